#!/bin/bash
# r02: peer kernel synchronisation -- arrive-only halo pushes (TCB_PEER_PUSH_ARRIVE)
# and 512- vs 256-thread CTAs (TCB_PEER_THREADS; half the barrier participants).
cd "$(dirname "$0")/.."
VARS="old:-DTCB_PEER_PUSH_ARRIVE=0 arr:-DTCB_PEER_PUSH_ARRIVE=1 old512:-DTCB_PEER_PUSH_ARRIVE=0+-DTCB_PEER_THREADS=512 arr512:-DTCB_PEER_PUSH_ARRIVE=1+-DTCB_PEER_THREADS=512"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/ps_$n.so $f; done; exit 0
fi
for rep in 1 2; do
for v in $VARS; do
  n=${v%%:*}
  for P in 2 4; do
    TCB200_LIB=tools/ps_$n.so python bench.py --workload slab20M_ms --partitions $P --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('slab20M_ms parts $P $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
  done
  TCB200_LIB=tools/ps_$n.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 --dist --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('dist world1 $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
done
done
