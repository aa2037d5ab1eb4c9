#!/bin/bash
# r02: merged x updates in the peer-memory PCG kernel (TCB_PEER_XMERGE) -- emulated
# partitions on one GPU and the torchrun world-1 leg (peer kernel + NCCL communicator of 1).
cd "$(dirname "$0")/.."
if [ "$1" == "build" ]; then
  bash tools/build_variant.sh tools/pm_0.so -DTCB_PEER_XMERGE=0
  bash tools/build_variant.sh tools/pm_1.so -DTCB_PEER_XMERGE=1
  exit 0
fi
for rep in 1 2; do
for n in pm_0 pm_1; do
  for P in 2 4; do
    TCB200_LIB=tools/$n.so python bench.py --workload slab20M_ms --partitions $P --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('slab20M_ms parts $P $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
  done
  TCB200_LIB=tools/$n.so timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus 1 --steps 20 --warmup 5 --dist --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('dist world1 $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
done
done
