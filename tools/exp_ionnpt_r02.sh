#!/bin/bash
# r02: TT2006 ionic kernel with k nodes per thread (TCB_ION_NPT), optionally with
# an L2 prefetch of the later nodes (TCB_ION_NPT_PF).
cd "$(dirname "$0")/.."
VARS="npt1:-DTCB_ION_NPT=1 npt2:-DTCB_ION_NPT=2 npt2pf:-DTCB_ION_NPT=2+-DTCB_ION_NPT_PF=1 npt4:-DTCB_ION_NPT=4"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/in_$n.so $f; done; exit 0
fi
for rep in 1 2 3; do
  for v in $VARS; do
    n=${v%%:*}
    TCB200_LIB=tools/in_$n.so python bench.py --workload slab10M_tt --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('slab10M_tt $n', round(d['value']/1e9,4), 'ionic_ms', round(r['ionic_ms_per_step'],4), 'clk', d['clocks']['sm_mhz'], 'cyc_k', round(r['ionic_ms_per_step']*d['clocks']['sm_mhz'],1))"
  done
done
