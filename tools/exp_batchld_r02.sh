#!/bin/bash
# r02: latency variant's matrix load policy (TCB_BATCH_MATLOAD): 0 evict-first,
# 1 cached, 2 L2 evict-last (mid-size matrices fit the 126 MB L2).
cd "$(dirname "$0")/.."
VARS="m0:-DTCB_BATCH_MATLOAD=0 m1:-DTCB_BATCH_MATLOAD=1 m2:-DTCB_BATCH_MATLOAD=2"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    bash tools/build_variant.sh tools/bl_$n.so $f; done; exit 0
fi
for rep in 1 2 3; do
  for W in nversion_dx0.1_tt:50 sphere655k_ms:50; do
    w=${W%%:*}; k=${W##*:}
    for v in $VARS; do
      n=${v%%:*}
      TCB200_LIB=tools/bl_$n.so python bench.py --workload $w --steps $k --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$w $n', round(d['value']/1e9,4), 'ms', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'clk', d['clocks']['sm_mhz'])"
    done
  done
done
