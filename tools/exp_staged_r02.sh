#!/bin/bash
# r02 PCG A/B at mid size: TMA-staged matrix (variant 1) with the batched gathers
# of variant 4 (TCB_STAGED_BATCH=1) vs variant 1 as is vs variant 4 / 0.
# Build here:  bash tools/exp_staged_r02.sh build ; run on the box: bash tools/exp_staged_r02.sh
cd "$(dirname "$0")/.."
if [ "$1" == "build" ]; then
  bash tools/build_variant.sh tools/sb_0.so -DTCB_STAGED_BATCH=0
  bash tools/build_variant.sh tools/sb_1.so -DTCB_STAGED_BATCH=1
  exit 0
fi
run() {  # lib workload variant steps
  TCB200_LIB=tools/$1.so python bench.py --workload $2 --pcg-variant $3 --steps $4 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$2 $1 v$3', round(d['value']/1e9,4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'it/step', d.get('pcg_iters_per_step'), 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  for W in nversion_dx0.1_tt:50 sphere655k_ms:50; do
    w=${W%%:*}; k=${W##*:}
    run sb_0 $w 4 $k; run sb_0 $w 1 $k; run sb_1 $w 1 $k
  done
  for W in biv3M_tt:20 sphere2.6M_ms:20 slab10M_tt:20; do
    w=${W%%:*}; k=${W##*:}
    run sb_0 $w 0 $k; run sb_0 $w 4 $k; run sb_1 $w 1 $k
  done
done
