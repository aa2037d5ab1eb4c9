#!/bin/bash
# r02: variant 2 (16-bit column offsets) with the per-slot bases broadcast by a
# shuffle (TCB_COMP_SHFL=1) vs variant 2 as is vs variant 0.
cd "$(dirname "$0")/.."
if [ "$1" == "build" ]; then
  bash tools/build_variant.sh tools/cs_0.so -DTCB_COMP_SHFL=0
  bash tools/build_variant.sh tools/cs_1.so -DTCB_COMP_SHFL=1
  exit 0
fi
run() {  # lib workload variant steps
  TCB200_LIB=tools/$1.so python bench.py --workload $2 --pcg-variant $3 --steps $4 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$2 $1 v$3', round(d['value']/1e9,4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'pcg_ms_it', round(r['pcg_ms_per_iter'],4), 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  for W in slab10M_tt slab20M_ms; do
    run cs_0 $W 0 20; run cs_0 $W 2 20; run cs_1 $W 2 20
  done
done
