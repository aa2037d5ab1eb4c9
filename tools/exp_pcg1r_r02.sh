#!/bin/bash
# r02: single-reduction PCG (variant 6) vs Algorithm 1's kernels (variant 4 / 0), in-tree library.
cd "$(dirname "$0")/.."
run() {  # workload variant steps
  python bench.py --workload $1 --pcg-variant $2 --steps $3 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1 v$2', round(d['value']/1e9,4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(r['frac'],3), 'it/step', d.get('pcg_iters_per_step'), 'clk', d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  for W in nversion_dx0.1_tt:50 sphere655k_ms:50 nversion_dx0.5_tt:200; do
    w=${W%%:*}; k=${W##*:}; run $w 4 $k; run $w 6 $k
  done
  for W in biv3M_tt:20 slab10M_tt:20; do
    w=${W%%:*}; k=${W##*:}; run $w 0 $k; run $w 4 $k; run $w 6 $k
  done
done
