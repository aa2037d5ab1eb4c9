#!/bin/bash
# Persistent PCG grid size: CTAs per SM capped (TCB_CG_PER_SM_CAP) -> fewer
# participants in each grid barrier vs fewer warps streaming.
cd "$(dirname "$0")/.."
VARS="c4:-DTCB_CG_PER_SM_CAP=4 c2:-DTCB_CG_PER_SM_CAP=2 c1:-DTCB_CG_PER_SM_CAP=1"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    [ -f tools/cap_$n.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
      $f -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
      -o tools/cap_$n.so -lgomp & done; wait; exit 0
fi
for W in nversion_dx0.1_tt biv3M_tt slab10M_tt; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/cap_$n.so python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W $n', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done
done
