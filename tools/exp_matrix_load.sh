#!/bin/bash
# Matrix load policy of the grid-engine PCG: evict-first streaming (__ldcs,
# default) vs cached (__ldg) -- matters for systems whose matrix could stay
# in the 126 MB L2 (configs[2]).
cd "$(dirname "$0")/.."
VARS="ldcs:-DTCB_MATRIX_LOAD=0 ldg:-DTCB_MATRIX_LOAD=1"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    [ -f tools/ml_$n.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
      $f -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
      -o tools/ml_$n.so -lgomp & done; wait; exit 0
fi
for W in nversion_dx0.1_tt biv3M_tt slab10M_tt; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/ml_$n.so python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W $n', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'])"
done
done
