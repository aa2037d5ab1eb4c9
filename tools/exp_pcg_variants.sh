#!/bin/bash
# Grid-engine PCG inner-loop variants on the default workload:
# row-product slot batching (TCB_ROW_BATCH) x CTAs/SM of the direct variant
# (TCB_DIRECT_MINB -> register cap).  Libraries are built here (tools/var_*.so)
# and selected with TCB200_LIB; each prints one bench line.
cd "$(dirname "$0")/.."
build() {  # name, extra flags
  [ -f tools/var_$1.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
    $2 -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
    -o tools/var_$1.so -lgomp
}
VARS="b0m4:-DTCB_ROW_BATCH=0 b4m4:-DTCB_ROW_BATCH=4 b8m3:-DTCB_ROW_BATCH=8+-DTCB_DIRECT_MINB=3 b8m2:-DTCB_ROW_BATCH=8+-DTCB_DIRECT_MINB=2"
if [ "$1" == "build" ]; then
  for v in $VARS; do build ${v%%:*} "$(echo ${v#*:} | tr + ' ')" & done; wait; exit 0
fi
W=${W:-slab20M_ms}
for v in $VARS; do
  n=${v%%:*}
  echo "== $n"
  TCB200_LIB=tools/var_$n.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n', d['value'], d['ms_per_step'], r['pcg_ms_per_iter'], r['frac'], d['pcg_iters_per_step'])"
done
