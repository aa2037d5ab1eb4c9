#!/bin/bash
# FP64 ionic kernel launch shapes: registers per
# thread (TCB_ION_MINB CTAs of 128 threads per SM) x grid-stride persistence.
cd "$(dirname "$0")/.."
VARS="p1m4:-DTCB_ION_MINB=4 p1m3:-DTCB_ION_MINB=3 p1m5:-DTCB_ION_MINB=5 p0m4:-DTCB_ION_MINB=4+-DTCB_ION_PERSIST=0"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    [ -f tools/ion_$n.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
      $f -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
      -o tools/ion_$n.so -lgomp & done; wait; exit 0
fi
for W in slab10M_tt slab10M_crn; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/ion_$n.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W $n', d['value'], d['ms_per_step'], 'ionic_ms', r['ionic_ms_per_step'])"
done
done
