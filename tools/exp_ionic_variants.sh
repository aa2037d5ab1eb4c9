#!/bin/bash
# FP64 ionic kernels: CTA size sweep (TCB_ION_THREADS), one node per thread.
# (An earlier sweep of grid-stride / register-capped shapes measured slower;
# DESIGN.md "Ionic kernel".)  Libraries are built here (tools/ion_*.so) and
# selected with TCB200_LIB.
cd "$(dirname "$0")/.."
VARS="t128:-DTCB_ION_THREADS=128 t256:-DTCB_ION_THREADS=256 t64:-DTCB_ION_THREADS=64"
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
