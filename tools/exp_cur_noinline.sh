#!/bin/bash
# Instruction-cache experiment: the current evaluation (twice per step) inlined
# twice (default) vs one out-of-line copy (TCB_CUR_NOINLINE=1).
cd "$(dirname "$0")/.."
VARS="inl:-DTCB_CUR_NOINLINE=0 noinl:-DTCB_CUR_NOINLINE=1"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    [ -f tools/cur_$n.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
      $f -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
      -o tools/cur_$n.so -lgomp & done; wait; exit 0
fi
for W in slab10M_tt slab10M_crn; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/cur_$n.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W $n', d['value'], d['ms_per_step'], 'ionic_ms', r['ionic_ms_per_step'])"
done
done
