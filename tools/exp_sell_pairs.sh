#!/bin/bash
# Slot-pair SELL layout (16-byte value / 8-byte index loads, TCB_SELL_PAIRS) and
# 16-byte row-pair streaming in the U phase (TCB_VEC_U), each on and off.
cd "$(dirname "$0")/.."
VARS="${VARS:-base:-DTCB_SELL_PAIRS=0+-DTCB_VEC_U=0 pairs:-DTCB_SELL_PAIRS=1+-DTCB_VEC_U=0 vecu:-DTCB_SELL_PAIRS=0+-DTCB_VEC_U=1 both:-DTCB_SELL_PAIRS=1+-DTCB_VEC_U=1}"
if [ "$1" == "build" ]; then
  for v in $VARS; do n=${v%%:*}; f=$(echo ${v#*:} | tr + ' ')
    [ -f tools/sp_$n.so ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
      $f -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp \
      -o tools/sp_$n.so -lgomp & done; wait; exit 0
fi
for W in ${WORKLOADS:-slab20M_ms slab10M_tt biv3M_tt nversion_dx0.1_tt}; do
for v in $VARS; do
  n=${v%%:*}
  TCB200_LIB=tools/sp_$n.so python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W $n', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'], 'iters', d['pcg_iters_per_step'])"
done
done
