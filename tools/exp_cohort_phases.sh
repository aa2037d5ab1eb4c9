#!/bin/bash
# Per-phase device timing of the cluster engine (globaltimer, CTA 0 thread 0),
# from an experiment build of the library with -DTCB_COHORT_PHASES.
set -e
cd "$(dirname "$0")/.."
L=tools/libtcb200_phases.so
[ -f $L ] || /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
  -DTCB_COHORT_PHASES -Xcompiler -fPIC,-fopenmp,-O3 -shared paper_2510_12011_b200/csrc/*.cu \
  paper_2510_12011_b200/csrc/*.cpp -o $L -lgomp
for m in ms tt2006; do
  for e in cluster cluster_streaming; do
    TCB200_LIB=$L python tools/run_small.py --engine $e --model $m --pre 60 --steps 100
  done
done
