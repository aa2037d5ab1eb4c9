#!/bin/bash
# Round-end verification at HEAD (run under gpurun): GPU tests, smoke, bench lines.
R=${1:-r01h}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err; echo bench=$?
timeout 300 python bench.py --workload cohort100_nversion05_tt --steps 50 --warmup 5 > gpurun_out/${R}_bench_cohort.json 2>&1; echo cohort=$?
timeout 300 python bench.py --workload nversion_dx0.5_tt --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_nversion05.json 2>&1; echo nv05=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${R}_bench_reference.json 2>&1; echo ref=$?
