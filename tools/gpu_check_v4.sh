python -m pytest tests -m gpu -x -q > gpurun_out/r01e_gputests_v4.log 2>&1; echo tests=$?
python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r01e_bench_nversion01.json 2>&1
python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline --pcg-variant 0 > gpurun_out/r01e_bench_nversion01_v0.json 2>&1
python bench.py --workload biv3M_tt --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r01e_bench_biv3M_tt.json 2>&1
