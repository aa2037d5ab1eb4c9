python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k sphere > gpurun_out/r01e_gputests_sphere.log 2>&1; echo tests=$?
python bench.py --workload sphere655k_ms --steps 50 > gpurun_out/r01e_bench_sphere655k_ms.json 2>&1
python bench.py --workload sphere2.6M_ms --steps 20 --no-cpu-baseline > gpurun_out/r01e_bench_sphere2.6M_ms.json 2>&1
python bench.py --workload sphere655k_ms --steps 50 --no-cpu-baseline --pcg-variant 0 > gpurun_out/r01e_bench_sphere655k_ms_v0.json 2>&1
