python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "step_io or state_injection" > gpurun_out/r01e_gputests_io.log 2>&1; echo tests=$?
python bench.py > gpurun_out/r01e_bench_default_io.json 2> gpurun_out/r01e_bench_default_io.err; echo bench=$?
python bench.py --workload slab10M_tt --no-cpu-baseline > gpurun_out/r01e_bench_slab10M_tt_io.json 2>&1
