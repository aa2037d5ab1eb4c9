python -m pytest tests -m gpu -x -q > gpurun_out/r01e_gputests_final.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01e_smoke_final.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/r01e_bench_default_final.json 2> gpurun_out/r01e_bench_default_final.err; echo bench=$?
python bench.py --workload nversion_dx0.1_tt --steps 50 --no-cpu-baseline > gpurun_out/r01e_bench_nversion01_final.json 2>&1
