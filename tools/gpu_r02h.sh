python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/exp_ionic_r02.sh > gpurun_out/r02h_exp_ionic.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_tests.log 2>&1
