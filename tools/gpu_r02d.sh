python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r02d_tests.log 2>&1
bash tools/exp_ionic_r02.sh > gpurun_out/r02d_exp_ionic.txt 2>&1
timeout 900 python tools/exp_overlap_r02.py > gpurun_out/r02d_exp_overlap.txt 2>&1
timeout 600 python tools/nversion_table3.py gpurun_out/r02d_nversion_table3.json > /dev/null 2> gpurun_out/r02d_nversion.err
