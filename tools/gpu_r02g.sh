python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/exp_zform_r02.sh > gpurun_out/r02g_exp_zform.txt 2>&1
TCB200_LIB=tools/pcg_zform.so timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -k "multislice or pcg_parity or trajectory" > gpurun_out/r02g_zform_tests.log 2>&1
timeout 900 python tools/exp_setup_parts.py 8 > gpurun_out/r02g_setup_parts.json 2>&1
