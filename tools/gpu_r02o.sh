bash tools/exp_xmerge_r02.sh > gpurun_out/r02o_exp_xmerge.txt 2>&1
TCB200_LIB=tools/pcg_xm.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "pcg_parity or trajectory or multislice" > gpurun_out/r02o_xm_tests.log 2>&1
