bash tools/exp_ionic_r02.sh > gpurun_out/r02l_exp_ionic.txt 2>&1
TCB200_LIB=tools/ion_all3.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_cohort.py -m gpu -q -x -k "ionic or trajectory or multislice or blow or cohort_parity" > gpurun_out/r02l_all3_tests.log 2>&1
