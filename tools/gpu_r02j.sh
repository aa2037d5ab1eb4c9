python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/exp_pipeline_r02.sh > gpurun_out/r02j_exp_pipeline.txt 2>&1
TCB_ION_RHS_CHUNKS=8 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_nversion.py -m gpu -q -x -k "multislice or trajectory or refinement or allocator or audit or ionic" > gpurun_out/r02j_pipeline_tests.log 2>&1
