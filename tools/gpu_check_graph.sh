python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "trajectory or pcg_parity or step_io" > gpurun_out/r01e_gputests_graph.log 2>&1; echo tests=$?
tools/exp_graph.sh > gpurun_out/r01e_exp_graph.txt 2>&1
