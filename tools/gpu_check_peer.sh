python -m pytest tests -m gpu -x -q > gpurun_out/r01e_gputests_peer.log 2>&1; echo tests=$?
python tools/exp_peer_batch.py > gpurun_out/r01e_exp_peer_batch.txt 2>&1
python tools/exp_peer_batch.py 400,250,25 >> gpurun_out/r01e_exp_peer_batch.txt 2>&1
