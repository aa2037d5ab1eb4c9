python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variant or pcg_parity or trajectory" > gpurun_out/r01e_v3_tests.log 2>&1; echo tests=$?
for W in nversion_dx0.1_tt biv3M_tt; do for V in 0 3; do
python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 1 --pcg-variant $V | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$W v$V', d['value'], d['ms_per_step'], 'pcg_ms_it', r['pcg_ms_per_iter'], 'frac', r['frac'], 'iters', d['pcg_iters_per_step'], 'ion', r['ionic_ms_per_step'])"
done; done > gpurun_out/r01e_exp_v3.txt 2>&1
