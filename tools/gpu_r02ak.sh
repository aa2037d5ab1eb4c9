mkdir -p gpurun_out
for rep in 1 2; do for W in slab10M_tt slab20M_ms; do for n in par0 par1; do
  TCB200_LIB=tools/un_$n.so python bench.py --workload $W --steps 20 --warmup 5 --windows 1 --no-cpu-baseline --e2e-steps 0 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$W $n', round(d['value']/1e9,4), 'frac', round(r['frac'],3), 'pcg_ms_it', round(r['pcg_ms_per_iter'],4), 'clk', d['clocks']['sm_mhz'])"
done; done; done > gpurun_out/r02ak_exp_parity.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02ak_gputests.log 2>&1
tail -2 gpurun_out/r02ak_gputests.log; cat gpurun_out/r02ak_exp_parity.txt
