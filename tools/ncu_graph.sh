# one g_S_kernel launch of the 20 M slab (variant 5) and the probe's stand-alone S phase
D="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --pcg-variant 5 --preroll 20"
$D > gpurun_out/r01e_plain_graph.log 2>&1
ncu --set full --clock-control none -k regex:"g_S_kernel" -s 60 -c 1 -o gpurun_out/r01e_full_graphS $D > gpurun_out/r01e_ncu_graphS.log 2>&1
ncu --set full --clock-control none -k regex:"sfull" -s 2 -c 2 -o gpurun_out/r01e_full_probeS tools/probe_bw.bin > gpurun_out/r01e_ncu_probeS.log 2>&1
