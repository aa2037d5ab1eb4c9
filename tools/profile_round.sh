#!/bin/bash
# One profiling pass (run under gpurun): plain bench lines, ncu launch lists of
# the same commands, and one ncu --set full capture of the kernels of one
# timed step.  Outputs land in gpurun_out/ and are summarised into profiles/.
set -x
R=${1:-r01}
B="python bench.py --steps 20 --warmup 5"
$B > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err
python bench.py --workload slab10M_tt --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_slab10M_tt.json 2>&1
python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_nversion01.json 2>&1
python bench.py --workload nversion_dx0.5_tt --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_nversion05.json 2>&1
# launch list of the default bench (timed region: skip preroll 500 x 3 + 200 stimulus + warmup)
C="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1"
$C > gpurun_out/${R}_plain_c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 1717 -c 64 --csv \
    --log-file gpurun_out/${R}_launches_slab20M_ms.csv $C > gpurun_out/${R}_ncu_launch.log 2>&1
# full capture: ionic + rhs + pcg of the first timed step (503 steps before)
D="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$D > gpurun_out/${R}_plain_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pcg_kernel|rhs_kernel|ionic_ms" -s 1509 -c 3 \
    -o gpurun_out/${R}_full_slab20M_ms $D > gpurun_out/${R}_ncu_full.log 2>&1
E="python bench.py --workload slab10M_tt --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$E > gpurun_out/${R}_plain_e.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pcg_kernel|rhs_kernel|ionic_tt" -s 1509 -c 3 \
    -o gpurun_out/${R}_full_slab10M_tt $E > gpurun_out/${R}_ncu_full_tt.log 2>&1
ls -la gpurun_out
