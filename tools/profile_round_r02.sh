#!/bin/bash
# One profiling pass (run under gpurun): plain bench lines, ncu launch lists of
# the same commands, and ncu --set full captures of the kernels of one timed
# step.  Outputs land in gpurun_out/ and are summarised into profiles/.
set -x
R=${1:-r02}
B="python bench.py --steps 20 --warmup 5"
{ time $B > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err ; } 2> gpurun_out/${R}_default_time.txt
for W in slab10M_tt slab10M_crn biv3M_tt; do
  python bench.py --workload $W --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_$W.json 2>&1
done
python bench.py --workload nversion_dx0.1_tt --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_nversion01.json 2>&1
python bench.py --workload nversion_dx0.5_tt --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_nversion05.json 2>&1
python bench.py --workload cohort100_nversion05_tt --steps 50 --warmup 5 > gpurun_out/${R}_bench_cohort.json 2>&1
python bench.py --workload sphere655k_ms --steps 50 --warmup 5 > gpurun_out/${R}_bench_sphere655k_ms.json 2>&1
python bench.py --workload sphere2.6M_ms --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${R}_bench_sphere2.6M_ms.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_reference.json 2>&1
# launch list of the default bench: step kernels only (setup kernels excluded by name);
# timed region = after the preroll (500 x 3 + 200 stimulus + 1 epilogue) and warmup (5 x 3 + 1)
C="python bench.py --steps 20 --warmup 5 --windows 1 --no-north-star --no-cpu-baseline --e2e-steps 1"
STEPK='regex:pcg_kernel|rhs_kernel|ionic_|stimulus_kernel|lat_epilogue|gather_kernel|scatter_kernel'
$C > gpurun_out/${R}_plain_c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$STEPK" -s 1717 -c 61 --csv \
    --log-file gpurun_out/${R}_launches_slab20M_ms.csv $C > gpurun_out/${R}_ncu_launch.log 2>&1
# full capture: ionic + rhs + pcg of the first timed step (503 steps before)
D="python bench.py --steps 2 --warmup 3 --windows 1 --no-north-star --no-cpu-baseline --e2e-steps 1"
$D > gpurun_out/${R}_plain_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pcg_kernel|rhs_kernel|ionic_ms" -s 1509 -c 3 \
    -o gpurun_out/${R}_full_slab20M_ms $D > gpurun_out/${R}_ncu_full.log 2>&1
for W in slab10M_tt slab10M_crn; do
  E="python bench.py --workload $W --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 1"
  $E > gpurun_out/${R}_plain_$W.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"pcg_kernel|rhs_kernel|ionic_" -s 1509 -c 3 \
      -o gpurun_out/${R}_full_$W $E > gpurun_out/${R}_ncu_full_$W.log 2>&1
done
# configs[2]: ionic + pcg of the first timed step (latency variant 4 under the automatic
# choice, RHS fused into the PCG kernel: two launches per step, 503 steps before)
E="python bench.py --workload nversion_dx0.1_tt --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 1"
$E > gpurun_out/${R}_plain_nversion01.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pcg_kernel|rhs_kernel|ionic_" -s 1006 -c 2 \
    -o gpurun_out/${R}_full_nversion01 $E > gpurun_out/${R}_ncu_full_nversion01.log 2>&1
# the N>1 leg at world size 1 (torchrun, peer-memory PCG with an NCCL communicator of 1)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 --dist > gpurun_out/${R}_bench_dist_world1.json \
    2> gpurun_out/${R}_bench_dist_world1.err
# FP64 instruction counts of the ionic kernels (bench.py's ionic_roofline)
bash tools/ncu_fp64.sh ${R}
# cluster engine: one launch of 20 steps of configs[0]
python tools/run_small.py > gpurun_out/${R}_plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cohort -s 1 -c 1 \
    -o gpurun_out/${R}_full_cluster_c1 python tools/run_small.py > gpurun_out/${R}_ncu_cluster.log 2>&1
ls -la gpurun_out
# weak-scaling leg at world size 1 (2.5 M nodes per GPU)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29518 bench.py --gpus 1 --steps 20 --warmup 5 --dist --weak > gpurun_out/${R}_bench_dist_weak_world1.json \
    2> gpurun_out/${R}_bench_dist_weak_world1.err
# wall time of the default run (what the driver runs)
/usr/bin/env bash -c "time python bench.py --no-north-star > /dev/null 2>&1" 2> gpurun_out/${R}_default_no_ns_time.txt
