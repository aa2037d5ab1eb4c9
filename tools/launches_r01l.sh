#!/bin/bash
# ncu launch list of the default bench at HEAD (step kernels of the timed region; see profile_round.sh)
R=${1:-r01l}
C="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1"
STEPK='regex:pcg_kernel|rhs_kernel|ionic_|stimulus_kernel|lat_epilogue|gather_kernel|scatter_kernel'
timeout 600 $C > gpurun_out/${R}_plain_c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$STEPK" -s 1717 -c 61 --csv \
    --log-file gpurun_out/${R}_launches_slab20M_ms.csv $C > gpurun_out/${R}_ncu_launch.log 2>&1
echo launches=$?
