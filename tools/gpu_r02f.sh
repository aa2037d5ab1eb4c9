bash tools/exp_ionic_r02.sh > gpurun_out/r02f_exp_ionic.txt 2>&1
timeout 900 python tools/exp_setup_parts.py 8 > gpurun_out/r02f_setup_parts.json 2>&1
E="python bench.py --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star"
for W in slab10M_tt slab10M_crn; do
  K=$([ $W == slab10M_tt ] && echo ionic_tt || echo ionic_crn)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 503 -c 1 -f -o gpurun_out/r02f_full_$W $E --workload $W > gpurun_out/r02f_ncu_$W.log 2>&1
done
