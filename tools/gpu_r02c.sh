set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
E="python bench.py --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 0 --no-north-star"
for W in slab10M_tt slab10M_crn; do
  K=$([ $W == slab10M_tt ] && echo ionic_tt || echo ionic_crn)
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s 503 -c 1 -f -o gpurun_out/r02c_full_$W $E --workload $W > gpurun_out/r02c_ncu_$W.log 2>&1
done
bash tools/ncu_fp64.sh r02c
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "allocator or partition or peer or split" > gpurun_out/r02c_tests.log 2>&1
bash tools/sanitize_r02.sh
