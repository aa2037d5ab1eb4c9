E="python bench.py --workload slab10M_tt --steps 2 --warmup 3 --windows 1 --no-cpu-baseline --e2e-steps 0"
TCB200_LIB=tools/ion_persist.so $E > gpurun_out/r02x_plain.log 2>&1 && \
TCB200_LIB=tools/ion_persist.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:ionic_persist -s 503 -c 1 -f -o gpurun_out/r02x_full_persist $E > gpurun_out/r02x_ncu.log 2>&1
