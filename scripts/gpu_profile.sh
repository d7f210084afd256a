# ncu evidence for profiles/: launch list (cold, serialised) + one full capture of the top kernels
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stencil_kernel|bdot_kernel|bupd_kernel|bicg_" -s 4000 -c 14 -o gpurun_out/prof ${CMD} > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out
