# One GPU call: parity tests, smoke, bench (default args), ncu launch list + full capture.
# Outputs under gpurun_out/ (scratch); summaries are copied into profiles/ by hand.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 3000 gpurun_out/bench.log
if [ -n "$NCU" ]; then
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_N:-8000} --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-chain_kernel|stencil_kernel|bdot_kernel|bupd_kernel|bicg_}" -s 4000 -c ${NCU_C:-16} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
ls -la gpurun_out
