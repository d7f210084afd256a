# ncu evidence at the c4 headline: launch list (cold, serialised) + one --set full capture of
# chain19 / bdot_bulk / bupd_gram(_bulk) launches.  Each ncu pass runs only after the same
# command exited 0 without ncu.  Scratch outputs in gpurun_out/.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
$CMD > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_N:-14000} --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-chain19_kernel|bdot_bulk|bupd_gram}" -s ${NCU_S:-3000} -c ${NCU_C:-6} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out | tail -5
