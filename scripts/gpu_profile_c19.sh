# chain19 detail capture at the c4 headline, exported to text on the box (the
# .ncu-rep itself can exceed gpurun's 64 MiB copy-back): details page, raw
# metrics and the per-source-line stall samples of 2 launches.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
$CMD > gpurun_out/plain.log 2>&1; echo plain=$?
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-chain19_kernel}" -s ${NCU_S:-3000} -c ${NCU_C:-2} -o /tmp/c19prof $CMD > gpurun_out/ncu_c19.log 2>&1; echo ncu=$?
ncu -i /tmp/c19prof.ncu-rep --page details --csv > gpurun_out/c19_details.csv 2>&1
ncu -i /tmp/c19prof.ncu-rep --page raw --csv > gpurun_out/c19_raw.csv 2>&1
ncu -i /tmp/c19prof.ncu-rep --page source --csv --print-source sass > gpurun_out/c19_sass.csv 2>&1
gzip -f gpurun_out/c19_*.csv
ls -la gpurun_out
