mkdir -p gpurun_out
for cfg in 5 0 1 5 1; do
RK_CHAIN_CFG=$cfg python bench.py --workload c3 --steps 5 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/c3_cfg${cfg}_$RANDOM.log 2>&1; echo cfg$cfg=$?
done
python - <<'P'
import json,glob
for f in sorted(glob.glob('gpurun_out/c3_cfg*.log')):
    for ln in open(f):
        if ln.startswith('{'):
            d=json.loads(ln); print(f, d['value'], d['iterations']['mean'], {k:(v['ms'],v['launches'],v['gbs']) for k,v in d['kernel_breakdown'].items()})
P
