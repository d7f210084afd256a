# A/B timing of librk run-time switches on the c4 headline (scratch outputs in gpurun_out/).
# usage: AB="RK_X=0 RK_X=1" bash scripts/ab_bench.sh
mkdir -p gpurun_out
ARGS=${ARGS:-"--steps 10 --warmup 5 --no-cpu-baseline --no-secondary --no-e2e"}
for rep in 1 2; do
for v in $AB; do
  tag=$(echo $v | sed "s|.*/||; s|=|_|g")
  env $v timeout 600 python bench.py $ARGS > gpurun_out/ab_${tag}_${rep}.log 2>&1
  echo "$v rep$rep: $(grep '^{' gpurun_out/ab_${tag}_${rep}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], "mv", d["iterations"]["mean"], "frac", d["roofline"]["frac"], {k: (v["ms"], v["gbs"]) for k, v in list(d["kernel_breakdown"].items())[:4]})')"
done
done
