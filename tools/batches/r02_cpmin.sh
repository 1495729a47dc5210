for cp in 0 0.05 0.1; do
  timeout 600 python bench.py --workload c4 --mix MI --steps 3 --warmup 2 --no-cpu --cp-min $cp --json-out gpurun_out/cpmin_mi_$cp.json > /dev/null 2>&1
  timeout 600 python bench.py --workload c4 --mix CI --steps 3 --warmup 2 --no-cpu --no-baselines --cp-min $cp --json-out gpurun_out/cpmin_ci_$cp.json > /dev/null 2>&1
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu --no-baselines --cp-min $cp --json-out gpurun_out/cpmin_c5_$cp.json > /dev/null 2>&1
done
for f in gpurun_out/cpmin_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],2))"; done
