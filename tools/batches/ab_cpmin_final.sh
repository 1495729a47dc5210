# R25 co-run threshold cp_min re-checked with the recalibrated profile: C5 and C4-MI
for r in 1 2; do
for c in 0.05 0.1 0.15 0.2; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu --cp-min $c > gpurun_out/ab13_c5_${c}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab13_c5_${c}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 cp_min $c run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab13_summary.txt
  timeout 300 python bench.py --workload c4 --mix MI --steps 5 --warmup 3 --no-baselines --no-cpu --cp-min $c > gpurun_out/ab13_mi_${c}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab13_mi_${c}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c4MI cp_min $c run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab13_summary.txt
done; done
