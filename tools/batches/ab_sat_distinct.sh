# A/B: hardware b_max vs saturation b_max + distinct kinds (R31, R31b); C5 and C4 per mix
timeout 600 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/ab4_gpumodel.log 2>&1; echo rc=$? >> gpurun_out/ab4_gpumodel.log
for r in 1 2; do
for b in hw sat; do
  timeout 300 python bench.py --bmax $b --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab4_c5_${b}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab4_c5_${b}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $b run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab4_summary.txt
  for m in CI MI MIX ALL; do
    timeout 300 python bench.py --workload c4 --mix $m --bmax $b --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab4_c4${m}_${b}_$r.log 2>&1
    python -c "import json;l=[x for x in open('gpurun_out/ab4_c4${m}_${b}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c4 $m $b run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab4_summary.txt
  done
done; done
