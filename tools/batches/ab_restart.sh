# engine experiment: restart the resident kernel so a newly launched partner holds the older warps
# (KL_RESTART_RESIDENT=1) -- scheduling tests under it, then C5 / C4-ALL A/B
KL_RESTART_RESIDENT=1 timeout 900 python -m pytest tests/test_gpu_sched.py tests/test_gpu_model.py -q -x > gpurun_out/ab14_tests.log 2>&1; echo rc=$? >> gpurun_out/ab14_tests.log
for r in 1 2; do
for v in base restart; do
  if [ $v = restart ]; then E="KL_RESTART_RESIDENT=1"; else E=""; fi
  env $E timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab14_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab14_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['engine_per_step'])" >> gpurun_out/ab14_summary.txt
  env $E timeout 300 python bench.py --workload c4 --mix ALL --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab14_c4_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab14_c4_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c4ALL $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab14_summary.txt
done; done
