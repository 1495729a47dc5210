# recalibrate every kind's profile for the current kernels (MM decoupled loop, MRIQ FP32x2, SPMV
# batched loads), then A/B the C5 queue: old profile vs new profile
timeout 2400 python tools/calibrate.py run gpurun_out/kl_profile_b200_new.json > gpurun_out/recal.log 2>&1; echo "calib rc $?" >> gpurun_out/recal.log
python - <<'PY'
import json
old = json.load(open("profiles/kl_profile_b200.json")); new = json.load(open("gpurun_out/kl_profile_b200_new.json"))
for k in ("cp_min", "level_mode"):
    new["config"][k] = old["config"][k]
new["config_notes"] = old.get("config_notes", {})
json.dump(new, open("gpurun_out/kl_profile_b200_new.json", "w"), indent=1)
PY
python tools/calibrate.py sat gpurun_out/kl_profile_b200_new.json >> gpurun_out/recal.log 2>&1
for r in 1 2; do
for v in old new; do
  if [ $v = new ]; then P="--profile gpurun_out/kl_profile_b200_new.json"; else P=""; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab6_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab6_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab6_summary.txt
done; done
