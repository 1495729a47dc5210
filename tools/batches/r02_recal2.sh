# recalibration for the final kernels (MM decoupled, MRIQ + BS FP32x2, SPMV batches): model error
# with it, and C5 A/B against the profile in use
timeout 2400 python tools/calibrate.py run gpurun_out/kl_profile_b200_final.json > gpurun_out/recal2.log 2>&1; echo "calib rc $?" >> gpurun_out/recal2.log
python - <<'PY'
import json
old = json.load(open("profiles/kl_profile_b200.json")); new = json.load(open("gpurun_out/kl_profile_b200_final.json"))
for k in ("cp_min", "level_mode"):
    new["config"][k] = old["config"][k]
new["config_notes"] = old.get("config_notes", {})
json.dump(new, open("gpurun_out/kl_profile_b200_final.json", "w"), indent=1)
PY
python tools/calibrate.py sat gpurun_out/kl_profile_b200_final.json >> gpurun_out/recal2.log 2>&1
KL_PROFILE=gpurun_out/kl_profile_b200_final.json timeout 1500 python tools/model_error.py gpurun_out/f3_model_error_final.json > gpurun_out/f3_me.log 2>&1; echo "me rc $?"
for r in 1 2; do
for v in inuse final; do
  if [ $v = final ]; then P="--profile gpurun_out/kl_profile_b200_final.json"; else P=""; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab12_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab12_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab12_summary.txt
done; done
