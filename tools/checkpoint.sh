#!/bin/bash
# Refresh every measured artefact on the GPU box (run under gpurun from the repo root).
# Outputs land in gpurun_out/ (copied into profiles/ by hand after review).
# CALIB=1: recalibrate the profile and re-measure the OPT pair table; OPT=1: the OPT table only;
# EXTRA=1: also the slice report, C5 on one GPU, C3 with the streaming kernel, ncu range replay,
# compute-sanitizer.
set -u
mkdir -p gpurun_out
echo "== gpu tests"; timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
if [ "${CALIB:-0}" = "1" ]; then
  echo "== calibrate"; timeout 900 python tools/calibrate.py run gpurun_out/kl_profile_b200.json > gpurun_out/calib.log 2>&1
  grep -E " fit |wrote" gpurun_out/calib.log | cut -c1-160
  cp gpurun_out/kl_profile_b200.json profiles/kl_profile_b200.json
fi
if [ "${CALIB:-0}" = "1" ] || [ "${OPT:-0}" = "1" ]; then
  echo "== OPT pair table (measured co-runs)"; timeout 1200 python tools/opt_table.py gpurun_out/opt_table.json > gpurun_out/opt_table.log 2>&1
  cp gpurun_out/opt_table.json profiles/r01_opt_table.json
  python tools/pruning_study.py gpurun_out/pruning_b200.json > gpurun_out/pruning_b200.log 2>&1
fi
echo "== bench c2"; timeout 900 python bench.py --json-out gpurun_out/bench_c2.json > gpurun_out/bench_c2.log 2>&1
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_c2.json"))
print({k: d.get(k) for k in ("value", "ms_per_step", "device_ms_per_step", "speedup_vs_sequential",
                             "speedup_vs_multistream", "clocks", "lease_conflicts", "host_decide_ms_per_step",
                             "model_ms_per_step")})
print("e2e", d["e2e"]["value"], "roofline", d["roofline"])
PY
echo "== bench c2 rule 0"; timeout 600 python bench.py --no-cpu --split-rule 0 --json-out gpurun_out/bench_c2_rule0.json > gpurun_out/bench_c2_rule0.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_c2_rule0.json'));print(d['value'], d['ms_per_step'], d['speedup_vs_sequential'])"
echo "== bench OPT"; timeout 600 python bench.py --no-cpu --no-baselines --opt profiles/r01_opt_table.json --json-out gpurun_out/bench_opt.json > gpurun_out/bench_opt.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_opt.json'));print(d['value'], d['ms_per_step'], d['device_ms_per_step'])"
echo "== bench c4"; timeout 900 python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu --json-out gpurun_out/bench_c4.json > gpurun_out/bench_c4.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print(d['value'], d['ms_per_step'], d['speedup_vs_sequential'], d['lease_conflicts'])"
echo "== model error"; timeout 900 python tools/model_error.py gpurun_out/model_error.json > gpurun_out/model_error.log 2>&1
python -c "import json;print(json.load(open('gpurun_out/model_error.json'))['summary'])" | cut -c1-300
echo "== ncu launch list"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-baselines --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "== ncu full (the persistent slice-launcher variant the bench runs, second launch)"
for k in MRIQ MM ST PC BS TEA SAD SPMV; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 1 -c 1 -o gpurun_out/prof_$k python tools/prof_target.py $k sched > gpurun_out/ncu_full_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_model_batch -c 1 -o gpurun_out/prof_MODEL python tools/model_bench.py 1 > gpurun_out/ncu_full_MODEL.log 2>&1
python tools/model_bench.py 20 > gpurun_out/model_bench.json
python tools/ncu_summary.py gpurun_out/ncu_summary.json gpurun_out/prof_*.ncu-rep > /dev/null 2>&1
# keep the dominant kernel's and the model's reports; the rest are summarised (gpurun_out merge cap)
for k in MM ST PC BS TEA SAD SPMV; do rm -f gpurun_out/prof_$k.ncu-rep; done
echo "== MC(1000)"; timeout 900 python tools/mc_cdf.py 1000 gpurun_out/mc_cdf.json 2>&1 | tail -1 | cut -c1-400
echo "== online"; timeout 900 python tools/online.py 320 gpurun_out/online.json 2>&1 | tail -3 | cut -c1-600
echo "== f1 study"; timeout 600 python tools/model3_study.py gpurun_out/model3_study.json 2>&1 | tail -3
echo "== model bench"; python tools/model_bench.py 20
echo "== launcher overhead"; python tools/launcher_overhead.py > gpurun_out/launcher_overhead.txt 2>&1; cat gpurun_out/launcher_overhead.txt
if [ "${EXTRA:-0}" = "1" ]; then
  echo "== slice report"; timeout 600 python bench.py --no-cpu --no-baselines --steps 5 --trace-out gpurun_out/step_trace.jsonl --json-out gpurun_out/bench_trace.json > /dev/null 2>&1
  python tools/slice_report.py gpurun_out/step_trace.jsonl gpurun_out/slices.json > gpurun_out/slices.txt 2>&1; head -20 gpurun_out/slices.txt
  echo "== C5 on one GPU"; timeout 1200 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu --json-out gpurun_out/bench_c5.json > gpurun_out/bench_c5.log 2>&1
  python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'], d['ms_per_step'], d['speedup_vs_sequential'])"
  echo "== C3 with the streaming kernel"; KL_C3_SYNTH=1 timeout 1200 python tools/model_error.py gpurun_out/model_error_synth.json > gpurun_out/model_error_synth.log 2>&1
  echo "== ncu range replay"; bash tools/ncu_range.sh
  echo "== sanitizers"; bash tools/sanitize.sh
fi
echo "== done"; ls gpurun_out
