# final artefacts with the recalibrated default profile: GPU tests, smoke, C5 headline (20 steps),
# C2, C4 per mix, one step's trace
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/y_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/y_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 --json-out gpurun_out/y_bench_c5_n1.json > gpurun_out/y_bench_c5.log 2>&1; echo "c5 rc $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --json-out gpurun_out/y_bench_c2.json > gpurun_out/y_bench_c2.log 2>&1; echo "c2 rc $?"
for m in CI MI MIX ALL; do
  timeout 600 python bench.py --workload c4 --mix $m --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/y_bench_c4_$m.json > gpurun_out/y_bench_c4_$m.log 2>&1; echo "c4 $m rc $?"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu --trace-out gpurun_out/y_c5_trace.jsonl > gpurun_out/y_trace.log 2>&1; echo "trace rc $?"
