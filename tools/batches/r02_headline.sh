# the round-2 headline line (C5, 20 steps) with the final bench, and one step's launch trace for
# the per co-scheduled slice report
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 --json-out gpurun_out/h_bench_c5_n1.json > gpurun_out/h_bench_c5.log 2>&1; echo "c5 rc $?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-baselines --no-cpu --trace-out gpurun_out/h_c5_trace.jsonl > gpurun_out/h_trace.log 2>&1; echo "trace rc $?"
