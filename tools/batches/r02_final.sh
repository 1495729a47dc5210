# full GPU test suite, sanitizers over every kind, smoke, and the default bench line (C5) + C2
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash tools/sanitize.sh > gpurun_out/sanitize_summary.txt 2>&1; grep -E "==|SUMMARY|invalid" gpurun_out/sanitize_summary.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --gpus 1 --steps 10 --warmup 3 --json-out gpurun_out/r02_bench_c5_n1.json > gpurun_out/bench_c5.log 2>&1; echo "bench rc $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --json-out gpurun_out/r02_bench_c2.json > gpurun_out/bench_c2.log 2>&1; echo "c2 rc $?"
rm -f gpurun_out/sanitizer_*.log
