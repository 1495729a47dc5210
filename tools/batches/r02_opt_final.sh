# f2 OPT comparator with the final kernels: measured pair table (paper size), C5 decided from it,
# and the steady-state model error
timeout 1500 python tools/opt_table.py gpurun_out/o_opt_table.json > gpurun_out/o_opt_table.log 2>&1; echo "opt rc $?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu --opt gpurun_out/o_opt_table.json --json-out gpurun_out/o_bench_opt.json > gpurun_out/o_bench_opt.log 2>&1; echo "bench opt rc $?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu --json-out gpurun_out/o_bench_model.json > gpurun_out/o_bench_model.log 2>&1; echo "bench model rc $?"
KL_STEADY=1 timeout 1800 python tools/model_error.py gpurun_out/o_model_error_steady.json > gpurun_out/o_me_steady.log 2>&1; echo "me steady rc $?"
