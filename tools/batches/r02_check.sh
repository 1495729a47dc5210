# full GPU suite, smoke, default bench (C5), ncu of MM plain (tensor pipe), MM solo probe
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/v13_gputest.log 2>&1; echo rc=$? >> gpurun_out/v13_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v13_smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --json-out gpurun_out/v13_bench.json > gpurun_out/v13_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_plain_pair --launch-skip 1 -c 1 -o gpurun_out/v13_mm_plain -f python tools/prof_target.py MM plain > gpurun_out/v13_ncu_mm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_persistent_pair --launch-skip 1 -c 1 -o gpurun_out/v13_mm_pers -f python tools/prof_target.py MM sched >> gpurun_out/v13_ncu_mm.log 2>&1
