# complete ncu launch list of one step of the default bench command (C5, no warm-up)
timeout 2700 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-baselines --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc $?"; wc -l gpurun_out/r02_launches_c5.csv
