# round-2 ncu evidence: per-kind --set full (plain grid and the persistent variant the bench runs),
# the model batch, and the launch list of the default bench command (C5, one step, no warm-up).
# Only summaries travel back (gpurun_out/ is capped at 64 MiB): reports are summarised, then
# removed except MRIQ's and MM's.
mkdir -p gpurun_out
for k in MRIQ PC ST BS TEA SAD SPMV MM; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 1 -c 1 -o gpurun_out/r02prof_${k}_persistent python tools/prof_target.py $k sched > /dev/null 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_plain -s 1 -c 1 -o gpurun_out/r02prof_${k}_plain python tools/prof_target.py $k plain > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_model_batch -c 1 -o gpurun_out/r02prof_MODEL python tools/model_bench.py 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_summary.json gpurun_out/r02prof_*.ncu-rep > /dev/null 2>&1
ncu -i gpurun_out/r02prof_MM_plain.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_mm_plain_source.csv 2>/dev/null
for f in gpurun_out/r02prof_*.ncu-rep; do case $f in *MRIQ_persistent*|*MM_plain*) ;; *) rm -f $f;; esac; done
timeout 1300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-baselines --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc $?"; du -sh gpurun_out; ls -la gpurun_out | head -20
