# end-of-round-2 artefacts with the final kernels (MM decoupled loop, MRIQ / BS FP32x2, SPMV
# batches): GPU tests, smoke, ncu --set full of every kind (plain + persistent) and the model
# batch, C5 headline (20 steps), C2, C4 per mix, launcher overhead, the C5 launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/z_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/z_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1
for k in MRIQ PC ST BS TEA SAD SPMV MM; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_persistent -s 1 -c 1 -o gpurun_out/r02prof_${k}_persistent python tools/prof_target.py $k sched > /dev/null 2>&1
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_plain -s 1 -c 1 -o gpurun_out/r02prof_${k}_plain python tools/prof_target.py $k plain > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_model_batch -c 1 -o gpurun_out/r02prof_MODEL python tools/model_bench.py 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/z_ncu_summary.json gpurun_out/r02prof_*.ncu-rep > /dev/null 2>&1
for f in gpurun_out/r02prof_*.ncu-rep; do case $f in *MRIQ_persistent*|*MM_plain*) ;; *) rm -f $f;; esac; done
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 --json-out gpurun_out/z_bench_c5_n1.json > gpurun_out/z_bench_c5.log 2>&1; echo "c5 rc $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --json-out gpurun_out/z_bench_c2.json > gpurun_out/z_bench_c2.log 2>&1; echo "c2 rc $?"
for m in CI MI MIX ALL; do
  timeout 600 python bench.py --workload c4 --mix $m --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/z_bench_c4_$m.json > gpurun_out/z_bench_c4_$m.log 2>&1; echo "c4 $m rc $?"
done
SPIN=1 timeout 600 python tools/launcher_overhead.py > gpurun_out/z_launcher_overhead.txt 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-baselines --no-cpu > gpurun_out/z_ncu_bench.log 2>&1
echo "launch list rc $?"; du -sh gpurun_out
