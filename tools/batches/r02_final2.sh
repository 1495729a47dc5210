# final round-2 measurements after the MM decoupled loop: C5 headline (20 steps), C2, C4 per mix,
# launcher overhead (host launch hidden)
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 --json-out gpurun_out/f_bench_c5_n1.json > gpurun_out/f_bench_c5.log 2>&1; echo "c5 rc $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --json-out gpurun_out/f_bench_c2.json > gpurun_out/f_bench_c2.log 2>&1; echo "c2 rc $?"
for m in CI MI MIX ALL; do
  timeout 600 python bench.py --workload c4 --mix $m --steps 5 --warmup 3 --no-cpu --json-out gpurun_out/f_bench_c4_$m.json > gpurun_out/f_bench_c4_$m.log 2>&1; echo "c4 $m rc $?"
done
SPIN=1 timeout 600 python tools/launcher_overhead.py > gpurun_out/f_launcher_overhead.txt 2>&1; echo "overhead rc $?"
