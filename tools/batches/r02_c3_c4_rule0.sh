set -x
timeout 900 python tools/c3_mm_stream.py gpurun_out/r02_c3_mm_stream.json > gpurun_out/c3.log 2>&1
for m in CI MI MIX ALL; do timeout 600 python bench.py --workload c4 --mix $m --steps 3 --warmup 2 --no-cpu --json-out gpurun_out/r02_bench_c4_$m.json > gpurun_out/c4_$m.log 2>&1; done
timeout 900 python bench.py --split-rule 0 --steps 3 --warmup 2 --no-cpu --json-out gpurun_out/r02_bench_c5_rule0.json > gpurun_out/c5r0.log 2>&1
tail -3 gpurun_out/c3.log
