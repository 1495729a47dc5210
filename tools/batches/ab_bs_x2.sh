# BS + ST FP32x2 (product) vs scalar (-DKL_BS_SCALAR -DKL_ST_SCALAR): GPU kernel tests, solo, C5 and C4-ALL A/B
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/ab7_kernels.log 2>&1; echo rc=$? >> gpurun_out/ab7_kernels.log
SPIN=1 KINDS=BS,ST timeout 300 python tools/launcher_overhead.py > gpurun_out/ab7_solo_x2.txt 2>&1
SPIN=1 KINDS=BS,ST KL_LIB_PATH=variants/libkl_bs_scalar.so timeout 300 python tools/launcher_overhead.py > gpurun_out/ab7_solo_scalar.txt 2>&1
for r in 1 2; do
for v in x2 scalar; do
  if [ $v = scalar ]; then L="KL_LIB_PATH=variants/libkl_bs_scalar.so"; else L=""; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab7_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab7_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab7_summary.txt
  env $L timeout 300 python bench.py --workload c4 --mix ALL --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab7_c4_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab7_c4_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c4ALL $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab7_summary.txt
done; done
