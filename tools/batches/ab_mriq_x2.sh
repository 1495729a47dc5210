# MRIQ FP32x2 (product) vs scalar (-DKL_MRIQ_SCALAR) build: GPU kernel tests, solo, C5 A/B
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/ab5_kernels.log 2>&1; echo rc=$? >> gpurun_out/ab5_kernels.log
SPIN=1 KINDS=MRIQ,SPMV timeout 300 python tools/launcher_overhead.py > gpurun_out/ab5_solo_x2.txt 2>&1
SPIN=1 KINDS=MRIQ,SPMV KL_LIB_PATH=variants/libkl_mriq_scalar.so timeout 300 python tools/launcher_overhead.py > gpurun_out/ab5_solo_scalar.txt 2>&1
for r in 1 2; do
for v in x2 scalar; do
  if [ $v = scalar ]; then L="KL_LIB_PATH=variants/libkl_mriq_scalar.so"; else L=""; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab5_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab5_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), 'mriq roof', round(d['roofline']['frac'],3))" >> gpurun_out/ab5_summary.txt
done; done
