# MRIQ two voxels per thread (-DKL_MRIQ_V2: fetched chunks of 2 virtual blocks) vs the product:
# kernel parity through the variant, solo plain/persistent, C5 A/B
KL_LIB_PATH=variants/libkl_mriq_v2.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "mriq or sliced or MRIQ" > gpurun_out/ab11_kernels.log 2>&1; echo rc=$? >> gpurun_out/ab11_kernels.log
SPIN=1 KINDS=MRIQ timeout 300 python tools/launcher_overhead.py > gpurun_out/ab11_solo_prod.txt 2>&1
KL_LIB_PATH=variants/libkl_mriq_v2.so SPIN=1 KINDS=MRIQ timeout 300 python tools/launcher_overhead.py > gpurun_out/ab11_solo_v2.txt 2>&1
for r in 1 2; do
for v in prod v2; do
  if [ $v = prod ]; then L=""; else L="KL_LIB_PATH=variants/libkl_mriq_v2.so"; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab11_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab11_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['parity']['MRIQ'])" >> gpurun_out/ab11_summary.txt
done; done
