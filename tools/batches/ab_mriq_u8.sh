# MRIQ FP32x2 loop unrolled 8 pairs (-DKL_MRIQ_U=8) vs 4 (product): solo and C5
SPIN=1 KINDS=MRIQ timeout 300 python tools/launcher_overhead.py > gpurun_out/ab16_solo_u4.txt 2>&1
KL_LIB_PATH=variants/libkl_u8.so SPIN=1 KINDS=MRIQ timeout 300 python tools/launcher_overhead.py > gpurun_out/ab16_solo_u8.txt 2>&1
for r in 1 2; do
for v in u4 u8; do
  if [ $v = u8 ]; then L="KL_LIB_PATH=variants/libkl_u8.so"; else L=""; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab16_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab16_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab16_summary.txt
done; done
