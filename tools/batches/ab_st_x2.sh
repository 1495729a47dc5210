# ST FP32x2 vs scalar (BS FP32x2 in all): solo (persistent spills at 32 registers), C5 A/B
for v in prod st_scalar st_minb12; do
  if [ $v = prod ]; then L=""; else L="KL_LIB_PATH=variants/libkl_$v.so"; fi
  env $L SPIN=1 KINDS=ST timeout 300 python tools/launcher_overhead.py > gpurun_out/ab8_solo_$v.txt 2>&1
done
for r in 1 2; do
for v in prod st_scalar st_minb12; do
  if [ $v = prod ]; then L=""; else L="KL_LIB_PATH=variants/libkl_$v.so"; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu > gpurun_out/ab8_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab8_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab8_summary.txt
done; done
