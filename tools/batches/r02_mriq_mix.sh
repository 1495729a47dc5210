# C5 with the MRIQ MUFU / FMA-polynomial mixes (KL_MRIQ_P of every 8 k-points on the FMA pipe):
# less MUFU in the MIO queue for MRIQ's partners
for v in base mriqp1 mriqp2; do
  KL_LIB_PATH=variants/libkl_$v.so timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-baselines --json-out gpurun_out/mix_$v.json > /dev/null 2>&1
  KINDS=MRIQ KL_LIB_PATH=variants/libkl_$v.so timeout 120 python tools/launcher_overhead.py 2>&1 | tail -1
  python -c "import json; d=json.load(open('gpurun_out/mix_$v.json')); print('$v', round(d['value'],1), round(d['ms_per_step'],1), d['parity']['MRIQ'])"
done
