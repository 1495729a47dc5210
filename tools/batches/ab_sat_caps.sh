# A/B: kinds' b_max limited to their solo saturation occupancy (cap_sweep_ms within 1 % of best)
for r in 1 2; do
for v in base m3 sat; do
  case $v in base) P="";; m3) P="--prof MRIQ.bmax=3";; sat) P="--prof MRIQ.bmax=3 --prof PC.bmax=4 --prof SAD.bmax=5 --prof TEA.bmax=12 --prof BS.bmax=8";; esac
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab2_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab2_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('$v run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab2_summary.txt
done; done
