# A/B: b_max at the solo saturation occupancy, 1 % and 2 % tolerance, C5 and C2
S1="--prof MRIQ.bmax=3 --prof PC.bmax=4 --prof SAD.bmax=5 --prof SPMV.bmax=4 --prof ST.bmax=14 --prof BS.bmax=8 --prof TEA.bmax=12"
S2="--prof MRIQ.bmax=3 --prof PC.bmax=4 --prof SAD.bmax=5 --prof SPMV.bmax=4 --prof ST.bmax=14 --prof BS.bmax=8 --prof TEA.bmax=10"
for r in 1 2; do
for v in base sat1 sat2; do
  case $v in base) P="";; sat1) P="$S1";; sat2) P="$S2";; esac
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab3_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab3_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab3_summary.txt
done
for v in base sat1; do
  case $v in base) P="";; sat1) P="$S1";; esac
  timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab3c2_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab3c2_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c2 $v run $r', round(d['value'],1), round(d['ms_per_step'],2))" >> gpurun_out/ab3_summary.txt
done; done
