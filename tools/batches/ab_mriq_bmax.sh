for r in 1 2; do
for v in 0 3 2; do
  if [ $v = 0 ]; then P=""; else P="--prof MRIQ.bmax=$v"; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab1_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab1_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('bmax=$v run $r', round(d['value'],1), round(d['ms_per_step'],1))" >> gpurun_out/ab1_summary.txt
done; done
