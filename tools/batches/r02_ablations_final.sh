# ablations on the final build: Eq.8 balanced ratio (split rule 0), C2's four occupancy levels,
# and the default, C5, 5 steps each (one box)
for v in base rule0 four; do
  case $v in base) P="";; rule0) P="--split-rule 0";; four) P="--levels four";; esac
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/abl_${v}.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/abl_${v}.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/abl_summary.txt
done
