# with the FP32x2 MRIQ: MRIQ's b_max 8 (hardware) vs 3 vs 2 on C5; MRIQ's solo cap sweep; a
# functional 2-rank run on one device (gloo)
SPIN=1 KINDS=MRIQ timeout 300 python - > gpurun_out/ab9_mriq_sweep.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, ".")
import torch, kl_inputs as G, paper_1303_5164_b200 as K
from paper_1303_5164_b200.workload import Instance
ctx = K.Context(device=0); i = Instance(G.gen("MRIQ", "paper"), "cuda")
for cap in range(1, 9):
    ctx.run_capped("MRIQ", i.grid, i.args, cap)
    print(cap, round(ctx.run_capped("MRIQ", i.grid, i.args, cap), 4), flush=True)
PY
for r in 1 2; do
for v in 8 3 2; do
  if [ $v = 8 ]; then P=""; else P="--prof MRIQ.bmax=$v"; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab9_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab9_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 mriq bmax $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab9_summary.txt
done; done
KL_BENCH_ONE_DEVICE=1 timeout 600 python bench.py --gpus 2 --backend gloo --size small --steps 2 --warmup 1 --no-baselines --no-cpu > gpurun_out/ab9_two_rank.log 2>&1; echo "two-rank rc $?" >> gpurun_out/ab9_summary.txt
