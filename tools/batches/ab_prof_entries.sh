# C5: the calibrated profile in use vs its MRIQ entry (and MM / SPMV entries) from the
# recalibration for the final kernels (profiles/kl_profile_b200_recal_r02.json)
for r in 1 2; do
for v in base mriq all; do
  case $v in base) P="";; mriq) P="--prof MRIQ.rm=0.0023391825723108827 --prof MRIQ.r=15.68911541746213 --prof MRIQ.ipb=119936.0 --prof MRIQ.ipc_max=0.4488409734168632 --prof MRIQ.pur=0.4389518234759327 --prof MRIQ.mur=0.0019739639659129044";; all) P="--prof MRIQ.rm=0.0023391825723108827 --prof MRIQ.r=15.68911541746213 --prof MRIQ.ipb=119936.0 --prof MRIQ.ipc_max=0.4488409734168632 --prof MRIQ.pur=0.4389518234759327 --prof MRIQ.mur=0.0019739639659129044 --prof MM.rm=0.0317181192844341 --prof MM.ipb=16799.06640625 --prof MM.pur=0.08033921198969646 --prof MM.mur=0.16878819324693284 --prof SPMV.rm=0.0370744752411292 --prof SPMV.ipb=143.0 --prof SPMV.pur=0.15460371379802565 --prof SPMV.mur=0.2119744176398089";; esac
  timeout 300 python bench.py --steps 5 --warmup 3 --no-baselines --no-cpu $P > gpurun_out/ab10_c5_${v}_$r.log 2>&1
  python -c "import json;l=[x for x in open('gpurun_out/ab10_c5_${v}_$r.log') if x.startswith('{')][-1];d=json.loads(l);print('c5 $v run $r', round(d['value'],1), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])" >> gpurun_out/ab10_summary.txt
done; done
