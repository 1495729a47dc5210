"""Record device facts (cudaDeviceProp) and host core count on the GPU box."""
import json, os, subprocess, torch
p = torch.cuda.get_device_properties(0)
d = {k: getattr(p, k) for k in dir(p) if not k.startswith('_') and isinstance(getattr(p, k), (int, float, str, bool))}
d['nproc'] = os.cpu_count()
try:
    d['lscpu'] = subprocess.run(['lscpu'], capture_output=True, text=True).stdout
except Exception as e:
    d['lscpu'] = str(e)
os.makedirs('gpurun_out', exist_ok=True)
json.dump(d, open('gpurun_out/devprobe.json', 'w'), indent=1, default=str)
print(json.dumps({k: v for k, v in d.items() if k != 'lscpu'}, default=str))
