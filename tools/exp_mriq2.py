import os, sys
sys.path.insert(0, os.getcwd())
import torch
import kl_inputs as G
import paper_1303_5164_b200 as K
from paper_1303_5164_b200.workload import Instance
ctx = K.Context(device=0)
d = G.gen("MRIQ", "paper")
a = Instance(d, "cuda"); b = Instance(d, "cuda", inputs=a.inputs)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); e1.synchronize(); return e0.elapsed_time(e1)
for rep in range(2):
    seq = t(lambda: (ctx.run_plain("MRIQ", a.grid, a.args, 0), ctx.run_plain("MRIQ", b.grid, b.args, 0)))
    def conc():
        ev = torch.cuda.Event(); ev.record()
        s1.wait_event(ev); s2.wait_event(ev)
        ctx.run_plain("MRIQ", a.grid, a.args, s1); ctx.run_plain("MRIQ", b.grid, b.args, s2)
        e1 = torch.cuda.Event(); e1.record(s1); torch.cuda.current_stream().wait_event(e1)
        e2 = torch.cuda.Event(); e2.record(s2); torch.cuda.current_stream().wait_event(e2)
    c = t(conc)
    solo = t(lambda: ctx.run_plain("MRIQ", a.grid, a.args, 0))
    print("solo", solo, "two sequential", seq, "two concurrent", c)
    for caps in [(2,6),(4,4),(8,0)]:
        r1, r2 = ctx.run_pair("MRIQ", a.grid, a.args, caps[0], "MRIQ", b.grid, b.args, caps[1] or 8)
        print(caps, "exec", r1.executed, r2.executed, "ms", (r1.t1_ns-r1.t0_ns)/1e6, (r2.t1_ns-r2.t0_ns)/1e6, "t0 diff us", (r2.t0_ns-r1.t0_ns)/1e3)
