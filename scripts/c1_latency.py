import torch, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device('cuda')
W = synth.ternary_weights(256, 512, 1)
pw = v.pack_weights(W, 4, device=dev)
A = torch.randint(-127, 128, (512, 8), dtype=torch.int8, device=dev)
s = torch.rand(8, device=dev)
out = torch.empty((256, 8), device=dev)
ws = v.workspace(dev)
def t(fn, n=200):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n): fn()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * n)
print("auto", v.plan_ws(256, 512, 8, 4), t(lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, ws=ws)))
for S in (1, 2, 4, 8):
    for tpw in (1, 2):
        print("slot S", S, "tpw", tpw, t(lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=v.slot_plan(tpw=tpw, splits=S), ws=ws)))
for w in (8, 12, 16):
    for S in (1, 2):
        try:
            print("k1", w, S, t(lambda: v.mpgemm_ex(pw, A, s, 0.02, out=out, plan=v.LaunchPlan(w, S))))
        except Exception as e: print("k1", w, S, e)
print("k1 auto", v.plan(256,512,8,4), t(lambda: v.mpgemm(pw, A, s, 0.02, out=out)))
