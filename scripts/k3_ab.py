"""K3 quantizer and the bench step (K3 + mpGeMM) under env knobs (development tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
dev = torch.device("cuda")
M, K, N = 6912, 2560, 256
W = torch.from_numpy(synth.ternary_weights(M, K, 2000, 0.4)).to(dev)
pw = v.pack_weights_device(W, 4)
x = torch.from_numpy(synth.activations_f32(K, N, 2100)).to(dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev)
s = torch.empty((N,), device=dev)
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def graph_time(fn, n=12):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            flush.zero_()
            if fn: fn()
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    return float(np.median(ts))
base = graph_time(None)
k3 = graph_time(lambda: v.quantize(x, q=q, scale=s)) - base
step = graph_time(lambda: (v.quantize(x, q=q, scale=s), v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws))) - base
k1 = graph_time(lambda: v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws)) - base
print(f"QCL={os.environ.get('VLUT_QCL', 'auto')}: K3 {k3:6.2f} us  K1 {k1:6.2f} us  step {step:6.2f} us", flush=True)
