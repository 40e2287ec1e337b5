"""Bench step variants on configs[1] (development tool): K3 + K1 (two
launches, PDL) vs vlut_quantize_mpgemm (one cooperative launch with the
quantizer as a grid-wide prologue).  L2 flushed outside each step's events."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
M, K, N, g = 6912, 2560, 256, 4
W = torch.from_numpy(synth.ternary_weights(M, K, 2000, 0.4)).to(dev)
pw = v.pack_weights_device(W, g)
x = torch.from_numpy(synth.activations_f32(K, N, 2001)).to(dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev)
s = torch.empty((N,), dtype=torch.float32, device=dev)
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
def two():
    v.quantize(x, q=q, scale=s, stream=st)
    v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)
def fused():
    v.quantize_mpgemm(pw, x, 0.02, q=q, scale=s, out=out, ws=ws, stream=st)
for name, fn in (("two_launches", two), ("fused", fused), ("two_launches", two), ("fused", fused)):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(200):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); fn(); b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print(f"{name:14s} step us mean {np.mean(ts):7.2f} med {np.median(ts):7.2f} min {np.min(ts):7.2f}")
