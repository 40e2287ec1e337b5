"""How much do the per-kernel events inside bench.py's step cost?  Times the
configs[1] step (flush outside, quantize + mpGeMM inside) with and without the
event between K3 and K1 (which blocks the programmatic-dependent-launch
overlap of K1's prologue with K3)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
if len(sys.argv) > 1:
    v.lib_path = sys.argv[1]
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
def step():
    v.quantize(x, q=q, scale=s, stream=st)
    v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)
for _ in range(20):
    step()
torch.cuda.synchronize()
for mode in ("inner_events", "outer_only", "no_flush_outer"):
    ts, k1 = [], []
    for i in range(100):
        if mode != "no_flush_outer":
            flush.zero_()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(st)
        v.quantize(x, q=q, scale=s, stream=st)
        if mode == "inner_events":
            e[1].record(st)
        v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)
        if mode == "inner_events":
            e[2].record(st)
        e[3].record(st)
        torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[3]))
        if mode == "inner_events":
            k1.append(e[1].elapsed_time(e[2]))
    print(mode, "step us mean %.2f med %.2f" % (np.mean(ts) * 1e3, np.median(ts) * 1e3),
          ("k1 us %.2f" % (np.mean(k1) * 1e3)) if k1 else "")

# K3 alone and K1 alone, each right after a flush
for name, fn in (("k3_only", lambda: v.quantize(x, q=q, scale=s, stream=st)),
                 ("k1_only", lambda: v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)),
                 ("k3_noflush", None)):
    ts = []
    for i in range(100):
        if fn is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        (fn or (lambda: v.quantize(x, q=q, scale=s, stream=st)))()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "us mean %.2f med %.2f" % (np.mean(ts) * 1e3, np.median(ts) * 1e3))

