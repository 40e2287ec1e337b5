"""A/B timing of two builds of libvlut.so on the same shapes (development
tool): python scripts/ab_lib.py [path/to/libvlut.so].  CUDA graph of
back-to-back launches over weight copies > 2x L2."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
if len(sys.argv) > 1:
    v.lib_path = sys.argv[1]
from paper_2512_06443_b200 import synth

def bench(runs, reps=60):
    for r in runs[:2]:
        r()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in runs:
            r()
    g.replay(); torch.cuda.synchronize()
    per = max(2, reps // len(runs))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(per):
        g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (per * len(runs))

dev = torch.device("cuda")
R_LU = 148 * 64 * 1965e6
for (M, K, N, g, plan) in [(6912, 2560, 256, 4, (12, 2)), (6912, 2560, 256, 4, (8, 3)),
                           (3072, 23040, 256, 4, (12, 4)), (6912, 2560, 2048, 4, None),
                           (3840, 2560, 2048, 4, None), (3072, 23040, 1024, 5, (12, 4))]:
    W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = max(1, -(-260_000_000 // pw0.nbytes))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev)
    out = torch.empty((M, N), device=dev)
    lp = v.LaunchPlan(*plan) if plan else None
    mk = (lambda p_: (lambda: v.mpgemm_ex(p_, A, s, 0.02, out=out, plan=lp))) if lp else \
         (lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out)))
    t = bench([mk(p) for p in pws])
    lk = M * (K // g) * N
    pl = lp or v.plan_ws(M, K, N, g)
    print(f"M={M} K={K} N={N} g={g} plan=w{pl.warps} s{pl.splits} sk{pl.streamk}: {t:8.2f} us  frac {lk / R_LU / (t * 1e-6):.3f}", flush=True)
    del pws, pw0, W
    torch.cuda.empty_cache()
