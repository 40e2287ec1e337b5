"""Compare plans under three timing methods (development tool):
(a) one launch per 256 MB L2 flush, events around it; (b) a CUDA graph of
back-to-back launches over weight copies > 2x L2; (c) events around each
launch, no flush.  python scripts/timing_methods.py M K N g plan[;plan...]
with plan = warps,splits,n_cta[,streamk,m_cta]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
R_LU = 148 * 64 * 1965e6
M, K, N, g = (int(x) for x in sys.argv[1:5])
plans = []
for t in sys.argv[5].split(";"):
    f = [int(x) for x in t.split(",")]
    plans.append(v.LaunchPlan(f[0], f[1], n_cta=f[2], streamk=f[3] if len(f) > 3 else 0,
                              m_cta=f[4] if len(f) > 4 else 0))
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw0 = v.pack_weights_device(W, g)
copies = max(2, -(-300_000_000 // pw0.nbytes))
pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev) * 0.01 + 1e-3
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
lk = M * (K // g) * N
for plan in plans:
    run = lambda p_: v.mpgemm_ws(p_, A, s, 0.02, out=out, plan=plan, ws=ws)
    for _ in range(3):
        run(pw0)
    torch.cuda.synchronize()
    res = {}
    for mode in ("flush", "noflush"):
        ts = []
        for i in range(20):
            if mode == "flush":
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run(pws[i % len(pws)])
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[mode] = float(np.median(ts))
    g_ = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_):
        for p_ in pws:
            run(p_)
    g_.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g_.replay()
    b.record()
    torch.cuda.synchronize()
    res["graph"] = a.elapsed_time(b) * 1e3 / (5 * len(pws))
    print(f"M={M} K={K} N={N} g={g} plan=w{plan.warps} s{plan.splits} n{plan.n_cta} sk{plan.streamk}: "
          + "  ".join(f"{k} {t:8.1f} us ({lk / R_LU / (t * 1e-6):.3f})" for k, t in res.items()),
          flush=True)
