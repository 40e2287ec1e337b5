"""Stream-K with 1 vs 2 output rows per lookup thread (development tool):
per-launch events after an L2 flush, median of 20, several big-N shapes."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
R_LU = 148 * 64 * 1965e6
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ws = v.workspace(dev)
shapes = [(3072, 23040, 1024, 4), (3072, 23040, 1024, 5), (3072, 23040, 256, 4), (3072, 23040, 256, 5),
          (3072, 23040, 4096, 5), (14336, 4096, 1024, 4), (4096, 14336, 1024, 4), (6144, 4096, 1024, 4),
          (4096, 4096, 1024, 4), (6912, 2560, 2048, 4), (3840, 2560, 2048, 4), (2560, 2560, 2048, 4),
          (6912, 2560, 256, 4), (4096, 14335, 1024, 5)]
for (M, K, N, g) in shapes:
    K = K - K % g
    W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
    pw = v.pack_weights_device(W, g)
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev) * 0.01 + 1e-3
    out = torch.empty((M, N), device=dev)
    res = {}
    for name, plan in (("auto", None), ("w16r1", v.LaunchPlan(16, 1, streamk=1)),
                       ("w12r1", v.LaunchPlan(12, 1, streamk=1)),
                       ("w12r2", v.LaunchPlan(12, 1, m_cta=768, streamk=1)),
                       ("w8r2", v.LaunchPlan(8, 1, m_cta=512, streamk=1))):
        run = lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
        for _ in range(2):
            run()
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); run(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = float(np.median(ts))
    lk = M * (K // g) * N
    pl = v.plan_ws(M, K, N, g)
    print(f"M={M:6d} K={K:6d} N={N:5d} g={g} auto[w{pl.warps} m{pl.m_cta} sk{pl.streamk}] " +
          " ".join(f"{k}={t:8.1f}us({lk / R_LU / (t * 1e-6):.3f})" for k, t in res.items()), flush=True)
