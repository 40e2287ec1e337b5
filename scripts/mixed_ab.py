"""Mixed g=5/g=4 schedule (f2) and g=5 with K padding vs pure g=4 on the K-not-multiple-of-5 linears
of configs 3 and 5 (development tool): per-launch events after an L2 flush."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ws = v.workspace(dev)
def t(fn, reps=20):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))
for (M, K, N) in [(6144, 4096, 1024), (4096, 14336, 1024), (14336, 4096, 1024), (2560, 6912, 2048)]:
    W = synth.ternary_weights(M, K, 1)
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev) * 0.01 + 1e-3
    out = torch.empty((M, N), device=dev)
    p4 = v.pack_weights(W, 4, device=dev)
    pm = v.pack_weights_mixed(W, device=dev)
    k5, k4 = v.group_schedule(K)
    p5 = v.pack_weights(W, 5, device=dev, pad_k=True)
    t4 = t(lambda: v.mpgemm_ws(p4, A, s, 0.02, out=out, ws=ws))
    tm = t(lambda: v.mpgemm_mixed(pm, A, s, 0.02, out=out, ws=ws))
    t5 = t(lambda: v.mpgemm_ws(p5, A, s, 0.02, out=out, ws=ws))
    pl = v.plan_ws(M, K, N, 5)
    print(f"M={M} K={K} N={N} (k5={k5}, k4={k4}): g4 {t4:8.1f} us  mixed {tm:8.1f} us ({t4 / tm:.3f}x)  "
          f"g5 padded {t5:8.1f} us ({t4 / t5:.3f}x) [w{pl.warps} m{pl.m_cta}]")
