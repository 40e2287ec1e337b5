"""Token-count sweep on the configs[1] weights (6912 x 2560, g = 4) with the
auto planner (development tool): per-launch events after an L2 flush for
N >= 128, a CUDA graph over weight copies (> 2x L2) below; prints the
chosen kernel, time, tokens/s and the fraction of max(T_hbm, T_lookup)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
if len(sys.argv) > 1:  # optional libvlut.so build to sweep
    v.lib_path = os.path.abspath(sys.argv[1])
dev = torch.device("cuda")
M, K, g = 6912, 2560, 4
R_LU = 148 * 64 * 1965e6
HBM = 6534.1e9
W = torch.from_numpy(synth.ternary_weights(M, K, 2000, 0.4)).to(dev)
pws = [v.pack_weights_device(W, g) for _ in range(60)]
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for N in (1, 2, 4, 8, 16, 32, 48, 64, 80, 96, 112, 128, 160, 192, 256, 512, 1024, 2048, 4096):
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev) * 0.01 + 1e-3
    out = torch.empty((M, N), device=dev)
    if N < 128:
        runs = [lambda p_=p_: v.mpgemm_ws(p_, A, s, 0.02, out=out, ws=ws) for p_ in pws]
        for r in runs[:2]: r()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for r in runs: r()
        gr.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): gr.replay()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e-3 / (5 * len(runs))
    else:
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); v.mpgemm_ws(pws[0], A, s, 0.02, out=out, ws=ws); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = float(np.median(ts))
    lk = M * (K // g) * N
    hb = M * K // g + K * N + 4 * N + 4 * M * N
    roof = max(lk / R_LU, hb / HBM)
    pl = v.plan_ws(M, K, N, g)
    kern = (f"K2 tpw={pl.tpw} nw={pl.nw} S={pl.splits}" if pl.slot else
            f"K1 w{pl.warps} m{pl.m_cta} n{pl.n_cta} S={pl.splits} sk={pl.streamk}")
    print(f"N={N:5d} {kern:28s} {t * 1e6:9.2f} us  {N / t / 1e6:8.3f} M tok/s  "
          f"frac {roof / t:.3f} ({'hbm' if hb / HBM > lk / R_LU else 'smem'})", flush=True)
