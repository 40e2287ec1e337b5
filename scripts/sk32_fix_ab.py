"""A/B of builds on the planner's stream-K shapes (development tool): per
library, per shape, a CUDA graph of back-to-back launches over weight copies
> 2x L2 (mean per launch) and the output compared with the first library's.
  python scripts/sk32_fix_ab.py lib1.so lib2.so ..."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

R_LU = 148 * 64 * 1965e6
SHAPES = [(3072, 23040, 256, 5), (3072, 23040, 256, 4), (3072, 23040, 1024, 5), (3072, 23040, 1024, 4),
          (6144, 4096, 1024, 4), (14336, 4096, 1024, 4), (3840, 2560, 2048, 4), (6912, 2560, 2048, 4),
          (6912, 2560, 256, 4)]
dev = torch.device("cuda")
libs = sys.argv[1:]
res = {}
refs = {}
for li, path in enumerate(libs):
    v.lib_path = path
    v._lib = None
    for attr in ("_LIB", "_lib_handle"):
        if hasattr(v, attr):
            setattr(v, attr, None)
    ws = v.workspace(dev)
    for (M, K, N, g) in SHAPES:
        W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
        pw0 = v.pack_weights_device(W, g)
        copies = max(2, -(-260_000_000 // pw0.nbytes))
        pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
        gen = torch.Generator(device=dev).manual_seed(7)
        A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev, generator=gen)
        s = torch.rand(N, device=dev, generator=gen)
        out = torch.empty((M, N), device=dev)
        runs = [(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, ws=ws)))(p) for p in pws]
        for r in runs[:2]:
            r()
        torch.cuda.synchronize()
        g_ = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_):
            for r in runs:
                r()
        g_.replay(); torch.cuda.synchronize()
        per = max(2, 40 // len(runs))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(per):
            g_.replay()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e3 / (per * len(runs))
        v.mpgemm_ws(pw0, A, s, 0.02, out=out, ws=ws); torch.cuda.synchronize()
        key = (M, K, N, g)
        same = True
        if li == 0:
            refs[key] = out.clone()
        else:
            same = torch.equal(out, refs[key])
        pl = v.plan_ws(M, K, N, g)
        lk = M * (K // g) * N
        print(f"{os.path.basename(path):22s} M={M:5d} K={K:5d} N={N:4d} g={g} w{pl.warps} sk{pl.streamk} "
              f"m{pl.m_cta}: {t:8.2f} us frac {lk / R_LU / (t * 1e-6):.3f} same={same}", flush=True)
        del pws, pw0, W
        torch.cuda.empty_cache()
