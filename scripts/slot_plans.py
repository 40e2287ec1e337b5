"""Forced K2 plans at small N (development tool): per (shape, nw, tpw,
splits) a CUDA graph of back-to-back launches over weight copies > 2x L2,
mean per launch, and the fraction of the shared-memory lookup roofline.
  python scripts/slot_plans.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from decode_bench import bench  # noqa: E402

R_LU = 148 * 64 * 1965e6
dev = torch.device("cuda")
ws = v.workspace(dev)
CASES = [(3072, 23040, 16, 4, [(8, 2, 0), (4, 2, 0), (2, 2, 0), (4, 2, 11), (4, 2, 33)]),
         (3072, 23040, 64, 4, [(8, 2, 0), (4, 2, 0), (8, 2, 6)]),
         (3072, 23040, 16, 5, [(2, 2, 0), (1, 2, 0)]),
         (6912, 2560, 16, 4, [(8, 2, 0), (4, 2, 0), (2, 2, 0)])]
for (M, K, N, g, plans) in CASES:
    W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    A, s = v.quantize(torch.randn(K, N, device=dev))
    out = torch.empty((M, N), device=dev)
    lk = M * (K // g) * N
    auto = v.plan_ws(M, K, N, g)
    for (nw, tpw, sp) in plans:
        pl = v.slot_plan(tpw=tpw, nw=nw, splits=sp)
        try:
            t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, plan=pl, ws=ws)))(p)
                       for p in pws]) * 1e-6
            print(f"M={M} K={K} N={N} g={g} nw={nw} tpw={tpw} splits={sp or 'auto'}: {t * 1e6:7.2f} us "
                  f"({lk / R_LU / t:.3f} of SMEM roof)   [planner: nw={auto.nw} S={auto.splits}]", flush=True)
        except Exception as e:
            print(f"M={M} K={K} N={N} g={g} nw={nw} tpw={tpw} splits={sp}: n/a {str(e)[:60]}")
    del pws, pw0
    torch.cuda.empty_cache()
