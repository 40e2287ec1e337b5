"""Mid-N (32..192) plans after the fp32 split-tile meeting (development tool):
planner's choice vs forced K1-32-SK 12 x 1 / 12 x 2, graph of back-to-back
launches over weight copies > 2x L2.   python scripts/midn_probe.py"""
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
for (M, K, g, Ns) in [(3072, 23040, 4, [32, 64, 128]), (6912, 2560, 4, [64, 96, 128, 192]),
                      (3072, 23040, 5, [32, 64, 128])]:
    W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    for N in Ns:
        A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
        s = torch.rand(N, device=dev)
        out = torch.empty((M, N), device=dev)
        lk = M * (K // g) * N
        auto = v.plan_ws(M, K, N, g)
        for name, pl in [("auto", None), ("sk32 12x1", v.LaunchPlan(12, 1, m_cta=384, n_cta=32, streamk=1)),
                         ("sk32 12x2", v.LaunchPlan(12, 1, m_cta=768, n_cta=32, streamk=1))]:
            try:
                t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, plan=pl, ws=ws)))(p)
                           for p in pws]) * 1e-6
                desc = (f"slot={auto.slot} nw={auto.nw} S={auto.splits} sk={auto.streamk} m={auto.m_cta} "
                        f"n={auto.n_cta}") if pl is None else ""
                print(f"M={M} K={K} N={N} g={g} {name:10s}: {t * 1e6:8.2f} us  frac {lk / R_LU / t:.3f}  {desc}",
                      flush=True)
            except Exception as e:
                print(f"M={M} K={K} N={N} g={g} {name}: n/a {str(e)[:80]}")
    del pws, pw0
    torch.cuda.empty_cache()
