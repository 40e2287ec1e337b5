"""Planner-model A/B (development tool): the auto plan's time over an N sweep
under run-time planner switches (env, read at launch), graph of back-to-back
launches over weight copies > 2x L2.   python scripts/planner_ab.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from decode_bench import bench  # noqa: E402

R_LU = 148 * 64 * 1965e6
MODELS = {"old": {"VLUT_SK32_MODEL_OLD": "1"}, "new": {}}
dev = torch.device("cuda")
ws = v.workspace(dev)
SW = [(6912, 2560, 4, [48, 64, 80, 96, 112, 128, 160, 192, 256, 512, 1024]),
      (3072, 23040, 4, [32, 48, 64, 96, 128, 192, 256]),
      (3072, 23040, 5, [32, 48, 64, 96, 128, 192, 256]),
      (4096, 4096, 4, [128, 256, 1024]), (2560, 6912, 4, [64, 128, 256, 2048])]
for (M, K, g, Ns) in SW:
    W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    for N in Ns:
        A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
        s = torch.rand(N, device=dev)
        out = torch.empty((M, N), device=dev)
        lk = M * (K // g) * N
        line = f"M={M:5d} K={K:5d} N={N:4d} g={g}:"
        for name, env in MODELS.items():
            for k in ("VLUT_SK32_MODEL_OLD",):
                os.environ.pop(k, None)
            os.environ.update(env)
            pl = v.plan_ws(M, K, N, g)
            t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, ws=ws)))(p) for p in pws]) * 1e-6
            tag = (f"K2" if pl.slot else f"{'SK' if pl.streamk else 'CL'}{pl.n_cta}w{pl.warps}m{pl.m_cta}s{pl.splits}")
            line += f"  {name} {t * 1e6:8.2f} ({lk / R_LU / t:.3f} {tag})"
        print(line, flush=True)
    del pws, pw0
    torch.cuda.empty_cache()
