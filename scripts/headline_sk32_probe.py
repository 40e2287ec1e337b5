"""configs[1] (6912 x 2560, N = 256, g = 4): the planner's K1-32 vs forced
K1-32-SK 12 x 1 / 12 x 2 after the fp32 split-tile meeting (development
tool); graph of back-to-back launches over weight copies > 2x L2."""
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
SHAPES = [(6912, 2560, 256, 4), (6912, 2560, 512, 4), (3840, 2560, 2048, 4)]
if os.environ.get("PROBE_SHAPES"):  # "M,K,N,g;M,K,N,g"
    SHAPES = [tuple(int(x) for x in t.split(",")) for t in os.environ["PROBE_SHAPES"].split(";")]
for (M, K, N, g) in SHAPES:
    W = torch.from_numpy(synth.ternary_weights(M, K, 1, 0.4)).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev)
    out = torch.empty((M, N), device=dev)
    lk = M * (K // g) * N
    for name, pl in [("auto", None), ("sk32 12x1", v.LaunchPlan(12, 1, m_cta=384, n_cta=32, streamk=1)),
                     ("sk32 12x2", v.LaunchPlan(12, 1, m_cta=768, n_cta=32, streamk=1))]:
        for envv in ("",) if os.environ.get("PROBE_SHAPES") else ("", "1"):
            if envv:
                os.environ["VLUT_SK32_INT_PARTIALS"] = "1"
            else:
                os.environ.pop("VLUT_SK32_INT_PARTIALS", None)
            t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, plan=pl, ws=ws)))(p)
                       for p in pws]) * 1e-6
            print(f"M={M} K={K} N={N} {name:10s} {'int32 partials' if envv else 'default meeting'}: "
                  f"{t * 1e6:8.2f} us frac {lk / R_LU / t:.3f}", flush=True)
    os.environ.pop("VLUT_SK32_INT_PARTIALS", None)
    del pws, pw0
    torch.cuda.empty_cache()
