"""Decode (N = 1 .. 16) timing of the planner's K2 launch (development tool):
  python scripts/decode_bench.py [libvlut.so ...]
For each build: (a) a CUDA graph of back-to-back mpGeMM launches over weight
copies > 2x L2 (every launch streams its weights from HBM), (b) the same with
a per-token quantizer (K3) before every mpGeMM -- a decode step's kernels.
Mean device time per launch (pair) and the fraction of the HBM roofline
(packed weights + activations + outputs at MEASURED_PEAKS' copy bandwidth)."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

try:
    HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
except Exception:
    HBM = 6534.1e9


def bench(runs, reps=200):
    for r in runs[:3]:
        r()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in runs:
            r()
    g.replay()
    torch.cuda.synchronize()
    per = max(3, reps // len(runs))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(per):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (per * len(runs))


def run(libpath):
    import importlib
    if libpath:
        v.lib_path = libpath
        v._lib = None
    dev = torch.device("cuda")
    ws = v.workspace(dev)
    res = []
    shapes = [(3072, 23040, 1, 4), (3072, 23040, 1, 5), (6912, 2560, 1, 4),
              (2560, 6912, 1, 4), (3072, 23040, 16, 4), (3072, 23040, 64, 4)]
    if os.environ.get("DECODE_SHAPES"):  # "M,K,N,g;M,K,N,g;..."
        shapes = [tuple(int(x) for x in t.split(",")) for t in os.environ["DECODE_SHAPES"].split(";")]
    for (M, K, N, g) in shapes:
        W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
        pw0 = v.pack_weights_device(W, g)
        copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
        pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
        x = torch.randn(K, N, device=dev)
        A, s = v.quantize(x)
        out = torch.empty((M, N), device=dev)
        hbm = pw0.nbytes + K * N + 4 * N + 4 * M * N
        t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, A, s, 0.02, out=out, ws=ws)))(p) for p in pws])
        def pair(p_):
            def f():
                v.quantize(x, q=A, scale=s)
                v.mpgemm_ws(p_, A, s, 0.02, out=out, ws=ws)
            return f
        tp = bench([pair(p) for p in pws])
        tf = None
        if N == 1 and hasattr(v, "mpgemm_decode"):
            xf = x[:, 0].contiguous()
            of = torch.empty((M,), device=dev)
            sf = torch.empty((1,), device=dev)
            tf = bench([(lambda p_: (lambda: v.mpgemm_decode(p_, xf, 0.02, out=of, scale_out=sf,
                                                              ws=ws)))(p) for p in pws])
        pl = v.plan_ws(M, K, N, g)
        r = dict(M=M, K=K, N=N, g=g, us=t, us_pair=tp, us_fused=tf,
                 frac_hbm=hbm / HBM / (t * 1e-6),
                 plan=f"slot={pl.slot} tpw={pl.tpw} nw={pl.nw} S={pl.splits}")
        res.append(r)
        fused = f"  fused decode {tf:7.2f} us" if tf is not None else ""
        print(f"{os.path.basename(libpath or 'libvlut.so'):24s} M={M:5d} K={K:5d} N={N:3d} g={g}: "
              f"{t:7.2f} us (frac HBM {r['frac_hbm']:.3f})  quantize+mpgemm {tp:7.2f} us{fused}  "
              f"[{r['plan']}]", flush=True)
        del pws, pw0, W
        torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    libs = sys.argv[1:] or [""]
    for lp in libs:
        run(lp)
