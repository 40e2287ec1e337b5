"""K2 (lane-slot / scalar-LUT) vs K1 timing sweep (development tool): CUDA
events around each launch, L2 flushed between launches (weights streamed from
HBM), median of reps.  Prints us, the fraction of the SMEM lookup roofline
(2 B per lookup-add at 148 x 128 B/clk x 1965 MHz) and of the HBM roofline
(packed weight + activation + output bytes at the measured copy bandwidth)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

R_LU = 148 * 64 * 1965e6  # int16 lookup-adds/s
HBM = 6534.1e9


def bench(runs, reps):
    """Mean device time per launch: one pass over `runs` (one launch per
    weight copy; the copies together exceed the 126 MB L2, so every launch
    streams its weights from HBM) is captured in a CUDA graph and replayed,
    so host launch overhead is not measured (event resolution on B200 is
    ~2 us, hence batches)."""
    for r in runs[:3]:
        r()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r in runs:
            r()
    g.replay()
    torch.cuda.synchronize()
    n = len(runs)
    per = max(2, (reps + n - 1) // n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(per):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / (per * n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    dev = torch.device("cuda")
    ws = v.workspace(dev)
    rows = []
    shapes = [(3072, 23040, N, g) for g in (4, 5) for N in (1, 4, 16, 64, 256)]
    shapes += [(6912, 2560, N, 4) for N in (1, 16, 256)]
    shapes += [(2560, 6912, 1, 4), (14336, 4096, 1, 4), (4096, 14336, 1, 4)]
    for (M, K, N, g) in shapes:
        W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
        pw0 = v.pack_weights_device(W, g)
        copies = int(min(64, max(1, -(-300_000_000 // pw0.nbytes))))
        pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
        A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
        s = torch.rand(N, device=dev) * 0.01 + 1e-3
        out = torch.empty((M, N), device=dev)
        lookups = M * (K // g) * N
        hbm_bytes = pw0.nbytes + K * N + 4 * N + 4 * M * N
        arms = {
            "k1_cluster": lambda pw: (lambda: v.mpgemm_ex(pw, A, s, 0.02, out=out,
                                                          plan=v.plan(M, K, N, g))),
            "k1_streamk": lambda pw: (lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out,
                                                          plan=v.LaunchPlan(16, 1, streamk=1),
                                                          ws=ws)),
            "k2_vec": lambda pw: (lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out,
                                                      plan=v.slot_plan(tpw=2), ws=ws)),
            "k2_scalar": lambda pw: (lambda: v.mpgemm_scalar_lut(pw, A, s, 0.02, out=out, ws=ws)),
            "auto_ws": lambda pw: (lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, ws=ws)),
        }
        if N > 64:
            arms.pop("k2_vec")
            arms.pop("k2_scalar")
        pl = v.plan_ws(M, K, N, g)
        for name, mk in arms.items():
            t = bench([mk(pw) for pw in pws], a.reps)
            r = dict(M=M, K=K, N=N, g=g, arm=name, us=t * 1e6, copies=copies,
                     frac_smem=(lookups / R_LU) / t, frac_hbm=(hbm_bytes / HBM) / t,
                     auto=f"slot={pl.slot} tpw={pl.tpw} nw={pl.nw} S={pl.splits} sk={pl.streamk}")
            rows.append(r)
            print(f"M={M:6d} K={K:6d} N={N:5d} g={g} {name:11s} us={r['us']:9.2f} "
                  f"smem={r['frac_smem']:.3f} hbm={r['frac_hbm']:.3f}  [{r['auto']}]", flush=True)
        del pws, pw0, W, A, out
        torch.cuda.empty_cache()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
