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


def bench(run, reps, flush):
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    dev = torch.device("cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ws = v.workspace(dev)
    rows = []
    shapes = [(3072, 23040, N, g) for g in (4, 5) for N in (1, 4, 16, 64, 256)]
    shapes += [(6912, 2560, N, 4) for N in (1, 16, 256)]
    shapes += [(2560, 6912, 1, 4), (14336, 4096, 1, 4), (4096, 14336, 1, 4)]
    for (M, K, N, g) in shapes:
        W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
        pw = v.pack_weights_device(W, g)
        A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
        s = torch.rand(N, device=dev) * 0.01 + 1e-3
        out = torch.empty((M, N), device=dev)
        lookups = M * (K // g) * N
        hbm_bytes = pw.nbytes + K * N + 4 * N + 4 * M * N
        arms = {
            "k1_cluster": lambda: v.mpgemm_ex(pw, A, s, 0.02, out=out, plan=v.plan(M, K, N, g)),
            "k1_streamk": lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out,
                                              plan=v.LaunchPlan(16, 1, streamk=1), ws=ws),
            "k2_vec": lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=v.slot_plan(tpw=2), ws=ws),
            "k2_scalar": lambda: v.mpgemm_scalar_lut(pw, A, s, 0.02, out=out, ws=ws),
            "auto_ws": lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, ws=ws),
        }
        pl = v.plan_ws(M, K, N, g)
        for name, run in arms.items():
            t, tmin = bench(run, a.reps, flush)
            r = dict(M=M, K=K, N=N, g=g, arm=name, us=t * 1e6, us_min=tmin * 1e6,
                     frac_smem=(lookups / R_LU) / t, frac_hbm=(hbm_bytes / HBM) / t,
                     auto=f"slot={pl.slot} tpw={pl.tpw} nw={pl.nw} S={pl.splits} sk={pl.streamk}")
            rows.append(r)
            print(f"M={M:6d} K={K:6d} N={N:5d} g={g} {name:11s} us={r['us']:9.2f} "
                  f"smem={r['frac_smem']:.3f} hbm={r['frac_hbm']:.3f}  [{r['auto']}]", flush=True)
        del pw, W, A, out
    if a.json:
        with open(a.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
