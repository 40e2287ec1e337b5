"""Quick kernel timing sweep (development tool): times vlut_mpgemm for the
BASELINE shapes with CUDA events, L2 flushed between launches, and prints
tokens/s, lookups/s and the fraction of the shared-memory lookup roofline."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
if os.environ.get("VLUT_LIB"):
    v.lib_path = os.environ["VLUT_LIB"]
from paper_2512_06443_b200 import synth  # noqa: E402

R_LU = 148 * 64 * 1965e6  # int16 lookup-adds/s at 128 B/clk/SM, 1965 MHz


def time_one(M, K, N, g, plan=None, reps=20, p_zero=None, ws=False):
    dev = torch.device("cuda")
    W = torch.from_numpy(synth.ternary_weights(M, K, 1, p_zero)).to(dev)
    pw = v.pack_weights_device(W, g)
    A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
    s = torch.rand(N, device=dev) * 0.01 + 1e-3
    out = torch.empty((M, N), device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    run = (lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan)) if ws else \
        (lambda: v.mpgemm_ex(pw, A, s, 0.02, out=out, plan=plan))
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
    t = float(np.median(ts))
    lookups = M * (K // g) * N
    pl = plan or (v.plan_ws(M, K, N, g) if ws else v.plan(M, K, N, g))
    return dict(M=M, K=K, N=N, g=g, plan=f"w{pl.warps} s{pl.splits} sk{pl.streamk}", us=t * 1e6,
                tok_s=N / t, gops=2 * M * K * N / t / 1e9, lookups_s=lookups / t,
                frac_roof=(lookups / R_LU) / t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plans", action="store_true")
    ap.add_argument("--ws", action="store_true", help="workspace path (stream-K allowed)")
    ap.add_argument("--shape", type=int, nargs=4, metavar=("M", "K", "N", "G"),
                    help="sweep every K1 plan (cluster w x s, stream-K w) on this shape only")
    a = ap.parse_args()
    rows = []
    if a.shape:
        M, K, N, g = a.shape
        rows.append(time_one(M, K, N, g, ws=True))
        for w in (8, 12, 16):
            rows.append(time_one(M, K, N, g, plan=v.LaunchPlan(w, 1, streamk=1), ws=True))
            for sp in range(1, 9):
                try:
                    rows.append(time_one(M, K, N, g, plan=v.LaunchPlan(w, sp)))
                except Exception as e:  # plan not launchable for this shape
                    print(f"w{w} s{sp}: {e}")
        for r in rows:
            print(f"M={r['M']:6d} K={r['K']:6d} N={r['N']:5d} g={r['g']} plan={r['plan'][:24]:24s} "
                  f"us={r['us']:9.2f} frac={r['frac_roof']:.3f}")
        return
    rows.append(time_one(6912, 2560, 256, 4, p_zero=0.4, ws=a.ws))
    for N in (256, 1024, 4096):
        for g in (4, 5):
            rows.append(time_one(3072, 23040, N, g, ws=a.ws))
    for lin in synth.CONFIGS[3].linears:
        rows.append(time_one(lin.M, lin.K, 1024, 4, ws=a.ws))
    for lin in synth.CONFIGS[5].linears:
        rows.append(time_one(lin.M, lin.K, 2048, 4, ws=a.ws))
    if a.plans:
        for w in (8, 12, 16):
            for sp in (1, 2, 3, 4, 5, 6, 7, 8):
                rows.append(time_one(6912, 2560, 256, 4, plan=v.LaunchPlan(w, sp)))
    for r in rows:
        print(f"M={r['M']:6d} K={r['K']:6d} N={r['N']:5d} g={r['g']} plan={r['plan'][:24]:24s} "
              f"us={r['us']:9.2f} frac={r['frac_roof']:.3f}")


if __name__ == "__main__":
    main()
