"""A/B timing of libvlut builds on K1 shapes (development tool):
  python scripts/k1_ab.py libA.so [libB.so ...]   ("" = the in-tree build)
Per (shape, plan): one launch per L2 flush, CUDA events around it, median of
reps; every build gets its own zeroed workspace.  Prints us and the fraction
of the shared-memory lookup roofline (148 x 128 B/clk x 1965 MHz, 2 B per
lookup-add)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

R_LU = 148 * 64 * 1965e6
SHAPES = [  # (M, K, N, g, plan-name)
    (6912, 2560, 256, 4, "auto"), (6912, 2560, 256, 4, "c12x2"),
    (3072, 23040, 256, 4, "auto"), (3072, 23040, 256, 5, "auto"), (3072, 23040, 256, 5, "w8r2"),
    (3072, 23040, 1024, 4, "auto"), (3072, 23040, 1024, 5, "auto"),
    (3072, 23040, 1024, 5, "w12r2"), (3072, 23040, 1024, 5, "w8r2"),
    (3072, 23040, 4096, 5, "auto"), (6144, 4096, 1024, 4, "auto"), (14336, 4096, 1024, 4, "auto"),
    (6912, 2560, 2048, 4, "auto"), (3840, 2560, 2048, 4, "auto"), (2560, 6912, 2048, 4, "auto"),
]
PLANS = {"auto": None, "c12x2": (12, 2, 0, 0), "w12r2": (12, 1, 768, 1), "w8r2": (8, 1, 512, 1),
         "w8r3": (8, 1, 768, 1), "w16r1": (16, 1, 0, 1), "w12r1": (12, 1, 0, 1),
         "n32w12": (12, 1, 0, 0, 32), "n32w16": (16, 1, 0, 0, 32), "n32w8": (8, 1, 0, 0, 32),
         "n32w12s2": (12, 2, 0, 0, 32), "n32w16s2": (16, 2, 0, 0, 32), "n32w8s2": (8, 2, 0, 0, 32),
         "n32w12s4": (12, 4, 0, 0, 32), "n32w12s8": (12, 8, 0, 0, 32), "n32w8s8": (8, 8, 0, 0, 32),
         "n32w16s8": (16, 8, 0, 0, 32), "n32w8s4": (8, 4, 0, 0, 32), "n32w16s4": (16, 4, 0, 0, 32),
         "sk32w12r1": (12, 1, 384, 1, 32), "sk32w16r1": (16, 1, 512, 1, 32),
         "sk32w12r2": (12, 1, 768, 1, 32), "sk32w16r2": (16, 1, 1024, 1, 32),
         "sk32w12r4": (12, 1, 1536, 1, 32), "sk32w12r3": (12, 1, 1152, 1, 32),
         "sk32w8r3": (8, 1, 768, 1, 32), "sk32w8r2": (8, 1, 512, 1, 32)}


def main():
    libs = sys.argv[1:] or [""]
    if os.environ.get("K1AB_SHAPES"):
        # "M,K,N,g,plan;M,K,N,g,plan;..."
        shapes = [tuple(int(x) for x in t.split(",")[:4]) + (t.split(",")[4],)
                  for t in os.environ["K1AB_SHAPES"].split(";")]
    elif os.environ.get("K1AB_PLANS"):
        keep = set(os.environ["K1AB_PLANS"].split(","))
        shapes = [s for s in SHAPES if s[4] in keep]
    else:
        shapes = SHAPES
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    reps = int(os.environ.get("K1AB_REPS", "15"))
    for (M, K, N, g, pn) in shapes:
        W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
        pw = v.pack_weights_device(W, g)
        A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
        s = torch.rand(N, device=dev) * 0.01 + 1e-3
        out = torch.empty((M, N), device=dev)
        lk = M * (K // g) * N
        row = f"M={M:5d} K={K:5d} N={N:4d} g={g} {pn:6s}"
        for lp in libs:
            v.lib_path = lp or os.path.join(os.path.dirname(v.__file__), "libvlut.so")
            v._lib = None
            ws = torch.zeros(int(v.lib().vlut_workspace_bytes()), dtype=torch.uint8, device=dev)
            pl = PLANS[pn]
            plan = None if pl is None else v.LaunchPlan(pl[0], pl[1], m_cta=pl[2], streamk=pl[3],
                                                         n_cta=pl[4] if len(pl) > 4 else 64)
            run = lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
            try:
                for _ in range(3):
                    run()
                torch.cuda.synchronize()
                if os.environ.get("K1AB_EVENTS"):
                    ts = []
                    for _ in range(reps):
                        flush.zero_()
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record()
                        run()
                        b.record()
                        torch.cuda.synchronize()
                        ts.append(a.elapsed_time(b) * 1e3)
                    t = float(np.median(ts))
                else:
                    # per-launch events resolve ~2 us on B200: time a CUDA graph of
                    # (L2 flush, launch) x n minus a graph of n flushes alone
                    def graph_time(with_run, n=12):
                        gr = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gr):
                            for _ in range(n):
                                flush.zero_()
                                if with_run:
                                    run()
                        gr.replay()
                        torch.cuda.synchronize()
                        best = []
                        for _ in range(3):
                            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            a.record()
                            gr.replay()
                            b.record()
                            torch.cuda.synchronize()
                            best.append(a.elapsed_time(b) * 1e3 / n)
                        return float(np.median(best))
                    t = graph_time(True) - graph_time(False)
                row += f" | {os.path.basename(lp) or 'tree'}: {t:8.1f} us {lk / R_LU / (t * 1e-6):.3f}"
            except Exception as e:  # plan not supported by this build
                row += f" | {os.path.basename(lp) or 'tree'}: n/a ({str(e)[:40]})"
            del ws
        print(row, flush=True)
        del pw, W, A, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
