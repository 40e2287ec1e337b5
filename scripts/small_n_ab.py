"""Small-N (K2 region) timing of one libvlut build with the planner's plans
(development tool): CUDA graph of back-to-back launches over weight copies
> 2x L2, mean per launch; checks the int32 result against the oracle on 8 rows.
  python scripts/small_n_ab.py [libvlut.so]"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_06443_b200 as v  # noqa: E402
if len(sys.argv) > 1:
    v.lib_path = sys.argv[1]
import oracle  # noqa: E402  (dev-tool check only)
from paper_2512_06443_b200 import synth  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from decode_bench import bench  # noqa: E402

R_LU = 148 * 64 * 1965e6
dev = torch.device("cuda")
ws = v.workspace(dev)
for (M, K, g, Ns) in [(3072, 23040, 4, [1, 4, 16, 32, 64]), (6912, 2560, 4, [1, 16, 64]),
                      (2560, 6912, 4, [16, 64]), (3072, 23040, 5, [16])]:
    Wn = synth.ternary_weights(M, K, 1)
    W = torch.from_numpy(Wn).to(dev)
    pw0 = v.pack_weights_device(W, g)
    copies = int(min(96, max(2, -(-300_000_000 // pw0.nbytes))))
    pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(copies - 1)]
    for N in Ns:
        A = synth.int8_activations(K, N, seed=N)
        Ad = torch.from_numpy(A).to(dev)
        s = torch.rand(N, device=dev)
        out = torch.empty((M, N), device=dev)
        t = bench([(lambda p_: (lambda: v.mpgemm_ws(p_, Ad, s, 0.02, out=out, ws=ws)))(p) for p in pws]) * 1e-6
        acc = v.mpgemm_acc_ws(pw0, Ad, ws=ws)
        torch.cuda.synchronize()
        rows = np.arange(0, M, M // 8)
        ok = np.array_equal(acc.cpu().numpy()[rows], oracle.gemm_i32(Wn[rows], A))
        pl = v.plan_ws(M, K, N, g)
        lk = M * (K // g) * N
        print(f"{os.path.basename(v.lib_path):18s} M={M:5d} K={K:5d} N={N:3d} g={g}: {t * 1e6:8.2f} us "
              f"(smem frac {lk / R_LU / t:.3f})  slot={pl.slot} nw={pl.nw} S={pl.splits} m={pl.m_cta} exact={ok}",
              flush=True)
    del pws, pw0
    torch.cuda.empty_cache()
