"""Per-CTA phase stamps of K1-32-SK (-DVLUT_TIMING build): entry, first table
ready (lookup thread 0), producer epilogue start, owner wait start / done,
lookups + epilogues done.   python scripts/sk32_phase_timing.py M K N g rpt"""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B
lib = os.path.join(ROOT, "abtmp", "libvlut_timing_sk32.so")
if not os.path.exists(lib):
    subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f not in ("-v", "-Xptxas")] +
                          ["-DVLUT_TIMING", "-o", lib] + B.SOURCES)
import paper_2512_06443_b200 as v
v.lib_path = lib
from paper_2512_06443_b200 import synth
M, K, N, g, rpt = (int(x) for x in sys.argv[1:6])
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev)
out = torch.empty((M, N), device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
L = v.lib()
L.vlut_debug_set_timing(ctypes.c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ws = v.workspace(dev)
plan = v.plan_ws(M, K, N, g)
print("plan", plan)
for it in range(4):
    flush.zero_(); torch.cuda.synchronize()
    buf.zero_(); torch.cuda.synchronize()
    v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
    torch.cuda.synchronize()
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
for i, n in enumerate("entry table0 owner_wait owner_go end producer_epi".split()):
    col = t[:, i if i < 5 else 5]
    col = col[col > 0]
    if len(col):
        rel = (col - t0) / 1000.0
        print(f"{n:12s} n={len(col):4d} min {rel.min():8.2f} med {np.median(rel):8.2f} max {rel.max():8.2f} us")
ow = t[(t[:, 2] > 0) & (t[:, 3] > 0)]
if len(ow):
    w = (ow[:, 3] - ow[:, 2]) / 1000.0
    print(f"owner spin   n={len(w)} min {w.min():.2f} med {np.median(w):.2f} max {w.max():.2f} us")
order = np.argsort(-t[:, 4])[:6]
print("latest CTAs (cta: entry table0 owner_wait owner_go end producer_epi, us):")
idx = np.nonzero(buf.view(-1, 8).cpu().numpy()[:, 0] > 0)[0]
for o in order:
    row = [(x - t0) / 1000.0 if x > 0 else float("nan") for x in t[o, :6]]
    print(f"  cta {idx[o]:4d}: " + " ".join(f"{x:8.2f}" for x in row))
