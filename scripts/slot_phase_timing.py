"""Build a -DVLUT_TIMING variant of libvlut and print per-CTA phase times of K2
(globaltimer stamps of thread 0): entry, first index tile landed, first table
built, lookup loop done, int32 tile in shared memory, split-K arrival done,
epilogue stored (last CTA of a tile only).
  python scripts/slot_phase_timing.py M K N g tpw"""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B
lib = "/tmp/libvlut_timing.so"
subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f != "-v" and f != "-Xptxas"] +
                      ["-DVLUT_TIMING", "-o", lib] + os.environ.get("VLUT_EXTRA", "").split() + B.SOURCES)
import paper_2512_06443_b200 as v
v.lib_path = lib
from paper_2512_06443_b200 import synth
M, K, N, g, tpw = (int(x) for x in sys.argv[1:6])
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev)
out = torch.empty((M, N), device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
L = v.lib()
rc = L.vlut_debug_set_timing(ctypes.c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ws = v.workspace(dev)
plan = v.slot_plan(tpw=tpw)
for it in range(4):
    flush.zero_(); torch.cuda.synchronize()
    buf.zero_()
    torch.cuda.synchronize()
    v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
    torch.cuda.synchronize()
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = os.environ.get("NAMES", "entry idx0 table0 loop_end tile_smem arrived stored idx_last").split()
print("CTAs", len(t), "rc", rc, v.plan_ws(M, K, N, g))
for i, n in enumerate(names):
    col = t[:, i]
    col = col[col > 0]
    if len(col) == 0:
        continue
    rel = (col - t0) / 1000.0
    print(f"{n:10s} n={len(col):4d} min {rel.min():8.2f}  med {np.median(rel):8.2f}  max {rel.max():8.2f} us")
