"""Per-CTA phase times of K3 (the per-token quantizer) from a -DVLUT_TIMING
build of libvlut (globaltimer stamps of thread 0; development tool):
entry, after griddepcontrol.wait, loads+local max done, CTA max in smem,
cluster.sync done, scales ready, codes stored, exit barrier passed.
  python scripts/k3_phase_timing.py K N"""
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B  # noqa: E402

lib = "/tmp/libvlut_timing.so"
subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f not in ("-v", "-Xptxas")] +
                      ["-DVLUT_TIMING", "-o", lib] + B.SOURCES +
                      os.environ.get("VLUT_EXTRA", "").split())
import paper_2512_06443_b200 as v  # noqa: E402

v.lib_path = lib
K, N = (int(a) for a in sys.argv[1:3])
dev = torch.device("cuda")
x = torch.randn(K, N, device=dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev)
s = torch.empty((N,), device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
L = v.lib()
L.vlut_debug_set_timing(__import__("ctypes").c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(5):
    flush.zero_()
    buf.zero_()
    torch.cuda.synchronize()
    a.record()
    v.quantize(x, q=q, scale=s)
    b.record()
    torch.cuda.synchronize()
print("events us", a.elapsed_time(b) * 1e3)
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["entry", "pdl_waited", "loaded", "cta_max", "cluster_sync", "scales", "stored", "exit"]
print("CTAs", len(t))
for i, nme in enumerate(names):
    col = t[:, i]
    col = col[col > 0]
    if len(col) == 0:
        continue
    rel = (col - t0) / 1000.0
    print(f"{nme:13s} n={len(col):4d} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f} us")
