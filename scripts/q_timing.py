"""Phase timing of the K3 quantizer (-DVLUT_TIMING build)."""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B
lib = "/tmp/libvlut_timing.so"
subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f not in ("-v", "-Xptxas")] +
                      ["-DVLUT_TIMING", "-o", lib] + B.SOURCES)
import paper_2512_06443_b200 as v
v.lib_path = lib
K, N = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
x = torch.randn(K, N, device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
v.lib().vlut_debug_set_timing(ctypes.c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for it in range(3):
    flush.zero_(); torch.cuda.synchronize(); buf.zero_(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); v.quantize(x); e1.record(); torch.cuda.synchronize()
print("event us", e0.elapsed_time(e1) * 1e3)
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
for i, n in enumerate(["entry", "pdl", "loaded", "cta_red", "csync", "scale", "stored", "exit"]):
    col = rel[:, i]
    print(f"{n:10s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
