"""Build a -DVLUT_TIMING variant of libvlut and print per-CTA phase times of K1
(globaltimer stamps): entry, TMEM alloc, first table ready, main loop done,
red tile written, cluster sync, epilogue stores, exit."""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B
lib = "/tmp/libvlut_timing.so"
subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f != "-v" and f != "-Xptxas"] +
                      ["-DVLUT_TIMING", "-o", lib] + B.SOURCES)
import paper_2512_06443_b200 as v
v.lib_path = lib
from paper_2512_06443_b200 import synth
M, K, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
# optional plan: warps splits n_cta
plan = v.LaunchPlan(int(sys.argv[4]), int(sys.argv[5]), n_cta=int(sys.argv[6])) if len(sys.argv) > 6 else None
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1, 0.4)).to(dev)
pw = v.pack_weights_device(W, 4)
A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev)
out = torch.empty((M, N), device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
# set the __device__ pointer via cudaMemcpyToSymbol equivalent: use cuda-python-free trick
L = v.lib()
rc = L.vlut_debug_set_timing(ctypes.c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for it in range(3):
    flush.zero_(); torch.cuda.synchronize()
    buf.zero_()
    torch.cuda.synchronize()
    v.mpgemm_ex(pw, A, s, 0.02, out=out, plan=plan) if plan else v.mpgemm(pw, A, s, 0.02, out=out)
    torch.cuda.synchronize()
t = buf.view(-1, 8).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["entry", "tmem", "table0", "loop_end", "red_written", "sync1", "reduced", "stored"]
print("plan", plan)
print("CTAs", len(t), "rc", rc)
for i, n in enumerate(names):
    col = rel[:, i]
    print(f"{n:12s} min {col.min():8.2f}  med {np.median(col):8.2f}  max {col.max():8.2f} us")
