"""K1 phase timing (-DVLUT_TIMING build) right after a flush, with and
without a K3 quantizer launch (+ synchronize) before the flush: which phase
of K1 gets slower after K3 (development tool)."""
import ctypes, os, subprocess, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_06443_b200 import build as B
lib = "/tmp/libvlut_timing.so"
subprocess.check_call([B.nvcc()] + [f for f in B.NVCC_FLAGS if f not in ("-v", "-Xptxas")] +
                      ["-DVLUT_TIMING", "-DVLUT_TIMING_EPI", "-o", lib] + B.SOURCES)
import paper_2512_06443_b200 as v
v.lib_path = lib
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
M, K, N = 6912, 2560, 256
pw = v.pack_weights_device(torch.from_numpy(synth.ternary_weights(M, K, 1, 0.4)).to(dev), 4)
x = torch.randn(K, N, device=dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev); s = torch.empty(N, device=dev)
v.quantize(x, q=q, scale=s)
q2 = torch.empty_like(q); s2 = torch.empty_like(s); xt = x.t().contiguous()
out = torch.empty((M, N), device=dev)
buf = torch.zeros(65536 * 8, dtype=torch.int64, device=dev)
v.lib().vlut_debug_set_timing(ctypes.c_void_p(buf.data_ptr()))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
names = ["entry", "tmem", "table0", "loop_end", "red_written", "sync1", "dsmem_loaded", "stored"]
xs = x.clone()
for mode in ("plain", "after_sum_x", "plain", "after_sum_x"):
    acc = []
    for it in range(6):
        if mode == "after_k3":
            v.quantize(x, q=q, scale=s)
        elif mode == "after_sum_x":
            x.sum()
        elif mode == "after_q_write":
            q.fill_(3)
        elif mode == "after_k3_other_x":
            v.quantize(xs, q=q2, scale=s2)
        elif mode == "after_quantize_t":
            v.quantize_t(xt, q=q2, scale=s2)
        torch.cuda.synchronize()
        buf.zero_()
        flush.zero_()
        v.mpgemm(pw, q, s, 0.02, out=out)
        torch.cuda.synchronize()
        t = buf.view(-1, 8).cpu().numpy().astype(np.int64)[:144]
        t0 = t[:, 0].min()
        acc.append((t - t0) / 1000.0)
    rel = np.median(np.stack(acc), axis=0)
    print(mode, " ".join(f"{n}={np.median(rel[:, i]):.2f}/{rel[:, i].max():.2f}" for i, n in enumerate(names)))
