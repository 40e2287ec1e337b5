"""Zero-copy input probe (development tool): the configs[1] step's fp32
activations read by the quantizer straight from pinned host memory (UVA)
versus an H2D copy followed by the quantizer; per-step time of a pipelined
back-to-back loop and of the pieces."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

dev = torch.device("cuda")
M, K, N, g = 6912, 2560, 256, 4
L = v.lib()
x = np.random.default_rng(0).standard_normal((K, N)).astype(np.float32)
xh = torch.from_numpy(x).pin_memory()
xd = torch.empty((K, N), device=dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev)
s = torch.empty((N,), device=dev)
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)


def quant(ptr):
    rc = L.vlut_quantize(ctypes.c_void_p(ptr), None, K, N, ctypes.c_void_p(q.data_ptr()),
                         ctypes.c_void_p(s.data_ptr()), sp)
    assert rc == 0, rc


def t(fn, n=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


quant(xd.data_ptr())
xd.copy_(xh)
quant(xd.data_ptr())
q_ref, s_ref = q.clone(), s.clone()
quant(xh.data_ptr())
torch.cuda.synchronize()
print("zero-copy codes == device codes:", bool(torch.equal(q, q_ref) and torch.equal(s, s_ref)))
print(f"quantize from device memory       {t(lambda: quant(xd.data_ptr())):7.1f} us")
print(f"H2D copy alone                    {t(lambda: xd.copy_(xh, non_blocking=True)):7.1f} us")
print(f"H2D copy + quantize               {t(lambda: (xd.copy_(xh, non_blocking=True), quant(xd.data_ptr()))):7.1f} us")
print(f"quantize from pinned host (UVA)   {t(lambda: quant(xh.data_ptr())):7.1f} us")
