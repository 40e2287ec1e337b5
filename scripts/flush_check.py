"""Does the L2 flush flush?  K1 at configs[1] timed right after different
256 MiB flushes (development tool): zero memset, non-zero fill, and a copy
of 256 MiB of random bytes; plus the DRAM bytes are visible in ncu runs."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
if len(sys.argv) > 1:
    v.lib_path = sys.argv[1]
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
M, K, N = 6912, 2560, 256
pw = v.pack_weights_device(torch.from_numpy(synth.ternary_weights(M, K, 1, 0.4)).to(dev), 4)
x = torch.randn(K, N, device=dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev); s = torch.empty(N, device=dev)
v.quantize(x, q=q, scale=s)
out = torch.empty((M, N), device=dev); ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
src = torch.randint(0, 255, (256 << 20,), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
modes = {
    "zero_memset": lambda: flush.zero_(),
    "fill_0x5a": lambda: flush.fill_(0x5A),
    "copy_random": lambda: flush.copy_(src),
    "none": lambda: None,
    "read_x_then_flush": lambda: (x.sum(), flush.zero_()),
}
for name, fl in list(modes.items()) * 2:
    ts = []
    for i in range(60):
        torch.cuda.synchronize()
        fl()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:12s} K1 mean {np.mean(ts):.2f} med {np.median(ts):.2f} us")
