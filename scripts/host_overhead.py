"""Host-side cost of one binding call (development tool): wall time of
back-to-back enqueues without synchronisation."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
M, K, N = 6912, 2560, 256
pw = v.pack_weights_device(torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev), 4)
x = torch.randn(K, N, device=dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev); s = torch.empty(N, device=dev)
out = torch.empty((M, N), device=dev); ws = v.workspace(dev); st = torch.cuda.current_stream()
for name, fn in [("quantize", lambda: v.quantize(x, q=q, scale=s, stream=st)),
                 ("mpgemm_ws", lambda: v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)),
                 ("mpgemm", lambda: v.mpgemm(pw, q, s, 0.02, out=out, stream=st))]:
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name}: host {1e6 * (t1 - t0) / n:.1f} us per call (enqueue only)")
