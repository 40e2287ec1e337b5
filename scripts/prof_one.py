"""One mpGeMM launch of a given plan for ncu (development tool):
  python scripts/prof_one.py M K N g warps splits n_cta [streamk] [m_cta]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
M, K, N, g, w, sp, nc = (int(x) for x in sys.argv[1:8])
sk = int(sys.argv[8]) if len(sys.argv) > 8 else 0
mc = int(sys.argv[9]) if len(sys.argv) > 9 else 0
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev) * 0.01 + 1e-3
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
plan = v.LaunchPlan(w, sp, m_cta=mc, n_cta=nc, streamk=sk)
for _ in range(3):
    flush.zero_()
    v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
torch.cuda.synchronize()
