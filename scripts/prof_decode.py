"""Decode launches for ncu (development tool):
  python scripts/prof_decode.py [libvlut.so] -- config 4 g = 4 N = 1, planner's K2
plan, a few launches each after an L2 flush (profile with -k regex:vlut_slot)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
if len(sys.argv) > 1:
    v.lib_path = os.path.abspath(sys.argv[1])
M, K, N, g = 3072, 23040, 1, 4
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev) * 0.01 + 1e-3
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    v.mpgemm_ws(pw, A, s, 0.02, out=out, ws=ws)
torch.cuda.synchronize()
print(v.plan_ws(M, K, N, g))
