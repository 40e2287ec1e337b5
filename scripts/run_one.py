"""Run one mpGeMM configuration a few times (for ncu captures):
python scripts/run_one.py M K N g arm [reps]; arm in k2_vec, k2_scalar, auto_ws, k1."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

M, K, N, g = (int(x) for x in sys.argv[1:5])
arm = sys.argv[5]
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 4
dev = torch.device("cuda")
pw = v.pack_weights_device(torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev), g)
A = torch.randint(-127, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev) * 0.01 + 1e-3
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
for _ in range(reps):
    if arm == "k2_vec":
        v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=v.slot_plan(tpw=2), ws=ws)
    elif arm == "k2_scalar":
        v.mpgemm_scalar_lut(pw, A, s, 0.02, out=out, ws=ws)
    elif arm == "auto_ws":
        v.mpgemm_ws(pw, A, s, 0.02, out=out, ws=ws)
    else:
        v.mpgemm(pw, A, s, 0.02, out=out)
torch.cuda.synchronize()
print("ok", M, K, N, g, arm, v.plan_ws(M, K, N, g))
