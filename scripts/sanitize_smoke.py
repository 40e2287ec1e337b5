"""Small invocations of every kernel family (K1 cluster + stream-K, K2 vector +
scalar + split-K, K3 + quantize_t + quantize_amax, packer, fused all-gather
emulation) for compute-sanitizer memcheck runs (development tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
ws = v.workspace(dev)
for (M, K, N, g) in [(385, 1024, 130, 4), (200, 1285, 17, 5), (1000, 1300, 5, 4), (64, 64, 1, 4)]:
    W = synth.ternary_weights(M, K, 1)
    pw = v.pack_weights(W, g, device=dev)
    pwd = v.pack_weights_device(torch.from_numpy(W).to(dev), g)
    x = torch.randn(K, N, device=dev)
    q, s = v.quantize(x)
    q2, s2 = v.quantize_t(x.t().contiguous())
    o1 = v.mpgemm(pw, q, s, 0.02)
    o2 = v.mpgemm_ws(pw, q, s, 0.02, ws=ws)
    o3 = v.mpgemm_ex(pw, q, s, 0.02, plan=v.LaunchPlan(8, 3))
    o4 = v.mpgemm_ws(pw, q, s, 0.02, plan=v.LaunchPlan(16, 1, streamk=1), ws=ws)
    if N <= 64:
        o5 = v.mpgemm_ws(pw, q, s, 0.02, plan=v.slot_plan(tpw=2), ws=ws)
        o6 = v.mpgemm_scalar_lut(pw, q, s, 0.02, ws=ws)
    amax = torch.zeros(N, dtype=torch.int32, device=dev)
    o7 = v.mpgemm_fused(pw, q, s, 0.02, amax=amax, ws=ws)
    qa, sa = v.quantize_amax(o7, amax)
    bufs = [torch.zeros((M, N), device=dev) for _ in range(2)]
    v.mpgemm_allgather(pw, q, s, 0.02, bufs[0], 0, [bufs[1].data_ptr()])
    torch.cuda.synchronize()
    print("ok", M, K, N, g, float((o1 - o2).abs().max()), float((o1 - bufs[1]).abs().max()))
