"""Soak test (development tool): random schedules, shapes and streams for a
fixed wall time, every result compared with the same call's first result
(all schedules are bit-identical, so any difference is a race or a
corrupted workspace).  python scripts/soak.py [seconds]"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
dev = torch.device("cuda")
rng = np.random.default_rng(7)
shapes = [(3072, 23040, 1, 4), (3072, 4608, 16, 4), (1100, 2560, 4, 5), (6912, 2560, 256, 4),
          (2560, 2560, 512, 4), (777, 1285, 64, 5), (64, 64, 2, 4), (4096, 4100, 96, 5)]
cases = []
for i, (M, K, N, g) in enumerate(shapes):
    W = torch.from_numpy(synth.ternary_weights(M, K, 70 + i)).to(dev)
    pw = v.pack_weights_device(W, g, pad_k=(K % g != 0))
    A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
    cases.append((pw, A, N))
plans = [None, v.LaunchPlan(8, 1), v.LaunchPlan(12, 2), v.LaunchPlan(16, 4),
         v.LaunchPlan(16, 1, streamk=1), v.LaunchPlan(12, 1, m_cta=768, streamk=1),
         v.LaunchPlan(8, 1, m_cta=512, streamk=1), v.slot_plan(tpw=2), v.slot_plan(tpw=1),
         v.slot_plan(tpw=2, splits=1), v.LaunchPlan(12, 1, n_cta=32), v.LaunchPlan(16, 2, n_cta=32),
         v.LaunchPlan(12, 1, m_cta=768, n_cta=32, streamk=1)]
streams = [torch.cuda.Stream() for _ in range(3)]
wss = [torch.zeros_like(v.workspace(dev)) for _ in streams]
refs = {}
launches = mism = 0
t0 = time.time()
pending = []
while time.time() - t0 < secs:
    si = int(rng.integers(0, 3))
    ci = int(rng.integers(0, len(cases)))
    pi = int(rng.integers(0, len(plans)))
    pw, A, N = cases[ci]
    plan = plans[pi]
    if plan is not None and plan.slot and N > 64:
        plan = None
    if plan is not None and plan.n_cta == 32 and N % 16:
        plan = None  # 32-token tiles need N % 16 == 0
    with torch.cuda.stream(streams[si]):
        acc = v.mpgemm_acc_ws(pw, A, plan=plan, ws=wss[si], stream=streams[si])
    pending.append((ci, pi, acc))
    launches += 1
    if len(pending) >= 64:
        torch.cuda.synchronize()
        for ci, pi, acc in pending:
            if ci not in refs:
                refs[ci] = acc.clone()
            elif not torch.equal(acc, refs[ci]):
                mism += 1
                print("MISMATCH case", ci, "plan", plans[pi], flush=True)
        pending.clear()
torch.cuda.synchronize()
print(f"soak: {launches} launches in {time.time() - t0:.0f} s on 3 streams, {mism} mismatches")
sys.exit(1 if mism else 0)
