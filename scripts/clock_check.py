"""SM clock (NVML) while a plan runs back to back for ~1.5 s (development
tool): python scripts/clock_check.py M K N g plan[;plan...] (warps,splits,n_cta[,streamk])"""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
R_LU = 148 * 64 * 1965e6
M, K, N, g = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1)).to(dev)
pw = v.pack_weights_device(W, g)
A = torch.randint(-128, 128, (K, N), dtype=torch.int8, device=dev)
s = torch.rand(N, device=dev) * 0.01 + 1e-3
out = torch.empty((M, N), device=dev)
ws = v.workspace(dev)
lk = M * (K // g) * N
for t in sys.argv[5].split(";"):
    f = [int(x) for x in t.split(",")]
    plan = v.LaunchPlan(f[0], f[1], n_cta=f[2], streamk=f[3] if len(f) > 3 else 0)
    run = lambda: v.mpgemm_ws(pw, A, s, 0.02, out=out, plan=plan, ws=ws)
    gr = torch.cuda.CUDAGraph()
    run(); torch.cuda.synchronize()
    with torch.cuda.graph(gr):
        for _ in range(50):
            run()
    gr.replay(); torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        t0 = time.perf_counter(); n = 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        while time.perf_counter() - t0 < 1.5:
            gr.replay(); n += 1
            torch.cuda.synchronize()
        b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / (n * 50)
    cs = clk.summary()
    print(f"plan {t:14s}: {us:8.2f} us/launch ({lk / R_LU / (us * 1e-6):.3f})  sm_mhz median "
          f"{cs.get('sm_mhz')} reasons {cs.get('reasons')}", flush=True)
