"""Fit per-launch fixed overhead of K1: time(K) = a + b * K at fixed plan."""
import sys, os, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v
from scripts.kbench import time_one
M, N = 6912, 256
for plan in [v.LaunchPlan(12, 2), v.LaunchPlan(12, 1)]:
    pts = []
    for K in (640, 1280, 2560, 5120, 10240):
        r = time_one(M, K, N, 4, plan=plan, reps=20)
        pts.append((K, r["us"]))
    Ks = np.array([p[0] for p in pts], float); ts = np.array([p[1] for p in pts])
    b, a = np.polyfit(Ks, ts, 1)
    print(json.dumps({"plan": str(plan), "points": pts, "fixed_us": a, "us_per_Kfeature": b}))
