"""Per-kernel times of one config-5 layer (N=2048) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
from paper_2512_06443_b200.sharded import RowShardedLinear
cfg = synth.CONFIGS[5]
dev = torch.device("cuda")
N = 2048
L = [RowShardedLinear(w, 4, synth.W_SCALE, device=dev, device_pack=True) for _, w in synth.config_weights(cfg, 0)]
x = torch.from_numpy(synth.activations_f32(2560, N, 5999)).to(dev)
def ev():
    return torch.cuda.Event(enable_timing=True)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = ev(), ev(); a.record(); r = fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), r
tq, (xq, xs) = t(lambda: v.quantize(x))
tqkv, qkv = t(lambda: L[0](xq, xs))
tq1, (q1, s1) = t(lambda: v.quantize(qkv[:2560]))
to, o = t(lambda: L[1](q1, s1))
tq2, (u, su) = t(lambda: v.quantize(o))
tg, gate = t(lambda: L[2](u, su))
tu, up = t(lambda: L[3](u, su))
tq3, (hq, hs) = t(lambda: v.quantize(gate, up))
td, d = t(lambda: L[4](hq, hs))
tq4, _ = t(lambda: v.quantize(d))
print(f"quantize x {tq:.1f}us  qkv {tqkv:.1f}  Q(qkv) {tq1:.1f}  o {to:.1f}  Q(o) {tq2:.1f}  gate {tg:.1f}  up {tu:.1f}  Q(g*u) {tq3:.1f}  down {td:.1f}  Q(d) {tq4:.1f}")
print("layer total us", tqkv + tq1 + to + tq2 + tg + tu + tq3 + td + tq4, " quantize share", (tq1+tq2+tq3+tq4)/(tqkv + tq1 + to + tq2 + tg + tu + tq3 + td + tq4))
