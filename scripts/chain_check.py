"""Config-5 chain timings (development tool): plain, fused (f1) and
overlapped f1 (token chunks, exchange on a side stream), N = 2048, L layers."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402
from paper_2512_06443_b200.sharded import LayerChain, RowShardedLinear  # noqa: E402
L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dev = torch.device("cuda")
cfg = synth.CONFIGS[5]
N = 2048
layers = [[RowShardedLinear(w, 4, synth.W_SCALE, device=dev, device_pack=True)
           for _, w in synth.config_weights(cfg, l)] for l in range(L)]
x = torch.from_numpy(synth.activations_f32(2560, N, 5999)).to(dev)
xq, xs = v.quantize(x)
for name, ch in (("plain", LayerChain(layers)), ("fused", LayerChain(layers, fused=True)),
                 ("chunks2", LayerChain(layers, fused=True, chunks=2)),
                 ("chunks4", LayerChain(layers, fused=True, chunks=4))):
    ch(xq, xs); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(); ch(xq, xs); b.record(); torch.cuda.synchronize()
        ts.append((a.elapsed_time(b), (time.perf_counter() - t0) * 1e3))
    print(name, [f"{t:.2f}/{w:.2f}" for t, w in ts], flush=True)
