"""A/B of the bench step's launch schedule over rotating inputs (> 2x L2):
seq = K3(i) -> K1(i) on one stream (the bench's graph); pipe = K3(i+1) on a
second stream overlapping K1(i) (double-buffered codes/scales), optionally
with a forced K3 cluster size (VLUT_QCL).  Checks every output against the
sequential schedule.   python scripts/pipeline_probe.py [steps]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_06443_b200 as v  # noqa: E402
from paper_2512_06443_b200 import synth  # noqa: E402

K_STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 200
M, K, N, g = 6912, 2560, 256, 4
dev = torch.device("cuda")
W = torch.from_numpy(synth.ternary_weights(M, K, 1, 0.4)).to(dev)
pw0 = v.pack_weights_device(W, g)
per = pw0.nbytes + K * N * 4 + M * N * 4
R = max(2, -(-2 * (126 << 20) // per))
pws = [pw0] + [v.pack_weights_device(W, g) for _ in range(R - 1)]
xs = [torch.randn(K, N, device=dev) for _ in range(R)]
outs = [torch.empty(M, N, device=dev) for _ in range(R)]
ws = v.workspace(dev)
qb = [torch.empty(K, N, dtype=torch.int8, device=dev) for _ in range(2)]
sb = [torch.empty(N, device=dev) for _ in range(2)]
torch.cuda.synchronize()


def seq():
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for i in range(K_STEPS):
            j = i % R
            v.quantize(xs[j], q=qb[0], scale=sb[0])
            v.mpgemm_ws(pws[j], qb[0], sb[0], synth.W_SCALE, out=outs[j], ws=ws)
    return gr


def pipe(prio):
    gr = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(priority=prio)
    evq = [torch.cuda.Event() for _ in range(K_STEPS)]
    evk = [torch.cuda.Event() for _ in range(K_STEPS)]
    with torch.cuda.graph(gr):
        cs = torch.cuda.current_stream()
        side.wait_stream(cs)
        for i in range(K_STEPS):
            j, b = i % R, i % 2
            with torch.cuda.stream(side):
                if i >= 2:
                    side.wait_event(evk[i - 2])
                v.quantize(xs[j], q=qb[b], scale=sb[b], stream=side)
                evq[i].record(side)
            cs.wait_event(evq[i])
            v.mpgemm_ws(pws[j], qb[b], sb[b], synth.W_SCALE, out=outs[j], ws=ws)
            evk[i].record(cs)
        cs.wait_stream(side)
    return gr


def timed(gr, reps=3):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / K_STEPS)
    return ts


g0 = seq()
g0.replay(); torch.cuda.synchronize()
ref = [o.clone() for o in outs]
print(f"seq            : {['%.2f' % t for t in timed(g0)]} us/step", flush=True)
for qcl in ["", "1", "2", "4"]:
    for prio in (0, -1):
        if qcl:
            os.environ["VLUT_QCL"] = qcl
        else:
            os.environ.pop("VLUT_QCL", None)
        gp = pipe(prio)
        for o in outs:
            o.fill_(float("nan"))
        gp.replay(); torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in zip(outs, ref))
        print(f"pipe qcl={qcl or 'auto'} prio={prio}: {['%.2f' % t for t in timed(gp)]} us/step  same={same}",
              flush=True)
os.environ.pop("VLUT_QCL", None)
print(f"seq again      : {['%.2f' % t for t in timed(g0)]} us/step")
