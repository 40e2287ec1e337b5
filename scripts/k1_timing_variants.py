import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2512_06443_b200 as v
from paper_2512_06443_b200 import synth
dev = torch.device("cuda")
M, K, N, g = 6912, 2560, 256, 4
W = synth.ternary_weights(M, K, 2000, 0.4)
pw = v.pack_weights_device(torch.from_numpy(W).to(dev), g)
x = torch.from_numpy(synth.activations_f32(K, N, 2001)).to(dev)
q = torch.empty((K, N), dtype=torch.int8, device=dev); s = torch.empty((N,), dtype=torch.float32, device=dev)
out = torch.empty((M, N), device=dev); ws = v.workspace(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream()
for _ in range(20):
    v.quantize(x, q=q, scale=s, stream=st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st)
torch.cuda.synchronize()
def run(mode, n=200):
    ts = []
    for i in range(n):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        if mode == "bench":
            flush.zero_(); e[0].record(st); v.quantize(x, q=q, scale=s, stream=st); e[1].record(st)
            flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "sync_first":
            torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k3_then_flush_sync":
            v.quantize(x, q=q, scale=s, stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k1_then_flush":
            v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k3_other_q":
            v.quantize(x, q=q2, scale=s2, stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k3_q_sleep":
            v.quantize(x, q=q, scale=s, stream=st); torch.cuda.synchronize(); torch.cuda._sleep(2000000); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "qcopy_then_flush":
            q.copy_(q3); s.copy_(s3); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k1c8_then_flush":
            v.mpgemm_ex(pw, q, s, 0.02, out=out, plan=v.LaunchPlan(12, 8), stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k1c4_then_flush":
            v.mpgemm_ex(pw, q, s, 0.02, out=out, plan=v.LaunchPlan(12, 4), stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k1c1_then_flush":
            v.mpgemm_ex(pw, q, s, 0.02, out=out, plan=v.LaunchPlan(12, 1), stream=st); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "small_then_flush":
            small.add_(1.0); torch.cuda.synchronize(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k1_sleep_flush":
            v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); torch.cuda.synchronize(); time.sleep(0.0002); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k3_noflush_k1":
            v.quantize(x, q=q, scale=s, stream=st); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "k3_pdl_step":
            flush.zero_(); e[2].record(st); v.quantize(x, q=q, scale=s, stream=st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        elif mode == "double_flush":
            flush.zero_(); flush.zero_(); e[2].record(st); v.mpgemm_ws(pw, q, s, 0.02, out=out, ws=ws, stream=st); e[3].record(st)
        torch.cuda.synchronize()
        ts.append(e[2].elapsed_time(e[3]) * 1e3)
    ts = np.array(ts)
    print(mode, "mean %.2f med %.2f min %.2f max %.2f" % (ts.mean(), np.median(ts), ts.min(), ts.max()))
q2 = torch.empty_like(q); s2 = torch.empty_like(s); q3 = q.clone(); s3 = s.clone()
import time
small = torch.zeros(1024, device=dev)
for m in ("sync_first", "k3_then_flush_sync", "small_then_flush", "k1_sleep_flush", "k1_then_flush", "k3_noflush_k1", "k3_pdl_step"):
    run(m)
