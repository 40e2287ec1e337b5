"""Host-resident batches through the Vec-LUT linear with copy/compute overlap.

A serving loop feeds activations from pinned host memory and reads results
back.  Run serially, one step is H2D (fp32 x) + quantize (K3) + mpGeMM (K1/K2)
+ D2H (fp32 out), and at BASELINE.json configs[1] the two PCIe copies take
longer than the kernels.  ``HostPipeline`` keeps ``depth`` device buffer
slots and three CUDA streams (H2D copy engine, compute, D2H copy engine)
chained by events, so step i+1's input upload and step i-1's result download
overlap step i's kernels (both copy directions run concurrently on separate
copy engines).  Every kernel is still the C-ABI path (``quantize``,
``mpgemm_ws``); torch only provides memory, streams and events.
"""
from __future__ import annotations

from typing import Callable, Optional

import paper_2512_06443_b200 as v


class HostPipeline:
    def __init__(self, W: "v.PackedWeights", w_scale: float, K: int, N: int, device,
                 depth: int = 2, ws=None, post: Optional[Callable] = None):
        """W: packed weights ([M][K]); per step x is fp32 [K][N] (token axis
        contiguous), the result fp32 [M][N].  ``post(out, stream, slot)``
        (optional) runs on the compute stream after the mpGeMM (e.g. an
        all-gather of row shards into a per-slot buffer) and returns the
        tensor to download."""
        import torch
        self.torch = torch
        self.W, self.w_scale, self.K, self.N = W, float(w_scale), K, N
        self.depth = depth
        self.dev = torch.device(device)
        self.ws = ws if ws is not None else v.workspace(self.dev)
        self.post = post
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.x = [torch.empty((K, N), dtype=torch.float32, device=self.dev) for _ in range(depth)]
        self.out = [torch.empty((W.M, N), dtype=torch.float32, device=self.dev)
                    for _ in range(depth)]
        self.q = torch.empty((K, N), dtype=torch.int8, device=self.dev)
        self.sc = torch.empty((N,), dtype=torch.float32, device=self.dev)
        ev = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
        self.ev_in = [ev() for _ in range(depth)]     # x slot uploaded
        self.ev_xfree = [ev() for _ in range(depth)]  # x slot consumed by the kernels
        self.ev_done = [ev() for _ in range(depth)]   # out slot written
        self.ev_ofree = [ev() for _ in range(depth)]  # out slot downloaded
        self.i = 0

    def submit(self, x_pin, o_pin) -> None:
        """Enqueue one step: x_pin (pinned fp32 [K][N]) -> o_pin (pinned fp32
        [M][N], or the rows ``result()`` selects).  Asynchronous."""
        slot = self.i % self.depth
        first = self.i < self.depth
        with self.torch.cuda.stream(self.s_in):
            if not first:
                self.s_in.wait_event(self.ev_xfree[slot])
            self.x[slot].copy_(x_pin, non_blocking=True)
            self.ev_in[slot].record(self.s_in)
        with self.torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(self.ev_in[slot])
            if not first:
                self.s_cmp.wait_event(self.ev_ofree[slot])
            v.quantize(self.x[slot], q=self.q, scale=self.sc, stream=self.s_cmp)
            self.ev_xfree[slot].record(self.s_cmp)
            v.mpgemm_ws(self.W, self.q, self.sc, self.w_scale, out=self.out[slot], ws=self.ws,
                        stream=self.s_cmp)
            res = self.out[slot]
            if self.post is not None:
                res = self.post(res, self.s_cmp, slot)
            self.ev_done[slot].record(self.s_cmp)
        with self.torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_done[slot])
            o_pin.copy_(res, non_blocking=True)
            self.ev_ofree[slot].record(self.s_out)
        self.i += 1

    def synchronize(self) -> None:
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.synchronize()


class BatchPipeline:
    """Independent device-resident activation batches through one Vec-LUT
    linear, the quantizer of batch i+1 overlapping the mpGeMM of batch i.

    The mpGeMM grid leaves SMs free (configs[1]: K1-32 runs 144 CTAs, one per
    SM, on the 148), and the quantizer launched with one-CTA clusters
    (``quantize(..., cluster=1)``, vlut_quantize_ex) fits them, so on a second
    stream it runs under the mpGeMM instead of before it: the step costs the
    mpGeMM alone (profiles/r02_pipeline.txt; an 8-CTA cluster cannot be
    placed on the free SMs and waits for the mpGeMM).  Codes and scales are
    double-buffered: batch i's quantizer waits for the mpGeMM of batch i-2
    (the last reader of its buffer), batch i's mpGeMM for its quantizer.
    Results are bit-identical to quantize-then-mpGeMM on one stream.

    ``submit`` enqueues on the caller's current stream (the mpGeMMs) and the
    pipeline's side stream (the quantizers) and can be captured in a CUDA
    graph; ``join`` makes the current stream wait for the side stream.  An
    input x must already be complete on the side stream's timeline: written
    before the first ``submit`` on the current stream, or signalled by the
    ``ready`` event passed with it.
    """

    def __init__(self, W: "v.PackedWeights", w_scale: float, K: int, N: int, device, ws=None,
                 plan=None):
        import torch
        self.torch = torch
        self.W, self.w_scale, self.K, self.N = W, float(w_scale), K, N
        self.dev = torch.device(device)
        # one workspace (allocated here, outside any graph capture); the
        # mpGeMMs are chained by events, so it is never used by two at once
        self.ws = ws if ws is not None else v.workspace(self.dev)
        self.plan = plan
        self.side = torch.cuda.Stream(self.dev)
        self.q = [torch.empty((K, N), dtype=torch.int8, device=self.dev) for _ in range(2)]
        self.sc = [torch.empty((N,), dtype=torch.float32, device=self.dev) for _ in range(2)]
        self.ev_q = [torch.cuda.Event() for _ in range(2)]  # codes of buffer b written
        self.ev_k = [torch.cuda.Event() for _ in range(2)]  # codes of buffer b consumed
        self.i = 0

    def submit(self, x, out, W: "Optional[v.PackedWeights]" = None, ready=None) -> None:
        """x: fp32 [K][N] on the device; out: fp32 [M][N]; W: packed weights
        for this batch (default: the pipeline's)."""
        torch = self.torch
        b = self.i % 2
        cs = torch.cuda.current_stream(self.dev)
        if self.i == 0:
            self.side.wait_stream(cs)
        with torch.cuda.stream(self.side):
            if ready is not None:
                self.side.wait_event(ready)
            if self.i >= 2:
                self.side.wait_event(self.ev_k[b])
            v.quantize(x, q=self.q[b], scale=self.sc[b], stream=self.side, cluster=1)
            self.ev_q[b].record(self.side)
        cs.wait_event(self.ev_q[b])
        if self.i >= 1:
            cs.wait_event(self.ev_k[1 - b])  # the previous mpGeMM (same workspace), any stream
        v.mpgemm_ws(W if W is not None else self.W, self.q[b], self.sc[b], self.w_scale, out=out,
                    ws=self.ws, plan=self.plan, stream=cs)
        self.ev_k[b].record(cs)
        self.i += 1

    def reset(self) -> None:
        """Start a new sequence (e.g. before capturing one in a CUDA graph):
        the next submit forks the side stream from the current one again."""
        self.i = 0

    def join(self) -> None:
        self.torch.cuda.current_stream(self.dev).wait_stream(self.side)
