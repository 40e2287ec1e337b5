"""Row-parallel ternary linears and the config-5 layer chain (e).

North star: "Linear layers are sharded by output rows across 1/2/4/8 GPUs of
one 8xB200 box, with an NCCL all-gather of outputs over NVLink."  Output row m
depends only on weight row m and all of A, so rank r of G packs the contiguous
rows [r*Mp, (r+1)*Mp) (Mp = ceil(M/G); the last shard may be short), computes
its fp32 shard with ``vlut_mpgemm`` and ``all_gather_into_tensor`` assembles
the token-contiguous [M][N] output on every rank.  The gathered result is
bit-identical to the 1-GPU result (each output element is computed by exactly
one rank with the same kernel arithmetic).

PyTorch is plumbing here (device memory, streams, process groups).  The
per-shard compute defaults to the CUDA path; tests inject other callables
(e.g. the CPU oracle under gloo) to check the partition / gather logic on CPU.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

__all__ = ["shard_rows", "RowShardedLinear", "LayerChain", "CHAIN_Q_ROWS", "PeerOutputs",
           "Chunk", "split_tokens", "join_tokens"]


def shard_rows(M: int, world: int, rank: int) -> Tuple[int, int, int]:
    """(row0, row1, Mp): rank's contiguous row range and the padded shard size."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    Mp = -(-M // world)
    r0 = min(M, rank * Mp)
    r1 = min(M, r0 + Mp)
    return r0, r1, Mp


def _dist():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist
    return None


class PeerOutputs:
    """Symmetric fp32 [M][N] output buffers on every rank for the fused
    all-gather (``vlut_mpgemm_allgather``): allocated with torch symmetric
    memory (CUDA IPC mappings; NVLink P2P on one NVSwitch box), so each rank
    holds device pointers to every peer's buffer and its K1 epilogue stores
    its row shard into all of them.  Two buffers per N alternate between
    calls: a rank can only be one call ahead of a peer (every call ends with a
    cross-GPU barrier on the stream), so it never overwrites a buffer a peer
    is still reading.  Plumbing only -- the stores are the kernel's.

    mode "multicast" (NVLS, when the device supports multicast objects): the
    kernel stores each unit ONCE to the buffer's multicast address and the
    NVSwitch replicates it into every rank's copy (the local one included);
    mode "unicast": one store to the local copy plus one per peer."""

    def __init__(self, group=None, mode: str = "auto"):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.symm = symm_mem
        self.group = group or dist.group.WORLD
        self.rank = dist.get_rank(self.group)
        self.world = dist.get_world_size(self.group)
        self.mode = mode
        self._bufs = {}
        self._turn = {}

    def _multicast_ok(self, device) -> bool:
        if self.mode == "unicast":
            return False
        try:
            from torch._C._distributed_c10d import _SymmetricMemory
            from torch._C._autograd import DeviceType
            import torch
            idx = torch.device(device).index
            if idx is None:
                idx = torch.cuda.current_device()
            return bool(_SymmetricMemory.has_multicast_support(DeviceType.CUDA, idx))
        except Exception:
            return False

    def get(self, M: int, N: int, device):
        """(buffer [M][N] fp32, store target (device pointer), [peer device
        pointers], barrier) for this call: the kernel stores to the target
        (the local copy, or the multicast address) and to each peer."""
        key = (M, N)
        if key not in self._bufs:
            import torch
            mc = self._multicast_ok(device)
            pair = []
            for _ in range(2):
                t = self.symm.empty((M, N), dtype=torch.float32, device=device)
                h = self.symm.rendezvous(t, self.group)
                mptr = int(getattr(h, "multicast_ptr", 0) or 0) if mc else 0
                if mptr:
                    target, peers = mptr, []
                else:
                    target = t.data_ptr()
                    peers = [int(h.buffer_ptrs[r]) for r in range(self.world) if r != self.rank]
                pair.append((t, target, peers, h))
            self._bufs[key] = pair
            self._turn[key] = 0
        i = self._turn[key]
        self._turn[key] = 1 - i
        t, target, peers, h = self._bufs[key][i]
        return t, target, peers, (lambda: h.barrier(channel=0))

    def multicast(self, M: int, N: int) -> bool:
        """True if get(M, N, ...) hands out a multicast address (store it
        with mpgemm_allgather(..., multicast=True))."""
        pair = self._bufs.get((M, N))
        return bool(pair) and pair[0][1] != pair[0][0].data_ptr()

    def transport(self, M: int, N: int, device) -> str:
        _, target, peers, _ = self.get(M, N, device)
        self.get(M, N, device)  # restore the alternation
        return "unicast" if (peers or self.world == 1) and target else "multicast"


class RowShardedLinear:
    """One ternary linear, row-sharded over the default process group.

    W: int8 trits [M][K] (host, full matrix; each rank keeps only its rows),
    g: 4 or 5, w_scale: per-tensor scale.  ``compute(shard, A, a_scale, out)``
    fills ``out`` ([rows][N] fp32) -- default: the CUDA kernel.
    """

    def __init__(self, W, g: int, w_scale: float, device=None,
                 compute: Optional[Callable] = None, pack: Optional[Callable] = None,
                 device_pack: bool = False, fused: Optional[Callable] = None,
                 quantize_amax: Optional[Callable] = None, peers: Optional[PeerOutputs] = None):
        dist = _dist()
        self.world = dist.get_world_size() if dist else 1
        self.rank = dist.get_rank() if dist else 0
        self.M, self.K = W.shape
        self.g = g
        self.w_scale = float(w_scale)
        self.r0, self.r1, self.Mp = shard_rows(self.M, self.world, self.rank)
        self.rows = self.r1 - self.r0
        self.device = device
        W_r = W[self.r0:self.r1]
        if pack is not None:
            self.shard = pack(np.ascontiguousarray(W_r), g)
        elif not self.rows:
            self.shard = None
        elif device_pack:
            # upload the trits and pack on the GPU (large weights; no validation)
            import torch
            import paper_2512_06443_b200 as v
            wd = torch.as_tensor(W_r, device=device or "cuda").contiguous()
            self.shard = v.pack_weights_device(wd, g)
            torch.cuda.current_stream().synchronize()
            del wd
        else:
            import paper_2512_06443_b200 as v
            self.shard = v.pack_weights(np.ascontiguousarray(W_r), g, device=device)
        self.peers = peers  # fused all-gather buffers (None: NCCL all_gather_into_tensor)
        self._compute = compute or self._cuda_compute
        self._fused = fused or self._cuda_fused
        if quantize_amax is None:
            def quantize_amax(x, amax, q, scale):
                import paper_2512_06443_b200 as v
                v.quantize_amax(x, amax, q=q, scale=scale)
        self._quantize_amax = quantize_amax

    def _cuda_fused(self, shard, A, a_scale, out, mul_in, amax, amax_rows):
        import paper_2512_06443_b200 as v
        v.mpgemm_fused(shard, A, a_scale, self.w_scale, out=out, mul_in=mul_in, amax=amax,
                       amax_rows=amax_rows, ws=v.workspace(A.device))

    def local(self, A, a_scale):
        """This rank's fp32 rows [rows][N] (no gather)."""
        import torch
        out = torch.empty((self.rows, A.shape[1]), dtype=torch.float32, device=A.device)
        if self.rows:
            self._compute(self.shard, A, a_scale, out)
        return out

    def forward_quantized(self, A, a_scale, q_rows: Optional[int] = None, mul_in=None):
        """Fused re-quantization (f1): the GEMM epilogue multiplies by mul_in
        (this rank's rows, optional) and produces per-token |out| maxima over
        the first q_rows global rows; the maxima are all-reduced (MAX) across
        ranks, each rank quantizes its own rows, and the int8 shards (4x fewer
        bytes than fp32) are all-gathered.  Returns (q [q_rows][N] int8,
        scale [N] fp32) on every rank -- bit-identical to quantizing the
        gathered fp32 output."""
        local, amax = self._fused_local(A, a_scale, q_rows, mul_in)
        return self._finish_quantized(local, amax, A.shape[1], q_rows)

    def _fused_local(self, A, a_scale, q_rows, mul_in):
        """This rank's fp32 rows (epilogue: * mul_in) and the per-token maxima
        of its rows below q_rows (int32 [N], float bits)."""
        import torch
        N = A.shape[1]
        dev = A.device
        q_rows = self.M if q_rows is None else q_rows
        amax = torch.zeros((N,), dtype=torch.int32, device=dev)
        local = torch.empty((max(self.rows, 1), N), dtype=torch.float32, device=dev)[:self.rows]
        arows = max(0, min(self.rows, q_rows - self.r0))
        if self.rows:
            self._fused(self.shard, A, a_scale, local, mul_in, amax, arows)
        return local, amax

    def _finish_quantized(self, local, amax, N, q_rows):
        """MAX all-reduce of the maxima, quantize this rank's rows with them,
        all-gather the int8 shards: (q [q_rows][N], scale [N])."""
        import torch
        dev = local.device
        q_rows = self.M if q_rows is None else q_rows
        d = _dist()
        if d is not None and self.world > 1:
            d.all_reduce(amax, op=d.ReduceOp.MAX)
        q_loc = torch.empty((self.Mp, N), dtype=torch.int8, device=dev)
        scale = torch.empty((N,), dtype=torch.float32, device=dev)
        if self.rows:
            self._quantize_amax(local, amax, q_loc[:self.rows], scale)
        else:
            self._quantize_amax(torch.zeros((1, N), dtype=torch.float32, device=dev), amax,
                                torch.empty((1, N), dtype=torch.int8, device=dev), scale)
        if self.world == 1:
            return q_loc[:q_rows], scale
        if self.rows < self.Mp:
            q_loc[self.rows:].zero_()
        full = torch.empty((self.Mp * self.world, N), dtype=torch.int8, device=dev)
        d.all_gather_into_tensor(full, q_loc)
        return full[:q_rows], scale

    def forward_quantized_chunks(self, chunks, q_rows: Optional[int] = None, mul_ins=None,
                                 comm=None):
        """f1 overlapped with compute: the tokens are split into chunks
        (per-token quantization makes them independent) and, per chunk, the
        fused mpGeMM runs on the compute (current) stream while the previous
        chunks' MAX all-reduce, quantization and int8 all-gather run on the
        `comm` stream -- the exchange of chunk i overlaps the compute of chunk
        i+1 (and of the next linear's earlier chunks).

        chunks: list of Chunk; mul_ins: per-chunk local rows [rows][Nc] or
        None.  Returns a list of Chunk (q [q_rows][Nc], scale [Nc], ready
        event on `comm`).  comm None (CPU / gloo): sequential, same values."""
        out = []
        for c, ch in enumerate(chunks):
            A, s = ch.wait()
            local, amax = self._fused_local(A, s, q_rows, None if mul_ins is None else mul_ins[c])
            if comm is None:
                q, sc = self._finish_quantized(local, amax, A.shape[1], q_rows)
                out.append(Chunk(q, sc))
                continue
            import torch
            cur = torch.cuda.current_stream(A.device)
            done = torch.cuda.Event()
            done.record(cur)
            with torch.cuda.stream(comm):
                comm.wait_event(done)
                # produced on `cur`, consumed on `comm`: keep the blocks alive
                local.record_stream(comm)
                amax.record_stream(comm)
                q, sc = self._finish_quantized(local, amax, A.shape[1], q_rows)
                ready = torch.cuda.Event()
                ready.record(comm)
            out.append(Chunk(q, sc, ready))
        return out

    def local_chunks(self, chunks):
        """This rank's fp32 rows per chunk (no gather; config 5's gate rows)."""
        return [self.local(*ch.wait()) for ch in chunks]

    def _cuda_compute(self, shard, A, a_scale, out):
        # workspace path: the planner may pick the stream-K schedule
        import paper_2512_06443_b200 as v
        v.mpgemm_ws(shard, A, a_scale, self.w_scale, out=out)

    def __call__(self, A, a_scale, out=None):
        """A: int8 [K][N] (replicated on every rank), a_scale: fp32 [N] ->
        fp32 [M][N] on every rank."""
        import torch
        N = A.shape[1]
        dev = A.device
        if self.world == 1:
            if out is None:
                out = torch.empty((self.M, N), dtype=torch.float32, device=dev)
            if self.rows:
                self._compute(self.shard, A, a_scale, out)
            return out
        if self.peers is not None:
            # fused all-gather: the K1 epilogue stores this rank's rows into
            # every rank's copy over NVLink; one cross-GPU barrier completes it
            import paper_2512_06443_b200 as v
            buf, target, peer_ptrs, barrier = self.peers.get(self.M, N, dev)
            if self.rows:
                v.mpgemm_allgather(self.shard, A, a_scale, self.w_scale, target, self.r0, peer_ptrs,
                                   multicast=self.peers.multicast(self.M, N))
            barrier()
            if out is not None:
                out.copy_(buf)
                return out
            return buf
        local = torch.empty((self.Mp, N), dtype=torch.float32, device=dev)
        if self.rows:
            self._compute(self.shard, A, a_scale, local[:self.rows])
        if self.rows < self.Mp:
            local[self.rows:].zero_()
        full = torch.empty((self.Mp * self.world, N), dtype=torch.float32, device=dev)
        _dist().all_gather_into_tensor(full, local)
        res = full[:self.M]
        if out is not None:
            out.copy_(res)
            return out
        return res


class Chunk:
    """A token chunk of the chain's int8 activations: q [K][Nc], scale [Nc]
    and, when produced on a side stream, the event that marks them ready."""

    __slots__ = ("q", "scale", "ready")

    def __init__(self, q, scale, ready=None):
        self.q, self.scale, self.ready = q, scale, ready

    def wait(self):
        """(q, scale), with the current stream ordered after their producer."""
        if self.ready is not None:
            import torch
            cur = torch.cuda.current_stream(self.q.device)
            cur.wait_event(self.ready)
            self.q.record_stream(cur)
            self.scale.record_stream(cur)
        return self.q, self.scale


def split_tokens(q, scale, n_chunks: int):
    """Split [K][N] int8 activations (+ scale [N]) into contiguous token chunks."""
    N = q.shape[1]
    bounds = [N * i // n_chunks for i in range(n_chunks + 1)]
    return [Chunk(q[:, a:b].contiguous(), scale[a:b].contiguous())
            for a, b in zip(bounds, bounds[1:]) if b > a]


def join_tokens(chunks):
    """Concatenate chunks back into ([K][N] int8, [N] fp32)."""
    import torch
    pairs = [ch.wait() for ch in chunks]
    return torch.cat([p[0] for p in pairs], 1), torch.cat([p[1] for p in pairs])


# Config 5 glue (reading c14): per layer
#   qkv = L_qkv(x); o = L_o(Q(qkv[0:2560])); u = Q(o);
#   h = L_gate(u) * L_up(u); x' = Q(L_down(Q(h)))
CHAIN_Q_ROWS = 2560


class LayerChain:
    """The 30-layer BitNet-2B-shaped prefill of ternary linears (config 5).

    layers: list of 5-tuples of RowShardedLinear (qkv, o, gate, up, down).
    quantize(x, y=None) -> (q, scale): default the CUDA quantizer (K3).
    """

    def __init__(self, layers: Sequence[Sequence[RowShardedLinear]], q_rows: int = CHAIN_Q_ROWS,
                 quantize: Optional[Callable] = None, fused: bool = False, chunks: int = 1,
                 comm_stream=None):
        """chunks > 1 (with fused): the f1 chain overlapped with compute --
        tokens split into `chunks` groups, each linear's exchange of chunk i
        on `comm_stream` while chunk i+1 computes (comm_stream None on a GPU:
        a new side stream; on CPU: sequential)."""
        self.fused = fused
        self.chunks = chunks
        self.comm = comm_stream
        self.layers = [tuple(l) for l in layers]
        self.q_rows = q_rows
        if quantize is None:
            import paper_2512_06443_b200 as v
            quantize = v.quantize
        self.quantize = quantize

    def layer_fused(self, l, xq, xs):
        """Same layer with fused re-quantization (f1): no separate amax pass,
        int8 gathers, and gate (.) up fused into the up-projection epilogue
        (the gate rows never leave their rank)."""
        L_qkv, L_o, L_gate, L_up, L_down = self.layers[l]
        q1, s1 = L_qkv.forward_quantized(xq, xs, q_rows=self.q_rows)
        u, su = L_o.forward_quantized(q1, s1)
        gate = L_gate.local(u, su)
        hq, hs = L_up.forward_quantized(u, su, mul_in=gate)
        return L_down.forward_quantized(hq, hs)

    def layer_chunked(self, l, chunks):
        """layer_fused over token chunks, exchange overlapped with compute."""
        L_qkv, L_o, L_gate, L_up, L_down = self.layers[l]
        c1 = L_qkv.forward_quantized_chunks(chunks, q_rows=self.q_rows, comm=self.comm)
        c2 = L_o.forward_quantized_chunks(c1, comm=self.comm)
        gates = L_gate.local_chunks(c2)
        c3 = L_up.forward_quantized_chunks(c2, mul_ins=gates, comm=self.comm)
        return L_down.forward_quantized_chunks(c3, comm=self.comm)

    def layer(self, l, xq, xs):
        if self.fused:
            return self.layer_fused(l, xq, xs)
        L_qkv, L_o, L_gate, L_up, L_down = self.layers[l]
        qkv = L_qkv(xq, xs)
        q1, s1 = self.quantize(qkv[:self.q_rows])
        o = L_o(q1, s1)
        u, su = self.quantize(o)
        gate = L_gate(u, su)
        up = L_up(u, su)
        hq, hs = self.quantize(gate, up)
        d = L_down(hq, hs)
        return self.quantize(d)

    def __call__(self, xq, xs, n_layers: Optional[int] = None):
        n = len(self.layers) if n_layers is None else n_layers
        if self.fused and self.chunks > 1:
            if self.comm is None and xq.is_cuda:
                import torch
                self.comm = torch.cuda.Stream(xq.device)
            ch = split_tokens(xq, xs, self.chunks)
            for l in range(n):
                ch = self.layer_chunked(l, ch)
            return join_tokens(ch)
        for l in range(n):
            xq, xs = self.layer(l, xq, xs)
        return xq, xs
