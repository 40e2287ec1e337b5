#!/usr/bin/env python
"""bench.py -- Vec-LUT ternary mpGeMM on B200: the driver's benchmark contract.

Workload (N=1 GPU): BASELINE.json configs[1], the BitNet-2B-shaped FFN-up
ternary linear, M=6912, K=2560, N=256 tokens, g=4, weights iid with
P(-1)=P(+1)=0.3, P(0)=0.4, per-tensor scale 0.02, activations N(0,1) fp32.
One step = one pass of the hot path over one batch: per-token int8 quantize
(a7, K3 kernel) -> fused Vec-LUT mpGeMM with fp32 dequant (a2-a6, K1 kernel)
[-> NCCL all-gather of row shards (a8) when --gpus > 1].  Weights are packed
once, offline (a1), before timing.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py re-launches
itself under torch.distributed.run with N ranks (one per GPU, 127.0.0.1
rendezvous); n_gpus reports the ranks that joined the process group.

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream
around each step's kernels; the L2 is flushed (256 MiB memset) between steps
outside those windows; the sum of per-step durations is the timed total, max
over ranks.  See DESIGN.md §Measurement.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2512_06443_b200 import synth  # noqa: E402

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT = 148
SMEM_BYTES_PER_CLK_SM = 128  # 32 banks x 4 B
SM_MAX_MHZ_FALLBACK = 1965.0
HBM_FALLBACK_GBS = 6650.0    # B200_PROFILING.md fallback



def plan_label(pl):
    """Kernel family and launch shape a LaunchPlan selects (vlut.h dispatch)."""
    if pl.slot:
        return f"K2 lane-slot tpw={pl.tpw} nw={pl.nw} splits={pl.splits}"
    fam = ("K1-32" if pl.n_cta == 32 else "K1") + ("-SK" if pl.streamk else "")
    return f"{fam} warps={pl.warps} m_cta={pl.m_cta} n_cta={pl.n_cta} splits={pl.splits}"

def load_peaks():
    try:
        with open(MEASURED_PEAKS) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK_GBS, "sm_max_mhz": SM_MAX_MHZ_FALLBACK}, "fallback"


# ------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, torch_dev):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self.ok = False
        self._stop = threading.Event()
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            # match the torch device to an NVML handle by UUID (the PCI-bus-id
            # lookup segfaults in this pynvml build)
            want = str(getattr(torch.cuda.get_device_properties(torch_dev), "uuid", "")).lower()
            self.h = None
            for i in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(h)
                u = (u.decode() if isinstance(u, bytes) else str(u)).lower()
                if want and want in u:
                    self.h = h
                    break
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(torch_dev.index or 0)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # keep benchmarking; report the absence
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(0.001)  # sparse: the sampler competes with the launch thread for the GIL

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    @staticmethod
    def merge(*samplers):
        """One summary over several sampling windows (timed steps + per-kernel
        passes): median SM clock over all samples, union of reasons."""
        ok = [c for c in samplers if c.ok]
        if not ok:
            return samplers[0].summary()
        smp = [x for c in ok for x in c.samples]
        reasons = 0
        for c in ok:
            reasons |= c.reasons
        rs = [name for bit, name in ClockSampler.REASONS.items() if reasons & bit and bit != 0x1]
        return {"sm_mhz": float(statistics.median(smp)) if smp else None,
                "sm_max_mhz": float(ok[0].max_mhz), "reasons": rs, "samples": len(smp),
                "windows": "timed steps + per-kernel passes"}

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit and bit != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": float(self.max_mhz), "reasons": rs, "samples": len(self.samples)}


# ------------------------------------------------------------------ helpers
def workload(args):
    cfg = synth.CONFIGS[2]
    lin = cfg.linears[0]
    return dict(cfg=cfg, M=lin.M, K=lin.K, N=cfg.N[0], g=cfg.g[0], p_zero=cfg.p_zero,
                w_seed=synth.weight_seed(cfg, 0, 0), x_seed=synth.act_seed(cfg, cfg.N[0]))


def bench_config(wl, world):
    """The `config` object of the JSON line -- identical for both arms (the
    driver compares them); implementation details go to other keys."""
    return {"workload": "configs[1]: BitNet-2B FFN-up ternary linear", "M": wl["M"],
            "K": wl["K"], "N": wl["N"], "g": wl["g"],
            "weights": "iid ternary P(0)=0.4 P(+-1)=0.3, seeded",
            "activations": "N(0,1) fp32, per-token int8 absmax quantized",
            "step": "per-token int8 quantize + ternary mpGeMM + fp32 dequant"
                    + (" + all-gather of output row shards" if world > 1 else ""),
            "parallelism": f"row-shard M over {world} GPU(s)" if world > 1 else "single GPU",
            "l2": ("inputs larger than L2: the K timed steps rotate over copies of the packed "
                   "weights, fp32 activations and outputs totalling > 2x the 126 MB L2, run "
                   "back to back (one CUDA graph of the K steps, events around it)" if world == 1
                   else "flushed between steps (256 MiB memset outside each step's event window)")}


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def maybe_spawn(args):
    """--gpus N > 1 without a torch.distributed launcher: re-run this script
    under torch.distributed.run with N ranks and return its exit code (rank 0
    prints the JSON line).  None when no spawn is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def comm_check(dist, dev):
    """The communicator every rank joined: its size and one all-reduce over
    it (sum of ones == world); logged to stderr and put in the JSON line."""
    import torch
    world = dist.get_world_size()
    t = torch.ones(1, device=dev)
    dist.all_reduce(t)
    ok = int(t.item()) == world
    print(f"[rank {dist.get_rank()}] {dist.get_backend()} communicator: nranks={world} "
          f"all_reduce_ok={ok}", file=sys.stderr, flush=True)
    return {"backend": dist.get_backend(), "nranks": world, "all_reduce_ok": ok}


def plumbing_main(args):
    """CPU check of the multi-rank bench plumbing (-m "not gpu" tests): the
    spawn, process-group join, row sharding with padding, the all-gather and
    the max-over-ranks timing, over gloo.  The per-shard compute, quantizer
    and reference are injected from a TEST module (args.plumbing, a file
    under tests/): bench.py itself computes nothing here, and the line says
    it is a plumbing check, not a measurement."""
    import importlib.util
    import torch
    import torch.distributed as dist
    from paper_2512_06443_b200.sharded import RowShardedLinear
    path = os.path.abspath(args.plumbing)
    if os.path.basename(os.path.dirname(path)) != "tests":
        raise SystemExit("--plumbing takes a module under tests/")
    spec = importlib.util.spec_from_file_location("bench_plumbing_hooks", path)
    hooks = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(hooks)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("gloo")
        world = dist.get_world_size()
    rank = dist.get_rank() if world > 1 else 0
    comm = comm_check(dist, torch.device("cpu")) if world > 1 else None
    M, K, N, g = 1001, 256, 32, 4  # M odd: the last shard is padded
    W = synth.ternary_weights(M, K, 2000, 0.4)
    x = synth.activations_f32(K, N, 2100)
    q, s = hooks.quantize(x)
    lin = RowShardedLinear(W, g, synth.W_SCALE, compute=hooks.compute(synth.W_SCALE),
                           pack=lambda w, g_: w)
    for _ in range(args.warmup):
        out = lin(q, s)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = lin(q, s)
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t[0])
    exact = bool(np.array_equal(out.numpy().view(np.int32),
                                hooks.reference(W, q, s, synth.W_SCALE).view(np.int32)))
    if world > 1:
        e = torch.tensor([1 if exact else 0])
        dist.all_reduce(e, op=dist.ReduceOp.MIN)
        exact = bool(e.item())
    if rank == 0:
        print(json.dumps({"impl": "plumbing-test", "metric": "plumbing check (not a measurement)",
                          "value": None, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "comm": comm,
                          "shard_rows": [list(map(int, sharded_rows(M, world, r)))
                                         for r in range(world)],
                          "gathered_equals_reference": exact,
                          "seconds_max_over_ranks": el}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0 if exact else 1


def sharded_rows(M, world, rank):
    from paper_2512_06443_b200.sharded import shard_rows
    return shard_rows(M, world, rank)


def algorithmic(M, K, N, g):
    lookups = M * (K // g) * N
    return dict(lookups=lookups, smem_bytes=2 * lookups,
                hbm_bytes=M * K // g + K * N + 4 * N + 4 * M * N, dense_ops=2 * M * K * N)


# ------------------------------------------------------------------ CPU oracle leg
def oracle_pipeline_rows(W, x, m0, m1, w_scale):
    """The oracle's step on rows [m0, m1): quantize (all tokens) -> int32 dot
    products -> fp32 dequant.  Test infrastructure, timed as the baseline."""
    import oracle
    q, s = oracle.quantize(x)
    acc = np.zeros((W.shape[0], x.shape[1]), np.int32)
    oracle.gemm_i32_rows(W, q, m0, m1, acc)
    return oracle.dequant_f32(acc[m0:m1], s, w_scale)


def cpu_baseline(W, x, N, budget_s=12.0, min_rows=32):
    import oracle
    oracle.build()
    M = W.shape[0]
    t0 = time.perf_counter()
    oracle_pipeline_rows(W, x, 0, min_rows, synth.W_SCALE)
    t_probe = time.perf_counter() - t0
    per_row = t_probe / min_rows
    rows = int(min(M, max(min_rows, budget_s / max(per_row, 1e-9))))
    t0 = time.perf_counter()
    done = 0
    reps = 0
    while True:
        oracle_pipeline_rows(W, x, 0, rows, synth.W_SCALE)
        done += rows
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or reps >= 50:
            break
    tok_s = N * (done / M) / el
    return {"value": tok_s, "unit": "tokens/s", "cores": oracle.num_threads(), "kind": "oracle",
            "omp_num_threads": oracle.omp_threads_env(), "build": " ".join(oracle.FLAGS),
            "sample": f"oracle quantize+int32 dot products+fp32 dequant on rows [0,{rows}) of "
                      f"the {M}-row workload, {reps} pass(es), {el:.1f} s; tokens/s scaled by "
                      f"rows/M", "seconds": el}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(args)
    M, K, N, g = wl["M"], wl["K"], wl["N"], wl["g"]
    W = synth.ternary_weights(M, K, wl["w_seed"], wl["p_zero"])
    x = synth.activations_f32(K, N, wl["x_seed"])
    import oracle
    oracle.build()
    # each step is the whole workload (all M rows) when the whole run fits
    # ~2.5 minutes, else a row sample sized to fit (scaled by M / rows)
    t0 = time.perf_counter()
    oracle_pipeline_rows(W, x, 0, 32, synth.W_SCALE)
    per_row = (time.perf_counter() - t0) / 32
    total_steps = args.steps + args.warmup
    step_budget = 150.0 / max(total_steps, 1)
    rows = int(min(M, max(8, step_budget / max(per_row, 1e-9))))
    for _ in range(args.warmup):
        oracle_pipeline_rows(W, x, 0, rows, synth.W_SCALE)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_pipeline_rows(W, x, 0, rows, synth.W_SCALE)
    el = time.perf_counter() - t0
    sec_per_full_step = el / args.steps * (M / rows)
    val = N / sec_per_full_step
    sample = ("each step: the whole workload (all rows)" if rows == M else
              f"each step: rows [0,{rows}) of {M}, time scaled by M/rows")
    line = {
        "impl": "reference", "metric": "ternary Vec-LUT mpGeMM tokens/s (configs[1])",
        "value": val, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec_per_full_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": bench_config(wl, args.gpus),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "kind": "oracle",
                         "cores": oracle.num_threads(),
                         "omp_num_threads": oracle.omp_threads_env(),
                         "build": " ".join(oracle.FLAGS),
                         "sample": "oracle quantize + int32 dot products + fp32 dequant; "
                                   + sample},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def vlut_launches_per_step(v, plan):
    """Our kernels per timed step: K3 quantize + the mpGeMM launch(es)."""
    return 1 + int(v.lib().vlut_launches_per_mpgemm())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="vlut", choices=["vlut", "reference"])
    ap.add_argument("--gather", default="p2p", choices=["p2p", "nccl"],
                    help="N>1: fused all-gather in the K1 epilogue (NVLink peer stores into "
                         "symmetric buffers) or mpGeMM + NCCL all_gather_into_tensor")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config 3/4 sweep")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-chain", action="store_true", help="skip the config-5 30-layer chain")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the step's kernels eagerly instead of replaying a CUDA graph")
    ap.add_argument("--chain-layers", type=int, default=30)
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clock warm-up loop, no cpu/sweep/e2e legs")
    ap.add_argument("--table", default="",
                    help="write SURVEY §8(d)'s per-(config, N, g) CSV (GPU timings, roofline "
                         "fractions, clocks, and the oracle's GOPS on a bounded row sample "
                         "as the cpu baseline of each row) to this path and exit")
    ap.add_argument("--plumbing", default="",
                    help="CPU check of the multi-rank plumbing over gloo with compute "
                         "injected from this tests/ module (not a measurement)")
    args = ap.parse_args()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    if args.plumbing:
        return plumbing_main(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.table:
        return config_table(args.table)
    if args.profile:
        args.no_cpu = args.no_sweep = args.no_e2e = args.no_chain = True

    import torch
    import torch.distributed as dist
    import paper_2512_06443_b200 as v

    from paper_2512_06443_b200.sharded import shard_rows
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    comm = None
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = comm_check(dist, dev)
        world = dist.get_world_size()  # the ranks that joined
    rank = dist.get_rank() if world > 1 else 0
    stream = torch.cuda.current_stream()

    peaks, peaks_src = load_peaks()
    wl = workload(args)
    M, K, N, g = wl["M"], wl["K"], wl["N"], wl["g"]
    alg = algorithmic(M, K, N, g)

    # ---- offline: weights (row shard of this rank) packed on device (a1)
    W = synth.ternary_weights(M, K, wl["w_seed"], wl["p_zero"])
    # rank's contiguous rows [r0, r1); shards padded to Mp rows for the gather
    r0, r1, Mp = shard_rows(M, world, rank)
    Ms = r1 - r0
    W_r = W[r0:r1]
    pw = v.pack_weights_device(torch.from_numpy(np.ascontiguousarray(W_r)).to(dev), g)
    x_host = synth.activations_f32(K, N, wl["x_seed"])
    x = torch.from_numpy(x_host).to(dev)
    q = torch.empty((K, N), dtype=torch.int8, device=dev)
    s = torch.empty((N,), dtype=torch.float32, device=dev)
    out_loc = torch.zeros((Mp, N), dtype=torch.float32, device=dev)  # pad rows stay 0
    out_r = out_loc[:Ms]
    gathered = torch.empty((Mp * world, N), dtype=torch.float32, device=dev) if world > 1 else None
    out_full = gathered[:M] if world > 1 else out_r
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    ws = v.workspace(dev)
    plan = v.plan_ws(Ms, K, N, g)

    # N > 1: the all-gather fused into the K1 epilogue (peer stores into
    # symmetric buffers + one cross-GPU barrier), validated once against the
    # NCCL path; any failure falls back to NCCL and says why
    gather = "none" if world == 1 else args.gather
    peer = None
    if world > 1 and gather == "p2p":
        try:
            from paper_2512_06443_b200.sharded import PeerOutputs
            peer = PeerOutputs()
            v.quantize(x, q=q, scale=s, stream=stream)
            v.mpgemm_ws(pw, q, s, synth.W_SCALE, out=out_r, ws=ws, stream=stream)
            dist.all_gather_into_tensor(gathered, out_loc)
            def validate(pe):
                for _ in range(2):  # both alternating buffers
                    buf, target, peers, barrier = pe.get(M, N, dev)
                    buf.fill_(float("nan"))
                    torch.cuda.synchronize()
                    dist.barrier()
                    v.mpgemm_allgather(pw, q, s, synth.W_SCALE, target, r0, peers,
                                       stream=stream, multicast=pe.multicast(M, N))
                    barrier()
                    torch.cuda.synchronize()
                    okt = torch.tensor([1 if torch.equal(buf, out_full) else 0], device=dev)
                    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
                    if int(okt.item()) != 1:
                        raise RuntimeError("fused all-gather result differs from NCCL")
            try:
                validate(peer)
                gather = "p2p " + peer.transport(M, N, dev)
            except Exception:
                if peer.transport(M, N, dev) != "multicast":
                    raise
                peer = PeerOutputs(mode="unicast")  # multicast failed: unicast peer stores
                validate(peer)
                gather = "p2p unicast (multicast failed validation)"
        except Exception as ex:  # keep measuring, on the NCCL path
            gather = f"nccl (p2p unavailable: {str(ex)[:120]})"
            peer = None

    def step(st=stream):
        v.quantize(x, q=q, scale=s, stream=st)
        if peer is not None:
            buf, target, peers, barrier = peer.get(M, N, dev)
            v.mpgemm_allgather(pw, q, s, synth.W_SCALE, target, r0, peers, stream=stream,
                               multicast=peer.multicast(M, N))
            barrier()
            return
        v.mpgemm_ws(pw, q, s, synth.W_SCALE, out=out_r, ws=ws, stream=st)
        if world > 1:
            dist.all_gather_into_tensor(gathered, out_loc)

    # ---- warm-up: W steps, plus >= 0.3 s of work so clocks leave idle
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while not args.profile and time.perf_counter() - t0 < 0.3:
        for _ in range(20):
            step()
        torch.cuda.synchronize()

    # ---- timed region: exactly K steps.  Only the step is bracketed by
    # events: an event between the quantizer and the mpGeMM would block the
    # programmatic-dependent-launch overlap of K1's prologue with K3's tail
    # (measured: +8 us per step), so the per-kernel durations for the
    # roofline come from a second pass of K steps in which each kernel is
    # timed alone right after its own L2 flush (events around the kernel).
    #
    # Launch mode (1 GPU): the step's two kernels are captured once in a CUDA
    # graph (the K3 -> K1 programmatic edge is kept) and the graph is replayed
    # each step -- per-kernel host launch latency (~4-5 us per eager launch,
    # measured: eager step 92.9 us vs 83.4 us in a graph) is not the path's
    # work; `launch.eager_ms_per_step` reports the eager number alongside.
    use_graph = world == 1 and not args.no_graph
    g_step = g_k3 = g_k1 = None
    if use_graph:
        g_step, g_k3, g_k1 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step):
            step(None)
        with torch.cuda.graph(g_k3):
            v.quantize(x, q=q, scale=s)
        with torch.cuda.graph(g_k1):
            v.mpgemm_ws(pw, q, s, synth.W_SCALE, out=out_r, ws=ws)
        for _ in range(3):
            g_step.replay()
        torch.cuda.synchronize()
    run_step = g_step.replay if use_graph else step
    run_k3 = g_k3.replay if use_graph else (lambda: v.quantize(x, q=q, scale=s, stream=stream))
    run_k1 = g_k1.replay if use_graph else (
        lambda: v.mpgemm_ws(pw, q, s, synth.W_SCALE, out=out_r, ws=ws, stream=stream))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush, outside the step's event window
            e = evs[i]
            e[0].record(stream)
            run_step()
            e[1].record(stream)
        torch.cuda.synchronize()
    eager_ms = None
    if use_graph:  # the same K steps launched eagerly, for reference
        eev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            eev[i][0].record(stream)
            step()
            eev[i][1].record(stream)
        torch.cuda.synchronize()
        eager_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in eev]))
    if world > 1:
        dist.barrier()
    # per-kernel passes (a second clock-sampling window: the timed steps above
    # last only a few ms), one
    # loop per kernel: each launch right after its own L2 flush, which runs on
    # the GPU while the host enqueues the event and the kernel (no host
    # submission latency in the window).  Separate loops because a preceding
    # K3 + synchronize measurably slows the next K1 launch (+6 us, idle-gap
    # effect, scripts/k1_timing_variants.py) -- inside the step, K1 follows
    # K3 back to back and takes ~step - K3.
    with ClockSampler(dev) as clk2:
        for i in range(args.steps):
            e = kev[i]
            flush.zero_()
            e[0].record(stream)
            run_k3()
            e[1].record(stream)
            torch.cuda.synchronize()
        for i in range(args.steps):
            e = kev[i]
            flush.zero_()
            e[2].record(stream)
            run_k1()
            e[3].record(stream)
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    k1_ms = [e[2].elapsed_time(e[3]) for e in kev]
    k3_ms = [e[0].elapsed_time(e[1]) for e in kev]
    total_ms = float(sum(step_ms))
    flushed = {"ms_per_step": total_ms / args.steps, "k1_ms_mean": float(np.mean(k1_ms)),
               "k3_ms_mean": float(np.mean(k3_ms)),
               "how": "each step (and each kernel) alone right after a 256 MiB L2 flush, CUDA "
                      "events around it: includes the idle-GPU launch latency of the first "
                      "kernel (~4-5 us)"}
    rotate = None
    if world == 1 and not args.no_graph:
        # Steady-state throughput with inputs larger than L2: R copies of the
        # packed weights, fp32 activations and outputs (R x 14 MB > 2 x the
        # 126 MB L2), step i uses copy i % R, the K steps run back to back
        # from one CUDA graph (no host launch gaps; every step's weights and
        # activations come from HBM).  The kernels' durations: graphs of K
        # back-to-back launches of each kernel alone over the same rotation.
        per_copy = pw.nbytes + x.numel() * 4 + out_r.numel() * 4
        R = max(2, -(-2 * (126 << 20) // per_copy))
        pws_r = [pw] + [v.pack_weights_device(torch.from_numpy(np.ascontiguousarray(W_r)).to(dev), g)
                        for _ in range(R - 1)]
        xs_r = [x] + [x.clone() for _ in range(R - 1)]
        outs_r = [out_r] + [torch.empty_like(out_r) for _ in range(R - 1)]
        torch.cuda.synchronize()

        def seq_graph(fn, end=None):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for i in range(args.steps):
                    fn(i % R)
                if end is not None:
                    end()
            gr.replay()
            torch.cuda.synchronize()
            return gr

        g_seq = seq_graph(lambda j: (v.quantize(xs_r[j], q=q, scale=s),
                                     v.mpgemm_ws(pws_r[j], q, s, synth.W_SCALE, out=outs_r[j], ws=ws)))
        g_k3s = seq_graph(lambda j: v.quantize(xs_r[j], q=q, scale=s))
        g_k1s = seq_graph(lambda j: v.mpgemm_ws(pws_r[j], q, s, synth.W_SCALE, out=outs_r[j], ws=ws))

        def timed(gr, reps=3):
            ts = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record(stream)
                gr.replay()
                b.record(stream)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return ts

        # the same K steps through pipeline.BatchPipeline: batch i+1's
        # quantizer (one-CTA clusters, side stream) runs on the SMs K1-32's
        # grid leaves free while batch i's mpGeMM runs; checked bit-identical
        # to the sequential schedule on every rotating output copy
        from paper_2512_06443_b200.pipeline import BatchPipeline
        bp = BatchPipeline(pw, synth.W_SCALE, K, N, dev, ws=ws)
        g_pipe = seq_graph(lambda j: bp.submit(xs_r[j], outs_r[j], W=pws_r[j]), end=bp.join)
        g_seq.replay()
        torch.cuda.synchronize()
        ref_outs = [o.clone() for o in outs_r]
        for o in outs_r:
            o.fill_(float("nan"))
        g_pipe.replay()
        torch.cuda.synchronize()
        pipe_same = all(torch.equal(a, b) for a, b in zip(outs_r, ref_outs))
        del ref_outs

        with ClockSampler(dev) as clk3:
            pipe_ts = timed(g_pipe)
            seq_ts = timed(g_seq)
            k1_ts = timed(g_k1s)
            k3_ts = timed(g_k3s)
        rotate = {"copies": R, "bytes_per_copy": int(per_copy),
                  "schedule": ("pipelined: batch i+1's quantizer (K3, one-CTA clusters, second "
                               "stream) overlaps batch i's mpGeMM (pipeline.BatchPipeline)"
                               if pipe_same else
                               "sequential (the pipelined schedule did not match it)"),
                  "pipelined_ms": pipe_ts, "pipelined_equals_sequential": pipe_same,
                  "seq_ms": seq_ts,
                  "seq_ms_per_step": float(seq_ts[0]) / args.steps,
                  "k1_ms_mean": float(np.median(k1_ts)) / args.steps,
                  "k3_ms_mean": float(np.median(k3_ts)) / args.steps}
        # the timed K steps: the first replay of the K-step graph is the
        # measurement (the other two confirm it)
        total_ms = float(pipe_ts[0] if pipe_same else seq_ts[0])
        k1_ms = [rotate["k1_ms_mean"]]
        k3_ms = [rotate["k3_ms_mean"]]
    if world > 1:
        t = torch.tensor([total_ms, float(np.mean(k1_ms))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, k1_mean = float(t[0]), float(t[1])
    else:
        k1_mean = float(np.mean(k1_ms))
    ms_per_step = total_ms / args.steps
    value = N * args.steps / (total_ms * 1e-3)  # whole-job tokens/s (all M rows)

    # ---- e2e through the public API from pinned host buffers: every step
    # uploads its fp32 input and downloads its fp32 result; HostPipeline
    # overlaps step i+1's upload and step i-1's download with step i's
    # kernels (separate copy-engine streams, 2 device buffer slots)
    e2e = None
    if not args.no_e2e:
        from paper_2512_06443_b200.pipeline import HostPipeline
        depth = 2
        x_pins = [torch.from_numpy(x_host).pin_memory() for _ in range(depth)]
        o_pins = [torch.empty((Ms, N), dtype=torch.float32).pin_memory() for _ in range(depth)]
        post = None
        if world > 1:
            locs = [torch.zeros((Mp, N), dtype=torch.float32, device=dev) for _ in range(depth)]
            fulls = [torch.empty((Mp * world, N), dtype=torch.float32, device=dev)
                     for _ in range(depth)]

            def post(res, st, slot):
                locs[slot][:Ms].copy_(res)
                dist.all_gather_into_tensor(fulls[slot], locs[slot])
                return res  # each rank downloads its own row shard
        pipe = HostPipeline(pw, synth.W_SCALE, K, N, dev, depth=depth, ws=ws, post=post)
        # >= 200 pipelined steps (~30 ms): the pipeline's fill and drain (one
        # upload, one download) stay < 1 % of the timed region
        e2e_steps = max(200, min(args.steps, 1000))
        for i in range(4):
            pipe.submit(x_pins[i % depth], o_pins[i % depth])
        pipe.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.s_in)
        for i in range(e2e_steps):
            pipe.submit(x_pins[i % depth], o_pins[i % depth])
        pipe.s_out.wait_stream(pipe.s_in)
        pipe.s_out.wait_stream(pipe.s_cmp)
        b.record(pipe.s_out)
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        # the downloaded result is the oracle-parity output (spot check)
        assert torch.equal(o_pins[(e2e_steps - 1) % depth], out_r.cpu()) or world > 1
        e2e = {"value": N * e2e_steps / (e2e_ms * 1e-3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(K * N * 4),
               "d2h_bytes_per_step": int(Ms * N * 4) * world, "steps": e2e_steps,
               "ms_per_step": e2e_ms / e2e_steps,
               "api": "paper_2512_06443_b200.pipeline.HostPipeline (quantize + mpgemm_ws per "
                      "step; H2D / compute / D2H on three streams, 2 buffer slots)"}

    if rank != 0:
        if not args.no_chain:
            chain_bench(v, dev, world, rank, args, peer=peer)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (K1)
    a_shard = algorithmic(Ms, K, N, g)
    sm_max = float(peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK))
    smem_peak_gbs = SM_COUNT * SMEM_BYTES_PER_CLK_SM * sm_max * 1e6 / 1e9
    achieved = a_shard["smem_bytes"] / (k1_mean * 1e-3) / 1e9
    # traffic: dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch
    # from an ncu --set full capture (ncu cannot run inside this timed
    # process); the file names the capture and the build it was taken of
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "k1_dram_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get("dram_bytes_per_launch")
            traffic_src = f"profiles/k1_dram_traffic.json <- {tj.get('source', '?')}"
        except Exception:
            traffic = None
    roofline = {
        "bound": "smem", "achieved": achieved, "peak": smem_peak_gbs, "unit": "GB/s",
        "frac": achieved / smem_peak_gbs, "traffic": traffic, "traffic_source": traffic_src,
        "kernel": ("vlut_mpgemm32_kernel (K1-32: 32-token tiles, paired-group tables)"
                   if plan.n_cta == 32 else "vlut_mpgemm_kernel (K1)")
                  + f" warps={plan.warps} splits={plan.splits}",
        "algorithmic_bytes_per_launch": a_shard["smem_bytes"],
        "per_unit": "2 B of shared-memory table read per int16 lookup-add; lookups = M*(K/g)*N",
        "peak_source": f"derived: {SM_COUNT} SMs x {SMEM_BYTES_PER_CLK_SM} B/clk x "
                       f"{sm_max:.0f} MHz (sm_max_mhz, {peaks_src})",
        "k1_ms_mean": k1_mean, "k3_quantize_ms_mean": float(np.mean(k3_ms)),
        "kernel_timing": ("K back-to-back launches of the kernel alone over the rotating "
                          "weight / activation / output copies (> 2x L2), one CUDA graph, "
                          "events around it: mean duration per launch"
                          if rotate is not None else
                          "per-kernel passes of K launches each: every launch right after its "
                          "own L2 flush, CUDA events around the kernel only, synchronize per "
                          "launch"),
        "hbm_achieved_gbs": a_shard["hbm_bytes"] / (k1_mean * 1e-3) / 1e9,
        "hbm_peak_gbs": float(peaks.get("hbm_gbs", HBM_FALLBACK_GBS)),
        "lookups_per_s": a_shard["lookups"] / (k1_mean * 1e-3),
    }

    line = {
        "metric": "ternary Vec-LUT mpGeMM tokens/s (configs[1])",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int16",
        "dtype_detail": "int8 activations x ternary (base-3 packed) weights; int16 LUT "
                        "lookup-adds, int32 accumulation, fp32 dequant",
        "data": "synthetic",
        "config": bench_config(wl, world),
        "kernels": "K3 quantize + fused Vec-LUT mpGeMM with fp32 dequant ("
                   + ("K1-32" if plan.n_cta == 32 else "K1") + ")"
                   + ((" with the all-gather of row shards fused into the epilogue "
                       "(NVLink peer stores + cross-GPU barrier)" if peer is not None
                       else " + NCCL all-gather of row shards") if world > 1 else ""),
        "gather": gather,
        "plan": plan.__dict__,
        "timing": ({"mode": "rotate", "detail": rotate, "flushed_latency": flushed}
                   if rotate is not None else {"mode": "flush", "detail": flushed}),
        "launch": {"mode": "cuda_graph" if use_graph else "eager",
                   "detail": ("quantize + mpGeMM captured once in a CUDA graph (programmatic "
                              "K3 -> K1 edge kept), replayed after each L2 flush; per-kernel "
                              "timing passes replay single-kernel graphs; the steady-state "
                              "(rotating) K steps: one graph of pipeline.BatchPipeline submits "
                              "(batch i+1's quantizer on a second stream under batch i's "
                              "mpGeMM), see timing.detail" if use_graph else
                              "eager launches"),
                   "eager_ms_per_step": eager_ms},
        "comm": comm,
        "gops": alg["dense_ops"] * args.steps / (total_ms * 1e-3) / 1e9,
        "gpu_launches": args.steps * vlut_launches_per_step(v, plan),
        "roofline": roofline,
        "e2e": e2e,
    }
    clocks = ClockSampler.merge(clk, clk2, *([clk3] if rotate is not None else []))
    line["clocks"] = clocks

    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(W, x_host, N)

    if world == 1 and not args.no_sweep:
        line["sweep"] = sweep(v, dev, stream, flush)

    if not args.no_chain:
        line["config5"] = chain_bench(v, dev, world, rank, args, peer=peer)

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    print(json.dumps(line), flush=True)
    return 0


def chain_bench(v, dev, world, rank, args, reps=5, peer=None):
    """BASELINE.json configs[4]: 30 BitNet-2B-shaped layers of ternary linears
    (QKV, O, gate, up, down), N = 2048 tokens, every linear row-sharded over
    the N GPUs with an NCCL all-gather (north star), int8 re-quantization
    between linears (reading c14).  Weights: seeded numpy ternary, packed on
    the device.  Times whole forwards with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2512_06443_b200.sharded import LayerChain, RowShardedLinear
    cfg = synth.CONFIGS[5]
    N = cfg.N[0]
    L = args.chain_layers
    layers = []
    for l in range(L):
        layers.append([RowShardedLinear(w, 4, synth.W_SCALE, device=dev, device_pack=True)
                       for _, w in synth.config_weights(cfg, l)])
    chain = LayerChain(layers)
    x = torch.from_numpy(synth.activations_f32(2560, N, synth.act_seed(cfg, N))).to(dev)
    xq, xs = v.quantize(x)
    chain(xq, xs)  # warm-up forward
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        chain(xq, xs)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts))
    # f1: fused re-quantization (epilogue maxima, int8 gathers, gate (.) up fused)
    fchain = LayerChain(layers, fused=True)
    fchain(xq, xs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tf = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fchain(xq, xs)
        b.record()
        torch.cuda.synchronize()
        tf.append(a.elapsed_time(b))
    t_f = float(np.median(tf))
    # f1 overlapped with compute: 2 token chunks; each linear's per-chunk
    # MAX all-reduce + quantize + int8 all-gather on a side stream while the
    # next chunk computes
    kchain = LayerChain(layers, fused=True, chunks=2)
    for _ in range(2):  # allocator steady state across the two streams
        kchain(xq, xs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tk = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        kchain(xq, xs)
        b.record()
        torch.cuda.synchronize()
        tk.append(a.elapsed_time(b))
    t_k = float(np.median(tk))
    # N > 1: every linear's all-gather fused into its K1 epilogue (peer stores)
    t_p = float("nan")
    if world > 1 and peer is not None:
        for lay in layers:
            for lin in lay:
                lin.peers = peer
        chain(xq, xs)
        torch.cuda.synchronize()
        dist.barrier()
        tp = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            chain(xq, xs)
            b.record()
            torch.cuda.synchronize()
            tp.append(a.elapsed_time(b))
        t_p = float(np.median(tp))
        for lay in layers:
            for lin in lay:
                lin.peers = None
    if world > 1:
        tt = torch.tensor([t, t_f, t_p, t_k], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, t_f, t_p, t_k = float(tt[0]), float(tt[1]), float(tt[2]), float(tt[3])
    lookups = L * N * sum(lin.M * lin.K // 4 for lin in cfg.linears)
    R_LU = SM_COUNT * 64 * SM_MAX_MHZ_FALLBACK * 1e6
    return {"config": 5, "layers": L, "N": N, "n_gpus": world, "ms_per_forward": t,
            "tokens_s": N / (t * 1e-3),
            "frac_smem_roofline": lookups / (R_LU * world) / (t * 1e-3),
            "fused_requant": {"ms_per_forward": t_f, "tokens_s": N / (t_f * 1e-3),
                              "frac_smem_roofline": lookups / (R_LU * world) / (t_f * 1e-3)},
            "fused_requant_overlapped": {"ms_per_forward": t_k, "tokens_s": N / (t_k * 1e-3),
                                         "chunks": 2,
                                         "frac_smem_roofline": lookups / (R_LU * world)
                                         / (t_k * 1e-3)},
            "fused_allgather": ({"ms_per_forward": t_p, "tokens_s": N / (t_p * 1e-3),
                                 "frac_smem_roofline": lookups / (R_LU * world) / (t_p * 1e-3)}
                                if t_p == t_p else None),
            "step": "per layer: 5 row-sharded Vec-LUT linears (+ all-gather when n_gpus > 1) "
                    "and 4 int8 re-quantizations; weights packed once before timing; "
                    "fused_requant = f1 (epilogue maxima, int8 all-gathers)"}


def sweep(v, dev, stream, flush, reps=10):
    """Configs 3 and 4 (BASELINE.json configs[2], configs[3]): K1 alone on
    resident int8 inputs, L2 flushed between launches; N = 256..4096."""
    import torch
    R_LU = SM_COUNT * 64 * SM_MAX_MHZ_FALLBACK * 1e6
    res = []

    ws = v.workspace(dev)

    def timeit(pw, A, sc, out):
        for _ in range(2):
            v.mpgemm_ws(pw, A, sc, synth.W_SCALE, out=out, ws=ws, stream=stream)
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            v.mpgemm_ws(pw, A, sc, synth.W_SCALE, out=out, ws=ws, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return float(np.median(ts))

    def timeit_batched(make_run, pws, reps=60):
        """Short launches (N <= 64): per-launch events have ~2 us resolution,
        so a CUDA graph of one launch per weight copy (copies > 2x L2: every
        launch streams its weights from HBM) is replayed and averaged.  The
        launches go to the current stream (the capture stream)."""
        runs = [make_run(pw) for pw in pws]
        for r in runs[:2]:
            r()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for r in runs:
                r()
        gr.replay()
        torch.cuda.synchronize()
        per = max(2, reps // len(runs))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(per):
            gr.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e-3 / (per * len(runs))

    hbm_peak = load_peaks()[0].get("hbm_gbs", HBM_FALLBACK_GBS) * 1e9
    c4 = synth.CONFIGS[4]
    lin = c4.linears[0]
    W4 = torch.from_numpy(synth.ternary_weights(lin.M, lin.K, synth.weight_seed(c4, 0, 0))).to(dev)
    for g in (4, 5):
        pw = v.pack_weights_device(W4, g)
        copies = max(1, -(-260_000_000 // pw.nbytes))
        pws = [pw] + [v.pack_weights_device(W4, g) for _ in range(copies - 1)]
        for N in c4.N:
            x = torch.from_numpy(synth.activations_f32(lin.K, N, synth.act_seed(c4, N))).to(dev)
            A, sc = v.quantize(x)
            out = torch.empty((lin.M, N), dtype=torch.float32, device=dev)
            lk = lin.M * (lin.K // g) * N
            hbm_bytes = pw.nbytes + lin.K * N + 4 * N + 4 * lin.M * N
            pl = v.plan_ws(lin.M, lin.K, N, g)
            if N <= 64:
                t = timeit_batched(lambda p_: (lambda: v.mpgemm_ws(
                    p_, A, sc, synth.W_SCALE, out=out, ws=ws)), pws)
                timing = "CUDA graph of back-to-back launches over weight copies > 2x L2"
            else:
                t = timeit(pw, A, sc, out)
                timing = "per-launch events, L2 flushed"
            kern = plan_label(pl)
            e = {"config": 4, "M": lin.M, "K": lin.K, "N": N, "g": g, "us": t * 1e6,
                 "kernel": kern, "timing": timing,
                 "tokens_s": N / t, "gops": 2 * lin.M * lin.K * N / t / 1e9,
                 "frac_smem_roofline": lk / R_LU / t,
                 "frac_hbm_roofline": hbm_bytes / hbm_peak / t}
            if N <= 64:
                # f4 comparator: the scalar LUT (1->1 lookups, one table per token)
                ts = timeit_batched(lambda p_: (lambda: v.mpgemm_scalar_lut(
                    p_, A, sc, synth.W_SCALE, out=out, ws=ws)), pws)
                e["scalar_lut_us"] = ts * 1e6
                e["vec_over_scalar_speedup"] = ts / t
            if N == 1:
                # a whole decode step: quantize + mpGeMM (two launches), and
                # the same step fused into one kernel (vlut_mpgemm_decode)
                xf = x[:, 0].contiguous()
                of = torch.empty((lin.M,), dtype=torch.float32, device=dev)
                sf = torch.empty((1,), dtype=torch.float32, device=dev)
                tq = timeit_batched(lambda p_: (lambda: (
                    v.quantize(x, q=A, scale=sc),
                    v.mpgemm_ws(p_, A, sc, synth.W_SCALE, out=out, ws=ws))), pws)
                tf = timeit_batched(lambda p_: (lambda: v.mpgemm_decode(
                    p_, xf, synth.W_SCALE, out=of, scale_out=sf, ws=ws)), pws)
                e["decode_step_us"] = tq * 1e6
                e["fused_decode_step_us"] = tf * 1e6
            res.append(e)
        del pw, pws
    c3 = synth.CONFIGS[3]
    tot = 0.0
    for j, lin in enumerate(c3.linears):
        Wd = torch.from_numpy(synth.ternary_weights(lin.M, lin.K, synth.weight_seed(c3, 0, j))).to(dev)
        pw = v.pack_weights_device(Wd, 4)
        x = torch.from_numpy(synth.activations_f32(lin.K, 1024, synth.act_seed(c3, 1024, j))).to(dev)
        A, sc = v.quantize(x)
        out = torch.empty((lin.M, 1024), dtype=torch.float32, device=dev)
        t = timeit(pw, A, sc, out)
        tot += t
        lk = lin.M * (lin.K // 4) * 1024
        res.append({"config": 3, "linear": lin.name, "M": lin.M, "K": lin.K, "N": 1024, "g": 4,
                    "us": t * 1e6, "frac_smem_roofline": lk / R_LU / t})
    res.append({"config": 3, "linear": "all 5 in sequence", "N": 1024, "us": tot * 1e6,
                "tokens_s": 1024 / tot})
    # mixed g=5/g=4 schedule (f2) on config 3's K = 4096 / 14336 linears
    for j in (0, 4):
        lin = c3.linears[j]
        W = synth.ternary_weights(lin.M, lin.K, synth.weight_seed(c3, 0, j))
        pm = v.pack_weights_mixed(W, device=dev)
        x = torch.from_numpy(synth.activations_f32(lin.K, 1024, synth.act_seed(c3, 1024, j))).to(dev)
        A, sc = v.quantize(x)
        out = torch.empty((lin.M, 1024), dtype=torch.float32, device=dev)
        for _ in range(2):
            v.mpgemm_mixed(pm, A, sc, synth.W_SCALE, out=out, ws=ws, stream=stream)
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            v.mpgemm_mixed(pm, A, sc, synth.W_SCALE, out=out, ws=ws, stream=stream)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        t = float(np.median(ts))
        k5, k4 = v.group_schedule(lin.K)
        lk = lin.M * (k5 // 5 + k4 // 4) * 1024
        res.append({"config": 3, "linear": lin.name + " (mixed g5/g4)", "M": lin.M, "K": lin.K,
                    "N": 1024, "k5": k5, "k4": k4, "bpw": 8.0 * (k5 / 5 + k4 / 4) / lin.K,
                    "us": t * 1e6, "frac_smem_roofline": lk / R_LU / t})
        # the same K with g = 5 and a zero-padded last group (VLUT_PACK_PAD_K):
        # same bytes per row, one launch
        p5 = v.pack_weights(W, 5, device=dev, pad_k=True)
        t5 = timeit(p5, A, sc, out)
        lk5 = lin.M * (-(-lin.K // 5)) * 1024
        res.append({"config": 3, "linear": lin.name + " (g5, padded K)", "M": lin.M, "K": lin.K,
                    "N": 1024, "bpw": 8.0 * (-(-lin.K // 5)) / lin.K, "us": t5 * 1e6,
                    "frac_smem_roofline": lk5 / R_LU / t5})
    return res


# ------------------------------------------------------------------ SURVEY §8(d) table
def config_table(path, oracle_budget_s=0.6):
    """One CSV row per (config, linear, N, g, G=1) of BASELINE.json's configs:
    median and min device time (>= 20 repeats and >= 100 ms of timed work;
    launches over weight copies > 2x L2 in a CUDA graph for N <= 64, else one
    launch per L2 flush with events around it), tokens/s, effective GOPS
    (2MKN/t), lookups/s, T_roof = max(T_hbm, T_lu) and T_roof / t, the SM
    clock under load, and the oracle's GOPS on a bounded row sample with the
    host's thread count (the cpu baseline of each row).  Configs 1..5 at
    G = 1; config 2 also with uniform weights (the path is data-independent);
    config 5 is its layer-0 linears (every layer has the same shapes)."""
    import csv
    import torch
    import oracle
    import paper_2512_06443_b200 as v
    oracle.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peaks, _ = load_peaks()
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS) * 1e9
    r_lu = SM_COUNT * 64 * peaks.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK) * 1e6
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ws = v.workspace(dev)
    cores = oracle.num_threads()
    oracle_cache = {}

    def oracle_gops(W, q, key):
        if key in oracle_cache:
            return oracle_cache[key]
        M, K = W.shape
        N = q.shape[1]
        acc = np.zeros((M, N), np.int32)
        oracle.gemm_i32_rows(W, q, 0, min(M, 2), acc)  # warm (threads, pages)
        rows = min(M, 4)
        while True:  # double the row sample until it takes >= the budget
            t0 = time.perf_counter()
            oracle.gemm_i32_rows(W, q, 0, rows, acc)
            t = time.perf_counter() - t0
            if t >= oracle_budget_s or rows == M:
                break
            rows = min(M, max(2 * rows, int(rows * oracle_budget_s / max(t, 1e-6))))
        oracle_cache[key] = (2.0 * rows * K * N / t / 1e9, f"rows [0,{rows}) of {M}, {t:.2f} s")
        return oracle_cache[key]

    rows_out = []

    def emit(cfg, lin, M, K, N, g, pz, pw, A, sc, out, W, q):
        lk = M * (K // g) * N
        hbm_b = pw.nbytes + K * N + 4 * N + 4 * M * N
        t_roof = max(hbm_b / hbm, lk / r_lu)
        pl = v.plan_ws(M, K, N, g)
        kern = plan_label(pl)
        call = lambda p_: (lambda: v.mpgemm_ws(p_, A, sc, synth.W_SCALE, out=out, ws=ws))
        with ClockSampler(dev) as clk:
            if N <= 64:
                # a CUDA graph of one launch per weight copy (copies > 2x L2:
                # every launch streams its weights from HBM), replayed
                copies = max(1, min(256, -(-260_000_000 // pw.nbytes)))
                Wd = torch.from_numpy(W).to(dev)
                pws = [pw] + [v.pack_weights_device(Wd, g) for _ in range(copies - 1)]
                del Wd
                runs = [call(p_) for p_ in pws]
                for r in runs[:3]:
                    r()
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for r in runs:
                        r()
                gr.replay()
                torch.cuda.synchronize()
                per = []
                t_start = time.perf_counter()
                while len(per) < 20 or sum(per) * len(runs) < 0.1:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    gr.replay()
                    b.record()
                    torch.cuda.synchronize()
                    per.append(a.elapsed_time(b) * 1e-3 / len(runs))
                    if time.perf_counter() - t_start > 20:
                        break
                timing = f"CUDA graph of {len(runs)} launches over weight copies, per-launch mean"
                del gr, runs, pws
            else:
                for _ in range(3):
                    call(pw)()
                torch.cuda.synchronize()
                per = []
                while len(per) < 20 or sum(per) < 0.1:
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    call(pw)()
                    b.record()
                    torch.cuda.synchronize()
                    per.append(a.elapsed_time(b) * 1e-3)
                timing = "one launch per L2 flush, events around it"
        t_med, t_min = float(np.median(per)), float(np.min(per))
        og, osample = oracle_gops(W, q, (cfg, lin, M, K, N, pz))
        ck = clk.summary()
        gops = 2.0 * M * K * N / t_med / 1e9
        rows_out.append({
            "config": cfg, "linear": lin, "M": M, "K": K, "N": N, "g": g, "G": 1,
            "weights": "uniform{-1,0,1}" if pz is None else f"P(0)={pz}",
            "kernel": kern, "t_median_us": round(t_med * 1e6, 3), "t_min_us": round(t_min * 1e6, 3),
            "repeats": len(per), "timing": timing, "tokens_s": round(N / t_med, 1),
            "gops": round(gops, 1), "lookups_s": round(lk / t_med, 1),
            "t_roof_us": round(t_roof * 1e6, 3),
            "bound": "hbm" if hbm_b / hbm > lk / r_lu else "smem",
            "frac_roof": round(t_roof / t_med, 4), "sm_mhz": ck.get("sm_mhz"),
            "throttle": "|".join(ck.get("reasons", [])), "host_cores": cores,
            "oracle_gops": round(og, 3), "oracle_sample": osample,
            "gpu_over_oracle": round(gops / og, 1)})
        print(json.dumps(rows_out[-1]), file=sys.stderr, flush=True)

    def one(cfg_idx, j, lin, N, g, pz):
        cfg = synth.CONFIGS[cfg_idx]
        W = synth.ternary_weights(lin.M, lin.K, synth.weight_seed(cfg, 0, j), pz)
        x = synth.activations_f32(lin.K, N, synth.act_seed(cfg, N, j))
        q, s = oracle.quantize(x)
        pw = v.pack_weights_device(torch.from_numpy(W).to(dev), g)
        A = torch.from_numpy(q).to(dev)
        sc = torch.from_numpy(s).to(dev)
        out = torch.empty((lin.M, N), dtype=torch.float32, device=dev)
        emit(cfg_idx, lin.name, lin.M, lin.K, N, g, pz, pw, A, sc, out, W, q)

    c = synth.CONFIGS
    one(1, 0, c[1].linears[0], 8, 4, None)
    one(2, 0, c[2].linears[0], 256, 4, c[2].p_zero)
    one(2, 0, c[2].linears[0], 256, 4, None)
    for j, lin in enumerate(c[3].linears):
        one(3, j, lin, 1024, 4, None)
    for g in c[4].g:
        for N in c[4].N:
            one(4, 0, c[4].linears[0], N, g, None)
    for j, lin in enumerate(c[5].linears):
        one(5, j, lin, 2048, 4, None)
    with open(path, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=list(rows_out[0].keys()))
        wr.writeheader()
        wr.writerows(rows_out)
    print(json.dumps({"table": path, "rows": len(rows_out)}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
