"""Hooks for ``bench.py --plumbing tests/bench_plumbing.py`` (test
infrastructure): the CPU oracle stands in for the per-shard CUDA compute so
the multi-rank bench plumbing (spawn, process-group join, row sharding with
padding, all-gather, max-over-ranks timing) can run under gloo without a GPU.
Not collected by pytest (no test_ prefix); test_bench_plumbing.py drives it."""
import numpy as np
import torch

import oracle


def quantize(x):
    q, s = oracle.quantize(np.ascontiguousarray(x))
    return torch.from_numpy(q), torch.from_numpy(s)


def compute(w_scale):
    def f(shard, A, a_scale, out):
        acc = oracle.gemm_i32(shard, A.numpy())
        out.copy_(torch.from_numpy(oracle.dequant_f32(acc, a_scale.numpy(), w_scale)))
    return f


def reference(W, q, s, w_scale):
    return oracle.dequant_f32(oracle.gemm_i32(W, q.numpy()), s.numpy(), w_scale)
