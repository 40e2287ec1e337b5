"""Stress: many back-to-back launches that alternate schedules (K1 cluster,
K1 stream-K with 1 and 2 rows per thread, K2 split-K in both meeting modes,
K2 without split) and shapes on shared workspaces and two streams, without
host synchronisation between them.  Every result must equal the result of
the same call made alone (all schedules are bit-identical):
this catches cross-launch races in the split-K arrival counters, generation
words, stream-K epoch flags and workspace zero-keeping.
"""
import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def v():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    import paper_2512_06443_b200 as vl
    return vl


def dev():
    return torch.device("cuda:0")


def test_interleaved_schedules_two_streams(v):
    shapes = [(3072, 23040, 1, 4), (3072, 4608, 16, 4), (1100, 2560, 4, 5), (6912, 2560, 256, 4),
              (2560, 2560, 512, 4), (777, 1285, 64, 5)]
    cases = []
    for i, (M, K, N, g) in enumerate(shapes):
        W = synth.ternary_weights(M, K, seed=50 + i)
        A = synth.int8_activations(K, N, seed=60 + i)
        pw = v.pack_weights(W, g, device=dev())
        rows = np.unique(np.concatenate([[0, M - 1], synth.rng(i).integers(0, M, size=8)]))
        ref = oracle.gemm_i32(W[rows], A)
        cases.append((pw, torch.from_numpy(A).to(dev()), M, N, rows, ref))
    plans = [None, v.LaunchPlan(12, 2), v.LaunchPlan(16, 1, streamk=1),
             v.LaunchPlan(12, 1, m_cta=768, streamk=1), v.slot_plan(tpw=2), v.slot_plan(tpw=1),
             v.slot_plan(tpw=2, splits=1)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    wss = [torch.zeros_like(v.workspace(dev())) for _ in streams]
    rng = synth.rng(123)
    pending = []
    for it in range(240):
        si = it % 2
        ci = int(rng.integers(0, len(cases)))
        pw, Ad, M, N, rows, ref = cases[ci]
        plan = plans[int(rng.integers(0, len(plans)))]
        if plan is not None and plan.slot and N > 64:
            plan = None
        with torch.cuda.stream(streams[si]):
            acc = v.mpgemm_acc_ws(pw, Ad, plan=plan, ws=wss[si], stream=streams[si])
        pending.append((acc, rows, ref, ci, plan))
        if len(pending) >= 24:
            torch.cuda.synchronize()
            for acc, rows, ref, ci, plan in pending:
                got = acc[torch.from_numpy(rows).to(dev())].cpu().numpy()
                assert np.array_equal(got, ref), (ci, plan)
            pending.clear()
    torch.cuda.synchronize()
    for acc, rows, ref, ci, plan in pending:
        got = acc[torch.from_numpy(rows).to(dev())].cpu().numpy()
        assert np.array_equal(got, ref), (ci, plan)
