"""Seeded random-shape parity sweep (GPU) of every public mpGeMM entry point
against the CPU oracle: the auto planner picks K1 cluster, K1 stream-K or K2
depending on the shape, so random (M, K, N, g) reach plan boundaries, ragged
M / K / N tails and tiny dimensions that hand-picked cases may miss.

Bar: int32 accumulators bit-exact; fp32 outputs bit-identical to the
oracle's fixed-order fp32 dequant.
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


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def shapes(n, seed):
    r = synth.rng(seed)
    out = []
    for _ in range(n):
        g = int(r.choice([4, 5]))
        M = int(r.choice([r.integers(1, 64), r.integers(64, 1200), r.integers(1200, 3100)]))
        K = g * int(r.choice([r.integers(1, 40), r.integers(40, 700)]))
        N = int(r.choice([r.integers(1, 17), r.integers(17, 80), r.integers(80, 300)]))
        out.append((M, K, N, g))
    return out


CASES = shapes(36, 2024)


@pytest.mark.parametrize("M,K,N,g", CASES)
def test_random_shape_all_entry_points(v, M, K, N, g):
    seed = M * 7 + K * 3 + N
    W = synth.ternary_weights(M, K, seed)
    x = synth.activations_f32(K, N, seed + 1)
    q, s = oracle.quantize(x)
    acc_ref = oracle.gemm_i32(W, q)
    ref32 = oracle.dequant_f32(acc_ref, s, synth.W_SCALE)
    pw = v.pack_weights(W, g, device=dev())
    qd, sd = to_dev(q), to_dev(s)
    ws = v.workspace(dev())
    # GPU quantizer == oracle quantizer
    qg, sg = v.quantize(to_dev(x))
    outs = {
        "mpgemm": v.mpgemm(pw, qd, sd, synth.W_SCALE),
        "mpgemm_ws": v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, ws=ws),
        "mpgemm_ex": v.mpgemm_ex(pw, qd, sd, synth.W_SCALE),
    }
    acc = v.mpgemm_acc_ws(pw, qd, ws=ws)
    acc_c = v.mpgemm_acc(pw, qd)
    fm = v.mpgemm_layout(pw, qd, sd, synth.W_SCALE)
    if N <= 64:
        outs["scalar_lut"] = v.mpgemm_scalar_lut(pw, qd, sd, synth.W_SCALE, ws=ws)
    torch.cuda.synchronize()
    assert np.array_equal(qg.cpu().numpy(), q) and np.array_equal(sg.cpu().numpy(), s)
    assert np.array_equal(acc.cpu().numpy(), acc_ref), "acc_ws"
    assert np.array_equal(acc_c.cpu().numpy(), acc_ref), "acc"
    for name, o in outs.items():
        assert np.array_equal(o.cpu().numpy().view(np.int32), ref32.view(np.int32)), name
    assert np.array_equal(fm.cpu().numpy().T.view(np.int32), ref32.view(np.int32)), "layout"


@pytest.mark.parametrize("M,K,N", [(M, K, N) for (M, K, N, g) in shapes(10, 7)])
def test_random_shape_mixed_schedule(v, M, K, N):
    """Mixed g=5/g=4 packing (f2) for arbitrary K (not a multiple of 4 or 5
    in general): the schedule's two parts chained through int32."""
    K = K + 1 + (M % 7)  # break divisibility on purpose
    try:
        k5, k4 = v.group_schedule(K)
    except v.VlutError:
        pytest.skip(f"K={K} not representable as 5a + 4b")
    assert k5 + k4 == K and k5 % 5 == 0 and k4 % 4 == 0
    W = synth.ternary_weights(M, K, M + K)
    x = synth.activations_f32(K, N, K + N)
    q, s = oracle.quantize(x)
    pm = v.pack_weights_mixed(W, device=dev())
    o = v.mpgemm_mixed(pm, to_dev(q), to_dev(s), synth.W_SCALE, ws=v.workspace(dev()))
    torch.cuda.synchronize()
    ref32 = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
    assert np.array_equal(o.cpu().numpy().view(np.int32), ref32.view(np.int32))
