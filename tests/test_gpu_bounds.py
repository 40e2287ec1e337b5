"""Out-of-bounds write guards for every kernel path (GPU).

Each output (and the split-K workspace) is a window inside a larger buffer
whose surrounding bytes hold a canary pattern; after the call the canaries
must be intact and the window must hold the oracle's result.  This is the
substitute for a memory checker on the GPU pool: a tile, tail or epilogue
store that lands outside [M][N] (or outside the workspace) fails here.
"""
import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

GUARD = 64 * 1024          # bytes of canary on each side (keeps 1 KB alignment)
CANARY = 0x5A


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


class Guarded:
    """A [shape] tensor of dtype inside a byte buffer with canaries around it."""

    def __init__(self, shape, dtype, fill=None):
        esz = torch.empty((), dtype=dtype).element_size()
        n = int(np.prod(shape)) if len(shape) else 1
        self.nbytes = n * esz
        self.raw = torch.full((GUARD * 2 + self.nbytes,), CANARY, dtype=torch.uint8, device=dev())
        win = self.raw[GUARD:GUARD + self.nbytes]
        if fill is not None:
            win.fill_(fill)
        self.t = win.view(dtype).view(*shape)

    def intact(self):
        torch.cuda.synchronize()
        r = self.raw.cpu().numpy()
        return bool(np.all(r[:GUARD] == CANARY) and np.all(r[GUARD + self.nbytes:] == CANARY))


SHAPES = [(33, 68, 3, 4), (64, 64, 1, 4), (385, 1024, 130, 4), (200, 1285, 17, 5),
          (1000, 1300, 5, 4), (777, 2565, 67, 5), (129, 640, 257, 4)]


def _case(v, M, K, N, g):
    W = synth.ternary_weights(M, K, seed=M + N)
    x = synth.activations_f32(K, N, seed=K + N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights(W, g, device=dev())
    return W, x, q, s, pw, oracle.gemm_i32(W, q)


def _plans(v, N):
    plans = [None, v.LaunchPlan(8, 1), v.LaunchPlan(12, 3), v.LaunchPlan(16, 2, streamk=1)]
    if N <= 64:
        plans += [v.slot_plan(tpw=1), v.slot_plan(tpw=2, splits=3)]
    return plans


@pytest.mark.parametrize("M,K,N,g", SHAPES)
def test_mpgemm_outputs_and_workspace_stay_in_bounds(v, M, K, N, g):
    W, x, q, s, pw, ref = _case(v, M, K, N, g)
    ref32 = oracle.dequant_f32(ref, s, synth.W_SCALE)
    qd, sd = to_dev(q), to_dev(s)
    ws = Guarded((int(v.workspace(dev()).numel()),), torch.uint8, fill=0)
    for plan in _plans(v, N):
        out = Guarded((M, N), torch.float32)
        v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, out=out.t, plan=plan, ws=ws.t)
        assert out.intact() and ws.intact(), plan
        assert np.array_equal(out.t.cpu().numpy().view(np.int32), ref32.view(np.int32)), plan
        acc = Guarded((M, N), torch.int32)
        v.mpgemm_acc_ws(pw, qd, out=acc.t, plan=plan, ws=ws.t)
        assert acc.intact() and ws.intact(), plan
        assert np.array_equal(acc.t.cpu().numpy(), ref), plan
    # the scalar-LUT comparator, with and without split-K
    if N <= 64:
        for use in (ws.t, None):
            out = Guarded((M, N), torch.float32)
            v.mpgemm_scalar_lut(pw, qd, sd, synth.W_SCALE, out=out.t, ws=use, use_ws=use is not None)
            assert out.intact() and ws.intact()
            assert np.array_equal(out.t.cpu().numpy().view(np.int32), ref32.view(np.int32))


@pytest.mark.parametrize("M,K,N,g", SHAPES[:5])
def test_fused_layout_and_quantizers_stay_in_bounds(v, M, K, N, g):
    W, x, q, s, pw, ref = _case(v, M, K, N, g)
    xd = to_dev(x)
    # K3: q [K][N] int8, scale [N]
    qg, sg = Guarded((K, N), torch.int8), Guarded((N,), torch.float32)
    v.quantize(xd, q=qg.t, scale=sg.t)
    assert qg.intact() and sg.intact()
    assert np.array_equal(qg.t.cpu().numpy(), q)
    qt, st = Guarded((K, N), torch.int8), Guarded((N,), torch.float32)
    v.quantize_t(xd.t().contiguous(), q=qt.t, scale=st.t)
    assert qt.intact() and st.intact()
    assert np.array_equal(qt.t.cpu().numpy(), q)
    # feature-major epilogue
    fm = Guarded((N, M), torch.float32)
    v.mpgemm_layout(pw, qg.t, sg.t, synth.W_SCALE, out=fm.t)
    assert fm.intact()
    ref32 = oracle.dequant_f32(ref, s, synth.W_SCALE)
    assert np.array_equal(fm.t.cpu().numpy().T.view(np.int32), ref32.view(np.int32))
    # fused re-quantization maxima (f1) and the amax quantizer
    amax = Guarded((N,), torch.int32, fill=0)
    out = Guarded((M, N), torch.float32)
    v.mpgemm_fused(pw, qg.t, sg.t, synth.W_SCALE, out=out.t, amax=amax.t)
    assert out.intact() and amax.intact()
    qa, sa = Guarded((M, N), torch.int8), Guarded((N,), torch.float32)
    v.quantize_amax(out.t, amax.t, q=qa.t, scale=sa.t)
    assert qa.intact() and sa.intact()
    q2, s2 = oracle.quantize(ref32)
    assert np.array_equal(qa.t.cpu().numpy(), q2)


@pytest.mark.parametrize("M,K,N,g,shards", [(385, 1024, 130, 4, 3), (1000, 1300, 5, 4, 2),
                                            (200, 1285, 17, 5, 4)])
def test_allgather_shards_stay_in_their_rows(v, M, K, N, g, shards):
    """Fused all-gather: each shard writes only its row band of out_full and
    of every peer buffer (two peers emulated on one device)."""
    W = synth.ternary_weights(M, K, seed=3)
    x = synth.activations_f32(K, N, seed=4)
    q, s = oracle.quantize(x)
    qd, sd = to_dev(q), to_dev(s)
    ref32 = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
    bounds = np.linspace(0, M, shards + 1).astype(int)
    for i in range(shards):
        r0, r1 = int(bounds[i]), int(bounds[i + 1])
        pw = v.pack_weights(np.ascontiguousarray(W[r0:r1]), g, device=dev())
        own, peer = Guarded((M, N), torch.float32, fill=0), Guarded((M, N), torch.float32, fill=0)
        v.mpgemm_allgather(pw, qd, sd, synth.W_SCALE, own.t, r0, [peer.t.data_ptr()])
        assert own.intact() and peer.intact()
        for b in (own, peer):
            o = b.t.cpu().numpy()
            assert np.array_equal(o[r0:r1].view(np.int32), ref32[r0:r1].view(np.int32))
            assert not o[:r0].any() and not o[r1:].any()


def test_empty_inputs_are_noops(v):
    """N = 0 (no tokens) through every entry point: status OK, nothing written."""
    M, K, g = 300, 640, 4
    W = synth.ternary_weights(M, K, seed=1)
    pw = v.pack_weights(W, g, device=dev())
    A = torch.empty((K, 0), dtype=torch.int8, device=dev())
    s = torch.empty((0,), dtype=torch.float32, device=dev())
    guard = Guarded((M, 1), torch.float32, fill=7)
    out = guard.t[:, :0]
    ws = v.workspace(dev())
    v.mpgemm(pw, A, s, synth.W_SCALE, out=out)
    v.mpgemm_ws(pw, A, s, synth.W_SCALE, out=out, ws=ws)
    v.mpgemm_ex(pw, A, s, synth.W_SCALE, out=out)
    v.mpgemm_scalar_lut(pw, A, s, synth.W_SCALE, out=out, ws=ws)
    v.mpgemm_layout(pw, A, s, synth.W_SCALE, out=torch.empty((0, M), device=dev()))
    q, sc = v.quantize(torch.empty((K, 0), device=dev()))
    torch.cuda.synchronize()
    assert guard.intact() and bool((guard.raw[GUARD:GUARD + guard.nbytes] == 7).all())
    assert q.numel() == 0 and sc.numel() == 0
