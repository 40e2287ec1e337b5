"""GPU parity of K2 -- the lane-slot kernel for small N (decode) and the
scalar-LUT (1->1) comparator --
against the CPU oracle, through the C ABI.

Bar: int32 accumulators bit-exact for every variant (g, nw, tpw), every split
of the K range and every tail; fp32 outputs bit-identical to the oracle's
fixed-order fp32 dequant and within 1e-6 of the fp64 definition.
"""
import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

REL_TOL = 1e-6


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


def check_fp32(got, acc_ref, a_scale, w_scale):
    ref = oracle.dequant_f64(acc_ref, a_scale, w_scale)
    g = got.astype(np.float64)
    nz = ref != 0
    assert np.all(g[~nz] == 0)
    rel = np.abs(g[nz] - ref[nz]) / np.abs(ref[nz])
    assert rel.size == 0 or rel.max() <= REL_TOL, rel.max()
    ref32 = oracle.dequant_f32(acc_ref, a_scale, w_scale)
    assert np.array_equal(got.view(np.int32), ref32.view(np.int32))


VARIANTS = [(4, nw, tpw) for tpw in (1, 2) for nw in (1, 2, 4, 8)] + \
           [(5, nw, tpw) for tpw in (1, 2) for nw in (1, 2)] + [(5, 4, 1)]

# (M, K, N): ragged M (not a multiple of 32 / of m_cta), K-tiles with a
# ragged last tile, N not a multiple of the CTA's token count
SHAPES_G4 = [(1, 4, 1), (33, 68, 3), (1000, 1300, 5), (1100, 2560, 17), (2100, 640, 1)]
SHAPES_G5 = [(1, 5, 1), (70, 85, 3), (2100, 1280, 5), (2500, 2565, 1)]


@pytest.mark.parametrize("g,nw,tpw", VARIANTS)
@pytest.mark.parametrize("splits", [1, 3, 0])
def test_slot_acc_every_variant_and_split(v, g, nw, tpw, splits):
    for (M, K, N) in (SHAPES_G4 if g == 4 else SHAPES_G5):
        W = synth.ternary_weights(M, K, seed=M + K)
        A = synth.int8_activations(K, N, seed=K + N)  # full int8 range incl. -128
        pw = v.pack_weights(W, g, device=dev())
        plan = v.slot_plan(tpw=tpw, nw=nw, splits=splits)
        acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=plan)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), oracle.gemm_i32(W, A)), (M, K, N)


@pytest.mark.parametrize("g,nw,tpw,N", [(4, 8, 2, 100), (4, 4, 1, 67), (5, 2, 2, 129), (4, 8, 2, 65)])
def test_slot_wide_n_global_activation_path(v, g, nw, tpw, N):
    """N > 64: activations are not staged by TMA (the builders read them from
    global memory), several N-tiles, ragged last N-tile; forced K2 plans."""
    M, K = 1100, 1280 if g == 4 else 1285
    W = synth.ternary_weights(M, K, seed=N)
    A = synth.int8_activations(K, N, seed=N + 1)
    pw = v.pack_weights(W, g, device=dev())
    ref = oracle.gemm_i32(W, A)
    for splits in (1, 0):
        acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=v.slot_plan(tpw=tpw, nw=nw, splits=splits))
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), ref)


@pytest.mark.parametrize("g,tpw", [(4, 1), (4, 2), (5, 1), (5, 2)])
def test_slot_adversarial_extremes(v, g, tpw):
    # every field at its bound: all-+1 / all--1 rows against -128 / +127,
    # long K (many SWAR widenings for tpw = 2)
    M, K, N = 96, 23040, 4
    W = np.ones((M, K), np.int8)
    W[1::2] = -1
    W[2::4] = 0
    A = np.full((K, N), -128, np.int8)
    A[:, 1::2] = 127
    pw = v.pack_weights(W, g, device=dev())
    for splits in (1, 7):
        acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=v.slot_plan(tpw=tpw, splits=splits))
        ref = oracle.gemm_i32(W, A)
        assert np.array_equal(acc.cpu().numpy(), ref)
    assert ref.min() == -128 * K


@pytest.mark.parametrize("M,K,N,g", [(6912, 2560, 1, 4), (1000, 1300, 7, 4), (2100, 1280, 16, 5),
                                     (3072, 4096, 16, 4)])
def test_slot_fp32_vector_and_scalar(v, M, K, N, g):
    W = synth.ternary_weights(M, K, seed=M)
    x = synth.activations_f32(K, N, seed=N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights(W, g, device=dev())
    ref = oracle.gemm_i32(W, q)
    o_vec = v.mpgemm_ws(pw, to_dev(q), to_dev(s), synth.W_SCALE, plan=v.slot_plan(tpw=2))
    o_sc = v.mpgemm_scalar_lut(pw, to_dev(q), to_dev(s), synth.W_SCALE)
    o_sc1 = v.mpgemm_scalar_lut(pw, to_dev(q), to_dev(s), synth.W_SCALE, use_ws=False)
    torch.cuda.synchronize()
    for o in (o_vec, o_sc, o_sc1):
        check_fp32(o.cpu().numpy(), ref, s, synth.W_SCALE)


@pytest.mark.parametrize("N,tpw", [(1, 1), (2, 2), (1, 2)])
def test_slot_counted_meeting_extremes(v, N, tpw):
    """Decode-size tiles meet through counted 64-bit atomics (count << 40 |
    sum of partial + 2^31): up to 148 partials per element, each at the int32
    extremes of its K range, positive and negative, must sum exactly, and
    again on the same workspace (each launch leaves its words zero)."""
    M, K, g = 1000, 46080, 4
    W = np.ones((M, K), np.int8)
    W[1::2] = -1
    W[2::4] = 0
    W[3::8, ::3] = 0
    A = np.full((K, N), -128, np.int8)
    A[::5] = 127
    pw = v.pack_weights(W, g, device=dev())
    ref = oracle.gemm_i32(W, A)
    ws = torch.zeros_like(v.workspace(dev()))
    for splits in (2, 45, 148):
        for rep in range(2):
            acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=v.slot_plan(tpw=tpw, splits=splits), ws=ws)
            torch.cuda.synchronize()
            assert np.array_equal(acc.cpu().numpy(), ref), (splits, rep)
    assert ref.min() < -2**20 and ref.max() > 2**20


def test_slot_workspace_stays_clean_and_deterministic(v):
    # the split-K workspace region must be zero again after every launch:
    # alternate shapes and variants on one workspace, compare each repeat
    ws = v.workspace(dev())
    cases = []
    for (M, K, N, g, tpw) in [(3072, 23040, 1, 4, 1), (1100, 2560, 17, 4, 2), (2100, 1280, 3, 5, 2)]:
        W = synth.ternary_weights(M, K, seed=K)
        A = synth.int8_activations(K, N, seed=N)
        cases.append((v.pack_weights(W, g, device=dev()), to_dev(A), tpw, oracle.gemm_i32(W, A)))
    for rep in range(3):
        for pw, Ad, tpw, ref in cases:
            acc = v.mpgemm_acc_ws(pw, Ad, plan=v.slot_plan(tpw=tpw), ws=ws)
            assert np.array_equal(acc.cpu().numpy(), ref)


def test_planner_uses_slot_for_small_n(v):
    # decode shapes go to K2 when a workspace is available, K1 otherwise stays valid
    p1 = v.plan_ws(3072, 23040, 1, 4)
    p16 = v.plan_ws(3072, 23040, 16, 4)
    assert p1.slot == 1 and p16.slot == 1
    assert p1.splits > 1 and p1.grid_ctas <= 148 * 2
    p256 = v.plan_ws(6912, 2560, 256, 4)
    assert p256.slot == 0 and p256.n_cta in (64, 32)  # K1 (64-token) or K1-32 tiles


@pytest.mark.parametrize("N,g", [(1, 4), (16, 4), (1, 5), (4, 5), (64, 4)])
def test_config4_full_size_slot_sampled(v, N, g):
    """BASELINE.json config 4 (Falcon3-10B FFN-down, 3072 x 23040) at decode
    token counts through the auto-planned workspace path (K2), GPU quantizer
    and device packer as bench.py runs them; sampled rows vs the oracle."""
    M, K = 3072, 23040
    seed = 4000 + N
    W = synth.ternary_weights(M, K, seed=seed)
    x = synth.activations_f32(K, N, seed=seed + 1)
    q, s = v.quantize(to_dev(x))
    pw = v.pack_weights_device(to_dev(W), g)
    out = v.mpgemm_ws(pw, q, s, synth.W_SCALE)
    o_sc = v.mpgemm_scalar_lut(pw, q, s, synth.W_SCALE)
    torch.cuda.synchronize()
    qr, sr = oracle.quantize(x)
    assert np.array_equal(q.cpu().numpy(), qr)
    pick = np.unique(np.concatenate([[0, M - 1], synth.rng(seed + 2).integers(0, M, size=40)]))
    acc_ref = oracle.gemm_i32(W[pick], qr)
    check_fp32(out.cpu().numpy()[pick], acc_ref, sr, synth.W_SCALE)
    check_fp32(o_sc.cpu().numpy()[pick], acc_ref, sr, synth.W_SCALE)


def test_north_star_mpgemm_uses_library_workspace(v):
    """vlut_mpgemm (no workspace argument) reaches the K2 decode path through
    the library's per-stream workspace: config 4 shape at N = 1 and 16, two
    streams, repeated calls -- all equal to the oracle."""
    M, K = 3072, 23040
    W = synth.ternary_weights(M, K, seed=9)
    pw = v.pack_weights(W, 4, device=dev())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for N in (1, 16):
        x = synth.activations_f32(K, N, seed=N)
        q, s = oracle.quantize(x)
        qd, sd = to_dev(q), to_dev(s)
        outs = []
        for st in streams:
            with torch.cuda.stream(st):
                for _ in range(2):
                    o = v.mpgemm(pw, qd, sd, synth.W_SCALE, stream=st)
                outs.append(o)
        torch.cuda.synchronize()
        pick = np.unique(np.concatenate([[0, M - 1], synth.rng(N).integers(0, M, size=40)]))
        ref = oracle.gemm_i32(W[pick], q)
        for o in outs:
            check_fp32(o.cpu().numpy()[pick], ref, s, synth.W_SCALE)


def test_north_star_mpgemm_under_graph_capture(v):
    """First vlut_mpgemm call on a stream inside a CUDA graph capture: the
    library must not allocate its workspace there (it falls back to the
    cluster schedules); the captured graph replays correctly."""
    M, K, N = 700, 1280, 8
    W = synth.ternary_weights(M, K, seed=21)
    x = synth.activations_f32(K, N, seed=22)
    q, s = oracle.quantize(x)
    pw = v.pack_weights(W, 4, device=dev())
    qd, sd = to_dev(q), to_dev(s)
    out = torch.empty((M, N), device=dev())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        v.mpgemm(pw, qd, sd, synth.W_SCALE, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    check_fp32(out.cpu().numpy(), oracle.gemm_i32(W, q), s, synth.W_SCALE)


@pytest.mark.parametrize("M,K,g,kind", [(3072, 23040, 4, "normal"), (3072, 23040, 5, "normal"),
                                        (6912, 2560, 4, "normal"), (1000, 1300, 4, "normal"),
                                        (70, 85, 5, "normal"), (2100, 1283, 5, "padk"),
                                        (700, 640, 4, "zeros"), (700, 640, 4, "huge"),
                                        (1000, 1300, 4, "unaligned")])
def test_fused_decode_matches_oracle(v, M, K, g, kind):
    """vlut_mpgemm_decode (N = 1): quantization inside the K2 decode kernel.
    The scale and the fp32 output must be bit-identical to the oracle's
    quantize -> int32 GEMM -> fp32 dequant, for ragged M / K, a zero-padded
    last g = 5 group, an all-zero token (scale 1), values at the int8 clamp and
    an unaligned x (scalar absmax path)."""
    W = synth.ternary_weights(M, K, seed=M + K)
    x = synth.activations_f32(K, 1, seed=K)[:, 0].copy()
    if kind == "zeros":
        x[:] = 0.0
    elif kind == "huge":
        x *= 1e30
        x[::7] = -3e38
    pw = v.pack_weights(W, g, device=dev(), pad_k=(kind == "padk"))
    q, s = oracle.quantize(x[:, None])
    ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)[:, 0]
    if kind == "unaligned":
        buf = torch.zeros(K + 1, dtype=torch.float32, device=dev())
        buf[1:] = to_dev(x)
        xd = buf[1:]
    else:
        xd = to_dev(x)
    for rep in range(2):  # the workspace words must be zero again after each launch
        out, sc = v.mpgemm_decode(pw, xd, synth.W_SCALE)
        torch.cuda.synchronize()
        assert np.array_equal(sc.cpu().numpy().view(np.int32), s.view(np.int32)), rep
        assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32)), rep


def test_fused_decode_global_code_path(v, monkeypatch):
    """The builders' fallback (each feature quantized from global memory when
    a CTA's K slice does not fit the activation ring), forced on."""
    monkeypatch.setenv("VLUT_DECODE_NO_RING", "1")
    for (M, K, g) in [(3072, 23040, 4), (2100, 1283, 5)]:
        W = synth.ternary_weights(M, K, seed=K)
        x = synth.activations_f32(K, 1, seed=M)[:, 0].copy()
        pw = v.pack_weights(W, g, device=dev(), pad_k=(K % g != 0))
        q, s = oracle.quantize(x[:, None])
        ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)[:, 0]
        out, sc = v.mpgemm_decode(pw, to_dev(x), synth.W_SCALE)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32))


def test_fused_decode_equals_quantize_then_scalar_lut(v):
    """The fused step and the two-launch step (quantize, then the scalar-LUT
    mpGeMM) are the same computation: identical bits, chained over 5 layers
    where each layer's output is the next one's input."""
    M = K = 2560
    pws = [v.pack_weights(synth.ternary_weights(M, K, seed=900 + i), 4, device=dev())
           for i in range(5)]
    x = to_dev(synth.activations_f32(K, 1, seed=31)[:, 0].copy())
    a = b = x
    for pw in pws:
        a, _ = v.mpgemm_decode(pw, a, synth.W_SCALE)
        qb, sb = v.quantize(b[:, None].contiguous())
        b = v.mpgemm_scalar_lut(pw, qb, sb, synth.W_SCALE)[:, 0].contiguous()
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
