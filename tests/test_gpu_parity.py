"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north star): int32 accumulators bit-exact; fp32 outputs within 1e-6
relative error of the fp64 definition (and, by fixed op order, bit-identical
to the oracle's fp32 dequant); quantizer codes and scales bit-exact.
"""
import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

REL_TOL = 1e-6  # north star: <= 1e-6 relative error on fp32 outputs


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


ALL_PLANS = [(w, s) for w in (8, 12, 16) for s in (1, 2, 3, 4, 5, 6, 7, 8)]


# ------------------------------------------------------------------ quantizer
@pytest.mark.parametrize("K,N", [(1, 1), (5, 3), (512, 8), (2560, 257), (6912, 64)])
def test_quantize_bit_exact(v, K, N):
    x = synth.activations_f32(K, N, seed=K + N)
    if N > 2:
        x[:, 1] = 0.0          # zero column -> scale 1
        x[:, 2] *= 1e-30       # tiny values
    q, s = v.quantize(to_dev(x))
    qr, sr = oracle.quantize(x)
    assert np.array_equal(s.cpu().numpy().view(np.int32), sr.view(np.int32))
    assert np.array_equal(q.cpu().numpy(), qr)


@pytest.mark.parametrize("cluster", [1, 2, 4, 8])
@pytest.mark.parametrize("K,N", [(2560, 256), (5, 3), (6912, 40), (23040, 16), (3, 1)])
def test_quantize_caller_cluster_bit_exact(v, K, N, cluster):
    """vlut_quantize_ex: every caller-chosen K3 cluster size gives the
    oracle's codes and scales bit for bit (incl. K < cluster, N = 1)."""
    x = synth.activations_f32(K, N, seed=3 * K + N)
    y = synth.activations_f32(K, N, seed=5 * K + N)
    for yy in (None, y):
        q, s = v.quantize(to_dev(x), None if yy is None else to_dev(yy), cluster=cluster)
        qr, sr = oracle.quantize(x if yy is None else (x * yy).astype(np.float32))
        assert np.array_equal(s.cpu().numpy().view(np.int32), sr.view(np.int32))
        assert np.array_equal(q.cpu().numpy(), qr)


def test_quantize_rejects_bad_cluster(v):
    x = to_dev(synth.activations_f32(64, 8, seed=1))
    for c in (-1, 3, 16):
        with pytest.raises(v.VlutError):
            v.quantize(x, cluster=c)


@pytest.mark.parametrize("K,N", [(2560, 1), (23040, 1), (6912, 2), (1000, 4), (4096, 8),
                                 (8192, 16), (12, 16), (4, 1), (65536, 2)])
@pytest.mark.parametrize("with_y", [False, True])
def test_quantize_small_n_flat_path(v, K, N, with_y):
    """Decode shapes (N in {1,2,4,8,16}: the flat K3f kernel), plain and
    x * y (config 5's gate (.) up glue): codes and scales bit-exact; a zero
    token column gets scale 1 and zero codes."""
    x = synth.activations_f32(K, N, seed=K + 7 * N)
    y = synth.activations_f32(K, N, seed=K + 9 * N) if with_y else None
    if N > 1:
        x[:, N - 1] = 0.0
    q, s = v.quantize(to_dev(x), None if y is None else to_dev(y))
    xr = x if y is None else (x * y).astype(np.float32)
    qr, sr = oracle.quantize(np.ascontiguousarray(xr))
    torch.cuda.synchronize()
    assert np.array_equal(s.cpu().numpy().view(np.int32), sr.view(np.int32))
    assert np.array_equal(q.cpu().numpy(), qr)


def test_quantize_half_boundaries(v):
    """Values whose quotient x / s sits on, or a few ulps around, a k + 1/2
    rounding boundary for every k in [-127, 126] and several scales: codes
    must be round-half-away of the IEEE quotient fl(x / s), as the oracle's
    (any shortcut through a reciprocal would differ on some of these)."""
    rng = synth.rng(77)
    N = 24
    amax = np.float32(rng.uniform(0.01, 50.0, N)).astype(np.float32)
    amax[0], amax[1] = np.float32(127.0), np.float32(1.0)
    cols = []
    for n in range(N):
        s = np.float32(amax[n] / np.float32(127.0))
        col = [amax[n], -amax[n]]
        for k in range(-127, 127):
            b = np.float32(np.float32(k + 0.5) * s)
            for d in (-3, -2, -1, 0, 1, 2, 3):
                x = b
                for _ in range(abs(d)):
                    x = np.nextafter(x, np.float32(np.inf if d > 0 else -np.inf), dtype=np.float32)
                if abs(x) <= amax[n]:
                    col.append(x)
        cols.append(np.array(col, np.float32))
    K = max(len(c) for c in cols)
    x = np.zeros((K, N), np.float32)
    for n, c in enumerate(cols):
        x[:len(c), n] = c
    q, s = v.quantize(to_dev(x))
    qr, sr = oracle.quantize(x)
    assert np.array_equal(s.cpu().numpy().view(np.int32), sr.view(np.int32))
    assert np.array_equal(q.cpu().numpy(), qr)


def test_quantize_mul_bit_exact(v):
    K, N = 700, 96
    a = synth.activations_f32(K, N, seed=1)
    b = synth.activations_f32(K, N, seed=2)
    q, s = v.quantize(to_dev(a), to_dev(b))
    qr, sr = oracle.quantize((a * b).astype(np.float32))
    assert np.array_equal(s.cpu().numpy(), sr) and np.array_equal(q.cpu().numpy(), qr)


# ------------------------------------------------------------------ packer
@pytest.mark.parametrize("M,K,g", [(1, 4, 4), (33, 200, 4), (100, 85, 5), (384, 2560, 4)])
def test_pack_roundtrip_and_device_packer(v, M, K, g):
    W = synth.ternary_weights(M, K, seed=M + K)
    pw = v.pack_weights(W, g, device=dev())
    assert np.array_equal(v.unpack_weights_host(pw), W)
    pd = v.pack_weights_device(to_dev(W), g)
    torch.cuda.synchronize()
    assert torch.equal(pw.payload, pd.payload)


def test_pack_rejects_invalid_trit(v):
    W = np.zeros((4, 8), np.int8)
    W[2, 5] = -2
    with pytest.raises(v.VlutError) as e:
        v.pack_weights(W, 4, device=dev())
    assert e.value.name == "VLUT_ERR_INVALID_TRIT"


# ------------------------------------------------------------------ mpGeMM, exact int32
SHAPES = [
    # (M, K, N, g) -- tails in every dimension, several tiles
    (1, 4, 1, 4), (7, 20, 3, 4), (32, 64, 64, 4), (33, 68, 65, 4), (100, 512, 8, 4),
    (256, 512, 8, 4), (385, 1024, 130, 4), (520, 1280, 63, 4), (1000, 260, 256, 4),
    (5, 5, 1, 5), (70, 85, 17, 5), (129, 640, 64, 5), (400, 1280, 100, 5), (777, 2560, 200, 5),
]


@pytest.mark.parametrize("M,K,N,g", SHAPES)
def test_mpgemm_acc_bit_exact_default_plan(v, M, K, N, g):
    W = synth.ternary_weights(M, K, seed=3 * M + K)
    A = synth.int8_activations(K, N, seed=N + 17)  # full int8 range incl. -128
    pw = v.pack_weights(W, g, device=dev())
    acc = v.mpgemm_acc(pw, to_dev(A))
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), oracle.gemm_i32(W, A))


@pytest.mark.parametrize("g", [4, 5])
@pytest.mark.parametrize("warps,splits", ALL_PLANS)
def test_mpgemm_acc_every_plan(v, g, warps, splits):
    M, K, N = 700, 64 * g * 5 + 4 * g, 150  # 5.25 K-tiles: ragged split ranges
    W = synth.ternary_weights(M, K, seed=11)
    A = synth.int8_activations(K, N, seed=12)
    pw = v.pack_weights(W, g, device=dev())
    acc = v.mpgemm_acc(pw, to_dev(A), plan=v.LaunchPlan(warps, splits))
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), oracle.gemm_i32(W, A))


# ------------------------------------------------------------------ K1-32 (32-token tiles)
SHAPES32 = [
    # (M, K, N, g) -- N % 16 == 0 (TMA staging); 16-token N tails, M / K tails
    (1, 4, 16, 4), (33, 68, 48, 4), (385, 1024, 144, 4), (520, 1280, 32, 4), (1000, 260, 256, 4),
    (5, 5, 16, 5), (129, 640, 80, 5), (400, 1280, 112, 5), (777, 2560, 208, 5),
]


@pytest.mark.parametrize("M,K,N,g", SHAPES32)
@pytest.mark.parametrize("warps,splits", [(12, 1), (16, 1), (8, 1), (12, 2), (16, 3), (8, 5)])
def test_mpgemm32_acc_and_fp32(v, M, K, N, g, warps, splits):
    """K1-32 (paired-group tables, 32-token tiles): int32 accumulators
    bit-exact, fp32 bit-identical to the oracle's fixed-order dequant, for
    every warp count and cluster split (ragged split ranges included)."""
    W = synth.ternary_weights(M, K, seed=5 * M + K)
    A = synth.int8_activations(K, N, seed=N + 29)  # full int8 range incl. -128
    s = synth.token_scales(N, seed=N)
    pw = v.pack_weights(W, g, device=dev())
    plan = v.LaunchPlan(warps, splits, n_cta=32)
    acc = v.mpgemm_acc(pw, to_dev(A), plan=plan)
    out = v.mpgemm_ex(pw, to_dev(A), to_dev(s), synth.W_SCALE, plan=plan)
    torch.cuda.synchronize()
    ref = oracle.gemm_i32(W, A)
    assert np.array_equal(acc.cpu().numpy(), ref)
    check_fp32(out.cpu().numpy(), ref, s, synth.W_SCALE)


@pytest.mark.parametrize("g", [4, 5])
def test_mpgemm32_adversarial_extremes(v, g):
    M, K, N = 64, 23040, 64
    W = np.ones((M, K), np.int8)
    W[1::2] = -1
    W[2::4] = 0
    A = np.full((K, N), -128, np.int8)
    A[:, 1::2] = 127
    A[:, 2::4] = 0
    pw = v.pack_weights(W, g, device=dev())
    acc = v.mpgemm_acc(pw, to_dev(A), plan=v.LaunchPlan(12, 1, n_cta=32)).cpu().numpy()
    ref = oracle.gemm_i32(W, A)
    assert np.array_equal(acc, ref)


def test_mpgemm32_rejects_unsupported(v):
    """32-token tiles need N % 16 == 0 and the plain epilogue."""
    M, K, g = 64, 64, 4
    pw = v.pack_weights(synth.ternary_weights(M, K, seed=1), g, device=dev())
    A = to_dev(synth.int8_activations(K, 24, seed=2))
    with pytest.raises(v.VlutError) as e:
        v.mpgemm_acc(pw, A, plan=v.LaunchPlan(12, 1, n_cta=32))
    assert e.value.name == "VLUT_ERR_UNSUPPORTED"


@pytest.mark.parametrize("g", [4, 5])
def test_mpgemm_adversarial_extremes(v, g):
    # |acc| up to 128 * K: all +1 weights against all -128 / +127 activations,
    # a long K (many SWAR flushes), every field at its bias bound
    M, K, N = 64, 23040 if g == 4 else 23040, 64
    W = np.ones((M, K), np.int8)
    W[1::2] = -1
    W[2::4] = 0
    A = np.full((K, N), -128, np.int8)
    A[:, 1::2] = 127
    pw = v.pack_weights(W, g, device=dev())
    acc = v.mpgemm_acc(pw, to_dev(A)).cpu().numpy()
    ref = oracle.gemm_i32(W, A)
    assert np.array_equal(acc, ref)
    assert ref.min() == -128 * K or ref.max() == 128 * K


def test_mpgemm_zero_and_negation(v):
    M, K, N = 300, 1024, 128
    A = synth.int8_activations(K, N, seed=5)
    Ad = to_dev(A)
    pz = v.pack_weights(np.zeros((M, K), np.int8), 4, device=dev())
    assert not v.mpgemm_acc(pz, Ad).any().item()
    W = synth.ternary_weights(M, K, seed=6)
    a = v.mpgemm_acc(v.pack_weights(W, 4, device=dev()), Ad)
    b = v.mpgemm_acc(v.pack_weights(-W, 4, device=dev()), Ad)
    assert torch.equal(a, -b)


# ------------------------------------------------------------------ fp32 epilogue
@pytest.mark.parametrize("M,K,N,g", [(256, 512, 8, 4), (385, 1024, 130, 4), (200, 1280, 96, 5)])
def test_mpgemm_fp32_matches_oracle(v, M, K, N, g):
    W = synth.ternary_weights(M, K, seed=M)
    x = synth.activations_f32(K, N, seed=N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights(W, g, device=dev())
    out = v.mpgemm(pw, to_dev(q), to_dev(s), synth.W_SCALE)
    torch.cuda.synchronize()
    check_fp32(out.cpu().numpy(), oracle.gemm_i32(W, q), s, synth.W_SCALE)


def test_unaligned_N_paths(v):
    # N % 16 != 0 (4-byte staging) and N odd (byte staging, scalar stores)
    for N in (4, 12, 9, 1):
        M, K = 96, 256
        W = synth.ternary_weights(M, K, seed=N)
        A = synth.int8_activations(K, N, seed=N + 1)
        s = synth.token_scales(N, seed=N + 2)
        pw = v.pack_weights(W, 4, device=dev())
        out = v.mpgemm(pw, to_dev(A), to_dev(s), 0.5)
        acc = v.mpgemm_acc(pw, to_dev(A))
        torch.cuda.synchronize()
        ref = oracle.gemm_i32(W, A)
        assert np.array_equal(acc.cpu().numpy(), ref)
        check_fp32(out.cpu().numpy(), ref, s, 0.5)


def test_determinism_across_plans(v):
    M, K, N = 1536, 2560, 256
    W = synth.ternary_weights(M, K, seed=2, p_zero=0.4)
    A = synth.int8_activations(K, N, seed=3)
    s = synth.token_scales(N, seed=4)
    pw = v.pack_weights(W, 4, device=dev())
    Ad, sd = to_dev(A), to_dev(s)
    outs = [v.mpgemm_ex(pw, Ad, sd, 0.02, plan=v.LaunchPlan(w, sp)) for w, sp in ALL_PLANS]
    outs.append(v.mpgemm(pw, Ad, sd, 0.02))
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32))


# ------------------------------------------------------------------ full BASELINE sizes, sampled
def sampled_rows_check(v, M, K, N, g, seed, p_zero=None, rows=48):
    W = synth.ternary_weights(M, K, seed=seed, p_zero=p_zero)
    x = synth.activations_f32(K, N, seed=seed + 1)
    xd = to_dev(x)
    q, s = v.quantize(xd)            # GPU quantizer, as bench.py runs it
    pw = v.pack_weights_device(to_dev(W), g)
    out = v.mpgemm(pw, q, s, synth.W_SCALE)
    torch.cuda.synchronize()
    qr, sr = oracle.quantize(x)
    assert np.array_equal(q.cpu().numpy(), qr) and np.array_equal(s.cpu().numpy(), sr)
    r = synth.rng(seed + 2)
    pick = np.unique(np.concatenate([[0, M - 1], r.integers(0, M, size=rows)]))
    acc_ref = oracle.gemm_i32(W[pick], qr)
    check_fp32(out.cpu().numpy()[pick], acc_ref, sr, synth.W_SCALE)


def test_config2_full_size_sampled(v):
    c = synth.CONFIGS[2]
    lin = c.linears[0]
    sampled_rows_check(v, lin.M, lin.K, 256, 4, seed=2000, p_zero=0.4)


@pytest.mark.parametrize("N,g", [(256, 4), (1024, 5), (4096, 4), (1, 4), (16, 5)])
def test_config4_full_size_sampled(v, N, g):
    sampled_rows_check(v, 3072, 23040, N, g, seed=4000 + N, rows=12 if N >= 1024 else 32)


@pytest.mark.parametrize("j", range(5))
def test_config3_linears_sampled(v, j):
    lin = synth.CONFIGS[3].linears[j]
    sampled_rows_check(v, lin.M, lin.K, 1024, 4, seed=3000 + j, rows=8)


# ------------------------------------------------------------------ config 5 chain (a7 + a2-a6)
def test_config5_chain_30_layers_sampled_tokens(v):
    """BASELINE.md's parity bar for config 5: bit-exact int8 re-quantization
    along the whole 30-layer chain.  Full BitNet-2B-shaped layer weights and
    N = 2048 tokens on the GPU, through BOTH the plain chain (LayerChain) and
    the fused re-quantization chain (LayerChain(fused=True), f1); the oracle
    re-runs the chain (oracle.config5_layer, reading c14) on 16 sampled token
    columns -- per-token quantization makes columns independent -- and codes
    and scales must be bit-identical after every one of the 30 layers.  The
    overlapped f1 chain (4 token chunks, exchange on a side stream) must
    equal both on every token.
    Layers are built one at a time (weights generated, packed, checked, freed)."""
    from paper_2512_06443_b200.sharded import LayerChain, RowShardedLinear
    cfg = synth.CONFIGS[5]
    N, n_layers = 2048, cfg.layers
    assert n_layers == 30
    x = synth.activations_f32(2560, N, synth.act_seed(cfg, N))
    xq, xs = v.quantize(to_dev(x))
    fq, fs = xq, xs
    kq, ks = xq, xs
    cols = np.unique(np.concatenate([[0, N - 1], synth.rng(5).integers(0, N, size=14)]))
    q_ref, s_ref = oracle.quantize(np.ascontiguousarray(x[:, cols]))
    for l in range(n_layers):
        lw = [w for _, w in synth.config_weights(cfg, l)]
        lay = [RowShardedLinear(w, 4, synth.W_SCALE, device=dev(), device_pack=True) for w in lw]
        xq, xs = LayerChain([lay]).layer(0, xq, xs)
        fq, fs = LayerChain([lay], fused=True).layer(0, fq, fs)
        # f1 overlapped: 4 token chunks, exchange/quantize on a side stream
        kq, ks = LayerChain([lay], fused=True, chunks=4)(kq, ks)
        q_ref, s_ref = oracle.config5_layer(lw, synth.W_SCALE, q_ref, s_ref, q_rows=2560)
        torch.cuda.synchronize()
        assert np.array_equal(xs.cpu().numpy()[cols].view(np.int32), s_ref.view(np.int32)), l
        assert np.array_equal(xq.cpu().numpy()[:, cols], q_ref), l
        assert np.array_equal(fs.cpu().numpy()[cols].view(np.int32), s_ref.view(np.int32)), l
        assert np.array_equal(fq.cpu().numpy()[:, cols], q_ref), l
        # the two chains agree on every token, not only the sampled ones
        assert torch.equal(xq, fq) and torch.equal(xs.view(torch.int32), fs.view(torch.int32)), l
        assert torch.equal(xq, kq) and torch.equal(xs.view(torch.int32), ks.view(torch.int32)), l
        del lay, lw


def test_bench_workload_full_matrix_exact_plan(v):
    """The launch bench.py times (BASELINE.json configs[1], 6912 x 2560,
    N = 256, g = 4, P(0) = 0.4 weights; the plan vlut_plan_ws picks, plain
    epilogue, the library-chosen schedule of vlut_mpgemm too), checked on the
    WHOLE 6912 x 256 output against the oracle: int32 accumulators bit-exact
    and fp32 outputs bit-identical to the fixed-order fp32 dequant (and within
    1e-6 of fp64)."""
    cfg = synth.CONFIGS[2]
    lin = cfg.linears[0]
    M, K, N, g = lin.M, lin.K, cfg.N[0], cfg.g[0]
    W = synth.ternary_weights(M, K, synth.weight_seed(cfg, 0, 0), cfg.p_zero)
    x = synth.activations_f32(K, N, synth.act_seed(cfg, N))
    xd = to_dev(x)
    q, s = v.quantize(xd)
    pw = v.pack_weights_device(to_dev(W), g)
    plan = v.plan_ws(M, K, N, g)
    out = v.mpgemm_ws(pw, q, s, synth.W_SCALE, plan=plan, ws=v.workspace(dev()))
    out_ns = v.mpgemm(pw, q, s, synth.W_SCALE)
    acc = v.mpgemm_acc_ws(pw, q, plan=plan, ws=v.workspace(dev()))
    torch.cuda.synchronize()
    q_ref, s_ref = oracle.quantize(x)
    assert np.array_equal(q.cpu().numpy(), q_ref)
    assert np.array_equal(s.cpu().numpy().view(np.int32), s_ref.view(np.int32))
    acc_ref = oracle.gemm_i32(W, q_ref)
    assert np.array_equal(acc.cpu().numpy(), acc_ref)
    check_fp32(out.cpu().numpy(), acc_ref, s_ref, synth.W_SCALE)
    check_fp32(out_ns.cpu().numpy(), acc_ref, s_ref, synth.W_SCALE)


def test_parity_harness_detects_single_trit_corruption(v):
    """an injected single-trit corruption in the payload must be
    reported.  One payload byte of a real (row, group) is changed ON THE
    DEVICE to another valid index (one trit flipped); the oracle comparison
    must then fail exactly on that output row, and restoring the byte must
    make it pass again.  Proves the parity checks above can fail."""
    M, K, N, g = 300, 640, 96, 4
    W = synth.ternary_weights(M, K, seed=481)
    x = synth.activations_f32(K, N, seed=482)
    q, s = oracle.quantize(x)
    qd, sd = to_dev(q), to_dev(s)
    pw = v.pack_weights(W, g, device=dev())
    ref = oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE)
    ok = v.mpgemm(pw, qd, sd, synth.W_SCALE)
    torch.cuda.synchronize()
    assert np.array_equal(ok.cpu().numpy().view(np.int32), ref.view(np.int32))
    m, k = 123, 37                       # row 123, group 37 (features 148..151)
    kt, j = divmod(k, 16)
    off = (kt * pw.desc.m_pad + m) * 16 + j
    old = int(pw.payload[off].item())
    assert old == oracle.pack_group(W[m, k * g:(k + 1) * g])
    trits = oracle.unpack_index(old, g).copy()
    trits[0] = 1 if trits[0] != 1 else -1     # flip one trit
    pw.payload[off] = oracle.pack_group(trits)
    # vlut.h: the payload must not be written by the kernel launched just
    # before the mpGeMM (weights are staged before griddepcontrol.wait)
    torch.cuda.synchronize()
    bad = v.mpgemm(pw, qd, sd, synth.W_SCALE)
    torch.cuda.synchronize()
    diff_rows = np.unique(np.nonzero(bad.cpu().numpy().view(np.int32) != ref.view(np.int32))[0])
    assert diff_rows.tolist() == [m]     # reported, and only where corrupted
    pw.payload[off] = old
    torch.cuda.synchronize()
    again = v.mpgemm(pw, qd, sd, synth.W_SCALE)
    torch.cuda.synchronize()
    assert np.array_equal(again.cpu().numpy().view(np.int32), ref.view(np.int32))
    # a byte outside [0, 3^g) is a corrupt payload for the host unpacker
    pw.payload[off] = 81
    with pytest.raises(v.VlutError) as e:
        v.unpack_weights_host(pw)
    assert e.value.name == "VLUT_ERR_INVALID_TRIT"


# ------------------------------------------------------------------ mixed g=5/g=4 schedule (f2)
@pytest.mark.parametrize("M,K,N", [(300, 4096, 130), (77, 22, 5), (500, 6912, 64), (64, 20, 16),
                                   (128, 16, 32)])
def test_mpgemm_mixed_matches_oracle(v, M, K, N):
    W = synth.ternary_weights(M, K, seed=K)
    x = synth.activations_f32(K, N, seed=N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights_mixed(W, device=dev())
    k5, k4 = v.group_schedule(K)
    assert (pw.w5 is None) == (k5 == 0) and (pw.w4 is None) == (k4 == 0)
    out = v.mpgemm_mixed(pw, to_dev(q), to_dev(s), synth.W_SCALE)
    out_ws = v.mpgemm_mixed(pw, to_dev(q), to_dev(s), synth.W_SCALE, ws=v.workspace(dev()))
    torch.cuda.synchronize()
    check_fp32(out.cpu().numpy(), oracle.gemm_i32(W, q), s, synth.W_SCALE)
    assert torch.equal(out.view(torch.int32), out_ws.view(torch.int32))
    # bits per weight of the logical mixed packing (near 1.6 for common shapes)
    bpw = 8.0 * (k5 / 5 + k4 / 4) / K
    assert bpw == pytest.approx(oracle.mixed_bits_per_weight(K))
    if K >= 100:
        assert bpw < 1.61


# ------------------------------------------------------------------ fused transpositions (f3)
@pytest.mark.parametrize("K,N", [(2560, 256), (6912, 40), (17, 3), (4096, 1000), (14336, 64)])
def test_quantize_t_feature_major_input(v, K, N):
    x = synth.rng(K + N).standard_normal((N, K), dtype=np.float32)  # framework layout [N][K]
    if N > 2:
        x[1] = 0.0
    q, s = v.quantize_t(to_dev(x))
    qr, sr = oracle.quantize(np.ascontiguousarray(x.T))
    assert np.array_equal(s.cpu().numpy().view(np.int32), sr.view(np.int32))
    assert np.array_equal(q.cpu().numpy(), qr)
    y = synth.rng(K).standard_normal((N, K), dtype=np.float32)
    q2, s2 = v.quantize_t(to_dev(x), to_dev(y))
    qr2, sr2 = oracle.quantize(np.ascontiguousarray((x * y).astype(np.float32).T))
    assert np.array_equal(s2.cpu().numpy(), sr2) and np.array_equal(q2.cpu().numpy(), qr2)


@pytest.mark.parametrize("M,K,N", [(6912, 2560, 256), (385, 1024, 130), (100, 512, 9)])
def test_mpgemm_feature_major_output_and_linear(v, M, K, N):
    W = synth.ternary_weights(M, K, seed=M + 1)
    x_nk = synth.rng(N).standard_normal((N, K), dtype=np.float32)
    pw = v.pack_weights(W, 4, device=dev())
    qr, sr = oracle.quantize(np.ascontiguousarray(x_nk.T))
    ref32 = oracle.dequant_f32(oracle.gemm_i32(W, qr), sr, synth.W_SCALE)  # [M][N]
    out_t = v.mpgemm_layout(pw, to_dev(qr), to_dev(sr), synth.W_SCALE, feature_major=True)
    y = v.linear(pw, to_dev(x_nk), synth.W_SCALE)
    torch.cuda.synchronize()
    assert out_t.shape == (N, M) and y.shape == (N, M)
    assert np.array_equal(out_t.cpu().numpy().view(np.int32), np.ascontiguousarray(ref32.T).view(np.int32))
    assert np.array_equal(y.cpu().numpy().view(np.int32), np.ascontiguousarray(ref32.T).view(np.int32))


# ------------------------------------------------------------------ stream-K schedule
@pytest.mark.parametrize("M,K,N,g", SHAPES + [(6912, 2560, 256, 4), (2560, 2560, 2048, 4)])
@pytest.mark.parametrize("warps,rpt", [(8, 1), (12, 1), (16, 1), (12, 2), (8, 2)])
def test_streamk_acc_bit_exact(v, M, K, N, g, warps, rpt):
    # rpt = output rows per lookup thread (m_cta = 32 * warps * rpt)
    W = synth.ternary_weights(M, K, seed=5 * M + K)
    A = synth.int8_activations(K, N, seed=N + 3)
    pw = v.pack_weights_device(to_dev(W), g)
    acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=v.LaunchPlan(warps, 1, m_cta=32 * warps * rpt, streamk=1))
    torch.cuda.synchronize()
    if M * N * K > 2e9:  # large case: sampled rows
        pick = np.unique(synth.rng(1).integers(0, M, size=24))
        assert np.array_equal(acc.cpu().numpy()[pick], oracle.gemm_i32(W[pick], A))
    else:
        assert np.array_equal(acc.cpu().numpy(), oracle.gemm_i32(W, A))


@pytest.mark.parametrize("M,K,N,g", SHAPES32 + [(6912, 2560, 256, 4), (2560, 2560, 2048, 4),
                                               (3072, 4600, 512, 5)])
@pytest.mark.parametrize("warps,rpt", [(12, 1), (16, 1), (12, 2)])
def test_streamk32_acc_and_fp32(v, M, K, N, g, warps, rpt):
    """K1-32 under stream-K (32-token tiles, 1 or 2 rows per lookup thread,
    split tiles combined through workspace partials): int32 bit-exact, fp32
    bit-identical to the oracle's fixed-order dequant."""
    W = synth.ternary_weights(M, K, seed=7 * M + K)
    A = synth.int8_activations(K, N, seed=N + 41)
    s = synth.token_scales(N, seed=N + 1)
    pw = v.pack_weights_device(to_dev(W), g)
    plan = v.LaunchPlan(warps, 1, m_cta=32 * warps * rpt, n_cta=32, streamk=1)
    ws = torch.zeros_like(v.workspace(dev()))
    acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=plan, ws=ws)
    out = v.mpgemm_ws(pw, to_dev(A), to_dev(s), synth.W_SCALE, plan=plan, ws=ws)
    torch.cuda.synchronize()
    if M * N * K > 2e9:  # large case: sampled rows
        pick = np.unique(synth.rng(2).integers(0, M, size=24))
        ref = oracle.gemm_i32(W[pick], A)
        assert np.array_equal(acc.cpu().numpy()[pick], ref)
        check_fp32(out.cpu().numpy()[pick], ref, s, synth.W_SCALE)
    else:
        ref = oracle.gemm_i32(W, A)
        assert np.array_equal(acc.cpu().numpy(), ref)
        check_fp32(out.cpu().numpy(), ref, s, synth.W_SCALE)


@pytest.mark.parametrize("M,K,N,g,rpt", [(3072, 23040, 256, 5, 2), (3072, 4600, 64, 5, 1),
                                         (3072, 4600, 512, 5, 1),
                                         (700, 2560, 96, 4, 2), (128, 140000, 32, 4, 1)])
def test_streamk32_split_meeting_repeated_launches(v, M, K, N, g, rpt):
    """K1-32-SK split tiles meet in fp32 accumulators when there are >= 2
    CTAs per tile (exact: every partial sum is an integer below 2^24; fewer
    CTAs per tile or K >= 131072 keep the int32 partials):
    three launches on one workspace with new activations stay bit-exact, and
    the accumulator region is all zero again after each launch."""
    W = synth.ternary_weights(M, K, seed=M + 3)
    pw = v.pack_weights_device(to_dev(W), g)
    plan = v.LaunchPlan(12, 1, m_cta=384 * rpt, n_cta=32, streamk=1)
    ws = torch.zeros_like(v.workspace(dev()))
    acc_bytes = 148 * 768 * 32 * 4
    big = M * N * K > 2e9
    pick = np.unique(synth.rng(5).integers(0, M, size=16)) if big else np.arange(M)
    for it in range(3):
        A = synth.int8_activations(K, N, seed=50 + it)
        if it == 1:
            A[:] = -128  # extreme partial sums: -128 * (K / 2) per CTA half
        acc = v.mpgemm_acc_ws(pw, to_dev(A), plan=plan, ws=ws)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy()[pick], oracle.gemm_i32(W[pick], A))
        assert int(torch.count_nonzero(ws[-acc_bytes:])) == 0


@pytest.mark.parametrize("M,K,N,g", [(6912, 2560, 256, 4), (3072, 23040, 1024, 5), (385, 1024, 130, 4)])
def test_streamk_fp32_and_planner_identity(v, M, K, N, g):
    W = synth.ternary_weights(M, K, seed=M)
    x = synth.activations_f32(K, N, seed=N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights_device(to_dev(W), g)
    qd, sd = to_dev(q), to_dev(s)
    o_sk = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=v.LaunchPlan(12, 1, streamk=1))
    o_sk2 = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=v.LaunchPlan(12, 1, m_cta=768, streamk=1))
    o_auto = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE)
    o_cl = v.mpgemm(pw, qd, sd, synth.W_SCALE)
    torch.cuda.synchronize()
    assert torch.equal(o_sk.view(torch.int32), o_cl.view(torch.int32))
    assert torch.equal(o_sk2.view(torch.int32), o_cl.view(torch.int32))
    assert torch.equal(o_auto.view(torch.int32), o_cl.view(torch.int32))
    pick = np.unique(np.concatenate([[0, M - 1], synth.rng(2).integers(0, M, size=16)]))
    check_fp32(o_sk.cpu().numpy()[pick], oracle.gemm_i32(W[pick], q), s, synth.W_SCALE)


# ------------------------------------------------------------------ fused re-quantization (f1)
FUSED_PLANS = {"cluster": None, "auto_ws": "ws", "sk16": (16, 1, 1), "sk12": (12, 1, 1),
               "sk8": (8, 1, 1), "cl12x3": (12, 3, 0), "sk12r2": (12, 1, 1, 768), "sk8r2": (8, 1, 1, 512)}


@pytest.mark.parametrize("M,K,N,rows", [(6912, 2560, 256, 6912), (3840, 2560, 200, 2560),
                                        (100, 512, 9, 37), (2560, 6912, 130, 2560)])
@pytest.mark.parametrize("how", list(FUSED_PLANS))
def test_mpgemm_fused_mul_and_amax(v, M, K, N, rows, how):
    W = synth.ternary_weights(M, K, seed=M + 5)
    x = synth.activations_f32(K, N, seed=N + 5)
    q, s = oracle.quantize(x)
    g = synth.rng(3).standard_normal((M, N), dtype=np.float32)
    pw = v.pack_weights(W, 4, device=dev())
    amax = torch.zeros((N,), dtype=torch.int32, device=dev())
    h = FUSED_PLANS[how]
    plan = (v.LaunchPlan(h[0], h[1], m_cta=h[3] if len(h) > 3 else 0, streamk=h[2])
            if isinstance(h, tuple) else None)
    ws = v.workspace(dev()) if h is not None else None
    out = v.mpgemm_fused(pw, to_dev(q), to_dev(s), synth.W_SCALE, mul_in=to_dev(g), amax=amax,
                         amax_rows=rows, plan=plan, ws=ws)
    torch.cuda.synchronize()
    ref = (oracle.dequant_f32(oracle.gemm_i32(W, q), s, synth.W_SCALE) * g).astype(np.float32)
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32))
    ref_amax = np.abs(ref[:rows]).max(0).astype(np.float32)
    assert np.array_equal(amax.cpu().numpy().view(np.float32), ref_amax)
    # quantize with the fused maxima == the oracle quantizer on those rows
    qq, ss = v.quantize_amax(out[:rows].contiguous(), amax)
    qr, sr = oracle.quantize(np.ascontiguousarray(ref[:rows]))
    torch.cuda.synchronize()
    assert np.array_equal(ss.cpu().numpy(), sr) and np.array_equal(qq.cpu().numpy(), qr)


# ------------------------------------------------------------------ host pipeline (e2e path)
@pytest.mark.parametrize("graph", [False, True])
def test_batch_pipeline_matches_oracle(v, graph):
    """pipeline.BatchPipeline (batch i+1's quantizer on a side stream under
    batch i's mpGeMM, double-buffered codes): every batch's output is
    bit-identical to the oracle, eager and captured in a CUDA graph replayed
    twice with new inputs; weights alternate between two matrices."""
    from paper_2512_06443_b200.pipeline import BatchPipeline
    M, K, N, steps = 1000, 2560, 96, 7
    Ws = [synth.ternary_weights(M, K, seed=90 + i) for i in range(2)]
    pws = [v.pack_weights(W, 4, device=dev()) for W in Ws]
    xs = [to_dev(synth.activations_f32(K, N, seed=100 + i)) for i in range(steps)]
    outs = [torch.full((M, N), float("nan"), device=dev()) for _ in range(steps)]
    bp = BatchPipeline(pws[0], synth.W_SCALE, K, N, dev())
    torch.cuda.synchronize()

    def run():
        bp.reset()
        for i in range(steps):
            bp.submit(xs[i], outs[i], W=pws[i % 2])
        bp.join()

    def check():
        for i in range(steps):
            x = xs[i].cpu().numpy()
            q, s = oracle.quantize(x)
            check_fp32(outs[i].cpu().numpy(), oracle.gemm_i32(Ws[i % 2], q), s, synth.W_SCALE)

    if not graph:
        run()
        torch.cuda.synchronize()
        check()
        return
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        run()
    for rep in range(2):
        for i in range(steps):
            xs[i].copy_(to_dev(synth.activations_f32(K, N, seed=200 + 10 * rep + i)))
            outs[i].fill_(float("nan"))
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        check()


def test_host_pipeline_matches_oracle(v):
    """bench.py's e2e path: pinned fp32 inputs -> HostPipeline (H2D, quantize,
    mpGeMM, D2H on three streams, 2 slots) -> pinned outputs; every step's
    download equals the oracle (different inputs per step catch slot races)."""
    from paper_2512_06443_b200.pipeline import HostPipeline
    M, K, N, g = 700, 1280, 96, 4
    W = synth.ternary_weights(M, K, seed=71)
    pw = v.pack_weights(W, g, device=dev())
    steps = 6
    xs = [synth.activations_f32(K, N, seed=80 + i) for i in range(steps)]
    x_pins = [torch.from_numpy(x).pin_memory() for x in xs]
    o_pins = [torch.empty((M, N), dtype=torch.float32).pin_memory() for _ in range(steps)]
    pipe = HostPipeline(pw, synth.W_SCALE, K, N, dev(), depth=2)
    for i in range(steps):
        pipe.submit(x_pins[i], o_pins[i])
    pipe.synchronize()
    for i in range(steps):
        q, s = oracle.quantize(xs[i])
        check_fp32(o_pins[i].numpy(), oracle.gemm_i32(W, q), s, synth.W_SCALE)


# ------------------------------------------------------------------ fused all-gather epilogue (a8)
@pytest.mark.parametrize("M,K,N,G", [(6912, 2560, 256, 2), (1000, 1280, 100, 3), (700, 260, 64, 8),
                                     (333, 512, 63, 4)])
def test_mpgemm_allgather_emulated_ranks(v, M, K, N, G):
    """Single-process emulation of G ranks (no rank waits on another): rank r
    computes rows [r0, r1) with vlut_mpgemm_allgather into its own buffer and
    the G-1 'peer' buffers; afterwards every buffer holds the full output,
    bit-identical to the oracle, and nothing outside the shards was touched."""
    from paper_2512_06443_b200.sharded import shard_rows
    W = synth.ternary_weights(M, K, seed=M + G)
    x = synth.activations_f32(K, N, seed=N + G)
    q, s = oracle.quantize(x)
    qd, sd = to_dev(q), to_dev(s)
    bufs = [torch.full((M + 4, N), float("nan"), device=dev()) for _ in range(G)]
    for r in range(G):
        r0, r1, _ = shard_rows(M, G, r)
        if r1 <= r0:
            continue
        pw = v.pack_weights(np.ascontiguousarray(W[r0:r1]), 4, device=dev())
        peers = [bufs[p].data_ptr() for p in range(G) if p != r]
        v.mpgemm_allgather(pw, qd, sd, synth.W_SCALE, bufs[r], r0, peers)
    torch.cuda.synchronize()
    ref = oracle.gemm_i32(W, q)
    for b in bufs:
        got = b.cpu().numpy()
        check_fp32(got[:M], ref, s, synth.W_SCALE)
        assert np.isnan(got[M:]).all()


def test_mpgemm_allgather_rejects_bad_peers(v):
    W = synth.ternary_weights(64, 64, seed=1)
    pw = v.pack_weights(W, 4, device=dev())
    A = to_dev(synth.int8_activations(64, 8, seed=2))
    s = to_dev(synth.token_scales(8, seed=3))
    out = torch.empty((64, 8), device=dev())
    with pytest.raises(v.VlutError):
        v.mpgemm_allgather(pw, A, s, 0.02, out, 0, [out.data_ptr() + 4])  # misaligned peer
    with pytest.raises(v.VlutError):
        v.mpgemm_allgather(pw, A, s, 0.02, out, 0, [out.data_ptr()] * 8)  # > 7 peers


class _SingleDeviceMulticast:
    """A multicast object with this one device as its only member (CUDA
    driver API): `mc` is the multicast address, `uc` the unicast mapping of
    the same physical memory.  Raises RuntimeError when unsupported."""

    def __init__(self, nbytes):
        from cuda.bindings import driver as cu
        self.cu = cu
        torch.zeros(1, device=dev())  # primary context current
        idx = torch.cuda.current_device()

        def ok(res, what=""):
            res = res if isinstance(res, tuple) else (res,)
            if res[0] != cu.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"CUDA driver {what}: {res[0]}")
            return res[1] if len(res) == 2 else res[1:]

        d = ok(cu.cuDeviceGet(idx))
        if not ok(cu.cuDeviceGetAttribute(
                cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d)):
            raise RuntimeError("no multicast support")
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = 1
        fd = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        prop.handleTypes = fd
        prop.size = nbytes
        gran = ok(cu.cuMulticastGetGranularity(
            prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "granularity")
        self.size = size = -(-nbytes // gran) * gran
        prop.size = size
        self.mc_handle = ok(cu.cuMulticastCreate(prop), "cuMulticastCreate")
        ok(cu.cuMulticastAddDevice(self.mc_handle, d), "cuMulticastAddDevice")
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = idx
        ap.requestedHandleTypes = fd
        self.mem = ok(cu.cuMemCreate(size, ap, 0), "cuMemCreate")
        ok(cu.cuMulticastBindMem(self.mc_handle, 0, self.mem, 0, size, 0), "cuMulticastBindMem")
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = idx
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.vas = []
        for h in (self.mem, self.mc_handle):
            va = ok(cu.cuMemAddressReserve(size, gran, 0, 0), "cuMemAddressReserve")
            ok(cu.cuMemMap(va, size, 0, h, 0), "cuMemMap")
            ok(cu.cuMemSetAccess(va, size, [acc], 1), "cuMemSetAccess")
            self.vas.append(va)
        self.uc, self.mc = int(self.vas[0]), int(self.vas[1])

    def close(self):
        cu = self.cu
        torch.cuda.synchronize()
        for va in self.vas:
            cu.cuMemUnmap(va, self.size)
            cu.cuMemAddressFree(va, self.size)
        cu.cuMulticastUnbind(self.mc_handle, 0, 0, self.size)
        cu.cuMemRelease(self.mem)
        cu.cuMemRelease(self.mc_handle)


@pytest.mark.parametrize("M,K,N", [(256, 512, 64), (1000, 1280, 100), (333, 512, 63)])
def test_mpgemm_allgather_multicast_single_device(v, M, K, N):
    """vlut_mpgemm_allgather_multicast on real multicast memory (a one-member
    multicast object): two emulated ranks store their row shards through the
    multicast address with multimem.st; the unicast view holds the whole
    output, bit-identical to the oracle, NaN past it."""
    from paper_2512_06443_b200.sharded import shard_rows
    nbytes = (M + 4) * N * 4
    try:
        mcb = _SingleDeviceMulticast(nbytes)
    except (ImportError, RuntimeError) as ex:
        pytest.skip(f"multicast object unavailable: {ex}")
    try:
        view = torch.full(((mcb.size // 4) // N, N), float("nan"), device=dev())
        mcb.cu.cuMemcpy(mcb.uc, view.data_ptr(), view.numel() * 4)
        W = synth.ternary_weights(M, K, seed=M + 7)
        x = synth.activations_f32(K, N, seed=N + 7)
        q, s = oracle.quantize(x)
        qd, sd = to_dev(q), to_dev(s)
        for r in range(2):
            r0, r1, _ = shard_rows(M, 2, r)
            pw = v.pack_weights(np.ascontiguousarray(W[r0:r1]), 4, device=dev())
            v.mpgemm_allgather(pw, qd, sd, synth.W_SCALE, mcb.mc, r0, multicast=True)
        torch.cuda.synchronize()
        mcb.cu.cuMemcpy(view.data_ptr(), mcb.uc, view.numel() * 4)
        torch.cuda.synchronize()
        got = view.cpu().numpy()
        check_fp32(got[:M], oracle.gemm_i32(W, q), s, synth.W_SCALE)
        assert np.isnan(got[M:]).all()
        with pytest.raises(v.VlutError):
            v.mpgemm_allgather(pw, qd, sd, synth.W_SCALE, mcb.mc + 4, 0, multicast=True)
    finally:
        mcb.close()


def test_peer_outputs_symmetric_memory_world1(v):
    """The symmetric-memory plumbing of the fused all-gather on a 1-rank
    NCCL group: allocation, rendezvous, alternating buffers, barrier."""
    import os
    import torch.distributed as dist
    from paper_2512_06443_b200.sharded import PeerOutputs
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev())
    try:
        W = synth.ternary_weights(128, 256, seed=5)
        x = synth.activations_f32(256, 64, seed=6)
        q, s = oracle.quantize(x)
        pw = v.pack_weights(W, 4, device=dev())
        for mode in ("unicast", "auto"):  # auto: the multicast address when supported
            po = PeerOutputs(mode=mode)
            b0, t0, peers0, bar0 = po.get(128, 64, dev())
            b1, t1, peers1, bar1 = po.get(128, 64, dev())
            b2, _, _, _ = po.get(128, 64, dev())
            assert peers0 == [] and peers1 == []
            assert b0.data_ptr() != b1.data_ptr() and b2.data_ptr() == b0.data_ptr()
            b0.fill_(float("nan"))
            v.mpgemm_allgather(pw, to_dev(q), to_dev(s), synth.W_SCALE, t0, 0, peers0,
                               multicast=po.multicast(128, 64))
            bar0()
            torch.cuda.synchronize()
            check_fp32(b0.cpu().numpy(), oracle.gemm_i32(W, q), s, synth.W_SCALE)
            print(mode, "transport:", po.transport(128, 64, dev()))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ padded packing (K % g != 0)
@pytest.mark.parametrize("M,K,g", [(33, 7, 4), (100, 4096, 5), (70, 14, 5), (384, 1283, 5)])
def test_padded_pack_roundtrip_and_device_packer(v, M, K, g):
    W = synth.ternary_weights(M, K, seed=M + K)
    with pytest.raises(v.VlutError) as e:
        v.pack_weights(W, g, device=dev())  # plain packing keeps rejecting g | K
    assert e.value.name == "VLUT_ERR_SHAPE"
    pw = v.pack_weights(W, g, device=dev(), pad_k=True)
    assert np.array_equal(v.unpack_weights_host(pw), W)
    pd = v.pack_weights_device(to_dev(W), g, pad_k=True)
    torch.cuda.synchronize()
    assert torch.equal(pw.payload, pd.payload)


PADDED_PLANS = {"auto": None, "auto_ws": "ws", "cluster12x2": (12, 2, 0, 0),
                "sk16": (16, 1, 1, 0), "sk12r2": (12, 1, 1, 768), "k2": "slot"}


@pytest.mark.parametrize("M,K,N,g", [(385, 4096, 130, 5), (200, 1283, 17, 5), (1000, 6, 5, 4),
                                     (777, 14336, 64, 5), (129, 2561, 256, 4)])
@pytest.mark.parametrize("how", list(PADDED_PLANS))
def test_padded_mpgemm_every_schedule(v, M, K, N, g, how):
    """g = 5 (or 4) over a K that g does not divide: the last group's missing
    features are zero trits and their activation rows read as 0 -- the
    result equals the definition over the true K for every schedule."""
    W = synth.ternary_weights(M, K, seed=K)
    x = synth.activations_f32(K, N, seed=N)
    q, s = oracle.quantize(x)
    pw = v.pack_weights(W, g, device=dev(), pad_k=True)
    qd, sd = to_dev(q), to_dev(s)
    h = PADDED_PLANS[how]
    if h is None:
        out = v.mpgemm(pw, qd, sd, synth.W_SCALE)
        acc = v.mpgemm_acc(pw, qd)
    elif h == "ws":
        out = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE)
        acc = v.mpgemm_acc_ws(pw, qd)
    elif h == "slot":
        if N > 64:
            pytest.skip("K2 covers N <= 64 from staged activations; wider N is tested elsewhere")
        out = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=v.slot_plan(tpw=2))
        acc = v.mpgemm_acc_ws(pw, qd, plan=v.slot_plan(tpw=1, splits=3))
    else:
        plan = v.LaunchPlan(h[0], h[1], m_cta=h[3], streamk=h[2])
        out = v.mpgemm_ws(pw, qd, sd, synth.W_SCALE, plan=plan)
        acc = v.mpgemm_acc_ws(pw, qd, plan=plan)
    torch.cuda.synchronize()
    acc_ref = oracle.gemm_i32(W, q)
    assert np.array_equal(acc.cpu().numpy(), acc_ref)
    check_fp32(out.cpu().numpy(), acc_ref, s, synth.W_SCALE)


def test_output_larger_than_2g_elements(v):
    """M x N > 2^31 output elements (9.6 GB fp32): every offset into out, the
    workspace and the epilogues must be 64-bit.  Sampled rows (first, last,
    random) and the last token column vs the oracle."""
    M, K, N, g = 40000, 20, 60000, 4
    W = synth.ternary_weights(M, K, seed=99)
    A = synth.int8_activations(K, N, seed=98)
    s = synth.token_scales(N, seed=97)
    pw = v.pack_weights(W, g, device=dev())
    Ad, sd = to_dev(A), to_dev(s)
    rows = np.unique(np.concatenate([[0, 1, M - 2, M - 1], synth.rng(5).integers(0, M, size=12)]))
    ref = oracle.dequant_f32(oracle.gemm_i32(W[rows], A), s, synth.W_SCALE)
    for how in ("auto", "cluster", "streamk"):
        if how == "auto":
            out = v.mpgemm(pw, Ad, sd, synth.W_SCALE)
        elif how == "cluster":
            out = v.mpgemm_ex(pw, Ad, sd, synth.W_SCALE)
        else:
            out = v.mpgemm_ws(pw, Ad, sd, synth.W_SCALE, plan=v.LaunchPlan(12, 1, m_cta=768, streamk=1))
        torch.cuda.synchronize()
        got = out[torch.from_numpy(rows).to(dev())].cpu().numpy()
        assert np.array_equal(got.view(np.int32), ref.view(np.int32)), how
        del out
        torch.cuda.empty_cache()


@pytest.mark.parametrize("a_off,o_off", [(1, 0), (4, 4), (8, 0), (0, 4)])
@pytest.mark.parametrize("N", [64, 256])
def test_misaligned_device_pointers(v, a_off, o_off, N):
    """A and out at byte offsets that break 16-byte alignment: the kernels
    fall back to 4-/1-byte activation staging (no TMA) and scalar stores;
    every schedule still bit-exact."""
    M, K, g = 700, 1280, 4
    W = synth.ternary_weights(M, K, seed=a_off + N)
    A = synth.int8_activations(K, N, seed=o_off + N)
    s = synth.token_scales(N, seed=N)
    pw = v.pack_weights(W, g, device=dev())
    abuf = torch.zeros(K * N + 64, dtype=torch.int8, device=dev())
    Ad = abuf[a_off:a_off + K * N].view(K, N)
    Ad.copy_(torch.from_numpy(A))
    obuf = torch.zeros(M * N + 16, dtype=torch.float32, device=dev())
    out = obuf[o_off // 4:o_off // 4 + M * N].view(M, N)
    sd = to_dev(s)
    ref = oracle.gemm_i32(W, A)
    plans = [None, v.LaunchPlan(12, 2), v.LaunchPlan(16, 1, streamk=1)]
    if N <= 64:
        plans.append(v.slot_plan(tpw=2))
    for plan in plans:
        out.zero_()
        v.mpgemm_ws(pw, Ad, sd, 0.5, out=out, plan=plan)
        torch.cuda.synchronize()
        check_fp32(out.cpu().numpy(), ref, s, 0.5)
