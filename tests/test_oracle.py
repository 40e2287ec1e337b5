"""Pins for the CPU oracle (oracle/).  CPU only (-m "not gpu").

Each test checks the oracle against something other than itself: a value the
paper prints (tests/golden/paper_values.json, with citations), a closed form,
an invariant, brute force on tiny inputs, or an independent library routine
(numpy int64 matmul, numpy.base_repr, decimal rounding, fractions).
"""
import itertools
from decimal import Decimal, ROUND_HALF_UP
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2512_06443_b200 import synth


def digits3(i, g):
    """Base-3 digits of i, LSD first, via numpy's base_repr (library)."""
    s = np.base_repr(i, 3).zfill(g)
    return [int(c) for c in reversed(s)]


# ------------------------------------------------------------------ GetSign
@pytest.mark.parametrize("g", [4, 5])
def test_get_sign_matches_base_repr(g):
    for i in range(3 ** g):
        d = digits3(i, g)
        for r in range(g):
            assert oracle.get_sign(i, r) == d[r] - 1


def test_worked_example_23(golden):
    ex = golden["worked_example_23"]
    i, g = ex["i"], ex["g"]
    # the paper's digit string (MSD first) is the base-3 numeral of 23
    assert sum(d * 3 ** (g - 1 - p) for p, d in enumerate(ex["base3_digits_msd_first"])) == i
    # Alg. 1 GetSign (LSD first; reading c1)
    assert [oracle.get_sign(i, r) for r in range(g)] == ex["alg1_trits_lsd_first"]
    # the same pattern is the paper's MSD-first pattern reversed
    assert ex["alg1_trits_lsd_first"] == list(reversed(ex["paper_pattern_msd_first"]))
    assert oracle.pack_group(ex["alg1_trits_lsd_first"]) == 23


# ------------------------------------------------------------------ packing
def test_pack_group_fixed_points(golden):
    assert oracle.pack_group([0, 0, 0, 0]) == oracle.zero_index(4) == 40
    assert oracle.pack_group([0] * 5) == oracle.zero_index(5) == 121
    assert oracle.pack_group([1] * 4) == golden["index_range"]["g4_max"]
    assert oracle.pack_group([1] * 5) == golden["index_range"]["g5_max"]
    assert oracle.pack_group([-1] * 4) == 0
    assert golden["table_rows"]["g4"] == 3 ** 4 and golden["table_rows"]["g5"] == 3 ** 5
    with pytest.raises(ValueError):
        oracle.pack_group([0, 2, 0, 0])


@pytest.mark.parametrize("g", [4, 5])
def test_pack_unpack_bijection(g):
    seen = set()
    for w in itertools.product([-1, 0, 1], repeat=g):
        i = oracle.pack_group(list(w))
        assert 0 <= i < 3 ** g
        assert list(oracle.unpack_index(i, g)) == list(w)
        seen.add(i)
    assert len(seen) == 3 ** g
    with pytest.raises(ValueError):
        oracle.unpack_index(3 ** g, g)  # 243 in a g=5 group is corrupt


@pytest.mark.parametrize("g", [4, 5])
def test_pack_matrix_roundtrip_and_bpw(g, golden):
    W = synth.ternary_weights(37, 20 * g, seed=11 + g)
    P = oracle.pack_matrix(W, g)
    assert P.shape == (37, 20)
    U = np.stack([np.concatenate([oracle.unpack_index(int(b), g) for b in row]) for row in P])
    assert np.array_equal(U, W)
    bpw = 8.0 * P.size / W.size
    key = "g4_I2" if g == 4 else "g5_I1"
    assert bpw == pytest.approx(golden["bits_per_weight"][key], abs=1e-12)
    assert oracle.pack_matrix(np.zeros((3, 4 * g), np.int8), g).tolist() == \
        [[oracle.zero_index(g)] * 4] * 3
    with pytest.raises(ValueError):
        oracle.pack_matrix(np.zeros((2, 4 * g + 1), np.int8), g)


# ------------------------------------------------------------------ GEMM definition
def test_gemm_brute_force_tiny():
    r = synth.rng(5)
    for _ in range(20):
        M, K, N = (int(x) for x in r.integers(1, 7, size=3))
        W = r.integers(-1, 2, size=(M, K)).astype(np.int8)
        A = r.integers(-128, 128, size=(K, N)).astype(np.int8)
        ref = [[sum(int(W[m, k]) * int(A[k, n]) for k in range(K)) for n in range(N)]
               for m in range(M)]
        assert oracle.gemm_i32(W, A).tolist() == ref


@pytest.mark.parametrize("M,K,N", [(64, 512, 8), (33, 100, 17), (5, 4096, 3), (128, 20, 129)])
def test_gemm_matches_numpy_int64(M, K, N):
    W = synth.ternary_weights(M, K, seed=M + K)
    A = synth.int8_activations(K, N, seed=N + 7)
    ref = W.astype(np.int64) @ A.astype(np.int64)
    assert np.array_equal(oracle.gemm_i32(W, A).astype(np.int64), ref)


def test_gemm_closed_forms():
    r = synth.rng(9)
    M, K = 12, 40
    W = synth.ternary_weights(M, K, seed=3)
    # A = c * I  =>  acc = c * W
    for c in (1, -1, 7, -128, 127):
        A = (np.eye(K, dtype=np.int64) * c).astype(np.int8)
        assert np.array_equal(oracle.gemm_i32(W, A), (W.astype(np.int32) * c))
    A = synth.int8_activations(K, 9, seed=4)
    # selector row: single +1 at column k0 => row of A
    S = np.zeros((3, K), np.int8)
    S[0, 5] = 1
    S[1, 0] = 1
    S[2, K - 1] = -1
    out = oracle.gemm_i32(S, A)
    assert np.array_equal(out[0], A[5].astype(np.int32))
    assert np.array_equal(out[1], A[0].astype(np.int32))
    assert np.array_equal(out[2], -A[K - 1].astype(np.int32))
    # all +1 => column sums ; W = 0 => 0
    assert np.array_equal(oracle.gemm_i32(np.ones((2, K), np.int8), A)[0],
                          A.astype(np.int64).sum(0).astype(np.int32))
    assert not oracle.gemm_i32(np.zeros((4, K), np.int8), A).any()
    # negation and linearity (kept in int8 range)
    assert np.array_equal(oracle.gemm_i32(-W, A), -oracle.gemm_i32(W, A))
    A1 = r.integers(-63, 64, size=(K, 9)).astype(np.int8)
    A2 = r.integers(-64, 64, size=(K, 9)).astype(np.int8)
    assert np.array_equal(oracle.gemm_i32(W, (A1 + A2).astype(np.int8)),
                          oracle.gemm_i32(W, A1) + oracle.gemm_i32(W, A2))
    # extreme: all +1 weights, all -128 activations, long K
    K2 = 23040
    assert oracle.gemm_i32(np.ones((1, K2), np.int8),
                           np.full((K2, 2), -128, np.int8)).tolist() == [[-128 * K2] * 2]


def test_gemm_rows_is_a_slice():
    W = synth.ternary_weights(50, 64, seed=1)
    A = synth.int8_activations(64, 10, seed=2)
    full = oracle.gemm_i32(W, A)
    part = np.zeros_like(full)
    oracle.gemm_i32_rows(W, A, 10, 31, part)
    assert np.array_equal(part[10:31], full[10:31])
    assert not part[:10].any() and not part[31:].any()


# ------------------------------------------------------------------ precompute (Eq. 1)
@pytest.mark.parametrize("g", [4, 5])
def test_vanilla_table_brute_force(g, golden):
    A = synth.int8_activations(g, 11, seed=20 + g)
    T, ops = oracle.precompute_vanilla(A, g)
    for w in itertools.product([-1, 0, 1], repeat=g):
        i = oracle.pack_group(list(w))
        assert np.array_equal(T[i], np.array(w, np.int64) @ A.astype(np.int64))
    z = oracle.zero_index(g)
    assert not T[z].any()
    assert np.array_equal(T[3 ** g - 1], A.astype(np.int32).sum(0))
    assert np.array_equal(T[0], -A.astype(np.int32).sum(0))
    for i in range(3 ** g):  # anti-symmetry
        assert np.array_equal(T[i], -T[3 ** g - 1 - i])
    key = "g4_vanilla" if g == 4 else "g5_vanilla"
    assert ops == golden["topological_ops"][key] == 2 * 3 ** (g - 1) * g


def test_worked_example_table_row(golden):
    ex = golden["worked_example_23"]
    A = synth.int8_activations(4, 13, seed=77)
    T, _ = oracle.precompute_vanilla(A, 4)
    # paper: index 23 gives -A0 + A1 + A3 with rows read MSD-first; under
    # Alg. 1's LSD-first GetSign (reading c1) the same combination applies to
    # the rows in reverse order.
    combo = ex["paper_row_combination"]
    ref = sum(combo["A%d" % p] * A[3 - p].astype(np.int32) for p in range(4))
    assert np.array_equal(T[23], ref)


@pytest.mark.parametrize("g", [4, 5])
def test_topological_equals_vanilla_and_op_count(g, golden):
    r = synth.rng(100 + g)
    for trial in range(200):
        N = int(r.integers(1, 40))
        A = r.integers(-128, 128, size=(g, N)).astype(np.int8)
        Tv, _ = oracle.precompute_vanilla(A, g)
        Tt, ops, order = oracle.precompute_topological(A, g)
        assert np.array_equal(Tv, Tt)
    key = "g4_topological" if g == 4 else "g5_topological"
    assert ops == golden["topological_ops"][key] == 3 ** g
    vk = "g4_vanilla" if g == 4 else "g5_vanilla"
    ratio = golden["topological_ops"][vk] / ops
    assert ratio == pytest.approx(2 * g / 3)
    if g == 5:
        assert round(ratio, 1) == golden["topological_ops"]["g5_speedup"]
    # spanning order: every index once, single-trit +/-1 steps
    assert sorted(order.tolist()) == list(range(3 ** g))
    for a, b in zip(order[:-1], order[1:]):
        da, db = digits3(int(a), g), digits3(int(b), g)
        diff = [x - y for x, y in zip(da, db) if x != y]
        assert len(diff) == 1 and abs(diff[0]) == 1


def test_topological_fragment_relations(golden):
    frag = golden["topological_fragment"]
    A = synth.int8_activations(4, 9, seed=5)
    T, _, _ = oracle.precompute_topological(A, 4)
    for a, b in frag["edges"]:
        da, db = digits3(a, 4), digits3(b, 4)
        r = [k for k in range(4) if da[k] != db[k]]
        assert len(r) == 1
        r = r[0]
        assert np.array_equal(T[b], T[a] + (db[r] - da[r]) * A[r].astype(np.int32))
    a, b = frag["negation_edge"]
    assert np.array_equal(T[b], -T[a])


# ------------------------------------------------------------------ Alg. 1 == definition
@pytest.mark.parametrize("g", [4, 5])
def test_alg1_lut_gemm_equals_definition(g):
    r = synth.rng(300 + g)
    for _ in range(10):
        M = int(r.integers(1, 40))
        K = g * int(r.integers(1, 30))
        N = int(r.integers(1, 20))
        W = r.integers(-1, 2, size=(M, K)).astype(np.int8)
        A = r.integers(-128, 128, size=(K, N)).astype(np.int8)
        idx = oracle.pack_matrix(W, g)
        assert np.array_equal(oracle.alg1_lut_gemm(idx, A, g), oracle.gemm_i32(W, A))
    bad = np.full((1, 1), 3 ** g, np.uint8)
    with pytest.raises(ValueError):
        oracle.alg1_lut_gemm(bad, np.zeros((g, 1), np.int8), g)


def test_scalar_lut_paradigm_counts():
    g, M, K, N = 4, 9, 48, 7
    W = synth.ternary_weights(M, K, seed=8)
    A = synth.int8_activations(K, N, seed=9)
    idx = oracle.pack_matrix(W, g)
    O, lookups = oracle.scalar_lut_gemm(idx, A, g)
    assert np.array_equal(O, oracle.gemm_i32(W, A))
    # 1->1 lookups: N x the vector LUT's M*(K/g) 1->N lookups
    assert lookups == N * M * (K // g)


# ------------------------------------------------------------------ INT16 hierarchy
def test_block_bound_paper_values(golden):
    bb = golden["block_bound"]
    assert oracle.paper_block_bound(4, bb["int8_max"]) == bb["g4_B"] == 64
    assert oracle.paper_block_bound(5, bb["int8_max"]) == 51


def test_hier_accumulate_adversarial():
    row = 4 * 127  # g * max(INT8) = 508
    exact = 64 * row
    assert oracle.hier_accumulate(np.full(64, row, np.int16), 64) == exact
    # B = 65 exceeds the bound: the INT16 block wraps
    assert oracle.hier_accumulate(np.full(65, row, np.int16), 65) != 65 * row
    assert oracle.hier_accumulate(np.full(65, row, np.int16), 64) == 65 * row
    r = synth.rng(3)
    rows = r.integers(-508, 509, size=5000).astype(np.int16)
    assert oracle.hier_accumulate(rows, 64) == int(rows.astype(np.int64).sum())


def test_full_lut_bytes_paper_number(golden):
    ls = golden["lut_size"]
    b = oracle.full_lut_bytes(ls["K"], ls["N"], ls["g"])
    assert b == 299_344_896
    assert abs(b / 2 ** 20 - ls["MiB"]) < ls["MiB_tolerance"]


# ------------------------------------------------------------------ quantizer
def test_quantize_special_cases():
    x = np.zeros((5, 3), np.float32)
    x[:, 1] = [127 * 0.5, -127 * 0.5, 0, 0.25, 0]
    x[:, 2] = [127.0, 2.5, -2.5, 0.5, -0.5]
    q, s = oracle.quantize(x)
    assert s[0] == 1.0 and not q[:, 0].any()           # zero column -> scale 1
    assert s[1] == 0.5 and q[:, 1].tolist() == [127, -127, 0, 1, 0]
    assert s[2] == 1.0 and q[:, 2].tolist() == [127, 3, -3, 1, -1]  # half away
    with pytest.raises(ValueError):
        oracle.quantize(np.array([[np.inf]], np.float32))


def test_quantize_against_decimal_rounding():
    x = synth.activations_f32(300, 16, seed=12)
    q, s = oracle.quantize(x)
    amax = np.abs(x).max(0)
    assert np.array_equal(s, (amax / np.float32(127)).astype(np.float32))
    t = (x / s[None, :]).astype(np.float32)  # IEEE single division (numpy)
    ref = np.vectorize(lambda v: int(Decimal(float(v)).quantize(Decimal(1), rounding=ROUND_HALF_UP)))(t)
    ref = np.clip(ref, -127, 127)
    assert np.array_equal(q.astype(np.int64), ref)
    err = np.abs(x.astype(np.float64) - q.astype(np.float64) * s.astype(np.float64))
    assert np.all(err <= s.astype(np.float64) / 2 * (1 + 1e-6) + 1e-12)


# ------------------------------------------------------------------ dequant
def test_dequant_exact_and_f32_order():
    acc = np.array([[0, 1, -7, 2 ** 23, -(2 ** 23) + 5, 123456]], np.int32)
    a_s = np.array([0.5, 0.013, 1.7, 3e-3, 0.25, 7.5e-4], np.float32)
    w = 0.02
    d64 = oracle.dequant_f64(acc, a_s, w)
    for j in range(acc.shape[1]):
        exact = Fraction(int(acc[0, j])) * Fraction(float(a_s[j])) * Fraction(float(np.float32(w)))
        assert abs(Fraction(float(d64[0, j])) - exact) <= abs(exact) * Fraction(1, 2 ** 52)
    d32 = oracle.dequant_f32(acc, a_s, w)
    ref32 = (acc.astype(np.float32) * (a_s * np.float32(w)).astype(np.float32)).astype(np.float32)
    assert np.array_equal(d32.view(np.int32), ref32.view(np.int32))
    nz = d64 != 0
    assert np.all(np.abs(d32[nz] - d64[nz]) / np.abs(d64[nz]) <= 1.2e-7)


def test_config5_layer_smoke():
    # tiny stand-in shapes (same glue as config 5; reading c14)
    K, N = 40, 6
    Ws = (synth.ternary_weights(60, K, 1), synth.ternary_weights(K, K, 2),
          synth.ternary_weights(80, K, 3), synth.ternary_weights(80, K, 4),
          synth.ternary_weights(K, 80, 5))
    xq, xs = oracle.quantize(synth.activations_f32(K, N, 6))
    q, s = oracle.config5_layer(Ws, synth.W_SCALE, xq, xs, q_rows=K)
    assert q.shape == (K, N) and s.shape == (N,)
    assert np.all(s > 0) and np.abs(q.astype(int)).max() <= 127


def test_config5_layer_identity_closed_form():
    """Pin of the config-5 glue (reading c14) by a special case with a closed
    form: identity weights (ternary 0/1) make every linear pass its input
    through up to the per-token scales, so x' = Q(Q(h)) with h = u * u and
    u = x: the final codes are round_half_away(x^2 / 127) for int8 codes x
    whose column reaches |x| = 127 (x^2 / 127 kept away from .5 ties), and
    the input's sign is lost.  A dropped re-quantization, the product taken
    before Q, a wrong q_rows slice or a sign error all change the codes."""
    K, N = 64, 5
    rng = synth.rng(11)
    xq = rng.integers(-127, 128, size=(K, N)).astype(np.int8)
    xq[0, :] = 127
    xq[1, :] = -127
    frac = (xq.astype(np.int64) ** 2 % 127) / 127.0
    xq[np.abs(frac - 0.5) < 0.02] = 3  # 9 / 127 is far from a tie
    xs = np.full(N, 0.05, np.float32)
    I = np.eye(K, dtype=np.int8)
    W_qkv = np.concatenate([I, np.zeros((2 * K, K), np.int8)])  # rows K.. are ignored
    q, s = oracle.config5_layer((W_qkv, I, I, I, I), synth.W_SCALE, xq, xs, q_rows=K)
    x2 = xq.astype(np.int64) ** 2
    expect = (2 * x2 + 127) // 254  # round half away of x^2 / 127 (non-negative)
    assert np.array_equal(q.astype(np.int64), expect)
    assert np.all(q >= 0)


# ------------------------------------------------------------------ mixed g=5/g=4 schedule (f2)
def test_group_schedule_examples():
    # (K=20, I1) -> all 5s; K=4096 mixed -> 816 fives then 4 fours,
    # BPW = 8*820/4096 ~ 1.6016; K=7 unrepresentable
    assert oracle.group_schedule(20) == (4, 0)
    assert oracle.group_schedule(4096) == (816, 4)
    assert oracle.mixed_bits_per_weight(4096) == pytest.approx(8 * 820 / 4096)
    assert round(oracle.mixed_bits_per_weight(4096), 4) == 1.6016
    for bad in (1, 2, 3, 6, 7, 11):
        with pytest.raises(ValueError):
            oracle.group_schedule(bad)


def test_group_schedule_properties():
    for K in range(12, 3000):
        b, a = oracle.group_schedule(K)
        assert 5 * b + 4 * a == K and a >= 0 and b >= 0
        # maximal b: one more 5-group never leaves a multiple of 4
        assert all((K - 5 * bb) % 4 for bb in range(b + 1, K // 5 + 1))
        bpw = oracle.mixed_bits_per_weight(K)
        assert 1.6 <= bpw <= 2.0
        if K >= 100:
            assert bpw < 1.7
    # the paper's shapes that 5 does not divide (P:445-447 motivation)
    for K in (4096, 6912, 14336):
        assert K % 5 and oracle.group_schedule(K)[0] > 0
