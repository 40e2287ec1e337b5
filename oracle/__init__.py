"""CPU oracle for the Vec-LUT ternary mpGeMM (arXiv 2512.06443).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product package ``paper_2512_06443_b200`` never imports it,
and the two share no code (the oracle is plain C in ``oracle/oracle.c`` plus
this numpy/ctypes marshalling layer).

Every function cites the passage it follows: ``P:n`` is a line of
``/root/reference/PAPER.md`` (LaTeX source), ``S:n`` a line of ``SPEC.md``.
Readings of silent/garbled points are listed in DESIGN.md (c1..c16).

Pinned by ``tests/test_oracle.py`` against paper numbers (``tests/golden``),
closed forms, invariants, brute force and numpy's int64 matmul.  No function
here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


FLAGS = ["-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
         "-fPIC", "-shared"]
_STAMP = _LIB_PATH + ".host"


def _host_key() -> str:
    """Compiler flags + this host's CPU model: -march=native code built on
    one machine must not run on another (the GPU box is not this container)."""
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith(("model name", "flags")):
                    model += line.strip() + "\n"
                    if line.startswith("flags"):
                        break
    except OSError:
        pass
    return " ".join(FLAGS) + "\n" + model


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O3 -march=native (plain C, OpenMP over rows,
    IEEE fp: no FMA contraction, no fast-math -- SURVEY §8(c)/(d)).  Rebuilt
    when the source is newer or the host CPU / flags differ."""
    key = _host_key()
    stale = force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC))
    if not stale:
        try:
            with open(_STAMP) as f:
                stale = f.read() != key
        except OSError:
            stale = True
    if stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc"] + FLAGS + [_SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
        with open(_STAMP, "w") as f:
            f.write(key)
    return _LIB_PATH


def omp_threads_env() -> str:
    """OMP_NUM_THREADS as seen by the oracle (unset -> all host threads)."""
    return os.environ.get("OMP_NUM_THREADS", "unset")


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB_PATH)
    P = ctypes.c_void_p
    I = ctypes.c_int
    L = ctypes.POINTER(ctypes.c_long)
    sig = {
        "oracle_num_threads": ([], I),
        "oracle_get_sign": ([I, I], I),
        "oracle_pack_group": ([P, I], I),
        "oracle_unpack_index": ([I, I, P], I),
        "oracle_pack_matrix": ([P, I, I, I, P], I),
        "oracle_gemm_i32": ([P, P, P, I, I, I], I),
        "oracle_gemm_i32_rows": ([P, P, P, I, I, I, I, I], I),
        "oracle_precompute_vanilla": ([P, I, I, P, L], None),
        "oracle_precompute_topological": ([P, I, I, P, L, P], None),
        "oracle_alg1_lut_gemm": ([P, P, P, I, I, I, I], I),
        "oracle_hier_accumulate": ([P, I, I], ctypes.c_int32),
        "oracle_dequant_f64": ([P, P, ctypes.c_float, P, I, I], None),
        "oracle_dequant_f32": ([P, P, ctypes.c_float, P, I, I], None),
        "oracle_quantize": ([P, I, I, P, P], I),
        "oracle_scalar_lut_gemm": ([P, P, P, I, I, I, I, L], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def zero_index(g: int) -> int:
    """Index of the all-zero pattern, (3^g - 1)/2: 40 / 121."""
    return (3 ** g - 1) // 2


def get_sign(i: int, r: int) -> int:
    """GetSign of Alg. 1, 0-based digit r, LSD first (c1)."""
    return int(_load().oracle_get_sign(int(i), int(r)))


def pack_group(trits) -> int:
    """idx = sum_r (w_r+1) 3^r.  ValueError on a bad trit."""
    t = np.ascontiguousarray(np.asarray(trits, dtype=np.int8))
    v = _load().oracle_pack_group(_p(t), int(t.size))
    if v < 0:
        raise ValueError("invalid trit")
    return int(v)


def unpack_index(idx: int, g: int) -> np.ndarray:
    """Inverse of pack_group.  ValueError if idx not in [0,3^g)."""
    out = np.zeros(g, dtype=np.int8)
    if _load().oracle_unpack_index(int(idx), int(g), _p(out)) != 0:
        raise ValueError("index out of range")
    return out


def pack_matrix(W: np.ndarray, g: int) -> np.ndarray:
    """Logical packed weights [M][K/g] uint8."""
    W = np.ascontiguousarray(W, dtype=np.int8)
    M, K = W.shape
    if K % g:
        raise ValueError("g does not divide K")
    out = np.zeros((M, K // g), dtype=np.uint8)
    rc = _load().oracle_pack_matrix(_p(W), M, K, g, _p(out))
    if rc == -1:
        raise ValueError("invalid trit")
    return out


def gemm_i32(W: np.ndarray, A: np.ndarray) -> np.ndarray:
    """acc = W @ A by direct int32 dot products (definition, §8c; Table 2
    P:294-320).  W int8 trits [M][K], A int8 [K][N] -> int32 [M][N]."""
    W = np.ascontiguousarray(W, dtype=np.int8)
    A = np.ascontiguousarray(A, dtype=np.int8)
    M, K = W.shape
    K2, N = A.shape
    assert K == K2
    acc = np.zeros((M, N), dtype=np.int32)
    if M and N:
        rc = _load().oracle_gemm_i32(_p(W), _p(A), _p(acc), M, K, N)
        assert rc == 0
    return acc


def gemm_i32_rows(W: np.ndarray, A: np.ndarray, m0: int, m1: int,
                  acc: np.ndarray) -> None:
    """Rows [m0, m1) of the definition into ``acc`` (bounded CPU sample)."""
    M, K = W.shape
    N = A.shape[1]
    rc = _load().oracle_gemm_i32_rows(_p(W), _p(A), _p(acc), M, K, N, m0, m1)
    assert rc == 0


def precompute_vanilla(A: np.ndarray, g: int):
    """Eq. 1 by enumeration.  A int8 [g][N] ->
    (T int32 [3^g][N], op count)."""
    A = np.ascontiguousarray(A, dtype=np.int8)
    N = A.shape[1]
    T = np.zeros((3 ** g, N), dtype=np.int32)
    ops = ctypes.c_long(0)
    _load().oracle_precompute_vanilla(_p(A), g, N, _p(T), ctypes.byref(ops))
    return T, int(ops.value)


def precompute_topological(A: np.ndarray, g: int):
    """Topological precompute along the base-3 reflected Gray code.
    Returns (T, op count, visiting order)."""
    A = np.ascontiguousarray(A, dtype=np.int8)
    N = A.shape[1]
    T = np.zeros((3 ** g, N), dtype=np.int32)
    order = np.zeros(3 ** g, dtype=np.int32)
    ops = ctypes.c_long(0)
    _load().oracle_precompute_topological(_p(A), g, N, _p(T), ctypes.byref(ops),
                                          _p(order))
    return T, int(ops.value), order


def alg1_lut_gemm(idx: np.ndarray, A: np.ndarray, g: int) -> np.ndarray:
    """Alg. 1 literally: vanilla tables + Eq. 2 lookups."""
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    A = np.ascontiguousarray(A, dtype=np.int8)
    M, KG = idx.shape
    K, N = A.shape
    assert KG * g == K
    O = np.zeros((M, N), dtype=np.int32)
    rc = _load().oracle_alg1_lut_gemm(_p(idx), _p(A), _p(O), M, K, N, g)
    if rc == -3:
        raise ValueError("corrupt index")
    assert rc == 0
    return O


def hier_accumulate(rows: np.ndarray, B: int) -> int:
    """INT16 block accumulation widened to INT32 every B rows."""
    rows = np.ascontiguousarray(rows, dtype=np.int16)
    return int(_load().oracle_hier_accumulate(_p(rows), int(rows.size), int(B)))


def paper_block_bound(g: int, int8_max: int = 127) -> int:
    """B <= floor(max(INT16) / (max(INT8) * g))."""
    return 32767 // (int8_max * g)


def full_lut_bytes(K: int, N: int, g: int) -> int:
    """(K/g) * 3^g * N * 2 bytes of an un-tiled INT16 vector LUT."""
    if K % g:
        raise ValueError("g does not divide K")
    return (K // g) * (3 ** g) * N * 2


def dequant_f64(acc: np.ndarray, a_scale: np.ndarray, w_scale: float) -> np.ndarray:
    """out = acc * a_scale[n] * w_scale in double (reading c7)."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    a_scale = np.ascontiguousarray(a_scale, dtype=np.float32)
    M, N = acc.shape
    out = np.zeros((M, N), dtype=np.float64)
    _load().oracle_dequant_f64(_p(acc), _p(a_scale), ctypes.c_float(w_scale),
                               _p(out), M, N)
    return out


def dequant_f32(acc: np.ndarray, a_scale: np.ndarray, w_scale: float) -> np.ndarray:
    """Fixed-op-order fp32 dequant: fl(fl(a_scale*w_scale) * (float)acc)."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    a_scale = np.ascontiguousarray(a_scale, dtype=np.float32)
    M, N = acc.shape
    out = np.zeros((M, N), dtype=np.float32)
    _load().oracle_dequant_f32(_p(acc), _p(a_scale), ctypes.c_float(w_scale),
                               _p(out), M, N)
    return out


def quantize(x: np.ndarray):
    """Per-token absmax int8 quantizer (P:102 w1.6A8, reading c8).
    x fp32 [K][N] -> (q int8 [K][N], scale fp32 [N])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    K, N = x.shape
    q = np.zeros((K, N), dtype=np.int8)
    s = np.zeros(N, dtype=np.float32)
    if _load().oracle_quantize(_p(x), K, N, _p(q), _p(s)) != 0:
        raise ValueError("non-finite input")
    return q, s


def scalar_lut_gemm(idx: np.ndarray, A: np.ndarray, g: int):
    """Scalar-LUT paradigm comparator: (O, lookups)."""
    idx = np.ascontiguousarray(idx, dtype=np.uint8)
    A = np.ascontiguousarray(A, dtype=np.int8)
    M, KG = idx.shape
    K, N = A.shape
    O = np.zeros((M, N), dtype=np.int32)
    cnt = ctypes.c_long(0)
    rc = _load().oracle_scalar_lut_gemm(_p(idx), _p(A), _p(O), M, K, N, g,
                                        ctypes.byref(cnt))
    assert rc == 0
    return O, int(cnt.value)


def mpgemm_f32(W: np.ndarray, A: np.ndarray, a_scale: np.ndarray,
               w_scale: float) -> np.ndarray:
    """Definition + fixed-order fp32 dequant (the value a chain re-quantizes)."""
    return dequant_f32(gemm_i32(W, A), a_scale, w_scale)


def config5_layer(Ws, w_scale: float, x_q: np.ndarray, x_s: np.ndarray,
                  q_rows: int):
    """One layer of config 5's fixed glue (reading c14):
    qkv = L_qkv(x); o = L_o(Q(qkv[0:q_rows])); u = Q(o);
    h = L_gate(u) * L_up(u) (one fp32 multiply); x' = Q(L_down(Q(h))).
    Ws = (W_qkv, W_o, W_gate, W_up, W_down) trits.  Returns (q, scale) of x'."""
    W_qkv, W_o, W_gate, W_up, W_down = Ws
    qkv = mpgemm_f32(W_qkv, x_q, x_s, w_scale)
    q1, s1 = quantize(np.ascontiguousarray(qkv[:q_rows]))
    o = mpgemm_f32(W_o, q1, s1, w_scale)
    u, su = quantize(o)
    gate = mpgemm_f32(W_gate, u, su, w_scale)
    up = mpgemm_f32(W_up, u, su, w_scale)
    h = (gate * up).astype(np.float32)
    hq, hs = quantize(h)
    d = mpgemm_f32(W_down, hq, hs, w_scale)
    return quantize(d)


def group_schedule(K: int):
    """Flexible sub-2-bit packing: split K into b groups
    of 5 followed by a groups of 4 with 5b + 4a = K, maximising b (reading of
    the footnote's condition).  Returns (b, a).  ValueError if no
    non-negative (a, b) exists (e.g. K in {1, 2, 3, 6, 7, 11})."""
    if K < 4:
        raise ValueError("unrepresentable K")
    for b in range(K // 5, -1, -1):
        if (K - 5 * b) % 4 == 0:
            return b, (K - 5 * b) // 4
    raise ValueError("unrepresentable K")


def mixed_bits_per_weight(K: int) -> float:
    """8 * (number of groups) / K for the mixed schedule."""
    b, a = group_schedule(K)
    return 8.0 * (a + b) / K
