/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the Vec-LUT
 * ternary mpGeMM (arXiv 2512.06443).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_2512_06443_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source),
 *            "S:n" = /root/reference/SPEC.md line n.
 *
 * Every function states the passage it follows.  There is no blocking,
 * no fusion, no LUT in the GEMM definition, no intrinsics.  Build:
 *   gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared oracle.c -o liboracle.so
 * (-ffp-contract=off: the fp32 dequant / quantizer must be IEEE single ops.)
 *
 * Pins (tests/test_oracle.py): every function below is checked against
 * something other than itself -- paper numbers (tests/golden/), closed forms,
 * invariants, brute force on tiny inputs, numpy's int64 matmul.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- info */
int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------ 3^g helper */
static int pow3(int g) { int p = 1; for (int i = 0; i < g; ++i) p *= 3; return p; }

/* ------------------------------------------------ GetSign  (Alg. 1)
 * GetSign(i, j) = floor(i / 3^(j-1)) mod 3 - 1, 1-based j.  0-based r here
 * (reading c1/c4 in DESIGN.md): trit r of index i is floor(i/3^r) mod 3 - 1,
 * least-significant digit first. */
int oracle_get_sign(int i, int r) {
  int p = 1;
  for (int t = 0; t < r; ++t) p *= 3;
  return (i / p) % 3 - 1;
}

/* ------------------------------------------------ weight packing (a1)
 * P:436-441 ("packs the ternary weights into bytes ... for direct LUT
 * indexing"), Fig. bit-map caption P:390 ("The LUT row index is equal to the
 * decimal value of packed weights").  idx = sum_r (w_r + 1) * 3^r.
 * Returns -1 on an invalid trit. */
int oracle_pack_group(const int8_t* trits, int g) {
  int idx = 0, p = 1;
  for (int r = 0; r < g; ++r) {
    int t = trits[r];
    if (t < -1 || t > 1) return -1;
    idx += (t + 1) * p;
    p *= 3;
  }
  return idx;
}

/* Inverse of pack_group.  Returns 0 on success, -1 if idx is
 * outside [0, 3^g) (footnote P:417). */
int oracle_unpack_index(int idx, int g, int8_t* trits) {
  if (idx < 0 || idx >= pow3(g)) return -1;
  for (int r = 0; r < g; ++r) trits[r] = (int8_t)oracle_get_sign(idx, r);
  return 0;
}

/* Row-major logical packing: W [M][K] trits -> idx [M][K/g] bytes, group k of
 * row m covers features k*g .. k*g+g-1 (reading c4).  This is the *logical*
 * content of the packed weights ("Packed weights W of shape M x K/g");
 * the tile permutation of the CUDA path is a layout choice and is checked
 * by unpacking, not by comparing bytes.  Returns -1 on an invalid trit,
 * -2 if g does not divide K. */
int oracle_pack_matrix(const int8_t* W, int M, int K, int g, uint8_t* idx) {
  if (g <= 0 || K % g != 0) return -2;
  int KG = K / g;
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < KG; ++k) {
      int v = oracle_pack_group(W + (size_t)m * K + (size_t)k * g, g);
      if (v < 0) return -1;
      idx[(size_t)m * KG + k] = (uint8_t)v;
    }
  return 0;
}

/* ------------------------------------------------ the definition (§8c)
 * acc[m][n] = sum_{k<K} W[m][k] * A[k][n]          (int32; no LUT)
 * Table 2: W x A = O, W in R^{M x K}, A in R^{K x N}; A and O are
 * token-contiguous.  The method is lossless, so this
 * plain dot product is exactly what Alg. 1 / Eq. 2 must reproduce.
 * W: int8 trits [M][K]; A: int8 [K][N]; acc: int32 [M][N].
 * A is first copied to AT [N][K] (a plain transpose; no arithmetic) so each
 * dot product walks K contiguously. */
int oracle_gemm_i32(const int8_t* W, const int8_t* A, int32_t* acc,
                    int M, int K, int N) {
  if (M <= 0 || N <= 0) return 0;
  int8_t* AT = (int8_t*)malloc((size_t)N * (size_t)(K > 0 ? K : 1));
  if (!AT) return -1;
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) AT[(size_t)n * K + k] = A[(size_t)k * N + n];
#pragma omp parallel for schedule(static)
  for (int m = 0; m < M; ++m) {
    const int8_t* w = W + (size_t)m * K;
    for (int n = 0; n < N; ++n) {
      const int8_t* a = AT + (size_t)n * K;
      int32_t s = 0;
      for (int k = 0; k < K; ++k) s += (int32_t)w[k] * (int32_t)a[k];
      acc[(size_t)m * N + n] = s;
    }
  }
  free(AT);
  return 0;
}

/* Same definition, row subset [m0, m1): used by the bounded cpu_baseline
 * sample (bench.py) so the sample is literally a slice of the workload. */
int oracle_gemm_i32_rows(const int8_t* W, const int8_t* A, int32_t* acc,
                         int M, int K, int N, int m0, int m1) {
  if (m0 < 0) m0 = 0;
  if (m1 > M) m1 = M;
  if (m1 <= m0) return 0;
  return oracle_gemm_i32(W + (size_t)m0 * K, A, acc + (size_t)m0 * N,
                         m1 - m0, K, N);
}

/* ------------------------------------------------ LUT precompute (a3)
 * Vanilla enumeration, Alg. 1 Precompute / Eq. 1 (P:401-403,
 * reading c2: the stray outer sum over i is dropped):
 *   T[i][n] = sum_{r<g} GetSign(i, r) * A[r][n],   i in [0, 3^g).
 * A: int8 [g][N] (the g feature rows of one group, token-contiguous).
 * T: int32 [3^g][N].  *ops counts row-vector add/sub operations, i.e. the
 * number of (i, r) with GetSign != 0 (Alg. 1 lines "Add" and "Sub"). */
void oracle_precompute_vanilla(const int8_t* A, int g, int N, int32_t* T,
                               long* ops) {
  int R = pow3(g);
  long cnt = 0;
  for (int i = 0; i < R; ++i) {
    for (int n = 0; n < N; ++n) T[(size_t)i * N + n] = 0;
    for (int r = 0; r < g; ++r) {
      int v = oracle_get_sign(i, r);
      if (v == 1) {
        for (int n = 0; n < N; ++n) T[(size_t)i * N + n] += A[(size_t)r * N + n];
        cnt++;
      } else if (v == -1) {
        for (int n = 0; n < N; ++n) T[(size_t)i * N + n] -= A[(size_t)r * N + n];
        cnt++;
      }
    }
  }
  if (ops) *ops = cnt;
}

/* Topological precompute: every entry after the first is derived
 * from an already-computed entry by ONE +/- row operation, so a table costs
 * 3^g row ops instead of 2*3^(g-1)*g.  The paper shows only a fragment of its
 * dependency graph (reading c11); this oracle walks the base-3
 * reflected Gray code starting at index 0 (all -1): consecutive codes differ
 * in one digit by +/-1.  Root T[0] = -sum_r A[r] is counted as 1 op (the
 * paper's count "3^g" = 1 root + 3^g - 1 derivations).
 * order_out (optional, length 3^g) receives the visiting order. */
void oracle_precompute_topological(const int8_t* A, int g, int N, int32_t* T,
                                   long* ops, int* order_out) {
  int R = pow3(g);
  int digit[8] = {0}, dir[8];
  for (int r = 0; r < g; ++r) dir[r] = 1;
  long cnt = 0;
  /* root: index 0, every trit -1 */
  for (int n = 0; n < N; ++n) {
    int32_t s = 0;
    for (int r = 0; r < g; ++r) s -= A[(size_t)r * N + n];
    T[n] = s;
  }
  cnt++;
  int cur = 0;
  if (order_out) order_out[0] = 0;
  for (int step = 1; step < R; ++step) {
    /* reflected ternary Gray code: move the lowest digit that can still move
     * in its current direction; digits below it reverse direction */
    int r = 0;
    while (r < g) {
      int nd = digit[r] + dir[r];
      if (nd >= 0 && nd <= 2) break;
      dir[r] = -dir[r];
      ++r;
    }
    int p = 1;
    for (int t = 0; t < r; ++t) p *= 3;
    digit[r] += dir[r];
    int nxt = cur + dir[r] * p;
    /* trit r moved by dir[r] => T[nxt] = T[cur] + dir[r] * A[r] */
    for (int n = 0; n < N; ++n)
      T[(size_t)nxt * N + n] = T[(size_t)cur * N + n] + dir[r] * A[(size_t)r * N + n];
    cnt++;
    cur = nxt;
    if (order_out) order_out[step] = cur;
  }
  if (ops) *ops = cnt;
}

/* ------------------------------------------------ Alg. 1 literally (a3+a4)
 * O[m][n] = sum_k T[k][W[m][k]][n]   (Eq. 2) with T from the
 * vanilla Precompute.  Exists to pin the paper's claim that the LUT route
 * equals the definition (tests compare it with oracle_gemm_i32); it is NOT
 * the definition itself.  idx: [M][K/g] packed bytes (row-major). */
int oracle_alg1_lut_gemm(const uint8_t* idx, const int8_t* A, int32_t* O,
                         int M, int K, int N, int g) {
  if (K % g) return -2;
  int KG = K / g, R = pow3(g);
  int32_t* T = (int32_t*)malloc(sizeof(int32_t) * (size_t)R * (size_t)(N > 0 ? N : 1));
  if (!T) return -1;
  memset(O, 0, sizeof(int32_t) * (size_t)M * (size_t)N);
  for (int k = 0; k < KG; ++k) {
    oracle_precompute_vanilla(A + (size_t)k * g * N, g, N, T, NULL);
    for (int m = 0; m < M; ++m) {
      int i = idx[(size_t)m * KG + k];
      if (i >= R) { free(T); return -3; }
      for (int n = 0; n < N; ++n) O[(size_t)m * N + n] += T[(size_t)i * N + n];
    }
  }
  free(T);
  return 0;
}

/* ------------------------------------------------ INT16-INT32 hierarchy
 * accumulate up to B looked-up INT16 rows in INT16, then widen to
 * INT32.  rows: int16 values (one token), count n.  Emulates the INT16 block
 * register with C int16_t wraparound (two's complement) so that a B beyond
 * the paper's bound visibly overflows.  Returns the INT32 total. */
int32_t oracle_hier_accumulate(const int16_t* rows, int n, int B) {
  int32_t total = 0;
  int16_t block = 0;
  int in_block = 0;
  for (int i = 0; i < n; ++i) {
    block = (int16_t)(uint16_t)((uint16_t)block + (uint16_t)rows[i]);
    if (++in_block == B) { total += block; block = 0; in_block = 0; }
  }
  total += block;
  return total;
}

/* ------------------------------------------------ dequant (a6)
 * "Scale" stage (Table 1); formula S:329-337 (reading c7):
 * out[m][n] = acc[m][n] * a_scale[n] * w_scale.
 * f64: the definition, in double (used with the north star's 1e-6 relative
 * tolerance). */
void oracle_dequant_f64(const int32_t* acc, const float* a_scale, float w_scale,
                        double* out, int M, int N) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      out[(size_t)m * N + n] = (double)acc[(size_t)m * N + n] *
                               (double)a_scale[n] * (double)w_scale;
}

/* f32, fixed op order (reading c7 / §8c): s = fl(a_scale[n] * w_scale),
 * out = fl((float)acc * s).  Config 5's chain re-quantizes these fp32 values,
 * so the chain oracle needs the exact IEEE single result; (float)acc is exact
 * for |acc| < 2^24. */
void oracle_dequant_f32(const int32_t* acc, const float* a_scale, float w_scale,
                        float* out, int M, int N) {
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      volatile float s = a_scale[n] * w_scale;
      volatile float a = (float)acc[(size_t)m * N + n];
      out[(size_t)m * N + n] = a * s;
    }
}

/* ------------------------------------------------ quantizer (a7)
 * Per-token symmetric absmax int8 quantization for the w1.6A8 setting named
 * at P:102; formula S:339-347 (reading c8):
 *   amax_n = max_k |x[k][n]|;  s_n = amax_n / 127 (s_n = 1 if amax_n == 0);
 *   q[k][n] = clamp(roundf(x[k][n] / s_n), -127, 127), roundf = half away
 *   from zero.  All in IEEE single precision (the kernel's precision, since
 *   fp decides an integer here).
 * x: fp32 [K][N] token-contiguous; q: int8 [K][N]; scale: fp32 [N].
 * Returns -1 on a non-finite input. */
int oracle_quantize(const float* x, int K, int N, int8_t* q, float* scale) {
  for (int n = 0; n < N; ++n) {
    float amax = 0.0f;
    for (int k = 0; k < K; ++k) {
      float v = x[(size_t)k * N + n];
      if (!isfinite(v)) return -1;
      float a = fabsf(v);
      if (a > amax) amax = a;
    }
    volatile float s = amax / 127.0f;
    if (amax == 0.0f) s = 1.0f;
    scale[n] = s;
    for (int k = 0; k < K; ++k) {
      volatile float t = x[(size_t)k * N + n] / s;
      float r = roundf(t);
      if (r > 127.0f) r = 127.0f;
      if (r < -127.0f) r = -127.0f;
      q[(size_t)k * N + n] = (int8_t)r;
    }
  }
  return 0;
}

/* ------------------------------------------------ scalar LUT comparator (f4)
 * The prior paradigm: one table per token, N separate
 * 1->1 lookups per index.  *lookups counts indexing events.  Pins the
 * paradigm-count claim: scalar = N x vector lookups. */
int oracle_scalar_lut_gemm(const uint8_t* idx, const int8_t* A, int32_t* O,
                           int M, int K, int N, int g, long* lookups) {
  if (K % g) return -2;
  int KG = K / g, R = pow3(g);
  long cnt = 0;
  int32_t* t = (int32_t*)malloc(sizeof(int32_t) * (size_t)R);
  int8_t* col = (int8_t*)malloc((size_t)g);
  if (!t || !col) { free(t); free(col); return -1; }
  memset(O, 0, sizeof(int32_t) * (size_t)M * (size_t)N);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < KG; ++k) {
      for (int r = 0; r < g; ++r) col[r] = A[(size_t)(k * g + r) * N + n];
      oracle_precompute_vanilla(col, g, 1, t, NULL);
      for (int m = 0; m < M; ++m) {
        O[(size_t)m * N + n] += t[idx[(size_t)m * KG + k]];
        cnt++;
      }
    }
  free(t); free(col);
  if (lookups) *lookups = cnt;
  return 0;
}
