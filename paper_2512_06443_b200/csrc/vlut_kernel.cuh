// vlut_kernel.cuh -- K1: fused Vec-LUT ternary mpGeMM for sm_100a.
//
// One CTA owns an (M-block of 32*WARPS rows) x (N-tile of 64 tokens) output
// tile and a contiguous range of K-tiles (16 weight groups each).  The CTAs
// of one thread-block cluster (size S along K) split the K range and reduce
// their int32 partials through distributed shared memory.  Per K-tile:
//
//   a2  cp.async stages the K-tile's activation rows A[16g][64] (int8) and
//       the CTA rows' 16-byte index vectors into shared memory, one K-tile
//       ahead of use (double-buffered).
//   a3  every warp builds whole sub-tables T[i][0:64] (Eq. 1) of the
//       K-tile's groups in shared memory, in the topological order of P:503-513:
//       one +/- row operation per table row, walking a base-3 reflected Gray
//       code over the low g-1 trits (the top trit splits a table into three
//       independent 3^(g-1)-row chains, one per warp task).  Rows are stored
//       token-contiguous, 128 B per row = 64 tokens x int16, as
//       biased 16-bit fields two tokens per 32-bit word:  field = T + 128 g.
//   a4  each thread owns ONE output row and all 64 tokens of the tile.  For
//       every group it reads its row's index byte and performs the 1->N vector
//       lookup (Alg. 1) as 8 LDS.128 of the indexed table row,
//       visiting the 16-byte chunks in the lane-rotated order (lane+s) mod 8:
//       the 8 lanes of an LDS.128 phase then always hit 8 different bank
//       groups whatever rows the data-dependent indices select (no bank
//       conflicts).  Two groups are summed per IADD3 into 16-bit SWAR fields
//       (INT16 intra-block accumulation); the fields are widened
//       into int32 registers every 48 groups (48 * 256 g <= 65535).
//   a5  after the K range: int32 tile -> shared memory (XOR-swizzled, conflict
//       free), cluster barrier, each CTA of the cluster sums 1/S of the rows
//       over all S CTAs via DSMEM.
//   a6  fp32 epilogue out = fl((float)acc * fl(a_scale[n] * w_scale)) with
//       coalesced 16-byte stores (or raw int32 for the test hook).
//
// Citations: P:n = /root/reference/PAPER.md line n.  See DESIGN.md for the
// roofline (shared-memory lookup bandwidth) and the byte/instruction budget.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace vlut {

namespace cg = cooperative_groups;

constexpr int kNcta = 64;             // tokens per CTA (N-tile)
constexpr int kKgTile = 16;           // groups per K-tile (16-byte index vector)
constexpr int kRowBytes = kNcta * 2;  // one table row: 64 tokens x int16
constexpr int kFlushTiles = 3;        // widen SWAR fields every 3 K-tiles = 48 groups

__host__ __device__ constexpr int pow3(int g) { return g == 0 ? 1 : 3 * pow3(g - 1); }

template <int G>
struct Cfg {
  static constexpr int R = pow3(G);             // table rows 3^g
  static constexpr int RP = R / 3;              // rows per chain (top trit fixed)
  static constexpr int GS = (G == 4) ? 16 : 4;  // groups per table sub-stage
  static constexpr int SUBS = kKgTile / GS;     // sub-stages per K-tile
  static constexpr int BIAS = 128 * G;          // field bias: T + BIAS in [0, 256 g]
  static constexpr int TAB_BYTES = GS * R * kRowBytes;
  static constexpr int A_ROWS = kKgTile * G;    // activation rows per K-tile
  static constexpr int A_BYTES = A_ROWS * kNcta;
  static constexpr int IDX_MASK = (G == 4) ? 0x7F : 0xFF;
  static_assert(kFlushTiles * kKgTile * 2 * BIAS <= 65535, "SWAR field overflow");
};

template <int G, int WARPS>
struct Layout {
  static constexpr int THREADS = WARPS * 32;
  static constexpr int MCTA = THREADS;                    // one output row per thread
  static constexpr int RED_BYTES = MCTA * kNcta * 4;      // int32 reduction tile
  static constexpr int TAB_REGION =
      Cfg<G>::TAB_BYTES > RED_BYTES ? Cfg<G>::TAB_BYTES : RED_BYTES;
  static constexpr int IDX_OFF = TAB_REGION;
  static constexpr int IDX_BYTES = MCTA * 16;
  static constexpr int A_OFF = IDX_OFF + 2 * IDX_BYTES;
  static constexpr int SMEM = A_OFF + 2 * Cfg<G>::A_BYTES;
};

// ---------------------------------------------------------------- Gray walk
// Base-3 reflected Gray code over D digits (compile time): step s changes
// digit[s] by dir[s] and lands on index idx[s].
template <int D>
struct GrayWalk {
  int digit[pow3(D)];
  int dir[pow3(D)];
  int idx[pow3(D)];
  constexpr GrayWalk() : digit(), dir(), idx() {
    int dg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int dr[8] = {1, 1, 1, 1, 1, 1, 1, 1};
    int cur = 0;
    idx[0] = 0;
    for (int s = 1; s < pow3(D); ++s) {
      int r = 0;
      while (r < D) {
        int nd = dg[r] + dr[r];
        if (nd >= 0 && nd <= 2) break;
        dr[r] = -dr[r];
        ++r;
      }
      int p = 1;
      for (int t = 0; t < r; ++t) p *= 3;
      dg[r] += dr[r];
      cur += dr[r] * p;
      digit[s] = r;
      dir[s] = dr[r];
      idx[s] = cur;
    }
  }
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];\n" : "=h"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------- params
struct Params {
  const uint8_t* payload;  // packed indices [kt][m_pad][16]
  const int8_t* A;         // [K][N]
  const float* a_scale;    // [N]
  float w_scale;
  float* out;              // [M][N] fp32 (or int32 when ACC_ONLY)
  int M, K, N;
  int m_pad, kg_tiles;
  int splits;              // cluster size along K
  int a_vec;               // 16, 4 or 1: activation staging width
  int out_vec4;            // 1 if out rows allow aligned 16-byte stores
};

// ---------------------------------------------------------------- staging (a2)
template <int G, int WARPS>
__device__ __forceinline__ void stage_tile(const Params& p, int kt, int buf, int m0, int n0,
                                           uint8_t* smem) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS>;
  const int tid = threadIdx.x;
  // index vectors: one 16-byte row per thread (rows past m_pad -> zero fill)
  {
    const int m = m0 + tid;
    const bool ok = m < p.m_pad;
    const uint8_t* src = ok ? p.payload + ((size_t)kt * p.m_pad + m) * 16 : p.payload;
    cp_async16(smem_u32(smem + L::IDX_OFF + buf * L::IDX_BYTES + tid * 16), src, ok ? 16 : 0);
  }
  // activation rows k0 .. k0 + 16g - 1, tokens n0 .. n0+63 (past K or N -> 0)
  const int k0 = kt * kKgTile * G;
  uint8_t* a_s = smem + L::A_OFF + buf * C::A_BYTES;
  if (p.a_vec == 16) {
    for (int c = tid; c < C::A_ROWS * 4; c += L::THREADS) {
      const int row = c >> 2, part = c & 3;
      const int k = k0 + row, n = n0 + part * 16;
      const bool ok = (k < p.K) && (n < p.N);
      const int8_t* src = ok ? p.A + (size_t)k * p.N + n : p.A;
      cp_async16(smem_u32(a_s + row * kNcta + part * 16), src, ok ? 16 : 0);
    }
  } else if (p.a_vec == 4) {
    for (int c = tid; c < C::A_ROWS * 16; c += L::THREADS) {
      const int row = c >> 4, part = c & 15;
      const int k = k0 + row, n = n0 + part * 4;
      const bool ok = (k < p.K) && (n < p.N);
      const int8_t* src = ok ? p.A + (size_t)k * p.N + n : p.A;
      cp_async4(smem_u32(a_s + row * kNcta + part * 4), src, ok ? 4 : 0);
    }
  } else {
    for (int c = tid; c < C::A_ROWS * kNcta; c += L::THREADS) {
      const int row = c / kNcta, col = c % kNcta;
      const int k = k0 + row, n = n0 + col;
      a_s[row * kNcta + col] = (k < p.K && n < p.N) ? (uint8_t)p.A[(size_t)k * p.N + n] : 0;
    }
  }
}

// ---------------------------------------------------------------- table build (a3)
// Walk the Gray code over the low D = g-1 trits, starting from T (row `base`).
template <int D, int S>
__device__ __forceinline__ void gray_walk(uint32_t row_addr0, uint32_t T, const uint32_t (&P)[8],
                                          const uint32_t (&Mn)[8]) {
  constexpr GrayWalk<D> gw{};
  constexpr int dig = gw.digit[S];
  constexpr int dir = gw.dir[S];
  constexpr int idx = gw.idx[S];
  T += (dir > 0) ? P[dig] : Mn[dig];
  sts32(row_addr0 + idx * kRowBytes, T);
  if constexpr (S + 1 < pow3(D)) gray_walk<D, S + 1>(row_addr0, T, P, Mn);
}

template <int G, int WARPS>
__device__ __forceinline__ void build_tables(uint32_t tab_s, uint32_t a_s, int sub) {
  using C = Cfg<G>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t K1 = 0x00010001u;
  constexpr uint32_t C128 = 128u * K1;
#pragma unroll 1
  for (int u = warp; u < C::GS * 3; u += WARPS) {
    const int j = u / 3;        // group within sub-stage
    const int part = u - 3 * j; // value of the top trit
    const int grp = sub * C::GS + j;  // group within the K-tile
    uint32_t P[8], Mn[8];
    uint32_t sumU = 0;
#pragma unroll
    for (int r = 0; r < G; ++r) {
      // tokens 2*lane, 2*lane+1 of activation row grp*g + r
      uint32_t x = lds_u16(a_s + (grp * G + r) * kNcta + 2 * lane);
      // int8 a -> u = a + 128 (XOR 0x80), spread the two bytes into 16-bit fields
      uint32_t U = __byte_perm(x ^ 0x8080u, 0u, 0x4140);
      P[r] = U - C128;   // +a_r as packed arithmetic delta
      Mn[r] = C128 - U;  // -a_r
      if (r < G - 1) sumU += U;
    }
    // start row: trits 0..g-2 = -1, top trit = part - 1
    //   T = BIAS + sum_{r<g-1} (-a_r) + (part-1) a_{g-1}
    uint32_t T = (uint32_t)C::BIAS * K1 - sumU + (uint32_t)(G - 1) * C128;
    if (part == 0) T += Mn[G - 1];
    if (part == 2) T += P[G - 1];
    const uint32_t row0 = tab_s + (uint32_t)((j * C::R + part * C::RP) * kRowBytes) + 4 * lane;
    sts32(row0, T);
    gray_walk<G - 1, 1>(row0, T, P, Mn);
  }
}

// ---------------------------------------------------------------- the kernel
template <int G, int WARPS, bool ACC_ONLY>
__global__ void __launch_bounds__(WARPS * 32, 1) vlut_mpgemm_kernel(const Params p) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS>;
  extern __shared__ __align__(1024) uint8_t smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int rank = blockIdx.x;  // split index (== rank in cluster)
  const int n0 = blockIdx.y * kNcta;
  const int m0 = blockIdx.z * L::MCTA;
  const int S = p.splits;
  const int kt_begin = (int)(((long long)rank * p.kg_tiles) / S);
  const int kt_end = (int)(((long long)(rank + 1) * p.kg_tiles) / S);
  const int ntiles = kt_end - kt_begin;

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = smem_u32(smem + L::IDX_OFF);
  const uint32_t a_s0 = smem_u32(smem + L::A_OFF);

  // lane-rotated chunk offsets: slot s of this lane holds tokens 8c..8c+7,
  // c = (lane + s) & 7
  uint32_t rot[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)(((lane + s) & 7) * 16);

  uint32_t sw[8][4];
  int32_t acc[8][8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) sw[s][q] = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[s][t] = 0;
  }

  if (ntiles > 0) {
    stage_tile<G, WARPS>(p, kt_begin, 0, m0, n0, smem);
    cp_async_commit();
  }
  int since_flush = 0;
#pragma unroll 1
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    cp_async_wait_all();
    __syncthreads();  // tile t visible; previous lookups done; buffer buf^1 free
    if (t + 1 < ntiles) {
      stage_tile<G, WARPS>(p, kt_begin + t + 1, buf ^ 1, m0, n0, smem);
      cp_async_commit();
    }
    const uint4 iw = lds128(idx_s + buf * L::IDX_BYTES + tid * 16);
    const uint32_t iwa[4] = {iw.x, iw.y, iw.z, iw.w};
    const uint32_t a_s = a_s0 + buf * C::A_BYTES;
#pragma unroll
    for (int sub = 0; sub < C::SUBS; ++sub) {
      if (sub > 0) __syncthreads();  // lookups of the previous sub-stage done
      build_tables<G, WARPS>(tab_s, a_s, sub);
      __syncthreads();               // tables visible
      // ---- lookup + accumulate (a4)
#pragma unroll
      for (int jp = 0; jp < C::GS / 2; ++jp) {
        constexpr int dummy = 0;
        (void)dummy;
        const int b0 = sub * C::GS + 2 * jp, b1 = b0 + 1;  // index bytes in the K-tile
        const uint32_t i0 = (iwa[b0 >> 2] >> (8 * (b0 & 3))) & C::IDX_MASK;
        const uint32_t i1 = (iwa[b1 >> 2] >> (8 * (b1 & 3))) & C::IDX_MASK;
        const uint32_t r0 = tab_s + (uint32_t)((2 * jp) * C::R * kRowBytes) + i0 * kRowBytes;
        const uint32_t r1 = tab_s + (uint32_t)((2 * jp + 1) * C::R * kRowBytes) + i1 * kRowBytes;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint4 v0 = lds128(r0 + rot[s]);
          const uint4 v1 = lds128(r1 + rot[s]);
          sw[s][0] += v0.x + v1.x;
          sw[s][1] += v0.y + v1.y;
          sw[s][2] += v0.z + v1.z;
          sw[s][3] += v0.w + v1.w;
        }
      }
    }
    if (++since_flush == kFlushTiles || t + 1 == ntiles) {
      // widen 16-bit fields into int32 (INT16 -> INT32)
      since_flush = 0;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[s][2 * q] += (int32_t)(sw[s][q] & 0xFFFFu);
          acc[s][2 * q + 1] += (int32_t)(sw[s][q] >> 16);
          sw[s][q] = 0;
        }
      }
    }
  }
  // remove the field bias: every group added BIAS to every token
  const int32_t bias_total = C::BIAS * kKgTile * ntiles;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int t = 0; t < 8; ++t) acc[s][t] -= bias_total;

  // ---- int32 tile -> shared (a5).  Row r (this thread), 16-byte unit u of
  // the 256-byte row stored at u ^ ((r >> 2) & 1): conflict-free for both the
  // lane-per-row writes below and the row-contiguous reads after.
  __syncthreads();  // all table reads done before the region is reused
  {
    const uint32_t red_s = tab_s;
    const int r = tid;
    const uint32_t swz = (uint32_t)((r >> 2) & 1);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const uint32_t c = (uint32_t)((lane + s) & 7);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t u = (2 * c + h) ^ swz;
        sts128(red_s + r * 256 + u * 16, (uint32_t)acc[s][4 * h], (uint32_t)acc[s][4 * h + 1],
               (uint32_t)acc[s][4 * h + 2], (uint32_t)acc[s][4 * h + 3]);
      }
    }
  }
  cg::cluster_group cluster = cg::this_cluster();
  if (S > 1) cluster.sync(); else __syncthreads();

  // ---- reduce across the cluster + epilogue (a5, a6)
  {
    const int rows_per = L::MCTA / S;
    const int r_begin = rank * rows_per;
    const int units = rows_per * 16;
    const int4* red_local = reinterpret_cast<const int4*>(smem);
#pragma unroll 1
    for (int e = tid; e < units; e += L::THREADS) {
      const int r = r_begin + (e >> 4);
      const int u = e & 15;
      const int pu = u ^ ((r >> 2) & 1);
      const int off = r * 16 + pu;  // in int4 units
      int4 v = red_local[off];
      for (int q = 0; q < S; ++q) {
        if (q == rank) continue;
        const int4* rem = cluster.map_shared_rank(red_local, q);
        const int4 w = rem[off];
        v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
      }
      const int m = m0 + r;
      const int n = n0 + 4 * u;
      if (m >= p.M || n >= p.N) continue;
      if constexpr (ACC_ONLY) {
        int32_t* o = reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n;
        if (p.out_vec4 && n + 3 < p.N) {
          *reinterpret_cast<int4*>(o) = v;
        } else {
          const int vv[4] = {v.x, v.y, v.z, v.w};
          for (int i = 0; i < 4 && n + i < p.N; ++i) o[i] = vv[i];
        }
      } else {
        float* o = p.out + (size_t)m * p.N + n;
        const int vv[4] = {v.x, v.y, v.z, v.w};
        float f[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float sc = (n + i < p.N) ? __fmul_rn(__ldg(p.a_scale + n + i), p.w_scale) : 0.f;
          f[i] = __fmul_rn((float)vv[i], sc);
        }
        if (p.out_vec4 && n + 3 < p.N) {
          *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
        } else {
          for (int i = 0; i < 4 && n + i < p.N; ++i) o[i] = f[i];
        }
      }
    }
  }
  if (S > 1) cluster.sync();  // keep this CTA's shared memory alive for readers
}

}  // namespace vlut
