// vlut_kernel.cuh -- K1: fused Vec-LUT ternary mpGeMM for sm_100a.
//
// One CTA owns an (M-block of 32*WARPS rows) x (N-tile of 64 tokens) output
// tile and a contiguous range of K-tiles (16 weight groups each).  The CTAs
// of one thread-block cluster (size S along K) split the K range and reduce
// their int32 partials through distributed shared memory.
//
//   a2  cp.async stages each K-tile's activation rows A[16g][64] (int8) and
//       the CTA rows' 16-byte index vectors into shared memory, triple
//       buffered, one K-tile ahead of its first use.
//   a3  sub-tables (Eq. 1) are built in shared memory in the
//       topological order of P:503-513 (one +/- row op per row, along base-3
//       reflected Gray codes).  Only the upper half of each table is stored:
//       T[i] = -T[3^g-1-i] (negating all trits negates the dot product), so
//       rows i >= z = (3^g-1)/2 are kept at position i - z ((3^g+1)/2 rows:
//       41 for g=4, 122 for g=5) and a lookup of i < z reads position z - i
//       and negates.  Rows are token-contiguous, 128 B = 64 tokens
//       x int16, stored as biased 16-bit fields two tokens per 32-bit word:
//       field = T + 128 g  (in [0, 256 g] for any int8 input).
//       Tables are double buffered: while the CTA looks up sub-stage u it
//       builds sub-stage u+1, with ONE barrier per sub-stage.
//   a4  each thread owns ONE output row and all 64 tokens of the tile.  Per
//       group it turns its index byte into (position, sign) and performs the
//       1->N vector lookup (Alg. 1) as 8 LDS.128 of the row, in
//       the lane-rotated chunk order (lane+s) mod 8: the 8 lanes of an
//       LDS.128 phase always hit 8 different bank groups, whatever rows the
//       data-dependent indices select.  Words are accumulated into 16-bit SWAR
//       fields (INT16 intra-block accumulation): negated lookups
//       add (w ^ -1) [ALU] or w * -1 [FMA pipe], with a per-row count of
//       negations that restores 2*bias - field at the widening step; fields
//       are widened into int32 registers every 48 groups (48 * 256 g < 2^16).
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
#include <cuda.h>
#include <cuda_runtime.h>

namespace vlut {

namespace cg = cooperative_groups;

constexpr int kNcta = 64;             // tokens per CTA (N-tile)
constexpr int kKgTile = 16;           // groups per K-tile (16-byte index vector)
constexpr int kRowBytes = kNcta * 2;  // one table row: 64 tokens x int16
constexpr int kFlushTiles = 3;        // widen SWAR fields every 3 K-tiles = 48 groups
constexpr int kStageBufs = 3;         // A / index staging buffers
#ifndef VLUT_TABLE_BUFS
#define VLUT_TABLE_BUFS 2
#endif
// mbarrier slots (byte offsets from MBAR_OFF): FULL[b], EMPTY[b], STAGE[s]
__host__ __device__ constexpr int mb_full(int b) { return 8 * b; }
__host__ __device__ constexpr int mb_empty(int b) { return 8 * VLUT_TABLE_BUFS + 8 * b; }
__host__ __device__ constexpr int mb_stage(int s) { return 16 * VLUT_TABLE_BUFS + 8 * s; }

__host__ __device__ constexpr int pow3(int g) { return g == 0 ? 1 : 3 * pow3(g - 1); }

template <int G>
struct Cfg {
  static constexpr int R = pow3(G);             // full table rows 3^g
  static constexpr int ZERO = (R - 1) / 2;      // index of the all-zero pattern
  static constexpr int HR = (R + 1) / 2;        // stored (half) rows
  // table buffers and groups per sub-stage: NBUF x GS x half rows is the
  // table region; more, smaller buffers let the builders run further ahead
  static constexpr int NBUF = VLUT_TABLE_BUFS;
  static constexpr int GS = (G == 4) ? (NBUF == 4 ? 8 : 16) : (NBUF == 4 ? 2 : 4);
  static constexpr int SUBS = kKgTile / GS;     // sub-stages per K-tile
  static constexpr int BIAS = 128 * G;          // field bias: T + BIAS in [0, 256 g]
  static constexpr int TAB_BYTES = GS * HR * kRowBytes;  // one table buffer
  static constexpr int A_ROWS = kKgTile * G;    // activation rows per K-tile
  static constexpr int A_BYTES = A_ROWS * kNcta;
  static constexpr int IDX_MASK = (G == 4) ? 0x7F : 0xFF;
  static_assert(kFlushTiles * kKgTile * 2 * BIAS <= 65535, "SWAR field overflow");
};

// WARPS lookup warps (one output row per thread) + kBuilderWarps table
// builders; threads = 32 * (WARPS + builders).  Two rows per lookup thread
// (768 rows per table) halve the table build per lookup, so two builder warps
// keep up there -- and the 64 threads freed raise the register budget from
// 128 to 144 per thread (two rows' SWAR fields are 64 registers).
constexpr int kBuilderWarps = 4;
#ifndef VLUT_BW_RPT2
#define VLUT_BW_RPT2 4
#endif
template <int WARPS, int RPT>
constexpr int kBW = (RPT == 2 && WARPS == 12) ? VLUT_BW_RPT2 : kBuilderWarps;
constexpr int kTmemCols = 256;  // int32 accumulators: 64 columns per 4 lookup warps

// RPT = output rows per lookup thread: 1 (K1, both schedules) or 2 (the
// stream-K variant with 12 lookup warps: 768 rows share every table, halving
// the table-build share of the shared-memory pipe).
template <int G, int WARPS, int RPT = 1>
struct Layout {
  static_assert(RPT == 1 || RPT == 2, "one or two rows per lookup thread");
  static constexpr int BW = kBW<WARPS, RPT>;              // builder warps
  static constexpr int NLT = WARPS * 32;                  // lookup threads
  static constexpr int THREADS = NLT + BW * 32;
  static constexpr int BUILDER0 = NLT;                    // first builder thread
  static constexpr int MCTA = NLT * RPT;                  // output rows per CTA
  static constexpr int RED_BYTES = NLT * kNcta * 4;       // int32 tile of one row block
  static constexpr int TMEM_COLS = 256 * RPT;             // 64 columns per 4 warps per row block
  static constexpr int TAB_REGION = Cfg<G>::NBUF * Cfg<G>::TAB_BYTES > RED_BYTES
                                        ? Cfg<G>::NBUF * Cfg<G>::TAB_BYTES : RED_BYTES;
  static constexpr int IDX_OFF = TAB_REGION;
  static constexpr int IDX_BYTES = MCTA * 16;
  static constexpr int A_OFF = IDX_OFF + kStageBufs * IDX_BYTES;
  static constexpr int MISC_OFF = A_OFF + kStageBufs * Cfg<G>::A_BYTES;  // tmem address
  static constexpr int MBAR_OFF = MISC_OFF + 16;  // FULL[NBUF], EMPTY[NBUF], STAGE[3] (8 B each)
  static constexpr int SCALE_OFF = MBAR_OFF + 96;  // fl(a_scale[n] * w_scale), 64 floats
  static constexpr int AMAX_OFF = SCALE_OFF + kNcta * 4;  // per-token |out| max of the CTA
  static constexpr int SMEM = AMAX_OFF + kNcta * 4;
  // epilogue: 16-byte output units per thread (upper bound, splits = 1)
  static constexpr int EPI_UNITS = (MCTA * 16 + THREADS - 1) / THREADS;
  static_assert(WARPS <= 16, "TMEM columns: at most 4 column blocks of 64");
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

// ---------------------------------------------------------------- debug timing
// Compiled only with -DVLUT_TIMING (scripts/phase_timing): %globaltimer
// stamps of CTA phases into g_vlut_timing[cta][8].
#ifdef VLUT_TIMING
__device__ unsigned long long* g_vlut_timing;
#define VLUT_STAMP(i)                                                                      \
  do {                                                                                     \
    if (threadIdx.x == 0 && g_vlut_timing) {                                               \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      const unsigned cta_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
      g_vlut_timing[cta_ * 8 + (i)] = t_;                                                  \
    }                                                                                      \
  } while (0)
#else
#define VLUT_STAMP(i) \
  do {                \
  } while (0)
#endif

// ---------------------------------------------------------------- barriers
// Named barrier 5: builder warps only.  Table handshake: mbarriers (lookup
// warps wait on FULL without arriving, so they never rendezvous with each
// other; one elected lane per warp arrives).
__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMEM helpers
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// ---------------------------------------------------------------- params
constexpr int kMaxPeers = 7;  // 8 GPUs of one NVSwitch box: 7 remote copies

struct alignas(64) Params {
  CUtensorMap a_map;       // 2D TMA map of A [K][N] int8, box 64 x 16g (a_vec == 16)
  const uint8_t* payload;  // packed indices [kt][m_pad][16]
  const int8_t* A;         // [K][N]
  const float* a_scale;    // [N]
  float w_scale;
  float* out;              // [M][N] fp32 (or int32 when ACC_ONLY)
  const int32_t* acc_in;   // optional int32 [M][N] added before the epilogue (may alias out)
  int M, K, N;
  int m_pad, kg_tiles;
  int splits;              // cluster size along K
  int a_vec;               // 16 (TMA), 4 or 1: activation staging width
  int a3d;                 // K1-32: a_map is the 3-D view [r][group][token] (K % g == 0)
  int out_vec4;            // 1 if out rows allow aligned 16-byte stores
  int out_t;               // 1: out is [N][M] (feature-major, fused output transposition)
  const float* mul_in;     // optional fp32 [M][N]: out = fl(out * mul_in) (gate (.) up glue)
  unsigned* amax_out;      // optional [N]: atomicMax of |out| (float bits) over rows < amax_rows
  int amax_rows;
  // fused all-gather (a8): the fp32 tile is also stored to n_peers remote
  // copies of the output (peer device pointers, NVLink P2P), each already
  // offset to this shard's first row, same [M][N] indexing as `out`
  float* peer_out[kMaxPeers];
  int n_peers;
  // 1: `out` is a multicast address (NVLS: the NVSwitch replicates each store
  // into every rank's copy); stored with multimem.st, the only access PTX
  // defines on a multimem address
  int out_mc;
};

// fp32 stores to a multicast (multimem) address
__device__ __forceinline__ void st_mc_v4(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_mc_f32(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;\n" ::"l"(p), "f"(v) : "memory");
}

// ---------------------------------------------------------------- staging (a2)
// Issued by the builder threads (bt in [0, 128)).  what: 1 = index vectors,
// 2 = activations, 3 = both; a commit group is closed after the activations.
template <int G, int WARPS, int RPT = 1>
__device__ __forceinline__ void stage_tile(const Params& p, int kt, int buf, int m0, int n0,
                                           uint8_t* smem, int bt, int what) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS, RPT>;
  constexpr int NB = L::BW * 32;
  if (what & 1) {
    // index vectors: one 16-byte row per CTA row (rows past m_pad -> zero fill)
    for (int r = bt; r < L::MCTA; r += NB) {
      const int m = m0 + r;
      const bool ok = m < p.m_pad;
      const uint8_t* src = ok ? p.payload + ((size_t)kt * p.m_pad + m) * 16 : p.payload;
      cp_async16(smem_u32(smem + L::IDX_OFF + buf * L::IDX_BYTES + r * 16), src, ok ? 16 : 0);
    }
  }
  if (!(what & 2)) return;
  // activation rows k0 .. k0 + 16g - 1, tokens n0 .. n0+63 (past K or N -> 0)
  const int k0 = kt * kKgTile * G;
  uint8_t* a_s = smem + L::A_OFF + buf * C::A_BYTES;
  if (p.a_vec == 16) {
    for (int c = bt; c < C::A_ROWS * 4; c += NB) {
      const int row = c >> 2, part = c & 3;
      const int k = k0 + row, n = n0 + part * 16;
      const bool ok = (k < p.K) && (n < p.N);
      const int8_t* src = ok ? p.A + (size_t)k * p.N + n : p.A;
      cp_async16(smem_u32(a_s + row * kNcta + part * 16), src, ok ? 16 : 0);
    }
  } else if (p.a_vec == 4) {
    for (int c = bt; c < C::A_ROWS * 16; c += NB) {
      const int row = c >> 4, part = c & 15;
      const int k = k0 + row, n = n0 + part * 4;
      const bool ok = (k < p.K) && (n < p.N);
      const int8_t* src = ok ? p.A + (size_t)k * p.N + n : p.A;
      cp_async4(smem_u32(a_s + row * kNcta + part * 4), src, ok ? 4 : 0);
    }
  } else {
    for (int c = bt; c < C::A_ROWS * kNcta; c += NB) {
      const int row = c / kNcta, col = c % kNcta;
      const int k = k0 + row, n = n0 + col;
      a_s[row * kNcta + col] = (k < p.K && n < p.N) ? (uint8_t)p.A[(size_t)k * p.N + n] : 0;
    }
  }
  cp_async_commit();
}

// TMA bulk staging (N % 16 == 0, 16-byte aligned A): builder warp 0 issues one
// bulk copy for the CTA's index rows of the tile (contiguous in the payload)
// and one per activation row; completion is counted on the stage's mbarrier.
// Rows past K / m_pad and columns past N are zero-filled with plain stores
// (disjoint bytes; ordered for the consumers by barrier 5 / FULL).
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(addr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
      : "memory");
}

template <int G, int WARPS, int RPT = 1>
__device__ __forceinline__ void stage_tile_bulk(const Params& p, int kt, int buf, int m0, int n0,
                                                uint8_t* smem, int bt, uint32_t stg_mbar,
                                                bool do_idx, bool do_act, bool arm) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS, RPT>;
  constexpr int NB = L::BW * 32;
  const int idx_rows = max(0, min(L::MCTA, p.m_pad - m0));
  const int k0 = kt * kKgTile * G;
  const int a_rows = max(0, min(C::A_ROWS, p.K - k0));
  const int a_cols = max(0, min(kNcta, p.N - n0));  // multiple of 16 (N % 16 == 0)
  uint8_t* idx_dst = smem + L::IDX_OFF + buf * L::IDX_BYTES;
  uint8_t* a_dst = smem + L::A_OFF + buf * C::A_BYTES;
  // zero fill of the parts no copy covers (tails only)
  if (do_idx)
    for (int i = idx_rows * 16 + bt * 16; i < L::MCTA * 16; i += NB * 16)
      *reinterpret_cast<uint4*>(idx_dst + i) = make_uint4(0, 0, 0, 0);
  (void)a_cols; (void)a_rows;
  if (bt < 32) {
    if (arm && bt == 0) {
      // the A box always delivers 16g x 64 bytes (out-of-range elements are
      // zero-filled by the TMA unit and count toward the transaction)
      const uint32_t bytes = (uint32_t)(idx_rows * 16 + C::A_BYTES);
      mbar_expect_tx(stg_mbar, bytes);
    }
    __syncwarp();
    if (do_idx && bt == 0 && idx_rows > 0)
      bulk_g2s(smem_u32(idx_dst), p.payload + ((size_t)kt * p.m_pad + m0) * 16,
               (uint32_t)(idx_rows * 16), stg_mbar);
    if (do_act && bt == 0) {
      if (p.a3d)  // [r][group][token]: box (64 tokens, 16 groups, g rows)
        tma_load_3d(smem_u32(a_dst), &p.a_map, n0, kt * kKgTile, 0, stg_mbar);
      else
        tma_load_2d(smem_u32(a_dst), &p.a_map, n0, k0, stg_mbar);
    }
  }
}

// ---------------------------------------------------------------- table build (a3)
// Walk the Gray code over D digits from the start row already in T.
template <int D, int S>
__device__ __forceinline__ void gray_walk(uint32_t row_addr0, uint32_t T, const uint32_t (&P)[8],
                                          const uint32_t (&Mn)[8]) {
  if constexpr (D > 0 && S < pow3(D)) {
    constexpr GrayWalk<D> gw{};
    constexpr int dig = gw.digit[S];
    constexpr int dir = gw.dir[S];
    constexpr int idx = gw.idx[S];
    T += (dir > 0) ? P[dig] : Mn[dig];
    sts32(row_addr0 + idx * kRowBytes, T);
    gray_walk<D, S + 1>(row_addr0, T, P, Mn);
  }
}

// Half table: position 0 = the zero pattern; block Lv (Lv = 0..g-1) = the
// patterns whose trits above Lv are 0, trit Lv = +1, trits below free; it
// occupies positions [(3^Lv+1)/2, (3^(Lv+1)+1)/2), position = (3^Lv+1)/2 +
// (base-3 value of the free digits d_0..d_{Lv-1}, d = trit + 1).
template <int G, int Lv>
__device__ __forceinline__ void build_blocks(uint32_t row0, uint32_t S, const uint32_t (&U)[8],
                                             const uint32_t (&P)[8], const uint32_t (&Mn)[8]) {
  if constexpr (Lv < G) {
    constexpr uint32_t K1 = 0x00010001u;
    constexpr uint32_t C128 = 128u * K1;
    // start: trit Lv = +1, trits below = -1:  T = BIAS + a_Lv - sum_{r<Lv} a_r
    const uint32_t T = (uint32_t)Cfg<G>::BIAS * K1 + U[Lv] - C128 - S + (uint32_t)Lv * C128;
    const uint32_t base = row0 + (uint32_t)(((pow3(Lv) + 1) / 2) * kRowBytes);
    sts32(base, T);
    gray_walk<Lv, 1>(base, T, P, Mn);
    build_blocks<G, Lv + 1>(row0, S + U[Lv], U, P, Mn);
  }
}

// Builder warp bw (of BW) builds the half tables of its groups of
// sub-stage [grp0, grp0 + GS) of the staged K-tile.
template <int G, int BW = kBuilderWarps>
__device__ __forceinline__ void build_tables(uint32_t tab_s, uint32_t a_s, int grp0, int bw,
                                             int lane) {
  using C = Cfg<G>;
  constexpr uint32_t K1 = 0x00010001u;
  constexpr uint32_t C128 = 128u * K1;
#pragma unroll 1
  for (int j = bw; j < C::GS; j += BW) {
    uint32_t U[8], P[8], Mn[8];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      // tokens 2*lane, 2*lane+1 of activation row (grp0+j)*g + r
      const uint32_t x = lds_u16(a_s + ((grp0 + j) * G + r) * kNcta + 2 * lane);
      // int8 a -> u = a + 128 (XOR 0x80), spread the two bytes into 16-bit fields
      U[r] = __byte_perm(x ^ 0x8080u, 0u, 0x4140);
      P[r] = U[r] - C128;   // +a_r as a packed arithmetic delta
      Mn[r] = C128 - U[r];  // -a_r
    }
    const uint32_t row0 = tab_s + (uint32_t)(j * C::HR * kRowBytes) + 4 * lane;
    sts32(row0, (uint32_t)C::BIAS * K1);  // the zero pattern
    build_blocks<G, 0>(row0, 0u, U, P, Mn);
  }
}

// ---------------------------------------------------------------- wide-store table build
// 16-byte-store builders (K1 and K1-32): lane = 8 q + ch writes chunk ch of
// a 128-byte table line for line set q, one STS.128 per warp fills four
// lines (four wavefronts, conflict-free) -- a quarter of the store
// instructions of the 4-byte form, which matters because the lookup warps
// keep the shared-memory queue full (K1-32: 94 -> 88 us on the headline).
// The half table (anti-symmetry as in K1: position 0 = the zero
// pattern, block Lv = trits above Lv zero, trit Lv = +1, trits below free, at
// positions (3^Lv+1)/2 + base-3 value of digits d_r = t_r + 1) is cut into
// sub-walks: unit (Lv, D, PF) fixes digits D .. Lv-1 to the base-3 number PF
// and walks digits 0 .. D-1 along the reflected Gray code from all -1 (one
// packed add per entry and word).  The units are spread over the builder
// warps of a pair group (g = 4: 2 warps x 4 pairs x 41 lines; g = 5: 4 warps
// x 4 pairs x 122 lines).
// P[r][w] = +a_r as packed arithmetic 16-bit deltas (U - 128 per field); the
// -a_r step is T - P (mod 2^32 the same as adding C128 - U), so no second
// delta array is held.
template <int G, int Lv, int D, int PF>
__device__ __forceinline__ void sub_walk(uint32_t row0, const uint32_t (&P)[G][4]) {
  constexpr uint32_t K1 = 0x00010001u;
  uint32_t T[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    T[w] = (uint32_t)Cfg<G>::BIAS * K1 + P[Lv][w];
#pragma unroll
    for (int r = 0; r < Lv; ++r) {
      if (r < D) {
        T[w] -= P[r][w];  // walked digits start at trit -1
      } else {
        const int d = (PF / pow3(r - D)) % 3;  // fixed digit (compile time)
        if (d == 2) T[w] += P[r][w];
        if (d == 0) T[w] -= P[r][w];
      }
    }
  }
  constexpr int pos0 = (pow3(Lv) + 1) / 2 + PF * pow3(D);
  sts128(row0 + pos0 * 128, T[0], T[1], T[2], T[3]);
  if constexpr (D > 0) {
    constexpr GrayWalk<D> gw{};
#pragma unroll
    for (int st = 1; st < pow3(D); ++st) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        if (gw.dir[st] > 0) T[w] += P[gw.digit[st]][w];
        else T[w] -= P[gw.digit[st]][w];
      }
      sts128(row0 + (pos0 + gw.idx[st]) * 128, T[0], T[1], T[2], T[3]);
    }
  }
}

template <int G>
__device__ __forceinline__ void zero_row(uint32_t row0) {
  constexpr uint32_t Z = (uint32_t)Cfg<G>::BIAS * 0x00010001u;
  sts128(row0, Z, Z, Z, Z);
}

// The units of one builder warp: g = 4, half h of the 41 lines (20 + 21);
// g = 5, quarter h of the 122 lines (31 + 31 + 30 + 30).  Balanced, because
// the slowest builder warp paces the table handshake.
template <int G>
__device__ __forceinline__ void build_units(int h, uint32_t row0, const uint32_t (&P)[G][4]) {
  if constexpr (G == 4) {
    if (h == 0) {
      zero_row<4>(row0);
      sub_walk<4, 0, 0, 0>(row0, P);
      sub_walk<4, 1, 1, 0>(row0, P);
      sub_walk<4, 3, 2, 0>(row0, P);
      sub_walk<4, 2, 1, 0>(row0, P);
      sub_walk<4, 2, 1, 1>(row0, P);
    } else {
      sub_walk<4, 3, 2, 1>(row0, P);
      sub_walk<4, 3, 2, 2>(row0, P);
      sub_walk<4, 2, 1, 2>(row0, P);
    }
  } else {
    if (h == 0) {
      sub_walk<5, 4, 2, 0>(row0, P);
      sub_walk<5, 4, 2, 1>(row0, P);
      sub_walk<5, 4, 2, 2>(row0, P);
      sub_walk<5, 1, 1, 0>(row0, P);
      sub_walk<5, 0, 0, 0>(row0, P);
    } else if (h == 1) {
      sub_walk<5, 4, 2, 3>(row0, P);
      sub_walk<5, 4, 2, 4>(row0, P);
      sub_walk<5, 4, 2, 5>(row0, P);
      sub_walk<5, 2, 1, 0>(row0, P);
      zero_row<5>(row0);
    } else if (h == 2) {
      sub_walk<5, 4, 2, 6>(row0, P);
      sub_walk<5, 4, 2, 7>(row0, P);
      sub_walk<5, 4, 2, 8>(row0, P);
      sub_walk<5, 2, 1, 1>(row0, P);
    } else {
      sub_walk<5, 3, 2, 0>(row0, P);
      sub_walk<5, 3, 2, 1>(row0, P);
      sub_walk<5, 3, 2, 2>(row0, P);
      sub_walk<5, 2, 1, 2>(row0, P);
    }
  }
}

// K1 (64-token rows): builder warp bw of BW builds its line sets -- at g = 4
// set s = four groups 4s .. 4s+3 of the 16-group sub-stage (all 41 lines),
// at g = 5 (4-group sub-stages) the four groups' quarter s of the 122 lines.
// Lane 8 q + ch: group q of the set, tokens 8 ch .. 8 ch + 7.
template <int G, int BW = kBuilderWarps>
__device__ __forceinline__ void build_tables_wide(uint32_t tab_s, uint32_t a_s, int grp0, int bw,
                                                  int lane, bool a3d = false) {
  using C = Cfg<G>;
  constexpr uint32_t K1 = 0x00010001u;
  constexpr uint32_t C128 = 128u * K1;
  constexpr int SETS = (G == 4) ? C::GS / 4 : 4;  // g=4: group sets; g=5: line quarters
  static_assert(G == 5 ? C::GS == 4 : C::GS % 4 == 0, "wide builder: 4 groups per set");
  const int q = lane >> 3, ch = lane & 7;
#pragma unroll 1
  for (int st = bw; st < SETS; st += BW) {
    const int j = (G == 4) ? 4 * st + q : q;  // group within the sub-stage
    uint32_t P[G][4];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      uint32_t x0, x1;
      asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n"
                   : "=r"(x0), "=r"(x1)
                   : "r"(a_s + (uint32_t)((a3d ? (r * kKgTile + grp0 + j) : ((grp0 + j) * G + r)) *
                                               kNcta + 8 * ch)));
      x0 ^= 0x80808080u;
      x1 ^= 0x80808080u;
      const uint32_t U[4] = {__byte_perm(x0, 0u, 0x4140), __byte_perm(x0, 0u, 0x4342),
                             __byte_perm(x1, 0u, 0x4140), __byte_perm(x1, 0u, 0x4342)};
#pragma unroll
      for (int w = 0; w < 4; ++w) P[r][w] = U[w] - C128;
    }
    const uint32_t row0 = tab_s + (uint32_t)(j * C::HR * kRowBytes + ch * 16);
    if constexpr (G == 4) {
      build_units<4>(0, row0, P);
      build_units<4>(1, row0, P);
    } else {
      build_units<5>(st, row0, P);
    }
  }
}

// table builder of K1 / K1-SK: wide 16-byte stores or the 4-byte form
#ifndef VLUT_WIDE_MAX_WARPS
#define VLUT_WIDE_MAX_WARPS 16
#endif
template <int WARPS>
constexpr bool kWideBuild = WARPS <= VLUT_WIDE_MAX_WARPS;

// ---------------------------------------------------------------- lookups (a4)
template <int WARPS>
constexpr int kLookupGP = (WARPS >= 16) ? 1 : 2;
// two rows per thread: with 12 warps one group per load batch (the second
// row's accumulators take the registers of the second batch); 8 warps have
// 170 registers per thread and keep two
template <int WARPS, int RPT>
constexpr int kLookupGP2 = (RPT > 1) ? (WARPS <= 8 ? 2 : 1) : kLookupGP<WARPS>;
// loads per batch of the one-group path: 4 where 8 would spill (two rows per
// thread with 12 warps: 64 SWAR registers live)
#ifndef VLUT_LB_RPT2
#define VLUT_LB_RPT2 8
#endif
#ifndef VLUT_LB_W16
#define VLUT_LB_W16 8
#endif
template <int WARPS, int RPT>
constexpr int kLookupLB = (RPT > 1 && WARPS >= 12) ? VLUT_LB_RPT2 : (WARPS >= 16 ? VLUT_LB_W16 : 8);

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr));
  return v;
}

// Groups [SUB*GS, SUB*GS+GS) of the K-tile; idx_row = shared address of this
// thread's 16-byte index row of the tile (one index byte per group: a 32-bit
// word is loaded when its first group comes up -- the same wavefronts as one
// LDS.128 per tile, without 4 live registers per row).  Chunk order: slot s
// of lane l reads the 16-byte chunk c = (l & 7) ^ s of the 128-byte table row
// (the 8 lanes of an LDS.128 phase hit 8 different bank groups whatever the
// rows; row addresses are 128-aligned, so the chunk address is one XOR:
// (row | rot[0]) ^ 16 s -- no per-slot offset registers), or, RX = false,
// c = (l + s) & 7 with rot[s] = 16 c.
// GP = groups per load batch: 2 (16 LDS.128 in flight, half the negations on
// the ALU pipe as XOR, half on the FMA pipe as multiply) or 1 (8 in flight,
// every negation a multiply: 32 fewer live registers, for the 16-warp
// variants whose 102-register budget would otherwise spill).
// LB (GP = 1 only): LDS.128 per load batch, 8 or 4 (16 fewer live registers
// for the variants whose budget would otherwise spill inside this loop).
// LAZY: index words loaded from shared memory when first needed (idx_row)
// instead of held in registers (iwa, loaded once per K-tile by the caller) --
// for the two-rows-per-thread variants; elsewhere the eager form spills less.
// RX: chunk order c = (lane & 7) ^ s (one XOR per load, no offset registers:
// the two-rows-per-thread variants) or c = (lane + s) & 7 (rot[s] offsets in
// registers, r + rot[s]: what the other variants allocate best).
template <bool RX>
__device__ __forceinline__ int chunk_of(int lane, int s) {
  return RX ? ((lane ^ s) & 7) : ((lane + s) & 7);
}

template <int G, int GP = 2, int LB = 8, bool LAZY = false, bool RX = false>
__device__ __forceinline__ void lookup_sub(const int SUB, uint32_t tab, const uint32_t (&iwa)[4],
                                           uint32_t idx_row, const uint32_t (&rot)[8],
                                           uint32_t (&sw)[8][4], int32_t& nneg) {
  using C = Cfg<G>;
  static_assert(LB == 8 || LB == 4, "loads per batch");
  uint32_t word = 0;
  if constexpr (GP == 1) {
#pragma unroll
    for (int j = 0; j < C::GS; ++j) {
      const int b = SUB * C::GS + j;
      if (j == 0 || (b & 3) == 0) word = LAZY ? lds32(idx_row + 4 * (b >> 2)) : iwa[b >> 2];
      const int i = (int)((word >> (8 * (b & 3))) & C::IDX_MASK);
      const int d = i - C::ZERO;
      const uint32_t m = (uint32_t)(d >> 31);
      const uint32_t pos = (uint32_t)((d ^ (int)m) - (int)m);
      nneg += (int)m;
      const uint32_t sg = m | 1u;
      const uint32_t r = tab + (uint32_t)(j * C::HR * kRowBytes) + pos * kRowBytes;
#pragma unroll
      for (int s0 = 0; s0 < 8; s0 += LB) {
        uint4 v[LB];
#pragma unroll
        for (int s = 0; s < LB; ++s)
          v[s] = lds128(RX ? ((r | rot[0]) ^ (uint32_t)(16 * (s0 + s))) : r + rot[s0 + s]);
#pragma unroll
        for (int s = 0; s < LB; ++s) {
          sw[s0 + s][0] += v[s].x * sg;
          sw[s0 + s][1] += v[s].y * sg;
          sw[s0 + s][2] += v[s].z * sg;
          sw[s0 + s][3] += v[s].w * sg;
        }
      }
    }
    return;
  }
#pragma unroll
  for (int jp = 0; jp < C::GS / 2; ++jp) {
    const int b0 = SUB * C::GS + 2 * jp, b1 = b0 + 1;  // index bytes in the K-tile
    if (jp == 0 || (b0 & 3) == 0) word = LAZY ? lds32(idx_row + 4 * (b0 >> 2)) : iwa[b0 >> 2];
    const int i0 = (int)((word >> (8 * (b0 & 3))) & C::IDX_MASK);
    const int i1 = (int)((word >> (8 * (b1 & 3))) & C::IDX_MASK);  // b0 even: same word
    const int d0 = i0 - C::ZERO, d1 = i1 - C::ZERO;
    const uint32_t m0 = (uint32_t)(d0 >> 31), m1 = (uint32_t)(d1 >> 31);  // 0 or ~0: negate
    const uint32_t p0 = (uint32_t)((d0 ^ (int)m0) - (int)m0);              // |d|
    const uint32_t p1 = (uint32_t)((d1 ^ (int)m1) - (int)m1);
    nneg += (int)m0 + (int)m1;  // minus the number of negated lookups
    const uint32_t sg0 = m0 | 1u, sg1 = m1 | 1u;  // +1 / -1
    const uint32_t r0 = tab + (uint32_t)((2 * jp) * C::HR * kRowBytes) + p0 * kRowBytes;
    const uint32_t r1 = tab + (uint32_t)((2 * jp + 1) * C::HR * kRowBytes) + p1 * kRowBytes;
    uint4 v0[8], v1[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      v0[s] = lds128(RX ? ((r0 | rot[0]) ^ (uint32_t)(16 * s)) : r0 + rot[s]);
      v1[s] = lds128(RX ? ((r1 | rot[0]) ^ (uint32_t)(16 * s)) : r1 + rot[s]);
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s < 4) {  // ALU pipe: XOR-negate, two groups per IADD3
        sw[s][0] += (v0[s].x ^ m0) + (v1[s].x ^ m1);
        sw[s][1] += (v0[s].y ^ m0) + (v1[s].y ^ m1);
        sw[s][2] += (v0[s].z ^ m0) + (v1[s].z ^ m1);
        sw[s][3] += (v0[s].w ^ m0) + (v1[s].w ^ m1);
      } else {      // FMA pipe: multiply-negate
        sw[s][0] += v0[s].x * sg0 + v1[s].x * sg1;
        sw[s][1] += v0[s].y * sg0 + v1[s].y * sg1;
        sw[s][2] += v0[s].z * sg0 + v1[s].z * sg1;
        sw[s][3] += v0[s].w * sg0 + v1[s].w * sg1;
      }
    }
  }
}

// Widen the SWAR fields into the int32 accumulators held in TMEM (INT16 ->
// INT32).  A negated lookup contributed ~w (s < 4) or -w (s >= 4)
// instead of the packed 2*BIAS - field; add the difference back per negation
// before splitting the fields.  TMEM column 8*s + t of this thread's lane
// holds token slot (s, t); `first` initialises instead of accumulating.
template <int G, bool ALL_MUL = false>
__device__ __forceinline__ void flush_tmem(uint32_t (&sw)[8][4], int32_t& nneg, uint32_t taddr,
                                           bool first) {
  constexpr uint32_t K1 = 0x00010001u;
  const uint32_t cnt = (uint32_t)(-nneg);
  const uint32_t corr_xor = cnt * (2u * Cfg<G>::BIAS * K1 + 1u);
  const uint32_t corr_mul = cnt * (2u * Cfg<G>::BIAS * K1);
#pragma unroll
  for (int h = 0; h < 4; ++h) {  // slots 2h, 2h+1 -> 16 columns
    uint32_t v[16];
    if (!first) {
      tmem_ld16(taddr + 16 * h, v);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int s = 2 * h + e;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t w = sw[s][q] + ((s < 4 && !ALL_MUL) ? corr_xor : corr_mul);
        v[8 * e + 2 * q] += w & 0xFFFFu;
        v[8 * e + 2 * q + 1] += w >> 16;
        sw[s][q] = 0;
      }
    }
    tmem_st16(taddr + 16 * h, v);
  }
  tmem_wait_st();
  nneg = 0;
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: the K1 prologue (mbarriers, TMEM, index
// staging) overlaps the tail of the kernel that produced A / a_scale.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ---------------------------------------------------------------- the kernel
template <int G, int WARPS, bool ACC_ONLY>
__global__ void __launch_bounds__((WARPS + kBW<WARPS, 1>) * 32, 1)
    vlut_mpgemm_kernel(const __grid_constant__ Params p) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS>;
  extern __shared__ __align__(1024) uint8_t smem[];
  VLUT_STAMP(0);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int rank = blockIdx.x;  // split index (== rank in cluster)
  const int n0 = blockIdx.y * kNcta;
  const int m0 = blockIdx.z * L::MCTA;
  const int S = p.splits;
  const int kt_begin = (int)(((long long)rank * p.kg_tiles) / S);
  const int kt_end = (int)(((long long)(rank + 1) * p.kg_tiles) / S);
  const int ntiles = kt_end - kt_begin;
  const int nsub = ntiles * C::SUBS;

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = smem_u32(smem + L::IDX_OFF);
  const uint32_t a_s0 = smem_u32(smem + L::A_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::MISC_OFF);
  float* scale_s = reinterpret_cast<float*>(smem + L::SCALE_OFF);
  const uint32_t mbar = smem_u32(smem + L::MBAR_OFF);  // FULL b at +8b, EMPTY b at +16+8b

  if (tid == L::BUILDER0) {
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(mbar + mb_full(b), kBuilderWarps);
      mbar_init(mbar + mb_empty(b), WARPS);
    }
    for (int st = 0; st < kStageBufs; ++st)
      mbar_init(mbar + mb_stage(st), 1);  // bulk-copy completion of a staged tile
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();  // mbarriers initialised

  uint32_t tmem_base = 0;
  if (warp >= WARPS) {
    // =========================== builder warps: staging + table builds
    const int bt = tid - L::BUILDER0;
    const int bw = warp - WARPS;
    const bool bulk = (p.a_vec == 16);
    if (ntiles > 0) {
      // the packed weights do not depend on the previous kernel: stage tile
      // 0's indices before waiting for it, then its activations
      if (bulk) {
        stage_tile_bulk<G, WARPS>(p, kt_begin, 0, m0, n0, smem, bt, mbar + mb_stage(0), true, false, true);
        pdl_wait();
        stage_tile_bulk<G, WARPS>(p, kt_begin, 0, m0, n0, smem, bt, mbar + mb_stage(0), false, true, false);
      } else {
        stage_tile<G, WARPS>(p, kt_begin, 0, m0, n0, smem, bt, /*what=*/1);
        pdl_wait();
        stage_tile<G, WARPS>(p, kt_begin, 0, m0, n0, smem, bt, /*what=*/2);
      }
    } else {
      pdl_wait();
    }
    if (!ACC_ONLY && bt < kNcta) {
      const int n = n0 + bt;
      scale_s[bt] = (n < p.N) ? __fmul_rn(__ldg(p.a_scale + n), p.w_scale) : 0.f;
    }
#pragma unroll 1
    for (int u = 0; u < nsub + C::NBUF; ++u) {
      if (u >= C::NBUF)  // lookups of u - NBUF done with this buffer
        mbar_wait(mbar + mb_empty(u % C::NBUF), ((u / C::NBUF) - 1) & 1);
      if (u >= nsub) continue;
      const int T = u / C::SUBS, sub = u - T * C::SUBS;
      if (sub == 0) {
        if (bulk) {
          if (T + 1 < ntiles) {
            const int b1 = (T + 1) % kStageBufs;
            stage_tile_bulk<G, WARPS>(p, kt_begin + T + 1, b1, m0, n0, smem, bt, mbar + mb_stage(b1),
                                      true, true, true);
          }
          mbar_wait(mbar + mb_stage(T % kStageBufs), (T / kStageBufs) & 1);
        } else if (T + 1 < ntiles) {
          stage_tile<G, WARPS>(p, kt_begin + T + 1, (T + 1) % kStageBufs, m0, n0, smem, bt, 3);
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          cp_async_wait_all();
        }
        bar_sync(5, kBuilderWarps * 32);  // tile T's A rows visible to all builders
      }
#ifndef VLUT_K1_NOBUILD  // (timing experiment only: tables left unbuilt)
      // 16-byte-store builders, except in the 16-warp variants (96-register
      // budget: the wide builders' 32-40 delta registers would spill there)
      if constexpr (kWideBuild<WARPS>)
        build_tables_wide<G, L::BW>(tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES),
                                    a_s0 + (uint32_t)((T % kStageBufs) * C::A_BYTES), sub * C::GS,
                                    bw, lane, p.a3d != 0);
      else
        build_tables<G, L::BW>(tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES),
                               a_s0 + (uint32_t)((T % kStageBufs) * C::A_BYTES), sub * C::GS, bw,
                               lane);
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + mb_full(u % C::NBUF));  // table u (and tile T's indices) ready
    }
  } else {
    // =========================== lookup warps: one output row per thread
    // TMEM for the int32 accumulators: allocated by warp 0 while the
    // builders already stage and build (lookup warps only wait for it)
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(kTmemCols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tmem_fence_before();
    bar_sync(6, L::MCTA);
    tmem_fence_after();
    tmem_base = *tmem_slot;
    VLUT_STAMP(1);
    // lane-rotated chunk order: slot s of this lane holds tokens 8c..8c+7,
    // c = (lane + s) & 7
    uint32_t rot[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)(chunk_of<false>(lane, s) * 16);
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    uint32_t sw[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int q = 0; q < 4; ++q) sw[s][q] = 0;
    int32_t nneg = 0;
    bool first = true;
    int since_flush = warp % kFlushTiles;  // stagger the widening across warps
    uint32_t iwa[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
#pragma unroll
      for (int sub = 0; sub < C::SUBS; ++sub) {
        const int u = t * C::SUBS + sub;
        mbar_wait(mbar + mb_full(u % C::NBUF), (u / C::NBUF) & 1);  // table u built
        if (u == 0) VLUT_STAMP(2);
        const uint32_t idx_row = idx_s + (uint32_t)((t % kStageBufs) * L::IDX_BYTES + tid * 16);
        if (sub == 0) {
          const uint4 iw = lds128(idx_row);
          iwa[0] = iw.x; iwa[1] = iw.y; iwa[2] = iw.z; iwa[3] = iw.w;
        }
        lookup_sub<G, kLookupGP<WARPS>, kLookupLB<WARPS, 1>>(
            sub, tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES), iwa, idx_row, rot, sw, nneg);
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar + mb_empty(u % C::NBUF));  // table buffer u & 1 free
      }
      if (++since_flush >= kFlushTiles || t + 1 == ntiles) {
        since_flush = 0;
        flush_tmem<G, kLookupGP<WARPS> == 1>(sw, nneg, taddr, first);
        first = false;
      }
    }
    pdl_wait();  // (no-op by now) formally orders the epilogue's a_scale reads
  }
  // allow the next kernel in the stream to start its own prologue
  pdl_launch_dependents();

  VLUT_STAMP(3);
  // ---- int32 tile -> shared (a5).  Row r (lookup thread), 16-byte unit u
  // of the 256-byte row stored at u ^ ((r >> 2) & 1): conflict-free for both
  // the lane-per-row writes below and the row-contiguous reads after.
  // epilogue rows of each cluster rank: rows_per (a multiple of 4), the last
  // rank(s) may own fewer
  const int rows_per = ((L::MCTA + S - 1) / S + 3) & ~3;
  tmem_fence_before();
  __syncthreads();  // every table read done before the region is reused
  tmem_fence_after();
  if (warp < WARPS) {
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    const int32_t bias_total = C::BIAS * kKgTile * ntiles;
    const uint32_t red_s = tab_s;
    const int r = tid;
    const uint32_t swz = (uint32_t)((r >> 2) & 1);
    uint32_t v[4][16];
    if (ntiles > 0) {
#pragma unroll
      for (int h = 0; h < 4; ++h) tmem_ld16(taddr + 16 * h, v[h]);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int i = 0; i < 16; ++i) v[h][i] = 0;
    }
    if (p.out_t) {
      // token-major tile T[n][row]: lanes write consecutive rows (bank = lane)
#pragma unroll
      for (int h = 0; h < 4; ++h) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = chunk_of<false>(lane, 2 * h + e);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            sts32(red_s + (uint32_t)(((8 * c + j) * L::MCTA + r) * 4), v[h][8 * e + j] - bias_total);
        }
      }
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int s = 2 * h + e;
          const uint32_t c = (uint32_t)chunk_of<false>(lane, s);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint32_t uu = (2 * c + hh) ^ swz;
            const uint32_t* x = v[h] + 8 * e + 4 * hh;
            sts128(red_s + r * 256 + uu * 16, x[0] - bias_total, x[1] - bias_total,
                   x[2] - bias_total, x[3] - bias_total);
          }
        }
      }
    }
  }
  VLUT_STAMP(4);
  tmem_fence_before();
  cg::cluster_group cluster = cg::this_cluster();
  if (S > 1) cluster.sync(); else __syncthreads();
  VLUT_STAMP(5);
  if (warp == 0) {
    tmem_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                 "n"(kTmemCols)
                 : "memory");
  }

  // ---- reduce across the cluster + epilogue (a5, a6): all loads of a
  // thread's units first (latency overlapped), then convert + store
  {
    const int r_begin = min(L::MCTA, rank * rows_per);
    const int my_rows = min(rows_per, L::MCTA - r_begin);
    const int units = my_rows * 16;
    const int4* red_local = reinterpret_cast<const int4*>(smem);
    // unit e -> int4 offset in the tile:
    //   [M][N] out: row r_begin + e/16, tokens 4(e%16)..+3 (XOR-swizzled row)
    //   [N][M] out: token e / (my_rows/4), rows r_begin + 4(e % (my_rows/4))..+3
    const int rq = max(1, my_rows >> 2);
    auto tile_off = [&](int e) -> int {
      if (p.out_t) return ((e / rq) * L::MCTA + r_begin) / 4 + (e % rq);
      const int r = r_begin + (e >> 4);
      return r * 16 + ((e & 15) ^ ((r >> 2) & 1));
    };
    // chunks of CH units per thread (all loads of a chunk first): the
    // 16-warp variants' 13 units x 2 int4 arrays would not fit 102 registers
    constexpr int CH = (WARPS >= 16) ? 4 : L::EPI_UNITS;
    float tok_max[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int c0 = 0; c0 < L::EPI_UNITS; c0 += CH) {
      int4 acc4[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = tid + (c0 + i) * L::THREADS;
        acc4[i] = make_int4(0, 0, 0, 0);
        if (e < units) acc4[i] = red_local[tile_off(e)];
      }
      {
        for (int q = 1; q < S; ++q) {
          const int4* rem = cluster.map_shared_rank(red_local, (rank + q) % S);
          int4 w4[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            const int e = tid + (c0 + i) * L::THREADS;
            w4[i] = make_int4(0, 0, 0, 0);
            if (e < units) w4[i] = rem[tile_off(e)];
          }
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            acc4[i].x += w4[i].x; acc4[i].y += w4[i].y; acc4[i].z += w4[i].z; acc4[i].w += w4[i].w;
          }
        }
      }
#ifdef VLUT_TIMING_EPI
      if (c0 == 0) VLUT_STAMP(6);
#endif
      if (p.out_t) {
        // fused output transposition: out[n][m .. m+3], one token scale
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int e = tid + (c0 + i) * L::THREADS;
          if (e >= units) continue;
          const int nl = e / rq;
          const int n = n0 + nl;
          const int m = m0 + r_begin + 4 * (e % rq);
          if (n >= p.N || m >= p.M) continue;
          const int4 vv4 = acc4[i];
          const int vv[4] = {vv4.x, vv4.y, vv4.z, vv4.w};
          if constexpr (ACC_ONLY) {
            int32_t* o = reinterpret_cast<int32_t*>(p.out) + (size_t)n * p.M + m;
            if (p.out_vec4 && m + 3 < p.M) *reinterpret_cast<int4*>(o) = vv4;
            else for (int k = 0; k < 4 && m + k < p.M; ++k) o[k] = vv[k];
          } else {
            float* o = p.out + (size_t)n * p.M + m;
            const float sc = scale_s[nl];
            float f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) f[k] = __fmul_rn((float)vv[k], sc);
            if (p.out_vec4 && m + 3 < p.M) *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
            else for (int k = 0; k < 4 && m + k < p.M; ++k) o[k] = f[k];
          }
        }
      } else
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = tid + (c0 + i) * L::THREADS;
        if (e >= units) continue;
        const int u = e & 15;  // == tid & 15 (THREADS is a multiple of 16)
        const int m = m0 + r_begin + (e >> 4);
        const int n = n0 + 4 * u;
        if (m >= p.M || n >= p.N) continue;
        int4 vv4 = acc4[i];
        if (p.acc_in) {  // chained K ranges (mixed g=5/g=4 schedule): add the prior partial
          const int32_t* src = p.acc_in + (size_t)m * p.N + n;
          if (p.out_vec4 && n + 3 < p.N) {
            const int4 w = __ldcg(reinterpret_cast<const int4*>(src));
            vv4.x += w.x; vv4.y += w.y; vv4.z += w.z; vv4.w += w.w;
          } else {
            int t4[4] = {0, 0, 0, 0};
            for (int k = 0; k < 4 && n + k < p.N; ++k) t4[k] = __ldcg(src + k);
            vv4.x += t4[0]; vv4.y += t4[1]; vv4.z += t4[2]; vv4.w += t4[3];
          }
        }
        if constexpr (ACC_ONLY) {
          int32_t* o = reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n;
          if (p.out_vec4 && n + 3 < p.N) {
            *reinterpret_cast<int4*>(o) = vv4;
          } else {
            const int vv[4] = {vv4.x, vv4.y, vv4.z, vv4.w};
            for (int k = 0; k < 4 && n + k < p.N; ++k) o[k] = vv[k];
          }
        } else {
          float* o = p.out + (size_t)m * p.N + n;
          const int vv[4] = {vv4.x, vv4.y, vv4.z, vv4.w};
          float f[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) f[k] = __fmul_rn((float)vv[k], scale_s[4 * u + k]);
          if (p.mul_in) {  // fused element-wise product (config 5: h = gate (.) up)
            const float* mi = p.mul_in + (size_t)m * p.N + n;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (n + k < p.N) f[k] = __fmul_rn(f[k], __ldg(mi + k));
          }
          if (p.amax_out && m < p.amax_rows) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (n + k < p.N) tok_max[k] = fmaxf(tok_max[k], fabsf(f[k]));
          }
          if (p.out_vec4 && n + 3 < p.N) {
            const float4 f4 = make_float4(f[0], f[1], f[2], f[3]);
            if (p.out_mc)
              st_mc_v4(o, f4);
            else
              *reinterpret_cast<float4*>(o) = f4;
            // fused all-gather: the same 16 bytes to every peer's copy (P2P
            // stores over NVLink, overlapping the other CTAs' compute)
            for (int pi = 0; pi < p.n_peers; ++pi)
              *reinterpret_cast<float4*>(p.peer_out[pi] + (size_t)m * p.N + n) = f4;
          } else {
            for (int k = 0; k < 4 && n + k < p.N; ++k) {
              if (p.out_mc)
                st_mc_f32(o + k, f[k]);
              else
                o[k] = f[k];
            }
            for (int pi = 0; pi < p.n_peers; ++pi)
              for (int k = 0; k < 4 && n + k < p.N; ++k) p.peer_out[pi][(size_t)m * p.N + n + k] = f[k];
          }
        }
      }
    }
    // remote reads done: arrive now, wait only before exit (the peers keep
    // their shared memory until every CTA of the cluster has read it)
    if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
#ifndef VLUT_TIMING_EPI
    VLUT_STAMP(6);
#endif
    if constexpr (!ACC_ONLY) {
      if (p.amax_out) {
        // fused re-quantization (f1): per-token |out| max of this CTA ->
        // global atomicMax on the float bits (non-negative floats order as
        // unsigned integers).  Thread's token quad: 4 (tid & 15) .. +3.
        unsigned* cta_max = reinterpret_cast<unsigned*>(smem + L::AMAX_OFF);
        if (tid < kNcta) cta_max[tid] = 0u;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tok_max[k] = fmaxf(tok_max[k], __shfl_xor_sync(0xffffffffu, tok_max[k], 16));
          if (lane < 16) atomicMax(cta_max + 4 * (tid & 15) + k, __float_as_uint(tok_max[k]));
        }
        __syncthreads();
        if (tid < kNcta && n0 + tid < p.N && cta_max[tid] != 0u)
          atomicMax(p.amax_out + n0 + tid, cta_max[tid]);
      }
    }
  }
  VLUT_STAMP(7);
  if (S > 1) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}

}  // namespace vlut
