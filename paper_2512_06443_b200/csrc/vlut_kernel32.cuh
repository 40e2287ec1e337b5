// vlut_kernel32.cuh -- K1-32: the fused Vec-LUT mpGeMM with 32-token tiles.
//
// K1 (vlut_kernel.cuh) stores a table row of 64 tokens = 128 bytes, one full
// bank line, so a lookup's 8 LDS.128 of one row are conflict-free in the
// lane-rotated order.  Its 64-token N-tile leaves the headline shape
// (6912 x 2560, N = 256) with 72 (384-row) tiles for 148 SMs: the K range is
// split over a cluster pair and the int32 partials (48 KB per CTA) cross
// distributed shared memory at ~8.5 B/clk each way (~3 us per launch).
//
// K1-32 halves the N-tile to 32 tokens (64-byte rows) and keeps every lookup
// conflict-free by PAIRING groups: line p of pair jp holds row p of group
// 2jp in bytes [0, 64) and row p of group 2jp+1 in bytes [64, 128) of one
// 128-byte bank line.  A lookup thread reads, for its output row, row pos0
// of group 2jp and row pos1 of group 2jp+1 (4 chunks each) in the order
// chunk v = (lane & 7) ^ s, s = 0..7: v < 4 is a chunk of the first half
// (group 2jp), v >= 4 of the second half (group 2jp+1), and the 8 lanes of an
// LDS.128 phase always cover the 8 bank groups whatever rows they read.  For
// lanes with (lane & 7) < 4 the first four steps read group 2jp; for the
// others group 2jp+1 -- so steps 0..3 read line LA and steps 4..7 line LB,
// (LA, LB) = (L0, L1) or (L1, L0) per lane.  Step s and s+4 land in the same
// SWAR slot k = s & 3 (tokens of chunk (lane ^ k) & 3): 16 accumulator
// registers instead of 32.  The same 2 bytes of shared memory per
// lookup-add, the same half-table build share per row, twice the tiles: the
// headline runs as 144 CTAs without split-K and without a DSMEM exchange.
//
// Everything else is K1's: builder warps stage index rows (one bulk copy)
// and the activation tile (2-D TMA, box 32 x 16g) and build the half tables
// along base-3 reflected Gray codes; one builder lane computes
// two tokens of one group's half-table rows, the two halves of a warp the
// two groups of a pair, so a warp-wide 4-byte store fills one bank line;
// SWAR fields (T + 128 g) widen into TMEM int32 every 48 groups;
// optional cluster split-K (DSMEM); fp32 epilogue
// out = fl((float)acc * fl(a_scale[n] * w_scale)) through a swizzled shared
// tile for coalesced 16-byte stores.
#pragma once
#include "vlut_kernel.cuh"

namespace vlut {

constexpr int kN32 = 32;  // tokens per CTA
// mbarrier slots of K1-32 (byte offsets): FULL[NB], EMPTY[NB], STAGE[NB + 1]
template <int NB>
__device__ __forceinline__ constexpr int m32_full(int b) { return 8 * b; }
template <int NB>
__device__ __forceinline__ constexpr int m32_empty(int b) { return 8 * NB + 8 * b; }
template <int NB>
__device__ __forceinline__ constexpr int m32_stage(int s) { return 16 * NB + 8 * s; }

template <int G, bool SK = false>
struct Cfg32 {
  static constexpr int R = pow3(G);
  static constexpr int ZERO = (R - 1) / 2;
  static constexpr int HR = (R + 1) / 2;            // stored half-table positions
#ifndef VLUT_K32_NBUF
#define VLUT_K32_NBUF 3
#endif
  // table buffers: K1-32 VLUT_K32_NBUF; the stream-K variant (index tiles of
  // up to 1536 rows) 3 at g = 4 (measured 0.2-1.1 % faster than 2,
  // profiles/r02_sk32_fixup.txt) and 2 at g = 5 (243-row pair tables)
#ifndef VLUT_SK32_NBUF4
#define VLUT_SK32_NBUF4 3
#endif
  static constexpr int NBUF = (G == 4 && !SK) ? VLUT_K32_NBUF : (G == 4 ? VLUT_SK32_NBUF4 : 2);
  static constexpr int GS = (G == 4) ? 16 : 8;      // groups per sub-stage (even)
  static constexpr int PAIRS = GS / 2;
  static constexpr int SUBS = kKgTile / GS;
  static constexpr int BIAS = 128 * G;
  static constexpr int PAIR_BYTES = HR * 128;       // one bank line per position
  static constexpr int TAB_BYTES = PAIRS * PAIR_BYTES;
  static constexpr int A_ROWS = kKgTile * G;
  static constexpr int A_BYTES = A_ROWS * kN32;     // 16g rows x 32 tokens
  static constexpr int IDX_MASK = (G == 4) ? 0x7F : 0xFF;
  // staging: while building tile T the builders stage tile T + AHEAD (its
  // index rows and activations land during AHEAD tiles of lookups: a tile
  // is only ~2 us of lookups here); the builders run up to NBUF tables ahead
  // of the lookup warps, which may still have to read the index rows of tile
  // T - NBUF + 1 -- so STAGE >= NBUF + AHEAD buffers
#ifndef VLUT_K32_AHEAD
#define VLUT_K32_AHEAD 2
#endif
  static constexpr int AHEAD = SK ? 1 : VLUT_K32_AHEAD;
  static constexpr int STAGE = NBUF + AHEAD;
  static_assert(STAGE * 8 + 16 * NBUF <= 96, "mbarrier region");
  static_assert(kFlushTiles * kKgTile * 2 * BIAS <= 65535, "SWAR field overflow");
};

// RPT output rows per lookup thread (row block rb = rows rb*NLT + tid); SK =
// the stream-K variant's buffer counts.
template <int G, int WARPS, int RPT = 1, bool SK = false>
struct Layout32 {
  using C = Cfg32<G, SK>;
  static constexpr int NLT = WARPS * 32;
  static constexpr int THREADS = NLT + kBuilderWarps * 32;
  static constexpr int BUILDER0 = NLT;
  static constexpr int MCTA = NLT * RPT;
  // int32 tile [row][32] of the cluster epilogue (the stream-K epilogue
  // works from registers: no tile)
  static constexpr int RED_BYTES = SK ? 0 : MCTA * kN32 * 4;
  static constexpr int CB = 32 * ((WARPS + 3) / 4);   // TMEM columns per row block
  static constexpr int TMEM_COLS = CB * RPT <= 32 ? 32 : CB * RPT <= 64 ? 64
                                   : CB * RPT <= 128 ? 128 : CB * RPT <= 256 ? 256 : 512;
  static_assert(CB * RPT <= 512, "TMEM columns");
  static constexpr int TAB_REGION = C::NBUF * C::TAB_BYTES > RED_BYTES
                                        ? C::NBUF * C::TAB_BYTES : RED_BYTES;
  static constexpr int IDX_OFF = TAB_REGION;
  static constexpr int IDX_BYTES = MCTA * 16;
  static constexpr int A_OFF = IDX_OFF + C::STAGE * IDX_BYTES;
  static constexpr int MISC_OFF = A_OFF + C::STAGE * C::A_BYTES;
  static constexpr int MBAR_OFF = MISC_OFF + 16;
  static constexpr int SCALE_OFF = MBAR_OFF + 96;
  static constexpr int SMEM = SCALE_OFF + kN32 * 4;
  static constexpr int EPI_UNITS = (MCTA * 8 + THREADS - 1) / THREADS;  // 16-B units / thread
  static_assert(WARPS <= 16, "TMEM: at most 4 column blocks of 32");
};

// ---------------------------------------------------------------- staging (a2)
template <int G, int WARPS, int RPT = 1, bool SK = false>
__device__ __forceinline__ void stage32(const Params& p, int kt, int buf, int m0, int n0,
                                        uint8_t* smem, int bt, uint32_t stg_mbar, bool do_idx,
                                        bool do_act, bool arm) {
  using C = Cfg32<G, SK>;
  using L = Layout32<G, WARPS, RPT, SK>;
  constexpr int NB = kBuilderWarps * 32;
  const int idx_rows = max(0, min(L::MCTA, p.m_pad - m0));
  const int k0 = kt * kKgTile * G;
  uint8_t* idx_dst = smem + L::IDX_OFF + buf * L::IDX_BYTES;
  uint8_t* a_dst = smem + L::A_OFF + buf * C::A_BYTES;
  if (do_idx)  // rows past m_pad: zero (index 0 rows are never looked up by valid rows)
    for (int i = idx_rows * 16 + bt * 16; i < L::MCTA * 16; i += NB * 16)
      *reinterpret_cast<uint4*>(idx_dst + i) = make_uint4(0, 0, 0, 0);
  if (bt < 32) {
    if (arm && bt == 0)  // the A box always delivers 16g x 32 bytes (OOB zero-filled)
      mbar_expect_tx(stg_mbar, (uint32_t)(idx_rows * 16 + C::A_BYTES));
    __syncwarp();
    if (do_idx && bt == 0 && idx_rows > 0)
      bulk_g2s(smem_u32(idx_dst), p.payload + ((size_t)kt * p.m_pad + m0) * 16,
               (uint32_t)(idx_rows * 16), stg_mbar);
    if (do_act && bt == 0) {
      if (p.a3d)  // [r][group][token]: box (32 tokens, 16 groups, g rows)
        tma_load_3d(smem_u32(a_dst), &p.a_map, n0, kt * kKgTile, 0, stg_mbar);
      else
        tma_load_2d(smem_u32(a_dst), &p.a_map, n0, k0, stg_mbar);
    }
  }
}

// ---------------------------------------------------------------- table build (a3)
// Wide-store builders: a builder warp writes FOUR pairs' lines at once with
// 16-byte stores.  Lane = 8 q + ch: q picks pair 4 pg + q of the warp's pair
// group pg, ch the 16-byte chunk of the 128-byte line (ch < 4: tokens
// 8 ch .. 8 ch + 7 of group 2jp, ch >= 4: of group 2jp+1), so one STS.128
// fills four lines (four wavefronts, conflict-free) and a table costs a
// quarter of the store instructions of 4-byte stores -- the lookup warps keep
// the shared-memory queue full, and builders issuing 4-byte stores could not
// keep up (measured: halving their stores took K1-32 from 94 to 86 us).
//
// The activation tile is staged either as [group][r][32 tokens] (2-D map)
// or, when K % g == 0, as [r][group][32 tokens] (3-D map): then the four
// groups a builder load phase reads (same r, consecutive groups) fall in
// four different 32-byte bank windows instead of one (4-way conflicts).
template <int G>
__device__ __forceinline__ void build_tables32(uint32_t tab_s, uint32_t a_s, int grp0, int bw,
                                               int lane, bool a3d) {
  using C = Cfg32<G>;
  // warps per pair group: g = 4 -> 2 (two groups of 4 pairs), g = 5 -> 4
  constexpr int WPG = kBuilderWarps / (C::PAIRS / 4);
  static_assert(C::PAIRS % 4 == 0 && kBuilderWarps % (C::PAIRS / 4) == 0, "builder split");
  constexpr uint32_t K1 = 0x00010001u;
  constexpr uint32_t C128 = 128u * K1;
  const int pg = bw / WPG, h = bw % WPG;
  const int q = lane >> 3, ch = lane & 7;
  const int jp = 4 * pg + q;
  const int jg = 2 * jp + (ch >> 2);  // group within the sub-stage
  const int c = ch & 3;               // tokens 8c .. 8c + 7
  uint32_t P[G][4];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    uint32_t x0, x1;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n"
                 : "=r"(x0), "=r"(x1)
                 : "r"(a_s + (uint32_t)((a3d ? (r * kKgTile + grp0 + jg) : ((grp0 + jg) * G + r)) *
                                             kN32 + 8 * c)));
    x0 ^= 0x80808080u;  // int8 a -> a + 128
    x1 ^= 0x80808080u;
    const uint32_t U[4] = {__byte_perm(x0, 0u, 0x4140), __byte_perm(x0, 0u, 0x4342),
                           __byte_perm(x1, 0u, 0x4140), __byte_perm(x1, 0u, 0x4342)};
#pragma unroll
    for (int w = 0; w < 4; ++w) P[r][w] = U[w] - C128;  // +a_r as a packed arithmetic delta
  }
  build_units<G>(h, tab_s + (uint32_t)(jp * C::PAIR_BYTES + ch * 16), P);
}

// ---------------------------------------------------------------- lookups (a4)
// Pairs [SUB*PAIRS, ...) of the K-tile.  PB pairs per load batch (8 LDS.128
// each).  Slots k < NX negate by XOR (ALU pipe), k >= NX by multiply (FMA
// pipe): the per-lane line selection adds ALU work, so fewer XOR slots than
// K1 keep the two integer pipes balanced.
#ifndef VLUT_K32_NX
#define VLUT_K32_NX 1
#endif
constexpr int kNX32 = VLUT_K32_NX;
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;  // PTX prmt default mode: selector msb = replicate the byte's sign
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Per-lane PRMT selectors of the index decode (computed once): a pair's two
// groups sit at bytes bb0, bb0 + 1 (bb0 in {0, 2}) of an index word; lane
// side `so` = 0 reads group 2jp in steps 0..3 (line A), so = 1 group 2jp+1.
//   pos[bb0/2][0|1]: byte of line A | B into the low byte (zeros above)
//   sgn[bb0/2][0|1]: that byte's sign (msb) replicated over all 32 bits
struct Sel32 {
  uint32_t pos[2][2], sgn[2][2];
  __device__ __forceinline__ void init(int so) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t xa = (uint32_t)(2 * h + so), xb = (uint32_t)(2 * h + 1 - so);
      pos[h][0] = 0x4440u | xa;
      pos[h][1] = 0x4440u | xb;
      sgn[h][0] = 0x8888u | (xa * 0x1111u);
      sgn[h][1] = 0x8888u | (xb * 0x1111u);
    }
  }
};

// Pairs [SUB*PAIRS, ...) of the K-tile.  PB pairs per load batch (8 LDS.128
// each).  Index decode per 4-group word with byte-SIMD ops: |i - z| for all
// four bytes in one VABSDIFF4, the signs in bit 7 of (i + 128 - z) (no
// carries: i + 128 - z < 256), the negation count by POPC; per pair two PRMTs
// pick the lane's line-A / line-B positions (no SELs), two more the signs.
// Slots k < NX negate by XOR (ALU pipe), k >= NX by multiply (FMA pipe).
template <int G, int PB>
__device__ __forceinline__ void lookup_sub32(const int SUB, uint32_t tab, const uint32_t (&iwa)[4],
                                             const uint32_t (&rot)[8], const Sel32& sel,
                                             uint32_t (&sw)[4][4], int32_t& nneg) {
  using C = Cfg32<G>;
  static_assert(C::PAIRS % PB == 0, "pairs per batch");
  constexpr uint32_t Z4 = (uint32_t)C::ZERO * 0x01010101u;
  constexpr uint32_t NB4 = (uint32_t)(128 - C::ZERO) * 0x01010101u;
  constexpr int NWD = C::GS / 4;  // index words of this sub-stage
  uint32_t aw[NWD], ntw[NWD];
#pragma unroll
  for (int wd = 0; wd < NWD; ++wd) {
    const uint32_t word = iwa[(SUB * C::GS) / 4 + wd];
    aw[wd] = __vabsdiffu4(word, Z4);               // |i - z| per byte
    ntw[wd] = ~(word + NB4);                       // bit 7 set <=> i < z (negate)
    nneg -= __popc(ntw[wd] & 0x80808080u);
  }
#pragma unroll
  for (int jb = 0; jb < C::PAIRS; jb += PB) {
    uint4 va[PB][4], vb[PB][4];
    uint32_t ma[PB], mb[PB];
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const int jp = jb + q;
      const int wd = (2 * jp) >> 2, h = jp & 1;  // word, byte pair (bytes 2h, 2h+1)
      const uint32_t base = tab + (uint32_t)(jp * C::PAIR_BYTES);
      const uint32_t la = base + prmt(aw[wd], 0u, sel.pos[h][0]) * 128u;
      const uint32_t lb = base + prmt(aw[wd], 0u, sel.pos[h][1]) * 128u;
      ma[q] = prmt(ntw[wd], 0u, sel.sgn[h][0]);
      mb[q] = prmt(ntw[wd], 0u, sel.sgn[h][1]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // lines are 128-aligned: + == |
        va[q][k] = lds128(la + rot[k]);
        vb[q][k] = lds128(lb + rot[k + 4]);
      }
    }
#pragma unroll
    for (int q = 0; q < PB; ++q) {
      const uint32_t sa = ma[q] * 2u + 1u, sb = mb[q] * 2u + 1u;  // +1 / -1
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < kNX32) {
          sw[k][0] += (va[q][k].x ^ ma[q]) + (vb[q][k].x ^ mb[q]);
          sw[k][1] += (va[q][k].y ^ ma[q]) + (vb[q][k].y ^ mb[q]);
          sw[k][2] += (va[q][k].z ^ ma[q]) + (vb[q][k].z ^ mb[q]);
          sw[k][3] += (va[q][k].w ^ ma[q]) + (vb[q][k].w ^ mb[q]);
        } else {
          sw[k][0] += va[q][k].x * sa + vb[q][k].x * sb;
          sw[k][1] += va[q][k].y * sa + vb[q][k].y * sb;
          sw[k][2] += va[q][k].z * sa + vb[q][k].z * sb;
          sw[k][3] += va[q][k].w * sa + vb[q][k].w * sb;
        }
      }
    }
  }
}

// Widen (INT16 -> INT32) the 4 slots into TMEM columns 8k .. 8k + 7.
template <int G>
__device__ __forceinline__ void flush32(uint32_t (&sw)[4][4], int32_t& nneg, uint32_t taddr,
                                        bool first) {
  constexpr uint32_t K1 = 0x00010001u;
  const uint32_t cnt = (uint32_t)(-nneg);
  const uint32_t corr_xor = cnt * (2u * Cfg32<G>::BIAS * K1 + 1u);
  const uint32_t corr_mul = cnt * (2u * Cfg32<G>::BIAS * K1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
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
      const int k = 2 * h + e;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t w = sw[k][q] + (k < kNX32 ? corr_xor : corr_mul);
        v[8 * e + 2 * q] += w & 0xFFFFu;
        v[8 * e + 2 * q + 1] += w >> 16;
        sw[k][q] = 0;
      }
    }
    tmem_st16(taddr + 16 * h, v);
  }
  tmem_wait_st();
  nneg = 0;
}

// ---------------------------------------------------------------- the kernel
template <int G, int WARPS, bool ACC_ONLY>
__global__ void __launch_bounds__((WARPS + kBuilderWarps) * 32, 1)
    vlut_mpgemm32_kernel(const __grid_constant__ Params p) {
  using C = Cfg32<G>;
  using L = Layout32<G, WARPS>;
#ifndef VLUT_K32_PB
#define VLUT_K32_PB 2
#endif
  constexpr int PB = VLUT_K32_PB;  // pairs per load batch: 8 PB LDS.128 in flight
  extern __shared__ __align__(1024) uint8_t smem[];
  VLUT_STAMP(0);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int rank = blockIdx.x;  // split index (== rank in cluster)
  const int n0 = blockIdx.y * kN32;
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
  const uint32_t mbar = smem_u32(smem + L::MBAR_OFF);

  if (tid == L::BUILDER0) {
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(mbar + m32_full<C::NBUF>(b), kBuilderWarps);
      mbar_init(mbar + m32_empty<C::NBUF>(b), WARPS);
    }
    for (int st = 0; st < C::STAGE; ++st) mbar_init(mbar + m32_stage<C::NBUF>(st), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  uint32_t tmem_base = 0;
  if (warp >= WARPS) {
    // =========================== builders: staging + table builds
    const int bt = tid - L::BUILDER0;
    const int bw = warp - WARPS;
    // weights are not an output of the previous kernel (vlut.h): the first
    // AHEAD tiles' index rows before griddepcontrol.wait, activations after
    const int pre = min(ntiles, C::AHEAD);
    for (int T = 0; T < pre; ++T)
      stage32<G, WARPS>(p, kt_begin + T, T, m0, n0, smem, bt, mbar + m32_stage<C::NBUF>(T), true,
                        false, true);
    pdl_wait();
    for (int T = 0; T < pre; ++T)
      stage32<G, WARPS>(p, kt_begin + T, T, m0, n0, smem, bt, mbar + m32_stage<C::NBUF>(T), false,
                        true, false);
    if (!ACC_ONLY && bt < kN32) {
      const int n = n0 + bt;
      scale_s[bt] = (n < p.N) ? __fmul_rn(__ldg(p.a_scale + n), p.w_scale) : 0.f;
    }
#pragma unroll 1
    for (int u = 0; u < nsub + C::NBUF; ++u) {
      if (u >= C::NBUF) mbar_wait(mbar + m32_empty<C::NBUF>(u % C::NBUF), ((u / C::NBUF) - 1) & 1);
      if (u >= nsub) continue;
      const int T = u / C::SUBS, sub = u - T * C::SUBS;
      if (sub == 0) {
        if (T + C::AHEAD < ntiles) {
          const int b1 = (T + C::AHEAD) % C::STAGE;
          stage32<G, WARPS>(p, kt_begin + T + C::AHEAD, b1, m0, n0, smem, bt,
                            mbar + m32_stage<C::NBUF>(b1), true, true, true);
        }
        mbar_wait(mbar + m32_stage<C::NBUF>(T % C::STAGE), (T / C::STAGE) & 1);
        bar_sync(5, kBuilderWarps * 32);  // tile T's rows visible to all builders
      }
#ifndef VLUT_K32_NOBUILD  // (timing experiment only: tables left unbuilt)
      build_tables32<G>(tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES),
                        a_s0 + (uint32_t)((T % C::STAGE) * C::A_BYTES), sub * C::GS, bw, lane,
                        p.a3d != 0);
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + m32_full<C::NBUF>(u % C::NBUF));
    }
  } else {
    // =========================== lookup warps: one output row per thread
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(L::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tmem_fence_before();
    bar_sync(6, L::MCTA);
    tmem_fence_after();
    tmem_base = *tmem_slot;
    VLUT_STAMP(1);
    uint32_t rot[8];  // chunk (lane & 7) ^ s of a 128-byte line
#pragma unroll
    for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)((((lane & 7) ^ s) & 7) * 16);
    Sel32 sel;
    sel.init((lane & 4) ? 1 : 0);  // lanes (lane & 7) >= 4 read group 2jp+1 first
    const uint32_t taddr =
        tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * (warp >> 2));
    uint32_t sw[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) sw[k][q] = 0;
    int32_t nneg = 0;
    bool first = true;
    int since_flush = warp % kFlushTiles;
    uint32_t iwa[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
#pragma unroll
      for (int sub = 0; sub < C::SUBS; ++sub) {
        const int u = t * C::SUBS + sub;
        mbar_wait(mbar + m32_full<C::NBUF>(u % C::NBUF), (u / C::NBUF) & 1);
        if (u == 0) VLUT_STAMP(2);
        if (sub == 0) {
          const uint4 iw = lds128(idx_s + (uint32_t)((t % C::STAGE) * L::IDX_BYTES + tid * 16));
          iwa[0] = iw.x; iwa[1] = iw.y; iwa[2] = iw.z; iwa[3] = iw.w;
        }
#ifndef VLUT_K32_NOLOOKUP  // (timing experiment only)
        lookup_sub32<G, PB>(sub, tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES), iwa, rot, sel,
                            sw, nneg);
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar + m32_empty<C::NBUF>(u % C::NBUF));
      }
      if (++since_flush >= kFlushTiles || t + 1 == ntiles) {
        since_flush = 0;
        flush32<G>(sw, nneg, taddr, first);
        first = false;
      }
    }
    pdl_wait();  // (no-op by now) formally orders the epilogue's a_scale reads
#ifndef VLUT_K32_TILE_EPI
    if (S == 1) {
      // ---- direct epilogue (no split-K): this thread's row is complete in
      // TMEM once its last flush is done -- read it back and store the fp32
      // (or int32) row straight to global memory, warp by warp, while slower
      // warps still look up (no block barrier, no shared tile).  Slot k of
      // this lane holds tokens 8c .. 8c+7, c = (lane ^ k) & 3.
      const int32_t bias_total = C::BIAS * kKgTile * ntiles;
      uint32_t v[2][16];
      if (ntiles > 0) {
        tmem_ld16(taddr, v[0]);
        tmem_ld16(taddr + 16, v[1]);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 16; ++i) v[h][i] = 0;
      }
      const int m = m0 + tid;
      if (m < p.M) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = (lane ^ k) & 3;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int n = n0 + 8 * c + 4 * hh;
            if (n >= p.N) continue;  // N % 16 == 0: a quad is all-in or all-out
            const uint32_t* x = v[k >> 1] + 8 * (k & 1) + 4 * hh;
            const int a0 = (int)(x[0] - bias_total), a1 = (int)(x[1] - bias_total);
            const int a2 = (int)(x[2] - bias_total), a3 = (int)(x[3] - bias_total);
            if constexpr (ACC_ONLY) {
              *reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n) =
                  make_int4(a0, a1, a2, a3);
            } else {
              const int ul = 8 * c + 4 * hh;
              *reinterpret_cast<float4*>(p.out + (size_t)m * p.N + n) =
                  make_float4(__fmul_rn((float)a0, scale_s[ul]), __fmul_rn((float)a1, scale_s[ul + 1]),
                              __fmul_rn((float)a2, scale_s[ul + 2]), __fmul_rn((float)a3, scale_s[ul + 3]));
            }
          }
        }
      }
      // TMEM is released by warp 0 once every lookup warp has read its columns
      tmem_fence_before();
      bar_sync(6, L::MCTA);
      if (warp == 0) {
        tmem_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                     "n"(L::TMEM_COLS)
                     : "memory");
      }
    }
#endif
  }
  pdl_launch_dependents();
#ifndef VLUT_K32_TILE_EPI
  if (S == 1) return;  // builders have nothing left; lookup warps stored their rows
#endif

  VLUT_STAMP(3);
  // ---- int32 tile -> shared (a5): row r = 128 bytes = 8 units of 4 tokens;
  // unit u of row r stored at position u ^ (r & 7) (conflict-free for the
  // lane-per-row writes here and the 8-threads-per-row reads below)
  const int rows_per = ((L::MCTA + S - 1) / S + 3) & ~3;
  tmem_fence_before();
  __syncthreads();  // every table read done before the region is reused
  tmem_fence_after();
  if (warp < WARPS) {
    const uint32_t taddr =
        tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * (warp >> 2));
    const int32_t bias_total = C::BIAS * kKgTile * ntiles;
    const int r = tid;
    uint32_t v[2][16];
    if (ntiles > 0) {
      tmem_ld16(taddr, v[0]);
      tmem_ld16(taddr + 16, v[1]);
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 16; ++i) v[h][i] = 0;
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 2 * h + e;
        const uint32_t c = (uint32_t)((lane ^ k) & 3);  // tokens 8c .. 8c+7 (units 2c, 2c+1)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const uint32_t uu = (2 * c + hh) ^ (uint32_t)(r & 7);
          const uint32_t* x = v[h] + 8 * e + 4 * hh;
          sts128(tab_s + (uint32_t)(r * 128) + uu * 16, x[0] - bias_total, x[1] - bias_total,
                 x[2] - bias_total, x[3] - bias_total);
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
                 "n"(L::TMEM_COLS)
                 : "memory");
  }

  // ---- reduce across the cluster + epilogue (a5, a6): unit e = row
  // r_begin + e / 8, tokens 4 (e % 8) .. + 3; eight consecutive threads store
  // one row's 128 bytes
  {
    const int r_begin = min(L::MCTA, rank * rows_per);
    const int my_rows = min(rows_per, L::MCTA - r_begin);
    const int units = my_rows * 8;
    const int4* red_local = reinterpret_cast<const int4*>(smem);
    auto tile_off = [&](int e) -> int {
      const int r = r_begin + (e >> 3);
      return r * 8 + ((e & 7) ^ (r & 7));
    };
    constexpr int CH = L::EPI_UNITS;
    int4 acc4[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int e = tid + i * L::THREADS;
      acc4[i] = make_int4(0, 0, 0, 0);
      if (e < units) acc4[i] = red_local[tile_off(e)];
    }
    for (int q = 1; q < S; ++q) {
      const int4* rem = cluster.map_shared_rank(red_local, (rank + q) % S);
      int4 w4[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = tid + i * L::THREADS;
        w4[i] = make_int4(0, 0, 0, 0);
        if (e < units) w4[i] = rem[tile_off(e)];
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        acc4[i].x += w4[i].x; acc4[i].y += w4[i].y; acc4[i].z += w4[i].z; acc4[i].w += w4[i].w;
      }
    }
    if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int e = tid + i * L::THREADS;
      if (e >= units) continue;
      const int u = e & 7;
      const int m = m0 + r_begin + (e >> 3);
      const int n = n0 + 4 * u;
      if (m >= p.M || n >= p.N) continue;  // N % 16 == 0: a unit is all-in or all-out
      if constexpr (ACC_ONLY) {
        *reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n) = acc4[i];
      } else {
        const int vv[4] = {acc4[i].x, acc4[i].y, acc4[i].z, acc4[i].w};
        float f[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] = __fmul_rn((float)vv[k], scale_s[4 * u + k]);
        *reinterpret_cast<float4*>(p.out + (size_t)m * p.N + n) = make_float4(f[0], f[1], f[2], f[3]);
      }
    }
  }
  VLUT_STAMP(7);
  if (S > 1) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}

}  // namespace vlut
