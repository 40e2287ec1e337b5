// vlut_kernel_slot.cuh -- K2: lane-slot LUT mpGeMM for small token counts
// (decode, N = 1 .. 64) and the scalar-LUT (1->1) comparator (f4).
//
// K1 (vlut_kernel.cuh) reads a 128-byte table row (64 tokens) per lookup and
// needs N >= 64 to fill it.  K2 keeps every lookup conflict-free for ANY
// token count by giving each lane of a warp its own shared-memory bank:
//
//   table layout  T[word pair][index i][word w & 1][slot s], 4-byte entries,
//                 one 256-byte row per index i (2 words x 32 slots).  Slot
//                 s = 16 c + j holds copy c (c = 0, 1) of the table of group
//                 j (0..15) of the K-tile, so bank(slot) = s.
//   lookups       lane l (x = l & 15) walks the 16 groups of ITS row in the
//                 XOR order j = step ^ x; at every step the 16 lanes of each
//                 half-warp read 16 different slots and the two halves the
//                 two copies: 32 lanes -> 32 banks, whatever indices they
//                 hold.  One PRMT forms the address (index byte -> bits 8..15,
//                 slot -> bits 0..7); one LDS.32 per lookup and word.
//   words         TPW = 1: a word is ONE token's int32 entry -> the scalar LUT
//                 of T-MAC (each token its own table, N lookups per index,
//                 P:84-85).  TPW = 2: a word packs two tokens as
//                 biased 16-bit fields (field = T + 128 g, as K1) -> a 1->2
//                 vector lookup (the Vec-LUT paradigm) at 2 B of
//                 shared memory per lookup-add, K1's roofline.
//   staging (a2)  a producer warp streams each K-tile's 16-byte index rows of
//                 the CTA (one contiguous block of the packed payload) and its
//                 activation rows A[16g][N] (contiguous: token axis innermost)
//                 into a 2-4 stage ring with cp.async.bulk + one mbarrier per
//                 stage, so HBM stays busy at N = 1 (bandwidth-bound) and the
//                 builders never wait on global-memory latency.
//   build (a3)    builder lanes own a slot: lane l computes ALL 3^g entries of
//                 group l & 15 in the topological order of P:503-513 (one add
//                 per entry), as 9 independent base-3 reflected Gray-code
//                 chains (one per value of the two top trits) for ILP, and
//                 stores one 128-byte wavefront per entry and word.  Full
//                 tables: no sign decode on the lookup path.
//   accumulate    TPW = 1: int32 registers.  TPW = 2: SWAR fields widened into
//                 int32 registers every 48 groups (INT16 -> INT32).
//   split-K (a5)  CTAs of one (M-block, N-tile) split its K-tiles.  The CTA's
//                 int32 tile goes through shared memory; with S > 1 it is
//                 added into a zero-kept workspace by bulk reduce-add copies
//                 (cp.reduce.async.bulk .add.s32: one per CTA when its rows
//                 are contiguous there) and the CTAs arrive at an acq_rel
//                 counter; the last to arrive re-arms it.  Tiles <= 8 KB
//                 (decode): each partial element is one counted 64-bit atomic
//                 add (kAtom64 below); whichever thread adds an element's last
//                 contribution finishes that element, nobody waits.  Larger
//                 tiles: the last one bumps the tile's generation word, the
//                 CTAs (co-resident: cooperative launch) wait for it and each
//                 finishes 1/S of the tile, so no single CTA serialises it.
//                 Integer addition is associative: bit-exact for every split.
//   epilogue (a6) out = fl((float)acc * fl(a_scale[n] * w_scale)), or raw int32.
//
// Citations: P:n = /root/reference/PAPER.md line n.  DESIGN.md §4 (K2) gives
// the byte/instruction budget and the rooflines (HBM at N = 1, shared memory
// otherwise).
#pragma once
#include <type_traits>

#include "vlut_kernel.cuh"
#include "vlut_kernel_sk.cuh"

namespace vlut {
namespace slot {

constexpr int kLW = 16;                           // lookup warps
constexpr int kBW = 2;                            // builder warps
constexpr int kLookupThreads = kLW * 32;
constexpr int kThreads = (kLW + kBW + 1) * 32;    // + 1 producer warp = 608
constexpr int kRowStride = 256;                   // bytes per table index row
constexpr int kSmemMax = 232448;                  // 227 KB opt-in per CTA
constexpr int kFlushTiles = 3;                    // TPW = 2: widen every 48 groups
constexpr int kMaxCounters = 8192;                // split-K tiles (2 counters each) in the workspace
constexpr int kActNMax = 64;                      // activations staged by TMA when N <= 64
constexpr int kMaxStages = 8;                     // staging ring depth (bytes in flight at N = 1)
#ifndef VLUT_SLOT_RAMP
#define VLUT_SLOT_RAMP 2
#endif
// stages issued before the first tile lands (0: no gate, every ring stage's
// index rows are requested up front, before griddepcontrol.wait)
constexpr int kRampStages = VLUT_SLOT_RAMP;
#ifndef VLUT_SLOT_PIECES
#define VLUT_SLOT_PIECES 1
#endif
constexpr int kIdxPieces = VLUT_SLOT_PIECES;  // bulk copies per staged index tile

// The index rows of one K-tile (one contiguous block of the payload) as
// kIdxPieces bulk copies completing on the stage's mbarrier.
__device__ __forceinline__ void stage_idx(uint32_t dst, const uint8_t* src, int bytes,
                                          uint32_t mbar) {
  if (kIdxPieces <= 1) {
    bulk_g2s(dst, src, (uint32_t)bytes, mbar);
    return;
  }
  const int piece = ((bytes + kIdxPieces - 1) / kIdxPieces + 15) & ~15;
  for (int o = 0; o < bytes; o += piece)
    bulk_g2s(dst + o, src + o, (uint32_t)min(piece, bytes - o), mbar);
}
#ifndef VLUT_SLOT_LAST_ONLY_BYTES
#define VLUT_SLOT_LAST_ONLY_BYTES 8192
#endif
constexpr int kLastOnlyBytes = VLUT_SLOT_LAST_ONLY_BYTES;  // split-K tiles up to this size: the last CTA finishes them
#ifndef VLUT_SLOT_BULK_SMALL
constexpr bool kRedRegs = true;   // last-only tiles: partials added by red.add from registers
#else
constexpr bool kRedRegs = false;  // (A/B) bulk reduce-add of the shared tile
#endif
#ifndef VLUT_SLOT_ATOM64
#define VLUT_SLOT_ATOM64 1
#endif
// last-only tiles (decode): every partial element goes out as ONE 64-bit
// atomic add carrying (1 << 40) + (partial + 2^31): bits 40.. count the
// contributions, bits 0..39 hold the biased sum (S <= 255 partials of < 2^32
// each cannot carry into the count).  The thread whose add returns count
// S - 1 holds the tile's last contribution to that element: it forms the sum
// (old + its own, minus S 2^31), runs the epilogue for it and re-zeroes the
// word.  No arrival counter, no CTA barrier, no read-back of the workspace:
// one L2 round trip instead of three (red -> acq_rel arrival -> loads).
constexpr bool kAtom64 = VLUT_SLOT_ATOM64 != 0;
#ifndef VLUT_SLOT_LDG
#define VLUT_SLOT_LDG 1
#endif
// One table word per lookup (NW = 1: decode, N <= 2): every lookup thread
// copies its OWN index rows (16 B per row and K-tile, lane-consecutive rows:
// coalesced) into its slots of the shared ring with cp.async, a whole ring
// (STAGES tiles) at entry -- the weights do not depend on the previous
// kernel -- and one tile per tile consumed, one commit group per tile
// (the thread reads back only what it copied: no CTA-wide handshake).
// Measured (scripts/hbm_floor.cu, 17.7 MB): one bulk-copy ring per SM
// streams it in >= 6.4 us, per-thread loads issued up front in 4.3-5.1 us.
// The producer then stages only the (tiny) activation tiles.
constexpr bool kCpIdxAll = VLUT_SLOT_LDG != 0;
constexpr int kAtom64MaxSplits = 255;
#ifndef VLUT_SLOT_A64_TOK
#define VLUT_SLOT_A64_TOK 2
#endif
// variants with at most this many tokens per CTA meet through the counted
// 64-bit atomics (whatever their tile size); wider ones keep the bulk
// reduce-add + generation handshake
constexpr int kA64MaxTok = VLUT_SLOT_A64_TOK;

#ifndef VLUT_SLOT_RPL_G4
#define VLUT_SLOT_RPL_G4 2
#endif
template <int G, int NW, int TPW>
struct SL {
  static constexpr int R = pow3(G);
  static constexpr int ZERO = (R - 1) / 2;
  static constexpr int RPL = (G == 4) ? VLUT_SLOT_RPL_G4 : 4;  // rows per lookup lane
  static constexpr int MCTA = 32 * kLW * RPL;     // 1024 (g=4) / 2048 (g=5)
  static constexpr int NTOK = NW * TPW;           // tokens per CTA
  static constexpr int NWP = (NW + 1) / 2;        // 256-B row blocks (word pairs)
  // Scalar LUT (TPW = 1) with 4+ words per lookup: half tables (anti-symmetry
  // T[i] = -T[3^g-1-i], positions p = |i - ZERO|, sign applied by a multiply
  // at lookup) halve the build, whose share grows with NW; the per-index
  // decode is shared by the NW words (measured: N = 16 53 -> 48 us).  The
  // SWAR vector words lose more on the lookup path than they save (reverted
  // there, DESIGN.md §4 K2).
  static constexpr bool HALF = (NW >= 4 && TPW == 1);
  static constexpr int ROWS = HALF ? (R + 1) / 2 : R;  // stored table rows
  static constexpr int TAB_BYTES = NWP * ROWS * kRowStride;
  static constexpr int IDX_BYTES = MCTA * 16;
  static constexpr int ACT_BYTES = kKgTile * G * kActNMax;  // one K-tile of A, N <= 64
  static constexpr int FIXED = 2 * TAB_BYTES + 32 + 16 * kMaxStages + 16;
  static constexpr int ST_FIT = (kSmemMax - FIXED) / (IDX_BYTES + ACT_BYTES);
  static constexpr int STAGES = ST_FIT < kMaxStages ? ST_FIT : kMaxStages;
  static constexpr int IDX_OFF = 2 * TAB_BYTES;
  static constexpr int ACT_OFF = IDX_OFF + STAGES * IDX_BYTES;
  static constexpr int MBAR_OFF = ACT_OFF + STAGES * ACT_BYTES;  // FULL[2] EMPTY[2] STG[S] IFREE[S]
  static constexpr int MISC_OFF = MBAR_OFF + 32 + 16 * kMaxStages;
  static constexpr int FUSE_OFF = MISC_OFF + 16;  // fused decode: 16 warp maxima + the scale
  static constexpr int SMEM = FUSE_OFF + 80;
  static constexpr int BIAS = (TPW == 2) ? 128 * G : 0;
  static_assert(TPW == 1 || TPW == 2, "1 or 2 tokens per table word");
  static_assert(STAGES >= 2, "staging ring needs two stages");
  static_assert(SMEM <= kSmemMax, "shared memory budget");
  static_assert(MCTA * NTOK * 4 <= 2 * TAB_BYTES, "int32 tile must fit the table region");
  static_assert(TPW == 1 || kFlushTiles * kKgTile * 2 * BIAS <= 65535, "SWAR field overflow");
};

struct SlotParams {
  const uint8_t* payload;  // packed indices [kt][m_pad][16]
  const int8_t* A;         // [K][N] int8, token axis contiguous
  const float* a_scale;    // [N]
  float w_scale;
  void* out;               // [M][N] fp32, or int32 when acc_only
  int M, K, N;
  int m_pad, kg_tiles;
  int splits;              // CTAs per (M-block, N-tile) along K (grid.x)
  int acc_only;
  int act_tma;             // 1: A is staged by bulk copies (N <= 64, 16-B aligned A)
  int32_t* ws_acc;         // splits > 1: int32 [M][N], all zero between launches
  unsigned* ws_cnt;        // splits > 1: per-tile (arrivals, generation) words; arrivals zero
                           // between launches, generation monotonic
  int last_only;           // splits > 1: 1 = the last CTA to arrive finishes the whole tile
                           // (small tiles), 0 = every CTA finishes 1/S of it
  // fused decode (vlut_mpgemm_decode, N = 1): the fp32 activations [K]; every
  // CTA takes their absmax itself (all of K, from L2 after the first reader),
  // s = amax / 127 (1 if 0), and its builders quantize q = clamp(round(x /
  // s), +-127) -- K3's arithmetic, bit for bit -- so no quantizer launch and
  // no int8 round trip.  A / a_scale unused; scale_out (optional) <- s.
  const float* xq;
  float* scale_out;
  int q_ring;              // fused decode: 1 = codes through shared memory when the CTA's
                           // slice fits the activation ring (0: per-tile global reads)
};

// K3's code (vlut_aux_kernels.cuh q_code): the same IEEE division and rounding
__device__ __forceinline__ int slot_q_code(float v, float s) {
  float r = roundf(__fdiv_rn(v, s));
  r = fminf(fmaxf(r, -127.f), 127.f);
  return (int)r;
}

__device__ __forceinline__ void red_add_s32(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_u64(unsigned long long* p, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;\n" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void bulk_red_add_s32(int32_t* dst, uint32_t src_s, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.s32 [%0], [%1], %2;\n" ::"l"(dst),
               "r"(src_s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// per-thread asynchronous 16-byte global -> shared copy (L1 bypassed)
__device__ __forceinline__ void cp_async16(uint32_t dst_s, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst_s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];\n" : "=r"(v) : "r"(addr));
  return v;
}

// Activation bytes of K-tile kt that the producer stages (rows [k0, k0+16g)
// of A, full N-wide rows, clipped to K and rounded down to 16 B; the rest of
// a ragged last tile is read from global memory by the builders).
__device__ __forceinline__ int act_tile_bytes(const SlotParams& p, int kt, int G) {
  const int k0 = kt * kKgTile * G;
  const int rows = min(kKgTile * G, p.K - k0);
  return (rows * p.N) & ~15;
}

// Builder chain: all entries whose two top trits are fixed by prefix PF
// (d_{G-2} = PF % 3, d_{G-1} = PF / 3), the lower G-2 trits walked along the
// base-3 reflected Gray code from all -1.  T enters as the entry with the
// lower digits at 0.
// Plain C++ stores (not volatile asm) so the compiler interleaves the nine
// independent chains; the mbarrier arrive (asm volatile, memory clobber)
// orders them before the lookups.
template <int G, int PF>
__device__ __forceinline__ void build_chain(uint8_t* row, uint32_t T, const uint32_t (&P)[8],
                                            const uint32_t (&Mn)[8]) {
  constexpr int D = G - 2;
  constexpr int STRIDE = pow3(D);
  constexpr GrayWalk<D> gw{};
  *reinterpret_cast<uint32_t*>(row + (PF * STRIDE) * kRowStride) = T;
#pragma unroll
  for (int s = 1; s < pow3(D); ++s) {
    T += (gw.dir[s] > 0) ? P[gw.digit[s]] : Mn[gw.digit[s]];
    *reinterpret_cast<uint32_t*>(row + (gw.idx[s] + PF * STRIDE) * kRowStride) = T;
  }
}

// Packed per-row activation deltas of one word: TPW = 1 -> (a, -a) as int32;
// TPW = 2 -> two tokens as arithmetic 16-bit fields (a0 + 65536 a1) and its
// negation.  base = BIAS (packed) minus the sum of the lower G-2 rows.
template <int G, int NW, int TPW>
__device__ __forceinline__ void build_word(uint8_t* row_addr, const uint32_t (&U)[G], int bw,
                                           bool split_chains) {
  using L = SL<G, NW, TPW>;
  uint32_t P[8], Mn[8];
  uint32_t base = (uint32_t)L::BIAS * (TPW == 2 ? 0x00010001u : 1u);
#pragma unroll
  for (int r = 0; r < G; ++r) {
    if constexpr (TPW == 1) {
      P[r] = U[r];
      Mn[r] = 0u - U[r];
    } else {
      P[r] = U[r] - 0x00800080u;   // +a as a packed arithmetic delta
      Mn[r] = 0x00800080u - U[r];  // -a
    }
    if (r < G - 2) base += Mn[r];  // lower trits all -1
  }
  const uint32_t c2[3] = {Mn[G - 2], 0u, P[G - 2]};
  const uint32_t c1[3] = {Mn[G - 1], 0u, P[G - 1]};
#define VLUT_CHAIN(PF)                                                  \
  if (!split_chains || ((PF) % kBW) == bw)                              \
    build_chain<G, PF>(row_addr, base + c2[(PF) % 3] + c1[(PF) / 3], P, Mn);
  VLUT_CHAIN(0) VLUT_CHAIN(1) VLUT_CHAIN(2) VLUT_CHAIN(3) VLUT_CHAIN(4)
  VLUT_CHAIN(5) VLUT_CHAIN(6) VLUT_CHAIN(7) VLUT_CHAIN(8)
#undef VLUT_CHAIN
}

// Half table of one scalar word (HALF): position 0 = the zero pattern; block
// Lv = the patterns whose trits above Lv are 0, trit Lv = +1 and lower trits
// free, at positions [(3^Lv+1)/2, (3^(Lv+1)+1)/2) (position = |i - ZERO|),
// each walked along the base-3 reflected Gray code from all-lower-trits -1
// (one add per entry).
template <int G, int Lv>
__device__ __forceinline__ void build_half_block(uint8_t* row, uint32_t S, const uint32_t (&P)[8],
                                                 const uint32_t (&Mn)[8]) {
  if constexpr (Lv < G) {
    constexpr int P0 = (pow3(Lv) + 1) / 2;
    uint32_t T = P[Lv] + S;  // trit Lv = +1, trits below -1 (S = their sum)
    *reinterpret_cast<uint32_t*>(row + P0 * kRowStride) = T;
    if constexpr (Lv > 0) {
      constexpr GrayWalk<Lv> gw{};
#pragma unroll
      for (int s = 1; s < pow3(Lv); ++s) {
        T += (gw.dir[s] > 0) ? P[gw.digit[s]] : Mn[gw.digit[s]];
        *reinterpret_cast<uint32_t*>(row + (P0 + gw.idx[s]) * kRowStride) = T;
      }
    }
    build_half_block<G, Lv + 1>(row, S + Mn[Lv], P, Mn);
  }
}

template <int G>
__device__ __forceinline__ void build_word_half(uint8_t* row_addr, const uint32_t (&U)[G]) {
  uint32_t P[8], Mn[8];
#pragma unroll
  for (int r = 0; r < G; ++r) {
    P[r] = U[r];
    Mn[r] = 0u - U[r];
  }
  *reinterpret_cast<uint32_t*>(row_addr) = 0u;  // the zero pattern
  build_half_block<G, 0>(row_addr, 0u, P, Mn);
}

// One activation value (token n of feature row k) for the builders: staged
// copy when it landed there, else global memory; 0 outside [K) x [N).
__device__ __forceinline__ int act_value(const SlotParams& p, uint32_t act_s, int act_bytes,
                                         int k0, int k, int n) {
  if (k >= p.K || n >= p.N) return 0;
  const int e = (k - k0) * p.N + n;
  if (e < act_bytes) return (int)(int8_t)lds_u8(act_s + e);
  return (int)__ldg(p.A + (size_t)k * p.N + n);
}

// FQ: the fused-decode instantiation (vlut_mpgemm_decode; NW = TPW = 1), a
// separate kernel so the int8-input kernels carry none of its code
template <int G, int NW, int TPW, bool FQ = false>
__global__ void __launch_bounds__(kThreads, 1) vlut_slot_kernel(const __grid_constant__ SlotParams p) {
  using L = SL<G, NW, TPW>;
  static_assert(!FQ || (NW == 1 && TPW == 1), "fused decode: one scalar word");
  constexpr bool kA64 = kAtom64 && L::NTOK <= kA64MaxTok;
  // per-thread copies where the ring is short (g = 5: 2 stages beside the
  // 243-row tables; a bulk stage is refilled only after all 16 lookup warps
  // and both builders released it): config 4 g = 5 N = 1 8.24 -> 7.61 us.
  // With the 8-stage g = 4 ring the bulk copies are as fast or faster
  // (7.54 vs 7.75 us; profiles/r02_decode.txt)
#ifdef VLUT_SLOT_CP_ALL  // (experiment) per-thread copies at every ring depth
  constexpr bool kLdgIdx = kCpIdxAll && NW == 1;
#else
  constexpr bool kLdgIdx = kCpIdxAll && NW == 1 && L::STAGES < 4;
#endif
  constexpr int PF = kLdgIdx ? L::STAGES : 2;  // kLdgIdx: tiles in flight per thread
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int rank = blockIdx.x;
  const int n0 = blockIdx.y * L::NTOK;
  const int m0 = blockIdx.z * L::MCTA;
  const int S = p.splits;
  const int kt0 = (int)(((long long)rank * p.kg_tiles) / S);
  const int kt1 = (int)(((long long)(rank + 1) * p.kg_tiles) / S);
  const int ntiles = kt1 - kt0;
  unsigned g0 = 0;  // split-K generation word before this CTA arrives (tid 0)
  VLUT_STAMP(0);

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = tab_s + L::IDX_OFF;
  const uint32_t act_s = tab_s + L::ACT_OFF;
  const uint32_t mbar = tab_s + L::MBAR_OFF;
  constexpr uint32_t IFREE0 = 32 + 8 * kMaxStages;
  // FULL[b] = mbar + 8b, EMPTY[b] = mbar + 16 + 8b, STG[s] = mbar + 32 + 8s,
  // IFREE[s] = mbar + 32 + 8 kMaxStages + 8s

  if (tid == 0) {
    mbar_init(mbar + 0, kBW);
    mbar_init(mbar + 8, kBW);
    mbar_init(mbar + 16, kLW);
    mbar_init(mbar + 24, kLW);
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(mbar + 32 + 8 * s, 1);
      mbar_init(mbar + IFREE0 + 8 * s, kLdgIdx ? kBW : kLW + kBW);  // ring slot readers
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kLW + kBW) {
    // =========================== producer: index + activation tiles -> ring (a2)
    if (lane == 0 && ntiles > 0) {
      const int rows = min(L::MCTA, p.m_pad - m0);
      // (1) the packed weights are not an output of the previous kernel
      // (vlut.h): the index rows of the first ring-full of tiles are
      // requested before griddepcontrol.wait, so at decode (HBM-bound) the
      // weight stream overlaps the previous kernel's tail
      const int pre = min(ntiles, kRampStages > 0 ? min(kRampStages, L::STAGES) : L::STAGES);
#pragma unroll 1
      for (int t = 0; t < pre; ++t) {
        const int kt = kt0 + t;
        const int ab = p.act_tma ? act_tile_bytes(p, kt, G) : 0;
        const uint32_t stg = mbar + 32 + 8 * t;
        mbar_expect_tx(stg, (uint32_t)((kLdgIdx ? 0 : rows * 16) + ab));
        if (!kLdgIdx)
          stage_idx(idx_s + (uint32_t)(t * L::IDX_BYTES), p.payload + ((size_t)kt * p.m_pad + m0) * 16,
                    rows * 16, stg);
      }
      // (2) activations come from the previous kernel (quantizer)
      pdl_wait();
#pragma unroll 1
      for (int t = 0; t < pre; ++t) {
        const int kt = kt0 + t;
        const int ab = p.act_tma ? act_tile_bytes(p, kt, G) : 0;
        if (ab > 0)
          bulk_g2s(act_s + (uint32_t)(t * L::ACT_BYTES), p.A + (size_t)kt * kKgTile * G * p.N,
                   (uint32_t)ab, mbar + 32 + 8 * t);
      }
      // (3) the rest through the ring as stages free up
#pragma unroll 1
      for (int t = pre; t < ntiles; ++t) {
        const int st = t % L::STAGES, use = t / L::STAGES;
        const int kt = kt0 + t;
        if (use > 0) mbar_wait(mbar + IFREE0 + 8 * st, (use - 1) & 1);
        // ramp (kRampStages > 0): only that many stages per CTA in flight
        // until the first tile lands
        if (kRampStages > 0 && t == kRampStages) mbar_wait(mbar + 32, 0);
        const int ab = p.act_tma ? act_tile_bytes(p, kt, G) : 0;
        const uint32_t stg = mbar + 32 + 8 * st;
        mbar_expect_tx(stg, (uint32_t)((kLdgIdx ? 0 : rows * 16) + ab));
        if (!kLdgIdx)
          stage_idx(idx_s + (uint32_t)(st * L::IDX_BYTES), p.payload + ((size_t)kt * p.m_pad + m0) * 16,
                    rows * 16, stg);
        if (ab > 0)
          bulk_g2s(act_s + (uint32_t)(st * L::ACT_BYTES), p.A + (size_t)kt * kKgTile * G * p.N,
                   (uint32_t)ab, stg);
      }
    }
  } else if (warp >= kLW) {
    // =========================== builders: full tables (a3)
    const int bw = warp - kLW;
    const int j = lane & 15;
    pdl_wait();  // the global-memory tail of A comes from the previous kernel
    float xs = 1.f;  // fused decode: the token's scale, from the lookup warps
    if constexpr (FQ) {
      bar_sync(2, (kLW + kBW) * 32);
      xs = *reinterpret_cast<const float*>(smem + L::FUSE_OFF + 64);
    }
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1, st = t % L::STAGES;
      const int kt = kt0 + t;
      const int k0 = kt * kKgTile * G;
      if (t >= 2) mbar_wait(mbar + 16 + 8 * b, ((t >> 1) - 1) & 1);  // lookups of t-2 done
      mbar_wait(mbar + 32 + 8 * st, (t / L::STAGES) & 1);             // tile t staged
      const int ab = p.act_tma ? act_tile_bytes(p, kt, G) : 0;
      const uint32_t as = act_s + (uint32_t)(st * L::ACT_BYTES);
      // activations of this lane's group j for every word it builds
      constexpr int WPB = (NW + kBW - 1) / kBW;
      uint32_t U[WPB][G];
      if (ab == kKgTile * G * p.N && p.N % L::NTOK == 0) {
        // fast path: the whole tile is staged and the CTA's NTOK tokens of a
        // row are one aligned NTOK-byte vector -> one shared load per row
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const uint32_t addr = as + (uint32_t)((j * G + r) * p.N + n0);
          uint32_t by[4] = {0u, 0u, 0u, 0u};
          if constexpr (L::NTOK == 16) {
            const uint4 q4 = *reinterpret_cast<const uint4*>(smem + (addr - tab_s));
            by[0] = q4.x; by[1] = q4.y; by[2] = q4.z; by[3] = q4.w;
          } else if constexpr (L::NTOK == 8) {
            const uint2 q2 = *reinterpret_cast<const uint2*>(smem + (addr - tab_s));
            by[0] = q2.x; by[1] = q2.y;
          } else if constexpr (L::NTOK == 4) {
            by[0] = *reinterpret_cast<const uint32_t*>(smem + (addr - tab_s));
          } else if constexpr (L::NTOK == 2) {
            by[0] = *reinterpret_cast<const uint16_t*>(smem + (addr - tab_s));
          } else {
            by[0] = *(smem + (addr - tab_s));
          }
#pragma unroll
          for (int wi = 0; wi < WPB; ++wi) {
            const int w = (NW == 1) ? 0 : bw + wi * kBW;
            const int t0 = (w * TPW) & 15;  // token of the word's first field (w < NW)
            const uint32_t src = by[(t0 >> 2) & 3];
            if constexpr (TPW == 1) {
              U[wi][r] = (uint32_t)(int32_t)(int8_t)(src >> (8 * (t0 & 3)));
            } else {
              // bytes t0, t0+1 (same word: t0 even) -> (a + 128) in 16-bit fields
              // selector nibbles (b, zero, b+1, zero), b = t0 & 3
              const uint32_t sel = 0x4140u + ((uint32_t)(t0 & 3) * 0x0101u);
              U[wi][r] = __byte_perm(src ^ 0x80808080u, 0u, sel);
            }
          }
        }
      } else {
#pragma unroll
        for (int wi = 0; wi < WPB; ++wi) {
          const int w = (NW == 1) ? 0 : bw + wi * kBW;
#pragma unroll
          for (int r = 0; r < G; ++r) {
            const int k = k0 + j * G + r;
            if constexpr (TPW == 1) {
              if constexpr (FQ) {  // fused decode (N = 1): the code the lookup warps stored, or now
                U[wi][r] = (p.q_ring && ntiles * kKgTile * G <= L::STAGES * L::ACT_BYTES)
                               ? (uint32_t)(int32_t)reinterpret_cast<const int8_t*>(
                                     smem + L::ACT_OFF)[t * kKgTile * G + j * G + r]
                               : (uint32_t)(k < p.K ? slot_q_code(__ldg(p.xq + k), xs) : 0);
              } else {
                U[wi][r] = (uint32_t)act_value(p, as, ab, k0, k, n0 + w);
              }
            } else {
              const int nn = n0 + 2 * w;
              U[wi][r] = (uint32_t)(act_value(p, as, ab, k0, k, nn) + 128) |
                         ((uint32_t)(act_value(p, as, ab, k0, k, nn + 1) + 128) << 16);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + IFREE0 + 8 * st);  // done with the ring slot's A rows
#pragma unroll
      for (int wi = 0; wi < WPB; ++wi) {
        const int w = (NW == 1) ? 0 : bw + wi * kBW;
        if (w < NW) {
          uint8_t* row = smem + b * L::TAB_BYTES + (w >> 1) * L::ROWS * kRowStride + (w & 1) * 128 +
                         4 * lane;
          if constexpr (L::HALF) build_word_half<G>(row, U[wi]);
          else build_word<G, NW, TPW>(row, U[wi], bw, NW == 1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + 8 * b);  // table t ready
    }
  } else {
    // =========================== lookup warps (a4)
    // per-(row, word, token-in-word) int32 results
    int32_t acc[L::RPL][NW][TPW];
#pragma unroll
    for (int q = 0; q < L::RPL; ++q)
#pragma unroll
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int e = 0; e < TPW; ++e) acc[q][w][e] = 0;
    const int x = lane & 15;
    const int qk = x >> 2;
    uint32_t selv[4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
      selv[b] = L::HALF ? (0x4440u | (uint32_t)(b ^ (x & 3)))  // index byte -> bits 0..7
                        : (0x5504u | ((uint32_t)(b ^ (x & 3)) << 4));
    uint32_t sw[L::RPL][NW];
#pragma unroll
    for (int q = 0; q < L::RPL; ++q)
#pragma unroll
      for (int w = 0; w < NW; ++w) sw[q][w] = 0;
    int since_flush = 0;
    // kLdgIdx: this thread's index rows of tile t -> its slots of ring stage
    // t % STAGES (cp.async, one commit group per tile, empty past the end)
    auto cp_tile = [&](int t) {
      if (t < ntiles) {
        const int st = t % L::STAGES;
#pragma unroll
        for (int q = 0; q < L::RPL; ++q) {
          const int r = q * kLookupThreads + warp * 32 + lane;
          if (m0 + q * kLookupThreads + warp * 32 < p.m_pad)
            cp_async16(idx_s + (uint32_t)(st * L::IDX_BYTES + r * 16),
                       p.payload + ((size_t)(kt0 + t) * p.m_pad + m0 + r) * 16);
        }
      }
      cp_async_commit();
    };
    // ramp: tiles 0 and 1 at entry; the rest of the ring once tile 0 has
    // landed (the first tile is not queued behind a whole ring of requests)
    if constexpr (kLdgIdx) {
      cp_tile(0);
      cp_tile(1);
    }
    if constexpr (FQ) {
      // fused decode: the token's absmax over all K (the weight stream is
      // already in flight), s = amax / 127, handed to the builders
      pdl_wait();  // x may be the previous kernel's output
      float mx = 0.f;
      // every load of a round issued before any use (one L2 round trip per
      // round, not per load: 12 x 16 B per thread covers K = 24576)
      constexpr int QU = 12;
      if ((p.K & 3) == 0 && (((uintptr_t)p.xq) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(p.xq);
        const int n4 = p.K / 4;
        for (int i0 = tid; i0 < n4; i0 += QU * kLookupThreads) {
          float4 a[QU];
#pragma unroll
          for (int u = 0; u < QU; ++u) {
            const int i = i0 + u * kLookupThreads;
            a[u] = i < n4 ? __ldg(x4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < QU; ++u)
            mx = fmaxf(fmaxf(mx, fabsf(a[u].x)),
                       fmaxf(fabsf(a[u].y), fmaxf(fabsf(a[u].z), fabsf(a[u].w))));
        }
      } else {
        for (int i0 = tid; i0 < p.K; i0 += QU * kLookupThreads) {
          float a[QU];
#pragma unroll
          for (int u = 0; u < QU; ++u) {
            const int i = i0 + u * kLookupThreads;
            a[u] = i < p.K ? __ldg(p.xq + i) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < QU; ++u) mx = fmaxf(mx, fabsf(a[u]));
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
      float* red = reinterpret_cast<float*>(smem + L::FUSE_OFF);
      if (lane == 0) red[warp] = mx;
      bar_sync(1, kLookupThreads);
      float a = red[0];
#pragma unroll
      for (int w = 1; w < kLW; ++w) a = fmaxf(a, red[w]);
      const float sc = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
      if (tid == 0) {
        red[16] = sc;
        if (p.scale_out && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) *p.scale_out = sc;
      }
      // this CTA's K slice quantized into the (otherwise unused) activation
      // ring, so the builders read codes from shared memory instead of
      // paying a global-memory round trip per K-tile
      const int nq = ntiles * kKgTile * G;
      if (p.q_ring && nq <= L::STAGES * L::ACT_BYTES) {
        int8_t* qs = reinterpret_cast<int8_t*>(smem + L::ACT_OFF);
        const int kb = kt0 * kKgTile * G;
        for (int e0 = tid; e0 < nq; e0 += QU * kLookupThreads) {
          float xv[QU];
#pragma unroll
          for (int u = 0; u < QU; ++u) {
            const int k = kb + e0 + u * kLookupThreads;
            xv[u] = (e0 + u * kLookupThreads < nq && k < p.K) ? __ldg(p.xq + k) : 0.f;
          }
#pragma unroll
          for (int u = 0; u < QU; ++u)
            if (e0 + u * kLookupThreads < nq) qs[e0 + u * kLookupThreads] = (int8_t)slot_q_code(xv[u], sc);
        }
      }
      bar_sync(2, (kLW + kBW) * 32);  // the builders wait here for red[16] and the codes
    }
    // one K-tile with table buffer B (compile time: the buffer offset folds
    // into the LDS immediate, one PRMT forms the rest of each address)
    auto tile = [&](auto Bc, int t) {
      constexpr int B = decltype(Bc)::value;
      uint4 v[L::RPL];
      if constexpr (kLdgIdx) {
        // this thread's rows of tile t have landed (groups younger than t's:
        // tile 0 -> tile 1's; later tiles -> PF - 1 of them)
        if (t == 0) {
          cp_async_wait<1>();
        } else {
          cp_async_wait<PF - 1>();
        }
        const int st = t % L::STAGES;
        if (t == 0) VLUT_STAMP(1);
        if (t == ntiles - 1) VLUT_STAMP(7);
#pragma unroll
        for (int q = 0; q < L::RPL; ++q) {
          const int r = q * kLookupThreads + warp * 32 + lane;
          v[q] = (m0 + q * kLookupThreads + warp * 32 < p.m_pad)
                     ? *reinterpret_cast<const uint4*>(smem + L::IDX_OFF + st * L::IDX_BYTES + r * 16)
                     : make_uint4(0, 0, 0, 0);
        }
        if (t == 0) {  // end of the ramp: the ring's other free slots (2 .. PF-1)
#pragma unroll 1
          for (int j = 2; j < PF; ++j) cp_tile(j);
        }
      } else {
        const int st = t % L::STAGES;
        mbar_wait(mbar + 32 + 8 * st, (t / L::STAGES) & 1);  // index rows landed
        if (t == 0) VLUT_STAMP(1);
        if (t == ntiles - 1) VLUT_STAMP(7);
#pragma unroll
        for (int q = 0; q < L::RPL; ++q) {
          const int r = q * kLookupThreads + warp * 32 + lane;
          v[q] = (m0 + q * kLookupThreads + warp * 32 < p.m_pad)
                     ? *reinterpret_cast<const uint4*>(smem + L::IDX_OFF + st * L::IDX_BYTES + r * 16)
                     : make_uint4(0, 0, 0, 0);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar + IFREE0 + 8 * st);  // ring slot's index rows consumed
      }
      mbar_wait(mbar + 8 * B, (t >> 1) & 1);           // table t built
      if (t == 0) VLUT_STAMP(2);
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        if (m0 + q * kLookupThreads + warp * 32 >= p.m_pad) continue;  // warp-uniform
        // Wp[c] = v[c ^ qk]: the word holding group (4c + k) ^ x
        const uint32_t t0 = (qk & 1) ? v[q].y : v[q].x;
        const uint32_t t1 = (qk & 1) ? v[q].x : v[q].y;
        const uint32_t t2 = (qk & 1) ? v[q].w : v[q].z;
        const uint32_t t3 = (qk & 1) ? v[q].z : v[q].w;
        const uint32_t Wp[4] = {(qk & 2) ? t2 : t0, (qk & 2) ? t3 : t1, (qk & 2) ? t0 : t2,
                                (qk & 2) ? t1 : t3};
#pragma unroll
        for (int s = 0; s < kKgTile; ++s) {
          // byte (s & 3) ^ (x & 3) of Wp[s >> 2] -> bits 8..15, slot offset
          // (4 lane) ^ (4 s) -> bits 0..7: the entry's offset i * 256 + 4 slot
          uint32_t off;
          int32_t sg = 1;
          if constexpr (L::HALF) {
            // position |i - ZERO| -> bits 8.., slot -> bits 0..7; sign +-1
            const int d = (int)__byte_perm(Wp[s >> 2], 0u, selv[s & 3]) - L::ZERO;
            const int m = d >> 31;
            sg = m | 1;
            off = ((uint32_t)((d ^ m) - m) << 8) | (uint32_t)((4 * lane) ^ (4 * s));
          } else {
            off = __byte_perm(Wp[s >> 2], (uint32_t)((4 * lane) ^ (4 * s)), selv[s & 3]);
          }
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint32_t val = *reinterpret_cast<const uint32_t*>(
                smem + (B * L::TAB_BYTES + (w >> 1) * L::ROWS * kRowStride + (w & 1) * 128) + off);
            if constexpr (TPW == 1) acc[q][w][0] += L::HALF ? (int32_t)val * sg : (int32_t)val;
            else sw[q][w] += val;
          }
        }
      }
      if constexpr (kLdgIdx) cp_tile(t + PF);  // refill the slot just read
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + 16 + 8 * B);  // table buffer B free
      if constexpr (TPW == 2) {
        if (++since_flush >= kFlushTiles || t + 1 == ntiles) {
          since_flush = 0;
#pragma unroll
          for (int q = 0; q < L::RPL; ++q)
#pragma unroll
            for (int w = 0; w < NW; ++w) {
              acc[q][w][0] += (int32_t)(sw[q][w] & 0xFFFFu);
              acc[q][w][1] += (int32_t)(sw[q][w] >> 16);
              sw[q][w] = 0;
            }
        }
      }
    };
#pragma unroll 1
    for (int t = 0; t < ntiles; t += 2) {
      tile(std::integral_constant<int, 0>{}, t);
      if (t + 1 < ntiles) tile(std::integral_constant<int, 1>{}, t + 1);
    }
    if constexpr (TPW == 2) {
      const int32_t bias_total = L::BIAS * kKgTile * ntiles;
#pragma unroll
      for (int q = 0; q < L::RPL; ++q)
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          acc[q][w][0] -= bias_total;
          acc[q][w][1] -= bias_total;
        }
    }
    VLUT_STAMP(3);
    // int32 tile -> shared memory [row][token] (the table region: every
    // lookup warp is past its last table read after this barrier)
    bar_sync(1, kLookupThreads);
    // dense [row][ld] with ld = min(N, NTOK): for N <= NTOK the CTA's rows are
    // one contiguous block of the [M][N] output / workspace
    int32_t* tile_s = reinterpret_cast<int32_t*>(smem);
    const int ld = min(p.N, L::NTOK);
#pragma unroll
    for (int q = 0; q < L::RPL; ++q) {
      if ((kRedRegs || kA64) && S > 1 && p.last_only) break;  // partials go out from registers below
      const int r = q * kLookupThreads + warp * 32 + lane;
      if constexpr (L::NTOK >= 4) {
        if (ld == L::NTOK) {  // 16-byte vector stores
          constexpr int NCH = L::NTOK / 4;
          int4 ch[NCH];
#pragma unroll
          for (int c = 0; c < NCH; ++c) {
            const int t0 = 4 * c;
            ch[c] = make_int4(acc[q][t0 / TPW][t0 % TPW], acc[q][(t0 + 1) / TPW][(t0 + 1) % TPW],
                              acc[q][(t0 + 2) / TPW][(t0 + 2) % TPW],
                              acc[q][(t0 + 3) / TPW][(t0 + 3) % TPW]);
          }
          if constexpr (NCH == 4) {
            // 64-byte rows: lanes l and l+2 share banks; writing chunk
            // (c + lane) & 3 in step c halves the conflicts (16- -> 8-way)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int cc = (c + lane) & 3;
              const int4 a = (cc & 1) ? ch[1] : ch[0];
              const int4 b = (cc & 1) ? ch[3] : ch[2];
              *reinterpret_cast<int4*>(tile_s + r * L::NTOK + 4 * cc) = (cc & 2) ? b : a;
            }
          } else {
#pragma unroll
            for (int c = 0; c < NCH; ++c)
              *reinterpret_cast<int4*>(tile_s + r * L::NTOK + 4 * c) = ch[c];
          }
          continue;
        }
      }
#pragma unroll
      for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int e = 0; e < TPW; ++e)
          if (w * TPW + e < ld) tile_s[r * ld + w * TPW + e] = acc[q][w][e];
    }
    fence_proxy_async_smem();  // the tile is read by bulk-reduce copies
    pdl_wait();  // epilogue reads a_scale / the workspace of the previous kernel
    if (kA64 && S > 1 && p.last_only) {
      // small split-K tiles (decode), counted 64-bit atomics (kAtom64 above):
      // all of the thread's adds first (their round trips overlap), then the
      // elements it completed
      unsigned long long* ws64 = reinterpret_cast<unsigned long long*>(p.ws_acc);
      const int ntok_v = min(L::NTOK, p.N - n0);
      unsigned long long old[L::RPL][NW][TPW];
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        const int m = m0 + q * kLookupThreads + warp * 32 + lane;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int e = 0; e < TPW; ++e) {
            old[q][w][e] = 0;
            if (m < p.M && w * TPW + e < ntok_v)
              old[q][w][e] = atom_add_u64(ws64 + (size_t)m * p.N + n0 + w * TPW + e,
                                          (1ull << 40) + (unsigned long long)((uint32_t)acc[q][w][e] ^ 0x80000000u));
          }
      }
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        const int m = m0 + q * kLookupThreads + warp * 32 + lane;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int e = 0; e < TPW; ++e) {
            const int c = w * TPW + e;
            if (m < p.M && c < ntok_v && (unsigned)(old[q][w][e] >> 40) == (unsigned)(S - 1)) {
              const unsigned long long low = (old[q][w][e] & ((1ull << 40) - 1)) +
                                             (unsigned long long)((uint32_t)acc[q][w][e] ^ 0x80000000u);
              const int32_t a = (int32_t)(uint32_t)(low - (unsigned long long)S * 0x80000000ull);
              const size_t o = (size_t)m * p.N + n0 + c;
              ws64[o] = 0ull;  // zero-kept for the next launch (after its griddepcontrol.wait)
              if (p.acc_only) {
                reinterpret_cast<int32_t*>(p.out)[o] = a;
              } else {
                const float sc = __fmul_rn(FQ ? *reinterpret_cast<const float*>(smem + L::FUSE_OFF + 64)
                                                : __ldg(p.a_scale + n0 + c), p.w_scale);
                reinterpret_cast<float*>(p.out)[o] = __fmul_rn((float)a, sc);
              }
            }
          }
      }
    } else if (kRedRegs && S > 1 && p.last_only) {
      // small split-K tiles (decode): each thread adds its partial rows
      // straight from registers into the zero-kept workspace (red.add, no
      // shared tile and no bulk copy to wait for); the arrival below -- a CTA
      // barrier, then thread 0's acq_rel atomic, whose release is cumulative
      // over the barrier -- orders them before the last CTA's reads
      const int ntok_v = min(L::NTOK, p.N - n0);
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        const int m = m0 + q * kLookupThreads + warp * 32 + lane;
        if (m >= p.M) continue;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int e = 0; e < TPW; ++e)
            if (w * TPW + e < ntok_v)
              red_add_s32(p.ws_acc + (size_t)m * p.N + n0 + w * TPW + e, acc[q][w][e]);
      }
    }
    // the tile's generation before this CTA arrives (it cannot move before
    // then; read after pdl_wait so a previous launch's bump is visible)
    if (tid == 0 && S > 1 && !p.last_only)
      g0 = ld_relaxed_gpu(p.ws_cnt + 2 * (blockIdx.z * gridDim.y + blockIdx.y) + 1);
  }
  pdl_launch_dependents();
  if (kA64 && S > 1 && p.last_only) {  // finished element by element above
    VLUT_STAMP(5);  // (thread 0: its own elements done)
    return;
  }
  __syncthreads();  // int32 tile complete
  VLUT_STAMP(4);

  // =========================== split-K reduction + epilogue (a5, a6)
  const int rows_valid = min(L::MCTA, p.M - m0);
  const int ntok_valid = min(L::NTOK, p.N - n0);
  const int ld = min(p.N, L::NTOK);
  const int elems = rows_valid * ntok_valid;
  const int32_t* tile_c = reinterpret_cast<const int32_t*>(smem);
  int e_begin = 0, e_end = elems;  // the slice of (row, token) elements this CTA finishes
  if (S > 1) {
    // (1) partial -> zero-kept workspace: one bulk reduce-add when the CTA's
    // rows are contiguous there (N <= NTOK), one per row when rows are >= 64 B
    const bool red_done = kRedRegs && p.last_only;  // added from registers above
    const bool contig = !red_done && (p.N <= L::NTOK) && ((elems & 3) == 0);
    const bool rowwise = !red_done && !contig && (p.N > L::NTOK) && (ntok_valid >= 16) &&
                         ((ntok_valid & 3) == 0) && ((p.N & 3) == 0);
    if (contig) {
      if (tid == 0) {
        bulk_red_add_s32(p.ws_acc + (size_t)m0 * p.N, tab_s, (uint32_t)(elems * 4));
        bulk_commit_wait_all();
      }
    } else if (rowwise) {
      if (warp < kLW) {
        for (int r = tid; r < rows_valid; r += kLookupThreads)
          bulk_red_add_s32(p.ws_acc + (size_t)(m0 + r) * p.N + n0, tab_s + (uint32_t)(r * ld * 4),
                           (uint32_t)(ntok_valid * 4));
        bulk_commit_wait_all();
      }
    } else if (!red_done && warp < kLW) {
#pragma unroll 4
      for (int e = tid; e < elems; e += kLookupThreads) {
        const int r = e / ntok_valid, c = e - r * ntok_valid;
        red_add_s32(p.ws_acc + (size_t)(m0 + r) * p.N + n0 + c, tile_c[r * ld + c]);
      }
    }
    fence_proxy_async_global();
    __syncthreads();
    // (2) arrive (the release of the acq_rel add covers this CTA's reductions:
    // completed, and ordered before it by the proxy fence).  The last CTA of
    // the tile to arrive re-arms the count.  last_only (small tiles): that CTA
    // alone goes on and finishes the whole tile, the others exit -- no
    // waiting.  Otherwise it also bumps the tile's generation word (release)
    // and every CTA (co-resident: cooperative launch) waits for that and
    // finishes 1/S of the tile.  Bounded spin: a schedule bug must fail
    // loudly, never hang.
    unsigned* cnt = p.ws_cnt + 2 * (blockIdx.z * gridDim.y + blockIdx.y);
    __shared__ int s_last;
    if (tid == 0) {
      const bool last = atom_add_acq_rel(cnt, 1u) == (unsigned)(S - 1);
      if (last) {
        cnt[0] = 0u;  // all S arrivals are in: re-arm for the next launch
        if (!p.last_only) st_release_gpu(cnt + 1, g0 + 1u);  // ordered after the reset
      } else if (!p.last_only) {
        unsigned spins = 0;
        while (ld_acquire_gpu(cnt + 1) == g0) {
          __nanosleep(32);
          if (++spins > (1u << 26)) __trap();
        }
      }
      s_last = last ? 1 : 0;
    }
    __syncthreads();
    VLUT_STAMP(5);
    // (3) this CTA finishes elements [e_begin, e_end) of the tile
    if (p.last_only) {
      if (!s_last) return;
    } else {
      e_begin = (int)(((long long)elems * rank) / S);
      e_end = (int)(((long long)elems * (rank + 1)) / S);
    }
  }
  if (warp < kLW) {
    // batches of EB elements per thread: every workspace load of a batch is
    // issued before its stores (out / ws may alias as far as the compiler
    // knows, so a fused load-store loop would serialise the L2 round trips)
    constexpr int EB = 8;
    for (int e0 = e_begin + tid; e0 < e_end; e0 += EB * kLookupThreads) {
      int32_t a[EB];
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        const int e = e0 + b * kLookupThreads;
        a[b] = 0;
        if (e < e_end) {
          const int r = e / ntok_valid, c = e - r * ntok_valid;
          if (S > 1) a[b] = __ldcg(p.ws_acc + (size_t)(m0 + r) * p.N + n0 + c);
          else a[b] = tile_c[r * ld + c];
        }
      }
#pragma unroll
      for (int b = 0; b < EB; ++b) {
        const int e = e0 + b * kLookupThreads;
        if (e >= e_end) break;
        const int r = e / ntok_valid, c = e - r * ntok_valid;
        const size_t o = (size_t)(m0 + r) * p.N + n0 + c;
        if (S > 1) __stcg(p.ws_acc + o, 0);  // keep the workspace zero for the next launch
        if (p.acc_only) {
          reinterpret_cast<int32_t*>(p.out)[o] = a[b];
        } else {
          const float sc = __fmul_rn(FQ ? *reinterpret_cast<const float*>(smem + L::FUSE_OFF + 64)
                                                : __ldg(p.a_scale + n0 + c), p.w_scale);
          reinterpret_cast<float*>(p.out)[o] = __fmul_rn((float)a[b], sc);
        }
      }
    }
  }
  VLUT_STAMP(6);
}

}  // namespace slot
}  // namespace vlut
