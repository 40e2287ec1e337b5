// vlut_kernel_slot.cuh -- K2: lane-slot LUT mpGeMM for small token counts
// (decode, N = 1 .. ~64) and the scalar-LUT (1->1) comparator (f4).
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
//                 hold.  One LDS.32 per lookup and word.
//   words         TPW = 1: a word is ONE token's int32 entry -> the scalar LUT
//                 of T-MAC (each token its own table, N lookups per index,
//                 P:84-85).  TPW = 2: a word packs two tokens as
//                 biased 16-bit fields (field = T + 128 g, as K1) -> a 1->2
//                 vector lookup (the Vec-LUT paradigm) at 2 B of
//                 shared memory per lookup-add, K1's roofline.
//   build (a3)    builder lanes own a slot: lane l computes ALL 3^g entries of
//                 group l & 15 along the base-3 reflected Gray code (one add
//                 per entry, the topological order of P:503-513) and stores
//                 one 128-byte wavefront per entry and word.  Full tables (no
//                 sign decode on the lookup path).
//   index tiles   a producer warp streams each K-tile's 16-byte index rows of
//                 the CTA (one contiguous block of the packed payload) into a
//                 3-4 stage ring with cp.async.bulk + mbarriers, so HBM stays
//                 busy at N = 1 where the kernel is bandwidth-bound.
//   accumulate    TPW = 1: int32 registers.  TPW = 2: SWAR fields widened into
//                 int32 registers every 48 groups (INT16 -> INT32).
//   split-K (a5)  CTAs of one (M-block, N-tile) split its K-tiles; with S > 1
//                 their int32 partials meet in a zero-kept workspace through
//                 red.global.add, and the last CTA to arrive (acq_rel counter)
//                 applies the epilogue, then re-zeroes the workspace and the
//                 counter.  Integer addition is associative: bit-exact for
//                 every split.
//   epilogue (a6) out = fl((float)acc * fl(a_scale[n] * w_scale)), or raw int32.
//
// Citations: P:n = /root/reference/PAPER.md line n.  DESIGN.md §4 (K2) gives
// the byte/instruction budget and the rooflines (HBM at N = 1, shared memory
// otherwise).
#pragma once
#include <type_traits>

#include "vlut_kernel.cuh"

namespace vlut {
namespace slot {

constexpr int kLW = 16;                           // lookup warps
constexpr int kBW = 2;                            // builder warps
constexpr int kThreads = (kLW + kBW + 1) * 32;    // + 1 producer warp = 608
constexpr int kRowStride = 256;                   // bytes per table index row
constexpr int kSmemMax = 232448;                  // 227 KB opt-in per CTA
constexpr int kFlushTiles = 3;                    // TPW = 2: widen every 48 groups
constexpr int kMaxCounters = 16384;               // split-K tile counters in the workspace

template <int G, int NW, int TPW>
struct SL {
  static constexpr int R = pow3(G);
  static constexpr int ZERO = (R - 1) / 2;
  static constexpr int RPL = (G == 4) ? 2 : 4;    // rows per lookup lane
  static constexpr int MCTA = 32 * kLW * RPL;     // 1024 (g=4) / 2048 (g=5)
  static constexpr int NTOK = NW * TPW;           // tokens per CTA
  static constexpr int NWP = (NW + 1) / 2;        // 256-B row blocks (word pairs)
  static constexpr int TAB_BYTES = NWP * R * kRowStride;
  static constexpr int IDX_BYTES = MCTA * 16;
  static constexpr int FIXED = 2 * TAB_BYTES + 1024;
  static constexpr int ST_FIT = (kSmemMax - FIXED) / IDX_BYTES;
  static constexpr int STAGES = ST_FIT < 4 ? ST_FIT : 4;
  static constexpr int IDX_OFF = 2 * TAB_BYTES;
  static constexpr int MBAR_OFF = IDX_OFF + STAGES * IDX_BYTES;  // FULL[2] EMPTY[2] STG[4] IFREE[4]
  static constexpr int MISC_OFF = MBAR_OFF + 96;
  static constexpr int SMEM = MISC_OFF + 16;
  static constexpr int BIAS = (TPW == 2) ? 128 * G : 0;
  static constexpr int WPB = (NW + kBW - 1) / kBW;  // words per builder warp
  static_assert(TPW == 1 || TPW == 2, "1 or 2 tokens per table word");
  static_assert(STAGES >= 2, "index ring needs two stages");
  static_assert(SMEM <= kSmemMax, "shared memory budget");
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
  int32_t* ws_acc;         // splits > 1: int32 [M][N], all zero between launches
  unsigned* ws_cnt;        // splits > 1: per-tile arrival counters, zero between launches
};

__device__ __forceinline__ void red_add_s32(int32_t* p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Gray walk over all 3^G entries from entry 0 (all trits -1) with packed
// deltas P[r] (+a_r) / Mn[r] (-a_r); entry i stored at row_addr + i * 256.
template <int G>
__device__ __forceinline__ void walk_full(uint32_t row_addr, uint32_t T, const uint32_t (&P)[8],
                                          const uint32_t (&Mn)[8]) {
  constexpr GrayWalk<G> gw{};
#pragma unroll
  for (int s = 1; s < pow3(G); ++s) {
    T += (gw.dir[s] > 0) ? P[gw.digit[s]] : Mn[gw.digit[s]];
    sts32(row_addr + gw.idx[s] * kRowStride, T);
  }
}

// Activation values a builder lane needs for one K-tile: group j of the tile,
// rows r < G, tokens of its words.  Packed per (word, row): TPW = 1 -> the
// int8 value as int32; TPW = 2 -> (a0 + 128) | (a1 + 128) << 16.
template <int G, int NW, int TPW>
__device__ __forceinline__ void load_act(const SlotParams& p, int kt, int j, int n0, int bw,
                                         uint32_t (&U)[SL<G, NW, TPW>::WPB][G]) {
  using L = SL<G, NW, TPW>;
#pragma unroll
  for (int wi = 0; wi < L::WPB; ++wi) {
    const int w = bw + wi * kBW;
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const int k = (kt * kKgTile + j) * G + r;
      uint32_t u = 0;
      if (w < NW && k < p.K) {
        const int8_t* row = p.A + (size_t)k * p.N;
        if constexpr (TPW == 1) {
          const int n = n0 + w;
          u = (n < p.N) ? (uint32_t)(int32_t)__ldg(row + n) : 0u;
        } else {
          const int n = n0 + 2 * w;
          const uint32_t a0 = (n < p.N) ? (uint32_t)((int)__ldg(row + n) + 128) : 128u;
          const uint32_t a1 = (n + 1 < p.N) ? (uint32_t)((int)__ldg(row + n + 1) + 128) : 128u;
          u = a0 | (a1 << 16);
        }
      } else if constexpr (TPW == 2) {
        u = 128u | (128u << 16);
      }
      U[wi][r] = u;
    }
  }
}

template <int G, int NW, int TPW>
__global__ void __launch_bounds__(kThreads, 1) vlut_slot_kernel(const __grid_constant__ SlotParams p) {
  using L = SL<G, NW, TPW>;
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

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = tab_s + L::IDX_OFF;
  const uint32_t mbar = tab_s + L::MBAR_OFF;
  // FULL[b] = mbar + 8b, EMPTY[b] = mbar + 16 + 8b, STG[s] = mbar + 32 + 8s, IFREE[s] = mbar + 64 + 8s
  volatile unsigned* last_flag = reinterpret_cast<volatile unsigned*>(smem + L::MISC_OFF);

  if (tid == 0) {
    mbar_init(mbar + 0, kBW);
    mbar_init(mbar + 8, kBW);
    mbar_init(mbar + 16, kLW);
    mbar_init(mbar + 24, kLW);
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(mbar + 32 + 8 * s, 1);
      mbar_init(mbar + 64 + 8 * s, kLW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // per-(row, word, token-in-word) int32 results of the lookup lanes
  int32_t acc[L::RPL][NW][TPW];
#pragma unroll
  for (int q = 0; q < L::RPL; ++q)
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int e = 0; e < TPW; ++e) acc[q][w][e] = 0;

  if (warp == kLW + kBW) {
    // =========================== producer: index tiles -> ring (a2)
    if (lane == 0 && ntiles > 0) {
      const int rows = min(L::MCTA, p.m_pad - m0);
#pragma unroll 1
      for (int t = 0; t < ntiles; ++t) {
        const int st = t % L::STAGES, use = t / L::STAGES;
        if (use > 0) mbar_wait(mbar + 64 + 8 * st, (use - 1) & 1);
        mbar_expect_tx(mbar + 32 + 8 * st, (uint32_t)(rows * 16));
        bulk_g2s(idx_s + (uint32_t)(st * L::IDX_BYTES),
                 p.payload + ((size_t)(kt0 + t) * p.m_pad + m0) * 16, (uint32_t)(rows * 16),
                 mbar + 32 + 8 * st);
      }
    }
  } else if (warp >= kLW) {
    // =========================== builders: full tables (a3)
    const int bw = warp - kLW;
    const int j = lane & 15;
    pdl_wait();  // A is produced by the previous kernel (quantizer)
    uint32_t U[L::WPB][G];
    if (ntiles > 0) load_act<G, NW, TPW>(p, kt0, j, n0, bw, U);
#pragma unroll 1
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1;
      uint32_t Un[L::WPB][G];
      if (t + 1 < ntiles) load_act<G, NW, TPW>(p, kt0 + t + 1, j, n0, bw, Un);
      if (t >= 2) mbar_wait(mbar + 16 + 8 * b, ((t >> 1) - 1) & 1);  // lookups of t-2 done
#pragma unroll
      for (int wi = 0; wi < L::WPB; ++wi) {
        const int w = bw + wi * kBW;
        if (w < NW) {
          uint32_t P[8], Mn[8];
          uint32_t T = (uint32_t)L::BIAS * (TPW == 2 ? 0x00010001u : 1u);
#pragma unroll
          for (int r = 0; r < G; ++r) {
            if constexpr (TPW == 1) {
              P[r] = U[wi][r];
              Mn[r] = 0u - U[wi][r];
            } else {
              P[r] = U[wi][r] - 0x00800080u;   // +a as a packed arithmetic delta
              Mn[r] = 0x00800080u - U[wi][r];  // -a
            }
            T += Mn[r];  // entry 0: every trit -1
          }
          const uint32_t row = tab_s + (uint32_t)(b * L::TAB_BYTES) +
                               (uint32_t)((w >> 1) * L::R * kRowStride) + (uint32_t)((w & 1) * 128) +
                               (uint32_t)(4 * lane);
          sts32(row, T);
          walk_full<G>(row, T, P, Mn);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + 8 * b);  // table t ready
      if (t + 1 < ntiles) {
#pragma unroll
        for (int wi = 0; wi < L::WPB; ++wi)
#pragma unroll
          for (int r = 0; r < G; ++r) U[wi][r] = Un[wi][r];
      }
    }
  } else {
    // =========================== lookup warps (a4)
    const int x = lane & 15;
    const int qk = x >> 2;
    uint32_t selv[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) selv[b] = 0x5504u | ((uint32_t)(b ^ (x & 3)) << 4);
    uint32_t sw[L::RPL][NW];
#pragma unroll
    for (int q = 0; q < L::RPL; ++q)
#pragma unroll
      for (int w = 0; w < NW; ++w) sw[q][w] = 0;
    int since_flush = 0;
    // one K-tile with table buffer B (compile time: the buffer offset folds
    // into the LDS immediate, one PRMT forms the rest of each address)
    auto tile = [&](auto Bc, int t) {
      constexpr int B = decltype(Bc)::value;
      const int st = t % L::STAGES;
      mbar_wait(mbar + 32 + 8 * st, (t / L::STAGES) & 1);  // index rows landed
      uint4 v[L::RPL];
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        const int r = q * (kLW * 32) + warp * 32 + lane;
        v[q] = (m0 + q * (kLW * 32) + warp * 32 < p.m_pad)
                   ? *reinterpret_cast<const uint4*>(smem + L::IDX_OFF + st * L::IDX_BYTES + r * 16)
                   : make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + 64 + 8 * st);  // ring slot free
      mbar_wait(mbar + 8 * B, (t >> 1) & 1);           // table t built
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        if (m0 + q * (kLW * 32) + warp * 32 >= p.m_pad) continue;  // warp-uniform
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
          const uint32_t off = __byte_perm(Wp[s >> 2], (uint32_t)((4 * lane) ^ (4 * s)), selv[s & 3]);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint32_t val = *reinterpret_cast<const uint32_t*>(
                smem + (B * L::TAB_BYTES + (w >> 1) * L::R * kRowStride + (w & 1) * 128) + off);
            if constexpr (TPW == 1) acc[q][w][0] += (int32_t)val;
            else sw[q][w] += val;
          }
        }
      }
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
    pdl_wait();  // epilogue reads a_scale / the workspace of the previous kernel
  }
  pdl_launch_dependents();

  // =========================== split-K reduction + epilogue (a5, a6)
  if (S > 1) {
    if (warp < kLW) {
#pragma unroll
      for (int q = 0; q < L::RPL; ++q) {
        const int m = m0 + q * (kLW * 32) + warp * 32 + lane;
        if (m >= p.M) continue;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int e = 0; e < TPW; ++e) {
            const int n = n0 + w * TPW + e;
            if (n < p.N) red_add_s32(p.ws_acc + (size_t)m * p.N + n, acc[q][w][e]);
          }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      unsigned* cnt = p.ws_cnt + (blockIdx.z * gridDim.y + blockIdx.y);
      const unsigned prev = atom_add_acq_rel(cnt, 1u);
      const bool last = (prev == (unsigned)(S - 1));
      if (last) *cnt = 0u;  // every CTA of the tile has arrived: re-arm for the next launch
      *last_flag = last ? 1u : 0u;
    }
    __syncthreads();
    if (*last_flag == 0u) return;
    __threadfence();
  }
  if (warp >= kLW) return;
#pragma unroll
  for (int q = 0; q < L::RPL; ++q) {
    const int m = m0 + q * (kLW * 32) + warp * 32 + lane;
    if (m >= p.M) continue;
#pragma unroll
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int e = 0; e < TPW; ++e) {
        const int n = n0 + w * TPW + e;
        if (n >= p.N) continue;
        int32_t a = acc[q][w][e];
        if (S > 1) {
          int32_t* src = p.ws_acc + (size_t)m * p.N + n;
          a = __ldcg(src);
          __stcg(src, 0);  // keep the workspace zero for the next launch
        }
        if (p.acc_only) {
          reinterpret_cast<int32_t*>(p.out)[(size_t)m * p.N + n] = a;
        } else {
          const float sc = __fmul_rn(__ldg(p.a_scale + n), p.w_scale);
          reinterpret_cast<float*>(p.out)[(size_t)m * p.N + n] = __fmul_rn((float)a, sc);
        }
      }
  }
}

}  // namespace slot
}  // namespace vlut
