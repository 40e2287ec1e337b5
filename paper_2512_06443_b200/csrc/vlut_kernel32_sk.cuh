// vlut_kernel32_sk.cuh -- K1-32-SK: K1-32 (32-token tiles, paired-group
// tables, vlut_kernel32.cuh) under the stream-K persistent schedule of K1-SK
// (vlut_kernel_sk.cuh): one CTA per SM takes an equal slice of the flattened
// (tile, K-tile) unit list, split tiles pass int32 partials through the
// workspace with partial-ready flags that their consumers reset.
//
// K1-32's accumulators are 16 SWAR registers per output row (32 tokens), so
// a lookup thread can own two rows (768 rows per CTA with 12 warps) without
// spilling -- K1's 64-token rows need 32 registers each and spill at two
// rows with 12 warps.  Many rows per CTA amortise the half-table build: at
// g = 5 (122 lines per pair) the build is 32 % of the lookup wavefronts at 384
// rows, 16 % at 768.  (Four rows, 1536 per CTA, spill again: measured 3-30 %
// slower, not instantiated.)
//
// Per unit the builders stage the unit's index rows (MCTA x 16 B, one bulk
// copy) and activation tile (3-D TMA box 32 x 16 x g, or 2-D when K % g
// != 0) one unit ahead and build the pair tables with 16-byte stores; the
// lookup warps run every row block's lookups per sub-stage (index words
// reloaded per row block: one 16-byte load, so only one block's words are
// live) and widen into TMEM (row block rb at column CB * rb).  Segment
// epilogues work per thread on its rows: TMEM -> registers; a producer
// stores its int32 rows to workspace slot `cta` and releases its flag; an
// owner waits for (and resets) its producers' flags, adds their rows and
// stores fp32; a whole tile stores fp32 directly.  Integer addition is exact:
// bit-identical to every other plan.
#pragma once
#include "vlut_kernel32.cuh"
#include "vlut_kernel_sk.cuh"

namespace vlut {

#ifndef VLUT_SK32_FIX_MLP
#define VLUT_SK32_FIX_MLP 2
#endif

__device__ __forceinline__ void red_add_v4f32(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

template <int G, int WARPS, int RPT, bool ACC_ONLY>
__device__ __forceinline__ void sk32_epilogue(const Params& p, const SkParams& sk, const SkSeg sg,
                                              int KT, int cta, int NCTA, int tid, int lane,
                                              uint32_t taddr0) {
  using C = Cfg32<G, true>;
  using L = Layout32<G, WARPS, RPT, true>;
  constexpr int NLT = L::NLT;
  const int m0 = (sg.tile / sk.NT) * L::MCTA, n0 = (sg.tile % sk.NT) * kN32;
  const int32_t bias_total = C::BIAS * kKgTile * (sg.kb - sg.ka);
  const bool producer = sg.kb < KT;
  const bool owner = !producer && sg.ka > 0;
  int c_lo = cta;
  // split tiles meet in fp32 (sk.acc): every partial and every partial sum
  // is an integer of magnitude <= K * 128 < 2^24 (the host enables it only
  // then), so fp32 adds are exact and order-free -- each producer red.adds
  // its rows into the accumulator of the tile's first producer CTA (no
  // owner-side read per producer), the owner reads that one slot, adds its
  // own rows and zeroes it for the next launch
  const bool red_mode = sk.acc != nullptr;
  const long long head = (long long)sg.tile * KT;
  if (producer) VLUT_STAMP(5);
  if (producer && red_mode) {
    c_lo = cta;
    while (c_lo > 0 && sk_begin(sk.U, NCTA, c_lo) > head) --c_lo;
  }
  if (owner) {
    VLUT_STAMP(2);
    // the tile's head units [tile*KT, tile*KT + ka) came from the preceding CTA(s)
    c_lo = cta - 1;
    while (c_lo > 0 && sk_begin(sk.U, NCTA, c_lo) > head) --c_lo;
    if (tid == 0) {
      for (int c2 = cta - 1; c2 >= c_lo; --c2) {
        unsigned spins = 0;  // bounded: a schedule bug must fail loudly, never hang
        while (ld_acquire_gpu(sk.flags + c2) != sk.epoch) {
          __nanosleep(64);
          if (++spins > (1u << 26)) __trap();
        }
        st_relaxed_gpu(sk.flags + c2, 0u);  // consumed: 0 again for the next launch
      }
    }
    bar_sync(6, NLT);
    VLUT_STAMP(3);
  }
#pragma unroll 1
  for (int rb = 0; rb < RPT; ++rb) {
    const int row = rb * NLT + tid;
    const int m = m0 + row;
    uint32_t v[2][16];
    tmem_ld16(taddr0 + (uint32_t)(L::CB * rb), v[0]);
    tmem_ld16(taddr0 + (uint32_t)(L::CB * rb) + 16, v[1]);
    tmem_wait_ld();
    // slot k = 2h + e of this lane: tokens 8c .. 8c+7, c = (lane ^ k) & 3,
    // as two 4-token quads (hh = 0, 1)
    int32_t a[4][2][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          a[k][hh][j] = (int32_t)(v[k >> 1][8 * (k & 1) + 4 * hh + j] - (uint32_t)bias_total);
    if (producer && red_mode) {
      float* arow = sk.acc + ((size_t)c_lo * L::MCTA + row) * kN32;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = (lane ^ k) & 3;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          red_add_v4f32(arow + 8 * c + 4 * hh, (float)a[k][hh][0], (float)a[k][hh][1],
                        (float)a[k][hh][2], (float)a[k][hh][3]);
      }
      continue;
    }
    if (producer) {
      int32_t* wrow = sk.ws + ((size_t)cta * L::MCTA + row) * kN32;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = (lane ^ k) & 3;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          __stcg(reinterpret_cast<int4*>(wrow + 8 * c + 4 * hh),
                 make_int4(a[k][hh][0], a[k][hh][1], a[k][hh][2], a[k][hh][3]));
      }
      continue;
    }
    if (owner && red_mode) {
      float* arow = sk.acc + ((size_t)c_lo * L::MCTA + row) * kN32;
      float4 w4[4][2];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = (lane ^ k) & 3;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          w4[k][hh] = __ldcg(reinterpret_cast<const float4*>(arow + 8 * c + 4 * hh));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = (lane ^ k) & 3;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          a[k][hh][0] += (int32_t)w4[k][hh].x; a[k][hh][1] += (int32_t)w4[k][hh].y;
          a[k][hh][2] += (int32_t)w4[k][hh].z; a[k][hh][3] += (int32_t)w4[k][hh].w;
          __stcg(reinterpret_cast<float4*>(arow + 8 * c + 4 * hh), make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
    } else if (owner) {
      // producers' rows read VLUT_SK32_FIX_MLP at a time (all loads in flight
      // before the adds): the fixup is a chain of L2 round trips, one per
      // batch -- at N = 256 a tile has ~5 producers (r02_sk32_fixup.txt)
      constexpr int FB = VLUT_SK32_FIX_MLP;
#pragma unroll 1
      for (int c2 = cta - 1; c2 >= c_lo; c2 -= FB) {
        int4 w4[FB][4][2];
#pragma unroll
        for (int f = 0; f < FB; ++f) {
          const int cf = c2 - f >= c_lo ? c2 - f : c2;  // past the last producer: re-read, unused
          const int32_t* prow = sk.ws + ((size_t)cf * L::MCTA + row) * kN32;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c = (lane ^ k) & 3;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              w4[f][k][hh] = __ldcg(reinterpret_cast<const int4*>(prow + 8 * c + 4 * hh));
          }
        }
#pragma unroll
        for (int f = 0; f < FB; ++f) {
          if (c2 - f < c_lo) break;
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              a[k][hh][0] += w4[f][k][hh].x; a[k][hh][1] += w4[f][k][hh].y;
              a[k][hh][2] += w4[f][k][hh].z; a[k][hh][3] += w4[f][k][hh].w;
            }
        }
      }
    }
    if (m >= p.M) continue;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = (lane ^ k) & 3;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int n = n0 + 8 * c + 4 * hh;
        if (n >= p.N) continue;  // N % 16 == 0: a quad is all-in or all-out
        if constexpr (ACC_ONLY) {
          *reinterpret_cast<int4*>(reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n) =
              make_int4(a[k][hh][0], a[k][hh][1], a[k][hh][2], a[k][hh][3]);
        } else {
          float f[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            f[j] = __fmul_rn((float)a[k][hh][j], __fmul_rn(__ldg(p.a_scale + n + j), p.w_scale));
          *reinterpret_cast<float4*>(p.out + (size_t)m * p.N + n) = make_float4(f[0], f[1], f[2], f[3]);
        }
      }
    }
  }
  if (producer) {
    __threadfence();
    bar_sync(6, NLT);
    if (tid == 0) st_release_gpu(sk.flags + cta, sk.epoch);
  }
}

// The raw-int32 variant's epilogue as a real call: inlined, ptxas spilled
// registers inside that variant's lookup loop (the fp32 variant is clean).
template <int G, int WARPS, int RPT>
__device__ __noinline__ void sk32_epilogue_acc(const Params& p, const SkParams& sk, const SkSeg sg,
                                               int KT, int cta, int NCTA, int tid, int lane,
                                               uint32_t taddr0) {
  sk32_epilogue<G, WARPS, RPT, true>(p, sk, sg, KT, cta, NCTA, tid, lane, taddr0);
}

template <int G, int WARPS, int RPT, bool ACC_ONLY>
__global__ void __launch_bounds__((WARPS + kBuilderWarps) * 32, 1)
    vlut_mpgemm32_sk_kernel(const __grid_constant__ Params p, const SkParams sk) {
  using C = Cfg32<G, true>;
  using L = Layout32<G, WARPS, RPT, true>;
  constexpr int PB = (RPT >= 4) ? 1 : 2;  // pairs per load batch (registers)
  extern __shared__ __align__(1024) uint8_t smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int cta = blockIdx.x;
  const int NCTA = gridDim.x;
  const int KT = p.kg_tiles;
  const long long u0 = sk_begin(sk.U, NCTA, cta), u1 = sk_begin(sk.U, NCTA, cta + 1);
  const int nunits = (int)(u1 - u0);
  const int nsub = nunits * C::SUBS;
  VLUT_STAMP(0);

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = smem_u32(smem + L::IDX_OFF);
  const uint32_t a_s0 = smem_u32(smem + L::A_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::MISC_OFF);
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

  if (warp >= WARPS) {
    // =========================== builders: staging + table builds over the unit list
    const int bt = tid - L::BUILDER0;
    const int bw = warp - WARPS;
    SkIter nxt;
    nxt.init(u0, u1, KT);
    auto tile_m0 = [&](int tile) { return (tile / sk.NT) * L::MCTA; };
    auto tile_n0 = [&](int tile) { return (tile % sk.NT) * kN32; };
    if (nunits > 0) {  // unit 0: index rows before griddepcontrol.wait, activations after
      const int m0 = tile_m0(nxt.seg.tile), n0 = tile_n0(nxt.seg.tile);
      stage32<G, WARPS, RPT, true>(p, nxt.kt, 0, m0, n0, smem, bt, mbar + m32_stage<C::NBUF>(0),
                                   true, false, true);
      pdl_wait();
      stage32<G, WARPS, RPT, true>(p, nxt.kt, 0, m0, n0, smem, bt, mbar + m32_stage<C::NBUF>(0),
                                   false, true, false);
      nxt.next();
    } else {
      pdl_wait();
    }
#pragma unroll 1
    for (int u = 0; u < nsub + C::NBUF; ++u) {
      if (u >= C::NBUF) mbar_wait(mbar + m32_empty<C::NBUF>(u % C::NBUF), ((u / C::NBUF) - 1) & 1);
      if (u >= nsub) continue;
      const int T = u / C::SUBS, sub = u - T * C::SUBS;
      if (sub == 0) {
        if (nxt.valid()) {  // unit T + 1
          const int b1 = (T + 1) % C::STAGE;
          stage32<G, WARPS, RPT, true>(p, nxt.kt, b1, tile_m0(nxt.seg.tile), tile_n0(nxt.seg.tile),
                                       smem, bt, mbar + m32_stage<C::NBUF>(b1), true, true, true);
          nxt.next();
        }
        mbar_wait(mbar + m32_stage<C::NBUF>(T % C::STAGE), (T / C::STAGE) & 1);
        bar_sync(5, kBuilderWarps * 32);
      }
      build_tables32<G>(tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES),
                        a_s0 + (uint32_t)((T % C::STAGE) * C::A_BYTES), sub * C::GS, bw, lane,
                        p.a3d != 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + m32_full<C::NBUF>(u % C::NBUF));
    }
  } else {
    // =========================== lookup warps (RPT rows per thread: tid + rb * NLT)
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(L::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tmem_fence_before();
    bar_sync(6, L::NLT);
    tmem_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    uint32_t rot[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)((((lane & 7) ^ s) & 7) * 16);
    Sel32 sel;
    sel.init((lane & 4) ? 1 : 0);
    const uint32_t taddr0 =
        tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(32 * (warp >> 2));
    uint32_t sw[RPT][4][4];
    int32_t nneg[RPT];
#pragma unroll
    for (int rb = 0; rb < RPT; ++rb) {
      nneg[rb] = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) sw[rb][k][q] = 0;
    }
    bool first = true;
    int since_flush = warp % kFlushTiles;
    SkIter cur;
    cur.init(u0, u1, KT);
#pragma unroll 1
    for (int t = 0; t < nunits; ++t) {
#pragma unroll
      for (int sub = 0; sub < C::SUBS; ++sub) {
        const int u = t * C::SUBS + sub;
        mbar_wait(mbar + m32_full<C::NBUF>(u % C::NBUF), (u / C::NBUF) & 1);
        if (u == 0) VLUT_STAMP(1);
#pragma unroll
        for (int rb = 0; rb < RPT; ++rb) {
          const uint4 iw = lds128(idx_s + (uint32_t)((t % C::STAGE) * L::IDX_BYTES +
                                                     (tid + rb * L::NLT) * 16));
          const uint32_t iwa[4] = {iw.x, iw.y, iw.z, iw.w};
          lookup_sub32<G, PB>(sub, tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES), iwa, rot, sel,
                              sw[rb], nneg[rb]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar + m32_empty<C::NBUF>(u % C::NBUF));
      }
      const bool seg_end = (cur.kt + 1 == cur.seg.kb);
      if (++since_flush >= kFlushTiles || seg_end) {
        since_flush = 0;
#pragma unroll
        for (int rb = 0; rb < RPT; ++rb)
          flush32<G>(sw[rb], nneg[rb], taddr0 + (uint32_t)(L::CB * rb), first);
        first = false;
      }
      if (seg_end) {
        if constexpr (ACC_ONLY)
          sk32_epilogue_acc<G, WARPS, RPT>(p, sk, cur.seg, KT, cta, NCTA, tid, lane, taddr0);
        else
          sk32_epilogue<G, WARPS, RPT, false>(p, sk, cur.seg, KT, cta, NCTA, tid, lane, taddr0);
        first = true;  // the next segment re-initialises TMEM
      }
      cur.next();
    }
    VLUT_STAMP(4);
    pdl_wait();
    tmem_fence_before();
    bar_sync(6, L::NLT);
    if (warp == 0) {
      tmem_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                   "n"(L::TMEM_COLS)
                   : "memory");
    }
  }
  pdl_launch_dependents();
}

}  // namespace vlut
