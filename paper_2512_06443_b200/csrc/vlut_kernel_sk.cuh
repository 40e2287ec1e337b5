// vlut_kernel_sk.cuh -- K1-SK: the Vec-LUT mpGeMM with stream-K persistent
// scheduling (one CTA per SM, no clusters).
//
// The tiles of the grid (32*WARPS rows x 64 tokens) times their K-tiles form
// a flat list of U work units (u = tile * KT + kt, tiles ordered N-fastest so
// CTAs working at the same time share weight rows in L2).  CTA c processes
// units [c*U/G, (c+1)*U/G): whatever the tile count, every SM gets the same
// amount of lookups (no wave quantization).  A CTA's range is cut into
// segments (a run of K-tiles of one tile):
//   * full      [0, KT)        -> epilogue straight from TMEM
//   * producer  [ka, kb < KT)  -> the tile continues in the next CTA(s): the
//                                 int32 partial goes to workspace slot c, then
//                                 flags[c] = 1 (release)
//   * owner     [ka > 0, KT)   -> waits (acquire) for the producers of the
//                                 tile's head, resets their flags to 0, adds
//                                 their partials, epilogue
// Every producer has exactly one owner, so every flag a launch sets is reset
// by the same launch: all flags are 0 between launches and the handshake
// needs no host-side state -- a captured CUDA graph can be replayed (the
// next launch's producers store only after its griddepcontrol.wait, i.e.
// after this launch's resets are performed).
// Execution order inside a CTA: middle full tiles, its last segment, its
// first segment -- producers never wait, owners wait last, so the dependency
// graph is acyclic and all G <= #SMs CTAs are co-resident: no deadlock.
// Integer partial sums are exact, so the result is bit-identical to every
// other plan.  The table build / lookup / accumulation machinery is K1's
// (vlut_kernel.cuh): builder warps stage (TMA) and build double-buffered half
// tables, lookup warps own one output row each and widen into TMEM.
#pragma once
#include "vlut_kernel.cuh"

namespace vlut {

// The g = 5 two-rows-per-thread 12-warp variant (128 registers, 64 of them
// SWAR fields) loads index words lazily and uses the XOR chunk order (A/B:
// config 4 g = 5 N = 1024 1089 -> 1073 us; at g = 4 the eager form is ~1.5 %
// faster on config 5's gate shape).
template <int G, int WARPS, int RPT>
#ifndef VLUT_SK_LAZY16
#define VLUT_SK_LAZY16 0
#endif
constexpr bool kLazyRx = (G == 5 && RPT == 2 && WARPS == 12) || (VLUT_SK_LAZY16 && WARPS == 16);

struct SkParams {
  int NT, MT;           // N-tiles, M-tiles
  long long U;          // units = NT * MT * KT
  int32_t* ws;          // [G][MCTA * 64] int32 partials
  unsigned* flags;      // [G] partial-ready flags: 0 between launches
  unsigned epoch;       // the 'ready' value (1)
  // K1-32-SK with K * 128 < 2^24: split tiles meet in fp32 accumulators
  // [G][MCTA * 32] (slot = the tile's first producer CTA), zero between
  // launches; nullptr: the int32 partial slots above
  float* acc;
};

struct SkSeg {
  int tile, ka, kb;
};

__device__ __forceinline__ long long sk_begin(long long U, int G, int c) {
  return U * (long long)c / G;
}

// segment j (execution order) of the unit range [u0, u1)
__device__ __forceinline__ SkSeg sk_seg(long long u0, long long u1, int KT, int j) {
  const long long tf = u0 / KT, tl = (u1 - 1) / KT;
  const int kf = (int)(u0 % KT), kl = (int)((u1 - 1) % KT) + 1;
  if (tf == tl) return {(int)tf, kf, kl};
  const int nmid = (int)(tl - tf - 1);
  if (j < nmid) return {(int)(tf + 1 + j), 0, KT};
  if (j == nmid) return {(int)tl, 0, kl};
  return {(int)tf, kf, KT};
}

__device__ __forceinline__ int sk_nseg(long long u0, long long u1, int KT) {
  if (u1 <= u0) return 0;
  return (int)((u1 - 1) / KT - u0 / KT + 1);
}

// iterator over the units of a CTA in execution order
struct SkIter {
  long long u0, u1;
  int KT, nseg, j, kt;
  SkSeg seg;
  __device__ __forceinline__ void init(long long a, long long b, int kt_count) {
    u0 = a;
    u1 = b;
    KT = kt_count;
    nseg = sk_nseg(a, b, kt_count);
    j = 0;
    if (nseg > 0) {
      seg = sk_seg(u0, u1, KT, 0);
      kt = seg.ka;
    }
  }
  __device__ __forceinline__ bool valid() const { return j < nseg; }
  __device__ __forceinline__ void next() {
    if (++kt >= seg.kb) {
      if (++j < nseg) {
        seg = sk_seg(u0, u1, KT, j);
        kt = seg.ka;
      }
    }
  }
};

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Segment epilogue of K1-SK, kept out of the lookup loop's register
// allocation (__noinline__): full tiles and producers straight from TMEM (one
// row per thread and row block, four 16-column chunks); the owner (always the
// CTA's last segment, so the table region is free) through a shared int32
// tile -- one row block of NLT rows at a time -- and a flat, coalesced
// reduction of the producers' partials.
template <int G, int WARPS, int RPT, bool ACC_ONLY>
__device__ __forceinline__ void sk_epilogue(const Params& p, const SkParams& sk, const SkSeg sg,
                                         int KT, int cta, int NCTA, int tid, int lane,
                                         uint32_t taddr0, uint32_t tab_s, const uint8_t* smem) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS, RPT>;
  constexpr int NLT = L::NLT;
  constexpr bool RX = kLazyRx<G, WARPS, RPT>;
  const int r = tid;  // row within a row block
  const int m0 = (sg.tile / sk.NT) * L::MCTA, n0 = (sg.tile % sk.NT) * kNcta;
  const int32_t bias_total = C::BIAS * kKgTile * (sg.kb - sg.ka);
  const bool producer = sg.kb < KT;
  const bool owner = !producer && sg.ka > 0;
  const long long head = (long long)sg.tile * KT;
  unsigned* cta_max = reinterpret_cast<unsigned*>(const_cast<uint8_t*>(smem) + L::AMAX_OFF);
  const bool want_max = !ACC_ONLY && p.amax_out != nullptr && !producer;
  if (want_max) {
    if (tid < kNcta) cta_max[tid] = 0u;
    bar_sync(6, NLT);
  }
  if (owner) {
    // the tile's units [tile*KT, tile*KT + ka) were produced by the
    // preceding CTA(s)
    int c_lo = cta - 1;
    while (c_lo > 0 && sk_begin(sk.U, NCTA, c_lo) > head) --c_lo;
    float tok_max[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
    for (int rb = 0; rb < RPT; ++rb) {
      // the owner segment is the CTA's last: every table read is done once
      // all lookup warps get here, so the table region holds the row block.
      // TMEM -> shared int32 tile (XOR-swizzled rows, as in K1)
      bar_sync(6, NLT);
      {
        const uint32_t swz = (uint32_t)((r >> 2) & 1);
        const uint32_t taddr = taddr0 + 256u * (uint32_t)rb;
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {
          uint32_t v[16];
          tmem_ld16(taddr + 16 * h, v);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const uint32_t c = (uint32_t)chunk_of<RX>(lane, 2 * h + e);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const uint32_t uu = (2 * c + hh) ^ swz;
              const uint32_t* x = v + 8 * e + 4 * hh;
              sts128(tab_s + r * 256 + uu * 16, x[0] - bias_total, x[1] - bias_total,
                     x[2] - bias_total, x[3] - bias_total);
            }
          }
        }
      }
      if (rb == 0 && tid == 0) {
        for (int c2 = cta - 1; c2 >= c_lo; --c2) {
          // bounded wait: a schedule bug must fail loudly, never hang
          unsigned spins = 0;
          while (ld_acquire_gpu(sk.flags + c2) != sk.epoch) {
            __nanosleep(64);
            if (++spins > (1u << 26)) __trap();
          }
          // consumed: back to 0 for the next launch (this launch sets it
          // only once, so no later store can race with the reset)
          st_relaxed_gpu(sk.flags + c2, 0u);
        }
      }
      bar_sync(6, NLT);
      // flat reduction: unit e = (row e/16 of the block, tokens 4(e%16)..+3),
      // UPT units per thread per round; all loads of a producer issued together
      constexpr int UPT = 4;
      const int4* red = reinterpret_cast<const int4*>(smem);
      const size_t blk = (size_t)rb * NLT * 16;  // int4 offset of the row block in a slot
#pragma unroll 1
      for (int half = 0; half < 16 / UPT; ++half) {
        int4 acc4[UPT];
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int e = tid + (half * UPT + i) * NLT;
          const int rr = e >> 4;
          acc4[i] = red[rr * 16 + ((e & 15) ^ ((rr >> 2) & 1))];
        }
        // PP producers per round, all their loads issued before any add: with
        // few tiles a tile has many producers and one round trip per producer
        // would serialise the fixup
        constexpr int PP = (WARPS >= 16) ? 2 : 4;
        int c2 = cta - 1;
        for (; c2 - (PP - 1) >= c_lo; c2 -= PP) {
          int4 w4[PP][UPT];
#pragma unroll
          for (int pp = 0; pp < PP; ++pp) {
            const int4* prow =
                reinterpret_cast<const int4*>(sk.ws + (size_t)(c2 - pp) * L::MCTA * kNcta) + blk;
#pragma unroll
            for (int i = 0; i < UPT; ++i) w4[pp][i] = __ldcg(prow + tid + (half * UPT + i) * NLT);
          }
#pragma unroll
          for (int pp = 0; pp < PP; ++pp)
#pragma unroll
            for (int i = 0; i < UPT; ++i) {
              acc4[i].x += w4[pp][i].x; acc4[i].y += w4[pp][i].y;
              acc4[i].z += w4[pp][i].z; acc4[i].w += w4[pp][i].w;
            }
        }
        for (; c2 >= c_lo; --c2) {
          const int4* prow = reinterpret_cast<const int4*>(sk.ws + (size_t)c2 * L::MCTA * kNcta) + blk;
          int4 w4[UPT];
#pragma unroll
          for (int i = 0; i < UPT; ++i) w4[i] = __ldcg(prow + tid + (half * UPT + i) * NLT);
#pragma unroll
          for (int i = 0; i < UPT; ++i) {
            acc4[i].x += w4[i].x; acc4[i].y += w4[i].y; acc4[i].z += w4[i].z; acc4[i].w += w4[i].w;
          }
        }
#pragma unroll
        for (int i = 0; i < UPT; ++i) {
          const int e = tid + (half * UPT + i) * NLT;
          const int mm = m0 + rb * NLT + (e >> 4), n = n0 + 4 * (e & 15);
          if (mm >= p.M || n >= p.N) continue;
          const int32_t x[4] = {acc4[i].x, acc4[i].y, acc4[i].z, acc4[i].w};
          if constexpr (ACC_ONLY) {
            int32_t* o = reinterpret_cast<int32_t*>(p.out) + (size_t)mm * p.N + n;
            if (p.out_vec4 && n + 3 < p.N) *reinterpret_cast<int4*>(o) = acc4[i];
            else for (int k = 0; k < 4 && n + k < p.N; ++k) o[k] = x[k];
          } else {
            float f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float sc = (n + k < p.N) ? __fmul_rn(__ldg(p.a_scale + n + k), p.w_scale) : 0.f;
              f[k] = __fmul_rn((float)x[k], sc);
            }
            if (p.mul_in) {
              const float* mi = p.mul_in + (size_t)mm * p.N + n;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (n + k < p.N) f[k] = __fmul_rn(f[k], __ldg(mi + k));
            }
            if (want_max && mm < p.amax_rows) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (n + k < p.N) tok_max[k] = fmaxf(tok_max[k], fabsf(f[k]));
            }
            float* o = p.out + (size_t)mm * p.N + n;
            if (p.out_vec4 && n + 3 < p.N) *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
            else for (int k = 0; k < 4 && n + k < p.N; ++k) o[k] = f[k];
          }
        }
      }
    }
    if (want_max) {
      // thread's token quad 4 (tid & 15) .. +3 is fixed: lanes l, l+16 share it
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        tok_max[k] = fmaxf(tok_max[k], __shfl_xor_sync(0xffffffffu, tok_max[k], 16));
        if (lane < 16) atomicMax(cta_max + 4 * (tid & 15) + k, __float_as_uint(tok_max[k]));
      }
      bar_sync(6, NLT);
      if (tid < kNcta && n0 + tid < p.N && cta_max[tid] != 0u)
        atomicMax(p.amax_out + n0 + tid, cta_max[tid]);
    }
    return;
  }
#pragma unroll 1
  for (int rb = 0; rb < RPT; ++rb) {
    const int rr = rb * NLT + r;  // row within the tile
    const int m = m0 + rr;
    const uint32_t taddr = taddr0 + 256u * (uint32_t)rb;
#pragma unroll 1
    for (int h = 0; h < 4; ++h) {
      uint32_t v[16];
      tmem_ld16(taddr + 16 * h, v);
      tmem_wait_ld();
      int32_t a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = (int32_t)(v[i] - bias_total);
      if (producer) {
        // int32 partial -> workspace slot [row][token] (the owner reads it
        // row-contiguous and coalesced)
        int32_t* wrow = sk.ws + ((size_t)cta * L::MCTA + rr) * kNcta;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = chunk_of<RX>(lane, 2 * h + e);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int32_t* x = a + 8 * e + 4 * hh;
            __stcg(reinterpret_cast<int4*>(wrow + 8 * c + 4 * hh), make_int4(x[0], x[1], x[2], x[3]));
          }
        }
        continue;
      }
      if (m >= p.M) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = chunk_of<RX>(lane, 2 * h + e);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int n = n0 + 8 * c + 4 * hh;
          if (n >= p.N) continue;
          const int32_t* x = a + 8 * e + 4 * hh;
          if constexpr (ACC_ONLY) {
            int32_t* o = reinterpret_cast<int32_t*>(p.out) + (size_t)m * p.N + n;
            if (p.out_vec4 && n + 3 < p.N) *reinterpret_cast<int4*>(o) = make_int4(x[0], x[1], x[2], x[3]);
            else for (int k = 0; k < 4 && n + k < p.N; ++k) o[k] = x[k];
          } else {
            float f[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float sc = (n + k < p.N) ? __fmul_rn(__ldg(p.a_scale + n + k), p.w_scale) : 0.f;
              f[k] = __fmul_rn((float)x[k], sc);
            }
            if (p.mul_in) {
              const float* mi = p.mul_in + (size_t)m * p.N + n;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                if (n + k < p.N) f[k] = __fmul_rn(f[k], __ldg(mi + k));
            }
            if (want_max && m < p.amax_rows) {
              for (int k = 0; k < 4 && n + k < p.N; ++k)
                atomicMax(cta_max + (n - n0) + k, __float_as_uint(fabsf(f[k])));
            }
            float* o = p.out + (size_t)m * p.N + n;
            if (p.out_vec4 && n + 3 < p.N) *reinterpret_cast<float4*>(o) = make_float4(f[0], f[1], f[2], f[3]);
            else for (int k = 0; k < 4 && n + k < p.N; ++k) o[k] = f[k];
          }
        }
      }
    }
  }
  if (want_max) {
    bar_sync(6, NLT);
    if (tid < kNcta && n0 + tid < p.N && cta_max[tid] != 0u)
      atomicMax(p.amax_out + n0 + tid, cta_max[tid]);
  }
  if (producer) {
    __threadfence();
    bar_sync(6, NLT);
    if (tid == 0) st_release_gpu(sk.flags + cta, sk.epoch);
  }
}

template <int G, int WARPS, int RPT, bool ACC_ONLY>
__global__ void __launch_bounds__((WARPS + kBW<WARPS, RPT>) * 32, 1)
    vlut_mpgemm_sk_kernel(const __grid_constant__ Params p, const SkParams sk) {
  using C = Cfg<G>;
  using L = Layout<G, WARPS, RPT>;
  constexpr int GP = kLookupGP2<WARPS, RPT>;
  constexpr bool RX = kLazyRx<G, WARPS, RPT>;
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

  const uint32_t tab_s = smem_u32(smem);
  const uint32_t idx_s = smem_u32(smem + L::IDX_OFF);
  const uint32_t a_s0 = smem_u32(smem + L::A_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::MISC_OFF);
  const uint32_t mbar = smem_u32(smem + L::MBAR_OFF);

  if (tid == L::BUILDER0) {
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(mbar + mb_full(b), L::BW);
      mbar_init(mbar + mb_empty(b), WARPS);
    }
    for (int st = 0; st < kStageBufs; ++st) mbar_init(mbar + mb_stage(st), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= WARPS) {
    // =========================== builders: staging + table builds over the unit list
    const int bt = tid - L::BUILDER0;
    const int bw = warp - WARPS;
    const bool bulk = (p.a_vec == 16);
    SkIter cur, nxt;
    cur.init(u0, u1, KT);
    nxt.init(u0, u1, KT);
    auto tile_m0 = [&](int tile) { return (tile / sk.NT) * L::MCTA; };
    auto tile_n0 = [&](int tile) { return (tile % sk.NT) * kNcta; };
    if (nunits > 0) {
      const int m0 = tile_m0(nxt.seg.tile), n0 = tile_n0(nxt.seg.tile);
      if (bulk) {
        stage_tile_bulk<G, WARPS, RPT>(p, nxt.kt, 0, m0, n0, smem, bt, mbar + mb_stage(0), true, false, true);
        pdl_wait();
        stage_tile_bulk<G, WARPS, RPT>(p, nxt.kt, 0, m0, n0, smem, bt, mbar + mb_stage(0), false, true, false);
      } else {
        stage_tile<G, WARPS, RPT>(p, nxt.kt, 0, m0, n0, smem, bt, 1);
        pdl_wait();
        stage_tile<G, WARPS, RPT>(p, nxt.kt, 0, m0, n0, smem, bt, 2);
      }
      nxt.next();
    } else {
      pdl_wait();
    }
#pragma unroll 1
    for (int u = 0; u < nsub + C::NBUF; ++u) {
      if (u >= C::NBUF)  // lookups of u - NBUF done with this buffer
        mbar_wait(mbar + mb_empty(u % C::NBUF), ((u / C::NBUF) - 1) & 1);
      if (u >= nsub) continue;
      const int T = u / C::SUBS, sub = u - T * C::SUBS;
      if (sub == 0) {
        if (T > 0) cur.next();
        if (nxt.valid()) {  // unit T+1
          const int b1 = (T + 1) % kStageBufs;
          const int m0 = tile_m0(nxt.seg.tile), n0 = tile_n0(nxt.seg.tile);
          if (bulk) {
            stage_tile_bulk<G, WARPS, RPT>(p, nxt.kt, b1, m0, n0, smem, bt, mbar + mb_stage(b1), true,
                                      true, true);
          } else {
            stage_tile<G, WARPS, RPT>(p, nxt.kt, b1, m0, n0, smem, bt, 3);
          }
          nxt.next();
          if (!bulk) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else if (!bulk) {
          cp_async_wait_all();
        }
        if (bulk) mbar_wait(mbar + mb_stage(T % kStageBufs), (T / kStageBufs) & 1);
        bar_sync(5, L::BW * 32);
      }
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
      __syncwarp();
      if (lane == 0) mbar_arrive(mbar + mb_full(u % C::NBUF));
    }
  } else {
    // =========================== lookup warps (RPT rows per thread: r, r + NLT)
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
    // slot s of this lane <-> 16-byte chunk chunk_of<RX>(lane, s) of a row
    uint32_t rot[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)(chunk_of<RX>(lane, s) * 16);
    // row block rb of this warp: lanes 32 (warp & 3).., columns 64 (warp >> 2) + 256 rb
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    uint32_t sw[RPT][8][4];
    int32_t nneg[RPT];
    uint32_t iwa[RPT][4];
#pragma unroll
    for (int rb = 0; rb < RPT; ++rb) {
      nneg[rb] = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) iwa[rb][q] = 0u;
#pragma unroll
      for (int s = 0; s < 8; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q) sw[rb][s][q] = 0;
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
        mbar_wait(mbar + mb_full(u % C::NBUF), (u / C::NBUF) & 1);
        constexpr bool LAZY = kLazyRx<G, WARPS, RPT>;  // index words from shared memory
#pragma unroll
        for (int rb = 0; rb < RPT; ++rb) {
          const uint32_t idx_row =
              idx_s + (uint32_t)((t % kStageBufs) * L::IDX_BYTES + (tid + rb * L::NLT) * 16);
          if (!LAZY && sub == 0) {
            const uint4 iw = lds128(idx_row);
            iwa[rb][0] = iw.x; iwa[rb][1] = iw.y; iwa[rb][2] = iw.z; iwa[rb][3] = iw.w;
          }
          lookup_sub<G, GP, kLookupLB<WARPS, RPT>, LAZY, RX>(
              sub, tab_s + (uint32_t)((u % C::NBUF) * C::TAB_BYTES), iwa[rb], idx_row, rot, sw[rb],
              nneg[rb]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(mbar + mb_empty(u % C::NBUF));
      }
      const bool seg_end = (cur.kt + 1 == cur.seg.kb);
      if (++since_flush >= kFlushTiles || seg_end) {
        since_flush = 0;
#pragma unroll
        for (int rb = 0; rb < RPT; ++rb)
          flush_tmem<G, GP == 1>(sw[rb], nneg[rb], taddr + 256u * (uint32_t)rb, first);
        first = false;
      }
      if (seg_end) {
        sk_epilogue<G, WARPS, RPT, ACC_ONLY>(p, sk, cur.seg, KT, cta, NCTA, tid, lane, taddr, tab_s,
                                             smem);
        first = true;  // the next segment re-initialises TMEM
      }
      cur.next();
    }
    pdl_wait();
    // TMEM release: every lookup warp is done with it
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
