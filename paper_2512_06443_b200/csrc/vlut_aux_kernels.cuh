// vlut_aux_kernels.cuh -- K3 per-token quantizer and the device-side packer.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include "vlut_kernel.cuh"  // VLUT_STAMP (debug timing only)

namespace vlut {

#ifndef VLUT_Q_EARLY_TRIGGER
#define VLUT_Q_EARLY_TRIGGER 1
#endif
// Quantizer PDL order.  The dependent mpGeMM launches once every CTA of the
// quantizer has triggered, and touches nothing but the packed weights (which
// no kernel writes) before its own griddepcontrol.wait -- which returns only
// after this quantizer completed, and this quantizer's wait after ITS
// predecessor (e.g. the previous layer's mpGeMM) completed: the chain stays
// ordered.  Triggering BEFORE waiting therefore lets the next mpGeMM launch
// (and start streaming its weights) while this quantizer still waits for
// the previous kernel, instead of only after it.  All CTAs of this grid are
// resident when the dependent launches, so it cannot starve them.
__device__ __forceinline__ void pdl_trigger_then_wait() {
  if (VLUT_Q_EARLY_TRIGGER) {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
  } else {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  }
}

// ---------------------------------------------------------------- K3 quantize (a7)
// A thread-block cluster of CL CTAs owns 16 consecutive tokens; CTA `rank`
// owns a contiguous 1/CL slice of the K rows.  Each thread loads float4s
// (4 tokens of one row; 4 threads cover a row's 64 contiguous bytes) into
// registers, the per-token absmax is reduced warp -> CTA -> cluster (DSMEM),
// and the codes are written from the registers (rows beyond the register
// cache are re-read).  IEEE single ops only (no fast math):
//   s = amax / 127 (1 if amax == 0), q = clamp(roundf(x / s), -127, 127).
#ifndef VLUT_QTHREADS
#define VLUT_QTHREADS 512
#endif
constexpr int kQThreads = VLUT_QTHREADS;  // kQRows rows x 4 float4 columns per pass
constexpr int kQRows = kQThreads / 4;
constexpr int kQTok = 16;                 // tokens per cluster
constexpr int kQCache = 768 / kQRows;     // float4 register cache per thread (768 rows per CTA)

// One operand's float4 (4 tokens of row k), zeros outside N.
template <bool ALIGNED>
__device__ __forceinline__ float4 q_load1(const float* x, int k, int N, int n) {
  const size_t o = (size_t)k * N + n;
  if (ALIGNED && n + 3 < N) return __ldg(reinterpret_cast<const float4*>(x + o));
  float t[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) t[i] = (n + i < N) ? __ldg(x + o + i) : 0.f;
  return make_float4(t[0], t[1], t[2], t[3]);
}

__device__ __forceinline__ float4 fmul4(float4 a, float4 b) {
  return make_float4(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y), __fmul_rn(a.z, b.z),
                     __fmul_rn(a.w, b.w));
}

template <bool ALIGNED>
__device__ __forceinline__ float4 q_load(const float* x, const float* y, int k, int N, int n) {
  const size_t o = (size_t)k * N + n;
  float4 a;
  if (ALIGNED && n + 3 < N) {
    a = __ldg(reinterpret_cast<const float4*>(x + o));
    if (y) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(y + o));
      a.x = __fmul_rn(a.x, b.x); a.y = __fmul_rn(a.y, b.y);
      a.z = __fmul_rn(a.z, b.z); a.w = __fmul_rn(a.w, b.w);
    }
  } else {
    float t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      t[i] = 0.f;
      if (n + i < N) t[i] = y ? __fmul_rn(__ldg(x + o + i), __ldg(y + o + i)) : __ldg(x + o + i);
    }
    a = make_float4(t[0], t[1], t[2], t[3]);
  }
  return a;
}

__device__ __forceinline__ int8_t q_code(float v, float s) {
  float r = roundf(__fdiv_rn(v, s));
  r = fminf(fmaxf(r, -127.f), 127.f);
  return (int8_t)r;
}

template <bool ALIGNED>
__global__ void __launch_bounds__(kQThreads)
    vlut_quantize_kernel(const float* __restrict__ x, const float* __restrict__ y, int K, int N,
                         int8_t* __restrict__ q, float* __restrict__ scale) {
  __shared__ float red[kQThreads / 32][kQTok];
  __shared__ float all_max[8][kQTok];  // [cluster rank][token]: every CTA's maxima
  __shared__ float s_scale[kQTok];
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = tid & 3;              // float4 column within the 16 tokens
  const int rsub = tid >> 2;            // row within a kQRows-row pass
  const int n = blockIdx.y * kQTok + col * 4;
  const int k_begin = (int)(((long long)rank * K) / CL);
  const int k_end = (int)(((long long)(rank + 1) * K) / CL);
  VLUT_STAMP(0);
  // PDL: x may be the previous kernel's output; let the next kernel launch early
  pdl_trigger_then_wait();
  VLUT_STAMP(1);
  float4 cache[kQCache];
  float m[4] = {0.f, 0.f, 0.f, 0.f};
  // every load of the register cache is issued before any use (a multiply
  // right behind each load would serialise the DRAM round trips)
#pragma unroll
  for (int i = 0; i < kQCache; ++i) {
    const int k = k_begin + rsub + kQRows * i;
    cache[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < k_end && n < N) cache[i] = q_load1<ALIGNED>(x, k, N, n);
  }
  if (y) {
    float4 yc[kQCache];
#pragma unroll
    for (int i = 0; i < kQCache; ++i) {
      const int k = k_begin + rsub + kQRows * i;
      yc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < k_end && n < N) yc[i] = q_load1<ALIGNED>(y, k, N, n);
    }
#pragma unroll
    for (int i = 0; i < kQCache; ++i) cache[i] = fmul4(cache[i], yc[i]);
  }
#pragma unroll
  for (int i = 0; i < kQCache; ++i) {
    m[0] = fmaxf(m[0], fabsf(cache[i].x)); m[1] = fmaxf(m[1], fabsf(cache[i].y));
    m[2] = fmaxf(m[2], fabsf(cache[i].z)); m[3] = fmaxf(m[3], fabsf(cache[i].w));
  }
  for (int k = k_begin + rsub + kQRows * kQCache; k < k_end; k += kQRows) {
    if (n >= N) break;
    const float4 a = q_load<ALIGNED>(x, y, k, N, n);
    m[0] = fmaxf(m[0], fabsf(a.x)); m[1] = fmaxf(m[1], fabsf(a.y));
    m[2] = fmaxf(m[2], fabsf(a.z)); m[3] = fmaxf(m[3], fabsf(a.w));
  }
  VLUT_STAMP(2);
  // warp: lanes with equal (lane & 3) share tokens -> reduce over lane bits 2..4
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int d = 4; d < 32; d <<= 1) m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], d));
  if (lane < 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red[warp][lane * 4 + i] = m[i];
  }
  __syncthreads();
  // push model: the 16 combining threads store this CTA's maxima into slot
  // `rank` of every cluster CTA's table (DSMEM stores), one cluster barrier
  // (release / acquire), then every CTA reduces its own table locally -- no
  // remote round trip, no second barrier (no remote access after it)
  if (tid < kQTok) {
    float a = red[0][tid];
#pragma unroll
    for (int w = 1; w < kQThreads / 32; ++w) a = fmaxf(a, red[w][tid]);
    for (int r = 0; r < CL; ++r) cluster.map_shared_rank(&all_max[0][0], r)[rank * kQTok + tid] = a;
  }
  VLUT_STAMP(3);
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  VLUT_STAMP(4);
  if (tid < kQTok) {
    float a = 0.f;
    for (int r = 0; r < CL; ++r) a = fmaxf(a, all_max[r][tid]);
    const float sc = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
    s_scale[tid] = sc;
    if (rank == 0 && blockIdx.y * kQTok + tid < N) scale[blockIdx.y * kQTok + tid] = sc;
  }
  __syncthreads();
  VLUT_STAMP(5);
  float s[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) s[i] = s_scale[col * 4 + i];
#pragma unroll
  for (int i = 0; i < kQCache; ++i) {
    const int k = k_begin + rsub + kQRows * i;
    if (k < k_end && n < N) {
      const size_t o = (size_t)k * N + n;
      const int8_t c0 = q_code(cache[i].x, s[0]), c1 = q_code(cache[i].y, s[1]);
      const int8_t c2 = q_code(cache[i].z, s[2]), c3 = q_code(cache[i].w, s[3]);
      if (ALIGNED && n + 3 < N) {
        const uint32_t packed = (uint32_t)(uint8_t)c0 | ((uint32_t)(uint8_t)c1 << 8) |
                                ((uint32_t)(uint8_t)c2 << 16) | ((uint32_t)(uint8_t)c3 << 24);
        *reinterpret_cast<uint32_t*>(q + o) = packed;
      } else {
        const int8_t c[4] = {c0, c1, c2, c3};
        for (int t = 0; t < 4 && n + t < N; ++t) q[o + t] = c[t];
      }
    }
  }
  for (int k = k_begin + rsub + kQRows * kQCache; k < k_end; k += kQRows) {
    if (n >= N) break;
    const float4 a = q_load<ALIGNED>(x, y, k, N, n);
    const float v[4] = {a.x, a.y, a.z, a.w};
    for (int t = 0; t < 4 && n + t < N; ++t) q[(size_t)k * N + n + t] = q_code(v[t], s[t]);
  }
  VLUT_STAMP(6);
}

// ---------------------------------------------------------------- K3f: small-N (decode) quantizer
// K3 gives each cluster 16 tokens and each thread 4 tokens of a row: at
// decode (N = 1) three quarters of its threads idle and one cluster of 8
// CTAs walks K rows in many serial passes (K = 23040: ~15 us).  K3f treats
// [K][N] fp32 (token axis contiguous) as ONE flat array of K*N/4 float4s:
// lane i of the float4 at flat element e = 4f + i is token e mod N; every
// thread strides by a multiple of N/4 float4s, so its four lanes keep fixed
// tokens (4 tid + i) mod N (N in {1, 2, 4, 8, 16}).  One cluster of CL CTAs
// splits the flat array, every load is issued before any use (one DRAM round
// trip), maxima are reduced warp -> CTA (shared atomicMax on float bits:
// |x| >= 0 orders like unsigned) -> cluster (DSMEM push, as K3), and codes
// are written from registers: int8 [K][N] has the same flat order, so four
// codes are one 4-byte store.  Same IEEE ops as K3: identical codes/scales.
constexpr int kQfThreads = 512;
constexpr int kQfCache = 8;  // float4 per thread: <= 8 CTAs x 512 x 8 x 16 B = 512 KiB of x
constexpr int kQfMaxCL = 8;

template <bool HAS_Y>
__global__ void __launch_bounds__(kQfThreads)
    vlut_quantize_flat_kernel(const float* __restrict__ x, const float* __restrict__ y, int K,
                              int N, int8_t* __restrict__ q, float* __restrict__ scale) {
  __shared__ unsigned red[16];
  __shared__ float all_max[kQfMaxCL][16];  // [cluster rank][token]
  __shared__ float s_scale[16];
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31;
  const long long total4 = (long long)K * N / 4;
  // CTA slice [f0, f1) of float4s, f0 a multiple of kQfThreads (a multiple
  // of N/4), so a thread's token pattern does not depend on its CTA
  const long long per =
      ((total4 + CL - 1) / CL + kQfThreads - 1) / kQfThreads * kQfThreads;
  const long long f0 = (long long)rank * per;
  const long long f1 = min(total4, f0 + per);
  if (tid < 16) red[tid] = 0u;
  pdl_trigger_then_wait();
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4 c[kQfCache];
#pragma unroll
  for (int j = 0; j < kQfCache; ++j) {
    const long long f = f0 + tid + (long long)j * kQfThreads;
    c[j] = (f < f1) ? __ldg(x4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if constexpr (HAS_Y) {
    const float4* y4 = reinterpret_cast<const float4*>(y);
    float4 yc[kQfCache];
#pragma unroll
    for (int j = 0; j < kQfCache; ++j) {
      const long long f = f0 + tid + (long long)j * kQfThreads;
      yc[j] = (f < f1) ? __ldg(y4 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < kQfCache; ++j) c[j] = fmul4(c[j], yc[j]);
  }
  float m[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < kQfCache; ++j) {
    m[0] = fmaxf(m[0], fabsf(c[j].x)); m[1] = fmaxf(m[1], fabsf(c[j].y));
    m[2] = fmaxf(m[2], fabsf(c[j].z)); m[3] = fmaxf(m[3], fabsf(c[j].w));
  }
  // lanes l and l ^ d (d >= N/4) hold the same tokens
  const int pat = N >= 4 ? N / 4 : 1;  // distinct lane patterns
#pragma unroll
  for (int i = 0; i < 4; ++i)
    for (int d = pat; d < 32; d <<= 1) m[i] = fmaxf(m[i], __shfl_xor_sync(0xffffffffu, m[i], d));
  __syncthreads();  // red[] initialised
  if (lane < pat) {
#pragma unroll
    for (int i = 0; i < 4; ++i) atomicMax(red + (4 * lane + i) % N, __float_as_uint(m[i]));
  }
  __syncthreads();
  if (tid < N) {
    const float a = __uint_as_float(red[tid]);
    for (int r = 0; r < CL; ++r) cluster.map_shared_rank(&all_max[0][0], r)[rank * 16 + tid] = a;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tid < N) {
    float a = 0.f;
    for (int r = 0; r < CL; ++r) a = fmaxf(a, all_max[r][tid]);
    const float sc = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
    s_scale[tid] = sc;
    if (rank == 0) scale[tid] = sc;
  }
  __syncthreads();
  float s[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) s[i] = s_scale[(4 * tid + i) % N];
#pragma unroll
  for (int j = 0; j < kQfCache; ++j) {
    const long long f = f0 + tid + (long long)j * kQfThreads;
    if (f < f1) {
      const uint32_t packed = (uint32_t)(uint8_t)q_code(c[j].x, s[0]) |
                              ((uint32_t)(uint8_t)q_code(c[j].y, s[1]) << 8) |
                              ((uint32_t)(uint8_t)q_code(c[j].z, s[2]) << 16) |
                              ((uint32_t)(uint8_t)q_code(c[j].w, s[3]) << 24);
      reinterpret_cast<uint32_t*>(q)[f] = packed;
    }
  }
}

// ---------------------------------------------------------------- K3t: fused transposition (f3)
// Feature-major input (frameworks hold activations [N][K]; the
// transposition to the token-contiguous [K][N] int8 layout is fused into the
// quantization pass).  A cluster of CL CTAs owns 16 tokens, CTA `rank` a
// contiguous K slice.  Phase 1: each warp owns 2 tokens and reduces |x| over
// its slice with coalesced float4 loads along K; the per-token maxima are
// combined over the cluster (DSMEM).  Phase 2: the slice is re-read (L2),
// quantized and transposed through shared memory into 16-byte rows of q.
constexpr int kQtTok = 16;

__global__ void __launch_bounds__(256)
    vlut_quantize_t_kernel(const float* __restrict__ x, const float* __restrict__ y, int K, int N,
                           int8_t* __restrict__ q, float* __restrict__ scale) {
  extern __shared__ __align__(16) uint8_t qt_smem[];  // [slice][16] int8 codes
  __shared__ float cta_amax[kQtTok];
  __shared__ float s_scale[kQtTok];
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.y * kQtTok;
  const bool vec = ((K & 3) == 0) && ((((uintptr_t)x) | ((uintptr_t)(y ? y : x))) & 15) == 0;
  // K split in whole float4s when vectorised
  const int gran = vec ? 4 : 1;
  const int units = K / gran;
  const int k_begin = gran * (int)(((long long)rank * units) / CL);
  const int k_end = gran * (int)(((long long)(rank + 1) * units) / CL);
  pdl_trigger_then_wait();
  auto load = [&](int n, int k) -> float {
    const size_t o = (size_t)n * K + k;
    return y ? __fmul_rn(__ldg(x + o), __ldg(y + o)) : __ldg(x + o);
  };
  // ---- phase 1: per-token |x| max over this CTA's K slice
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int t = 2 * warp + h, n = n0 + t;
    float m = 0.f;
    if (n < N) {
      if (vec) {
        for (int k = k_begin + 4 * lane; k < k_end; k += 128) {
          const size_t o = (size_t)n * K + k;
          float4 a = __ldg(reinterpret_cast<const float4*>(x + o));
          if (y) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(y + o));
            a.x = __fmul_rn(a.x, b.x); a.y = __fmul_rn(a.y, b.y);
            a.z = __fmul_rn(a.z, b.z); a.w = __fmul_rn(a.w, b.w);
          }
          m = fmaxf(fmaxf(m, fabsf(a.x)), fmaxf(fabsf(a.y), fmaxf(fabsf(a.z), fabsf(a.w))));
        }
      } else {
        for (int k = k_begin + lane; k < k_end; k += 32) m = fmaxf(m, fabsf(load(n, k)));
      }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, d));
    if (lane == 0) cta_amax[t] = m;
  }
  cluster.sync();
  if (tid < kQtTok) {
    float a = 0.f;
    for (int r = 0; r < CL; ++r) a = fmaxf(a, cluster.map_shared_rank(cta_amax, r)[tid]);
    const float sc = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
    s_scale[tid] = sc;
    if (rank == 0 && n0 + tid < N) scale[n0 + tid] = sc;
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  // ---- phase 2: quantize into the shared [slice][16] tile (coalesced reads
  // along K per token), then 16-byte rows of q[k][n0 .. n0+15]
  const int slice = k_end - k_begin;
  for (int e = tid; e < slice * kQtTok; e += blockDim.x) {
    const int t = e / slice, kk = e - t * slice;
    const int n = n0 + t;
    int8_t c = 0;
    if (n < N) c = q_code(load(n, k_begin + kk), s_scale[t]);
    qt_smem[kk * kQtTok + t] = (uint8_t)c;
  }
  __syncthreads();
  const bool full16 = (n0 + kQtTok <= N) && ((N & 15) == 0) && ((((uintptr_t)q) & 15) == 0);
  for (int kk = tid; kk < slice; kk += blockDim.x) {
    int8_t* dst = q + (size_t)(k_begin + kk) * N + n0;
    if (full16) {
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(qt_smem + kk * kQtTok);
    } else {
      for (int t = 0; t < kQtTok && n0 + t < N; ++t) dst[t] = (int8_t)qt_smem[kk * kQtTok + t];
    }
  }
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}

// ---------------------------------------------------------------- K3a: quantize with known amax (f1)
// The per-token |x| maxima were produced by the producing GEMM's epilogue
// (vlut_mpgemm_fused), so quantization is one elementwise pass:
// s_n = amax_n / 127 (1 if 0), q = clamp(roundf(x / s_n), +-127).  4 tokens
// per thread (float4 in, 4 codes out), grid-stride.
__global__ void __launch_bounds__(256)
    vlut_quantize_amax_kernel(const float* __restrict__ x, const unsigned* __restrict__ amax,
                              int K, int N, int8_t* __restrict__ q, float* __restrict__ scale) {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int n4 = (N + 3) / 4;
  const long long total = (long long)K * n4;
  const bool vec = ((N & 3) == 0) && ((((uintptr_t)x) & 15) == 0) && ((((uintptr_t)q) & 3) == 0);
  const long long stride = (long long)gridDim.x * blockDim.x;
  constexpr int U = 4;  // units per thread and round: all loads issued before any use
  for (long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; e0 < total;
       e0 += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = e0 + u * stride;
      v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (vec && e < total) {
        const int k = (int)(e / n4), n = 4 * (int)(e % n4);
        v[u] = __ldg(reinterpret_cast<const float4*>(x + (size_t)k * N + n));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long e = e0 + u * stride;
      if (e >= total) break;
      const int k = (int)(e / n4), n = 4 * (int)(e % n4);
      float s[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = (n + i < N) ? __uint_as_float(__ldg(amax + n + i)) : 0.f;
        s[i] = (a == 0.f) ? 1.f : __fdiv_rn(a, 127.f);
      }
      if (k == 0)
        for (int i = 0; i < 4 && n + i < N; ++i) scale[n + i] = s[i];
      const size_t o = (size_t)k * N + n;
      if (vec) {
        const uint32_t packed = (uint32_t)(uint8_t)q_code(v[u].x, s[0]) |
                                ((uint32_t)(uint8_t)q_code(v[u].y, s[1]) << 8) |
                                ((uint32_t)(uint8_t)q_code(v[u].z, s[2]) << 16) |
                                ((uint32_t)(uint8_t)q_code(v[u].w, s[3]) << 24);
        *reinterpret_cast<uint32_t*>(q + o) = packed;
      } else {
        for (int i = 0; i < 4 && n + i < N; ++i) q[o + i] = q_code(__ldg(x + o + i), s[i]);
      }
    }
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ---------------------------------------------------------------- device packer (a1)
// One thread per payload byte [kt][m][j]: index = sum_r (w_r + 1) 3^r of
// group kt*16 + j of row m; padding -> the zero index.
__global__ void vlut_pack_kernel(const int8_t* __restrict__ w, int M, int K, int g, int m_pad,
                                 int kg_tiles, uint8_t* __restrict__ payload) {
  const long long total = (long long)kg_tiles * m_pad * 16;
  const int KG = (K + g - 1) / g;  // a partial last group (padded packing) reads zero trits
  const int zero = (g == 4) ? 40 : 121;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(e & 15);
    const long long rest = e >> 4;
    const int m = (int)(rest % m_pad);
    const int kt = (int)(rest / m_pad);
    const int k = kt * 16 + j;
    int idx = zero;
    if (m < M && k < KG) {
      const int8_t* src = w + (size_t)m * K + (size_t)k * g;
      idx = 0;
      int p3 = 1;
      for (int r = 0; r < g; ++r) {
        int t = (k * g + r < K) ? src[r] : 0;
        t = t < -1 ? -1 : (t > 1 ? 1 : t);
        idx += (t + 1) * p3;
        p3 *= 3;
      }
    }
    payload[e] = (uint8_t)idx;
  }
}

}  // namespace vlut
