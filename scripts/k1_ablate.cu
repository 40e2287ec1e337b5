// k1_ablate.cu -- development ablation of K1's main loop on one B200:
// reuses the device functions of csrc/vlut_kernel.cuh (lookup_sub,
// build_tables, flush_tmem) on synthetic indices and measures shared-memory
// bytes/clk/SM for progressively more of the real loop:
//   mode 0: lookups only (12 lookup warps, random indices, XOR/IMAD negation)
//   mode 1: + FULL/EMPTY named-barrier handshake with 4 idle builder warps
//   mode 2: + builders really build the half tables (Gray walks, STS)
//   mode 3: + TMEM flush every 3 K-tiles
//   mode 4: + builders stage A and index tiles from HBM with cp.async (Params)
//   mode 5: + lookup warps take their indices from the staged tiles
// Ablations of single design choices:
//   mode 10: mode 0 with the naive chunk order (no lane rotation): the 8
//            lanes of an LDS.128 phase hit the same bank group
//   mode 11: mode 0 with plain int32 accumulation (every 16-bit field
//            widened on every lookup) instead of SWAR fields
//   mode 12: mode 2 with the vanilla table build (every row summed from its
//            g activations) instead of the topological walk
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o k1_ablate k1_ablate.cu
#include <cstdio>
#include "../paper_2512_06443_b200/csrc/vlut_kernel.cuh"

using namespace vlut;

// vanilla build: every half-table row of a group summed from
// scratch over its g trits (g-1 packed adds per row) instead of one add along
// the Gray walk; same rows, same stores
template <int G>
__device__ __forceinline__ void build_tables_vanilla(uint32_t tab_s, uint32_t a_s, int grp0, int bw,
                                                     int lane) {
  using CC = Cfg<G>;
  constexpr uint32_t K1 = 0x00010001u;
  constexpr uint32_t C128 = 128u * K1;
  for (int j = bw; j < CC::GS; j += kBuilderWarps) {
    uint32_t P[8], Mn[8];
#pragma unroll
    for (int r = 0; r < G; ++r) {
      const uint32_t x = lds_u16(a_s + ((grp0 + j) * G + r) * kNcta + 2 * lane);
      const uint32_t U = __byte_perm(x ^ 0x8080u, 0u, 0x4140);
      P[r] = U - C128;
      Mn[r] = C128 - U;
    }
    const uint32_t row0 = tab_s + (uint32_t)(j * CC::HR * kRowBytes) + 4 * lane;
#pragma unroll
    for (int pos = 0; pos < CC::HR; ++pos) {
      int idx = CC::ZERO + pos;  // upper half: idx >= zero
      uint32_t T = (uint32_t)CC::BIAS * K1;
#pragma unroll
      for (int r = 0; r < G; ++r) {
        const int d = idx % 3;
        idx /= 3;
        T += (d == 2) ? P[r] : ((d == 0) ? Mn[r] : 0u);
      }
      sts32(row0 + pos * kRowBytes, T);
    }
  }
}

// plain int32 accumulation: both 16-bit fields of every looked-up word are
// widened and added on every lookup (2 extra ops per word, 64 accumulators)
template <int G>
__device__ __forceinline__ void lookup_int32(uint32_t tab, const uint32_t (&iwa)[4],
                                             const uint32_t (&rot)[8], int32_t (&acc)[64]) {
  using CC = Cfg<G>;
#pragma unroll
  for (int b = 0; b < CC::GS; ++b) {
    const int i = (int)((iwa[b >> 2] >> (8 * (b & 3))) & CC::IDX_MASK);
    const int d = i - CC::ZERO;
    const int m = d >> 31;
    const uint32_t pos = (uint32_t)((d ^ m) - m);
    const uint32_t r = tab + (uint32_t)(b * CC::HR * kRowBytes) + pos * kRowBytes;
    uint4 v[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) v[s] = lds128(r + rot[s]);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const uint32_t w[4] = {v[s].x, v[s].y, v[s].z, v[s].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int lo = (int)(w[q] & 0xFFFFu) - CC::BIAS, hi = (int)(w[q] >> 16) - CC::BIAS;
        acc[8 * s + 2 * q] += m ? -lo : lo;
        acc[8 * s + 2 * q + 1] += m ? -hi : hi;
      }
    }
  }
}
constexpr int G = 4, W = 12;
using C = Cfg<G>;
constexpr int THREADS = (W + kBuilderWarps) * 32;
// staging buffers live after the tables (the kernel layout's IDX/A offsets,
// rebased so that they start at STAGE_BASE + IDX_OFF)
constexpr int STAGE_BASE = 2 * Cfg<G>::TAB_BYTES + Cfg<G>::A_BYTES + 64 - Layout<G, W>::IDX_OFF;

template <int MODE>
struct Mode {
  static constexpr bool HANDSHAKE = (MODE >= 1 && MODE <= 7) || MODE == 12;
  static constexpr bool BUILD = (MODE >= 2 && MODE <= 7);
  static constexpr bool VANILLA = MODE == 12;
  static constexpr bool FLUSH = MODE >= 3 && MODE <= 7;
  static constexpr bool STAGE = MODE >= 4 && MODE <= 7;
};

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) ablate(int ntiles, unsigned long long* cyc, uint32_t* sink,
                                                      Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t tab_s = smem_u32(smem);
  const uint32_t a_s = smem_u32(smem + 2 * C::TAB_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * C::TAB_BYTES + C::A_BYTES);
  const uint32_t mbar = smem_u32(smem + 2 * C::TAB_BYTES + C::A_BYTES + 16);
  if (tid == 32) {
    mbar_init(mbar + 0, kBuilderWarps); mbar_init(mbar + 8, kBuilderWarps);
    mbar_init(mbar + 16, W); mbar_init(mbar + 24, W);
  }
  for (int i = tid; i < (2 * C::TAB_BYTES + C::A_BYTES) / 4; i += THREADS)
    reinterpret_cast<uint32_t*>(smem)[i] = (i * 2654435761u) & 0x01FF01FFu;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)), "n"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const long long t0 = clock64();
  uint32_t out = 0;
  if (warp >= W) {
    const int bw = warp - W;
    for (int u = 0; u < ntiles + 2; ++u) {
      if (Mode<MODE>::HANDSHAKE && u >= 2) mbar_wait(mbar + 16 + 8 * (u & 1), ((u >> 1) - 1) & 1);
      if (u >= ntiles) continue;
      if (Mode<MODE>::STAGE) {
        if (u + 1 < ntiles) {
          if (MODE != 6) stage_tile<G, W>(p, u + 1, (u + 1) % kStageBufs, 0, 0, smem + STAGE_BASE, tid - W * 32, 3);
          if (MODE != 7) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
          if (MODE != 7) cp_async_wait_all();
        }
        if (MODE != 7) bar_sync(5, kBuilderWarps * 32);
      }
      if (Mode<MODE>::VANILLA) build_tables_vanilla<G>(tab_s + (u & 1) * C::TAB_BYTES, a_s, 0, bw, lane);
      else if (Mode<MODE>::BUILD) build_tables<G>(tab_s + (u & 1) * C::TAB_BYTES,
                                     MODE >= 4 ? smem_u32(smem + STAGE_BASE + Layout<G, W>::A_OFF + (u % kStageBufs) * C::A_BYTES) : a_s,
                                     0, bw, lane);
      if (Mode<MODE>::HANDSHAKE) { __syncwarp(); if (lane == 0) mbar_arrive(mbar + 8 * (u & 1)); }
    }
  } else {
    uint32_t rot[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) rot[s] = (uint32_t)((MODE == 10 ? s : ((lane + s) & 7)) * 16);
    int32_t acc32[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc32[i] = 0;
    const uint32_t taddr = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    uint32_t sw[8][4];
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int q = 0; q < 4; ++q) sw[s][q] = 0;
    int32_t nneg = 0;
    uint32_t x = 12345u + tid * 747796405u;
    int since = 0;
    bool first = true;
    for (int t = 0; t < ntiles; ++t) {
      if (Mode<MODE>::HANDSHAKE) mbar_wait(mbar + 8 * (t & 1), (t >> 1) & 1);
      uint32_t iwa[4];
      if (MODE == 5) {
        const uint4 iw = lds128(smem_u32(smem + STAGE_BASE + Layout<G, W>::IDX_OFF) + (t % kStageBufs) * Layout<G, W>::IDX_BYTES + tid * 16);
        iwa[0] = iw.x % 81u; iwa[1] = iw.y; iwa[2] = iw.z; iwa[3] = iw.w;
      } else
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x = x * 1664525u + 1013904223u;
        // four random indices in [0, 81)
        uint32_t w = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) w |= (((x >> (7 * b)) & 127u) % 81u) << (8 * b);
        iwa[i] = w;
      }
      if (MODE == 11) lookup_int32<G>(tab_s + (t & 1) * C::TAB_BYTES, iwa, rot, acc32);
      else lookup_sub<G>(0, tab_s + (t & 1) * C::TAB_BYTES, iwa, rot, sw, nneg);
      if (Mode<MODE>::HANDSHAKE) { __syncwarp(); if (lane == 0) mbar_arrive(mbar + 16 + 8 * (t & 1)); }
      if (Mode<MODE>::FLUSH && (++since == 3 || t + 1 == ntiles)) {
        since = 0;
        flush_tmem<G>(sw, nneg, taddr, first);
        first = false;
      }
    }
#pragma unroll
    for (int s = 0; s < 8; ++s)
#pragma unroll
      for (int q = 0; q < 4; ++q) out += sw[s][q];
#pragma unroll
    for (int i = 0; i < 64; ++i) out += (uint32_t)acc32[i];
  }
  const long long t1 = clock64();
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) {
    tmem_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(kTmemCols) : "memory");
  }
  sink[blockIdx.x * THREADS + tid] = out;
  if (tid == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE>
void run(int sms, int ntiles) {
  const int smem = 2 * C::TAB_BYTES + C::A_BYTES + 64 + 3 * Layout<G, W>::IDX_BYTES + 3 * C::A_BYTES;
  cudaFuncSetAttribute(ablate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, sms * 8);
  cudaMalloc(&sink, sms * THREADS * 4);
  // a real packed-index / activation stream in HBM (values random, in range)
  Params p = {};
  const int M = W * 32, K = ntiles * 16 * G, N = 64;
  uint8_t* payload; int8_t* A;
  cudaMalloc(&payload, (size_t)ntiles * M * 16);
  cudaMalloc(&A, (size_t)K * N);
  cudaMemset(payload, 40, (size_t)ntiles * M * 16);
  cudaMemset(A, 3, (size_t)K * N);
  p.payload = payload; p.A = A; p.M = M; p.K = K; p.N = N; p.m_pad = M; p.kg_tiles = ntiles;
  p.splits = 1; p.a_vec = 16; p.out_vec4 = 1;
  ablate<MODE><<<sms, THREADS, smem>>>(4, cyc, sink, p);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  ablate<MODE><<<sms, THREADS, smem>>>(ntiles, cyc, sink, p);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mc = 0;
  for (int i = 0; i < sms; ++i) mc += h[i];
  mc /= sms;
  const double lookup_bytes = (double)W * 32 * ntiles * 16 * 128;  // rows x groups x 128 B
  const double build_bytes = (Mode<MODE>::BUILD || Mode<MODE>::VANILLA) ? (double)ntiles * 16 * C::HR * 128 : 0;
  printf("mode=%d: lookups %.1f B/clk/SM, lookups+build %.1f B/clk/SM  (%.3f ms, %.0f MHz) err=%s\n",
         MODE, lookup_bytes / mc, (lookup_bytes + build_bytes) / mc, ms, mc / (ms * 1e-3) / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms, 400);
  run<1>(sms, 400);
  run<2>(sms, 400);
  run<3>(sms, 400);
  run<4>(sms, 400);
  run<5>(sms, 400);
  run<6>(sms, 400);
  run<7>(sms, 400);
  run<10>(sms, 400);
  run<11>(sms, 400);
  run<12>(sms, 400);
  return 0;
}
