// HBM read floor for the decode point (development tool, not product code):
// how long does one kernel need just to READ config 4's packed weights
// (3072 x 5760 B = 17.7 MB at g = 4) from HBM?  That is the practical bound
// for K2 at N = 1.  Variants, each timed as a CUDA graph of R back-to-back
// launches over R distinct copies (R x 17.7 MB > 2x the 126 MB L2, so every
// launch streams from HBM), per-launch mean:
//   ldg  : grid = 148 x k CTAs, 256 threads, unrolled ld.global.nc.v4 (8 per
//          thread in flight), xor-reduce so the loads are live
//   bulk : one CTA per SM, cp.async.bulk chunks into a shared-memory ring,
//          S stages of C bytes, mbarrier per stage (K2's staging shape)
//   pdl  : the bulk variant launched with programmatic stream serialisation,
//          each kernel triggering its dependents at entry (a decode chain of
//          independent weight streams overlapping each other's tails)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_floor hbm_floor.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n16, uint32_t* sink) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  size_t i = tid;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = __ldg(p + i); acc ^= v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x12345679u) sink[0] = acc;
}

// CTA b reads its contiguous chunk [b*per, (b+1)*per); every thread issues
// all U of its 16-byte loads before using any (K2's "whole share up front")
template <int U>
__global__ void ldg_chunk_kernel(const uint4* __restrict__ p, size_t n16, uint32_t* sink) {
  const size_t per = (size_t)U * blockDim.x;
  const size_t b0 = blockIdx.x * per;
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const size_t i = b0 + (size_t)u * blockDim.x + threadIdx.x;
    v[u] = i < n16 ? __ldg(p + i) : make_uint4(0, 0, 0, 0);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  if (acc == 0x12345679u) sink[0] = acc;
}

// K2's decode pattern: CTA (s, mb) reads rows [mb*1024, +1024) of K-tiles
// [s*T, (s+1)*T) of a [kt][M][16] payload; thread = 2 rows (tid, tid+512).
// CP: cp.async into shared memory (one group, wait all); else LDG to regs.
template <bool CP, int T>
__global__ void __launch_bounds__(512) k2pat_kernel(const uint8_t* __restrict__ pay, int M, int kgt,
                                                    uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int s = blockIdx.x, mb = blockIdx.y;
  uint32_t acc = 0;
  if (CP) {
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = q * 512 + threadIdx.x;
        const int kt = s * T + t, row = mb * 1024 + r;
        if (kt < kgt && row < M) {
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + ((size_t)t * 1024 + r) * 16);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(pay + ((size_t)kt * M + row) * 16) : "memory");
        }
      }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(sm + ((size_t)t * 1024 + q * 512 + threadIdx.x) * 16);
        acc ^= v.x ^ v.w;
      }
  } else {
    uint4 v[T][2];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int kt = s * T + t, row = mb * 1024 + q * 512 + threadIdx.x;
        v[t][q] = (kt < kgt && row < M) ? __ldg(reinterpret_cast<const uint4*>(pay + ((size_t)kt * M + row) * 16))
                                        : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < 2; ++q) acc ^= v[t][q].x ^ v[t][q].w;
  }
  if (acc == 0x12345679u) sink[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W;\n}" :: "r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

// one CTA per SM; CTA b reads bytes [b*per, (b+1)*per) in chunks of C through
// S stages.  Warp 0 lane 0 produces, all 4 warps consume (xor over the chunk).
template <bool PDL>
__global__ void bulk_kernel(const uint8_t* __restrict__ p, size_t total, int C, int S, uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 32;
  uint8_t* ring = sm + 512;
  if (PDL) asm volatile("griddepcontrol.launch_dependents;");
  size_t per = (total + gridDim.x - 1) / gridDim.x;
  per = (per + 15) & ~(size_t)15;
  size_t beg = blockIdx.x * per, end = min(total, beg + per);
  int nch = beg >= end ? 0 : (int)((end - beg + C - 1) / C);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], blockDim.x / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < min(nch, S); ++c) {
      uint32_t bytes = (uint32_t)min((size_t)C, end - (beg + (size_t)c * C));
      mbar_expect(&full[c], bytes);
      bulk_g2s(ring + (size_t)c * C, p + beg + (size_t)c * C, bytes, &full[c]);
    }
  }
  uint32_t acc = 0;
  for (int c = 0; c < nch; ++c) {
    int s = c % S;
    uint32_t ph = (c / S) & 1;
    mbar_wait(&full[s], ph);
    uint32_t bytes = (uint32_t)min((size_t)C, end - (beg + (size_t)c * C));
    const uint4* q = (const uint4*)(ring + (size_t)s * C);
    for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) { uint4 v = q[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(&empty[s])) : "memory");
    if (threadIdx.x == 0 && c + S < nch) {
      mbar_wait(&empty[s], ph);
      int cn = c + S;
      uint32_t nb = (uint32_t)min((size_t)C, end - (beg + (size_t)cn * C));
      mbar_expect(&full[s], nb);
      bulk_g2s(ring + (size_t)s * C, p + beg + (size_t)cn * C, nb, &full[s]);
    }
  }
  if (acc == 0x12345679u) sink[0] = acc;
}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? (size_t)atof(argv[1]) : (size_t)3072 * 5760;
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int R = (int)std::max<size_t>(4, (300u << 20) / bytes + 1);
  std::vector<uint8_t*> bufs(R);
  for (auto& b : bufs) { CK(cudaMalloc(&b, bytes)); CK(cudaMemset(b, 1, bytes)); }
  uint32_t* sink; CK(cudaMalloc(&sink, 4));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  printf("bytes %zu (%.2f MB), copies %d (%.0f MB), SMs %d\n", bytes, bytes / 1e6, R, R * bytes / 1e6, nsm);

  auto time_graph = [&](auto launch_one) -> double {
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int r = 0; r < R; ++r) launch_one(r);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    std::vector<double> ts;
    for (int it = 0; it < 7; ++it) {
      CK(cudaEventRecord(e0, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms * 1e3 / R);
    }
    std::sort(ts.begin(), ts.end());
    CK(cudaGraphExecDestroy(ge)); CK(cudaGraphDestroy(g));
    return ts[ts.size() / 2];
  };
  auto report = [&](const char* name, double us) {
    printf("%-34s %7.2f us  %6.0f GB/s\n", name, us, bytes / us / 1e3);
  };

  for (int k : {1, 2, 4, 8, 16}) {
    for (int thr : {256, 512}) {
      double us = time_graph([&](int r) {
        ldg_kernel<<<nsm * k, thr, 0, st>>>((const uint4*)bufs[r], bytes / 16, sink);
      });
      char nm[64]; snprintf(nm, 64, "ldg grid=%dx%d thr=%d", nsm, k, thr); report(nm, us);
    }
  }
  {
    const size_t n16 = bytes / 16;
    auto chunk = [&](auto Uc, int thr) {
      constexpr int U = decltype(Uc)::value;
      const int grid = (int)((n16 + (size_t)U * thr - 1) / ((size_t)U * thr));
      double us = time_graph([&](int r) {
        ldg_chunk_kernel<U><<<grid, thr, 0, st>>>((const uint4*)bufs[r], n16, sink);
      });
      char nm[64]; snprintf(nm, 64, "ldg-chunk U=%d thr=%d grid=%d", U, thr, grid); report(nm, us);
    };
    chunk(std::integral_constant<int, 16>{}, 512);
    chunk(std::integral_constant<int, 8>{}, 1024);
    chunk(std::integral_constant<int, 8>{}, 512);
    chunk(std::integral_constant<int, 4>{}, 512);
    chunk(std::integral_constant<int, 4>{}, 256);
    chunk(std::integral_constant<int, 16>{}, 256);
    chunk(std::integral_constant<int, 32>{}, 256);
  }
  CK(cudaFuncSetAttribute(bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(bulk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (int C : {2048, 4096, 8192, 16384, 32768}) {
    for (int S : {2, 4, 6, 16, 32}) {
      if ((size_t)C * S + 512 > 220 * 1024) continue;
      for (int pdl = 0; pdl < 2; ++pdl) {
        double us = time_graph([&](int r) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(nsm); cfg.blockDim = dim3(128);
          cfg.dynamicSmemBytes = (size_t)C * S + 512; cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
          if (pdl) CK(cudaLaunchKernelEx(&cfg, bulk_kernel<true>, (const uint8_t*)bufs[r], bytes, C, S, sink));
          else CK(cudaLaunchKernelEx(&cfg, bulk_kernel<false>, (const uint8_t*)bufs[r], bytes, C, S, sink));
        });
        char nm[64]; snprintf(nm, 64, "bulk C=%d S=%d%s", C, S, pdl ? " pdl" : ""); report(nm, us);
      }
    }
  }
  // 2 CTAs per SM (smaller rings)
  for (int C : {8192, 16384}) {
    int S = 4;
    double us = time_graph([&](int r) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nsm * 2); cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = (size_t)C * S + 512; cfg.stream = st;
      CK(cudaLaunchKernelEx(&cfg, bulk_kernel<false>, (const uint8_t*)bufs[r], bytes, C, S, sink));
    });
    char nm[64]; snprintf(nm, 64, "bulk 2/SM C=%d S=%d", C, S); report(nm, us);
  }
  // K2's decode access pattern (config 4 g = 4 only: 3072 rows x 360 K-tiles)
  if (bytes == (size_t)3072 * 5760) {
    auto k2 = [&](auto CPc, auto Tc) {
      constexpr bool CP = decltype(CPc)::value;
      constexpr int T = decltype(Tc)::value;
      const int smem = CP ? T * 1024 * 16 : 0;
      CK(cudaFuncSetAttribute(k2pat_kernel<CP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      dim3 grid((360 + T - 1) / T, 3);
      double us = time_graph([&](int r) { k2pat_kernel<CP, T><<<grid, 512, smem, st>>>(bufs[r], 3072, 360, sink); });
      char nm[64]; snprintf(nm, 64, "k2-pattern %s T=%d (%d CTAs)", CP ? "cp.async" : "ldg", T, grid.x * 3); report(nm, us);
    };
    // the same loads with a large dynamic shared-memory allocation (less L1)
    for (int sk : {0, 64, 128, 160, 200, 220}) {
      CK(cudaFuncSetAttribute(k2pat_kernel<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      dim3 grid(45, 3);
      double us = time_graph([&](int r) { k2pat_kernel<false, 8><<<grid, 512, sk * 1024, st>>>(bufs[r], 3072, 360, sink); });
      char nm[64]; snprintf(nm, 64, "k2-pattern ldg T=8 smem=%dKB", sk); report(nm, us);
    }
    for (int sk : {128, 160, 200, 220}) {
      CK(cudaFuncSetAttribute(k2pat_kernel<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      dim3 grid(45, 3);
      double us = time_graph([&](int r) { k2pat_kernel<true, 8><<<grid, 512, sk * 1024, st>>>(bufs[r], 3072, 360, sink); });
      char nm[64]; snprintf(nm, 64, "k2-pattern cp.async T=8 smem=%dKB", sk); report(nm, us);
    }
    k2([]{ return std::false_type{}; }(), std::integral_constant<int, 8>{});
    k2(std::true_type{}, std::integral_constant<int, 8>{});
    k2(std::false_type{}, std::integral_constant<int, 4>{});
    k2(std::true_type{}, std::integral_constant<int, 4>{});
    k2(std::false_type{}, std::integral_constant<int, 2>{});
    k2(std::true_type{}, std::integral_constant<int, 2>{});
  }
  // empty-kernel launch floor in the same graph form
  double us = time_graph([&](int r) { ldg_kernel<<<nsm, 256, 0, st>>>((const uint4*)bufs[r], 0, sink); });
  report("empty (n=0) launch", us);
  return 0;
}
