// smem_bw.cu -- K5 microbenchmark: achievable shared-memory LDS.128 bandwidth
// on this GPU for the Vec-LUT lookup pattern (data-dependent 128-byte rows,
// lane-rotated 16-byte chunks), with and without the SWAR accumulate work.
// Prints bytes/clk/SM from SM clock cycles and from wall time.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o smem_bw smem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

// MODE 0: LDS.128 + xor-reduce (minimal ALU); MODE 1: + per-word IADD3 into
// 32 SWAR accumulators like the kernel; ROWS: table rows; ITERS: groups.
template <int MODE>
__global__ void __launch_bounds__(512, 1) bw_kernel(int iters, uint32_t seed, unsigned long long* cyc,
                                                     uint32_t* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  for (int i = tid; i < 41 * 16 * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = i * 2654435761u;
  __syncthreads();
  uint32_t rot[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) rot[s] = ((lane + s) & 7) * 16;
  uint32_t sw[8][4];
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) sw[s][q] = 0;
  uint32_t x = seed ^ (tid * 747796405u);
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int g = 0; g < 16; g += 2) {
      x = x * 1664525u + 1013904223u;
      const uint32_t r0 = base + (g * 41 + ((x >> 8) % 41)) * 128;
      const uint32_t r1 = base + ((g + 1) * 41 + ((x >> 20) % 41)) * 128;
      uint4 v0[8], v1[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        v0[s] = lds128(r0 + rot[s]);
        v1[s] = lds128(r1 + rot[s]);
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (MODE == 0) {
          sw[s][0] ^= v0[s].x ^ v1[s].y;
        } else {
          sw[s][0] += v0[s].x + v1[s].x;
          sw[s][1] += v0[s].y + v1[s].y;
          sw[s][2] += v0[s].z + v1[s].z;
          sw[s][3] += v0[s].w + v1[s].w;
        }
      }
    }
  }
  const long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += sw[s][q];
  sink[blockIdx.x * blockDim.x + tid] = acc;
  if (tid == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int MODE>
void run(int threads, int iters, int sms) {
  const int smem = 41 * 16 * 128;
  cudaFuncSetAttribute(bw_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  cudaMalloc(&sink, sms * threads * 4);
  bw_kernel<MODE><<<sms, threads, smem>>>(10, 1, cyc, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bw_kernel<MODE><<<sms, threads, smem>>>(iters, 7, cyc, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[1024];
  cudaMemcpy(h, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mc = 0;
  for (int i = 0; i < sms; ++i) mc += h[i];
  mc /= sms;
  const double bytes_per_block = (double)threads * iters * 16 * 8 * 16;  // lanes*iters*groups*8 LDS*16B
  printf("mode=%d threads=%d: %.1f B/clk/SM (clock64), %.2f TB/s chip (wall %.3f ms), eff clk %.0f MHz\n",
         MODE, threads, bytes_per_block / mc, bytes_per_block * sms / (ms * 1e-3) / 1e12, ms,
         mc / (ms * 1e-3) / 1e6);
  cudaFree(cyc);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {256, 384, 512}) {
    run<0>(t, 2000, sms);
    run<1>(t, 2000, sms);
  }
  return 0;
}
