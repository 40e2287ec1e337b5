// Split-K meeting cost at decode (development tool, not product code): how
// fast can C CTAs x 256 threads each add R partials into M distinct 64-bit
// words with atom.add.u64 (returning the old value, as K2's counted meeting
// does), alone and after streaming a 17.7 MB payload with per-thread loads?
// Graph of back-to-back launches over payload copies > 2x L2, mean per launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atom_floor atom_floor.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

// grid (S, MB): CTA (s, mb) owns rows [mb*256*R, (mb+1)*256*R) and K-tiles
// [s*T, (s+1)*T) of a [kt][M][16] payload; thread loads its R rows x T tiles
// up front (if LOAD), then adds one value per row into ws[row] (u64).
template <int R, int T, bool LOAD, bool RET>
__global__ void __launch_bounds__(256) meet_kernel(const uint4* __restrict__ pay, int M, int kgt,
                                                   unsigned long long* ws, uint32_t* sink) {
  const int s = blockIdx.x, mb = blockIdx.y;
  uint32_t acc[R];
#pragma unroll
  for (int q = 0; q < R; ++q) acc[q] = 1u;
  if (LOAD) {
    uint4 v[R][T];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int row = mb * 256 * R + q * 256 + threadIdx.x;
        const int kt = s * T + t;
        v[q][t] = (kt < kgt && row < M) ? __ldg(pay + (size_t)kt * M + row) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int q = 0; q < R; ++q)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[q] += (v[q][t].x ^ v[q][t].y ^ v[q][t].z ^ v[q][t].w) & 0xFF;
  }
  unsigned long long old[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int row = mb * 256 * R + q * 256 + threadIdx.x;
    old[q] = 0;
    if (row < M) {
      if (RET)
        asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old[q]) : "l"(ws + row), "l"((unsigned long long)acc[q]) : "memory");
      else
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(ws + row), "l"((unsigned long long)acc[q]) : "memory");
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int q = 0; q < R; ++q) x ^= (uint32_t)old[q];
  if (x == 0x12345679u) sink[0] = x;
}

int main() {
  const int M = 3072, kgt = 360;  // config 4, g = 4
  const size_t bytes = (size_t)kgt * M * 16;
  const int Rc = 18;
  std::vector<uint4*> bufs(Rc);
  for (auto& b : bufs) { CK(cudaMalloc(&b, bytes)); CK(cudaMemset(b, 1, bytes)); }
  unsigned long long* ws; CK(cudaMalloc(&ws, M * 8)); CK(cudaMemset(ws, 0, M * 8));
  uint32_t* sink; CK(cudaMalloc(&sink, 4));
  cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto time_graph = [&](auto launch_one) -> double {
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int r = 0; r < Rc; ++r) launch_one(r);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    std::vector<double> ts;
    for (int it = 0; it < 7; ++it) {
      CK(cudaEventRecord(e0, st)); CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ts.push_back(ms * 1e3 / Rc);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
  };
  auto run = [&](const char* name, auto kern, int R, int T) {
    dim3 grid((kgt + T - 1) / T, (M + 256 * R - 1) / (256 * R));
    double us = time_graph([&](int r) { kern<<<grid, 256, 0, st>>>(bufs[r], M, kgt, ws, sink); });
    printf("%-28s R=%d T=%d grid=%dx%d (%d CTAs, %d atomics): %6.2f us\n", name, R, T, grid.x, grid.y,
           grid.x * grid.y, grid.x * M, us);
  };
  run("atom only", meet_kernel<4, 2, false, true>, 4, 2);
  run("red only", meet_kernel<4, 2, false, false>, 4, 2);
  run("load only-ish (red)", meet_kernel<4, 2, true, false>, 4, 2);
  run("load + atom", meet_kernel<4, 2, true, true>, 4, 2);
  run("load + atom", meet_kernel<4, 4, true, true>, 4, 4);
  run("load + atom", meet_kernel<2, 4, true, true>, 2, 4);
  run("load + atom", meet_kernel<4, 3, true, true>, 4, 3);
  run("load + atom", meet_kernel<2, 2, true, true>, 2, 2);
  run("load + atom", meet_kernel<4, 8, true, true>, 4, 8);
  run("atom only", meet_kernel<4, 4, false, true>, 4, 4);
  run("atom only", meet_kernel<4, 8, false, true>, 4, 8);
  return 0;
}
