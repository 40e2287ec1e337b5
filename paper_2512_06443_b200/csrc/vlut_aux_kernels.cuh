// vlut_aux_kernels.cuh -- K3 per-token quantizer and the device-side packer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vlut {

// ---------------------------------------------------------------- K3 quantize (a7)
// One CTA owns 32 tokens (one warp-width of contiguous fp32 columns) and all K
// rows: pass 1 computes the per-token absmax (each warp strides over rows,
// 128-byte coalesced row segments, 8 loads in flight), pass 2 re-reads (from
// L2) and writes int8 codes.  IEEE single ops only (no fast math):
// s = amax / 127 (1 if amax == 0), q = clamp(roundf(x / s), -127, 127).
constexpr int kQuantWarps = 16;

__global__ void __launch_bounds__(kQuantWarps * 32)
    vlut_quantize_kernel(const float* __restrict__ x, const float* __restrict__ y, int K, int N,
                         int8_t* __restrict__ q, float* __restrict__ scale) {
  __shared__ float red[kQuantWarps][32];
  __shared__ float s_scale[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + lane;
  const bool ok = n < N;
  float amax = 0.f;
  if (ok) {
    int k = warp;
    for (; k + 7 * kQuantWarps < K; k += 8 * kQuantWarps) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const size_t o = (size_t)(k + i * kQuantWarps) * N + n;
        v[i] = y ? __fmul_rn(__ldg(x + o), __ldg(y + o)) : __ldg(x + o);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[i]));
    }
    for (; k < K; k += kQuantWarps) {
      const size_t o = (size_t)k * N + n;
      const float v = y ? __fmul_rn(__ldg(x + o), __ldg(y + o)) : __ldg(x + o);
      amax = fmaxf(amax, fabsf(v));
    }
  }
  red[warp][lane] = amax;
  __syncthreads();
  if (warp == 0) {
    float m = red[0][lane];
#pragma unroll
    for (int w = 1; w < kQuantWarps; ++w) m = fmaxf(m, red[w][lane]);
    const float s = (m == 0.f) ? 1.f : __fdiv_rn(m, 127.f);
    s_scale[lane] = s;
    if (ok) scale[n] = s;
  }
  __syncthreads();
  if (!ok) return;
  const float s = s_scale[lane];
  for (int k = warp; k < K; k += kQuantWarps) {
    const size_t o = (size_t)k * N + n;
    const float v = y ? __fmul_rn(__ldg(x + o), __ldg(y + o)) : __ldg(x + o);
    float r = roundf(__fdiv_rn(v, s));
    r = fminf(fmaxf(r, -127.f), 127.f);
    q[o] = (int8_t)r;
  }
}

// ---------------------------------------------------------------- device packer (a1)
// One thread per payload byte [kt][m][j]: index = sum_r (w_r + 1) 3^r of
// group kt*16 + j of row m; padding -> the zero index.
__global__ void vlut_pack_kernel(const int8_t* __restrict__ w, int M, int K, int g, int m_pad,
                                 int kg_tiles, uint8_t* __restrict__ payload) {
  const long long total = (long long)kg_tiles * m_pad * 16;
  const int KG = K / g;
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
        int t = src[r];
        t = t < -1 ? -1 : (t > 1 ? 1 : t);
        idx += (t + 1) * p3;
        p3 *= 3;
      }
    }
    payload[e] = (uint8_t)idx;
  }
}

}  // namespace vlut
