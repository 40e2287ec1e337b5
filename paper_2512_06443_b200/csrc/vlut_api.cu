// vlut_api.cu -- host side of libvlut.so: argument validation, the weight
// packer (a1), the launch planner and the launches.  See include/vlut.h for
// the contract of every entry point.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/vlut.h"
#include "vlut_aux_kernels.cuh"
#include "vlut_kernel.cuh"
#include "vlut_kernel32.cuh"
#include "vlut_kernel32_sk.cuh"
#include "vlut_kernel_sk.cuh"
#include "vlut_kernel_slot.cuh"
#include <atomic>

namespace {

thread_local std::string g_err;

// Peer destinations of the next launch (vlut_mpgemm_allgather -> run_mpgemm),
// thread-local so concurrent callers on other threads are unaffected.
struct PeerTls {
  int n = 0;
  int mc = 0;  // the output pointer is a multicast address
  float* ptr[vlut::kMaxPeers] = {};
};
thread_local PeerTls g_peer_tls;

vlut_status fail(vlut_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

vlut_status ok() {
  g_err.clear();
  return VLUT_OK;
}

#define VLUT_CUDA_TRY(expr)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(VLUT_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));        \
  } while (0)

struct DeviceInfo {
  bool init = false;
  int sms = 0;
  int smem_optin = 0;
  int cc_major = 0, cc_minor = 0;
};

std::mutex g_mu;
DeviceInfo g_dev[64];

vlut_status device_info(DeviceInfo* out) {
  int dev = 0;
  VLUT_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(VLUT_ERR_CUDA, "device ordinal %d out of range", dev);
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceInfo& d = g_dev[dev];
  if (!d.init) {
    VLUT_CUDA_TRY(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    VLUT_CUDA_TRY(
        cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    VLUT_CUDA_TRY(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    VLUT_CUDA_TRY(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    d.init = true;
  }
  *out = d;
  return VLUT_OK;
}

inline bool valid_g(int g) { return g == 4 || g == 5; }

inline int pow3i(int g) { return g == 4 ? 81 : 243; }

bool layout_of(int M, int K, int g, int flags, int* m_pad, int* kg_tiles, size_t* bytes) {
  if (M <= 0 || K <= 0 || !valid_g(g) || (flags & ~VLUT_PACK_PAD_K)) return false;
  if (K % g && !(flags & VLUT_PACK_PAD_K)) return false;
  const long long mp = ((long long)M + VLUT_M_TILE - 1) / VLUT_M_TILE * VLUT_M_TILE;
  const long long kgt = ((long long)((K + g - 1) / g) + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const long long b = kgt * mp * 16;
  if (mp > (1LL << 30) || kgt > (1LL << 30) || b <= 0) return false;
  *m_pad = (int)mp;
  *kg_tiles = (int)kgt;
  *bytes = (size_t)b;
  return true;
}

vlut_status check_desc(const vlut_packed_weights* W, int M, int K) {
  if (!W) return fail(VLUT_ERR_INVALID_ARGUMENT, "W descriptor is NULL");
  if (W->magic != VLUT_MAGIC || W->version != VLUT_VERSION)
    return fail(VLUT_ERR_CORRUPT_DESCRIPTOR, "bad descriptor magic/version");
  int mp = 0, kgt = 0;
  size_t bytes = 0;
  if (!layout_of(W->M, W->K, W->g, W->flags, &mp, &kgt, &bytes) || W->m_pad != mp ||
      W->kg_tiles != kgt || W->payload_bytes != (int64_t)bytes || W->m_tile != VLUT_M_TILE ||
      W->kg_tile != VLUT_KG_TILE || !W->payload)
    return fail(VLUT_ERR_CORRUPT_DESCRIPTOR, "descriptor fields inconsistent");
  if (((uintptr_t)W->payload) & 15) return fail(VLUT_ERR_MISALIGNED, "payload not 16-B aligned");
  if (W->M != M || W->K != K)
    return fail(VLUT_ERR_SHAPE, "shape (M=%d,K=%d) does not match descriptor (M=%d,K=%d)", M,
                K, W->M, W->K);
  return VLUT_OK;
}

// ------------------------------------------------------------ TMA descriptor
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

vlut_status encode_a_map(CUtensorMap* map, const int8_t* A, int K, int N, int g,
                         int box_n = vlut::kNcta) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  static cudaError_t get_err = cudaSuccess;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    get_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (get_err == cudaSuccess && q == cudaDriverEntryPointSuccess) fn = (EncodeTiledFn)f;
  });
  if (!fn) return fail(VLUT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(get_err));
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
  const cuuint64_t strides[1] = {(cuuint64_t)N};
  const cuuint32_t box[2] = {(cuuint32_t)box_n, (cuuint32_t)(vlut::kKgTile * g)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)A, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VLUT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return VLUT_OK;
}

// 3-D view of A for K1-32: dims (N tokens, K/g groups, g rows of a group),
// strides (g*N, N) bytes -- the box (32, 16, g) lands in shared memory as
// [r][group][token] (conflict-free builder loads, vlut_kernel32.cuh)
vlut_status encode_a_map3d(CUtensorMap* map, const int8_t* A, int K, int N, int g,
                           int box_n = vlut::kN32) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  });
  if (!fn) return fail(VLUT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)(K / g), (cuuint64_t)g};
  const cuuint64_t strides[2] = {(cuuint64_t)g * N, (cuuint64_t)N};
  const cuuint32_t box[3] = {(cuuint32_t)box_n, (cuuint32_t)vlut::kKgTile, (cuuint32_t)g};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)A, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(VLUT_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
  return VLUT_OK;
}

// ------------------------------------------------------------ planner
int smem_bytes_for(int g, int warps, int rpt = 1) {
  if (rpt == 2) {
    if (warps == 8) return g == 4 ? vlut::Layout<4, 8, 2>::SMEM : vlut::Layout<5, 8, 2>::SMEM;
    return g == 4 ? vlut::Layout<4, 12, 2>::SMEM : vlut::Layout<5, 12, 2>::SMEM;
  }
  if (g == 4) {
    if (warps == 8) return vlut::Layout<4, 8>::SMEM;
    if (warps == 12) return vlut::Layout<4, 12>::SMEM;
    return vlut::Layout<4, 16>::SMEM;
  }
  if (warps == 8) return vlut::Layout<5, 8>::SMEM;
  if (warps == 12) return vlut::Layout<5, 12>::SMEM;
  return vlut::Layout<5, 16>::SMEM;
}

// ------------------------------------------------------------ occupancy
template <int G, int WARPS, bool ACC>
cudaError_t prepare_kernel() {
  using L = vlut::Layout<G, WARPS>;
  static std::once_flag flags[64];
  static cudaError_t errs[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::call_once(flags[dev & 63], [&] {
    errs[dev & 63] = cudaFuncSetAttribute(vlut::vlut_mpgemm_kernel<G, WARPS, ACC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  });
  return errs[dev & 63];
}

// Co-resident clusters of size S for a variant (cudaOccupancyMaxActiveClusters,
// cached per device): clusters larger than 2 can strand SMs of a GPC.
template <int G, int WARPS>
int active_clusters(int S) {
  using L = vlut::Layout<G, WARPS>;
  static std::mutex mu;
  static int cache[64][9];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || S < 1 || S > 8) return 0;
  std::lock_guard<std::mutex> lk(mu);
  int& c = cache[dev & 63][S];
  if (c == 0) {
    if (prepare_kernel<G, WARPS, false>() != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)S, 1, 1);
    cfg.blockDim = dim3(L::THREADS, 1, 1);
    cfg.dynamicSmemBytes = L::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, vlut::vlut_mpgemm_kernel<G, WARPS, false>, &cfg) !=
            cudaSuccess ||
        n <= 0) {
      cudaGetLastError();
      n = -1;  // cluster size unusable
    }
    c = n;
  }
  return c;
}

// K1-32 (32-token tiles): kernel attribute + co-resident clusters
template <int G, int WARPS, bool ACC>
cudaError_t prepare_kernel32() {
  using L = vlut::Layout32<G, WARPS>;
  static std::once_flag flags[64];
  static cudaError_t errs[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::call_once(flags[dev & 63], [&] {
    errs[dev & 63] = cudaFuncSetAttribute(vlut::vlut_mpgemm32_kernel<G, WARPS, ACC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  });
  return errs[dev & 63];
}

template <int G, int WARPS>
int active_clusters32(int S) {
  using L = vlut::Layout32<G, WARPS>;
  static std::mutex mu;
  static int cache[64][9];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || S < 1 || S > 8) return 0;
  std::lock_guard<std::mutex> lk(mu);
  int& c = cache[dev & 63][S];
  if (c == 0) {
    if (prepare_kernel32<G, WARPS, false>() != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)S, 1, 1);
    cfg.blockDim = dim3(L::THREADS, 1, 1);
    cfg.dynamicSmemBytes = L::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, vlut::vlut_mpgemm32_kernel<G, WARPS, false>, &cfg) !=
            cudaSuccess ||
        n <= 0) {
      cudaGetLastError();
      n = -1;
    }
    c = n;
  }
  return c;
}

int active_clusters32_for(int g, int warps, int S) {
  if (g == 4) {
    if (warps == 8) return active_clusters32<4, 8>(S);
    if (warps == 12) return active_clusters32<4, 12>(S);
    return active_clusters32<4, 16>(S);
  }
  if (warps == 8) return active_clusters32<5, 8>(S);
  if (warps == 12) return active_clusters32<5, 12>(S);
  return active_clusters32<5, 16>(S);
}

int smem_bytes32_for(int g, int warps) {
  if (g == 4)
    return warps == 8 ? vlut::Layout32<4, 8>::SMEM
                      : (warps == 12 ? vlut::Layout32<4, 12>::SMEM : vlut::Layout32<4, 16>::SMEM);
  return warps == 8 ? vlut::Layout32<5, 8>::SMEM
                    : (warps == 12 ? vlut::Layout32<5, 12>::SMEM : vlut::Layout32<5, 16>::SMEM);
}

int active_clusters_for(int g, int warps, int S) {
  if (g == 4) {
    if (warps == 8) return active_clusters<4, 8>(S);
    if (warps == 12) return active_clusters<4, 12>(S);
    return active_clusters<4, 16>(S);
  }
  if (warps == 8) return active_clusters<5, 8>(S);
  if (warps == 12) return active_clusters<5, 12>(S);
  return active_clusters<5, 16>(S);
}

inline bool valid_split(int warps, int S) { return warps > 0 && S >= 1 && S <= 8; }

// Workspace layout (caller-provided, zeroed once):
//   [0, SK)             stream-K int32 partials [sms][768 x 64] (m_cta <= 768)
//   [SK, SK + 4096)     stream-K partial-ready flags (0 between launches)
//   [.., + 64 KB)       K2 split-K arrival counters (kept zero between launches)
//   [.., + 16 MB)       K2 split-K int32 accumulators [M][N] (kept zero)
size_t sk_part_bytes(int sms) { return (size_t)sms * 768 * 64 * 4; }  // max m_cta 768
size_t slot_cnt_off(int sms) { return sk_part_bytes(sms) + 4096; }
size_t slot_acc_off(int sms) { return slot_cnt_off(sms) + (size_t)vlut::slot::kMaxCounters * 8; }
constexpr size_t kSlotAccBytes = (size_t)16 << 20;
size_t sk32_acc_off(int sms) { return slot_acc_off(sms) + kSlotAccBytes; }
// K1-32-SK fp32 split-tile accumulators: one [768][32] slot per CTA, zero between launches
size_t sk_workspace_bytes(int sms) { return sk32_acc_off(sms) + (size_t)sms * 768 * 32 * 4; }

// Best stream-K plan (persistent, grid = #SMs): every CTA gets ceil(U / sms)
// K-tile units; cost in the same SMEM-cycle units as plan_for.
double plan_sk(int M, int K, int N, int g, int sms, vlut_launch_plan* best) {
  const int KG = (K + g - 1) / g;  // padded packing: the last group may be partial
  const int kgt = (KG + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const int NT = (N + vlut::kNcta - 1) / vlut::kNcta;
  const int half_rows = (pow3i(g) + 1) / 2;
  double best_cost = 1e300;
  // (warps, rows per lookup thread): 12 warps x 2 rows = 768 rows share each table
  const int warps_opts[5] = {16, 12, 8, 12, 8};
  const int rpt_opts[5] = {1, 1, 1, 2, 2};
  for (int wi = 0; wi < 5; ++wi) {
    const int warps = warps_opts[wi];
    const int rpt = rpt_opts[wi];
    if (rpt == 2 && getenv("VLUT_NO_RPT2")) continue;
    const int mcta = 32 * warps * rpt;
    const long long MT = (M + mcta - 1) / mcta;
    const long long U = MT * NT * kgt;
    const long long grid = U < sms ? U : sms;
    const double units = (double)((U + grid - 1) / grid);
    // two rows per thread, relative cost per lookup row (measured against 16
    // warps x 1 row, scripts/rpt_ab.py): 12 warps with one group per load
    // batch keep the pipe ~5 % less busy at g = 4 (~1 % at g = 5); 8 warps
    // with two groups per batch ~8 % less at g = 4 and ~1 % more at g = 5
    const double row_cost =
        rpt == 2 ? (warps == 8 ? (g == 4 ? 1.08 : 0.99) : (g == 4 ? 1.05 : 1.01)) : 1.0;
    double cost = units * VLUT_KG_TILE * ((double)mcta * row_cost + half_rows);
    cost += 6000.0;                             // start + last epilogue
    cost += (double)mcta * 256.0 * 3.0 / 64.0;  // partial write + read + output
    // the owner of a split tile reads every producer's int32 partial
    // (mcta x 64 x 4 B) one after another at ~64 B/clk: with few tiles a
    // tile is split over many CTAs and this serial fixup dominates
    const double per_tile = (double)grid / (double)(MT * NT);
    if (per_tile > 1.0) cost += (per_tile - 1.0) * (double)mcta * 256.0 / 64.0;
    if (cost < best_cost * 0.995) {
      best_cost = cost;
      best->warps = warps;
      best->splits = 1;
      best->m_cta = mcta;
      best->n_cta = vlut::kNcta;
      best->grid_ctas = (int)grid;
      best->smem_bytes = smem_bytes_for(g, warps, rpt);
      best->streamk = 1;
    }
  }
  return best_cost;
}

// Cost model in shared-memory cycles (DESIGN.md §4 planner):
//   per K-tile   16 groups x (m_cta lookup rows + (3^g+1)/2 half-table rows)
//                (one 128-B wavefront per row and group)
//   per CTA      tiles x per-tile + fixed start/epilogue + DSMEM reduction of
//                (S-1)/S of the m_cta x 256 B int32 tile at ~16 B/clk
//   total        waves x per-CTA, waves = ceil(CTAs / (active clusters x S))
double plan_for(int M, int K, int N, int g, int sms, vlut_launch_plan* best) {
  const int KG = (K + g - 1) / g;  // padded packing: the last group may be partial
  const int kgt = (KG + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const int NT = (N + vlut::kNcta - 1) / vlut::kNcta;
  const int half_rows = (pow3i(g) + 1) / 2;
  double best_cost = 1e300;
  const int warps_opts[3] = {16, 12, 8};
  const int split_opts[8] = {1, 2, 3, 4, 5, 6, 7, 8};
  for (int wi = 0; wi < 3; ++wi) {
    const int warps = warps_opts[wi];
    const int mcta = 32 * warps;
    const long long MT = (M + mcta - 1) / mcta;
    for (int si = 0; si < 8; ++si) {
      const int S = split_opts[si];
      if (!valid_split(warps, S) || S > kgt) continue;
      const long long ctas = MT * NT * S;
      if (ctas > 65535LL * 65535LL) continue;
      int clusters = active_clusters_for(g, warps, S);
      if (clusters < 0) continue;
      if (clusters == 0) clusters = sms / S;  // no device query possible
      const long long slots = (long long)clusters * S;
      if (slots <= 0) continue;
      const long long waves = (ctas + slots - 1) / slots;
      const double tiles = (double)((kgt + S - 1) / S);
      double per_cta = tiles * VLUT_KG_TILE * (double)(mcta + half_rows);
      per_cta += 6000.0;  // start (first tile + table) and epilogue
      if (S > 1) per_cta += (double)(S - 1) / S * mcta * 256.0 / 16.0;
      const double cost = waves * per_cta;
      if (cost < best_cost * 0.995) {
        best_cost = cost;
        best->warps = warps;
        best->splits = S;
        best->m_cta = mcta;
        best->n_cta = vlut::kNcta;
        best->grid_ctas = (int)ctas;
        best->smem_bytes = smem_bytes_for(g, warps);
        best->streamk = 0;
      }
    }
  }
  return best_cost;
}

// K1-32 (32-token tiles, paired-group tables): the same shared-memory cycle
// units as plan_for -- a 32-token row is half a 128-byte wavefront -- with
// the lookup path's extra ALU work (per-lane line selection) charged as a
// factor, a cheaper epilogue (no DSMEM exchange at splits = 1) and the
// DSMEM reduction of 128-byte rows when split.
#ifndef VLUT_K32_FACTOR
#define VLUT_K32_FACTOR 1.00
#endif
double plan_for32(int M, int K, int N, int g, int sms, vlut_launch_plan* best) {
  const int KG = (K + g - 1) / g;
  const int kgt = (KG + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const int NT = (N + vlut::kN32 - 1) / vlut::kN32;
  const int half_rows = (pow3i(g) + 1) / 2;
  double best_cost = 1e300;
  if (getenv("VLUT_NO_K32")) return best_cost;
  const int warps_opts[3] = {16, 12, 8};
  for (int wi = 0; wi < 3; ++wi) {
    const int warps = warps_opts[wi];
    const int mcta = 32 * warps;
    const long long MT = (M + mcta - 1) / mcta;
    for (int S = 1; S <= 8; ++S) {
      if (S > kgt) continue;
      const long long ctas = MT * NT * S;
      if (ctas > 65535LL * 65535LL) continue;
      int clusters = active_clusters32_for(g, warps, S);
      if (clusters < 0) continue;
      if (clusters == 0) clusters = sms / S;
      const long long slots = (long long)clusters * S;
      if (slots <= 0) continue;
      const long long waves = (ctas + slots - 1) / slots;
      const double tiles = (double)((kgt + S - 1) / S);
      double per_cta = tiles * VLUT_KG_TILE * 0.5 * (double)(mcta + half_rows) * VLUT_K32_FACTOR;
      per_cta += 4000.0;  // start (first tile + table) and epilogue
      if (S > 1) per_cta += (double)(S - 1) / S * mcta * 128.0 / 16.0 + 1500.0;
      const double cost = waves * per_cta;
      if (cost < best_cost * 0.995) {
        best_cost = cost;
        best->warps = warps;
        best->splits = S;
        best->m_cta = mcta;
        best->n_cta = vlut::kN32;
        best->grid_ctas = (int)ctas;
        best->smem_bytes = smem_bytes32_for(g, warps);
        best->streamk = 0;
      }
    }
  }
  return best_cost;
}

// K1-32 under stream-K (vlut_kernel32_sk.cuh): (warps, rows per thread) in
// {12 x 1, 16 x 1, 12 x 2}; same cost units as plan_sk (half wavefronts
// per 32-token row), plus the per-thread-row partial traffic of split tiles.
#ifndef VLUT_SK32_FACTOR
#define VLUT_SK32_FACTOR 1.00
#endif
int smem_bytes_sk32(int g, int warps, int rpt) {
#define S32(G_, W_, R_) \
  if (g == G_ && warps == W_ && rpt == R_) return vlut::Layout32<G_, W_, R_, true>::SMEM;
  S32(4, 12, 1) S32(4, 16, 1) S32(4, 12, 2)
  S32(5, 12, 1) S32(5, 16, 1) S32(5, 12, 2)
#undef S32
  return 0;
}

double plan_sk32(int M, int K, int N, int g, int sms, vlut_launch_plan* best) {
  const int KG = (K + g - 1) / g;
  const int kgt = (KG + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const int NT = (N + vlut::kN32 - 1) / vlut::kN32;
  const int half_rows = (pow3i(g) + 1) / 2;
  double best_cost = 1e300;
  if (getenv("VLUT_NO_SK32") || getenv("VLUT_NO_K32")) return best_cost;
  // 12 warps x 2 rows is planned (and 12 x 1 at g = 5, below): 16 x 1 lost
  // to the cluster K1-32 and K1-SK everywhere it was measured, 16 x 2 and
  // 12 x 4 rows spill (3-30 % slower).  The split-tile epilogues work per thread row
  // (~16 B/clk): a CTA typically has a producer and an owner segment.
  // 12 x 1 as well at g = 5, where it replaces K1-SK at mid N (config 4
  // N = 64: 115.8 -> 107.4 us); at g = 4 its cost model also picks it where
  // the cluster K1-32 is faster (configs[1] weights N = 80 / 96: 39.5 -> 45.3
  // us; profiles/r02_sk32_plan_r1.txt), so g = 4 plans 12 x 2 only
  const int warps_opts[2] = {12, 12};
  const int rpt_opts[2] = {2, 1};
  // end of round 2: with the fp32 split-tile meeting 12 x 1 also wins at
  // g = 4 once K is long (config 4 N = 64 99.3 -> 92.7 us, config 5 down
  // N = 128 62.5 -> 56.2 us); at K = 2560 (40 K-tiles) it still loses to the
  // cluster K1-32 at N = 80 / 96 (profiles/r02_planner_ab.txt)
  const int n_opts = (g == 5 || kgt >= 64) ? 2 : 1;
  for (int wi = 0; wi < n_opts; ++wi) {
    const int warps = warps_opts[wi], rpt = rpt_opts[wi];
    if (smem_bytes_sk32(g, warps, rpt) > 232448) continue;  // 227 KB opt-in per CTA
    const int mcta = 32 * warps * rpt;
    const long long MT = (M + mcta - 1) / mcta;
    const long long U = MT * NT * kgt;
    const long long grid = U < sms ? U : sms;
    const double units = (double)((U + grid - 1) / grid);
    double cost = units * VLUT_KG_TILE * 0.5 * ((double)mcta * VLUT_SK32_FACTOR + half_rows);
    cost += 4000.0 + 16.0 * mcta;
    const double per_tile = (double)grid / (double)(MT * NT);
    // the owner's fixup: one producer's rows per L2 round trip with int32
    // partials; with the fp32 meeting (fewer tiles than CTAs, K * 128 <
    // 2^24) producers reduce in L2 and the owner reads one slot
    double fix = per_tile - 1.0;
    const bool f32_meet = (long long)K * 128 < (1LL << 24) && 2 * MT * NT <= grid;
    if (f32_meet && !getenv("VLUT_SK32_MODEL_OLD") && fix > 1.0) fix = 1.0;
    if (per_tile > 1.0) cost += fix * (double)mcta * 128.0 / 16.0;
    if (cost < best_cost * 0.995) {
      best_cost = cost;
      best->warps = warps;
      best->splits = 1;
      best->m_cta = mcta;
      best->n_cta = vlut::kN32;
      best->grid_ctas = (int)grid;
      best->smem_bytes = smem_bytes_sk32(g, warps, rpt);
      best->streamk = 1;
    }
  }
  return best_cost;
}

// ------------------------------------------------------------ K2 (lane-slot) planner
// K2 variants: (nw, tpw) with n_cta = nw * tpw tokens per CTA.
inline bool slot_variant_ok(int g, int nw, int tpw) {
  if (!(tpw == 1 || tpw == 2)) return false;
  if (!(nw == 1 || nw == 2 || nw == 4 || nw == 8)) return false;
  return g == 4 || nw <= 2 || (nw == 4 && tpw == 1);  // g = 5: half tables at 4 scalar words
}
inline int slot_mcta(int g) { return g == 4 ? 32 * vlut::slot::kLW * VLUT_SLOT_RPL_G4 : 2048; }
int slot_smem(int g, int nw, int tpw);

// The narrowest variant covering N tokens in one N-tile (capped at the widest).
int slot_default_nw(int g, int N, int tpw) {
  const int maxnw = g == 4 ? 8 : (tpw == 1 ? 4 : 2);
  int nw = 1;
  while (nw < maxnw && nw * tpw < N) nw *= 2;
  return nw;
}

// Cost in shared-memory cycles of one SM (the K1 planner's unit): per K-tile
// lookups (m_cta * 16 groups * nw words / 32 lanes per wavefront) + the table
// build (nw * 3^g wavefronts) + the index reads (m_cta / 8); an index tile of
// m_cta * 16 B must also arrive from HBM (~22 B/clk/SM when all SMs stream);
// split-K adds the red.global traffic of the partial tile.
double plan_slot(int M, int K, int N, int g, int sms, int tpw, int nw_force, int S_force,
                 bool have_ws, vlut_launch_plan* out) {
  const int KG = (K + g - 1) / g;  // padded packing: the last group may be partial
  const int kgt = (KG + VLUT_KG_TILE - 1) / VLUT_KG_TILE;
  const int nw = nw_force > 0 ? nw_force : slot_default_nw(g, N, tpw);
  if (!slot_variant_ok(g, nw, tpw)) return 1e300;
  const int ntok = nw * tpw, mcta = slot_mcta(g);
  const long long NTt = (N + ntok - 1) / ntok, MT = (M + mcta - 1) / mcta;
  const long long tiles = NTt * MT;
  int S = 1;
  if (S_force > 0) {
    S = S_force;
  } else if (have_ws && tiles <= vlut::slot::kMaxCounters &&
             (size_t)M * (size_t)N * 4 <= kSlotAccBytes) {
    S = (int)(sms / tiles);  // one wave: split-K CTAs must be co-resident
    if (S < 1) S = 1;
    if (S > kgt) S = kgt;
    // the makespan is ceil(kgt / S) K-tiles: use the fewest CTAs that reach
    // it (fewer partial tiles to reduce, no idle tail on the others)
    const int per = (kgt + S - 1) / S;
    S = (kgt + per - 1) / per;
  }
  if (S > kgt) S = kgt;
  if (S < 1) S = 1;
  const long long ctas = tiles * S;
  const long long waves = (ctas + sms - 1) / sms;
  const double kt_per = (double)((kgt + S - 1) / S);
  // table rows: full 3^g, half tables for the scalar LUT from 4 words on
  const double rows = (nw >= 4 && tpw == 1) ? (pow3i(g) + 1) / 2.0 : (double)pow3i(g);
  const double smem_tile = mcta * 16.0 * nw / 32.0 + (double)nw * rows + mcta / 8.0;
  const double hbm_tile = mcta * 16.0 / 22.0;
  double per_cta = kt_per * (smem_tile > hbm_tile ? smem_tile : hbm_tile) + 3000.0;
  if (S > 1) per_cta += mcta * (double)ntok / 32.0 * 8.0;
  const double cost = (double)waves * per_cta;
  if (out) {
    memset(out, 0, sizeof(*out));
    out->warps = vlut::slot::kLW;
    out->splits = S;
    out->m_cta = mcta;
    out->n_cta = ntok;
    out->grid_ctas = (int)(ctas > 0x7fffffff ? 0x7fffffff : ctas);
    out->smem_bytes = slot_smem(g, nw, tpw);
    out->streamk = 0;
    out->slot = 1;
    out->tpw = tpw;
    out->nw = nw;
  }
  return cost;
}

// ------------------------------------------------------------ launches
template <int G, int NW, int TPW, bool FQ = false>
vlut_status launch_slot(const vlut::slot::SlotParams& p, int S, int NTt, int MT, cudaStream_t st) {
  using L = vlut::slot::SL<G, NW, TPW>;
  auto kern = vlut::slot::vlut_slot_kernel<G, NW, TPW, FQ>;
  static std::once_flag flags[64];
  static cudaError_t errs[64];
  int dev = 0;
  VLUT_CUDA_TRY(cudaGetDevice(&dev));
  std::call_once(flags[dev & 63], [&] {
    errs[dev & 63] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  });
  VLUT_CUDA_TRY(errs[dev & 63]);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S, (unsigned)NTt, (unsigned)MT);
  cfg.blockDim = dim3(vlut::slot::kThreads, 1, 1);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // split-K CTAs of a tile wait for each other (generation handshake): all
  // CTAs must be co-resident.  Last-only tiles never wait: no cooperative
  // launch, so the grid may overlap its neighbours (PDL).
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = (S > 1 && !(p.last_only && !getenv("VLUT_SLOT_COOP_ALWAYS"))) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  return VLUT_OK;
}

#define VLUT_SLOT_VARIANTS(X) \
  X(4, 1, 1) X(4, 2, 1) X(4, 4, 1) X(4, 8, 1) X(4, 1, 2) X(4, 2, 2) X(4, 4, 2) X(4, 8, 2) \
  X(5, 1, 1) X(5, 2, 1) X(5, 4, 1) X(5, 1, 2) X(5, 2, 2)

int slot_smem(int g, int nw, int tpw) {
#define X(G_, NW_, TPW_) \
  if (g == G_ && nw == NW_ && tpw == TPW_) return vlut::slot::SL<G_, NW_, TPW_>::SMEM;
  VLUT_SLOT_VARIANTS(X)
#undef X
  return 0;
}

vlut_status dispatch_slot(int g, int nw, int tpw, const vlut::slot::SlotParams& p, int S, int NTt,
                          int MT, cudaStream_t st) {
  if (p.xq) {  // fused decode: one scalar word
    if (nw == 1 && tpw == 1 && g == 4) return launch_slot<4, 1, 1, true>(p, S, NTt, MT, st);
    if (nw == 1 && tpw == 1 && g == 5) return launch_slot<5, 1, 1, true>(p, S, NTt, MT, st);
    return fail(VLUT_ERR_UNSUPPORTED, "fused decode: nw = tpw = 1 only");
  }
#define X(G_, NW_, TPW_) \
  if (g == G_ && nw == NW_ && tpw == TPW_) return launch_slot<G_, NW_, TPW_>(p, S, NTt, MT, st);
  VLUT_SLOT_VARIANTS(X)
#undef X
  return fail(VLUT_ERR_UNSUPPORTED, "no K2 variant for g=%d nw=%d tpw=%d", g, nw, tpw);
}

template <int G, int WARPS, bool ACC>
vlut_status launch_k1(const vlut::Params& p, int S, int NT, int MT, cudaStream_t st) {
  using L = vlut::Layout<G, WARPS>;
  auto kern = vlut::vlut_mpgemm_kernel<G, WARPS, ACC>;
  VLUT_CUDA_TRY((prepare_kernel<G, WARPS, ACC>()));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S, (unsigned)NT, (unsigned)MT);
  cfg.blockDim = dim3(L::THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the prologue overlaps the previous kernel
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  return VLUT_OK;
}

template <int G, int WARPS, bool ACC>
vlut_status launch_k1_32(const vlut::Params& p, int S, int NT, int MT, cudaStream_t st) {
  using L = vlut::Layout32<G, WARPS>;
  auto kern = vlut::vlut_mpgemm32_kernel<G, WARPS, ACC>;
  VLUT_CUDA_TRY((prepare_kernel32<G, WARPS, ACC>()));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)S, (unsigned)NT, (unsigned)MT);
  cfg.blockDim = dim3(L::THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)S;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  // no cluster attribute without split-K (a plain launch; the S = 1 path
  // never touches the cluster)
  cfg.numAttrs = (S > 1 || getenv("VLUT_K32_CLUSTER1")) ? 2 : 1;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
  return VLUT_OK;
}

template <int G, int WARPS, int RPT, bool ACC>
vlut_status launch_sk32(const vlut::Params& p, const vlut::SkParams& sk, int grid,
                        cudaStream_t st) {
  using L = vlut::Layout32<G, WARPS, RPT, true>;
  auto kern = vlut::vlut_mpgemm32_sk_kernel<G, WARPS, RPT, ACC>;
  static std::once_flag flags[64];
  static cudaError_t errs[64];
  int dev = 0;
  VLUT_CUDA_TRY(cudaGetDevice(&dev));
  std::call_once(flags[dev & 63], [&] {
    errs[dev & 63] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  });
  VLUT_CUDA_TRY(errs[dev & 63]);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(L::THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // owners wait for producers: co-resident
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p, sk));
  return VLUT_OK;
}

template <bool ACC>
vlut_status dispatch_sk32(int g, int warps, int rpt, const vlut::Params& p,
                          const vlut::SkParams& sk, int grid, cudaStream_t st) {
#define D32(G_, W_, R_) \
  if (g == G_ && warps == W_ && rpt == R_) return launch_sk32<G_, W_, R_, ACC>(p, sk, grid, st);
  D32(4, 12, 1) D32(4, 16, 1) D32(4, 12, 2)
  D32(5, 12, 1) D32(5, 16, 1) D32(5, 12, 2)
#undef D32
  return fail(VLUT_ERR_UNSUPPORTED, "no K1-32 stream-K variant g=%d warps=%d rows=%d", g, warps, rpt);
}

template <bool ACC>
vlut_status dispatch32(int g, int warps, const vlut::Params& p, int S, int NT, int MT,
                       cudaStream_t st) {
  if (g == 4) {
    if (warps == 8) return launch_k1_32<4, 8, ACC>(p, S, NT, MT, st);
    if (warps == 12) return launch_k1_32<4, 12, ACC>(p, S, NT, MT, st);
    if (warps == 16) return launch_k1_32<4, 16, ACC>(p, S, NT, MT, st);
  } else {
    if (warps == 8) return launch_k1_32<5, 8, ACC>(p, S, NT, MT, st);
    if (warps == 12) return launch_k1_32<5, 12, ACC>(p, S, NT, MT, st);
    if (warps == 16) return launch_k1_32<5, 16, ACC>(p, S, NT, MT, st);
  }
  return fail(VLUT_ERR_UNSUPPORTED, "no K1-32 variant for g=%d warps=%d", g, warps);
}

template <int G, int WARPS, bool ACC, int RPT = 1>
vlut_status launch_sk(const vlut::Params& p, const vlut::SkParams& sk, int grid,
                      cudaStream_t st) {
  using L = vlut::Layout<G, WARPS, RPT>;
  auto kern = vlut::vlut_mpgemm_sk_kernel<G, WARPS, RPT, ACC>;
  static std::once_flag flags[64];
  static cudaError_t errs[64];
  int dev = 0;
  VLUT_CUDA_TRY(cudaGetDevice(&dev));
  std::call_once(flags[dev & 63], [&] {
    errs[dev & 63] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  });
  VLUT_CUDA_TRY(errs[dev & 63]);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(L::THREADS, 1, 1);
  cfg.dynamicSmemBytes = L::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // owners spin on their producers' flags: every CTA must be co-resident
  // (grid <= #SMs, one CTA per SM), which a cooperative launch guarantees
  // whatever else holds SMs (NCCL kernels, other streams)
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p, sk));
  return VLUT_OK;
}

template <bool ACC>
vlut_status dispatch_sk(int g, int warps, int rpt, const vlut::Params& p, const vlut::SkParams& sk,
                        int grid, cudaStream_t st) {
  if (rpt == 2) {
    if (warps == 12) return g == 4 ? launch_sk<4, 12, ACC, 2>(p, sk, grid, st)
                                   : launch_sk<5, 12, ACC, 2>(p, sk, grid, st);
    if (warps == 8) return g == 4 ? launch_sk<4, 8, ACC, 2>(p, sk, grid, st)
                                  : launch_sk<5, 8, ACC, 2>(p, sk, grid, st);
    return fail(VLUT_ERR_UNSUPPORTED, "two rows per thread: 8 or 12 warps");
  }
  if (g == 4) {
    if (warps == 8) return launch_sk<4, 8, ACC>(p, sk, grid, st);
    if (warps == 12) return launch_sk<4, 12, ACC>(p, sk, grid, st);
    if (warps == 16) return launch_sk<4, 16, ACC>(p, sk, grid, st);
  } else {
    if (warps == 8) return launch_sk<5, 8, ACC>(p, sk, grid, st);
    if (warps == 12) return launch_sk<5, 12, ACC>(p, sk, grid, st);
    if (warps == 16) return launch_sk<5, 16, ACC>(p, sk, grid, st);
  }
  return fail(VLUT_ERR_UNSUPPORTED, "no stream-K variant for g=%d warps=%d", g, warps);
}

template <bool ACC>
vlut_status dispatch(int g, int warps, const vlut::Params& p, int S, int NT, int MT,
                     cudaStream_t st) {
  if (g == 4) {
    if (warps == 8) return launch_k1<4, 8, ACC>(p, S, NT, MT, st);
    if (warps == 12) return launch_k1<4, 12, ACC>(p, S, NT, MT, st);
    if (warps == 16) return launch_k1<4, 16, ACC>(p, S, NT, MT, st);
  } else {
    if (warps == 8) return launch_k1<5, 8, ACC>(p, S, NT, MT, st);
    if (warps == 12) return launch_k1<5, 12, ACC>(p, S, NT, MT, st);
    if (warps == 16) return launch_k1<5, 16, ACC>(p, S, NT, MT, st);
  }
  return fail(VLUT_ERR_UNSUPPORTED, "no kernel variant for g=%d warps=%d", g, warps);
}

// K2 launch for a validated call (sizes, descriptor, pointers checked by the
// caller).  plan.slot must be 1; nw/tpw/splits 0 = heuristic.
constexpr int kSlotAutoMaxN = 64;

vlut_status run_slot(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                     float w_scale, void* out, int M, int K, int N, vlut_launch_plan plan,
                     void* ws, size_t ws_bytes, void* stream, bool acc_only, const DeviceInfo& d,
                     const float* xq = nullptr, float* scale_out = nullptr) {
  const int g = W->g;
  const int tpw = plan.tpw ? plan.tpw : 2;
  const bool have_ws = ws != nullptr;
  if (have_ws) {
    if (ws_bytes < sk_workspace_bytes(d.sms))
      return fail(VLUT_ERR_BUFFER_TOO_SMALL, "workspace needs %zu bytes", sk_workspace_bytes(d.sms));
    if (((uintptr_t)ws) & 15) return fail(VLUT_ERR_MISALIGNED, "workspace not 16-B aligned");
  }
  if (plan.nw && !slot_variant_ok(g, plan.nw, tpw))
    return fail(VLUT_ERR_UNSUPPORTED, "no K2 variant for g=%d nw=%d tpw=%d", g, plan.nw, tpw);
  if (!(tpw == 1 || tpw == 2)) return fail(VLUT_ERR_INVALID_ARGUMENT, "tpw must be 1 or 2");
  vlut_launch_plan pl = {};
  plan_slot(M, K, N, g, d.sms, tpw, plan.nw, plan.splits, have_ws, &pl);
  const int S = pl.splits;
  const long long NTt = (N + pl.n_cta - 1) / pl.n_cta;
  const long long MT = (M + pl.m_cta - 1) / pl.m_cta;
  if (NTt > 65535 || MT > 65535 || S > 65535) return fail(VLUT_ERR_SHAPE, "grid too large");
  if (S > 1) {
    if (!have_ws) return fail(VLUT_ERR_INVALID_ARGUMENT, "K2 split-K (splits=%d) needs a workspace", S);
    if (NTt * MT * S > d.sms)
      return fail(VLUT_ERR_UNSUPPORTED, "K2 split-K needs all %lld CTAs co-resident (%d SMs)",
                  NTt * MT * S, d.sms);
    if (NTt * MT > vlut::slot::kMaxCounters || (size_t)M * (size_t)N * 4 > kSlotAccBytes)
      return fail(VLUT_ERR_SHAPE, "M*N too large for K2 split-K workspace");
  }
  if (pl.smem_bytes > d.smem_optin)
    return fail(VLUT_ERR_UNSUPPORTED, "needs %d B shared memory, device allows %d", pl.smem_bytes,
                d.smem_optin);
  vlut::slot::SlotParams p;
  memset(&p, 0, sizeof(p));
  p.payload = static_cast<const uint8_t*>(W->payload);
  p.A = A;
  p.a_scale = a_scale;
  p.w_scale = w_scale;
  p.out = out;
  p.M = M;
  p.K = K;
  p.N = N;
  p.m_pad = W->m_pad;
  p.kg_tiles = W->kg_tiles;
  p.splits = S;
  p.acc_only = acc_only ? 1 : 0;
  p.act_tma = (!xq && N <= vlut::slot::kActNMax && (((uintptr_t)A) & 15) == 0) ? 1 : 0;
  p.xq = xq;
  p.scale_out = scale_out;
  p.q_ring = getenv("VLUT_DECODE_NO_RING") ? 0 : 1;  // (test switch: the fallback path)
  if (have_ws) {
    p.ws_cnt = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + slot_cnt_off(d.sms));
    p.ws_acc = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + slot_acc_off(d.sms));
  }
  // last_only: no CTA waits for another.  Variants with few tokens per CTA
  // meet through counted 64-bit atomics (8-byte words, at most 255
  // partials); the others let the last CTA finish tiles up to 8 KB
  if (vlut::slot::kAtom64 && pl.nw * tpw <= vlut::slot::kA64MaxTok)
    p.last_only = (S <= vlut::slot::kAtom64MaxSplits && (size_t)M * (size_t)N * 8 <= kSlotAccBytes)
                      ? 1 : 0;
  else
    p.last_only =
        ((long long)pl.m_cta * std::min(N, pl.n_cta) * 4 <= vlut::slot::kLastOnlyBytes) ? 1 : 0;
  vlut_status st = dispatch_slot(g, pl.nw, tpw, p, S, (int)NTt, (int)MT,
                                 static_cast<cudaStream_t>(stream));
  if (st != VLUT_OK) return st;
  return ok();
}

// K1-32 preconditions: TMA activation staging (N % 16 == 0, 16-B aligned A),
// 16-byte output stores, the plain fp32 (or raw int32) epilogue.
bool k32_ok(const void* A, const void* out, int N, const int32_t* acc_in, int out_t,
            const float* mul_in, const unsigned* amax_out) {
  return N % 16 == 0 && ((((uintptr_t)A) | ((uintptr_t)out)) & 15) == 0 && !acc_in && !out_t &&
         !mul_in && !amax_out && !getenv("VLUT_NO_K32");
}

vlut_status run_mpgemm(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                       float w_scale, void* out, int M, int K, int N,
                       const vlut_launch_plan* plan_in, void* stream, bool acc_only,
                       const int32_t* acc_in = nullptr, int out_t = 0, void* ws = nullptr,
                       size_t ws_bytes = 0, const float* mul_in = nullptr,
                       unsigned* amax_out = nullptr, int amax_rows = 0) {
  if (M < 0 || K <= 0 || N < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes M=%d K=%d N=%d", M, K, N);
  if (M == 0 || N == 0) return ok();
  vlut_status st = check_desc(W, M, K);
  if (st != VLUT_OK) return st;
  if (!A || !out || (!acc_only && !a_scale))
    return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL device pointer");
  if (((uintptr_t)out) & 3) return fail(VLUT_ERR_MISALIGNED, "out not 4-B aligned");
  if (!acc_only && (((uintptr_t)a_scale) & 3))
    return fail(VLUT_ERR_MISALIGNED, "a_scale not 4-B aligned");
  if ((long long)N > (1LL << 30)) return fail(VLUT_ERR_SHAPE, "N too large");
  DeviceInfo d;
  st = device_info(&d);
  if (st != VLUT_OK) return st;
  vlut_launch_plan plan = {};
  const bool plain_epilogue = !acc_in && !out_t && !mul_in && !amax_out;
  if (plan_in) {
    plan = *plan_in;
    if (plan.slot) {
      if (!plain_epilogue)
        return fail(VLUT_ERR_UNSUPPORTED, "K2 plan: no acc_in / transposed / fused epilogue");
      return run_slot(W, A, a_scale, w_scale, out, M, K, N, plan, ws, ws_bytes, stream, acc_only,
                      d);
    }
    if (!(plan.warps == 8 || plan.warps == 12 || plan.warps == 16) ||
        !valid_split(plan.warps, plan.splits))
      return fail(VLUT_ERR_INVALID_ARGUMENT, "invalid plan warps=%d splits=%d", plan.warps,
                  plan.splits);
    if (plan.streamk && (!ws || acc_in || out_t))
      return fail(VLUT_ERR_INVALID_ARGUMENT, "stream-K plan needs a workspace and [M][N] output");
    // m_cta selects the rows per lookup thread: 0 or 32 * warps -> 1; 64 * warps
    // -> 2 (stream-K with 8 or 12 warps; 32-token stream-K with 12 warps)
    if (plan.n_cta == vlut::kN32 && plan.streamk) {
      const int r = plan.m_cta ? plan.m_cta / (32 * plan.warps) : 1;
      if ((plan.m_cta && plan.m_cta % (32 * plan.warps)) || !smem_bytes_sk32(W->g, plan.warps, r))
        return fail(VLUT_ERR_UNSUPPORTED,
                    "32-token stream-K: 12 or 16 warps x 1 row, or 12 warps x 2 rows");
    } else if (plan.m_cta && plan.m_cta != 32 * plan.warps &&
        !(plan.m_cta == 64 * plan.warps && plan.warps <= 12 && plan.streamk))
      return fail(VLUT_ERR_UNSUPPORTED, "m_cta=%d: 32*warps, or 64*warps (8/12 warps) stream-K",
                  plan.m_cta);
  } else {
    double c_best = plan_for(M, K, N, W->g, d.sms, &plan);
    if (ws && !acc_in && !out_t) {
      vlut_launch_plan sk_plan = {};
      const double c_sk = plan_sk(M, K, N, W->g, d.sms, &sk_plan);
      if (c_sk < c_best) {
        plan = sk_plan;
        c_best = c_sk;
      }
    }
    if (k32_ok(A, out, N, acc_in, out_t, mul_in, amax_out)) {
      vlut_launch_plan p32 = {};
      const double c32 = plan_for32(M, K, N, W->g, d.sms, &p32);
      if (c32 < c_best) {
        plan = p32;
        c_best = c32;
      }
      if (ws) {
        vlut_launch_plan s32 = {};
        const double cs32 = plan_sk32(M, K, N, W->g, d.sms, &s32);
        if (cs32 < c_best) {
          plan = s32;
          c_best = cs32;
        }
      }
    }
    if (plain_epilogue && N <= kSlotAutoMaxN) {
      vlut_launch_plan sl = {};
      const bool have_ws = ws && ws_bytes >= sk_workspace_bytes(d.sms) && ((uintptr_t)ws & 15) == 0;
      // N = 1: one token, the scalar and the vector LUT coincide; a 1-token
      // word (tpw = 1) wastes no half-words
      const double c_sl = plan_slot(M, K, N, W->g, d.sms, N == 1 ? 1 : 2, 0, 0, have_ws, &sl);
      if (c_sl < c_best)
        return run_slot(W, A, a_scale, w_scale, out, M, K, N, sl, have_ws ? ws : nullptr,
                        ws_bytes, stream, acc_only, d);
    }
  }
  if (plan.streamk && ws_bytes < sk_workspace_bytes(d.sms))
    return fail(VLUT_ERR_BUFFER_TOO_SMALL, "stream-K workspace needs %zu bytes",
                sk_workspace_bytes(d.sms));
  if (plan.streamk && (((uintptr_t)ws) & 15)) return fail(VLUT_ERR_MISALIGNED, "workspace not 16-B aligned");
  if (plan.splits > W->kg_tiles) plan.splits = 1;
  const bool n32 = plan.n_cta == vlut::kN32 && !plan.streamk;
  const bool sk32 = plan.n_cta == vlut::kN32 && plan.streamk;
  if (sk32 && (!k32_ok(A, out, N, acc_in, out_t, mul_in, amax_out) || g_peer_tls.n))
    return fail(VLUT_ERR_UNSUPPORTED,
                "32-token tiles: N %% 16 == 0, 16-B aligned A / out, plain epilogue only");
  if (n32) {
    if (!k32_ok(A, out, N, acc_in, out_t, mul_in, amax_out) || g_peer_tls.n)
      return fail(VLUT_ERR_UNSUPPORTED,
                  "32-token tiles: N %% 16 == 0, 16-B aligned A / out, plain epilogue only");
    if (plan.m_cta && plan.m_cta != 32 * plan.warps)
      return fail(VLUT_ERR_UNSUPPORTED, "32-token tiles: m_cta = 32 * warps");
    const int smem32 = smem_bytes32_for(W->g, plan.warps);
    if (smem32 > d.smem_optin)
      return fail(VLUT_ERR_UNSUPPORTED, "needs %d B shared memory, device allows %d", smem32,
                  d.smem_optin);
  }
  const int rpt = sk32 ? (plan.m_cta ? plan.m_cta / (32 * plan.warps) : 1)
                  : (plan.streamk && plan.m_cta == 64 * plan.warps) ? 2 : 1;
  const int smem = sk32 ? smem_bytes_sk32(W->g, plan.warps, rpt)
                        : smem_bytes_for(W->g, plan.warps, rpt);
  if (smem > d.smem_optin)
    return fail(VLUT_ERR_UNSUPPORTED, "needs %d B shared memory, device allows %d", smem,
                d.smem_optin);
  vlut::Params p;
  memset(&p, 0, sizeof(p));
  p.payload = static_cast<const uint8_t*>(W->payload);
  p.A = A;
  p.a_scale = a_scale;
  p.w_scale = w_scale;
  p.out = static_cast<float*>(out);
  p.acc_in = acc_in;
  p.M = M;
  p.K = K;
  p.N = N;
  p.m_pad = W->m_pad;
  p.kg_tiles = W->kg_tiles;
  p.splits = plan.splits;
  const uintptr_t ap = (uintptr_t)A;
  p.a_vec = (N % 16 == 0 && (ap & 15) == 0) ? 16 : ((N % 4 == 0 && (ap & 3) == 0) ? 4 : 1);
  if (p.a_vec == 16) {
    // [r][group][token] staging (conflict-free wide-builder loads) whenever
    // K % g == 0; K1's 4-byte builders (kWideBuild false) read [group][r]
    const int wq = plan.warps;
    const bool t32 = n32 || sk32;
    const bool wide = t32 || (wq <= VLUT_WIDE_MAX_WARPS);
    p.a3d = (wide && K % W->g == 0 && !getenv("VLUT_NO_A3D")) ? 1 : 0;
    st = p.a3d ? encode_a_map3d(&p.a_map, A, K, N, W->g, t32 ? vlut::kN32 : vlut::kNcta)
               : encode_a_map(&p.a_map, A, K, N, W->g, t32 ? vlut::kN32 : vlut::kNcta);
    if (st != VLUT_OK) return st;
  }
  p.out_t = out_t;
  p.n_peers = g_peer_tls.n;
  p.out_mc = g_peer_tls.mc;
  for (int i = 0; i < g_peer_tls.n; ++i) p.peer_out[i] = g_peer_tls.ptr[i];
  if ((p.n_peers || p.out_mc) && (plan.streamk || n32 || sk32 || acc_only || out_t || acc_in))
    return fail(VLUT_ERR_UNSUPPORTED, "fused all-gather: cluster schedule, fp32 [M][N] output only");
  p.mul_in = mul_in;
  p.amax_out = amax_out;
  p.amax_rows = amax_rows;
  p.out_vec4 = ((out_t ? M : N) % 4 == 0 && (((uintptr_t)out) & 15) == 0) ? 1 : 0;
  const int mcta = 32 * plan.warps * rpt;
  const long long NT = (N + (sk32 ? vlut::kN32 : vlut::kNcta) - 1) / (sk32 ? vlut::kN32 : vlut::kNcta);
  const long long MT = (M + mcta - 1) / mcta;
  if (NT > 65535 || MT > 65535) return fail(VLUT_ERR_SHAPE, "grid too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (plan.streamk) {
    vlut::SkParams sk;
    sk.NT = (int)NT;
    sk.MT = (int)MT;
    sk.U = MT * NT * (long long)W->kg_tiles;
    sk.ws = static_cast<int32_t*>(ws);
    sk.flags = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + sk_part_bytes(d.sms));
    sk.epoch = 1u;  // flags are reset by their consumers: graph-replay safe
    int grid = (int)(sk.U < d.sms ? sk.U : d.sms);
    if (const char* e = getenv("VLUT_SK_GRID")) {  // (experiment) override the persistent grid
      const int gx = atoi(e);
      if (gx > 0 && gx < grid) grid = gx;
    }
    // K1-32-SK: split tiles meet in fp32 accumulators (exact while every
    // partial sum stays below 2^24) when there are at least two CTAs per
    // tile -- several producers per tile, whose reads would chain in the
    // owner's fixup; with ~1 producer per tile the int32 partial stores are
    // cheaper than the L2 reductions (6912 x 2560 N = 512, 144 tiles: 154.7
    // vs 158.5 us; profiles/r02_sk32_fixup.txt)
    const bool acc_f32 = sk32 && (long long)K * 128 < (1LL << 24) && 2 * MT * NT <= grid &&
                         !getenv("VLUT_SK32_INT_PARTIALS");
    sk.acc = acc_f32 ? reinterpret_cast<float*>(static_cast<char*>(ws) + sk32_acc_off(d.sms)) : nullptr;
    if (sk32)
      st = acc_only ? dispatch_sk32<true>(W->g, plan.warps, rpt, p, sk, grid, s)
                    : dispatch_sk32<false>(W->g, plan.warps, rpt, p, sk, grid, s);
    else
      st = acc_only ? dispatch_sk<true>(W->g, plan.warps, rpt, p, sk, grid, s)
                    : dispatch_sk<false>(W->g, plan.warps, rpt, p, sk, grid, s);
    if (st != VLUT_OK) return st;
    return ok();
  }
  if (n32) {
    const long long NT32 = (N + vlut::kN32 - 1) / vlut::kN32;
    if (NT32 > 65535) return fail(VLUT_ERR_SHAPE, "grid too large");
    st = acc_only ? dispatch32<true>(W->g, plan.warps, p, plan.splits, (int)NT32, (int)MT, s)
                  : dispatch32<false>(W->g, plan.warps, p, plan.splits, (int)NT32, (int)MT, s);
    if (st != VLUT_OK) return st;
    return ok();
  }
  st = acc_only ? dispatch<true>(W->g, plan.warps, p, plan.splits, (int)NT, (int)MT, s)
                : dispatch<false>(W->g, plan.warps, p, plan.splits, (int)NT, (int)MT, s);
  if (st != VLUT_OK) return st;
  return ok();
}

}  // namespace

// Library-owned workspaces of vlut_mpgemm (the north-star signature has no
// workspace argument).  At most kWsCap per device, each bound to one stream
// by its process-unique id (cudaStreamGetId: ids are never reused, so a
// recycled stream handle cannot alias a workspace with work still in flight,
// and cudaStreamPerThread / the legacy stream resolve to their own streams).
// Calls on one stream are ordered, so they share that stream's workspace.  A
// new stream beyond the cap takes the least recently used entry after a
// device-wide synchronisation (its previous stream may still be using it) and
// re-zeroes it on the new stream.  g_ws_mu is held from the lookup through
// the launch, so an eviction can never rebind a workspace between the lookup
// and the launch that uses it.  Never allocates or evicts inside a stream
// capture: the call then runs without a workspace (cluster schedules only).
struct WsEntry {
  int dev;
  unsigned long long sid;
  void* ptr;
  size_t bytes;
  unsigned long long last;
};
constexpr int kWsCap = 4;
std::mutex g_ws_mu;
std::vector<WsEntry> g_ws;
unsigned long long g_ws_tick = 0;

bool internal_workspace_locked(void* stream, void** ws, size_t* bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  DeviceInfo d;
  if (device_info(&d) != VLUT_OK) return false;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;
  }
  unsigned long long sid = 0;
  if (cudaStreamGetId(st, &sid) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int n_dev = 0;
  WsEntry* lru = nullptr;
  for (auto& e : g_ws) {
    if (e.dev != dev) continue;
    if (e.sid == sid) {
      e.last = ++g_ws_tick;
      *ws = e.ptr;
      *bytes = e.bytes;
      return true;
    }
    ++n_dev;
    if (!lru || e.last < lru->last) lru = &e;
  }
  const size_t need = sk_workspace_bytes(d.sms);
  WsEntry* slot = nullptr;
  if (n_dev >= kWsCap && lru) {
    // the LRU entry's stream may still run work that uses it
    if (cudaDeviceSynchronize() != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    slot = lru;
  } else {
    void* p = nullptr;
    if (cudaMalloc(&p, need) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    g_ws.push_back({dev, 0ull, p, need, 0ull});
    slot = &g_ws.back();
  }
  if (cudaMemsetAsync(slot->ptr, 0, slot->bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return false;  // the entry stays cached (still unbound to this stream)
  }
  slot->sid = sid;
  slot->last = ++g_ws_tick;
  *ws = slot->ptr;
  *bytes = slot->bytes;
  return true;
}

// ================================================================ C ABI
extern "C" {

const char* vlut_last_error(void) { return g_err.c_str(); }

#ifdef VLUT_TIMING
int vlut_debug_set_timing(void* dev_buf) {
  return (int)cudaMemcpyToSymbol(vlut::g_vlut_timing, &dev_buf, sizeof(void*));
}
#endif

const char* vlut_version(void) { return "vlut-b200 0.1 (sm_100a)"; }

int vlut_launches_per_mpgemm(void) { return 1; }

int vlut_active_clusters(int g, int warps, int splits) {
  if (!valid_g(g) || !(warps == 8 || warps == 12 || warps == 16) || !valid_split(warps, splits))
    return 0;
  return active_clusters_for(g, warps, splits);
}

size_t vlut_packed_bytes_ex(int M, int K, int g, int flags) {
  int mp = 0, kgt = 0;
  size_t b = 0;
  if (!layout_of(M, K, g, flags, &mp, &kgt, &b)) return 0;
  return b;
}

size_t vlut_packed_bytes(int M, int K, int g) { return vlut_packed_bytes_ex(M, K, g, 0); }

static vlut_status fill_desc(int M, int K, int g, int flags, void* payload_dev,
                             size_t payload_bytes, vlut_packed_weights* desc_out, int* m_pad,
                             int* kgt) {
  if (!desc_out || !payload_dev) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!valid_g(g)) return fail(VLUT_ERR_INVALID_ARGUMENT, "g must be 4 or 5 (got %d)", g);
  if (M <= 0 || K <= 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "M, K must be > 0");
  if (flags & ~VLUT_PACK_PAD_K) return fail(VLUT_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  if (K % g && !(flags & VLUT_PACK_PAD_K))
    return fail(VLUT_ERR_SHAPE, "g=%d does not divide K=%d", g, K);
  size_t need = 0;
  if (!layout_of(M, K, g, flags, m_pad, kgt, &need)) return fail(VLUT_ERR_SHAPE, "size overflow");
  if (payload_bytes < need)
    return fail(VLUT_ERR_BUFFER_TOO_SMALL, "payload needs %zu bytes, got %zu", need,
                payload_bytes);
  if (((uintptr_t)payload_dev) & 15) return fail(VLUT_ERR_MISALIGNED, "payload not 16-B aligned");
  memset(desc_out, 0, sizeof(*desc_out));
  desc_out->magic = VLUT_MAGIC;
  desc_out->version = VLUT_VERSION;
  desc_out->M = M;
  desc_out->K = K;
  desc_out->g = g;
  desc_out->m_pad = *m_pad;
  desc_out->kg_tiles = *kgt;
  desc_out->m_tile = VLUT_M_TILE;
  desc_out->kg_tile = VLUT_KG_TILE;
  desc_out->flags = flags;
  desc_out->payload_bytes = (int64_t)need;
  desc_out->payload = payload_dev;
  return VLUT_OK;
}

vlut_status vlut_pack_weights_ex(const int8_t* w, int M, int K, int g, int flags,
                                 void* payload_dev, size_t payload_bytes,
                                 vlut_packed_weights* desc_out, void* stream) {
  if (!w) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL weights");
  vlut_packed_weights d;
  int mp = 0, kgt = 0;
  vlut_status st = fill_desc(M, K, g, flags, payload_dev, payload_bytes, &d, &mp, &kgt);
  if (st != VLUT_OK) return st;
  const int KG = (K + g - 1) / g;  // last group padded with zero trits (VLUT_PACK_PAD_K)
  const uint8_t zero = (uint8_t)((pow3i(g) - 1) / 2);
  std::vector<uint8_t> host((size_t)d.payload_bytes, zero);
  for (int m = 0; m < M; ++m) {
    const int8_t* row = w + (size_t)m * K;
    for (int k = 0; k < KG; ++k) {
      int idx = 0, p3 = 1;
      for (int r = 0; r < g; ++r) {
        const int f = k * g + r;
        const int t = f < K ? row[f] : 0;
        if (t < -1 || t > 1)
          return fail(VLUT_ERR_INVALID_TRIT, "invalid trit %d at (%d,%d)", t, m, f);
        idx += (t + 1) * p3;
        p3 *= 3;
      }
      host[((size_t)(k / VLUT_KG_TILE) * mp + m) * 16 + (k % VLUT_KG_TILE)] = (uint8_t)idx;
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VLUT_CUDA_TRY(cudaMemcpyAsync(payload_dev, host.data(), host.size(), cudaMemcpyHostToDevice, s));
  VLUT_CUDA_TRY(cudaStreamSynchronize(s));
  *desc_out = d;
  return ok();
}

vlut_status vlut_pack_weights(const int8_t* w, int M, int K, int g, void* payload_dev,
                              size_t payload_bytes, vlut_packed_weights* desc_out,
                              void* stream) {
  return vlut_pack_weights_ex(w, M, K, g, 0, payload_dev, payload_bytes, desc_out, stream);
}

vlut_status vlut_pack_weights_device_ex(const int8_t* w_dev, int M, int K, int g, int flags,
                                        void* payload_dev, size_t payload_bytes,
                                        vlut_packed_weights* desc_out, void* stream) {
  if (!w_dev) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL weights");
  vlut_packed_weights d;
  int mp = 0, kgt = 0;
  vlut_status st = fill_desc(M, K, g, flags, payload_dev, payload_bytes, &d, &mp, &kgt);
  if (st != VLUT_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long total = d.payload_bytes;
  const int threads = 256;
  long long blocks = (total + threads - 1) / threads;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  vlut::vlut_pack_kernel<<<(unsigned)blocks, threads, 0, s>>>(
      w_dev, M, K, g, mp, kgt, static_cast<uint8_t*>(payload_dev));
  VLUT_CUDA_TRY(cudaGetLastError());
  // The mpGeMM kernels stage weight tiles BEFORE griddepcontrol.wait (the
  // payload is not an output of the previous kernel -- see vlut.h).  An
  // event record after the packing kernel makes the next launch on this
  // stream an ordinary (not programmatic) dependent: it starts only after
  // the packing kernel has completed and its stores are visible.
  {
    static std::mutex mu;
    static cudaEvent_t ev[64] = {};
    int dev = 0;
    VLUT_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!ev[dev & 63]) VLUT_CUDA_TRY(cudaEventCreateWithFlags(&ev[dev & 63], cudaEventDisableTiming));
    VLUT_CUDA_TRY(cudaEventRecord(ev[dev & 63], s));
  }
  *desc_out = d;
  return ok();
}

vlut_status vlut_pack_weights_device(const int8_t* w_dev, int M, int K, int g,
                                     void* payload_dev, size_t payload_bytes,
                                     vlut_packed_weights* desc_out, void* stream) {
  return vlut_pack_weights_device_ex(w_dev, M, K, g, 0, payload_dev, payload_bytes, desc_out,
                                     stream);
}

vlut_status vlut_unpack_weights_host(const vlut_packed_weights* desc, const uint8_t* payload,
                                     int8_t* w) {
  if (!desc || !payload || !w) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL argument");
  int mp = 0, kgt = 0;
  size_t bytes = 0;
  if (desc->magic != VLUT_MAGIC ||
      !layout_of(desc->M, desc->K, desc->g, desc->flags, &mp, &kgt, &bytes) ||
      desc->m_pad != mp || desc->kg_tiles != kgt)
    return fail(VLUT_ERR_CORRUPT_DESCRIPTOR, "bad descriptor");
  const int g = desc->g, K = desc->K, KG = (K + g - 1) / g, R = pow3i(g);
  for (int m = 0; m < desc->M; ++m)
    for (int k = 0; k < KG; ++k) {
      int idx = payload[((size_t)(k / VLUT_KG_TILE) * mp + m) * 16 + (k % VLUT_KG_TILE)];
      if (idx >= R) return fail(VLUT_ERR_INVALID_TRIT, "corrupt payload byte %d at (%d,%d)", idx, m, k);
      for (int r = 0; r < g; ++r) {
        if (k * g + r < K) w[(size_t)m * K + k * g + r] = (int8_t)(idx % 3 - 1);
        idx /= 3;
      }
    }
  return ok();
}

vlut_status vlut_plan(int M, int K, int N, int g, vlut_launch_plan* plan) {
  if (!plan) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL plan");
  if (M <= 0 || K <= 0 || N <= 0 || !valid_g(g)) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes");
  DeviceInfo d;
  vlut_status st = device_info(&d);
  if (st != VLUT_OK) return st;
  memset(plan, 0, sizeof(*plan));
  const double c = plan_for(M, K, N, g, d.sms, plan);
  vlut_launch_plan p32 = {};
  if (N % 16 == 0 && !getenv("VLUT_NO_K32") && plan_for32(M, K, N, g, d.sms, &p32) < c) *plan = p32;
  return ok();
}

vlut_status vlut_mpgemm(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                        float w_scale, float* out, int M, int K, int N, void* stream) {
  // the north-star signature has no workspace argument: use the library's
  // per-(device, stream) workspace so every schedule (stream-K, K2 split-K)
  // is available; without one, only the cluster schedules
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::lock_guard<std::mutex> lk(g_ws_mu);  // held through the launch (see above)
  if (M > 0 && N > 0) internal_workspace_locked(stream, &ws, &ws_bytes);
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, nullptr, stream, false, nullptr, 0, ws,
                    ws_bytes);
}

int vlut_cached_workspaces(void) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  return (int)g_ws.size();
}

vlut_status vlut_release_workspaces(void) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  int cur = 0;
  VLUT_CUDA_TRY(cudaGetDevice(&cur));
  vlut_status st = VLUT_OK;
  while (!g_ws.empty()) {
    WsEntry e = g_ws.back();
    cudaError_t err = cudaSetDevice(e.dev);
    if (err == cudaSuccess) err = cudaDeviceSynchronize();  // its stream may still use it
    if (err == cudaSuccess) err = cudaFree(e.ptr);
    if (err != cudaSuccess) {
      st = fail(VLUT_ERR_CUDA, "releasing a workspace on device %d: %s", e.dev,
                cudaGetErrorString(err));
      break;
    }
    g_ws.pop_back();
  }
  cudaSetDevice(cur);
  return st == VLUT_OK ? ok() : st;
}

vlut_status vlut_mpgemm_ex(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                           float w_scale, float* out, int M, int K, int N,
                           const vlut_launch_plan* plan, void* stream) {
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, plan, stream, false);
}

vlut_status vlut_mpgemm_acc(const vlut_packed_weights* W, const int8_t* A, int32_t* acc_out,
                            int M, int K, int N, const vlut_launch_plan* plan, void* stream) {
  return run_mpgemm(W, A, nullptr, 0.f, acc_out, M, K, N, plan, stream, true);
}

size_t vlut_workspace_bytes(void) {
  DeviceInfo d;
  if (device_info(&d) != VLUT_OK) return 0;
  return sk_workspace_bytes(d.sms);
}

vlut_status vlut_mpgemm_ws(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                           float w_scale, float* out, int M, int K, int N,
                           const vlut_launch_plan* plan, void* workspace, size_t ws_bytes,
                           void* stream) {
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, plan, stream, false, nullptr, 0,
                    workspace, ws_bytes);
}

vlut_status vlut_mpgemm_acc_ws(const vlut_packed_weights* W, const int8_t* A, int32_t* acc_out,
                               int M, int K, int N, const vlut_launch_plan* plan,
                               void* workspace, size_t ws_bytes, void* stream) {
  return run_mpgemm(W, A, nullptr, 0.f, acc_out, M, K, N, plan, stream, true, nullptr, 0,
                    workspace, ws_bytes);
}

vlut_status vlut_mpgemm_scalar_lut(const vlut_packed_weights* W, const int8_t* A,
                                   const float* a_scale, float w_scale, float* out, int M, int K,
                                   int N, const vlut_launch_plan* plan, void* workspace,
                                   size_t ws_bytes, void* stream) {
  vlut_launch_plan pl = {};
  if (plan) pl = *plan;
  pl.slot = 1;
  pl.tpw = 1;
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, &pl, stream, false, nullptr, 0,
                    workspace, ws_bytes);
}

vlut_status vlut_mpgemm_decode(const vlut_packed_weights* W, const float* x, float w_scale,
                               float* out, float* scale_out, int M, int K, void* workspace,
                               size_t ws_bytes, void* stream) {
  if (M < 0 || K <= 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes M=%d K=%d", M, K);
  if (M == 0) return ok();
  vlut_status st = check_desc(W, M, K);
  if (st != VLUT_OK) return st;
  if (!x || !out) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL device pointer");
  if ((((uintptr_t)x) | ((uintptr_t)out) | ((uintptr_t)scale_out)) & 3)
    return fail(VLUT_ERR_MISALIGNED, "x / out / scale_out not 4-B aligned");
  DeviceInfo d;
  st = device_info(&d);
  if (st != VLUT_OK) return st;
  std::unique_lock<std::mutex> lk(g_ws_mu, std::defer_lock);
  if (!workspace) {  // the library's per-stream workspace, as vlut_mpgemm
    lk.lock();
    internal_workspace_locked(stream, &workspace, &ws_bytes);
  }
  const bool have_ws = workspace && ws_bytes >= sk_workspace_bytes(d.sms) &&
                       ((uintptr_t)workspace & 15) == 0;
  vlut_launch_plan sl = {};
  plan_slot(M, K, 1, W->g, d.sms, 1, 1, 0, have_ws, &sl);  // one scalar word: N = 1
  return run_slot(W, nullptr, nullptr, w_scale, out, M, K, 1, sl, have_ws ? workspace : nullptr,
                  ws_bytes, stream, false, d, x, scale_out);
}

vlut_status vlut_mpgemm_allgather(const vlut_packed_weights* W, const int8_t* A,
                                  const float* a_scale, float w_scale, float* out_full, int M,
                                  int K, int N, int row0, void* const* peer_full, int n_peers,
                                  void* stream) {
  if (n_peers < 0 || n_peers > vlut::kMaxPeers)
    return fail(VLUT_ERR_INVALID_ARGUMENT, "n_peers must be in [0, %d]", vlut::kMaxPeers);
  if (!out_full || row0 < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad output / row0");
  if (n_peers > 0 && !peer_full) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL peer pointer table");
  for (int i = 0; i < n_peers; ++i)
    if (!peer_full[i] || (((uintptr_t)peer_full[i]) & 15))
      return fail(VLUT_ERR_MISALIGNED, "peer buffer %d NULL or not 16-B aligned", i);
  if (M == 0 || N == 0) return ok();
  g_peer_tls.n = n_peers;
  for (int i = 0; i < n_peers; ++i)
    g_peer_tls.ptr[i] = static_cast<float*>(peer_full[i]) + (size_t)row0 * N;
  // cluster schedule (its epilogue carries the peer stores)
  vlut_launch_plan pl = {};
  DeviceInfo d;
  vlut_status st = device_info(&d);
  if (st == VLUT_OK) {
    plan_for(M, K, N, W ? W->g : 4, d.sms, &pl);
    st = run_mpgemm(W, A, a_scale, w_scale, out_full + (size_t)row0 * N, M, K, N, &pl, stream,
                    false);
  }
  g_peer_tls.n = 0;
  return st;
}

vlut_status vlut_mpgemm_allgather_multicast(const vlut_packed_weights* W, const int8_t* A,
                                            const float* a_scale, float w_scale, float* out_mc,
                                            int M, int K, int N, int row0, void* stream) {
  if (!out_mc || row0 < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad output / row0");
  if (((uintptr_t)out_mc) & 15) return fail(VLUT_ERR_MISALIGNED, "multicast address not 16-B aligned");
  if (M == 0 || N == 0) return ok();
  g_peer_tls.n = 0;
  g_peer_tls.mc = 1;
  vlut_launch_plan pl = {};
  DeviceInfo d;
  vlut_status st = device_info(&d);
  if (st == VLUT_OK) {
    plan_for(M, K, N, W ? W->g : 4, d.sms, &pl);
    st = run_mpgemm(W, A, a_scale, w_scale, out_mc + (size_t)row0 * N, M, K, N, &pl, stream,
                    false);
  }
  g_peer_tls.mc = 0;
  return st;
}

vlut_status vlut_plan_ws(int M, int K, int N, int g, vlut_launch_plan* plan) {
  if (!plan) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL plan");
  if (M <= 0 || K <= 0 || N <= 0 || !valid_g(g)) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes");
  DeviceInfo d;
  vlut_status st = device_info(&d);
  if (st != VLUT_OK) return st;
  memset(plan, 0, sizeof(*plan));
  vlut_launch_plan skp = {}, slp = {};
  double c = plan_for(M, K, N, g, d.sms, plan);
  const double c_sk = plan_sk(M, K, N, g, d.sms, &skp);
  if (c_sk < c) {
    *plan = skp;
    c = c_sk;
  }
  vlut_launch_plan p32 = {}, s32 = {};
  if (N % 16 == 0 && !getenv("VLUT_NO_K32")) {
    const double c32 = plan_for32(M, K, N, g, d.sms, &p32);
    if (c32 < c) {
      *plan = p32;
      c = c32;
    }
    const double cs32 = plan_sk32(M, K, N, g, d.sms, &s32);
    if (cs32 < c) {
      *plan = s32;
      c = cs32;
    }
  }
  if (N <= kSlotAutoMaxN && plan_slot(M, K, N, g, d.sms, N == 1 ? 1 : 2, 0, 0, true, &slp) < c)
    *plan = slp;
  return ok();
}

vlut_status vlut_mpgemm_fused(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                              float w_scale, float* out, int M, int K, int N, const float* mul_in,
                              unsigned* amax_out, int amax_rows, const vlut_launch_plan* plan,
                              void* ws, size_t ws_bytes, void* stream) {
  if ((mul_in && (((uintptr_t)mul_in) & 3)) || (amax_out && (((uintptr_t)amax_out) & 3)))
    return fail(VLUT_ERR_MISALIGNED, "mul_in / amax_out not 4-B aligned");
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, plan, stream, false, nullptr, 0,
                    ws, ws_bytes, mul_in, amax_out, amax_rows < 0 ? 0 : amax_rows);
}

vlut_status vlut_quantize_amax(const float* x, const unsigned* amax, int K, int N, int8_t* q,
                               float* scale, void* stream) {
  if (K < 0 || N < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes");
  if (K == 0 || N == 0) return ok();
  if (!x || !amax || !q || !scale) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  DeviceInfo d;
  vlut_status st = device_info(&d);
  if (st != VLUT_OK) return st;
  const long long total = (long long)K * ((N + 3) / 4);
  long long blocks = (total + 255) / 256;
  if (blocks > (long long)d.sms * 8) blocks = (long long)d.sms * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_amax_kernel, x, amax, K, N, q, scale));
  return ok();
}

vlut_status vlut_group_schedule(int K, int* k5, int* k4) {
  if (!k5 || !k4) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL argument");
  for (int b = K / 5; b >= 0 && K >= 4; --b) {
    if ((K - 5 * b) % 4 == 0) {
      *k5 = 5 * b;
      *k4 = K - 5 * b;
      return ok();
    }
  }
  return fail(VLUT_ERR_SHAPE, "K=%d is not 5b + 4a with a, b >= 0", K);
}

vlut_status vlut_mpgemm_mixed_ws(const vlut_packed_weights* W5, const vlut_packed_weights* W4,
                                 const int8_t* A, const float* a_scale, float w_scale,
                                 float* out, int M, int K, int N, void* ws, size_t ws_bytes,
                                 void* stream);

vlut_status vlut_mpgemm_mixed(const vlut_packed_weights* W5, const vlut_packed_weights* W4,
                              const int8_t* A, const float* a_scale, float w_scale, float* out,
                              int M, int K, int N, void* stream) {
  return vlut_mpgemm_mixed_ws(W5, W4, A, a_scale, w_scale, out, M, K, N, nullptr, 0, stream);
}

vlut_status vlut_mpgemm_mixed_ws(const vlut_packed_weights* W5, const vlut_packed_weights* W4,
                                 const int8_t* A, const float* a_scale, float w_scale,
                                 float* out, int M, int K, int N, void* ws, size_t ws_bytes,
                                 void* stream) {
  int k5 = 0, k4 = 0;
  vlut_status st = vlut_group_schedule(K, &k5, &k4);
  if (st != VLUT_OK) return st;
  if (M == 0 || N == 0) return ok();
  if (k5 && (!W5 || W5->g != 5 || W5->K != k5))
    return fail(VLUT_ERR_SHAPE, "W5 must hold the first %d features with g=5", k5);
  if (k4 && (!W4 || W4->g != 4 || W4->K != k4))
    return fail(VLUT_ERR_SHAPE, "W4 must hold the last %d features with g=4", k4);
  if (!A) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL A");
  if (k4 == 0)
    return run_mpgemm(W5, A, a_scale, w_scale, out, M, k5, N, nullptr, stream, false, nullptr, 0,
                      ws, ws_bytes);
  if (k5 == 0)
    return run_mpgemm(W4, A, a_scale, w_scale, out, M, k4, N, nullptr, stream, false, nullptr, 0,
                      ws, ws_bytes);
  // g=5 groups first: raw int32 partial into `out` (same size), then the g=4
  // groups on the remaining activation rows add it before the fp32 epilogue
  st = run_mpgemm(W5, A, nullptr, 0.f, out, M, k5, N, nullptr, stream, true, nullptr, 0, ws,
                  ws_bytes);
  if (st != VLUT_OK) return st;
  return run_mpgemm(W4, A + (size_t)k5 * N, a_scale, w_scale, out, M, k4, N, nullptr, stream,
                    false, reinterpret_cast<const int32_t*>(out));
}

vlut_status vlut_mpgemm_layout(const vlut_packed_weights* W, const int8_t* A,
                               const float* a_scale, float w_scale, float* out, int M, int K,
                               int N, int flags, void* stream) {
  if (flags & ~VLUT_OUT_FEATURE_MAJOR) return fail(VLUT_ERR_INVALID_ARGUMENT, "unknown flags %d", flags);
  return run_mpgemm(W, A, a_scale, w_scale, out, M, K, N, nullptr, stream, false, nullptr,
                    (flags & VLUT_OUT_FEATURE_MAJOR) ? 1 : 0);
}

vlut_status vlut_quantize_t(const float* x, const float* y, int K, int N, int8_t* q,
                            float* scale, void* stream) {
  if (K < 0 || N < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes");
  if (K == 0 || N == 0) return ok();
  if (!x || !q || !scale) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long tok_blocks = (N + vlut::kQtTok - 1) / vlut::kQtTok;
  if (tok_blocks > 65535) return fail(VLUT_ERR_SHAPE, "N too large");
  // cluster size along K: >= 2 waves of CTAs when possible, slices <= 2048 rows
  int CL = 1;
  while (CL < 8 && (tok_blocks * CL < 296 || (long long)K > (long long)CL * 2048)) CL *= 2;
  while (CL > 1 && K < 4 * CL) CL /= 2;  // at least one float4 per CTA
  const int slice_max = (K + CL - 1) / CL + 4;
  const size_t smem = (size_t)slice_max * vlut::kQtTok;
  if (smem > 200 * 1024) return fail(VLUT_ERR_SHAPE, "K too large for vlut_quantize_t");
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(vlut::vlut_quantize_t_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  VLUT_CUDA_TRY(attr);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)CL, (unsigned)tok_blocks, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_t_kernel, x, y, K, N, q, scale));
  return ok();
}

vlut_status vlut_linear(const vlut_packed_weights* W, const float* x, float w_scale, float* y,
                        int M, int K, int N, int8_t* q_ws, float* s_ws, void* stream) {
  if (!q_ws || !s_ws) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL workspace");
  vlut_status st = vlut_quantize_t(x, nullptr, K, N, q_ws, s_ws, stream);
  if (st != VLUT_OK) return st;
  return vlut_mpgemm_layout(W, q_ws, s_ws, w_scale, y, M, K, N, VLUT_OUT_FEATURE_MAJOR, stream);
}

vlut_status vlut_quantize(const float* x, const float* y, int K, int N, int8_t* q, float* scale,
                          void* stream) {
  return vlut_quantize_ex(x, y, K, N, q, scale, 0, stream);
}

vlut_status vlut_quantize_ex(const float* x, const float* y, int K, int N, int8_t* q,
                             float* scale, int cluster, void* stream) {
  if (!(cluster == 0 || cluster == 1 || cluster == 2 || cluster == 4 || cluster == 8))
    return fail(VLUT_ERR_INVALID_ARGUMENT, "cluster must be 0, 1, 2, 4 or 8");
  if (K < 0 || N < 0) return fail(VLUT_ERR_INVALID_ARGUMENT, "bad sizes");
  if (K == 0 || N == 0) return ok();
  if (!x || !q || !scale) return fail(VLUT_ERR_INVALID_ARGUMENT, "NULL pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // decode shapes (N in {1,2,4,8,16}, flat float4 access possible, fits the
  // register cache of one cluster): K3f, one cluster over the flat array
  {
    const long long total4 = (long long)K * N / 4;
    const bool pow2n = N == 1 || N == 2 || N == 4 || N == 8 || N == 16;
    const bool flat_ok = pow2n && ((long long)K * N) % 4 == 0 &&
                         ((((uintptr_t)x) | ((uintptr_t)(y ? y : x))) & 15) == 0 &&
                         (((uintptr_t)q) & 3) == 0 &&
                         total4 <= (long long)vlut::kQfMaxCL * vlut::kQfThreads * vlut::kQfCache;
    if (flat_ok && !cluster && !getenv("VLUT_NO_QFLAT")) {
      // CTAs: ~2 float4 per thread in flight, at most one cluster of 8
      long long CLl = (total4 + 2LL * vlut::kQfThreads - 1) / (2LL * vlut::kQfThreads);
      while (CLl < vlut::kQfMaxCL && total4 > CLl * vlut::kQfThreads * vlut::kQfCache) ++CLl;
      const int CLf = (int)std::max(1LL, std::min<long long>(vlut::kQfMaxCL, CLl));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)CLf, 1, 1);
      cfg.blockDim = dim3(vlut::kQfThreads, 1, 1);
      cfg.stream = s;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)CLf;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      if (y)
        VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_flat_kernel<true>, x, y, K, N, q, scale));
      else
        VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_flat_kernel<false>, x, y, K, N, q, scale));
      return ok();
    }
  }
  // cluster size along K: enough CTAs that every row fits the register cache
  // when possible (<= 8, portable), and >= ~2 waves of CTAs over the GPU.
  const long long tok_blocks = (N + vlut::kQTok - 1) / vlut::kQTok;
  int CL = 1;
  while (CL < 8 && ((long long)K > (long long)CL * vlut::kQRows * vlut::kQCache || tok_blocks * CL < 296))
    CL *= 2;
  if (CL > K) CL = 1;
  if (cluster) CL = cluster;  // caller-chosen (e.g. 1: fits the SMs a concurrent mpGeMM leaves idle)
  if (const char* e = getenv("VLUT_QCL")) {  // (development A/B knob)
    const int c = atoi(e);
    if (c == 1 || c == 2 || c == 4 || c == 8) CL = c;
  }
  if (tok_blocks > 65535) return fail(VLUT_ERR_SHAPE, "N too large");
  const bool aligned = (N % 4 == 0) && ((((uintptr_t)x) | ((uintptr_t)(y ? y : x))) & 15) == 0 &&
                       (((uintptr_t)q) & 3) == 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)CL, (unsigned)tok_blocks, 1);
  cfg.blockDim = dim3(vlut::kQThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the prologue overlaps the previous kernel
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (aligned)
    VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_kernel<true>, x, y, K, N, q, scale));
  else
    VLUT_CUDA_TRY(cudaLaunchKernelEx(&cfg, vlut::vlut_quantize_kernel<false>, x, y, K, N, q, scale));
  return ok();
}

}  // extern "C"
