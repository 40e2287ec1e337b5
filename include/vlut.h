/*
 * vlut.h -- C ABI of libvlut.so: the B200 (sm_100a) Vec-LUT ternary mpGeMM.
 *
 * Method: Vec-LUT, arXiv 2512.06443.  "P:n" cites /root/reference/PAPER.md
 * line n (LaTeX source), "S:n" SPEC.md line n.  The notation follows the
 * paper's Table 2: W x A = O, W in {-1,0,1}^{M x K} (ternary
 * weights), A in int8^{K x N} (activations, token axis N contiguous,
 * P:430-434), O in R^{M x N} (output, token axis contiguous).  g in {4,5} is
 * the weight group size; a group of g trits is one base-3 byte index
 * into a 3^g-row table of the group's signed
 * activation sums (Eq. 1).
 *
 * Conventions for every entry point:
 *   - Plain C types only.  "dev" pointers are CUDA device pointers, "host"
 *     pointers are ordinary host memory.  `stream` is a cudaStream_t passed
 *     as void* (0 = legacy default stream).
 *   - The caller owns every buffer.  The library allocates device memory in
 *     one place only: vlut_mpgemm (the north-star signature, which has no
 *     workspace argument) keeps a bounded cache of workspaces (~60 MB each on
 *     B200): at most 4 per device, each bound to one stream by its
 *     process-unique id (cudaStreamGetId -- a destroyed-then-recycled stream
 *     handle never aliases an old entry).  Created and zeroed on a stream's
 *     first call; a fifth stream takes the least recently used entry after a
 *     device-wide synchronisation.  Never allocated, evicted or used inside a
 *     stream capture (a captured vlut_mpgemm runs the cluster schedule).
 *     vlut_release_workspaces() frees them all.  Other global state: a
 *     thread-local error string and per-device property/attribute caches.
 *   - Weight payloads are read before the kernels' griddepcontrol.wait
 *     (programmatic dependent launch overlaps the weight stream with the
 *     tail of the previous kernel): a payload must NOT be written by the
 *     kernel launched immediately before an mpGeMM call on the same stream.
 *     Payloads written by vlut_pack_weights (which synchronises) and
 *     vlut_pack_weights_device (which ends with an event record on its
 *     stream, turning the next launch into an ordinary dependent) satisfy
 *     this.  Activations, scales and accumulators may come from the previous
 *     kernel.
 *   - Arguments are validated on the host before anything is launched.  On
 *     failure nothing is launched, a status != VLUT_OK is returned and
 *     vlut_last_error() describes it.  Nothing aborts or throws across the ABI.
 *   - Work is enqueued on `stream` and is asynchronous: a device fault
 *     surfaces at the caller's next synchronisation, not as a return value.
 *   - Results are deterministic and bit-identical for every launch plan
 *     (integer accumulation is exact and associative; fp32 epilogue op order
 *     is fixed).
 *   - Thread-safe and reentrant for distinct output buffers.
 */
#ifndef VLUT_H_
#define VLUT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VLUT_OK = 0,
  VLUT_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative size, bad g     */
  VLUT_ERR_INVALID_TRIT = 2,     /* a weight outside {-1,0,1}      */
  VLUT_ERR_SHAPE = 3,            /* g does not divide K, M/K/N mismatch with the descriptor, size overflow */
  VLUT_ERR_BUFFER_TOO_SMALL = 4, /* payload buffer smaller than vlut_packed_bytes() */
  VLUT_ERR_MISALIGNED = 5,       /* a device pointer not aligned as documented */
  VLUT_ERR_CORRUPT_DESCRIPTOR = 6, /* bad magic/version/fields in vlut_packed_weights */
  VLUT_ERR_CUDA = 7,             /* a CUDA runtime call or launch failed   */
  VLUT_ERR_UNSUPPORTED = 8       /* a plan the device cannot run (e.g. cluster size) */
} vlut_status;

#define VLUT_MAGIC 0x31544C56u /* "VLT1" little-endian */
#define VLUT_VERSION 1u
#define VLUT_KG_TILE 16 /* groups per packed K-tile (one 16-byte index vector per row) */
#define VLUT_M_TILE 32  /* row padding granularity of the packed payload */

/*
 * Packed ternary weights (a1; P:284 offline stage, P:436-441 tile-contiguous
 * layout).  A POD value the caller keeps next to the payload buffer.
 *
 * Payload layout (device, `payload_bytes` bytes, 16-byte aligned):
 *   byte payload[kt][m][j]   kt in [0, kg_tiles), m in [0, m_pad), j in [0,16)
 *   = index of group (kt*16 + j) of weight row m, where group k of row m
 *     covers features k*g .. k*g+g-1 (reading c4) and
 *     index = sum_{r<g} (W[m][k*g+r] + 1) * 3^r  (Alg. 1 GetSign, P:382;
 *     least-significant trit first, reading c1).
 *   With VLUT_PACK_PAD_K, K need not be a multiple of g: the last group
 *   reads zero trits for its features >= K (they contribute exactly 0).
 *   Rows m >= M and groups k >= ceil(K/g) hold the all-zero index (3^g-1)/2
 *   (40 for g=4, 121 for g=5) and contribute exactly 0.
 * The K-tile index is outermost, matching the K->M loop order of Alg. 1
 * (P:441); within a tile the 16 index bytes of one row are contiguous so one
 * 16-byte load fetches a row's indices for 16 groups, and a CTA's rows of one
 * K-tile form one contiguous, coalesced block.
 */
typedef struct {
  uint32_t magic;          /* VLUT_MAGIC                                  */
  uint32_t version;        /* VLUT_VERSION                                */
  int32_t M, K, g;         /* logical shape; g in {4,5}                   */
  int32_t m_pad;           /* M rounded up to VLUT_M_TILE                 */
  int32_t kg_tiles;        /* ceil(ceil(K/g) / VLUT_KG_TILE)              */
  int32_t m_tile, kg_tile; /* VLUT_M_TILE, VLUT_KG_TILE                   */
  int32_t flags;           /* 0, or VLUT_PACK_PAD_K                        */
  int64_t payload_bytes;   /* kg_tiles * m_pad * 16                        */
  const void* payload;     /* device pointer (caller-owned)               */
} vlut_packed_weights;

/*
 * Launch plan of the fused mpGeMM kernel (K1).  m_cta = 32*warps output rows
 * per CTA, n_cta = 64 tokens per CTA, `splits` CTAs of one thread-block
 * cluster share an (M-block, N-tile) and split its K range; their int32
 * partials are reduced through distributed shared memory (a5).
 */
typedef struct {
  int32_t warps;        /* 8, 12 or 16                                      */
  int32_t splits;       /* 1..8 (cluster size along K)                        */
  int32_t m_cta;        /* 32 * warps; stream-K only: 64 * warps (8 or 12
                           warps) = two output rows per lookup thread       */
  int32_t n_cta;        /* 64                                               */
  int32_t grid_ctas;    /* total CTAs launched                              */
  int32_t smem_bytes;   /* dynamic shared memory per CTA                    */
  int32_t streamk;      /* 1: stream-K persistent schedule (needs a workspace) */
  int32_t slot;         /* 1: K2 lane-slot kernel (small N / decode / scalar-LUT comparator):
                           m_cta = 1024 (g=4) or 2048 (g=5), n_cta = nw * tpw, `splits`
                           CTAs along K (> 1 needs a workspace)                       */
  int32_t tpw;          /* K2 tokens per 4-byte table word: 1 = scalar LUT (1->1 lookups,
                           one table per token), 2 = vector LUT (1->2)       */
  int32_t nw;           /* K2 table words per lookup: 1, 2, 4 or 8 (g=5: 1 or 2)      */
} vlut_launch_plan;

/* Payload bytes for an M x K ternary matrix packed with group size g
 * (kg_tiles * m_pad * 16).  Returns 0 if the arguments are invalid (M<=0,
 * K<=0, g not in {4,5}, g does not divide K) or the size overflows. */
size_t vlut_packed_bytes(int M, int K, int g);

/* Packing flag: K need not be a multiple of g; the last group of every row is
 * completed with zero trits (features >= K; the kernels read those activation
 * rows as 0).  The same ceil(K/5) bytes per row as the paper's mixed g=5/g=4
 * schedule -- never more -- but one g for the whole K range, so
 * one launch.  A B200 alternative to the mixed schedule. */
#define VLUT_PACK_PAD_K 1

/* vlut_packed_bytes / vlut_pack_weights / vlut_pack_weights_device with
 * packing flags (0 = the plain functions). */
size_t vlut_packed_bytes_ex(int M, int K, int g, int flags);
vlut_status vlut_pack_weights_ex(const int8_t* w_trits_host, int M, int K, int g, int flags,
                                 void* payload_dev, size_t payload_bytes,
                                 vlut_packed_weights* desc_out, void* stream);
vlut_status vlut_pack_weights_device_ex(const int8_t* w_trits_dev, int M, int K, int g, int flags,
                                        void* payload_dev, size_t payload_bytes,
                                        vlut_packed_weights* desc_out, void* stream);

/*
 * Pack ternary weights (a1, offline).
 *   w_trits_host : host, int8 [M][K] row-major, values in {-1,0,1}.
 *   payload_dev  : device, >= vlut_packed_bytes(M,K,g) bytes, 16-B aligned.
 *   desc_out     : host, filled on success (payload = payload_dev).
 * Validates every trit (VLUT_ERR_INVALID_TRIT, nothing written), packs on the
 * host and copies to the device with cudaMemcpyAsync on `stream`, then
 * synchronises `stream` (the host staging buffer is freed before return).
 */
vlut_status vlut_pack_weights(const int8_t* w_trits_host, int M, int K, int g,
                              void* payload_dev, size_t payload_bytes,
                              vlut_packed_weights* desc_out, void* stream);

/*
 * Same packing, done on the device from device-resident trits (for large
 * weights; one launch, asynchronous).  Invalid trits are not detected here
 * beyond being mapped into range; use vlut_pack_weights for validation.
 *   w_trits_dev : device int8 [M][K].   Other arguments as above.
 */
vlut_status vlut_pack_weights_device(const int8_t* w_trits_dev, int M, int K, int g,
                                     void* payload_dev, size_t payload_bytes,
                                     vlut_packed_weights* desc_out, void* stream);

/* Inverse of the packing, on the host (tests, checkpoint export):
 * payload_host (kg_tiles*m_pad*16 bytes, as described by desc) -> int8 trits
 * [M][K].  Returns VLUT_ERR_INVALID_TRIT on a byte >= 3^g (corrupt payload,
 * S:164).  Padding bytes are not inspected. */
vlut_status vlut_unpack_weights_host(const vlut_packed_weights* desc,
                                     const uint8_t* payload_host, int8_t* w_trits_host);

/* Planner input: co-resident thread-block clusters of `splits` K1 CTAs of
 * the (g, warps) variant on the current device (cudaOccupancyMaxActiveClusters);
 * -1 if that cluster size cannot run, 0 on bad arguments. */
int vlut_active_clusters(int g, int warps, int splits);

/* The heuristic launch plan for (M, K, N, g) on the current device. */
vlut_status vlut_plan(int M, int K, int N, int g, vlut_launch_plan* plan);

/*
 * Vec-LUT mpGeMM with fp32 dequant epilogue (a2-a6):
 *   out[m][n] = fl( (float)acc[m][n] * fl(a_scale[n] * w_scale) )
 *   acc[m][n] = sum_k W[m][k] * A[k][n]   (exact int32; Alg. 1 + Eq. 2,
 *              P:326-351; tables per Eq. 1, topological order
 *              P:503-513; INT16->INT32 hierarchical accumulation P:483-491)
 *   W       : packed weights (desc->M == M, desc->K == K).
 *   A       : device int8 [K][N], token axis contiguous; any
 *             int8 value including -128.
 *   a_scale : device fp32 [N], per-token activation scale.
 *   w_scale : per-tensor weight scale (reading c7).
 *   out     : device fp32 [M][N], token axis contiguous.
 * M == 0 or N == 0 is a no-op returning VLUT_OK.  A, out need 4-byte
 * alignment; 16-byte alignment and N % 16 == 0 take the vectorised path.
 * The planner may choose any schedule (cluster split-K, stream-K, K2 for small
 * N) using the library's workspace for `stream` (see Conventions).
 */
vlut_status vlut_mpgemm(const vlut_packed_weights* W, const int8_t* A,
                        const float* a_scale, float w_scale, float* out,
                        int M, int K, int N, void* stream);

/* As vlut_mpgemm with an explicit plan (NULL = heuristic).  Any valid plan
 * gives bit-identical results. */
vlut_status vlut_mpgemm_ex(const vlut_packed_weights* W, const int8_t* A,
                           const float* a_scale, float w_scale, float* out,
                           int M, int K, int N, const vlut_launch_plan* plan,
                           void* stream);

/*
 * Stream-K persistent schedule (one CTA per SM; every SM gets the same number
 * of K-tile work units whatever the tile count; split tiles are combined
 * through int32 partials in a caller-provided workspace).  Same results as
 * vlut_mpgemm.  The planner picks stream-K, the cluster split-K schedule or,
 * for small N, the K2 lane-slot kernel (split-K through the workspace) by its
 * cost model (plan == NULL) unless plan->streamk / plan->slot forces one.
 *   workspace : device, >= vlut_workspace_bytes() bytes, 16-B aligned, ZEROED
 *               ONCE before its first use, and used by one stream at a time.
 *               Regions: stream-K partials and partial-ready flags (each
 *               flag is set by its producer CTA and reset by its consumer in
 *               the same launch), K2 split-K arrival counts and int32
 *               accumulators (at decode-size tiles: counted 64-bit words,
 *               count << 40 | biased sum; every K2 launch leaves them zero
 *               again) and
 *               per-tile generation words (monotonic, read on the device),
 *               and K1-32-SK fp32 split-tile accumulators (producers red.add
 *               integer-valued partials, exact below 2^24; the tile's owner
 *               reads and re-zeroes them in the same launch).
 *               No host-side per-launch state: captured CUDA graphs may be
 *               replayed.  A launch that fails asynchronously can leave the
 *               zero-kept regions dirty: re-zero the workspace before reusing
 *               it after any CUDA error.  Stream-K and K2 split-K launches whose CTAs
 *               wait for each other are cooperative (all co-resident);
 *               K2's decode-size tiles meet without waiting and are not.
 * vlut_workspace_bytes() returns 0 without a CUDA device (~60 MB on B200).
 */
size_t vlut_workspace_bytes(void);
vlut_status vlut_mpgemm_ws(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                           float w_scale, float* out, int M, int K, int N,
                           const vlut_launch_plan* plan, void* workspace, size_t ws_bytes,
                           void* stream);
vlut_status vlut_mpgemm_acc_ws(const vlut_packed_weights* W, const int8_t* A, int32_t* acc_out,
                               int M, int K, int N, const vlut_launch_plan* plan,
                               void* workspace, size_t ws_bytes, void* stream);
/* The plan vlut_mpgemm_ws would choose (stream-K or cluster split-K). */
vlut_status vlut_plan_ws(int M, int K, int N, int g, vlut_launch_plan* plan);

/*
 * Scalar-LUT comparator and decode path (f4):
 * the K2 kernel with one table PER TOKEN and one 1->1 lookup per (row, group,
 * token) -- the T-MAC paradigm the paper contrasts with Vec-LUT -- laid out
 * so every lookup is a conflict-free 4-byte shared-memory read.  At N = 1 it
 * is also the Vec-LUT (one token: the two paradigms coincide) and the planner
 * uses it for decode.  Same results and contract as vlut_mpgemm_ws
 * (workspace may be NULL: then no split-K).  plan may be NULL (heuristic
 * nw); plan->slot/tpw are forced to 1/1.
 */
vlut_status vlut_mpgemm_scalar_lut(const vlut_packed_weights* W, const int8_t* A,
                                   const float* a_scale, float w_scale, float* out, int M, int K,
                                   int N, const vlut_launch_plan* plan, void* workspace,
                                   size_t ws_bytes, void* stream);

/*
 * Fused decode step (one token, N = 1): the per-token int8 quantization of
 * the activation (s = absmax / 127, 1 if absmax is 0; q =
 * clamp(round-half-away(x / s), +-127)) and the scalar-LUT mpGeMM + fp32
 * dequant of vlut_mpgemm_scalar_lut in ONE launch: every CTA of the K2 decode
 * kernel takes the absmax of x itself and its table builders quantize the
 * features they need, so there is no quantizer launch and no int8 round trip
 * (the scalar LUT for decoding).  Results are bit-identical to
 * vlut_quantize followed by vlut_mpgemm_scalar_lut.
 *   x         : device fp32 [K] (the token's activations; 16-B alignment and
 *               K % 4 == 0 take the vector path), may be the previous
 *               kernel's output (read after griddepcontrol.wait)
 *   out       : device fp32 [M]
 *   scale_out : device fp32 [1] <- s, or NULL
 *   workspace : as vlut_mpgemm_ws, or NULL for the library's per-stream one
 * Errors: INVALID_ARGUMENT, SHAPE / CORRUPT_DESCRIPTOR (descriptor), MISALIGNED
 * (x / out / scale_out not 4-B aligned), CUDA.
 */
vlut_status vlut_mpgemm_decode(const vlut_packed_weights* W, const float* x, float w_scale,
                               float* out, float* scale_out, int M, int K, void* workspace,
                               size_t ws_bytes, void* stream);

/* Raw int32 accumulators, no scales (bit-exact test hook):
 *   acc_out : device int32 [M][N].  Other arguments as vlut_mpgemm_ex. */
vlut_status vlut_mpgemm_acc(const vlut_packed_weights* W, const int8_t* A,
                            int32_t* acc_out, int M, int K, int N,
                            const vlut_launch_plan* plan, void* stream);

/*
 * Flexible sub-2-bit packing: split K into b groups of
 * g=5 followed by a groups of g=4, 5b + 4a = K, b maximal.  k5 = 5b, k4 = 4a
 * features.  VLUT_ERR_SHAPE if K has no such split (K in {1,2,3,6,7,11}).
 */
vlut_status vlut_group_schedule(int K, int* k5, int* k4);

/*
 * mpGeMM over a mixed schedule: W5 packs features [0, k5) with g=5 (NULL if
 * k5 == 0), W4 packs features [k5, K) with g=4 (NULL if k4 == 0); both have
 * M rows.  Same result and contract as vlut_mpgemm on the whole K (two
 * launches: the g=5 part writes raw int32 partials into `out`, the g=4 part
 * adds them before the fp32 epilogue).
 */
vlut_status vlut_mpgemm_mixed(const vlut_packed_weights* W5, const vlut_packed_weights* W4,
                              const int8_t* A, const float* a_scale, float w_scale, float* out,
                              int M, int K, int N, void* stream);
/* Same with a stream-K workspace (see vlut_mpgemm_ws; may be NULL). */
vlut_status vlut_mpgemm_mixed_ws(const vlut_packed_weights* W5, const vlut_packed_weights* W4,
                                 const int8_t* A, const float* a_scale, float w_scale,
                                 float* out, int M, int K, int N, void* ws, size_t ws_bytes,
                                 void* stream);

/*
 * Fused feature-major transpositions: frameworks hold activations
 * and outputs as [N][K] / [N][M] (feature axis contiguous).
 *   flags & VLUT_OUT_FEATURE_MAJOR: `out` is written as [N][M] (the K1
 *   epilogue writes the transposed tile; same values as vlut_mpgemm).
 */
#define VLUT_OUT_FEATURE_MAJOR 1
vlut_status vlut_mpgemm_layout(const vlut_packed_weights* W, const int8_t* A,
                               const float* a_scale, float w_scale, float* out, int M, int K,
                               int N, int flags, void* stream);

/* vlut_quantize on feature-major input: x, y device fp32 [N][K] (y may be
 * NULL) -> q device int8 [K][N] (token-contiguous, the layout the mpGeMM
 * consumes) and scale [N]; same codes and scales as vlut_quantize(x^T). */
vlut_status vlut_quantize_t(const float* x, const float* y, int K, int N, int8_t* q,
                            float* scale, void* stream);

/* A framework-layout ternary linear: y[N][M] = dequant(W x quant(x)^T) for
 * x fp32 [N][K]; q_ws (int8 [K][N]) and s_ws (fp32 [N]) are caller-provided
 * device workspaces.  Two launches (vlut_quantize_t, vlut_mpgemm_layout). */
vlut_status vlut_linear(const vlut_packed_weights* W, const float* x, float w_scale, float* y,
                        int M, int K, int N, int8_t* q_ws, float* s_ws, void* stream);

/*
 * Fused re-quantization (f1): vlut_mpgemm_ws (ws may be NULL: cluster schedule
 * only; plan may be NULL: the planner chooses, as in vlut_mpgemm_ws) whose epilogue
 * optionally multiplies the fp32 output element-wise by mul_in [M][N]
 * (config 5's gate (.) up glue: out = fl(out * mul_in)) and atomically maxes
 * |out| of rows m < amax_rows into amax_out[N] (IEEE float bits as unsigned;
 * the caller zeroes amax_out before the call).  mul_in / amax_out may be NULL.
 * vlut_quantize_amax then quantizes x [K][N] with those maxima in one pass
 * (s = amax/127, 1 if 0; q = clamp(roundf(x/s), +-127)) -- the same codes and
 * scales as vlut_quantize(x).  In the row-sharded path the per-rank maxima
 * are all-reduced (MAX) before quantizing, and int8 shards are gathered.
 */
vlut_status vlut_mpgemm_fused(const vlut_packed_weights* W, const int8_t* A, const float* a_scale,
                              float w_scale, float* out, int M, int K, int N, const float* mul_in,
                              unsigned* amax_out, int amax_rows, const vlut_launch_plan* plan,
                              void* ws, size_t ws_bytes, void* stream);
vlut_status vlut_quantize_amax(const float* x, const unsigned* amax, int K, int N, int8_t* q,
                               float* scale, void* stream);

/*
 * Row-sharded mpGeMM with the all-gather fused into the epilogue (a8, §8e):
 * this rank computes rows [row0, row0 + M) of an [M_total][N] output (W holds
 * those M rows) and its K1 epilogue stores every 16-byte output unit to
 *   out_full + row0*N (local, device)  and  peer_full[i] + row0*N, i < n_peers
 * -- the other ranks' full output buffers, mapped into this process (CUDA IPC
 * / symmetric memory; NVLink P2P stores), so the gather overlaps the other
 * CTAs' compute instead of following the kernel.  The caller orders the
 * peers' reads after every rank's launch (a cross-GPU barrier on the stream).
 *   peer_full : host array of n_peers device pointers (each 16-B aligned,
 *               >= (row0 + M) * N floats); n_peers <= 7 (8 GPUs).
 * Cluster split-K schedule; plain fp32 epilogue.  Same values as vlut_mpgemm.
 */
vlut_status vlut_mpgemm_allgather(const vlut_packed_weights* W, const int8_t* A,
                                  const float* a_scale, float w_scale, float* out_full, int M,
                                  int K, int N, int row0, void* const* peer_full, int n_peers,
                                  void* stream);

/*
 * The same with the all-gather done by the NVSwitch (NVLS multicast): out_mc
 * is the multicast address of the ranks' [M_total][N] fp32 buffers (e.g.
 * torch symmetric memory's multicast_ptr; 16-B aligned).  The K1 epilogue
 * stores every 16-byte unit ONCE, with multimem.st (the only access PTX
 * defines on a multimem address), and the switch replicates it into every
 * rank's copy, this rank's included.  Ordering as above (a cross-GPU barrier
 * before any rank reads).  Errors: VLUT_ERR_INVALID_ARGUMENT (NULL address,
 * row0 < 0), VLUT_ERR_MISALIGNED; otherwise as vlut_mpgemm.
 */
vlut_status vlut_mpgemm_allgather_multicast(const vlut_packed_weights* W, const int8_t* A,
                                            const float* a_scale, float w_scale, float* out_mc,
                                            int M, int K, int N, int row0, void* stream);

/*
 * Per-token absmax int8 quantizer (a7; w1.6A8 named at P:102; formula
 * S:339-347, reading c8), IEEE single precision throughout:
 *   x'[k][n] = x[k][n] * (y ? y[k][n] : 1)      (fp32 multiply, config 5's
 *                                                gate (.) up glue, c14)
 *   amax_n = max_k |x'[k][n]|, s_n = amax_n / 127 (1 if amax_n == 0)
 *   q[k][n] = clamp(roundf(x'[k][n] / s_n), -127, 127)
 *   x, y : device fp32 [K][N] (y may be NULL);  q : device int8 [K][N];
 *   scale : device fp32 [N].
 * Non-finite inputs are not detected (the caller's responsibility).
 */
vlut_status vlut_quantize(const float* x, const float* y, int K, int N,
                          int8_t* q, float* scale, void* stream);

/*
 * vlut_quantize with the K3 cluster size chosen by the caller: cluster 0 =
 * the library's choice (== vlut_quantize); 1, 2, 4 or 8 = that many CTAs per
 * 16-token block (fewer, narrower launches).  Cluster 1 is for running the
 * quantizer of the NEXT independent batch on a second stream while an
 * mpGeMM holds most SMs: its one-CTA clusters fit the SMs the mpGeMM grid
 * leaves free (configs[1]: 144 of 148), where an 8-CTA cluster would wait
 * for the mpGeMM to finish (profiles/r02_pipeline.txt).  Same codes and
 * scales, bit for bit, for every cluster size.  Errors as vlut_quantize, and
 * VLUT_ERR_INVALID_ARGUMENT for any other cluster value.
 */
vlut_status vlut_quantize_ex(const float* x, const float* y, int K, int N, int8_t* q,
                             float* scale, int cluster, void* stream);

/* The library's vlut_mpgemm workspaces (see Conventions): the number
 * currently cached (all devices), and a release of all of them (synchronises
 * each device that holds one, then frees; the next vlut_mpgemm call on a
 * stream re-creates its workspace).  Call release only when no other thread
 * is inside a libvlut call. */
int vlut_cached_workspaces(void);
vlut_status vlut_release_workspaces(void);

/* Number of kernel launches one vlut_mpgemm/vlut_mpgemm_acc call enqueues
 * (1: the whole path, split-K reduction included, is one cluster launch). */
int vlut_launches_per_mpgemm(void);

/* Message for the last failing call on this thread ("" if none). */
const char* vlut_last_error(void);

/* Library version string. */
const char* vlut_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VLUT_H_ */
