// gather.cu -- Gather and Stitch row movers, plus the library's
// status/diagnostic entry points.
//
// Both movers are HBM-bound row copies: one warp per row, 16-byte vector
// accesses (a 512-wide fp32 row is 128 float4 = 4 per lane), two rows in flight per warp.  A
// shared-memory-staged bulk-TMA Gather (gather_bulk_kernel) is kept as a measured alternative
// (TFS_GATHER_BULK=1 builds; slower on B200, see there).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace tfs {

static thread_local char g_last_error[512] = {0};
static std::atomic<long long> g_launches{0};

void launched(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_last_error(const char* where, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorName(e),
           cudaGetErrorString(e));
}

int32_t device_supported() {
  static std::mutex mu;
  static int cached[64];
  static bool init = false;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return TFS_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lk(mu);
  if (!init) {
    for (int i = 0; i < 64; ++i) cached[i] = -1;
    init = true;
  }
  if (cached[dev] < 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached[dev] = (major == 10 && minor == 0) ? TFS_OK : TFS_ERR_UNSUPPORTED;
  }
  return cached[dev];
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TFS_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return kNumSMsB200;
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : kNumSMsB200;
  }
  return cached[dev];
}

// ------------------------------------------------------------------------------------------------
// table2 / out2 (nullable): a width-1 companion gathered with the same ids (e.g. b with W).
template <bool BF16OUT>
__global__ void __launch_bounds__(256) gather_vec4_kernel(const float* __restrict__ table,
                                                          int64_t rows, int32_t dim,
                                                          const int64_t* __restrict__ ids,
                                                          int64_t n, void* __restrict__ out,
                                                          const float* __restrict__ table2,
                                                          float* __restrict__ out2,
                                                          tfs_device_error* err) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int n4 = dim >> 2;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t j0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 2; j0 < n; j0 += nwarps * 2) {
    int64_t id[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u;
      id[u] = j < n ? __ldg(ids + j) : 0;
      ok[u] = j < n && id[u] >= 0 && id[u] < rows;
      if (j < n && !ok[u] && id[u] != -1 && lane == 0) report_error(err, TFS_ERR_OUT_OF_RANGE, j);
    }
    if (table2 != nullptr && lane < 2) {  // lanes 0 / 1: the companion values of the two rows
      const bool okl = lane == 0 ? ok[0] : ok[1];
      if (okl) out2[j0 + lane] = __ldg(table2 + (lane == 0 ? id[0] : id[1]));
    }
    for (int c0 = 0; c0 < n4; c0 += 128) {  // 4 float4 per lane per row per sweep
      float4 v[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4* src = (const float4*)(table + id[u] * dim);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          v[u][q] = (ok[u] && c < n4) ? __ldg(src + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
        const int64_t j = j0 + u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          if (c >= n4) continue;
          if (BF16OUT) {
            uint2 p;
            p.x = pack_bf16x2(v[u][q].x, v[u][q].y);
            p.y = pack_bf16x2(v[u][q].z, v[u][q].w);
            ((uint2*)out)[j * n4 + c] = p;
          } else {
            ((float4*)out)[j * n4 + c] = v[u][q];
          }
        }
      }
    }
  }
}

template <bool BF16OUT>
__global__ void gather_scalar_kernel(const float* __restrict__ table, int64_t rows, int32_t dim,
                                     const int64_t* __restrict__ ids, int64_t n,
                                     void* __restrict__ out, tfs_device_error* err) {
  pdl_enter();
  const int64_t total = n * dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / dim;
    const int c = (int)(e - j * dim);
    const int64_t id = ids[j];
    if (id < 0 || id >= rows) {
      if (c == 0 && id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, j);
      continue;
    }
    const float v = table[id * dim + c];
    if (BF16OUT)
      ((uint16_t*)out)[e] = f32_to_bf16_bits(v);
    else
      ((float*)out)[e] = v;
  }
}

// Stitch: out[positions[j]] = rows[j].  With validation, claim[p] = min j claiming p.
__global__ void stitch_claim_kernel(const int64_t* positions, int64_t n,
                                    unsigned long long* claim, tfs_device_error* err) {
  pdl_enter();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = positions[j];
    if (p < 0 || p >= n)
      report_error(err, TFS_ERR_BAD_POSITIONS, j);
    else
      atomicMin(claim + p, (unsigned long long)j);
  }
}

__global__ void __launch_bounds__(256) stitch_vec4_kernel(const int64_t* __restrict__ positions,
                                                          const uint4* __restrict__ rows,
                                                          int64_t n, int64_t row_vecs,
                                                          uint4* __restrict__ out,
                                                          const unsigned long long* claim,
                                                          tfs_device_error* err) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t j = blockIdx.x * 8 + (threadIdx.x >> 5); j < n; j += nwarps) {
    const int64_t p = __ldg(positions + j);
    bool ok = p >= 0 && p < n;
    if (claim != nullptr && ok && claim[p] != (unsigned long long)j) {
      ok = false;
      if (lane == 0) report_error(err, TFS_ERR_BAD_POSITIONS, j);
    }
    if (!ok) continue;
    const uint4* src = rows + j * row_vecs;
    uint4* dst = out + p * row_vecs;
    for (int64_t c0 = 0; c0 < row_vecs; c0 += 128) {
      uint4 v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t c = c0 + q * 32 + lane;
        if (c < row_vecs) v[q] = __ldg(src + c);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t c = c0 + q * 32 + lane;
        if (c < row_vecs) dst[c] = v[q];
      }
    }
  }
}

__global__ void stitch_word_kernel(const int64_t* __restrict__ positions,
                                   const uint32_t* __restrict__ rows, int64_t n,
                                   int64_t row_words, uint32_t* __restrict__ out,
                                   const unsigned long long* claim, tfs_device_error* err) {
  pdl_enter();
  const int64_t total = n * row_words;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / row_words;
    const int64_t c = e - j * row_words;
    const int64_t p = positions[j];
    bool ok = p >= 0 && p < n;
    if (claim != nullptr && ok && claim[p] != (unsigned long long)j) {
      ok = false;
      if (c == 0) report_error(err, TFS_ERR_BAD_POSITIONS, j);
    }
    if (ok) out[p * row_words + c] = rows[e];
  }
}

#ifndef TFS_GRID_PER_SM
#define TFS_GRID_PER_SM 8
#endif
static int grid_for_rows(int64_t n, int rows_per_warp) {
  const int64_t blocks = cdiv(cdiv(n, rows_per_warp), 8);
  return (int)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)TFS_GRID_PER_SM * num_sms()));
}

// ---- Gather through bulk TMA (an A/B alternative, OFF in the product build) -------------------
// Measured round 2 (profiles/r2_ab_gather_bulk.log, r2_ncu_gather_bulk_Z.txt): 2x SLOWER than the
// register-staged kernel at Z (gather E 50 vs 25 us) and no faster at X.  The copies complete
// at ~9 B/clk per SM whatever the ring depth (2 / 4 / 6 slots per warp: 76 / 50 / 54 us), with
// DRAM at 15-19 % busy: one 2 KB cp.async.bulk per row is bound by the copy engine's per-request
// rate, not by bytes in flight.  The register kernel keeps 2 rows x 2 KB per warp in flight and
// is bound by the L2 -> SM traffic of the duplicated (Zipf) rows.
// Each warp owns a contiguous run of `per` output rows and a ring of kGDepth row slots in shared
// memory.  Lane r of a 32-row group reads id r (coalesced) and validates it; lane 0 then keeps
// kGDepth rows in flight as cp.async.bulk copies (table row -> slot, completion on the slot's
// mbarrier); the warp converts each landed row (fp32 -> bf16 RNE, or fp32 as is) with 16-byte
// shared loads and writes it with coalesced stores, then refills the slot with the row kGDepth
// ahead.  A single persistent wave (CTAs per SM from the occupancy calculator): 3 CTAs x 8 warps
// x 4 slots x 2 KB = 192 KB of row loads in flight per SM at d = 512, with ~40 registers a
// thread, where the register-staged kernel above held 4 KB per warp in registers.
#ifndef TFS_GATHER_BULK
#define TFS_GATHER_BULK 0  // 1: A/B builds only (tools/build_variant.py)
#endif
constexpr int kGDepth = 4;
constexpr int kGWarps = 8;
constexpr int kGMaxRowBytes = 4096;

__host__ __device__ inline uint32_t gslot_bytes(int32_t dim) {
  return ((uint32_t)dim * 4u + 127u) & ~127u;
}
constexpr int kGBarBytes = (kGWarps * kGDepth * 8 + 127) / 128 * 128;  // the slots' mbarriers
inline size_t gather_bulk_smem(int32_t dim) {
  return kGBarBytes + (size_t)kGWarps * kGDepth * gslot_bytes(dim);
}

template <bool BF16OUT>
__global__ void __launch_bounds__(kGWarps * 32) gather_bulk_kernel(
    const float* __restrict__ table, int64_t rows, int32_t dim, const int64_t* __restrict__ ids,
    int64_t n, int64_t per, void* __restrict__ out, const float* __restrict__ table2,
    float* __restrict__ out2, tfs_device_error* err) {
  pdl_enter();
  extern __shared__ __align__(128) uint8_t gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rb = (uint32_t)dim * 4u, sb = gslot_bytes(dim);
  uint64_t* bar = reinterpret_cast<uint64_t*>(gsm) + warp * kGDepth;
  uint8_t* ring = gsm + kGBarBytes + (size_t)warp * kGDepth * sb;
  if (lane < kGDepth) bulk::init(bar + lane, 1);
  bulk::fence_init();
  __syncwarp();
  const int n4 = dim >> 2;
  const int64_t j0 = ((int64_t)blockIdx.x * kGWarps + warp) * per;
  const int64_t j1 = min(n, j0 + per);
  uint32_t q0 = 0;  // rows this warp has put through its ring (slot = q % depth, phase = q / depth)
  for (int64_t c0 = j0; c0 < j1; c0 += 32) {
    const int cnt = (int)min((int64_t)32, j1 - c0);
    int64_t id = -1;
    bool ok = false;
    if (lane < cnt) {
      id = __ldg(ids + c0 + lane);
      ok = id >= 0 && id < rows;
      if (!ok && id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, c0 + lane);
      if (ok && table2 != nullptr) out2[c0 + lane] = __ldg(table2 + id);
    }
    const uint32_t okm = __ballot_sync(0xffffffffu, ok);
    const int nok = __popc(okm);
    // lane k: the position (in this group) of the k-th valid row
    const int kth = lane < nok ? (int)__fns(okm, 0, lane + 1) : 0;
    auto issue = [&](int k) {  // all lanes call (shuffles); lane 0 issues row k's copy
      const int r = __shfl_sync(0xffffffffu, kth, k);
      const int64_t idr = __shfl_sync(0xffffffffu, id, r);
      if (lane == 0) {
        const uint32_t q = q0 + (uint32_t)k, s = q % kGDepth;
        bulk::fence_proxy();
        bulk::expect_tx(bar + s, rb);
        bulk::g2s(ring + s * sb, table + idr * dim, rb, bar + s);
      }
    };
    for (int k = 0; k < min(kGDepth, nok); ++k) issue(k);
    for (int k = 0; k < nok; ++k) {
      const uint32_t q = q0 + (uint32_t)k, s = q % kGDepth;
      bulk::wait(bar + s, (q / kGDepth) & 1u);
      const int64_t j = c0 + __shfl_sync(0xffffffffu, kth, k);
      const float4* src = reinterpret_cast<const float4*>(ring + s * sb);
      for (int c = lane; c < n4; c += 32) {
        const float4 v = src[c];
        if (BF16OUT) {
          uint2 p;
          p.x = pack_bf16x2(v.x, v.y);
          p.y = pack_bf16x2(v.z, v.w);
          reinterpret_cast<uint2*>(out)[j * n4 + c] = p;
        } else {
          reinterpret_cast<float4*>(out)[j * n4 + c] = v;
        }
      }
      __syncwarp();  // every lane has read slot s
      if (k + kGDepth < nok) issue(k + kGDepth);
    }
    q0 += (uint32_t)nok;
  }
}

// Launch the bulk gather when the rows qualify (dim % 4 == 0, 16-byte-aligned table and out,
// rows <= 4 KB); returns false (nothing launched) otherwise.
static bool launch_gather_bulk(const float* table, int64_t rows, int32_t dim,
                               const int64_t* ids, int64_t n, void* out, bool bf,
                               const float* table2, float* out2, tfs_device_error* err,
                               cudaStream_t st, int32_t* rc) {
  *rc = TFS_OK;
  if (!TFS_GATHER_BULK || dim % 4 != 0 || (size_t)dim * 4 > (size_t)kGMaxRowBytes || (uintptr_t)table % 16 != 0 ||
      (uintptr_t)out % 16 != 0)
    return false;
  const size_t smem = gather_bulk_smem(dim);
  auto kern = bf ? gather_bulk_kernel<true> : gather_bulk_kernel<false>;
  // CTAs per SM by (device, dtype, dim / 4); the kernel's smem limit is set once per device to
  // the widest row's footprint (the attribute is per kernel, not per launch)
  static int per_sm[8][2][kGMaxRowBytes / 16 + 1];
  static bool attr_set[8][2];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 8) return false;
  if (!attr_set[dev][bf ? 1 : 0]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)gather_bulk_smem(kGMaxRowBytes / 4)) != cudaSuccess) {
      *rc = TFS_ERR_CUDA;
      set_last_error("gather_bulk_kernel attributes", cudaGetLastError());
      return true;
    }
    attr_set[dev][bf ? 1 : 0] = true;
  }
  int& cps = per_sm[dev][bf ? 1 : 0][dim / 4];
  if (cps == 0) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kGWarps * 32, smem);
    cps = std::max(1, b);
  }
  const int64_t warps_cap = (int64_t)num_sms() * cps * kGWarps;
  const int64_t per = std::max<int64_t>(1, cdiv(n, warps_cap));
  const int grid = (int)std::max<int64_t>(1, cdiv(cdiv(n, per), kGWarps));
  ::tfs::launch(kern, grid, kGWarps * 32, smem, st, table, rows, dim, ids, n, per, out, table2, out2, err);
  ::tfs::launched();
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error("gather_bulk_kernel launch", e);
    *rc = TFS_ERR_CUDA;
  }
  return true;
}

}  // namespace tfs

using namespace tfs;

extern "C" int32_t tfs_version(void) { return 200; }

extern "C" int64_t tfs_debug_launch_count(void) { return g_launches.load(); }

extern "C" const char* tfs_status_string(int32_t s) {
  switch (s) {
    case TFS_OK: return "ok";
    case TFS_ERR_INVALID_ARGUMENT: return "invalid argument";
    case TFS_ERR_OUT_OF_RANGE: return "id out of range";
    case TFS_ERR_BAD_POSITIONS: return "stitch positions are not a permutation";
    case TFS_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case TFS_ERR_CUDA: return "CUDA error";
    case TFS_ERR_UNSUPPORTED: return "unsupported device (libtfs needs sm_100a)";
    case TFS_ERR_SAMPLER_EXHAUSTED: return "sampler draw budget exhausted";
    case TFS_ERR_CAPACITY: return "route slot capacity exceeded";
    case TFS_ERR_COMM_TIMEOUT: return "device barrier timed out (a peer never arrived)";
    default: return "unknown status";
  }
}

extern "C" int32_t tfs_last_error_detail(char* buf, size_t len) {
  if (buf == nullptr || len == 0) return TFS_ERR_INVALID_ARGUMENT;
  strncpy(buf, g_last_error, len - 1);
  buf[len - 1] = 0;
  return TFS_OK;
}

extern "C" int32_t tfs_device_check(int32_t device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
    return TFS_ERR_UNSUPPORTED;
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  return (major == 10 && minor == 0) ? TFS_OK : TFS_ERR_UNSUPPORTED;
}

extern "C" int32_t tfs_gather(const void* table, int64_t rows, int32_t dim, int32_t table_dtype,
                              const int64_t* ids, int64_t n, void* out, int32_t out_dtype,
                              tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0);
  TFS_REQUIRE(table_dtype == TFS_F32 && (out_dtype == TFS_F32 || out_dtype == TFS_BF16));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && ids && out);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  const bool bf = out_dtype == TFS_BF16;
  const bool vec = (dim % 4 == 0) && ((uintptr_t)table % 16 == 0) &&
                   ((uintptr_t)out % (bf ? 8 : 16) == 0);
  int32_t brc = TFS_OK;
  if (launch_gather_bulk((const float*)table, rows, dim, ids, n, out, bf, nullptr, nullptr, err,
                         st, &brc))
    return brc;
  if (vec) {
    const int grid = grid_for_rows(n, 2);
    if (bf)
      ::tfs::launch(gather_vec4_kernel<true>, grid, 256, 0, st, (const float*)table, rows, dim, ids, n, out,
                                                     nullptr, nullptr, err);
    else
      ::tfs::launch(gather_vec4_kernel<false>, grid, 256, 0, st, (const float*)table, rows, dim, ids, n, out,
                                                      nullptr, nullptr, err);
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n * dim, 256), 8ll * num_sms()));
    if (bf)
      ::tfs::launch(gather_scalar_kernel<true>, grid, 256, 0, st, (const float*)table, rows, dim, ids, n, out, err);
    else
      ::tfs::launch(gather_scalar_kernel<false>, grid, 256, 0, st, (const float*)table, rows, dim, ids, n, out, err);
  }
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

// Gather in slot layout (owner side of a fixed-capacity route): entry (o, s), o < R, s < cap,
// reads id ids[o * ids_stride + s] and writes its row to out + o * out_stride + s * dim.
// Padding ids (-1) leave their row unwritten.  fp32 only.
template <bool VEC>
__global__ void __launch_bounds__(256) gather_slots_kernel(const float* __restrict__ table,
                                                           int64_t rows, int32_t dim,
                                                           const int64_t* __restrict__ ids,
                                                           int64_t ids_stride, int64_t cap,
                                                           int64_t n, float* __restrict__ out,
                                                           int64_t out_stride,
                                                           tfs_device_error* err) {
  pdl_enter();
  const int cols = VEC ? dim >> 2 : dim;
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols;
    const int c = (int)(e - i * cols);
    const int64_t o = i / cap, sl = i - o * cap;
    const int64_t id = __ldg(ids + o * ids_stride + sl);
    if (id < 0 || id >= rows) {
      if (c == 0 && id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      continue;
    }
    float* dst = out + o * out_stride + sl * dim;
    if (VEC)
      reinterpret_cast<float4*>(dst)[c] = __ldg(reinterpret_cast<const float4*>(table + id * dim) + c);
    else
      dst[c] = __ldg(table + id * dim + c);
  }
}

extern "C" int32_t tfs_gather_slots(const float* table, int64_t rows, int32_t dim,
                                    const int64_t* ids, int64_t ids_stride, int32_t num_slots,
                                    int64_t cap, float* out, int64_t out_stride,
                                    tfs_device_error* err, void* stream) {
  TFS_REQUIRE(dim >= 1 && rows >= 0 && num_slots >= 1 && cap >= 1 && ids_stride >= cap &&
              out_stride >= cap * dim);
  TFS_REQUIRE(table && ids && out);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  const int64_t n = (int64_t)num_slots * cap;
  const bool vec = dim % 4 == 0 && out_stride % 4 == 0 && ((uintptr_t)table % 16 == 0) &&
                   ((uintptr_t)out % 16 == 0);
  const int64_t total = n * (vec ? dim / 4 : dim);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 8ll * num_sms()));
  if (vec)
    ::tfs::launch(gather_slots_kernel<true>, grid, 256, 0, st, table, rows, dim, ids, ids_stride, cap, n, out,
                                                   out_stride, err);
  else
    ::tfs::launch(gather_slots_kernel<false>, grid, 256, 0, st, table, rows, dim, ids, ids_stride, cap, n,
                                                    out, out_stride, err);
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

// One-sided routed Gather (R > 1 over NVLink): out[t] = row (id div R) of the shard of owner
// id mod R, read through that owner's table pointer (peer memory).  Part, the id route, the
// owner Gather, the row route and Stitch in one kernel.
template <bool VEC, bool BF16OUT>
__global__ void __launch_bounds__(256) gather_peers_kernel(const float* const* __restrict__ shards,
                                                           int64_t shard_rows, int32_t dim,
                                                           const int64_t* __restrict__ ids,
                                                           int64_t n, int64_t vocab, int32_t R,
                                                           void* __restrict__ out,
                                                           const float* const* __restrict__ shards2,
                                                           float* __restrict__ out2,
                                                           tfs_device_error* err) {
  pdl_enter();
  const int cols = VEC ? dim >> 2 : dim;
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / cols;
    const int c = (int)(e - t * cols);
    const int64_t id = __ldg(ids + t);
    if (id < 0 || id >= vocab) {
      if (c == 0 && id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, t);
      continue;
    }
    const int64_t o = id % R, local = id / R;
    if (local >= shard_rows) continue;
    const float* src = shards[o] + local * dim;
    if (shards2 != nullptr && c == 0) out2[t] = shards2[o][local];
    if (VEC) {
      const float4 v = reinterpret_cast<const float4*>(src)[c];
      if (BF16OUT)
        reinterpret_cast<uint2*>(out)[t * cols + c] =
            make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
      else
        reinterpret_cast<float4*>(out)[t * cols + c] = v;
    } else {
      if (BF16OUT)
        reinterpret_cast<uint16_t*>(out)[t * dim + c] = f32_to_bf16_bits(src[c]);
      else
        reinterpret_cast<float*>(out)[t * dim + c] = src[c];
    }
  }
}

// The same, one warp per row (16-byte vector rows): the id, its owner and local row are read
// and divided once per row (the element-wise kernel above repeats two 64-bit divisions for
// every 16 bytes), and each lane keeps 2 rows x 4 float4 of peer loads in flight.
template <bool BF16OUT>
__global__ void __launch_bounds__(256) gather_peers_rows_kernel(
    const float* const* __restrict__ shards, int64_t shard_rows, int32_t dim,
    const int64_t* __restrict__ ids, int64_t n, int64_t vocab, int32_t R, void* __restrict__ out,
    const float* const* __restrict__ shards2, float* __restrict__ out2, tfs_device_error* err) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int n4 = dim >> 2;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t j0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 2; j0 < n; j0 += nwarps * 2) {
    const float4* src[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u;
      const int64_t id = j < n ? __ldg(ids + j) : -1;
      ok[u] = id >= 0 && id < vocab;
      if (j < n && !ok[u] && id != -1 && lane == 0) report_error(err, TFS_ERR_OUT_OF_RANGE, j);
      const int64_t o = ok[u] ? id % R : 0, local = ok[u] ? id / R : 0;
      ok[u] = ok[u] && local < shard_rows;
      src[u] = ok[u] ? reinterpret_cast<const float4*>(shards[o] + local * dim) : nullptr;
      if (ok[u] && shards2 != nullptr && lane == 0) out2[j] = shards2[o][local];
    }
    for (int c0 = 0; c0 < n4; c0 += 128) {
      float4 v[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          v[u][q] = (ok[u] && c < n4) ? src[u][c] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
        const int64_t j = j0 + u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          if (c >= n4) continue;
          if (BF16OUT)
            reinterpret_cast<uint2*>(out)[j * n4 + c] =
                make_uint2(pack_bf16x2(v[u][q].x, v[u][q].y), pack_bf16x2(v[u][q].z, v[u][q].w));
          else
            reinterpret_cast<float4*>(out)[j * n4 + c] = v[u][q];
        }
      }
    }
  }
}

// Launch the peer Gather: warp-per-row kernel for 16-byte vector rows, else element-wise.
static int32_t launch_gather_peers(const float* const* shards, int64_t shard_rows, int32_t dim,
                                   const int64_t* ids, int64_t n, int64_t vocab, int32_t R,
                                   void* out, bool bf, const float* const* shards2, float* out2,
                                   tfs_device_error* err, cudaStream_t st) {
  const bool vec = dim % 4 == 0 && ((uintptr_t)out % (bf ? 8 : 16) == 0);
  if (vec) {
    const int grid = grid_for_rows(n, 2);
    auto k = bf ? gather_peers_rows_kernel<true> : gather_peers_rows_kernel<false>;
    ::tfs::launch(k, grid, 256, 0, st, shards, shard_rows, dim, ids, n, vocab, R, out, shards2,
                  out2, err);
  } else {
    const int64_t total = n * dim;
    const int grid =
        (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 16ll * num_sms()));
    auto k = bf ? gather_peers_kernel<false, true> : gather_peers_kernel<false, false>;
    ::tfs::launch(k, grid, 256, 0, st, shards, shard_rows, dim, ids, n, vocab, R, out, shards2,
                  out2, err);
  }
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_gather_peers(const float* const* shards, int64_t shard_rows, int32_t dim,
                                    const int64_t* ids, int64_t n, int64_t vocab,
                                    int32_t num_shards, void* out, int32_t out_dtype,
                                    tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && shard_rows >= 0 && vocab >= 1 && num_shards >= 1);
  TFS_REQUIRE(out_dtype == TFS_F32 || out_dtype == TFS_BF16);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(shards && ids && out);
  TFS_SUPPORTED();
  return launch_gather_peers(shards, shard_rows, dim, ids, n, vocab, num_shards, out,
                             out_dtype == TFS_BF16, nullptr, nullptr, err, as_stream(stream));
}

extern "C" int32_t tfs_gather_peers2(const float* const* shards, int64_t shard_rows, int32_t dim,
                                     const float* const* shards2, const int64_t* ids, int64_t n,
                                     int64_t vocab, int32_t num_shards, void* out,
                                     int32_t out_dtype, float* out2, tfs_device_error* err,
                                     void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && shard_rows >= 0 && vocab >= 1 && num_shards >= 1);
  TFS_REQUIRE(out_dtype == TFS_F32 || out_dtype == TFS_BF16);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(shards && shards2 && ids && out && out2);
  TFS_SUPPORTED();
  return launch_gather_peers(shards, shard_rows, dim, ids, n, vocab, num_shards, out,
                             out_dtype == TFS_BF16, shards2, out2, err, as_stream(stream));
}

// Peer Gather from the owners' bf16 mirrors: one warp per row, 16-byte copies (8 bf16), two
// rows x 4 vectors of peer loads in flight per lane.
__global__ void __launch_bounds__(256) gather_peers_bf16_kernel(
    const uint16_t* const* __restrict__ shards, int64_t shard_rows, int32_t dim,
    const int64_t* __restrict__ ids, int64_t n, int64_t vocab, int32_t R,
    uint16_t* __restrict__ out, const float* const* __restrict__ shards2,
    float* __restrict__ out2, tfs_device_error* err) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int n8 = dim >> 3;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  for (int64_t j0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 2; j0 < n; j0 += nwarps * 2) {
    const uint4* src[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t j = j0 + u;
      const int64_t id = j < n ? __ldg(ids + j) : -1;
      ok[u] = id >= 0 && id < vocab;
      if (j < n && !ok[u] && id != -1 && lane == 0) report_error(err, TFS_ERR_OUT_OF_RANGE, j);
      const int64_t o = ok[u] ? id % R : 0, local = ok[u] ? id / R : 0;
      ok[u] = ok[u] && local < shard_rows;
      src[u] = ok[u] ? reinterpret_cast<const uint4*>(shards[o] + local * dim) : nullptr;
      if (ok[u] && shards2 != nullptr && lane == 0) out2[j] = shards2[o][local];
    }
    for (int c0 = 0; c0 < n8; c0 += 128) {
      uint4 v[2][4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          v[u][q] = (ok[u] && c < n8) ? src[u][c] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = c0 + q * 32 + lane;
          if (c < n8) reinterpret_cast<uint4*>(out)[(j0 + u) * n8 + c] = v[u][q];
        }
      }
    }
  }
}

extern "C" int32_t tfs_gather_peers2_bf16(const uint16_t* const* shards, int64_t shard_rows,
                                          int32_t dim, const float* const* shards2,
                                          const int64_t* ids, int64_t n, int64_t vocab,
                                          int32_t num_shards, uint16_t* out, float* out2,
                                          tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && shard_rows >= 0 && vocab >= 1 && num_shards >= 1);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(shards && shards2 && ids && out && out2);
  TFS_REQUIRE(dim % 8 == 0 && ((uintptr_t)out & 15) == 0);
  TFS_SUPPORTED();
  ::tfs::launch(gather_peers_bf16_kernel, grid_for_rows(n, 2), 256, 0, as_stream(stream),
                shards, shard_rows, dim, ids, n, vocab, num_shards, out, shards2, out2, err);
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_gather2(const float* table, int64_t rows, int32_t dim, const float* table2,
                               const int64_t* ids, int64_t n, void* out, int32_t out_dtype,
                               float* out2, tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0);
  TFS_REQUIRE(out_dtype == TFS_F32 || out_dtype == TFS_BF16);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && table2 && ids && out && out2);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  const bool bf = out_dtype == TFS_BF16;
  const bool vec = (dim % 4 == 0) && ((uintptr_t)table % 16 == 0) &&
                   ((uintptr_t)out % (bf ? 8 : 16) == 0);
  if (!vec) {  // unaligned / odd widths: the two plain gathers
    int32_t rc = tfs_gather(table, rows, dim, TFS_F32, ids, n, out, out_dtype, err, stream);
    if (rc != TFS_OK) return rc;
    return tfs_gather(table2, rows, 1, TFS_F32, ids, n, out2, TFS_F32, err, stream);
  }
  int32_t brc = TFS_OK;
  if (launch_gather_bulk(table, rows, dim, ids, n, out, bf, table2, out2, err, st, &brc))
    return brc;
  const int grid = grid_for_rows(n, 2);
  if (bf)
    ::tfs::launch(gather_vec4_kernel<true>, grid, 256, 0, st, table, rows, dim, ids, n, out, table2, out2,
                                                   err);
  else
    ::tfs::launch(gather_vec4_kernel<false>, grid, 256, 0, st, table, rows, dim, ids, n, out, table2, out2,
                                                    err);
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" size_t tfs_stitch_workspace_bytes(int64_t n) {
  return (size_t)std::max<int64_t>(n, 1) * sizeof(unsigned long long) + 256;
}

extern "C" int32_t tfs_stitch(const int64_t* positions, const void* rows, int64_t n,
                              int64_t row_bytes, void* out, void* ws, size_t ws_bytes,
                              tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && row_bytes >= 4 && row_bytes % 4 == 0);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(positions && rows && out);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  unsigned long long* claim = nullptr;
  if (err != nullptr) {
    if (ws == nullptr || ws_bytes < tfs_stitch_workspace_bytes(n)) return TFS_ERR_WORKSPACE_TOO_SMALL;
    claim = (unsigned long long*)ws;
    TFS_CUDA_TRY(cudaMemsetAsync(claim, 0xff, sizeof(unsigned long long) * n, st));
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4ll * num_sms()));
    ::tfs::launch(stitch_claim_kernel, g, 256, 0, st, positions, n, claim, err); ::tfs::launched();
  }
  const bool vec = row_bytes % 16 == 0 && ((uintptr_t)rows % 16 == 0) && ((uintptr_t)out % 16 == 0);
  if (vec) {
    ::tfs::launch(stitch_vec4_kernel, grid_for_rows(n, 1), 256, 0, st, 
        positions, (const uint4*)rows, n, row_bytes / 16, (uint4*)out, claim, err); ::tfs::launched();
  } else {
    const int64_t words = row_bytes / 4;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n * words, 256), 8ll * num_sms()));
    ::tfs::launch(stitch_word_kernel, g, 256, 0, st, positions, (const uint32_t*)rows, n, words,
                                          (uint32_t*)out, claim, err); ::tfs::launched();
  }
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}
