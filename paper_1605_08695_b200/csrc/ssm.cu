// ssm.cu -- sampled softmax forward + backward (DESIGN.md §3 O9-O11).
//
// Two operand modes behind one entry point (tfs_sampled_softmax_fwd_bwd):
//  * TFS_BF16 (the performance path): the three contractions Z = h W_s^T, dh = G W_s and
//    dW_s = G^T h run on the tcgen05 tensor cores (umma.cuh) with the softmax fused into the
//    GEMM epilogues.  Z is never materialised: pass 1 keeps per-row (max, sum-exp) of each
//    half tile, a row combine forms lse, and pass 2 recomputes Z tile by tile and writes
//    G = c exp(Z - lse) straight to bf16 (both layouts, so every GEMM stays K-major).
//  * TFS_F32 (parity mode, max rel err 1e-5): fp32 SIMT tiles, Z materialised in fp32.
// Every reduction has a fixed order (split-K partials are summed in split order), so outputs
// are run-to-run bit-identical.
#include <algorithm>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <mutex>

#include "umma.cuh"

namespace tfs {

// =============================================================================================
// tcgen05 GEMM host side
namespace umma {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

// Tensor map of one operand.  K-major [rows x K]: box {BK, box_rows}; MN-major [K x rows]:
// box {64 (MN), BK} -- the kernel issues rows/64 such boxes per stage.  128-byte swizzle.
static int32_t make_tmap(CUtensorMap* map, const Operand& op, uint64_t rows, uint64_t k,
                         uint32_t box_rows) {
  auto fn = encode_fn();
  if (fn == nullptr) return TFS_ERR_CUDA;
  if (((uintptr_t)op.base & 15) != 0 || (op.ld * 2) % 16 != 0) return TFS_ERR_INVALID_ARGUMENT;
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)op.ld * 2};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (op.mn) {
    dims[0] = rows; dims[1] = k;
    box[0] = kMNBox; box[1] = BK;
  } else {
    dims[0] = k; dims[1] = rows;
    box[0] = BK; box[1] = box_rows;
  }
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(op.base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TFS_OK : TFS_ERR_INVALID_ARGUMENT;
}

// Store map of an epilogue output: row-major [rows x cols] (x depth planes `plane` elements
// apart), element size esize, box = 64 bytes x 32 rows, 64-byte swizzle (the staging layout).
static int32_t make_store_map(CUtensorMap* map, CUtensorMapDataType dt, int esize, void* base,
                              uint64_t cols, uint64_t rows, uint64_t ld, uint64_t depth,
                              uint64_t plane) {
  auto fn = encode_fn();
  if (fn == nullptr) return TFS_ERR_CUDA;
  if (((uintptr_t)base & 15) != 0 || (ld * esize) % 16 != 0 || (plane * esize) % 16 != 0)
    return TFS_ERR_INVALID_ARGUMENT;
  const cuuint32_t rank = depth > 1 ? 3 : 2;
  cuuint64_t dims[3] = {cols, rows, depth};
  cuuint64_t strides[2] = {ld * esize, plane * esize};
  cuuint32_t box[3] = {(cuuint32_t)(64 / esize), 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt, rank, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TFS_OK : TFS_ERR_INVALID_ARGUMENT;
}

int tiles_of(int M, int N, int ct) { return (int)(cdiv(M, ct * BM) * cdiv(N, BN)); }

int effective_split(int K, int ksplit) {
  const int kb = (int)cdiv(K, BK);
  ksplit = std::max(1, std::min(ksplit, kb));
  const int per = (int)cdiv(kb, ksplit);
  return (int)cdiv(kb, per);
}

size_t part_floats(int M, int N, int ksplit) {
  return ksplit > 1 ? (size_t)ksplit * M * N : 0;
}

// ct: CTAs per tile of the launch (kSoftmaxCta / kStoreCta); each CTA loads bn / ct B rows.
static int32_t fill_problem(Problem& p, Operand A, Operand B, int M, int N, int K, int ksplit,
                            int ct, int bn = BN) {
  if (M <= 0 || N <= 0 || K <= 0 || bn < 32 || bn > BN || bn % 32 != 0)
    return TFS_ERR_INVALID_ARGUMENT;
  int32_t rc = make_tmap(&p.ta, A, (uint64_t)M, (uint64_t)K, BM);
  if (rc != TFS_OK) return rc;
  rc = make_tmap(&p.tb, B, (uint64_t)N, (uint64_t)K, (uint32_t)(bn / ct));
  if (rc != TFS_OK) return rc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.bn = bn;
  p.num_m = (int)cdiv(M, ct * BM);
  p.num_n = (int)cdiv(N, bn);
  p.kb_total = (int)cdiv(K, BK);
  ksplit = std::max(1, std::min(ksplit, p.kb_total));
  p.kb_per_split = (int)cdiv(p.kb_total, ksplit);
  p.ksplit = (int)cdiv(p.kb_total, p.kb_per_split);
  p.fd_ks = FastDiv::make((uint32_t)p.ksplit);
  p.fd_m = FastDiv::make((uint32_t)p.num_m);
  p.fd_n = FastDiv::make((uint32_t)p.num_n);
  p.units = p.num_m * p.num_n * p.ksplit;
  p.a_mn = A.mn;
  p.b_mn = B.mn;
  p.n_fast = (int64_t)M * K * 2 > (48ll << 20) ? 1 : 0;  // A (bf16) beyond ~40% of L2
  return TFS_OK;
}

// As many pipeline stages as the widest B tile of the launch leaves room for (Params).
template <int MODE, int CT>
static void stage_plan(Params& P) {
  int bmax = 0;
  for (int i = 0; i < P.nprob; ++i) bmax = std::max(bmax, P.p[i].bn / CT * BK * 2);
  P.b_stride = (bmax + 1023) / 1024 * 1024;
  const int fixed = (MODE == kStats && !TFS_SSM_ZPASS ? 0 : kEpiSmem) + kCbSmem + kBarBytes;
  P.stages =
      std::min<int>(kMaxStages,
                    ((int)kSmemBytes - fixed) / (ksub_of(MODE) * (A_BYTES + P.b_stride)));
}

// sms: the SMs a persistent launch may use (<= 0: every SM) -> its CTA groups of ct CTAs.
static int groups_or_all(int sms, int ct) {
  const int all = num_sms() / ct;
  return sms > 0 ? std::max(1, std::min(sms / ct, all)) : all;
}

#ifndef TFS_GEMM_DYN
#define TFS_GEMM_DYN 1  // STATS / GRAD claim tiles dynamically (umma.cuh; 0: static round robin)
#endif
#ifndef TFS_GEMM_PRIO
#define TFS_GEMM_PRIO 0
#endif
template <int MODE, bool LAB, int MC>
static int32_t launch_params_mc(Params P, int sms, cudaStream_t st) {
  constexpr int CT = MODE == kStore ? kStoreCta : kSoftmaxCta;
  constexpr int CL = CT * MC;
  stage_plan<MODE, CT>(P);
  static bool attr_done = false;
  if (!attr_done) {
    TFS_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE, LAB, CT, MC>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmemBytes));
    attr_done = true;
  }
  // persistent: one CTA (or CTA pair: a cluster of 2 on one TPC) per SM (or per two SMs)
  const int groups = std::min(P.total_units, groups_or_all(sms, CL));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(CL * groups));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (pdl_enabled()) {  // programmatic dependent launch (common.cuh)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (TFS_GEMM_PRIO) {  // A/B: the GEMM's CTAs dispatched before pending side-stream CTAs
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    attr[na].id = cudaLaunchAttributePriority;
    attr[na++].val.priority = hi;
  }
  if (CL > 1) {  // CTA pairs / multicast pairs: a cluster of 2 (else a plain launch)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CL;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
#ifdef TFS_GEMM_TRACE
  cudaEvent_t tr_ev[2];
  const bool tr_on = std::getenv("TFS_TRACE_DUMP") != nullptr;
  if (tr_on) {
    cudaEventCreate(&tr_ev[0]);
    cudaEventCreate(&tr_ev[1]);
    cudaEventRecord(tr_ev[0], st);
  }
#endif
  TFS_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_kernel<MODE, LAB, CT, MC>, P));
#ifdef TFS_GEMM_TRACE
  if (tr_on) cudaEventRecord(tr_ev[1], st);
#endif
  launched();
  TFS_LAUNCH_CHECK();
#ifdef TFS_GEMM_TRACE
  if (std::getenv("TFS_TRACE_DUMP") != nullptr) {  // eager calls only (synchronizes)
    cudaStreamSynchronize(st);
    static unsigned long long h[4][512];
    cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
    fprintf(stderr, "TRACE mode=%d units=%d grid=%d stages=%d:", MODE, P.total_units,
            (int)cfg.gridDim.x, P.stages);
    for (int i = 0; i < 512; ++i)
      if (h[MODE][i]) fprintf(stderr, " %d:%lld", i, (long long)(h[MODE][i] - h[MODE][0]));
    fprintf(stderr, "\n");
    static unsigned long long zero[4][512];
    cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
    // per-CTA spans: entry spread, setup, last exit, vs the event-timed launch
    static unsigned long long sp[4][160][3];
    cudaMemcpyFromSymbol(sp, g_span, sizeof(sp));
    float ev_ms = 0.f;
    cudaEventElapsedTime(&ev_ms, tr_ev[0], tr_ev[1]);
    unsigned long long e0 = ~0ull, e1 = 0, s1 = 0, x0 = ~0ull, x1 = 0;
    const int nc = std::min<int>((int)cfg.gridDim.x, 160);
    for (int b = 0; b < nc; ++b) {
      e0 = std::min(e0, sp[MODE][b][0]);
      e1 = std::max(e1, sp[MODE][b][0]);
      s1 = std::max(s1, sp[MODE][b][1] - sp[MODE][b][0]);
      x0 = std::min(x0, sp[MODE][b][2]);
      x1 = std::max(x1, sp[MODE][b][2]);
    }
    fprintf(stderr,
            "SPAN mode=%d event_us=%.2f entry_spread_us=%.2f max_setup_us=%.2f "
            "first_exit_us=%.2f last_exit_us=%.2f\n",
            MODE, ev_ms * 1e3, (e1 - e0) * 1e-3, s1 * 1e-3, (x0 - e0) * 1e-3, (x1 - e0) * 1e-3);
    cudaEventDestroy(tr_ev[0]);
    cudaEventDestroy(tr_ev[1]);
  }
#endif
  if (std::getenv("TFS_DEBUG_SYNC") != nullptr) {  // diagnostics: attribute faults to a mode
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      static const char* names[] = {"gemm_kernel<STATS>", "gemm_kernel<GRAD>", "gemm_kernel<STORE>"};
      set_last_error(names[MODE], e);
      return TFS_ERR_CUDA;
    }
  }
  return TFS_OK;
}

// mc: 2 = the logits / gradient GEMM shares B tiles across a cluster of 2 (softmax_mc).
template <int MODE, bool LAB = false>
static int32_t launch_params(Params P, int sms, cudaStream_t st, int mc = 1) {
  if constexpr (MODE == kStore) {
    return launch_params_mc<MODE, LAB, 1>(P, sms, st);
  } else {
    return mc == 2 ? launch_params_mc<MODE, LAB, 2>(P, sms, st)
                   : launch_params_mc<MODE, LAB, 1>(P, sms, st);
  }
}

// Multicast B in the logits / gradient GEMMs (gemm_kernel's MC = 2) for tall problems: A/B
// round 2 (profiles/r2_ab_mcast_b.log): Z STATS 539 -> 520 us, GRAD 807 -> 782 us; no gain at X
// (B = 2,560 rows: 184.0 vs 185.6 us), so below TFS_MCAST_MIN_ROWS rows every CTA loads its B.
#ifndef TFS_MCAST_MIN_ROWS
#define TFS_MCAST_MIN_ROWS 16384
#endif
static int softmax_mc(int M) { return (TFS_MCAST_B && M >= TFS_MCAST_MIN_ROWS) ? 2 : 1; }

int pick_bn(int M, int N, int sms) {
  const int mc = softmax_mc(M);
  const int64_t groups = groups_or_all(sms, kSoftmaxCta * mc);
  int best = BN;
  int64_t best_cost = -1;
  for (int bn = BN; bn >= 128; bn -= 32) {
    const int64_t tiles = cdiv(M, kSoftmaxCta * mc * BM) * cdiv(N, bn);
    const int64_t cost = cdiv(tiles, groups) * bn;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

int32_t launch_stats_or_grad(int mode, Operand A, Operand B, int M, int N, int K, int bn,
                             int groups, EpiParams ep, void* G, int64_t ldG,
                             cudaStream_t st) {
  if (A.mn || B.mn) return TFS_ERR_INVALID_ARGUMENT;
  Params P{};
  const int mc = softmax_mc(M);
  int32_t rc = fill_problem(P.p[0], A, B, M, N, K, 1, kSoftmaxCta * mc, bn);
  if (rc != TFS_OK) return rc;
  P.nprob = 1;
  P.total_units = P.p[0].units;
  if (mode == kGrad) {
    rc = make_store_map(&ep.tG, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, G, (uint64_t)N,
                        (uint64_t)M, (uint64_t)ldG, 1, 0);
    if (rc != TFS_OK) return rc;
  } else if (ep.zstore) {  // STATS also writes the fp32 logits Z [M x ldG]
    rc = make_store_map(&ep.tZ, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, G, (uint64_t)N,
                        (uint64_t)M, (uint64_t)ldG, 1, 0);
    if (rc != TFS_OK) return rc;
  }
  P.ep = ep;
  if (ep.label_in)
    return mode == kStats ? launch_params<kStats, true>(P, groups, st, mc)
                          : launch_params<kGrad, true>(P, groups, st, mc);
  return mode == kStats ? launch_params<kStats>(P, groups, st, mc)
                        : launch_params<kGrad>(P, groups, st, mc);
}

// Up to two STORE GEMMs in one persistent launch; the caller orders them by unit size.
int32_t launch_store(const Gemm* g, int count, int groups, cudaStream_t st) {
  if (count < 1 || count > 2) return TFS_ERR_INVALID_ARGUMENT;
  Params P{};
  P.nprob = count;
  P.total_units = 0;
  for (int i = 0; i < count; ++i) {
    Problem& p = P.p[i];
    int32_t rc = fill_problem(p, g[i].A, g[i].B, g[i].M, g[i].N, g[i].K, g[i].ksplit, kStoreCta);
    if (rc != TFS_OK) return rc;
    if (p.ksplit > 1) {
      if (g[i].part == nullptr || g[i].g != nullptr) return TFS_ERR_INVALID_ARGUMENT;
      rc = make_store_map(&p.to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g[i].part, (uint64_t)p.N,
                          (uint64_t)p.M, (uint64_t)p.N, (uint64_t)p.ksplit,
                          (uint64_t)p.M * p.N);
    } else {
      rc = make_store_map(&p.to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g[i].out, (uint64_t)p.N,
                          (uint64_t)p.M, (uint64_t)g[i].ldo, 1, 0);
    }
    if (rc != TFS_OK) return rc;
    p.g = g[i].g;
    p.wt = g[i].wt;
    p.ldw = g[i].ldw;
    p.wt_bf16 = g[i].wt_bf16;
    P.total_units += p.units;
  }
  return launch_params<kStore>(P, groups, st);
}

}  // namespace umma

// =============================================================================================
// Shared small kernels
__device__ __forceinline__ float block_sum_256(float v, float* red) {
  // fixed-order tree over 256 threads
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const float r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ float block_max_256(float v, float* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  const float r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) loss_sum_kernel(const float* loss, int64_t B, float c,
                                                       float* out) {
  pdl_enter();
  __shared__ float red[256];
  float acc = 0.f;
  for (int64_t t = threadIdx.x; t < B; t += 256) acc += loss[t];
  const float s = block_sum_256(acc, red);
  if (threadIdx.x == 0) *out = c * s;
}

// =============================================================================================
// fp32 parity path (SIMT)
enum SimtEpi : int { kSimtLogits = 0, kSimtDh = 1, kSimtStore = 2 };

struct SimtParams {
  const float* b_s;
  const float* le_s;
  const int64_t* sampled;
  const int64_t* labels;
  int remove_hits;
  const float* g;       // kSimtDh: g_t
  const float* w_true;  // kSimtDh
  float* out;
  int64_t ldo;
};

template <int EPI>
__global__ void __launch_bounds__(256) simt_gemm_kernel(int M, int N, int K, const float* A,
                                                        int64_t sam, int64_t sak, const float* B,
                                                        int64_t sbk, int64_t sbn, SimtParams p) {
  pdl_enter();
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;
      const int mm = sam == 1 ? (e & 63) : (e >> 4);
      const int kk = sam == 1 ? (e >> 6) : (e & 15);
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? A[(int64_t)m * sam + (int64_t)k * sak] : 0.f;
      const int nn = sbn == 1 ? (e & 63) : (e >> 4);
      const int kb = sbn == 1 ? (e >> 6) : (e & 15);
      const int n = n0 + nn, kq = k0 + kb;
      Bs[kb][nn] = (n < N && kq < K) ? B[(int64_t)kq * sbk + (int64_t)n * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (EPI == kSimtLogits) {
        const bool excl = p.remove_hits && p.sampled[n] == p.labels[m];
        v = excl ? -INFINITY : v + (p.b_s[n] - (p.le_s ? p.le_s[n] : 0.f));
      } else if (EPI == kSimtDh) {
        v = v + p.g[m] * p.w_true[(int64_t)m * p.ldo + n];
      }
      p.out[(int64_t)m * p.ldo + n] = v;
    }
  }
}

// One CTA per token: true logit, lse, loss, g, dW_true, db_true; Z row -> G row in place.
__global__ void __launch_bounds__(256) f32_row_kernel(
    int64_t S, int32_t d, const float* h, const float* w_true, const float* b_true,
    const float* le_true, float c, float* ZG, int64_t ldz, float* loss, float* lse_out,
    float* dw_true, float* db_true) {
  pdl_enter();
  __shared__ float red[256];
  const int64_t t = blockIdx.x;
  const float* ht = h + t * d;
  const float* wt = w_true + t * d;
  float part = 0.f;
  for (int k = threadIdx.x; k < d; k += 256) part = fmaf(ht[k], wt[k], part);
  const float z = block_sum_256(part, red) + b_true[t] - (le_true ? le_true[t] : 0.f);
  float* row = ZG + t * ldz;
  float mx = z;
  for (int64_t j = threadIdx.x; j < S; j += 256) mx = fmaxf(mx, row[j]);
  const float mu = block_max_256(mx, red);
  float se = threadIdx.x == 0 ? expf(z - mu) : 0.f;
  for (int64_t j = threadIdx.x; j < S; j += 256) se += expf(row[j] - mu);
  const float lse = mu + logf(block_sum_256(se, red));
  const float g = c * (expf(z - lse) - 1.f);
  for (int64_t j = threadIdx.x; j < S; j += 256) {
    const float zz = row[j];
    row[j] = zz == -INFINITY ? 0.f : c * expf(zz - lse);
  }
  for (int k = threadIdx.x; k < d; k += 256) dw_true[t * d + k] = g * ht[k];
  if (threadIdx.x == 0) {
    if (loss) loss[t] = lse - z;
    if (lse_out) lse_out[t] = lse;
    db_true[t] = g;
  }
}

// db_s[j] = sum_t G[t, j] in increasing t.
__global__ void colsum_kernel(const float* G, int64_t B, int64_t S, int64_t ldg, float* out) {
  pdl_enter();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= S) return;
  float acc = 0.f;
  for (int64_t t = 0; t < B; ++t) acc += G[t * ldg + j];
  out[j] = acc;
}

// =============================================================================================
// bf16 tensor-core path: small kernels around the GEMMs
// fp32 -> bf16 (RNE), 4 elements per thread.
__global__ void to_bf16_kernel(const float* src, int64_t n, uint16_t* dst) {
  pdl_enter();
  const int64_t n4 = n >> 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    reinterpret_cast<uint2*>(dst)[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = f32_to_bf16_bits(src[i]);
}

// db_s[j] = sum_t G[t, j] over the bf16 G [B x ldG]: block = 32 columns (4 x 16-byte chunks)
// x 64 row groups; each thread sums its rows in order (8 loads in flight), then the 64 partials
// are added in row-group order (fixed summation order, no atomics).  Also returns the candidate
// map to all-zero (the GRAD pass was its last reader), and one extra block forms
// loss_sum = c * sum_t loss_t (fixed-order tree) when loss_sum != nullptr.
// GROUPS row groups per block (4 GROUPS threads): 64 when there are enough 32-column blocks to
// fill the GPU, 256 for narrow G (few column blocks: more rows in flight per block).
constexpr int kColsumChunks = 4;
#ifndef TFS_COLSUM_GROUPS
#define TFS_COLSUM_GROUPS 128  // A/B round 2: X colsum 12.4 -> 11.3 us (64), 15.2 (32)
#endif
#ifndef TFS_COLSUM_G256
#define TFS_COLSUM_G256 0
#endif
template <int GROUPS>
__global__ void __launch_bounds__(kColsumChunks * GROUPS) g_colsum_kernel(
    const uint16_t* G, int64_t B, int64_t S, int64_t ldG, float* db_s, const int64_t* sampled,
    int2* cmap, int64_t vocab, const float* loss, float c, float* loss_sum) {
  pdl_enter();
  constexpr int kColsumGroups = GROUPS, kColsumThreads = kColsumChunks * GROUPS;
  __shared__ float red[kColsumGroups][kColsumChunks * 8 + 1];
  const int64_t ncol_blocks = cdiv_dev(S, kColsumChunks * 8);
  if (blockIdx.x >= ncol_blocks) {  // the loss-sum block
    float acc = 0.f;
    for (int64_t t = threadIdx.x; t < B; t += kColsumThreads) acc += loss[t];
    float* r = &red[0][0];
    r[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kColsumThreads / 2; s > 0; s >>= 1) {
      if (threadIdx.x < s) r[threadIdx.x] += r[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) *loss_sum = c * r[0];
    return;
  }
  if (cmap != nullptr) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < S;
         j += ncol_blocks * blockDim.x) {
      const int64_t k = sampled[j];
      if (k >= 0 && k < vocab) cmap[k] = make_int2(0, 0);
    }
  }
  const int chunk = threadIdx.x % kColsumChunks, rg = threadIdx.x / kColsumChunks;
  const int64_t c0 = (int64_t)blockIdx.x * (kColsumChunks * 8) + chunk * 8;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto add8 = [&](const uint4& x) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc[2 * k] += __uint_as_float(w[k] << 16);
      acc[2 * k + 1] += __uint_as_float(w[k] & 0xffff0000u);
    }
  };
  if (c0 < S) {
    constexpr int U = GROUPS >= 256 ? 4 : 8;  // independent row loads in flight per thread
    const uint16_t* p = G + c0;
    int64_t r = rg;
    for (; r + (U - 1) * kColsumGroups < B; r += U * kColsumGroups) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        x[u] = __ldg(reinterpret_cast<const uint4*>(p + (r + u * kColsumGroups) * ldG));
#pragma unroll
      for (int u = 0; u < U; ++u) add8(x[u]);
    }
    for (; r < B; r += kColsumGroups) add8(__ldg(reinterpret_cast<const uint4*>(p + r * ldG)));
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[rg][chunk * 8 + k] = acc[k];
  __syncthreads();
  // fixed-order tree over the row groups: 8 parts of 32 groups, then the 8 part sums
  constexpr int kCols = kColsumChunks * 8, kParts = 8;
  __shared__ float part[kParts][kCols];
  if (threadIdx.x < kParts * kCols) {
    const int col = threadIdx.x % kCols, pt = threadIdx.x / kCols;
    float sum = 0.f;
    for (int g = pt * (kColsumGroups / kParts); g < (pt + 1) * (kColsumGroups / kParts); ++g)
      sum += red[g][col];
    part[pt][col] = sum;
  }
  __syncthreads();
  if (threadIdx.x < kCols) {
    const int64_t col = (int64_t)blockIdx.x * kCols + threadIdx.x;
    float sum = 0.f;
#pragma unroll
    for (int pt = 0; pt < kParts; ++pt) sum += part[pt][threadIdx.x];
    if (col < S) db_s[col] = sum;
  }
}

// db_s[j] = sum over the GRAD epilogue's 32-row slab partials colpart[q * ld + j], q = 0, 1, ...
// (fixed order: 32 row groups of slabs summed in slab order, then the groups in group order);
// also returns the candidate map to all-zero (the GRAD pass was its last reader), and one
// extra block forms loss_sum = c * sum_t loss_t (fixed-order tree) when loss_sum != nullptr.
constexpr int kDbGroups = 32, kDbCols = 32;
__global__ void __launch_bounds__(kDbGroups * kDbCols) db_colpart_kernel(
    const float* colpart, int64_t nslabs, int64_t ld, int64_t S, float* db_s,
    const int64_t* sampled, int2* cmap, int64_t vocab, const float* loss, int64_t B, float c,
    float* loss_sum) {
  pdl_enter();
  __shared__ float red[kDbGroups][kDbCols + 1];
  const int64_t ncol_blocks = cdiv_dev(S, kDbCols);
  const int tid = threadIdx.x;
  if (blockIdx.x >= ncol_blocks) {  // the loss-sum block
    float acc = 0.f;
    for (int64_t t = tid; t < B; t += blockDim.x) acc += loss[t];
    float* r = &red[0][0];
    r[tid] = acc;
    __syncthreads();
    for (int s2 = (int)blockDim.x / 2; s2 > 0; s2 >>= 1) {
      if (tid < s2) r[tid] += r[tid + s2];
      __syncthreads();
    }
    if (tid == 0) *loss_sum = c * r[0];
    return;
  }
  if (cmap != nullptr) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + tid; j < S; j += ncol_blocks * blockDim.x) {
      const int64_t k = sampled[j];
      if (k >= 0 && k < vocab) cmap[k] = make_int2(0, 0);
    }
  }
  const int col = tid % kDbCols, g = tid / kDbCols;
  const int64_t j = (int64_t)blockIdx.x * kDbCols + col;
  float acc = 0.f;
  if (j < S) {
    int64_t q = g;
    for (; q + 7 * kDbGroups < nslabs; q += 8 * kDbGroups) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(colpart + (q + u * kDbGroups) * ld + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; q < nslabs; q += kDbGroups) acc += __ldg(colpart + q * ld + j);
  }
  red[g][col] = acc;
  __syncthreads();
  if (g == 0) {
    float sum = 0.f;
    for (int k = 0; k < kDbGroups; ++k) sum += red[k][col];
    if (j < S) db_s[j] = sum;
  }
}

// ---- operand conversion + column parameters + candidate map, one launch ---------------------
// h and W_s -> bf16 (RNE).  Per column (padded to a multiple of the 256-column tile):
// cb[j] = (b_s[j] - [Q] log_ec_s[j]) * log2(e) (-inf beyond S), sid[j] = s_j (-1 beyond S).
// With accidental-hit removal and a vocabulary bound, the candidate map (first in the
// workspace, zero between calls) receives, for every id k among the candidates,
//   cmap[k] = {max over j with s_j = k of (2^30 - j), max of (j + 1)}
// (integer atomics: order-independent), so the epilogue finds the columns [lo, hi] that hold a
// row's label with one load and compares ids only in chunks that intersect that range.
constexpr int32_t kMapLoBase = 1 << 30;
__global__ void __launch_bounds__(256) prep_kernel(const float* h, int64_t nh4, const float* w_s,
                                                   int64_t nw4, uint16_t* hb, uint16_t* wsb,
                                                   const float* b_s, const float* le_s,
                                                   const int64_t* sampled, int64_t S,
                                                   int64_t S_pad, int2* cmap, int64_t vocab,
                                                   float* cb, int32_t* sid) {
  pdl_enter();
  constexpr int U = 4;  // independent loads in flight per thread
  const int64_t total = nh4 + nw4 + S_pad;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e0 < total; e0 += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      v[u] = e < nh4 ? __ldg(reinterpret_cast<const float4*>(h) + e)
                     : (e < nh4 + nw4 ? __ldg(reinterpret_cast<const float4*>(w_s) + (e - nh4))
                                      : make_float4(0.f, 0.f, 0.f, 0.f));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * stride;
      if (e < nh4 + nw4) {
        const uint2 o = make_uint2(pack_bf16x2(v[u].x, v[u].y), pack_bf16x2(v[u].z, v[u].w));
        if (e < nh4)
          reinterpret_cast<uint2*>(hb)[e] = o;
        else
          reinterpret_cast<uint2*>(wsb)[e - nh4] = o;
      } else if (e < total) {
        const int64_t j = e - nh4 - nw4;
        if (j < S) {
          const int64_t k = sampled[j];
          cb[j] = (b_s[j] - (le_s ? le_s[j] : 0.f)) * umma::kLog2e;
          sid[j] = (int32_t)k;
          if (cmap != nullptr && k >= 0 && k < vocab) {
            int32_t* m = reinterpret_cast<int32_t*>(cmap + k);
            atomicMax(m, kMapLoBase - (int32_t)j);
            atomicMax(m + 1, (int32_t)j + 1);
          }
        } else {
          cb[j] = -INFINITY;
          sid[j] = -1;
        }
      }
    }
  }
}

// Four consecutive operand values as bf16-rounded floats: from fp32 (rounded here, RNE) or
// from bf16 bits (TFS_BF16_OPERANDS).  Element index i4 counts groups of four.
template <bool BIN>
__device__ __forceinline__ float4 ld4_bf(const void* p, int64_t i4) {
  if (BIN) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p) + i4);
    return make_float4(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                       __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
  }
  const float4 v = __ldg(reinterpret_cast<const float4*>(p) + i4);
  return make_float4(bf16_round(v.x), bf16_round(v.y), bf16_round(v.z), bf16_round(v.w));
}

// Warp per token: true logit on bf16-rounded operands, combine the per-half-tile (max, sum)
// partials (log2 domain) in tile order, then loss / g / dW_true / db_true.
template <bool BIN>
__global__ void __launch_bounds__(256) bf16_combine_kernel(
    int64_t B, int32_t d, const void* h, const void* w_true, const float* b_true,
    const float* le_true, const float2* stats, int nparts, float c, float* loss, float* lse_out,
    float* dw_true, float* db_true) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= B) return;
  // d % 64 == 0 on this path: vector loads.  Every load of the token -- h and w_true (kept in
  // registers for dw_true = g h when d <= 512), its bias and the stats partials (when at most
  // 128) -- is issued before any result is needed: one memory round trip.
  const int n4 = d >> 2;
  const int64_t r4 = t * n4;  // this token's first group of four
  const float2* st_t = stats + t * nparts;  // this token's partials, contiguous
  const bool regs = n4 <= 128 && nparts <= 128;
  float4 a[4], b[4];
  float2 sp[4];
  float part = 0.f;
  const float bt = b_true[t], lt = le_true ? le_true[t] : 0.f;
  if (regs) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = lane + 32 * u;
      a[u] = k < n4 ? ld4_bf<BIN>(h, r4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      b[u] = k < n4 ? ld4_bf<BIN>(w_true, r4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      sp[u] = k < nparts ? st_t[k] : make_float2(-INFINITY, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      part = fmaf(a[u].x, b[u].x, part);
      part = fmaf(a[u].y, b[u].y, part);
      part = fmaf(a[u].z, b[u].z, part);
      part = fmaf(a[u].w, b[u].w, part);
    }
  } else {
    for (int k0 = lane; k0 < n4; k0 += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + 32 * u;
        a[u] = k < n4 ? ld4_bf<BIN>(h, r4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
        b[u] = k < n4 ? ld4_bf<BIN>(w_true, r4 + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        part = fmaf(a[u].x, b[u].x, part);
        part = fmaf(a[u].y, b[u].y, part);
        part = fmaf(a[u].z, b[u].z, part);
        part = fmaf(a[u].w, b[u].w, part);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const float z = part + bt - lt;
  const float z2 = z * umma::kLog2e;
  float m = z2;
  if (regs) {
#pragma unroll
    for (int u = 0; u < 4; ++u) m = fmaxf(m, sp[u].x);
  } else {
    for (int p = lane; p < nparts; p += 32) m = fmaxf(m, st_t[p].x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = lane == 0 ? exp2f(z2 - m) : 0.f;
  if (regs) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (sp[u].y > 0.f) s += sp[u].y * exp2f(sp[u].x - m);
  } else {
    for (int p = lane; p < nparts; p += 32) {
      const float2 st = st_t[p];
      if (st.y > 0.f) s += st.y * exp2f(st.x - m);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = (m + log2f(s)) * 0.6931471805599453f;
  const float g = c * (expf(z - lse) - 1.f);
  float4* dw4 = reinterpret_cast<float4*>(dw_true + t * d);
  if (regs) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = lane + 32 * u;
      if (k < n4) dw4[k] = make_float4(g * a[u].x, g * a[u].y, g * a[u].z, g * a[u].w);
    }
  } else {
    for (int k = lane; k < n4; k += 32) {
      const float4 x = ld4_bf<BIN>(h, r4 + k);
      dw4[k] = make_float4(g * x.x, g * x.y, g * x.z, g * x.w);
    }
  }
  if (lane == 0) {
    if (loss) loss[t] = lse - z;
    lse_out[t] = lse;
    db_true[t] = g;
  }
}

// out = sum_s part[s] (split order) [+ g[row] * bf16(wt)] (float4 columns; N % 4 == 0); wt is
// fp32 (rounded here) or bf16 bits (BIN).
template <bool BIN>
__global__ void split_finalize_kernel(const float* part, int nsplit, int64_t M, int32_t N,
                                      const float* g, const void* wt, float* out) {
  pdl_enter();
  const int n4 = N / 4;
  const int64_t total = M * n4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / n4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nsplit; ++s) {
      const float4 x = reinterpret_cast<const float4*>(part)[s * total + e];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    if (g != nullptr) {
      const float gr = g[row];
      const float4 w = ld4_bf<BIN>(wt, e);
      acc.x += gr * w.x;
      acc.y += gr * w.y;
      acc.z += gr * w.z;
      acc.w += gr * w.w;
    }
    reinterpret_cast<float4*>(out)[e] = acc;
  }
}

// ---- workspace layouts --------------------------------------------------------------------------
struct F32Ws {
  float* Z;
};
struct Bf16Ws {
  uint16_t *hb, *wsb, *G;
  float2* stats;
  float *cb, *part_dh, *part_dws, *colpart;
  float* Z;  // [B x Spad] fp32 logits (log2 units) from the STATS pass (TFS_SSM_ZPASS)
  int32_t* sid;
  unsigned* sched;  // zero region after the candidate map: dynamic-schedule counters
  int64_t Sp, Spad, ldh, nslabs;
  int ks_dh, ks_dws;
};




// Split-K plan for the backward pair (dW_s: M=S, K=B; dh: M=B, K=S; both N=d) run in one
// persistent launch: aim for ~2 units per CTA pair of roughly equal k-block count.
#ifndef TFS_BWD_UNITS_PER_GROUP
#define TFS_BWD_UNITS_PER_GROUP 2
#endif
static void plan_backward(int64_t B, int64_t S, int32_t d, int* ks_dh, int* ks_dws) {
  constexpr int ct = umma::kStoreCta;
  const int64_t t_dh = umma::tiles_of((int)B, d, ct), t_dws = umma::tiles_of((int)S, d, ct);
  const int64_t kb_dh = cdiv(S, umma::BK), kb_dws = cdiv(B, umma::BK);
  const int64_t work = t_dh * kb_dh + t_dws * kb_dws;
  const int64_t target =
      std::max<int64_t>(16, cdiv(work, TFS_BWD_UNITS_PER_GROUP * (num_sms() / ct)));
  auto split = [&](int64_t kb) {
    if (kb <= target + target / 4) return 1;
    return (int)std::min<int64_t>(16, cdiv(kb, target));
  };
  *ks_dh = umma::effective_split((int)S, split(kb_dh));
  *ks_dws = umma::effective_split((int)B, split(kb_dws));
}

// The candidate map (bf16 path, vocab > 0) comes first: offset 0, size depending on vocab only,
// so a zero-filled workspace stays valid across calls of any shape.
static size_t map_bytes(int64_t vocab) {
  return vocab > 0 ? ((size_t)vocab * sizeof(int2) + 255) / 256 * 256 : 0;
}
static size_t ws_layout(int64_t B, int64_t S, int32_t d, int32_t dtype, int64_t vocab, F32Ws* f,
                        Bf16Ws* w, void* base) {
  Carver c(base, (size_t)-1);
  c.used = map_bytes(vocab);
  // 256 zero bytes: the tcgen05 GEMMs' dynamic tile-schedule counters (STATS [0, 2), GRAD
  // [4, 6)), zero before a call and left zero by it, like the map
  unsigned* sched = c.take<unsigned>(64);
  if (dtype == TFS_F32) {
    float* Z = c.take<float>((size_t)std::max<int64_t>(B * S, 1));
    if (f) f->Z = Z;
    return c.used + 256;
  }
  const int64_t Sp = (S + 7) / 8 * 8;
  // sized for any STATS / GRAD tile width in [128, 256] (chosen at launch, pick_bn)
  const int num_n = (int)cdiv(S, 128);
  const int64_t Spad = std::max<int64_t>(num_n, 1) * 128 + 256;
  int ks_dh = 1, ks_dws = 1;
  if (S > 0 && B > 0) plan_backward(B, S, d, &ks_dh, &ks_dws);
  Bf16Ws x;
  x.ldh = d;
  x.hb = c.take<uint16_t>(B * x.ldh);
  x.wsb = c.take<uint16_t>(S * d);
  x.G = c.take<uint16_t>(B * Sp);
  x.stats = c.take<float2>((size_t)2 * num_n * B);
  x.part_dh = c.take<float>(umma::part_floats((int)B, d, ks_dh));
  x.part_dws = c.take<float>(umma::part_floats((int)S, d, ks_dws));
  x.cb = c.take<float>(Spad);
  x.sid = c.take<int32_t>(Spad);
  x.nslabs = cdiv(std::max<int64_t>(B, 1), 2 * umma::BM) * 2 * 4;  // GRAD: 32-row slabs (MC <= 2)
  x.colpart = c.take<float>((size_t)x.nslabs * Spad);
  x.Z = TFS_SSM_ZPASS ? c.take<float>((size_t)std::max<int64_t>(B, 1) * Spad) : nullptr;
  x.sched = TFS_GEMM_DYN ? sched : nullptr;
  x.Sp = Sp;
  x.Spad = Spad;
  x.ks_dh = ks_dh;
  x.ks_dws = ks_dws;
  if (w) *w = x;
  return c.used + 256;
}

static int grid1d(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, threads), 8ll * num_sms()));
}

// Optional instrumentation events (tfs_ssm_args::timing_events).
static void mark(const tfs_ssm_args* a, int i, cudaStream_t st) {
  if (a->timing_events != nullptr && a->timing_events[i] != nullptr)
    cudaEventRecord(static_cast<cudaEvent_t>(a->timing_events[i]), st);
}

static int32_t ssm_f32(const tfs_ssm_args* a, void* ws, cudaStream_t st) {
  F32Ws w;
  ws_layout(a->B, a->S, a->dim, TFS_F32, a->vocab, &w, nullptr, ws);
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const int hits = (a->flags & TFS_REMOVE_ACCIDENTAL_HITS) ? 1 : 0;
  const float* le_s = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_s : nullptr;
  const float* le_t = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_true : nullptr;
  mark(a, 0, st);  // fp32 path: events 0 (start), 2 (after the logits GEMM), 7 (end) only
  if (S > 0) {  // Z = h W_s^T + b_s - logQ (excluded -> -inf)
    SimtParams p{a->b_s, le_s, a->sampled, a->labels, hits, nullptr, nullptr, w.Z, S};
    dim3 grid((unsigned)cdiv(S, 64), (unsigned)cdiv(B, 64));
    ::tfs::launch(simt_gemm_kernel<kSimtLogits>, grid, 256, 0, st, (int)B, (int)S, d, a->h, d, 1, a->w_s, 1,
                                                         d, p);
    launched();
  }
  mark(a, 2, st);
  ::tfs::launch(f32_row_kernel, (unsigned)B, 256, 0, st, S, d, a->h, a->w_true, a->b_true, le_t,
                                              a->grad_scale, w.Z, S, a->loss, a->lse, a->dw_true,
                                              a->db_true);
  launched();
  {  // dh = G W_s + g * w_true
    SimtParams p{nullptr, nullptr, nullptr, nullptr, 0, a->db_true, a->w_true, a->dh, d};
    dim3 grid((unsigned)cdiv(d, 64), (unsigned)cdiv(B, 64));
    ::tfs::launch(simt_gemm_kernel<kSimtDh>, grid, 256, 0, st, (int)B, d, (int)S, w.Z, S, 1, a->w_s, d, 1, p);
    launched();
  }
  if (S > 0) {  // dW_s = G^T h ; db_s = column sums of G
    SimtParams p{nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, a->dw_s, d};
    dim3 grid((unsigned)cdiv(d, 64), (unsigned)cdiv(S, 64));
    ::tfs::launch(simt_gemm_kernel<kSimtStore>, grid, 256, 0, st, (int)S, d, (int)B, w.Z, 1, S, a->h, d, 1, p);
    launched();
    ::tfs::launch(colsum_kernel, (unsigned)cdiv(S, 256), 256, 0, st, w.Z, B, S, S, a->db_s);
    launched();
  }
  mark(a, 7, st);
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}


// Everything the phases of the tensor-core path share: workspace slices, epilogue parameters,
// the STATS / GRAD tile width.
struct Bf16Plan {
  Bf16Ws w;
  umma::EpiParams ep;
  int bn, num_n;
  int groups;  // SMs the persistent GEMMs may use (0: every SM; tfs_ssm_args.sm_reserve)
  bool bin;
};

static void bf16_plan(const tfs_ssm_args* a, void* ws, Bf16Plan* p) {
  ws_layout(a->B, a->S, a->dim, TFS_BF16, a->vocab, nullptr, &p->w, ws);
  const bool hits = (a->flags & TFS_REMOVE_ACCIDENTAL_HITS) != 0;
  const bool label_in = (a->flags & TFS_LABEL_IN_CANDIDATES) != 0;
  p->groups = a->sm_reserve > 0 ? std::max(2, num_sms() - a->sm_reserve) : 0;  // SMs
  p->bn = a->S > 0 ? umma::pick_bn((int)a->B, (int)a->S, p->groups) : umma::BN;
  p->num_n = (int)cdiv(a->S, p->bn);
  p->bin = (a->flags & TFS_BF16_OPERANDS) != 0;  // h, w_true, w_s given in bf16
  if (p->bin) {  // already rounded by the producer (e.g. a bf16 Gather): no conversion pass
    p->w.hb = static_cast<uint16_t*>(const_cast<void*>(static_cast<const void*>(a->h)));
    p->w.wsb = static_cast<uint16_t*>(const_cast<void*>(static_cast<const void*>(a->w_s)));
  }
  const int64_t V = (hits || label_in) ? a->vocab : 0;
  umma::EpiParams& ep = p->ep;
  ep = umma::EpiParams{};
  ep.cb = p->w.cb;
  ep.sid = p->w.sid;
  ep.labels = (hits || label_in) ? a->labels : nullptr;
  ep.cmap = V > 0 ? reinterpret_cast<int2*>(ws) : nullptr;
  ep.vocab = V;
  ep.S_pad = (int)p->w.Spad;
  ep.stats = p->w.stats;
  ep.nparts = 2 * p->num_n;
  ep.lse = a->lse;
  ep.c = a->grad_scale;
  ep.label_in = label_in ? 1 : 0;
}

// Operands in bf16 (row-major; every GEMM reads them K- or MN-major as it needs), column
// parameters and the candidate map: one launch.
static int32_t bf16_prep(const tfs_ssm_args* a, const Bf16Plan& p, cudaStream_t st) {
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const float* le_s = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_s : nullptr;
  const int64_t nconv = p.bin ? 0 : (B + S) * d / 4;
  ::tfs::launch(prep_kernel, grid1d(nconv / 4 + p.w.Spad), 256, 0, st, 
      a->h, p.bin ? 0 : B * d / 4, a->w_s, p.bin ? 0 : S * d / 4, p.w.hb, p.w.wsb, a->b_s, le_s,
      a->sampled, S, p.w.Spad, const_cast<int2*>(p.ep.cmap), p.ep.vocab, p.w.cb, p.w.sid);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

// The gradient pass from the stored logits (TFS_SSM_ZPASS): G = c exp(Z - lse) = 2^(v - goff)
// in bf16, with the label column (label_in) at c (p - 1) and the label's logit to zlab -- the
// arithmetic of the GRAD epilogue (umma.cuh) on the same v, so G is bit-identical -- plus the
// column sums of each 32-row slab of the bf16 G in row order (the colpart layout the GRAD
// epilogue writes; db_colpart_kernel finishes db_s).  Block: 32 rows x 256 columns, lane =
// column (32-column loads and 64-byte stores per row, coalesced), all 32 row loads in flight.
template <bool LAB>
__global__ void __launch_bounds__(256) g_from_z_kernel(
    const float* __restrict__ Z, int64_t ldz, int64_t B, int64_t S, const float* __restrict__ lse,
    float c, const int64_t* __restrict__ labels, const int2* __restrict__ cmap, int64_t vocab,
    int S_pad, const int32_t* __restrict__ sid, uint16_t* __restrict__ G, int64_t ldG,
    float* __restrict__ colpart, int64_t colpart_ld, float* __restrict__ zlab) {
  pdl_enter();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int64_t col = ((int64_t)blockIdx.y * 8 + warp) * 32 + lane;
  const int nrows = (int)min((int64_t)32, B - r0);
  // lane r: row r0 + r's constants (as the GRAD epilogue forms them)
  const int64_t row_l = r0 + lane;
  float goff_l = 0.f;
  int32_t y_l = -2;
  int hlo_l = 1 << 30, hhi_l = -1;
  if (row_l < B) {
    if (LAB && labels != nullptr) {
      const int64_t yl = __ldg(labels + row_l);
      y_l = (int32_t)yl;
      if (cmap == nullptr) {
        hlo_l = 0;
        hhi_l = S_pad;
      } else if (yl >= 0 && yl < vocab) {
        const int2 m = __ldg(cmap + yl);
        if (m.y > 0) {
          hlo_l = (1 << 30) - m.x;
          hhi_l = m.y - 1;
        }
      }
    }
    goff_l = __ldg(lse + row_l) * umma::kLog2e - log2f(c);
  }
  const bool col_ok = col < S;
  const int32_t sid_c = (LAB && col_ok) ? __ldg(sid + col) : -1;
  float v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r)
    v[r] = (r < nrows && col_ok) ? __ldg(Z + (r0 + r) * ldz + col) : -INFINITY;
  float cs = 0.f;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float goff = __shfl_sync(0xffffffffu, goff_l, r);
    float g;
    if (LAB) {
      const int32_t y = __shfl_sync(0xffffffffu, y_l, r);
      const int lo = __shfl_sync(0xffffffffu, hlo_l, r), hi = __shfl_sync(0xffffffffu, hhi_l, r);
      const bool lab = col >= lo && col <= hi && sid_c == y;
      if (lab && r < nrows) zlab[r0 + r] = v[r] * umma::kLn2;
      g = umma::fast_exp2(v[r] - goff) - (lab ? c : 0.f);
    } else {
      g = umma::fast_exp2(v[r] - goff);
    }
    const uint16_t gb = f32_to_bf16_bits(g);
    if (r < nrows && col_ok) {
      G[(r0 + r) * ldG + col] = gb;
      cs += __uint_as_float((uint32_t)gb << 16);
    }
  }
  if (col_ok) colpart[(r0 >> 5) * colpart_ld + col] = cs;
}

// Pass 1: per-row (max, sum 2^x) of each half tile, log2 domain.
// zstore: also keep the logits (fp32 Z) for the gradient pass (the full fwd+bwd call).
static int32_t bf16_stats(const tfs_ssm_args* a, const Bf16Plan& p, bool zstore,
                          cudaStream_t st) {
  const umma::Operand hK{p.w.hb, p.w.ldh, false}, wsK{p.w.wsb, a->dim, false};
  umma::EpiParams ep = p.ep;
  ep.zstore = (zstore && p.w.Z != nullptr) ? 1 : 0;
  ep.sched = p.w.sched;
  return umma::launch_stats_or_grad(umma::kStats, hK, wsK, (int)a->B, (int)a->S, a->dim, p.bn,
                                    p.groups, ep, ep.zstore ? p.w.Z : nullptr, p.w.Spad, st);
}

// dW_s = G^T h and dh = G W_s [+ g * bf16(w_true)] from the bf16 G, in one persistent launch.
static int32_t bf16_store(const tfs_ssm_args* a, const Bf16Plan& p, const float* g_true,
                          const void* w_true, cudaStream_t st) {
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const Bf16Ws& w = p.w;
  using umma::Operand;
  int32_t rc = TFS_OK;
  // dW_s = G^T h (A = G MN-major, B = h MN-major) and dh = G W_s + g * bf16(w_true)
  // (A = G K-major, B = W_s MN-major) in one persistent launch; split partials are reduced in
  // split order by the finalize pass, which also adds the true-class term of dh.
  umma::Gemm g[2];
  const bool dws_split = w.ks_dws > 1, dh_split = w.ks_dh > 1;
  g[0] = umma::Gemm{Operand{w.G, w.Sp, true}, Operand{w.hb, w.ldh, true}, (int)S, d, (int)B,
                    w.ks_dws, a->dw_s, d, w.part_dws, nullptr, nullptr, 0, 0};
  g[1] = umma::Gemm{Operand{w.G, w.Sp, false}, Operand{w.wsb, d, true}, (int)B, d, (int)S,
                    w.ks_dh, a->dh, d, w.part_dh, dh_split ? nullptr : g_true,
                    dh_split ? nullptr : w_true, d, p.bin ? 1 : 0};
  // larger units first so the static round-robin schedule balances the SMs
  const int64_t u0 = cdiv(B, umma::BK) / w.ks_dws, u1 = cdiv(S, umma::BK) / w.ks_dh;
  if (u1 > u0) std::swap(g[0], g[1]);
  rc = umma::launch_store(g, 2, p.groups, st);
  if (rc != TFS_OK) return rc;
  mark(a, 6, st);
  if (dws_split) {  // dW_s first: the softmax-row gradients are then final (rows_ready_event)
    ::tfs::launch(split_finalize_kernel<false>, grid1d(S * d / 4), 256, 0, st,
                  w.part_dws, w.ks_dws, S, d, nullptr, nullptr, a->dw_s);
    launched();
  }
  if (a->rows_ready_event != nullptr &&
      cudaEventRecord(static_cast<cudaEvent_t>(a->rows_ready_event), st) != cudaSuccess)
    return TFS_ERR_CUDA;
  if (dh_split) {
    auto fin = p.bin ? split_finalize_kernel<true> : split_finalize_kernel<false>;
    ::tfs::launch(fin, grid1d(B * d / 4), 256, 0, st, w.part_dh, w.ks_dh, B, d, g_true, w_true, a->dh);
    launched();
  }
  TFS_LAUNCH_CHECK();
  mark(a, 7, st);
  return TFS_OK;
}

// Pass 2 onwards (S > 0): G = c exp(Z - lse) -> bf16 G; db_s = column sums of G (+ loss sum);
// dW_s = G^T h and dh = G W_s [+ g * bf16(w_true)] in one persistent launch.
static int32_t bf16_backward(const tfs_ssm_args* a, const Bf16Plan& p, const float* g_true,
                             const void* w_true, float* zlab, cudaStream_t st, bool z_stored = false) {
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const Bf16Ws& w = p.w;
  umma::EpiParams ep = p.ep;
  ep.zlab = zlab;
  if (z_stored && w.Z != nullptr) {  // G (and the db_s slab partials) from the stored logits
    const dim3 grid((unsigned)cdiv(B, 32), (unsigned)cdiv(S, 256));
    auto gk = ep.label_in ? g_from_z_kernel<true> : g_from_z_kernel<false>;
    ::tfs::launch(gk, grid, 256, 0, st, w.Z, w.Spad, B, S, a->lse, a->grad_scale, ep.labels,
                  ep.cmap, ep.vocab, ep.S_pad, ep.sid, w.G, w.Sp, w.colpart, w.Spad, zlab);
    launched();
    mark(a, 4, st);
    const int64_t ncb = cdiv(S, kDbCols);
    ::tfs::launch(db_colpart_kernel, (unsigned)(ncb + (a->loss_sum ? 1 : 0)), kDbGroups * kDbCols,
                  0, st, w.colpart, cdiv(B, 32), w.Spad, S, a->db_s, a->sampled,
                  const_cast<int2*>(ep.cmap), ep.vocab, a->loss, B, a->grad_scale, a->loss_sum);
    launched();
    mark(a, 5, st);
    return bf16_store(a, p, g_true, w_true, st);
  }
  // db_s = column sums of G.  When G is larger than L2 can keep (Z: 1 GB), the GRAD epilogue
  // sums each 32-row slab it stages (+8 us on X's GRAD, but no 1 GB re-read: Z -4.5 %, A/B
  // round 2, profiles/r2_ab_grad_colsum.log); otherwise a separate pass over G is cheaper.
  const bool fused_colsum = B * S * 2 > (64ll << 20);
  if (fused_colsum) {
    ep.colpart = w.colpart;
    ep.colpart_ld = w.Spad;
  }
  using umma::Operand;
  const Operand hK{w.hb, w.ldh, false}, wsK{w.wsb, d, false};
  ep.sched = w.sched ? w.sched + 4 : nullptr;
  int32_t rc = umma::launch_stats_or_grad(umma::kGrad, hK, wsK, (int)B, (int)S, d, p.bn,
                                          p.groups, ep, w.G,
                                          w.Sp, st);
  if (rc != TFS_OK) return rc;
  mark(a, 4, st);
  if (fused_colsum) {
    const int64_t ncb = cdiv(S, kDbCols);
    ::tfs::launch(db_colpart_kernel, (unsigned)(ncb + (a->loss_sum ? 1 : 0)), kDbGroups * kDbCols, 0, st, 
        w.colpart, w.nslabs, w.Spad, S, a->db_s, a->sampled, const_cast<int2*>(ep.cmap),
        ep.vocab, a->loss, B, a->grad_scale, a->loss_sum);
  } else {
    const int64_t ncb = cdiv(S, kColsumChunks * 8);
    const bool narrow = TFS_COLSUM_G256 || ncb < num_sms();  // 256 row groups per column block
    constexpr int kWide = TFS_COLSUM_GROUPS;  // row groups per column block (enough blocks)
    auto colsum = narrow ? g_colsum_kernel<256> : g_colsum_kernel<kWide>;
    ::tfs::launch(colsum, (unsigned)(ncb + (a->loss_sum ? 1 : 0)),
                  kColsumChunks * (narrow ? 256 : kWide), 0, st, w.G, B, S, w.Sp, a->db_s,
                  a->sampled, const_cast<int2*>(ep.cmap), ep.vocab, a->loss, a->grad_scale,
                  a->loss_sum);
  }
  launched();
  mark(a, 5, st);
  return bf16_store(a, p, g_true, w_true, st);
}

static int32_t ssm_bf16(const tfs_ssm_args* a, void* ws, cudaStream_t st) {
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const float* le_t = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_true : nullptr;
  mark(a, 0, st);
  Bf16Plan p;
  bf16_plan(a, ws, &p);
  int32_t rc = bf16_prep(a, p, st);
  if (rc != TFS_OK) return rc;
  mark(a, 1, st);
  if (S > 0) {
    rc = bf16_stats(a, p, true, st);
    if (rc != TFS_OK) return rc;
  }
  mark(a, 2, st);
  auto combine = p.bin ? bf16_combine_kernel<true> : bf16_combine_kernel<false>;
  ::tfs::launch(combine, (unsigned)cdiv(B, 8), 256, 0, st, B, d, a->h, a->w_true, a->b_true, le_t,
                                                p.w.stats, 2 * p.num_n, a->grad_scale, a->loss,
                                                a->lse, a->dw_true, a->db_true);
  launched();
  TFS_LAUNCH_CHECK();
  mark(a, 3, st);
  if (S == 0) {  // no candidates: dh = g * bf16(w_true)
    auto fin = p.bin ? split_finalize_kernel<true> : split_finalize_kernel<false>;
    ::tfs::launch(fin, grid1d(B * d / 4), 256, 0, st, nullptr, 0, B, d, a->db_true, a->w_true, a->dh);
    launched();
    TFS_LAUNCH_CHECK();
    return TFS_OK;
  }
  return bf16_backward(a, p, a->db_true, a->w_true, nullptr, st, /*z_stored=*/true);
}

// Warp per row: (max, sum) over all of the row's half-tile partials, log2 domain, combined in a
// fixed order (lane-strided, then a butterfly).
__global__ void __launch_bounds__(256) row_stats_kernel(const float2* stats, int nparts,
                                                        int64_t B, float2* out) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= B) return;
  const float2* st_t = stats + t * nparts;
  float m = -INFINITY;
  for (int q = lane; q < nparts; q += 32) m = fmaxf(m, st_t[q].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  if (m > -INFINITY)
    for (int q = lane; q < nparts; q += 32) {
      const float2 x = st_t[q];
      if (x.y > 0.f) s += x.y * exp2f(x.x - m);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[t] = make_float2(m, s);
}

}  // namespace tfs

using namespace tfs;

#ifdef TFS_GEMM_TRACE
// Diagnostic builds only (not in include/tfs.h): the per-CTA globaltimer spans (entry, setup
// done, exit; ns) of the last launch of each GEMM kind, [3][160][3], e.g. after a graph replay
// (tools/gemm_spans_step.py).
extern "C" int32_t tfs_trace_gemm_spans(unsigned long long* out) {
  static unsigned long long h[4][160][3];
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpyFromSymbol(h, umma::g_span, sizeof(h)) != cudaSuccess)
    return TFS_ERR_CUDA;
  std::memcpy(out, h, 3 * sizeof(h[0]));
  return TFS_OK;
}
// globaltimer markers in stream order (around a step replay): slot < 8
__device__ unsigned long long g_stamp[8];
__global__ void trace_stamp_kernel(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_stamp[slot & 7] = t;
}
extern "C" int32_t tfs_trace_stamp(int32_t slot, void* stream) {
  trace_stamp_kernel<<<1, 1, 0, as_stream(stream)>>>(slot);
  return cudaGetLastError() == cudaSuccess ? TFS_OK : TFS_ERR_CUDA;
}
extern "C" int32_t tfs_trace_stamps(unsigned long long* out) {
  if (cudaDeviceSynchronize() != cudaSuccess ||
      cudaMemcpyFromSymbol(out, g_stamp, sizeof(g_stamp)) != cudaSuccess)
    return TFS_ERR_CUDA;
  return TFS_OK;
}
#endif

extern "C" size_t tfs_ssm_workspace_bytes(int64_t B, int64_t S, int32_t dim, int32_t operand_dtype,
                                          int64_t vocab) {
  return ws_layout(B, S, dim, operand_dtype, vocab, nullptr, nullptr, nullptr);
}

extern "C" int32_t tfs_sampled_softmax_fwd_bwd(const tfs_ssm_args* a, void* ws, size_t ws_bytes,
                                               void* stream) {
  TFS_REQUIRE(a != nullptr);
  TFS_REQUIRE(a->B >= 0 && a->S >= 0 && a->dim >= 1 && a->B < (1ll << 31) && a->S < (1ll << 31));
  TFS_REQUIRE(a->operand_dtype == TFS_F32 || a->operand_dtype == TFS_BF16);
  if (a->B == 0) {
    TFS_SUPPORTED();
    cudaStream_t st = as_stream(stream);
    if (a->S > 0) {
      TFS_REQUIRE(a->dw_s && a->db_s);
      TFS_CUDA_TRY(cudaMemsetAsync(a->dw_s, 0, sizeof(float) * a->S * a->dim, st));
      TFS_CUDA_TRY(cudaMemsetAsync(a->db_s, 0, sizeof(float) * a->S, st));
    }
    if (a->loss_sum) TFS_CUDA_TRY(cudaMemsetAsync(a->loss_sum, 0, sizeof(float), st));
    if (a->rows_ready_event != nullptr)
      TFS_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(a->rows_ready_event), st));
    return TFS_OK;
  }
  TFS_REQUIRE(a->h && a->labels && a->w_true && a->b_true && a->dh && a->dw_true && a->db_true);
  TFS_REQUIRE(!(a->flags & TFS_SUBTRACT_LOG_Q) || (a->log_ec_true && (a->S == 0 || a->log_ec_s)));
  TFS_REQUIRE(a->S == 0 || (a->sampled && a->w_s && a->b_s && a->dw_s && a->db_s));
  TFS_REQUIRE(!(a->flags & TFS_BF16_OPERANDS) || a->operand_dtype == TFS_BF16);
  TFS_REQUIRE(!(a->flags & TFS_LABEL_IN_CANDIDATES));  // the split calls' mode only
  if (a->operand_dtype == TFS_BF16) {
    TFS_REQUIRE(a->dim % 64 == 0 && a->lse != nullptr);
    TFS_REQUIRE(((uintptr_t)a->h & 15) == 0 && ((uintptr_t)a->dh & 15) == 0);
    TFS_REQUIRE(((uintptr_t)a->w_true & 15) == 0 && ((uintptr_t)a->dw_true & 15) == 0);
    TFS_REQUIRE(((uintptr_t)a->dw_s & 15) == 0 || a->S == 0);
  }
  TFS_SUPPORTED();
  if (ws_bytes < tfs_ssm_workspace_bytes(a->B, a->S, a->dim, a->operand_dtype, a->vocab))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  TFS_REQUIRE(((uintptr_t)ws & 255) == 0);
  cudaStream_t st = as_stream(stream);
  TFS_REQUIRE(a->loss_sum == nullptr || a->loss != nullptr);
  int32_t rc = a->operand_dtype == TFS_BF16 ? ssm_bf16(a, ws, st) : ssm_f32(a, ws, st);
  if (rc != TFS_OK) return rc;
  const bool fused_sum = a->operand_dtype == TFS_BF16 && a->S > 0;  // done by g_colsum_kernel
  if (a->loss_sum && !fused_sum) {
    ::tfs::launch(loss_sum_kernel, 1, 256, 0, st, a->loss, a->B, a->grad_scale, a->loss_sum); ::tfs::launched();
    TFS_LAUNCH_CHECK();
  }
  // (the bf16 path with candidates records rows_ready_event itself, before the dh reduction)
  if (a->rows_ready_event != nullptr && !fused_sum)
    TFS_CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(a->rows_ready_event), st));
  return TFS_OK;
}

// ---- the two halves of a vocabulary-sharded full softmax ------------------------------------
static int32_t check_split_args(const tfs_ssm_args* a, void* ws, size_t ws_bytes) {
  TFS_REQUIRE(a != nullptr);
  TFS_REQUIRE(a->operand_dtype == TFS_BF16 && a->B >= 1 && a->S >= 1 && a->B < (1ll << 31) &&
              a->S < (1ll << 31) && a->dim >= 64 && a->dim % 64 == 0);
  TFS_REQUIRE(a->h && a->sampled && a->w_s && a->b_s);
  TFS_REQUIRE(((uintptr_t)a->h & 15) == 0 && ((uintptr_t)a->w_s & 15) == 0);
  TFS_REQUIRE(!(a->flags & TFS_SUBTRACT_LOG_Q) || a->log_ec_s);
  const bool hits = (a->flags & TFS_REMOVE_ACCIDENTAL_HITS) != 0;
  const bool label_in = (a->flags & TFS_LABEL_IN_CANDIDATES) != 0;
  TFS_REQUIRE(!(hits && label_in));
  TFS_REQUIRE(!(hits || label_in) || a->labels);
  TFS_SUPPORTED();
  if (ws_bytes < tfs_ssm_workspace_bytes(a->B, a->S, a->dim, TFS_BF16, a->vocab))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  TFS_REQUIRE(((uintptr_t)ws & 255) == 0);
  return TFS_OK;
}

extern "C" int32_t tfs_ssm_partial_stats(const tfs_ssm_args* a, float* row_stats, void* ws,
                                         size_t ws_bytes, void* stream) {
  int32_t rc = check_split_args(a, ws, ws_bytes);
  if (rc != TFS_OK) return rc;
  TFS_REQUIRE(row_stats != nullptr && ((uintptr_t)row_stats & 7) == 0);
  cudaStream_t st = as_stream(stream);
  Bf16Plan p;
  bf16_plan(a, ws, &p);
  if ((rc = bf16_prep(a, p, st)) != TFS_OK) return rc;
  if ((rc = bf16_stats(a, p, false, st)) != TFS_OK) return rc;
  ::tfs::launch(row_stats_kernel, (unsigned)cdiv(a->B, 8), 256, 0, st, p.w.stats, 2 * p.num_n, a->B,
                                                            reinterpret_cast<float2*>(row_stats));
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_ssm_backward_from_lse(const tfs_ssm_args* a, float* z_label, void* ws,
                                             size_t ws_bytes, void* stream) {
  int32_t rc = check_split_args(a, ws, ws_bytes);
  if (rc != TFS_OK) return rc;
  TFS_REQUIRE(a->lse && a->dh && a->dw_s && a->db_s);
  TFS_REQUIRE(((uintptr_t)a->dh & 15) == 0 && ((uintptr_t)a->dw_s & 15) == 0);
  TFS_REQUIRE(a->loss == nullptr && a->loss_sum == nullptr);
  const bool label_in = (a->flags & TFS_LABEL_IN_CANDIDATES) != 0;
  TFS_REQUIRE(!label_in || z_label != nullptr);
  cudaStream_t st = as_stream(stream);
  Bf16Plan p;
  bf16_plan(a, ws, &p);
  return bf16_backward(a, p, nullptr, nullptr, label_in ? z_label : nullptr, st);
}

// Diagnostics: C[ks][M x N] (fp32) = A[M x K] . B[N x K]^T with bf16 operands on the tcgen05
// path.  Exposed for the GEMM unit test only.
extern "C" size_t tfs_debug_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K,
                                                 int32_t ksplit) {
  const int ks = umma::effective_split(K, ksplit);
  return umma::part_floats(M, N, ks) * sizeof(float) + 256;
}

extern "C" int32_t tfs_debug_gemm_bf16(const void* A, int64_t lda, int32_t a_mn, const void* B,
                                       int64_t ldb, int32_t b_mn, int32_t M, int32_t N, int32_t K,
                                       int32_t ksplit, float* C, void* ws, size_t ws_bytes,
                                       void* stream) {
  TFS_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0 && lda % 8 == 0 && ldb % 8 == 0 &&
              N % 4 == 0);
  TFS_SUPPORTED();
  if (ws_bytes < tfs_debug_gemm_workspace_bytes(M, N, K, ksplit)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  const int ks = umma::effective_split(K, ksplit);
  Carver c(ws, ws_bytes);
  float* part = c.take<float>(umma::part_floats(M, N, ks));
  umma::Gemm g{umma::Operand{A, lda, a_mn != 0}, umma::Operand{B, ldb, b_mn != 0}, M, N, K, ks,
               C, N, part, nullptr, nullptr, 0, 0};
  int32_t rc = umma::launch_store(&g, 1, 0, st);
  if (rc != TFS_OK || ks == 1) return rc;
  ::tfs::launch(split_finalize_kernel<false>, grid1d((int64_t)M * N / 4), 256, 0, st, part, ks, M, N, nullptr,
                                                                    nullptr, C);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_ssm_grad_from_logits(void) { return TFS_SSM_ZPASS ? 1 : 0; }
