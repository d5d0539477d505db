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

template <int MODE, bool A_MN, bool B_MN>
static int32_t launch_mode(const CUtensorMap& ta, const CUtensorMap& tb, const Shape& g,
                           const EpiParams& ep, int grid, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    TFS_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<MODE, A_MN, B_MN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kSmemBytes));
    attr_done = true;
  }
  gemm_kernel<MODE, A_MN, B_MN><<<grid, kThreads, kSmemBytes, st>>>(ta, tb, g, ep);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

int32_t launch(int mode, Operand A, Operand B, int M, int N, int K, int ksplit,
               const EpiParams& ep, cudaStream_t st, int* ksplit_eff) {
  if (M <= 0 || N <= 0 || K <= 0) return TFS_ERR_INVALID_ARGUMENT;
  CUtensorMap ta, tb;
  int32_t rc = make_tmap(&ta, A, (uint64_t)M, (uint64_t)K, BM);
  if (rc != TFS_OK) return rc;
  rc = make_tmap(&tb, B, (uint64_t)N, (uint64_t)K, BN);
  if (rc != TFS_OK) return rc;
  Shape g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.num_m = (int)cdiv(M, BM);
  g.num_n = (int)cdiv(N, BN);
  g.kb_total = (int)cdiv(K, BK);
  ksplit = std::max(1, std::min(ksplit, g.kb_total));
  g.kb_per_split = (int)cdiv(g.kb_total, ksplit);
  g.ksplit = (int)cdiv(g.kb_total, g.kb_per_split);
  g.num_units = g.num_m * g.num_n * g.ksplit;
  if (ksplit_eff) *ksplit_eff = g.ksplit;
  const int grid = std::min(g.num_units, num_sms());
  const int sel = (A.mn ? 1 : 0) | (B.mn ? 2 : 0);
  switch (mode) {
    case kStats:
      if (sel != 0) return TFS_ERR_INVALID_ARGUMENT;
      return launch_mode<kStats, false, false>(ta, tb, g, ep, grid, st);
    case kGrad:
      if (sel != 0) return TFS_ERR_INVALID_ARGUMENT;
      return launch_mode<kGrad, false, false>(ta, tb, g, ep, grid, st);
    default:
      switch (sel) {
        case 0: return launch_mode<kStore, false, false>(ta, tb, g, ep, grid, st);
        case 1: return launch_mode<kStore, true, false>(ta, tb, g, ep, grid, st);
        case 2: return launch_mode<kStore, false, true>(ta, tb, g, ep, grid, st);
        default: return launch_mode<kStore, true, true>(ta, tb, g, ep, grid, st);
      }
  }
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

// Per-column epilogue parameters, padded to a multiple of the 256-column tile:
// cb[j] = (b_s[j] - [Q] log_ec_s[j]) * log2(e) (-inf beyond S), sid[j] = s_j (-1 beyond S);
// per-row label y32[t] (-2 = never matches when accidental hits are kept).
__global__ void column_params_kernel(const float* b_s, const float* le_s, const int64_t* sampled,
                                     int64_t S, int64_t S_pad, const int64_t* labels, int64_t B,
                                     int remove_hits, float* cb, int32_t* sid, int32_t* y32) {
  const int64_t total = S_pad + B;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < S) {
      cb[e] = (b_s[e] - (le_s ? le_s[e] : 0.f)) * umma::kLog2e;
      sid[e] = (int32_t)sampled[e];
    } else if (e < S_pad) {
      cb[e] = -INFINITY;
      sid[e] = -1;
    } else {
      const int64_t t = e - S_pad;
      y32[t] = remove_hits ? (int32_t)labels[t] : -2;
    }
  }
}

// Warp per token: true logit on bf16-rounded operands, combine the per-half-tile (max, sum)
// partials (log2 domain) in tile order, then loss / g / dW_true / db_true.
__global__ void __launch_bounds__(256) bf16_combine_kernel(
    int64_t B, int32_t d, const float* h, const float* w_true, const float* b_true,
    const float* le_true, const float2* stats, int nparts, float c, float* loss, float* lse_out,
    float* dw_true, float* db_true) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= B) return;
  const float* ht = h + t * d;
  const float* wt = w_true + t * d;
  float part = 0.f;
  for (int k = lane; k < d; k += 32) part = fmaf(bf16_round(ht[k]), bf16_round(wt[k]), part);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const float z = part + b_true[t] - (le_true ? le_true[t] : 0.f);
  const float z2 = z * umma::kLog2e;
  float m = z2;
  for (int p = lane; p < nparts; p += 32) m = fmaxf(m, stats[(int64_t)p * B + t].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = lane == 0 ? exp2f(z2 - m) : 0.f;
  for (int p = lane; p < nparts; p += 32) {
    const float2 st = stats[(int64_t)p * B + t];
    if (st.y > 0.f) s += st.y * exp2f(st.x - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = (m + log2f(s)) * 0.6931471805599453f;
  const float g = c * (expf(z - lse) - 1.f);
  for (int k = lane; k < d; k += 32) dw_true[t * d + k] = g * bf16_round(ht[k]);
  if (lane == 0) {
    if (loss) loss[t] = lse - z;
    lse_out[t] = lse;
    db_true[t] = g;
  }
}

// dh = sum_s part[s] (split order) + g * bf16(w_true)
__global__ void dh_finalize_kernel(const float* part, int nsplit, int64_t split_stride, int64_t B,
                                   int32_t d, const float* g, const float* w_true, float* dh) {
  const int64_t total = B * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float acc = part[e];
    for (int s = 1; s < nsplit; ++s) acc += part[s * split_stride + e];
    const int64_t t = e / d;
    dh[e] = acc + g[t] * bf16_round(w_true[e]);
  }
}

__global__ void split_sum_kernel(const float* part, int nsplit, int64_t split_stride,
                                 int64_t total, float* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float acc = part[e];
    for (int s = 1; s < nsplit; ++s) acc += part[s * split_stride + e];
    out[e] = acc;
  }
}

// db_s[j] = sum over the 4*num_m row-quarter partials in order.
__global__ void dbs_finalize_kernel(const float* part, int nrows, int64_t S, float* db_s) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= S) return;
  float acc = 0.f;
  for (int r = 0; r < nrows; ++r) acc += part[(int64_t)r * S + j];
  db_s[j] = acc;
}

// ---- workspace layouts --------------------------------------------------------------------------
struct F32Ws {
  float* Z;
};
struct Bf16Ws {
  uint16_t *hb, *wsb, *G;
  float2* stats;
  float *dbs_part, *dh_part, *dws_part, *cb;
  int32_t *sid, *y32;
  int64_t Sp, Spad;
  int ks_dh, ks_dws;
};

static int pick_split(int64_t M, int64_t N, int64_t K) {
  const int64_t base = cdiv(M, umma::BM) * cdiv(N, umma::BN);
  const int64_t kb = cdiv(K, umma::BK);
  int64_t ks = cdiv(num_sms(), base);
  ks = std::max<int64_t>(1, std::min<int64_t>({ks, kb, 8}));
  return (int)ks;
}

static size_t ws_layout(int64_t B, int64_t S, int32_t d, int32_t dtype, F32Ws* f, Bf16Ws* w,
                        void* base) {
  Carver c(base, (size_t)-1);
  if (dtype == TFS_F32) {
    float* Z = c.take<float>((size_t)std::max<int64_t>(B * S, 1));
    if (f) f->Z = Z;
    return c.used + 256;
  }
  const int64_t Sp = (S + 7) / 8 * 8;
  const int64_t Spad = std::max<int64_t>(cdiv(S, umma::BN), 1) * umma::BN;
  const int num_m = (int)cdiv(B, umma::BM);
  const int num_n = (int)cdiv(S, umma::BN);
  const int ks_dh = pick_split(B, d, S), ks_dws = pick_split(S, d, B);
  Bf16Ws x;
  x.hb = c.take<uint16_t>(B * d);
  x.wsb = c.take<uint16_t>(S * d);
  x.G = c.take<uint16_t>(B * Sp);
  x.stats = c.take<float2>((size_t)2 * num_n * B);
  x.dbs_part = c.take<float>((size_t)4 * num_m * S);
  x.dh_part = c.take<float>((size_t)ks_dh * B * d);
  x.dws_part = c.take<float>((size_t)(ks_dws > 1 ? ks_dws : 0) * S * d);
  x.cb = c.take<float>(Spad);
  x.sid = c.take<int32_t>(Spad);
  x.y32 = c.take<int32_t>(B);
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

static int32_t ssm_f32(const tfs_ssm_args* a, void* ws, cudaStream_t st) {
  F32Ws w;
  ws_layout(a->B, a->S, a->dim, TFS_F32, &w, nullptr, ws);
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const int hits = (a->flags & TFS_REMOVE_ACCIDENTAL_HITS) ? 1 : 0;
  const float* le_s = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_s : nullptr;
  const float* le_t = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_true : nullptr;
  if (S > 0) {  // Z = h W_s^T + b_s - logQ (excluded -> -inf)
    SimtParams p{a->b_s, le_s, a->sampled, a->labels, hits, nullptr, nullptr, w.Z, S};
    dim3 grid((unsigned)cdiv(S, 64), (unsigned)cdiv(B, 64));
    simt_gemm_kernel<kSimtLogits><<<grid, 256, 0, st>>>((int)B, (int)S, d, a->h, d, 1, a->w_s, 1,
                                                         d, p);
    launched();
  }
  f32_row_kernel<<<(unsigned)B, 256, 0, st>>>(S, d, a->h, a->w_true, a->b_true, le_t,
                                              a->grad_scale, w.Z, S, a->loss, a->lse, a->dw_true,
                                              a->db_true);
  launched();
  {  // dh = G W_s + g * w_true
    SimtParams p{nullptr, nullptr, nullptr, nullptr, 0, a->db_true, a->w_true, a->dh, d};
    dim3 grid((unsigned)cdiv(d, 64), (unsigned)cdiv(B, 64));
    simt_gemm_kernel<kSimtDh><<<grid, 256, 0, st>>>((int)B, d, (int)S, w.Z, S, 1, a->w_s, d, 1, p);
    launched();
  }
  if (S > 0) {  // dW_s = G^T h ; db_s = column sums of G
    SimtParams p{nullptr, nullptr, nullptr, nullptr, 0, nullptr, nullptr, a->dw_s, d};
    dim3 grid((unsigned)cdiv(d, 64), (unsigned)cdiv(S, 64));
    simt_gemm_kernel<kSimtStore><<<grid, 256, 0, st>>>((int)S, d, (int)B, w.Z, 1, S, a->h, d, 1, p);
    launched();
    colsum_kernel<<<(unsigned)cdiv(S, 256), 256, 0, st>>>(w.Z, B, S, S, a->db_s);
    launched();
  }
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

static int32_t ssm_bf16(const tfs_ssm_args* a, void* ws, cudaStream_t st) {
  Bf16Ws w;
  ws_layout(a->B, a->S, a->dim, TFS_BF16, nullptr, &w, ws);
  const int64_t B = a->B, S = a->S;
  const int32_t d = a->dim;
  const int hits = (a->flags & TFS_REMOVE_ACCIDENTAL_HITS) ? 1 : 0;
  const float* le_s = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_s : nullptr;
  const float* le_t = (a->flags & TFS_SUBTRACT_LOG_Q) ? a->log_ec_true : nullptr;
  const int num_m = (int)cdiv(B, umma::BM), num_n = (int)cdiv(S, umma::BN);

  // Operands in bf16 (row-major; every GEMM reads them K- or MN-major as it needs).
  to_bf16_kernel<<<grid1d(B * d / 4), 256, 0, st>>>(a->h, B * d, w.hb);
  launched();
  if (S > 0) {
    to_bf16_kernel<<<grid1d(S * d / 4), 256, 0, st>>>(a->w_s, S * d, w.wsb);
    launched();
  }
  column_params_kernel<<<grid1d(w.Spad + B), 256, 0, st>>>(
      a->b_s, le_s, a->sampled, S, w.Spad, a->labels, B, hits, w.cb, w.sid, w.y32);
  launched();
  TFS_LAUNCH_CHECK();

  using umma::Operand;
  umma::EpiParams ep{};
  ep.cb = w.cb;
  ep.sid = w.sid;
  ep.y = w.y32;
  int32_t rc;
  const Operand hK{w.hb, d, false}, wsK{w.wsb, d, false};
  if (S > 0) {  // pass 1: per-row (max, sum 2^x) of each half tile, log2 domain
    ep.stats = w.stats;
    rc = umma::launch(umma::kStats, hK, wsK, (int)B, (int)S, d, 1, ep, st, nullptr);
    if (rc != TFS_OK) return rc;
  }
  bf16_combine_kernel<<<(unsigned)cdiv(B, 8), 256, 0, st>>>(
      B, d, a->h, a->w_true, a->b_true, le_t, w.stats, 2 * num_n, a->grad_scale, a->loss,
      a->lse, a->dw_true, a->db_true);
  launched();
  TFS_LAUNCH_CHECK();
  if (S > 0) {  // pass 2: G = c exp(Z - lse) -> bf16 G; column partial sums for db_s
    ep.lse = a->lse;
    ep.c = a->grad_scale;
    ep.G = w.G;
    ep.ldG = w.Sp;
    ep.dbs_part = w.dbs_part;
    rc = umma::launch(umma::kGrad, hK, wsK, (int)B, (int)S, d, 1, ep, st, nullptr);
    if (rc != TFS_OK) return rc;
    dbs_finalize_kernel<<<(unsigned)cdiv(S, 256), 256, 0, st>>>(w.dbs_part, 4 * num_m, S, a->db_s);
    launched();
  }
  // dh = G W_s (split-K partials) + g * bf16(w_true):  A = G K-major, B = W_s MN-major.
  int ks = 1;
  if (S > 0) {
    umma::EpiParams e2{};
    e2.out = w.dh_part;
    e2.ldo = d;
    e2.split_stride = B * d;
    rc = umma::launch(umma::kStore, Operand{w.G, w.Sp, false}, Operand{w.wsb, d, true}, (int)B, d,
                      (int)S, w.ks_dh, e2, st, &ks);
    if (rc != TFS_OK) return rc;
  } else {
    TFS_CUDA_TRY(cudaMemsetAsync(w.dh_part, 0, sizeof(float) * B * d, st));
  }
  dh_finalize_kernel<<<grid1d(B * d), 256, 0, st>>>(w.dh_part, ks, B * d, B, d, a->db_true,
                                                    a->w_true, a->dh);
  launched();
  // dW_s = G^T h:  A = G MN-major, B = h MN-major.
  if (S > 0) {
    umma::EpiParams e3{};
    const bool split = w.ks_dws > 1;
    e3.out = split ? w.dws_part : a->dw_s;
    e3.ldo = d;
    e3.split_stride = S * d;
    int ks2 = 1;
    rc = umma::launch(umma::kStore, Operand{w.G, w.Sp, true}, Operand{w.hb, d, true}, (int)S, d,
                      (int)B, w.ks_dws, e3, st, &ks2);
    if (rc != TFS_OK) return rc;
    if (split) {
      split_sum_kernel<<<grid1d(S * d), 256, 0, st>>>(w.dws_part, ks2, S * d, S * d, a->dw_s);
      launched();
    }
  }
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

}  // namespace tfs

using namespace tfs;

extern "C" size_t tfs_ssm_workspace_bytes(int64_t B, int64_t S, int32_t dim, int32_t operand_dtype) {
  return ws_layout(B, S, dim, operand_dtype, nullptr, nullptr, nullptr);
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
    return TFS_OK;
  }
  TFS_REQUIRE(a->h && a->labels && a->w_true && a->b_true && a->dh && a->dw_true && a->db_true);
  TFS_REQUIRE(!(a->flags & TFS_SUBTRACT_LOG_Q) || (a->log_ec_true && (a->S == 0 || a->log_ec_s)));
  TFS_REQUIRE(a->S == 0 || (a->sampled && a->w_s && a->b_s && a->dw_s && a->db_s));
  if (a->operand_dtype == TFS_BF16) {
    TFS_REQUIRE(a->dim % 64 == 0 && a->lse != nullptr);
    TFS_REQUIRE(((uintptr_t)a->h & 15) == 0 && ((uintptr_t)a->dh & 15) == 0);
    TFS_REQUIRE(((uintptr_t)a->dw_s & 15) == 0 || a->S == 0);
  }
  TFS_SUPPORTED();
  if (ws_bytes < tfs_ssm_workspace_bytes(a->B, a->S, a->dim, a->operand_dtype))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  TFS_REQUIRE(((uintptr_t)ws & 255) == 0);
  cudaStream_t st = as_stream(stream);
  int32_t rc = a->operand_dtype == TFS_BF16 ? ssm_bf16(a, ws, st) : ssm_f32(a, ws, st);
  if (rc != TFS_OK) return rc;
  if (a->loss_sum) {
    TFS_REQUIRE(a->loss != nullptr);
    loss_sum_kernel<<<1, 256, 0, st>>>(a->loss, a->B, a->grad_scale, a->loss_sum); ::tfs::launched();
    TFS_LAUNCH_CHECK();
  }
  return TFS_OK;
}

// Diagnostics: C[ks][M x N] (fp32) = A[M x K] . B[N x K]^T with bf16 operands on the tcgen05
// path.  Exposed for the GEMM unit test only.
extern "C" int32_t tfs_debug_gemm_bf16(const void* A, int64_t lda, int32_t a_mn, const void* B,
                                       int64_t ldb, int32_t b_mn, int32_t M, int32_t N, int32_t K,
                                       int32_t ksplit, float* C, int32_t* out_ksplit,
                                       void* stream) {
  TFS_REQUIRE(A && B && C && M > 0 && N > 0 && K > 0 && lda % 8 == 0 && ldb % 8 == 0);
  TFS_SUPPORTED();
  umma::EpiParams e{};
  e.out = C;
  e.ldo = N;
  e.split_stride = (int64_t)M * N;
  int ks = 1;
  int32_t rc = umma::launch(umma::kStore, umma::Operand{A, lda, a_mn != 0},
                            umma::Operand{B, ldb, b_mn != 0}, M, N, K, ksplit, e,
                            as_stream(stream), &ks);
  if (out_ksplit) *out_ksplit = ks;
  return rc;
}
