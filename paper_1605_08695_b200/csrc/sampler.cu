// sampler.cu -- the log-uniform candidate sampler of the sampled softmax (P:715-717,
// P:1173-1175; readings R-6..R-10, R-17, R-24 in DESIGN.md §3).
//
// Unique mode needs "the first S distinct draws in draw order" -- an inherently sequential
// definition.  It is computed in parallel and exactly: every draw i writes k_i and does
// atomicMin(firstpos[k_i], i) (the minimum is order-independent), so draw i is a first
// occurrence iff firstpos[k_i] == i; a CTA-ordered prefix count of those flags then gives each
// first occurrence its rank in draw order.  The draw budget N is fixed at init (Chernoff bound),
// so a call never needs the host (graph-capturable); the per-id scratch is restored at the end.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace tfs {

struct Philox4 {
  uint32_t x, y, z, w;
};

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds, key bumped by the Weyl constants.
__device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

struct SamplerState {
  const uint64_t* thr;  // [V] inverse-CDF thresholds
  int32_t* firstpos;    // [V] scratch, INT32_MAX between calls
};

static SamplerState carve_state(void* state, int64_t vocab) {
  Carver c(state, (size_t)-1);
  uint64_t* thr = c.take<uint64_t>(vocab);
  int32_t* fp = c.take<int32_t>(vocab);
  return SamplerState{thr, fp};
}

__device__ __forceinline__ int64_t draw_id(const uint64_t* thr, int64_t V, double log_v1,
                                           uint32_t i, uint64_t step, uint32_t replica,
                                           uint64_t seed) {
  const Philox4 w = philox4x32_10(
      Philox4{i, (uint32_t)(step >> 32), (uint32_t)step, replica}, (uint32_t)seed,
      (uint32_t)(seed >> 32));
  const uint64_t m = ((((uint64_t)w.x) << 32) | w.y) >> 11;  // 53-bit integer
  // Float guess of the inverse CDF (fp32 is close enough: the integer fix-up below walks to
  // the exact k = min{k : m < Thr[k]} from any start), then the exact fix-up.
  const float guess = __expf((float)m * 0x1p-53f * (float)log_v1) - 1.0f;
  int64_t k = guess < 0.f ? 0 : (guess > 2147483647.f ? V - 1 : (int64_t)guess);
  k = k < 0 ? 0 : (k > V - 1 ? V - 1 : k);
  while (k > 0 && m < thr[k - 1]) --k;
  while (m >= thr[k]) ++k;
  return k;
}

// The log-uniform law puts ~half of the draws on the 1024 most frequent ids: their
// first-position minima are taken in shared memory first (one global atomicMin per CTA and id
// instead of one per draw -- id 0 alone gets ~5% of all draws).  min is order-independent.
constexpr int kHotIds = 1024;
__global__ void __launch_bounds__(256) sample_draw_kernel(const uint64_t* thr, int64_t V,
                                                          double log_v1, int64_t N, uint64_t seed,
                                                          uint64_t step, const uint64_t* step_dev,
                                                          uint32_t replica, int unique,
                                                          int32_t* draws, int32_t* firstpos,
                                                          int64_t* out_direct) {
  pdl_enter();
  __shared__ int32_t hot[kHotIds];
  if (step_dev != nullptr) step = *step_dev;
  if (unique) {
    for (int j = threadIdx.x; j < kHotIds; j += blockDim.x) hot[j] = 0x7fffffff;
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = draw_id(thr, V, log_v1, (uint32_t)i, step, replica, seed);
    if (unique) {
      draws[i] = (int32_t)k;
      if (k < kHotIds)
        atomicMin(hot + k, (int32_t)i);
      else
        atomicMin(firstpos + k, (int32_t)i);
    } else {
      out_direct[i] = k;
    }
  }
  if (unique) {
    __syncthreads();
    for (int j = threadIdx.x; j < kHotIds && j < V; j += blockDim.x)
      if (hot[j] != 0x7fffffff) atomicMin(firstpos + j, hot[j]);
  }
}

constexpr int kSelThreads = 256, kSelItems = 4, kSelTile = kSelThreads * kSelItems;

__device__ __forceinline__ uint32_t cta_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t ws[kSelThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  uint32_t base = 0, all = 0;
  for (int w = 0; w < kSelThreads / 32; ++w) {
    if (w < warp) base += ws[w];
    all += ws[w];
  }
  __syncthreads();
  if (total) *total = all;
  return base + x - v;
}

__global__ void __launch_bounds__(kSelThreads) sample_count_kernel(const int32_t* draws,
                                                                   const int32_t* firstpos,
                                                                   int64_t N, uint32_t* blk_cnt) {
  pdl_enter();
  const int64_t base = (int64_t)blockIdx.x * kSelTile + threadIdx.x * kSelItems;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    if (i < N && firstpos[draws[i]] == (int32_t)i) ++c;
  }
  uint32_t total;
  cta_exclusive_scan(c, &total);
  if (threadIdx.x == 0) blk_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kSelThreads) sample_select_kernel(
    const int32_t* draws, const int32_t* firstpos, int64_t N, const uint32_t* blk_cnt, int nblk,
    int32_t S, int64_t* out_sampled, int64_t* out_num_tries, tfs_device_error* err) {
  pdl_enter();
  __shared__ uint32_t s_pre, s_all;
  if (threadIdx.x < 32) {
    uint32_t pre = 0, all = 0;
    for (int b = threadIdx.x; b < nblk; b += 32) {
      const uint32_t c = blk_cnt[b];
      all += c;
      if (b < (int)blockIdx.x) pre += c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (threadIdx.x == 0) {
      s_pre = pre;
      s_all = all;
    }
  }
  __syncthreads();
  if (s_all < (uint32_t)S) {  // budget exhausted (probability < 1e-21 with the init budget)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      report_error(err, TFS_ERR_SAMPLER_EXHAUSTED, N);
      *out_num_tries = N;
    }
  }
  if (s_pre >= (uint32_t)S) return;
  const int64_t base = (int64_t)blockIdx.x * kSelTile + threadIdx.x * kSelItems;
  bool f[kSelItems];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    f[j] = i < N && firstpos[draws[i]] == (int32_t)i;
    c += f[j];
  }
  uint32_t rank = s_pre + cta_exclusive_scan(c, nullptr);
#pragma unroll
  for (int j = 0; j < kSelItems; ++j) {
    if (!f[j]) continue;
    if (rank < (uint32_t)S) {
      out_sampled[rank] = draws[base + j];
      if (rank == (uint32_t)S - 1) *out_num_tries = base + j + 1;
    }
    ++rank;
  }
}

// Expected counts (R-10, R-24) and scratch restore.
__device__ __forceinline__ float log_expected_count(int64_t k, int64_t V, double log_v1,
                                                    int unique, int64_t T, int32_t S) {
  const double p = log1p(1.0 / (double)(k + 1)) / log_v1;  // ln((k+2)/(k+1)) / ln(V+1)
  const double ec = unique ? -expm1((double)T * log1p(-p)) : (double)S * p;
  return (float)log(ec);
}

__global__ void sample_finish_kernel(const int32_t* draws, int32_t* firstpos, int64_t N, int unique,
                                     int64_t V, double log_v1, int32_t S,
                                     const int64_t* out_sampled, const int64_t* labels,
                                     int64_t n_labels, const int64_t* num_tries, float* les,
                                     float* ley, tfs_device_error* err) {
  pdl_enter();
  const int64_t T = unique ? *num_tries : (int64_t)S;
  const int64_t nl = (int64_t)S + n_labels;
  const int64_t total = (unique && N > nl) ? N : nl;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (unique && e < N) firstpos[draws[e]] = 0x7fffffff;
    if (e < S) {
      int64_t k = out_sampled[e];
      k = k < 0 ? 0 : (k >= V ? V - 1 : k);
      les[e] = log_expected_count(k, V, log_v1, unique, T, S);
    } else if (e < (int64_t)S + n_labels) {
      const int64_t t = e - S;
      const int64_t k = labels[t];
      if (k < 0 || k >= V) {
        report_error(err, TFS_ERR_OUT_OF_RANGE, t);
        ley[t] = 0.f;
      } else {
        ley[t] = log_expected_count(k, V, log_v1, unique, T, S);
      }
    }
  }
}

__global__ void set_i64_kernel(int64_t* p, int64_t v) {
  pdl_enter(); *p = v; }

// Commit of a sample drawn ahead of time: copy (s, log ec(s), T) into the step's buffers and
// form the labels' log expected counts with that T.
__global__ void sample_commit_kernel(int64_t V, double log_v1, int unique, int32_t S,
                                     const int64_t* s_in, const float* les_in,
                                     const int64_t* T_in, const int64_t* labels, int64_t n_labels,
                                     int64_t* s_out, float* les_out, float* ley_out,
                                     int64_t* T_out, int64_t* labels_out, tfs_device_error* err) {
  pdl_enter();
  const int64_t T = unique ? *T_in : (int64_t)S;
  const int64_t total = (int64_t)S + n_labels;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e == 0) *T_out = *T_in;
    if (e < S) {
      s_out[e] = s_in[e];
      les_out[e] = les_in[e];
    } else {
      const int64_t t = e - S;
      const int64_t k = labels[t];
      if (labels_out != nullptr) labels_out[t] = k;
      if (k < 0 || k >= V) {
        report_error(err, TFS_ERR_OUT_OF_RANGE, t);
        ley_out[t] = 0.f;
      } else {
        ley_out[t] = log_expected_count(k, V, log_v1, unique, T, S);
      }
    }
  }
}

}  // namespace tfs

using namespace tfs;

extern "C" size_t tfs_sampler_state_bytes(int64_t vocab) {
  Carver c(nullptr, 0);
  c.take<uint64_t>(vocab);
  c.take<int32_t>(vocab);
  return c.used + 256;
}

// Draw budget: smallest N such that P(#distinct in N draws < S) <= 1e-21 by Bernstein's
// inequality on the number X of ids never drawn (a sum of negatively associated indicators
// with mean M(N) = sum_k (1 - p_k)^N): fewer than S distinct <=> X >= V - S + 1.
static int64_t draw_budget(int64_t V, int32_t S) {
  std::vector<double> lq((size_t)V);
  const double lv1 = std::log((double)V + 1.0);
  for (int64_t k = 0; k < V; ++k) lq[k] = std::log1p(-std::log1p(1.0 / (double)(k + 1)) / lv1);
  auto ok = [&](int64_t N) {
    double M = 0.0;
    for (int64_t k = 0; k < V; ++k) M += std::exp((double)N * lq[k]);
    const double t = (double)(V - S + 1) - M;
    return t > 0 && t * t / (2.0 * (M + t / 3.0)) >= 48.4;  // exp(-48.4) < 1e-21
  };
  int64_t lo = std::max<int64_t>(S, 1), hi = (1ll << 31) - 1;
  if (!ok(hi)) return hi;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (ok(mid)) hi = mid; else lo = mid + 1;
  }
  return lo;
}

extern "C" int32_t tfs_sampler_init(int64_t vocab, int32_t num_sampled, int32_t unique,
                                    void* state, int64_t* out_max_draws, void* stream) {
  TFS_REQUIRE(vocab >= 1 && vocab < (1ll << 31) - 1 && num_sampled >= 0 && state && out_max_draws);
  TFS_REQUIRE(!unique || num_sampled <= vocab);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  // Inverse-CDF thresholds Thr[k] = floor(2^53 ln(k+2) / ln(V+1)) in host long double (R-17).
  std::vector<uint64_t> thr((size_t)vocab);
  const long double lden = logl((long double)vocab + 1.0L);
  for (int64_t k = 0; k < vocab; ++k)
    thr[k] = (uint64_t)floorl(ldexpl(logl((long double)(k + 2)) / lden, 53));
  thr[vocab - 1] = 1ull << 53;
  SamplerState s = carve_state(state, vocab);
  TFS_CUDA_TRY(cudaMemcpyAsync((void*)s.thr, thr.data(), sizeof(uint64_t) * vocab,
                               cudaMemcpyHostToDevice, st));
  TFS_CUDA_TRY(cudaMemsetAsync(s.firstpos, 0x7f, sizeof(int32_t) * vocab, st));
  // 0x7f7f7f7f > any draw index: "not seen".
  TFS_CUDA_TRY(cudaStreamSynchronize(st));
  *out_max_draws = unique ? draw_budget(vocab, num_sampled) : num_sampled;
  return TFS_OK;
}

extern "C" size_t tfs_sampler_workspace_bytes(int64_t max_draws) {
  Carver c(nullptr, 0);
  c.take<int32_t>(max_draws);
  c.take<uint32_t>(cdiv(max_draws, kSelTile) + 1);
  return c.used + 256;
}

extern "C" int32_t tfs_log_uniform_sample(const void* state, int64_t vocab, int32_t num_sampled,
                                          int32_t unique, int64_t max_draws, uint64_t seed,
                                          uint64_t step, const uint64_t* step_dev,
                                          uint32_t replica, const int64_t* labels,
                                          int64_t n_labels, int64_t* out_sampled,
                                          float* out_log_ec_sampled, float* out_log_ec_labels,
                                          int64_t* out_num_tries, void* ws, size_t ws_bytes,
                                          tfs_device_error* err, void* stream) {
  TFS_REQUIRE(state && vocab >= 1 && num_sampled >= 0 && n_labels >= 0 && out_num_tries);
  TFS_REQUIRE(!unique || (num_sampled <= vocab && max_draws >= num_sampled));
  TFS_REQUIRE(max_draws < (1ll << 31));
  TFS_REQUIRE(num_sampled == 0 || (out_sampled && out_log_ec_sampled));
  TFS_REQUIRE(n_labels == 0 || (labels && out_log_ec_labels));
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  SamplerState s = carve_state((void*)state, vocab);
  const double log_v1 = std::log((double)vocab + 1.0);
  if (num_sampled == 0) {
    ::tfs::launch(set_i64_kernel, 1, 1, 0, st, out_num_tries, 0); ::tfs::launched();
  } else if (!unique) {
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(num_sampled, 256), 4 * num_sms()));
    ::tfs::launch(sample_draw_kernel, g, 256, 0, st, s.thr, vocab, log_v1, num_sampled, seed, step, step_dev, replica,
                                          0, nullptr, nullptr, out_sampled); ::tfs::launched();
    ::tfs::launch(set_i64_kernel, 1, 1, 0, st, out_num_tries, num_sampled); ::tfs::launched();
  } else {
    if (ws_bytes < tfs_sampler_workspace_bytes(max_draws)) return TFS_ERR_WORKSPACE_TOO_SMALL;
    Carver c(ws, ws_bytes);
    int32_t* draws = c.take<int32_t>(max_draws);
    const int nblk = (int)cdiv(max_draws, kSelTile);
    uint32_t* blk = c.take<uint32_t>(nblk + 1);
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(max_draws, 256), num_sms()));
    ::tfs::launch(sample_draw_kernel, g, 256, 0, st, s.thr, vocab, log_v1, max_draws, seed, step, step_dev, replica,
                                          1, draws, s.firstpos, nullptr); ::tfs::launched();
    ::tfs::launch(sample_count_kernel, nblk, kSelThreads, 0, st, draws, s.firstpos, max_draws, blk); ::tfs::launched();
    ::tfs::launch(sample_select_kernel, nblk, kSelThreads, 0, st, draws, s.firstpos, max_draws, blk, nblk,
                                                       num_sampled, out_sampled, out_num_tries, err); ::tfs::launched();
    TFS_LAUNCH_CHECK();
    const int64_t total = std::max<int64_t>(max_draws, num_sampled + n_labels);
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 4 * num_sms()));
    ::tfs::launch(sample_finish_kernel, g2, 256, 0, st, draws, s.firstpos, max_draws, 1, vocab, log_v1,
                                             num_sampled, out_sampled, labels, n_labels,
                                             out_num_tries, out_log_ec_sampled, out_log_ec_labels,
                                             err); ::tfs::launched();
    TFS_LAUNCH_CHECK();
    return TFS_OK;
  }
  const int64_t total = (int64_t)num_sampled + n_labels;
  if (total > 0) {
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 4 * num_sms()));
    ::tfs::launch(sample_finish_kernel, g2, 256, 0, st, nullptr, nullptr, 0, unique, vocab, log_v1,
                                             num_sampled, out_sampled, labels, n_labels,
                                             out_num_tries, out_log_ec_sampled, out_log_ec_labels,
                                             err); ::tfs::launched();
  }
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_sample_commit(int64_t vocab, int32_t num_sampled, int32_t unique,
                                     const int64_t* sampled, const float* log_ec_sampled,
                                     const int64_t* num_tries, const int64_t* labels,
                                     int64_t n_labels, int64_t* out_sampled,
                                     float* out_log_ec_sampled, float* out_log_ec_labels,
                                     int64_t* out_num_tries, int64_t* out_labels,
                                     tfs_device_error* err, void* stream) {
  TFS_REQUIRE(vocab >= 1 && num_sampled >= 0 && n_labels >= 0 && num_tries && out_num_tries);
  TFS_REQUIRE(num_sampled == 0 || (sampled && log_ec_sampled && out_sampled && out_log_ec_sampled));
  TFS_REQUIRE(n_labels == 0 || (labels && out_log_ec_labels));
  TFS_SUPPORTED();
  const int64_t total = std::max<int64_t>(1, (int64_t)num_sampled + n_labels);
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 4 * num_sms()));
  ::tfs::launch(sample_commit_kernel, g, 256, 0, as_stream(stream), 
      vocab, std::log((double)vocab + 1.0), unique, num_sampled, sampled, log_ec_sampled,
      num_tries, labels, n_labels, out_sampled, out_log_ec_sampled, out_log_ec_labels,
      out_num_tries, out_labels, err);
  ::tfs::launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}
