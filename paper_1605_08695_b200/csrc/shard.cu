// shard.cu -- cross-shard pieces of the vocabulary-sharded full softmax (P:706-714,
// P:1159-1166): the (max, sum) combine into lse, the pull-reduce of dh partials, the loss over
// the labels a shard owns, and the dense SGD of a shard's W / b with its bf16 operand shadow.
// Peer buffers are read with plain loads through symmetric-memory pointers (NVLink P2P).
#include "common.cuh"

#include <algorithm>

namespace tfs {
namespace {

constexpr float kLn2f = 0.6931471805599453f;

// lse[t] from the R shards' (m, s) pairs, in rank order.
__global__ void lse_combine_peers_kernel(const float* const* tab, int R, int64_t n, float* lse) {
  pdl_enter();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  float m = -INFINITY;
  for (int r = 0; r < R; ++r) m = fmaxf(m, tab[r][2 * t]);
  float s = 0.f;
  if (m > -INFINITY)
    for (int r = 0; r < R; ++r) {
      const float2 x = reinterpret_cast<const float2*>(tab[r])[t];
      if (x.y > 0.f) s += x.y * exp2f(x.x - m);
    }
  lse[t] = (m + log2f(s)) * kLn2f;
}

template <bool VEC>
__global__ void reduce_peers_kernel(const float* const* tab, int R, int64_t offset, int64_t n,
                                    float* out) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    const int64_t n4 = n / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 acc = reinterpret_cast<const float4*>(tab[0] + offset)[i];
      for (int r = 1; r < R; ++r) {
        const float4 x = reinterpret_cast<const float4*>(tab[r] + offset)[i];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
      reinterpret_cast<float4*>(out)[i] = acc;
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      float acc = tab[0][offset + i];
      for (int r = 1; r < R; ++r) acc += tab[r][offset + i];
      out[i] = acc;
    }
  }
}

// One block: per-thread partial sums over a fixed strided range, then a fixed tree.
__global__ void __launch_bounds__(1024) label_loss_kernel(const float* lse, const float* zl,
                                                          const int64_t* labels, int64_t n, int R,
                                                          int shard, float c, float* out) {
  pdl_enter();
  __shared__ float red[1024];
  float acc = 0.f;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    const int64_t y = labels[t];
    if (y >= 0 && y % R == shard) acc += lse[t] - zl[t];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = c * red[0];
}

__global__ void dense_sgd_kernel(float4* table, const float4* grad, int64_t n, float lr,
                                 uint2* shadow) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = n / 4;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i0 < n % 4) {  // tail elements (n % 4 of them)
    const int64_t e = n4 * 4 + i0;
    float* t = reinterpret_cast<float*>(table);
    t[e] -= lr * reinterpret_cast<const float*>(grad)[e];
    if (shadow != nullptr) reinterpret_cast<uint16_t*>(shadow)[e] = f32_to_bf16_bits(t[e]);
  }
  for (int64_t i = i0; i < n4; i += stride) {
    float4 w = table[i];
    const float4 g = grad[i];
    w.x -= lr * g.x;
    w.y -= lr * g.y;
    w.z -= lr * g.z;
    w.w -= lr * g.w;
    table[i] = w;
    if (shadow != nullptr) shadow[i] = make_uint2(pack_bf16x2(w.x, w.y), pack_bf16x2(w.z, w.w));
  }
}

int grid_for(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8ll * num_sms()));
}

}  // namespace
}  // namespace tfs

using namespace tfs;

extern "C" int32_t tfs_lse_combine_peers(const float* const* stats_tab, int32_t R, int64_t n,
                                         float* lse, void* stream) {
  TFS_REQUIRE(R >= 1 && n >= 0);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(stats_tab && lse);
  TFS_SUPPORTED();
  ::tfs::launch(lse_combine_peers_kernel, (unsigned)cdiv(n, 256), 256, 0, as_stream(stream), stats_tab, R, n,
                                                                                 lse);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_reduce_peers(const float* const* src_tab, int32_t R, int64_t offset,
                                    int64_t n, float* out, void* stream) {
  TFS_REQUIRE(R >= 1 && n >= 0 && offset >= 0);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(src_tab && out);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  const bool vec = n % 4 == 0 && offset % 4 == 0 && ((uintptr_t)out & 15) == 0;
  if (vec)
    ::tfs::launch(reduce_peers_kernel<true>, grid_for(n / 4), 256, 0, st, src_tab, R, offset, n, out);
  else
    ::tfs::launch(reduce_peers_kernel<false>, grid_for(n), 256, 0, st, src_tab, R, offset, n, out);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_label_loss_sum(const float* lse, const float* z_label,
                                      const int64_t* labels, int64_t n, int32_t R, int32_t shard,
                                      float c, float* out, void* stream) {
  TFS_REQUIRE(R >= 1 && shard >= 0 && shard < R && n >= 0 && out);
  TFS_REQUIRE(n == 0 || (lse && z_label && labels));
  TFS_SUPPORTED();
  ::tfs::launch(label_loss_kernel, 1, 1024, 0, as_stream(stream), lse, z_label, labels, n, R, shard, c, out);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_dense_sgd(float* table, const float* grad, int64_t n, float lr,
                                 void* shadow, void* stream) {
  TFS_REQUIRE(n >= 0);
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && grad && ((uintptr_t)table & 15) == 0 && ((uintptr_t)grad & 15) == 0);
  TFS_REQUIRE(((uintptr_t)shadow & 7) == 0);
  TFS_SUPPORTED();
  ::tfs::launch(dense_sgd_kernel, grid_for(n / 4 + 1), 256, 0, as_stream(stream), 
      reinterpret_cast<float4*>(table), reinterpret_cast<const float4*>(grad), n, lr,
      static_cast<uint2*>(shadow));
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}
