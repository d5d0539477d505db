// sort.cu -- Part, the stable digit-sort engine it shares with the LSD radix sort,
// and the deterministic sort-by-id segmented reductions behind the sparse gradient path:
// tfs_sort_reduce (gradient rows summed per id before routing) and
// tfs_scatter_add_sgd (ScatterAdd/SGD "-=" on the owner shard).
//
// Design: HBM/latency-bound integer work.  A tile of 4096 items per 256-thread
// CTA; per-tile digit histograms; every CTA computes its own global offsets from the (small)
// histogram table, so a pass is two launches with no separate scan.  Within a tile the rank
// of an item among equal digits is computed with warp __match_any_sync + popc and a per-round
// warp-order prefix, which makes the scatter stable (original order kept: R-2).  Floating
// point sums over duplicate ids run in increasing original position inside each segment
// (fixed order, no float atomics: run-to-run bit-identical, R-16).
#include <algorithm>

#include "common.cuh"

namespace tfs {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 items per CTA
constexpr int kMaxBuckets = 256;
constexpr int kLongSeg = 256;  // segments longer than this are summed by a whole CTA

struct DigitSrc {
  int mode;
  const int64_t* ids;
  const int32_t* assign;
  int64_t vocab;
  int32_t nshards;
  const uint32_t* keys;
  int shift;
  int nbuckets;
};

__device__ __forceinline__ int digit_of(const DigitSrc& s, int64_t i, tfs_device_error* err) {
  if (s.mode == kDigitRadix) return (int)((s.keys[i] >> s.shift) & 0xffu);
  if (s.mode == kDigitMod) {
    int64_t id = s.ids[i];
    if (id < 0 || id >= s.vocab) {
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      return 0;
    }
    return (int)(id % s.nshards);
  }
  int32_t a = s.assign[i];
  if (a < 0 || a >= s.nshards) {
    report_error(err, TFS_ERR_OUT_OF_RANGE, i);
    return 0;
  }
  return a;
}

// Exclusive scan of one value per thread over a 256-thread CTA (fixed order).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[kSortWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  uint32_t base = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) {
    uint32_t ws = warp_sums[w];
    if (w < warp) base += ws;
    all += ws;
  }
  __syncthreads();
  if (total) *total = all;
  return base + x - v;
}

__global__ void __launch_bounds__(kSortThreads) digit_hist_kernel(DigitSrc src, int64_t n,
                                                                  uint32_t* hist, int ntiles,
                                                                  tfs_device_error* err) {
  __shared__ uint32_t cnt[kMaxBuckets];
  const int nb = src.nbuckets;
  for (int b = threadIdx.x; b < nb; b += kSortThreads) cnt[b] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = base + (int64_t)j * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&cnt[digit_of(src, i, err)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kSortThreads) hist[(int64_t)b * ntiles + blockIdx.x] = cnt[b];
}

struct PartSink {  // tfs_partition outputs
  int64_t* local;
  int64_t* positions;
  int64_t* counts;
  __device__ void put(const DigitSrc& s, uint32_t pos, int64_t i) const {
    int64_t id = s.ids[i];
    local[pos] = s.mode == kDigitMod ? id / s.nshards : id;
    positions[pos] = i;
  }
};

struct RadixSink {  // one LSD pass
  const uint32_t* vals_in;
  uint32_t* keys_out;
  uint32_t* vals_out;
  __device__ void put(const DigitSrc& s, uint32_t pos, int64_t i) const {
    keys_out[pos] = s.keys[i];
    vals_out[pos] = vals_in ? vals_in[i] : (uint32_t)i;
  }
};

template <class Sink>
__global__ void __launch_bounds__(kSortThreads) digit_scatter_kernel(DigitSrc src, int64_t n,
                                                                     const uint32_t* hist,
                                                                     int ntiles, Sink sink,
                                                                     int64_t* counts_out) {
  __shared__ uint32_t running[kMaxBuckets];
  __shared__ uint32_t wcnt[kSortWarps][kMaxBuckets];
  const int nb = src.nbuckets;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = blockIdx.x;

  // Global base of every bucket for this tile: all earlier buckets + this bucket in earlier tiles.
  uint32_t tot = 0, pre = 0;
  if (tid < nb) {
    const uint32_t* h = hist + (int64_t)tid * ntiles;
    for (int t = 0; t < ntiles; ++t) {
      uint32_t c = h[t];
      tot += c;
      if (t < tile) pre += c;
    }
  }
  uint32_t excl = block_exclusive_scan(tid < nb ? tot : 0u, nullptr);
  if (tid < nb) {
    running[tid] = excl + pre;
    if (counts_out != nullptr && tile == 0) counts_out[tid] = (int64_t)tot;
  }
  __syncthreads();

  const int64_t base = (int64_t)tile * kSortTile;
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + (int64_t)j * kSortThreads + tid;
    const bool valid = i < n;
    const int dg = valid ? digit_of(src, i, nullptr) : -1;
    for (int b = tid; b < kSortWarps * nb; b += kSortThreads) wcnt[b / nb][b % nb] = 0;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    const uint32_t rank = __popc(peers & lanemask_lt());
    if (valid && rank == 0) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    if (tid < nb) {
      uint32_t p = running[tid];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        uint32_t c = wcnt[w][tid];
        wcnt[w][tid] = p;
        p += c;
      }
      running[tid] = p;
    }
    __syncthreads();
    if (valid) sink.put(src, wcnt[warp][dg] + rank, i);
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------------
// Radix sort of (key, val) pairs.
size_t radix_sort_ws_bytes(int64_t n) {
  Carver c(nullptr, 0);
  int64_t ntiles = cdiv(n, kSortTile);
  c.take<uint32_t>(n);
  c.take<uint32_t>(n);
  c.take<uint32_t>((size_t)kMaxBuckets * ntiles + 1);
  return c.used + 256;
}

int32_t radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                         uint32_t* vals_out, int64_t n, int key_bits, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  if (n == 0) return TFS_OK;
  Carver c(ws, ws_bytes);
  const int ntiles = (int)cdiv(n, kSortTile);
  uint32_t* tk = c.take<uint32_t>(n);
  uint32_t* tv = c.take<uint32_t>(n);
  uint32_t* hist = c.take<uint32_t>((size_t)kMaxBuckets * ntiles + 1);
  if (!c.fits()) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int passes = key_bits <= 8 ? 1 : (key_bits + 7) / 8;
  // Ping-pong so that the last pass lands in keys_out / vals_out.
  const uint32_t* ksrc = keys_in;
  const uint32_t* vsrc = vals_in;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    uint32_t* kd = to_out ? keys_out : tk;
    uint32_t* vd = to_out ? vals_out : tv;
    DigitSrc s{kDigitRadix, nullptr, nullptr, 0, 0, ksrc, 8 * p, 256};
    digit_hist_kernel<<<ntiles, kSortThreads, 0, st>>>(s, n, hist, ntiles, nullptr);
    digit_scatter_kernel<RadixSink><<<ntiles, kSortThreads, 0, st>>>(
        s, n, hist, ntiles, RadixSink{vsrc, kd, vd}, nullptr);
    TFS_LAUNCH_CHECK();
    ksrc = kd;
    vsrc = vd;
  }
  return TFS_OK;
}

}  // namespace tfs

using namespace tfs;

// ================================================================================================
// Part
extern "C" size_t tfs_partition_workspace_bytes(int64_t n, int32_t num_shards) {
  (void)num_shards;
  return (size_t)kMaxBuckets * cdiv(n, kSortTile) * sizeof(uint32_t) + 256;
}

extern "C" int32_t tfs_partition(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                                 const int32_t* assignments, int64_t* out_local,
                                 int64_t* out_positions, int64_t* out_counts, void* ws,
                                 size_t ws_bytes, tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && num_shards >= 1 && num_shards <= kMaxBuckets && n < (1ll << 31));
  TFS_REQUIRE(out_counts != nullptr);
  TFS_REQUIRE(n == 0 || (ids && out_local && out_positions));
  TFS_REQUIRE(assignments != nullptr || vocab >= 1);
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TFS_CUDA_TRY(cudaMemsetAsync(out_counts, 0, sizeof(int64_t) * num_shards, st));
    return TFS_OK;
  }
  if (ws_bytes < tfs_partition_workspace_bytes(n, num_shards)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int ntiles = (int)cdiv(n, kSortTile);
  uint32_t* hist = (uint32_t*)ws;
  DigitSrc s{assignments ? kDigitAssign : kDigitMod, ids, assignments, vocab, num_shards,
             nullptr, 0, num_shards};
  digit_hist_kernel<<<ntiles, kSortThreads, 0, st>>>(s, n, hist, ntiles, err);
  digit_scatter_kernel<PartSink><<<ntiles, kSortThreads, 0, st>>>(
      s, n, hist, ntiles, PartSink{out_local, out_positions, out_counts}, out_counts);
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

// ================================================================================================
// Segmented reductions over id-sorted gradient rows.
namespace tfs {

static int bits_for(uint64_t max_value) {
  int b = 1;
  while (b < 32 && (max_value >> b) != 0) ++b;
  return b;
}

// keys for ScatterAdd: key = id (invalid -> sentinel `rows`); for sort_reduce: key =
// owner * nloc + local.
__global__ void make_keys_kernel(const int64_t* ids, int64_t n, int64_t limit, int32_t R,
                                 int64_t nloc, int composite, uint32_t* keys, uint32_t* vals,
                                 tfs_device_error* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t id = ids[i];
    uint32_t key;
    if (id < 0 || id >= limit) {
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      key = composite ? (uint32_t)(R * nloc) : (uint32_t)limit;  // sorts last, skipped later
    } else {
      key = composite ? (uint32_t)((id % R) * nloc + id / R) : (uint32_t)id;
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

// Segment heads of a sorted key array: per-tile head counts, then per-tile starts.
__global__ void __launch_bounds__(kSortThreads) heads_count_kernel(const uint32_t* k, int64_t n,
                                                                   uint32_t* tile_cnt) {
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)threadIdx.x * kSortItems;
  uint32_t c = 0;
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = base + j;
    if (i < n && (i == 0 || k[i] != k[i - 1])) ++c;
  }
  uint32_t total;
  block_exclusive_scan(c, &total);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kSortThreads) heads_write_kernel(const uint32_t* k, int64_t n,
                                                                   const uint32_t* tile_cnt,
                                                                   int ntiles,
                                                                   uint32_t* seg_start,
                                                                   int64_t* num_unique) {
  __shared__ uint32_t tile_base;
  if (threadIdx.x < 32) {
    uint32_t pre = 0, all = 0;
    for (int t = threadIdx.x; t < ntiles; t += 32) {
      uint32_t c = tile_cnt[t];
      all += c;
      if (t < (int)blockIdx.x) pre += c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (threadIdx.x == 0) {
      tile_base = pre;
      if (blockIdx.x == 0) {
        *num_unique = all;
        seg_start[all] = (uint32_t)n;  // sentinel end of the last segment
      }
    }
  }
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)threadIdx.x * kSortItems;
  uint32_t c = 0;
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = base + j;
    if (i < n && (i == 0 || k[i] != k[i - 1])) ++c;
  }
  uint32_t pos = tile_base + block_exclusive_scan(c, nullptr);
  for (int j = 0; j < kSortItems; ++j) {
    int64_t i = base + j;
    if (i < n && (i == 0 || k[i] != k[i - 1])) seg_start[pos++] = (uint32_t)i;
  }
}

struct SegJob {
  const uint32_t* keys;       // sorted keys
  const uint32_t* perm;       // original index of each sorted position
  const uint32_t* seg_start;  // [U + 1]
  const int64_t* num_unique;  // device U
  const float* rows;          // [n x dim] gradient rows (original order)
  const float* rows2;         // optional [n] companion values
  int32_t dim;
  uint32_t invalid_key;       // keys >= invalid_key are skipped (bad ids)
  // apply mode (ScatterAdd-SGD): table[key] -= lr * sum
  float* table;
  float* table2;
  float lr;
  // write mode (sort_reduce): out_local[s], out_rows[s]
  int64_t* out_local;
  float* out_rows;
  float* out_rows2;
  int64_t nloc;
  uint32_t* long_list;
  uint32_t* long_count;
};

// Row sums are accumulated in fp64 (one rounding to fp32 at the end), in increasing original
// position: the fixed order makes them run-to-run bit-identical (R-16) and fp64 keeps
// thousand-way duplicate sums (Zipf heavy hitters) within the fp32 parity bound.
struct D4 {
  double x, y, z, w;
};

__device__ __forceinline__ void add4(D4& a, const float4& v) {
  a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
}

// Sum of rows perm[a..b) (in order) for the float4 columns c4_0 + 32*v + lane this lane owns.
template <int V>
__device__ __forceinline__ void sum_rows_vec4(const SegJob& j, uint32_t a, uint32_t b, int c4_0,
                                              D4 (&acc)[V]) {
  const int lane = threadIdx.x & 31;
  const int n4 = j.dim >> 2;
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = D4{0.0, 0.0, 0.0, 0.0};
  uint32_t i = a;
  for (; i + 1 < b; i += 2) {  // two rows in flight
    const float4* r0 = (const float4*)(j.rows + (int64_t)j.perm[i] * j.dim);
    const float4* r1 = (const float4*)(j.rows + (int64_t)j.perm[i + 1] * j.dim);
    float4 x0[V], x1[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = c4_0 + v * 32 + lane;
      x0[v] = c < n4 ? __ldg(r0 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      x1[v] = c < n4 ? __ldg(r1 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      add4(acc[v], x0[v]);
      add4(acc[v], x1[v]);
    }
  }
  if (i < b) {
    const float4* r0 = (const float4*)(j.rows + (int64_t)j.perm[i] * j.dim);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int c = c4_0 + v * 32 + lane;
      if (c < n4) add4(acc[v], __ldg(r0 + c));
    }
  }
}

// ScatterAdd-SGD: T = fl32(T - lr * g) evaluated in fp64; sort_reduce: out = fl32(g).
__device__ __forceinline__ void emit_vec4(const SegJob& j, uint32_t s, uint32_t key, int c4,
                                          const D4& v) {
  if (j.table != nullptr) {
    float4* t = (float4*)(j.table + (int64_t)key * j.dim) + c4;
    float4 w = *t;
    const double lr = (double)j.lr;
    w.x = (float)((double)w.x - lr * v.x);
    w.y = (float)((double)w.y - lr * v.y);
    w.z = (float)((double)w.z - lr * v.z);
    w.w = (float)((double)w.w - lr * v.w);
    *t = w;
  } else {
    ((float4*)(j.out_rows + (int64_t)s * j.dim))[c4] =
        make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
  }
}

__device__ __forceinline__ void emit_scalar(const SegJob& j, uint32_t s, uint32_t key, int c,
                                            double v) {
  if (j.table != nullptr) {
    float* t = j.table + (int64_t)key * j.dim + c;
    *t = (float)((double)*t - (double)j.lr * v);
  } else {
    j.out_rows[(int64_t)s * j.dim + c] = (float)v;
  }
}

__device__ __forceinline__ void emit_companion(const SegJob& j, uint32_t s, uint32_t key,
                                               double v) {
  if (j.table != nullptr) {
    if (j.table2) j.table2[key] = (float)((double)j.table2[key] - (double)j.lr * v);
  } else if (j.out_rows2) {
    j.out_rows2[s] = (float)v;
  }
}

// One warp per (short) segment.
__global__ void __launch_bounds__(256) seg_sum_kernel(SegJob j) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t U = *j.num_unique;
  for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < U;
       s += warps) {
    const uint32_t a = j.seg_start[s], b = j.seg_start[s + 1];
    const uint32_t key = j.keys[a];
    if (key >= j.invalid_key) continue;
    if (j.out_local) j.out_local[s] = (int64_t)(key % (uint32_t)j.nloc);
    if (b - a > (uint32_t)kLongSeg) {
      if (lane == 0) j.long_list[atomicAdd(j.long_count, 1u)] = (uint32_t)s;
      continue;
    }
    if ((j.dim & 3) == 0) {
      const int n4 = j.dim >> 2;
      for (int c4_0 = 0; c4_0 < n4; c4_0 += 4 * 32) {
        D4 acc[4];
        sum_rows_vec4<4>(j, a, b, c4_0, acc);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c4 = c4_0 + v * 32 + lane;
          if (c4 < n4) emit_vec4(j, (uint32_t)s, key, c4, acc[v]);
        }
      }
    } else {
      for (int c = lane; c < j.dim; c += 32) {
        double acc = 0.0;
        for (uint32_t i = a; i < b; ++i) acc += j.rows[(int64_t)j.perm[i] * j.dim + c];
        emit_scalar(j, (uint32_t)s, key, c, acc);
      }
    }
    if (j.rows2 != nullptr && lane == 0) {
      double acc = 0.0;
      for (uint32_t i = a; i < b; ++i) acc += j.rows2[j.perm[i]];
      emit_companion(j, (uint32_t)s, key, acc);
    }
  }
}

// One CTA per long segment: 8 warps sum 8 contiguous pieces (in order), then the pieces are
// added in piece order.  The split depends only on the segment length: deterministic.
__global__ void __launch_bounds__(256) seg_sum_long_kernel(SegJob j) {
  extern __shared__ double part[];  // [8][dim] + [8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cnt = *j.long_count;
  for (uint32_t q = blockIdx.x; q < cnt; q += gridDim.x) {
    const uint32_t s = j.long_list[q];
    const uint32_t a = j.seg_start[s], b = j.seg_start[s + 1];
    const uint32_t key = j.keys[a];
    const uint32_t len = b - a;
    const uint32_t pa = a + (uint32_t)(((uint64_t)len * warp) / 8);
    const uint32_t pb = a + (uint32_t)(((uint64_t)len * (warp + 1)) / 8);
    for (int c = lane; c < j.dim; c += 32) {
      double acc = 0.0;
      for (uint32_t i = pa; i < pb; ++i) acc += j.rows[(int64_t)j.perm[i] * j.dim + c];
      part[warp * j.dim + c] = acc;
    }
    if (j.rows2 != nullptr && lane == 0) {
      double acc = 0.0;
      for (uint32_t i = pa; i < pb; ++i) acc += j.rows2[j.perm[i]];
      part[8 * j.dim + warp] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < j.dim; c += blockDim.x) {
      double acc = part[c];
      for (int w = 1; w < 8; ++w) acc += part[w * j.dim + c];
      emit_scalar(j, s, key, c, acc);
    }
    if (j.rows2 != nullptr && threadIdx.x == 0) {
      double acc = part[8 * j.dim];
      for (int w = 1; w < 8; ++w) acc += part[8 * j.dim + w];
      emit_companion(j, s, key, acc);
    }
    __syncthreads();
  }
}

__global__ void owner_counts_kernel(const uint32_t* keys, const uint32_t* seg_start,
                                    const int64_t* num_unique, int32_t R, int64_t nloc,
                                    uint32_t invalid_key, int64_t* counts) {
  const int o = threadIdx.x;
  if (o >= R) return;
  const int64_t U = *num_unique;
  auto first_ge = [&](int64_t owner) {  // first segment whose owner >= `owner`
    int64_t lo = 0, hi = U;
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      uint32_t k = keys[seg_start[mid]];
      int64_t ow = k >= invalid_key ? R : (int64_t)(k / (uint32_t)nloc);
      if (ow < owner) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  counts[o] = first_ge(o + 1) - first_ge(o);
}

struct SegScratch {
  uint32_t *k0, *v0, *k1, *v1, *seg_start, *tile_cnt, *long_list, *long_count;
  int64_t* num_unique;
  void* sort_ws;
  size_t sort_ws_bytes;
};

static size_t seg_scratch_bytes(int64_t n, SegScratch* s, void* ws, size_t cap) {
  Carver c(ws, cap);
  int64_t ntiles = cdiv(n, kSortTile);
  uint32_t* k0 = c.take<uint32_t>(n);
  uint32_t* v0 = c.take<uint32_t>(n);
  uint32_t* k1 = c.take<uint32_t>(n);
  uint32_t* v1 = c.take<uint32_t>(n);
  uint32_t* ss = c.take<uint32_t>(n + 1);
  uint32_t* tc = c.take<uint32_t>(ntiles + 1);
  uint32_t* ll = c.take<uint32_t>(n / kLongSeg + 1);
  uint32_t* lc = c.take<uint32_t>(1);
  int64_t* nu = c.take<int64_t>(1);
  size_t rs = radix_sort_ws_bytes(n);
  char* rws = c.take<char>(rs);
  if (s) *s = SegScratch{k0, v0, k1, v1, ss, tc, ll, lc, nu, rws, rs};
  return c.used + 256;
}

static int32_t sort_and_segment(const int64_t* ids, int64_t n, int64_t limit, int32_t R,
                                int64_t nloc, int composite, uint32_t key_max, SegScratch& s,
                                tfs_device_error* err, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>(cdiv(n, 256), 4 * num_sms());
  make_keys_kernel<<<grid, 256, 0, st>>>(ids, n, limit, R, nloc, composite, s.k0, s.v0, err);
  TFS_LAUNCH_CHECK();
  int32_t rc = radix_sort_pairs(s.k0, s.v0, s.k1, s.v1, n, bits_for(key_max), s.sort_ws,
                                s.sort_ws_bytes, st);
  if (rc != TFS_OK) return rc;
  const int ntiles = (int)cdiv(n, kSortTile);
  heads_count_kernel<<<ntiles, kSortThreads, 0, st>>>(s.k1, n, s.tile_cnt);
  heads_write_kernel<<<ntiles, kSortThreads, 0, st>>>(s.k1, n, s.tile_cnt, ntiles, s.seg_start,
                                                      s.num_unique);
  TFS_CUDA_TRY(cudaMemsetAsync(s.long_count, 0, sizeof(uint32_t), st));
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

static int32_t run_segments(SegJob& j, int64_t n, cudaStream_t st) {
  const int64_t warps_needed = n;  // U <= n
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(warps_needed, 8), 8 * num_sms()));
  seg_sum_kernel<<<grid, 256, 0, st>>>(j);
  const size_t smem = (size_t)(8 * j.dim + 8) * sizeof(double);
  if (smem > 48 * 1024) {
    TFS_CUDA_TRY(cudaFuncSetAttribute(seg_sum_long_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const int lgrid = (int)std::max<int64_t>(1, std::min<int64_t>(n / kLongSeg + 1, num_sms()));
  seg_sum_long_kernel<<<lgrid, 256, smem, st>>>(j);
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

}  // namespace tfs

// ================================================================================================
extern "C" size_t tfs_scatter_add_sgd_workspace_bytes(int64_t n, int32_t dim) {
  (void)dim;
  return seg_scratch_bytes(n, nullptr, nullptr, 0);
}

extern "C" int32_t tfs_scatter_add_sgd(float* table, int64_t rows, int32_t dim, const int64_t* ids,
                                       const float* grad_rows, int64_t n, float lr, float* table2,
                                       const float* grad2, void* ws, size_t ws_bytes,
                                       tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0 && rows < (1ll << 31) - 1 && n < (1ll << 31));
  TFS_REQUIRE((table2 == nullptr) == (grad2 == nullptr));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && ids && grad_rows);
  TFS_REQUIRE(dim % 4 != 0 || (((uintptr_t)table | (uintptr_t)grad_rows) & 15) == 0);
  TFS_SUPPORTED();
  SegScratch s;
  if (ws_bytes < seg_scratch_bytes(n, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  int32_t rc = sort_and_segment(ids, n, rows, 1, rows + 1, 0, (uint32_t)rows, s, err, st);
  if (rc != TFS_OK) return rc;
  SegJob j{};
  j.keys = s.k1; j.perm = s.v1; j.seg_start = s.seg_start; j.num_unique = s.num_unique;
  j.rows = grad_rows; j.rows2 = grad2; j.dim = dim; j.invalid_key = (uint32_t)rows;
  j.table = table; j.table2 = table2; j.lr = lr;
  j.nloc = rows + 1; j.long_list = s.long_list; j.long_count = s.long_count;
  return run_segments(j, n, st);
}

extern "C" size_t tfs_sort_reduce_workspace_bytes(int64_t n, int32_t dim) {
  (void)dim;
  return seg_scratch_bytes(n, nullptr, nullptr, 0);
}

extern "C" int32_t tfs_sort_reduce(const int64_t* ids, int64_t n, int64_t vocab,
                                   int32_t num_shards, const float* rows, int32_t dim,
                                   const float* rows2, int64_t* out_local, float* out_rows,
                                   float* out_rows2, int64_t* out_counts, int64_t* out_num_unique,
                                   void* ws, size_t ws_bytes, tfs_device_error* err,
                                   void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && vocab >= 1 && num_shards >= 1 && num_shards <= 1024);
  TFS_REQUIRE(n < (1ll << 31) && vocab + num_shards < (1ll << 32) - 1);
  TFS_REQUIRE(out_counts && out_num_unique);
  TFS_REQUIRE((rows2 == nullptr) == (out_rows2 == nullptr));
  TFS_SUPPORTED();
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    TFS_CUDA_TRY(cudaMemsetAsync(out_counts, 0, sizeof(int64_t) * num_shards, st));
    TFS_CUDA_TRY(cudaMemsetAsync(out_num_unique, 0, sizeof(int64_t), st));
    return TFS_OK;
  }
  TFS_REQUIRE(ids && rows && out_local && out_rows);
  SegScratch s;
  if (ws_bytes < seg_scratch_bytes(n, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int64_t nloc = cdiv(vocab, num_shards);
  const uint32_t invalid = (uint32_t)(num_shards * nloc);
  int32_t rc = sort_and_segment(ids, n, vocab, num_shards, nloc, 1, invalid, s, err, st);
  if (rc != TFS_OK) return rc;
  SegJob j{};
  j.keys = s.k1; j.perm = s.v1; j.seg_start = s.seg_start; j.num_unique = s.num_unique;
  j.rows = rows; j.rows2 = rows2; j.dim = dim; j.invalid_key = invalid;
  j.out_local = out_local; j.out_rows = out_rows; j.out_rows2 = out_rows2; j.nloc = nloc;
  j.long_list = s.long_list; j.long_count = s.long_count;
  rc = run_segments(j, n, st);
  if (rc != TFS_OK) return rc;
  owner_counts_kernel<<<1, 1024, 0, st>>>(s.k1, s.seg_start, s.num_unique, num_shards, nloc,
                                          invalid, out_counts);
  TFS_LAUNCH_CHECK();
  // (With bad ids, U also counts their sentinel segment; outputs are unspecified then.)
  TFS_CUDA_TRY(cudaMemcpyAsync(out_num_unique, s.num_unique, sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, st));
  return TFS_OK;
}
