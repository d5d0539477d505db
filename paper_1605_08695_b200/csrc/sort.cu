// sort.cu -- Part, the stable digit-sort engine it shares with the LSD radix sort,
// and the deterministic sort-by-id segmented reductions behind the sparse gradient path:
// tfs_sort_reduce (gradient rows summed per id before routing) and
// tfs_scatter_add_sgd (ScatterAdd/SGD "-=" on the owner shard).
//
// Design: latency/HBM-bound integer work.  A tile of 1024 items per 256-thread
// CTA; per-tile digit histograms; every CTA computes its own global offsets from the (small)
// histogram table, so a pass is two launches with no separate scan.  Within a tile the rank
// of an item among equal digits comes from warp __match_any_sync + popc and a per-round
// warp-order prefix, which makes the scatter stable (original order kept: R-2).
//
// Segmented sums over the id-sorted rows use a FIXED reduction structure (R-16): the sorted
// array is cut into 16-row chunks (one warp each, all row addresses known up front, so the row
// loads are issued back to back); inside a chunk a segment's rows are added in sorted order in
// fp64; a segment that crosses chunk boundaries is finished by adding its per-chunk partials in
// chunk order.  The structure depends only on the segment lengths, so results are
// run-to-run bit-identical, and fp64 keeps thousand-way Zipf duplicates inside the fp32 bound.
#include <algorithm>

#include "common.cuh"

namespace tfs {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 4;
constexpr int kSortTile = kSortThreads * kSortItems;  // 1024 items per CTA
constexpr int kMaxBuckets = 256;
constexpr int kChunk = 16;  // sorted rows per warp in the segmented sums

struct DigitSrc {
  int mode;
  const int64_t* ids;
  const int32_t* assign;
  int64_t vocab;
  int32_t nshards;
  const uint32_t* keys;
  const uint32_t* vals;
  int shift;
  int nbuckets;
};

// One input element: its bucket plus what the sink needs to write it out.
struct Item {
  int digit;
  int64_t a;   // partition: id;  radix: key
  uint32_t b;  // radix: value
};

__device__ __forceinline__ Item load_item(const DigitSrc& s, int64_t i, tfs_device_error* err) {
  Item it;
  if (s.mode == kDigitRadix) {
    const uint32_t k = s.keys[i];
    it.a = k;
    it.b = s.vals ? s.vals[i] : (uint32_t)i;
    it.digit = (int)((k >> s.shift) & 0xffu);
    return it;
  }
  const int64_t id = s.ids[i];
  it.a = id;
  it.b = 0;
  if (s.mode == kDigitMod) {
    if (id < 0 || id >= s.vocab) {
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      it.digit = 0;
    } else {
      it.digit = (int)(id % s.nshards);
    }
  } else {
    const int32_t a = s.assign[i];
    if (a < 0 || a >= s.nshards) {
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      it.digit = 0;
    } else {
      it.digit = a;
    }
  }
  return it;
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
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  int dg[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {  // all loads first
    const int64_t i = base + (int64_t)j * kSortThreads + threadIdx.x;
    dg[j] = i < n ? load_item(src, i, err).digit : -1;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kSortItems; ++j)
    if (dg[j] >= 0) atomicAdd(&cnt[dg[j]], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kSortThreads) hist[(int64_t)b * ntiles + blockIdx.x] = cnt[b];
}

struct PartSink {  // tfs_partition outputs
  int64_t* local;
  int64_t* positions;
  __device__ void put(const DigitSrc& s, uint32_t pos, int64_t i, const Item& it) const {
    local[pos] = s.mode == kDigitMod ? it.a / s.nshards : it.a;
    positions[pos] = i;
  }
};

struct RadixSink {  // one LSD pass
  uint32_t* keys_out;
  uint32_t* vals_out;
  __device__ void put(const DigitSrc&, uint32_t pos, int64_t, const Item& it) const {
    keys_out[pos] = (uint32_t)it.a;
    vals_out[pos] = it.b;
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
  const int tid = threadIdx.x, warp = tid >> 5;
  const int tile = blockIdx.x;
  const int64_t base = (int64_t)tile * kSortTile;

  // Issue every global load up front: this tile's items and this bucket's histogram column.
  Item it[kSortItems];
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + (int64_t)j * kSortThreads + tid;
    if (i < n)
      it[j] = load_item(src, i, nullptr);
    else
      it[j].digit = -1;
  }
  uint32_t tot = 0, pre = 0;
  if (tid < nb) {
    const uint32_t* h = hist + (int64_t)tid * ntiles;
    for (int t = 0; t < ntiles; ++t) {
      const uint32_t c = h[t];
      tot += c;
      if (t < tile) pre += c;
    }
  }
  // Global base of every bucket for this tile: all earlier buckets + this bucket in earlier tiles.
  const uint32_t excl = block_exclusive_scan(tid < nb ? tot : 0u, nullptr);
  if (tid < nb) {
    running[tid] = excl + pre;
    if (counts_out != nullptr && tile == 0) counts_out[tid] = (int64_t)tot;
  }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int dg = it[j].digit;
    for (int b = tid; b < kSortWarps * nb; b += kSortThreads) wcnt[b / nb][b % nb] = 0;
    __syncthreads();
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    const uint32_t rank = __popc(peers & lanemask_lt());
    if (dg >= 0 && rank == 0) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    if (tid < nb) {
      uint32_t p = running[tid];
#pragma unroll
      for (int w = 0; w < kSortWarps; ++w) {
        const uint32_t c = wcnt[w][tid];
        wcnt[w][tid] = p;
        p += c;
      }
      running[tid] = p;
    }
    __syncthreads();
    if (dg >= 0) sink.put(src, wcnt[warp][dg] + rank, base + (int64_t)j * kSortThreads + tid, it[j]);
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
    DigitSrc s{kDigitRadix, nullptr, nullptr, 0, 0, ksrc, vsrc, 8 * p, 256};
    digit_hist_kernel<<<ntiles, kSortThreads, 0, st>>>(s, n, hist, ntiles, nullptr);
    launched();
    digit_scatter_kernel<RadixSink><<<ntiles, kSortThreads, 0, st>>>(
        s, n, hist, ntiles, RadixSink{kd, vd}, nullptr);
    launched();
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
             nullptr, nullptr, 0, num_shards};
  digit_hist_kernel<<<ntiles, kSortThreads, 0, st>>>(s, n, hist, ntiles, err);
  launched();
  digit_scatter_kernel<PartSink><<<ntiles, kSortThreads, 0, st>>>(
      s, n, hist, ntiles, PartSink{out_local, out_positions}, out_counts);
  launched();
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

// keys for ScatterAdd: key = id (invalid -> sentinel `limit`); for sort_reduce: key =
// owner * nloc + local (invalid -> R * nloc).  Invalid keys sort last and are skipped.
__global__ void make_keys_kernel(const int64_t* ids, int64_t n, int64_t limit, int32_t R,
                                 int64_t nloc, int composite, uint32_t* keys, uint32_t* vals,
                                 tfs_device_error* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = ids[i];
    uint32_t key;
    if (id < 0 || id >= limit) {
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
      key = composite ? (uint32_t)(R * nloc) : (uint32_t)limit;
    } else {
      key = composite ? (uint32_t)((id % R) * nloc + id / R) : (uint32_t)id;
    }
    keys[i] = key;
    vals[i] = (uint32_t)i;
  }
}

// Segment heads of a sorted key array: per-tile head counts, then per-tile starts and the
// segment index of every sorted position.
__global__ void __launch_bounds__(kSortThreads) heads_count_kernel(const uint32_t* k, int64_t n,
                                                                   uint32_t* tile_cnt) {
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)threadIdx.x * kSortItems;
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + j;
    if (i < n && (i == 0 || k[i] != k[i - 1])) ++c;
  }
  uint32_t total;
  block_exclusive_scan(c, &total);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kSortThreads) heads_write_kernel(
    const uint32_t* k, int64_t n, const uint32_t* tile_cnt, int ntiles, uint32_t* seg_start,
    uint32_t* seg_of, int64_t* num_unique) {
  __shared__ uint32_t tile_base;
  if (threadIdx.x < 32) {
    uint32_t pre = 0, all = 0;
    for (int t = threadIdx.x; t < ntiles; t += 32) {
      const uint32_t c = tile_cnt[t];
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
  const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)threadIdx.x * kSortItems;
  bool head[kSortItems];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + j;
    head[j] = i < n && (i == 0 || k[i] != k[i - 1]);
    c += head[j];
  }
  __syncthreads();
  uint32_t pos = tile_base + block_exclusive_scan(c, nullptr);
#pragma unroll
  for (int j = 0; j < kSortItems; ++j) {
    const int64_t i = base + j;
    if (i >= n) break;
    if (head[j]) seg_start[pos++] = (uint32_t)i;
    seg_of[i] = pos - 1;
  }
}

struct SegJob {
  const uint32_t* keys;       // sorted keys
  const uint32_t* perm;       // original index of each sorted position
  const uint32_t* seg_start;  // [U + 1]
  const uint32_t* seg_of;     // [n] segment of each sorted position
  const int64_t* num_unique;  // device U
  int64_t n;
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
  // partials of segments crossing chunk boundaries: slot 2c = the piece in chunk c of the
  // segment that started before chunk c; slot 2c+1 = the piece of the segment that starts in
  // chunk c and continues after it.
  double* part;   // [2 * nchunks x dim]
  double* part2;  // [2 * nchunks]
};

struct D4 {
  double x, y, z, w;
};

__device__ __forceinline__ void add4(D4& a, const float4& v) {
  a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
}

// ScatterAdd-SGD: T = fl32(T - lr * g) evaluated in fp64; sort_reduce: out = fl32(g).
__device__ __forceinline__ void emit4(const SegJob& j, uint32_t s, uint32_t key, int c4,
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

__device__ __forceinline__ void emit1(const SegJob& j, uint32_t s, uint32_t key, int c, double v) {
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

// Where the piece of segment s that lives in chunk `chunk` goes: -1 = it is the whole segment
// (emit now), else the partial slot index.
__device__ __forceinline__ int64_t piece_slot(const SegJob& j, uint32_t s, int64_t chunk) {
  const int64_t c0 = (int64_t)j.seg_start[s] / kChunk;
  const int64_t c1 = ((int64_t)j.seg_start[s + 1] - 1) / kChunk;
  if (c0 == c1) return -1;
  return chunk == c0 ? 2 * chunk + 1 : 2 * chunk;
}

// One warp per chunk of kChunk sorted rows, float4 columns (dim % 4 == 0).
__global__ void __launch_bounds__(256) seg_chunk_vec4_kernel(SegJob j) {
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t base = chunk * kChunk;
  if (base >= j.n) return;
  const int cnt = (int)min((int64_t)kChunk, j.n - base);
  uint32_t perm_l = 0, seg_l = 0;
  float r2_l = 0.f;
  if (lane < cnt) {
    perm_l = j.perm[base + lane];
    seg_l = j.seg_of[base + lane];
    if (j.rows2) r2_l = j.rows2[perm_l];
  }
  const int n4 = j.dim >> 2;
  for (int c4_0 = 0; c4_0 < n4; c4_0 += 128) {
    D4 acc[4];
    double acc2 = 0.0;
    uint32_t cur = __shfl_sync(0xffffffffu, seg_l, 0);
    auto flush = [&](uint32_t s) {
      const uint32_t key = j.keys[j.seg_start[s]];
      if (key >= j.invalid_key) return;
      const int64_t slot = piece_slot(j, s, chunk);
      if (slot < 0) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c4 = c4_0 + v * 32 + lane;
          if (c4 < n4) emit4(j, s, key, c4, acc[v]);
        }
        if (j.rows2 && lane == 0 && c4_0 == 0) emit_companion(j, s, key, acc2);
      } else {
        double* p = j.part + slot * j.dim;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c4 = c4_0 + v * 32 + lane;
          if (c4 < n4) {
            p[4 * c4 + 0] = acc[v].x;
            p[4 * c4 + 1] = acc[v].y;
            p[4 * c4 + 2] = acc[v].z;
            p[4 * c4 + 3] = acc[v].w;
          }
        }
        if (j.rows2 && lane == 0 && c4_0 == 0) j.part2[slot] = acc2;
      }
    };
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[v] = D4{0.0, 0.0, 0.0, 0.0};
    for (int r0 = 0; r0 < cnt; r0 += 4) {
      float4 x[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // four rows' loads in flight
        const uint32_t pr = __shfl_sync(0xffffffffu, perm_l, r0 + u);
        const float4* row = (const float4*)(j.rows + (int64_t)pr * j.dim);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c4 = c4_0 + v * 32 + lane;
          x[u][v] = (r0 + u < cnt && c4 < n4) ? __ldg(row + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (r0 + u >= cnt) break;
        const uint32_t s = __shfl_sync(0xffffffffu, seg_l, r0 + u);
        const float r2 = __shfl_sync(0xffffffffu, r2_l, r0 + u);
        if (s != cur) {
          flush(cur);
          cur = s;
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[v] = D4{0.0, 0.0, 0.0, 0.0};
          acc2 = 0.0;
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) add4(acc[v], x[u][v]);
        acc2 += r2;
      }
    }
    flush(cur);
  }
}

// Scalar columns (any dim): same structure, one column per lane per 32-column block.
__global__ void __launch_bounds__(256) seg_chunk_scalar_kernel(SegJob j) {
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t base = chunk * kChunk;
  if (base >= j.n) return;
  const int cnt = (int)min((int64_t)kChunk, j.n - base);
  uint32_t perm_l = 0, seg_l = 0;
  float r2_l = 0.f;
  if (lane < cnt) {
    perm_l = j.perm[base + lane];
    seg_l = j.seg_of[base + lane];
    if (j.rows2) r2_l = j.rows2[perm_l];
  }
  for (int c0 = 0; c0 < j.dim; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0, acc2 = 0.0;
    uint32_t cur = __shfl_sync(0xffffffffu, seg_l, 0);
    auto flush = [&](uint32_t s) {
      const uint32_t key = j.keys[j.seg_start[s]];
      if (key >= j.invalid_key) return;
      const int64_t slot = piece_slot(j, s, chunk);
      if (slot < 0) {
        if (c < j.dim) emit1(j, s, key, c, acc);
        if (j.rows2 && lane == 0 && c0 == 0) emit_companion(j, s, key, acc2);
      } else {
        if (c < j.dim) j.part[slot * j.dim + c] = acc;
        if (j.rows2 && lane == 0 && c0 == 0) j.part2[slot] = acc2;
      }
    };
    for (int r = 0; r < cnt; ++r) {
      const uint32_t pr = __shfl_sync(0xffffffffu, perm_l, r);
      const uint32_t s = __shfl_sync(0xffffffffu, seg_l, r);
      const float r2 = __shfl_sync(0xffffffffu, r2_l, r);
      const float xv = c < j.dim ? j.rows[(int64_t)pr * j.dim + c] : 0.f;
      if (s != cur) {
        flush(cur);
        cur = s;
        acc = 0.0;
        acc2 = 0.0;
      }
      acc += xv;
      acc2 += r2;
    }
    flush(cur);
  }
}

// One warp per segment: out_local, and the chunk-order sum of the partials of segments that
// cross chunk boundaries.
__global__ void __launch_bounds__(256) seg_cross_kernel(SegJob j) {
  const int lane = threadIdx.x & 31;
  const int64_t U = *j.num_unique;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t s = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); s < U; s += warps) {
    const uint32_t a = j.seg_start[s], b = j.seg_start[s + 1];
    const uint32_t key = j.keys[a];
    if (key >= j.invalid_key) continue;
    if (j.out_local && lane == 0) j.out_local[s] = (int64_t)(key % (uint32_t)j.nloc);
    const int64_t c0 = a / kChunk, c1 = (b - 1) / kChunk;
    if (c0 == c1) continue;
    for (int c = lane; c < j.dim; c += 32) {
      double acc = j.part[(2 * c0 + 1) * j.dim + c];
      for (int64_t ch = c0 + 1; ch <= c1; ++ch) acc += j.part[(2 * ch) * j.dim + c];
      emit1(j, (uint32_t)s, key, c, acc);
    }
    if (j.rows2 && lane == 0) {
      double acc = j.part2[2 * c0 + 1];
      for (int64_t ch = c0 + 1; ch <= c1; ++ch) acc += j.part2[2 * ch];
      emit_companion(j, (uint32_t)s, key, acc);
    }
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
      const int64_t mid = (lo + hi) / 2;
      const uint32_t k = keys[seg_start[mid]];
      const int64_t ow = k >= invalid_key ? R : (int64_t)(k / (uint32_t)nloc);
      if (ow < owner) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  counts[o] = first_ge(o + 1) - first_ge(o);
}

struct SegScratch {
  uint32_t *k0, *v0, *k1, *v1, *seg_start, *seg_of, *tile_cnt;
  double *part, *part2;
  int64_t* num_unique;
  void* sort_ws;
  size_t sort_ws_bytes;
};

static size_t seg_scratch_bytes(int64_t n, int32_t dim, SegScratch* s, void* ws, size_t cap) {
  Carver c(ws, cap);
  const int64_t ntiles = cdiv(n, kSortTile);
  const int64_t nchunks = cdiv(n, kChunk);
  SegScratch x;
  x.k0 = c.take<uint32_t>(n);
  x.v0 = c.take<uint32_t>(n);
  x.k1 = c.take<uint32_t>(n);
  x.v1 = c.take<uint32_t>(n);
  x.seg_start = c.take<uint32_t>(n + 1);
  x.seg_of = c.take<uint32_t>(n);
  x.tile_cnt = c.take<uint32_t>(ntiles + 1);
  x.part = c.take<double>((size_t)2 * nchunks * dim);
  x.part2 = c.take<double>((size_t)2 * nchunks);
  x.num_unique = c.take<int64_t>(1);
  x.sort_ws_bytes = radix_sort_ws_bytes(n);
  x.sort_ws = c.take<char>(x.sort_ws_bytes);
  if (s) *s = x;
  return c.used + 256;
}

static int32_t sort_and_segment(const int64_t* ids, int64_t n, int64_t limit, int32_t R,
                                int64_t nloc, int composite, uint32_t key_max, SegScratch& s,
                                tfs_device_error* err, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>(cdiv(n, 256), 4 * num_sms());
  make_keys_kernel<<<grid, 256, 0, st>>>(ids, n, limit, R, nloc, composite, s.k0, s.v0, err);
  launched();
  TFS_LAUNCH_CHECK();
  int32_t rc = radix_sort_pairs(s.k0, s.v0, s.k1, s.v1, n, bits_for(key_max), s.sort_ws,
                                s.sort_ws_bytes, st);
  if (rc != TFS_OK) return rc;
  const int ntiles = (int)cdiv(n, kSortTile);
  heads_count_kernel<<<ntiles, kSortThreads, 0, st>>>(s.k1, n, s.tile_cnt);
  launched();
  heads_write_kernel<<<ntiles, kSortThreads, 0, st>>>(s.k1, n, s.tile_cnt, ntiles, s.seg_start,
                                                      s.seg_of, s.num_unique);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

static void bind(SegJob& j, const SegScratch& s, int64_t n) {
  j.keys = s.k1;
  j.perm = s.v1;
  j.seg_start = s.seg_start;
  j.seg_of = s.seg_of;
  j.num_unique = s.num_unique;
  j.n = n;
  j.part = s.part;
  j.part2 = s.part2;
}

static int32_t run_segments(SegJob& j, int64_t n, cudaStream_t st) {
  const int64_t nchunks = cdiv(n, kChunk);
  const int grid = (int)std::max<int64_t>(1, cdiv(nchunks, 8));
  if ((j.dim & 3) == 0 && ((uintptr_t)j.rows & 15) == 0)
    seg_chunk_vec4_kernel<<<grid, 256, 0, st>>>(j);
  else
    seg_chunk_scalar_kernel<<<grid, 256, 0, st>>>(j);
  launched();
  const int cgrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 8 * num_sms()));
  seg_cross_kernel<<<cgrid, 256, 0, st>>>(j);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

}  // namespace tfs

// ================================================================================================
extern "C" size_t tfs_scatter_add_sgd_workspace_bytes(int64_t n, int32_t dim) {
  return seg_scratch_bytes(n, dim, nullptr, nullptr, 0);
}

extern "C" int32_t tfs_scatter_add_sgd(float* table, int64_t rows, int32_t dim, const int64_t* ids,
                                       const float* grad_rows, int64_t n, float lr, float* table2,
                                       const float* grad2, void* ws, size_t ws_bytes,
                                       tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0 && rows < (1ll << 31) - 1 && n < (1ll << 31));
  TFS_REQUIRE((table2 == nullptr) == (grad2 == nullptr));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && ids && grad_rows);
  TFS_REQUIRE(dim % 4 != 0 || ((uintptr_t)table & 15) == 0);
  TFS_SUPPORTED();
  SegScratch s;
  if (ws_bytes < seg_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  int32_t rc = sort_and_segment(ids, n, rows, 1, rows + 1, 0, (uint32_t)rows, s, err, st);
  if (rc != TFS_OK) return rc;
  SegJob j{};
  bind(j, s, n);
  j.rows = grad_rows;
  j.rows2 = grad2;
  j.dim = dim;
  j.invalid_key = (uint32_t)rows;
  j.table = table;
  j.table2 = table2;
  j.lr = lr;
  j.nloc = rows + 1;
  return run_segments(j, n, st);
}

extern "C" size_t tfs_sort_reduce_workspace_bytes(int64_t n, int32_t dim) {
  return seg_scratch_bytes(n, dim, nullptr, nullptr, 0);
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
  TFS_REQUIRE(dim % 4 != 0 || ((uintptr_t)out_rows & 15) == 0);
  SegScratch s;
  if (ws_bytes < seg_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int64_t nloc = cdiv(vocab, num_shards);
  const uint32_t invalid = (uint32_t)(num_shards * nloc);
  int32_t rc = sort_and_segment(ids, n, vocab, num_shards, nloc, 1, invalid, s, err, st);
  if (rc != TFS_OK) return rc;
  SegJob j{};
  bind(j, s, n);
  j.rows = rows;
  j.rows2 = rows2;
  j.dim = dim;
  j.invalid_key = invalid;
  j.out_local = out_local;
  j.out_rows = out_rows;
  j.out_rows2 = out_rows2;
  j.nloc = nloc;
  rc = run_segments(j, n, st);
  if (rc != TFS_OK) return rc;
  owner_counts_kernel<<<1, 1024, 0, st>>>(s.k1, s.seg_start, s.num_unique, num_shards, nloc,
                                          invalid, out_counts);
  launched();
  TFS_LAUNCH_CHECK();
  // (With bad ids, U also counts their sentinel segment; outputs are unspecified then.)
  TFS_CUDA_TRY(cudaMemcpyAsync(out_num_unique, s.num_unique, sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, st));
  return TFS_OK;
}
