// sort.cu -- Part, the stable digit-sort engine it shares with the LSD radix sort,
// and the deterministic sort-by-id segmented reductions behind the sparse gradient path:
// tfs_sort_reduce (gradient rows summed per id before routing) and
// tfs_scatter_add_sgd (ScatterAdd/SGD "-=" on the owner shard).
//
// Design: latency/HBM-bound integer work.  A tile of 1024 items per 256-thread
// CTA; per-tile digit histograms; every CTA computes its own global offsets from the (small)
// histogram table, so a pass is two launches with no separate scan.  Within a tile the rank
// of an item among equal digits comes from an 8-ballot warp digit match + popc and a per-round
// warp-order prefix, which makes the scatter stable (original order kept: R-2).
//
// Segmented sums over the id-sorted rows use a FIXED reduction structure (R-16): the sorted
// array is cut into windows of 8 (short inputs) or 32 rows, one CTA each (thread = float4
// column; warp 0 builds the window's row program in shared memory); inside a window a
// segment's rows are added in sorted order in fp64; a segment that crosses window edges leaves
// one partial per window, and the last arriver of each block of 16 windows, then of the blocks,
// adds them in window / block order -- in the same launch.  The structure depends only on the
// segment lengths, so results are run-to-run bit-identical, and fp64 keeps thousand-way Zipf
// duplicates inside the fp32 bound.
#include <algorithm>

#include "common.cuh"

namespace tfs {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortItems = 4;
constexpr int kSortTile = kSortThreads * kSortItems;  // 1024 items per CTA
constexpr int kMaxBuckets = 256;
// Sorted rows per window of the segmented sums: 32 for long inputs, 8 for short ones (more
// windows in flight); scratch is sized for the smallest.
#ifndef TFS_SEG_CHUNK
#define TFS_SEG_CHUNK 32
#endif
constexpr int kChunk = TFS_SEG_CHUNK;
#ifndef TFS_SEG_CHUNK_MIN
#define TFS_SEG_CHUNK_MIN 8
#endif
constexpr int kChunkMin = TFS_SEG_CHUNK_MIN;
#ifndef TFS_SEG_SHORT_N
#define TFS_SEG_SHORT_N 40000  // below this many rows: 8-row windows
#endif


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

// Lanes holding the same 8-bit digit as this lane (valid lanes only): 8 ballots, one per digit
// bit -- much cheaper than a general match on this part.
__device__ __forceinline__ uint32_t match_digit8(int dg, bool valid) {
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  uint32_t peers = valid ? vmask : 0u;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const bool bit = (dg >> b) & 1;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__global__ void __launch_bounds__(kSortThreads) digit_hist_kernel(DigitSrc src, int64_t n,
                                                                  uint32_t* hist, int ntiles,
                                                                  tfs_device_error* err) {
  pdl_enter();
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
  pdl_enter();
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
    const uint32_t peers = match_digit8(dg & 0xff, dg >= 0);
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
    ::tfs::launch(digit_hist_kernel, ntiles, kSortThreads, 0, st, s, n, hist, ntiles, nullptr);
    launched();
    ::tfs::launch(digit_scatter_kernel<RadixSink>, ntiles, kSortThreads, 0, st, 
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
// One shard: the stable partition is the identity (local = id, position = i, count = n); only
// the id range check remains.
__global__ void partition_one_kernel(const int64_t* ids, int64_t n, int64_t vocab,
                                     int64_t* local, int64_t* positions, int64_t* counts,
                                     tfs_device_error* err) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = ids[i];
    if (id < 0 || id >= vocab) report_error(err, TFS_ERR_OUT_OF_RANGE, i);
    local[i] = id;
    positions[i] = i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[0] = n;
}

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
  if (num_shards == 1 && assignments == nullptr) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4ll * num_sms()));
    ::tfs::launch(partition_one_kernel, grid, 256, 0, st, ids, n, vocab, out_local, out_positions,
                                               out_counts, err);
    launched();
    TFS_LAUNCH_CHECK();
    return TFS_OK;
  }
  if (ws_bytes < tfs_partition_workspace_bytes(n, num_shards)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int ntiles = (int)cdiv(n, kSortTile);
  uint32_t* hist = (uint32_t*)ws;
  DigitSrc s{assignments ? kDigitAssign : kDigitMod, ids, assignments, vocab, num_shards,
             nullptr, nullptr, 0, num_shards};
  ::tfs::launch(digit_hist_kernel, ntiles, kSortThreads, 0, st, s, n, hist, ntiles, err);
  launched();
  ::tfs::launch(digit_scatter_kernel<PartSink>, ntiles, kSortThreads, 0, st, 
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

// Ids read densely (cap == 0) or from a slot layout: id i = slot (i / cap, i % cap) at
// p[o * stride + s].
struct IdsView {
  const int64_t* p;
  int64_t cap, stride;
};
__device__ __forceinline__ int64_t load_id(const IdsView& v, int64_t i) {
  if (v.cap == 0) return v.p[i];
  const int64_t o = i / v.cap;
  return v.p[o * v.stride + (i - o * v.cap)];
}

// keys for ScatterAdd: key = id (invalid -> sentinel `limit`); for sort_reduce: key =
// owner * nloc + local (invalid -> R * nloc).  Invalid keys sort last and are skipped.
__global__ void make_keys_kernel(IdsView ids, int64_t n, int64_t limit, int32_t R,
                                 int64_t nloc, int composite, uint32_t* keys, uint32_t* vals,
                                 tfs_device_error* err) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = load_id(ids, i);
    uint32_t key;
    if (id < 0 || id >= limit) {
      if (id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, i);  // -1: padding, skipped
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
  pdl_enter();
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
  pdl_enter();
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
  // apply mode (ScatterAdd-SGD): table[key] -= lr * sum; or sparse Momentum / Adagrad with the
  // fp32 slot tables slot / slot2 (opt 1 / 2, reading R-29)
  float* table;
  float* table2;
  float lr;
  int opt;
  double mu;
  float* slot;
  float* slot2;
  uint16_t* mirror;  // optional bf16 copy of the table, kept in step (tfs_sparse_opt.mirror)
  // write mode (sort_reduce): out_local[u], out_rows[u]; with slot_base (route_reduce) the row
  // of segment u (owner o = key / nloc) goes to slot o * cap + (u - slot_base[o]) instead
  int64_t* out_local;
  float* out_rows;
  float* out_rows2;
  const int64_t* slot_base;
  int64_t cap;
  int64_t out_stride, out2_stride;  // per-owner slot region strides of out_rows / out_rows2
  float* const* out_tab;            // or per-owner region bases (+ out_off / out2_off)
  float* const* out2_tab;
  int64_t out_off, out2_off;
  // input rows in slot layout (row_cap > 0): row i = slot (i / row_cap, i % row_cap) at
  // rows + o * row_stride + s * dim (rows2 + o * row2_stride + s)
  int64_t row_cap, row_stride, row2_stride;
  int64_t nloc;
  int32_t chunk;  // rows per window (kChunk or kChunkMin)
  // apply mode: sums of the segments that lie inside one chunk, [U x dim] (+ [U])
  float* sums;
  float* sums2;
  // partials of segments crossing chunk boundaries: slot 2c = the piece in chunk c of the
  // segment that started before chunk c; slot 2c+1 = the piece of the segment that starts in
  // chunk c and continues after it.
  double* part;   // [2 * nchunks x dim]
  double* part2;  // [2 * nchunks]
  // Second level for segments that cross chunk boundaries: chunk_info[c] = (segment of the
  // piece in slot 2c, segment of the piece in slot 2c+1), -1 where absent; the crossing
  // segments are listed in cross_list (order irrelevant).
  int2* chunk_info;
  uint32_t* cross_list;
  uint32_t* cross_count;
  // Fused crossing reduction (vec path): arrival counters, zero between calls (the last
  // arriver resets them): per partial slot (the level-1 run of a segment inside a block of
  // kRunWin windows is keyed by its first slot) and per segment (level 2).
  uint32_t* win_cnt;
  uint32_t* seg_cnt;
};

struct D4 {
  double x, y, z, w;
};

// Where segment u's results go in write mode: float offset of its row in out_rows, offset in
// out_rows2, index in out_local.  row < 0: dropped (slot capacity exceeded).
struct OutPos {
  float* row;     // nullptr: dropped
  float* r2;      // nullptr when there is no companion stream
  int64_t local;  // index into out_local
};
__device__ __forceinline__ OutPos seg_out_pos(const SegJob& j, int64_t u, uint32_t key) {
  if (j.slot_base == nullptr)
    return OutPos{j.out_rows + u * j.dim, j.out_rows2 ? j.out_rows2 + u : nullptr, u};
  const int64_t o = key / (uint32_t)j.nloc;
  const int64_t s = u - j.slot_base[o];
  if (s >= j.cap) return OutPos{nullptr, nullptr, -1};
  if (j.out_tab != nullptr)  // owner o's inbox, written over NVLink
    return OutPos{j.out_tab[o] + j.out_off + s * j.dim,
                  j.out2_tab ? j.out2_tab[o] + j.out2_off + s : nullptr, -1};
  return OutPos{j.out_rows + o * j.out_stride + s * j.dim,
                j.out_rows2 ? j.out_rows2 + o * j.out2_stride + s : nullptr, -1};
}
// Float offset of input row i (and of its rows2 value).
__device__ __forceinline__ int64_t row_off(const SegJob& j, uint32_t i) {
  if (j.row_cap == 0) return (int64_t)i * j.dim;
  const int64_t o = i / j.row_cap;
  return o * j.row_stride + ((int64_t)i - o * j.row_cap) * j.dim;
}
__device__ __forceinline__ int64_t row2_off(const SegJob& j, uint32_t i) {
  if (j.row_cap == 0) return i;
  const int64_t o = i / j.row_cap;
  return o * j.row2_stride + ((int64_t)i - o * j.row_cap);
}

__device__ __forceinline__ void add4(D4& a, const float4& v) {
  a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
}
__device__ __forceinline__ void add4(D4& a, const D4& v) {
  a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
}
__device__ __forceinline__ float4 to_f4(const D4& v) {
  return make_float4((float)v.x, (float)v.y, (float)v.z, (float)v.w);
}

// One optimizer step of an fp32 element given the fp64 sum g of its gradients (R-29); s is the
// element's slot value (updated; unused for SGD).
template <int OPT>
__device__ __forceinline__ float opt_step(const SegJob& j, float w, double g, float& s) {
  const double lr = (double)j.lr;
  if (OPT == 1) {
    s = (float)(j.mu * (double)s + g);
    return (float)((double)w - lr * (double)s);
  }
  if (OPT == 2) {
    s = (float)((double)s + g * g);
    return (float)((double)w - lr * g / sqrt((double)s));
  }
  return (float)((double)w - lr * g);
}
// The step on four columns of row `key` (slot row at the same offset as the table row).
template <int OPT>
__device__ __forceinline__ float4 opt_step4(const SegJob& j, float4 w, const D4& g, int64_t key,
                                            int c4) {
  if (OPT == 0) {
    float dummy = 0.f;
    return make_float4(opt_step<0>(j, w.x, g.x, dummy), opt_step<0>(j, w.y, g.y, dummy),
                       opt_step<0>(j, w.z, g.z, dummy), opt_step<0>(j, w.w, g.w, dummy));
  }
  float4* sp = reinterpret_cast<float4*>(j.slot + key * j.dim) + c4;
  float4 sv = *sp;
  w = make_float4(opt_step<OPT>(j, w.x, g.x, sv.x), opt_step<OPT>(j, w.y, g.y, sv.y),
                  opt_step<OPT>(j, w.z, g.z, sv.z), opt_step<OPT>(j, w.w, g.w, sv.w));
  *sp = sv;
  return w;
}
// The companion (width-1) table's step with its slot2.
template <int OPT>
__device__ __forceinline__ void opt_step2(const SegJob& j, int64_t key, double g2) {
  float s = OPT ? j.slot2[key] : 0.f;
  j.table2[key] = opt_step<OPT>(j, j.table2[key], g2, s);
  if (OPT) j.slot2[key] = s;
}

// Where a finished piece of one segment goes (warp-uniform decision).
struct PieceDst {
  int kind;  // 0 whole segment, 1 head slot (started before the chunk), 2 tail slot
  int64_t slot;
};
__device__ __forceinline__ PieceDst piece_dst(bool starts_before, bool ends_after, int64_t chunk) {
  if (starts_before) return PieceDst{1, 2 * chunk};
  if (ends_after) return PieceDst{2, 2 * chunk + 1};
  return PieceDst{0, 0};
}

// One CTA per window of kChunk sorted rows, all columns (thread = one float4 column group,
// looping when dim / 4 exceeds the CTA).  The window's segment structure (heads, ends, whole
// segments, crossings) is computed once by warp 0 and is uniform across the CTA, so the column
// threads run branch-uniform: every row of a batch of 8 -- and the table row of every whole
// segment ending in the batch -- is loaded at once, each segment's rows are added in sorted
// order in fp64, and a whole segment is applied (T = fl32(T - lr g), or Momentum / Adagrad) or
// written; pieces of segments crossing the window's edges go to the partial slots (2c: the
// piece of the segment that started before window c; 2c + 1: the piece of the segment that
// starts in c and continues after it) and the segment to cross_list.
#ifndef TFS_WIN_BATCH
#define TFS_WIN_BATCH 8
#endif
constexpr int kWinBatch = TFS_WIN_BATCH;  // rows per two pipelined half-batches
constexpr int kRunWin = 16;  // windows per level-1 block of a crossing segment

template <int OPT, bool WR>
__device__ __forceinline__ void seg_finish_vec4(const SegJob& j, uint32_t s, int c4, const D4& acc,
                                                bool col0, double acc2);

// acc += the partial slots slot(0), slot(1), ..., slot(n - 1) of column group c4, added in
// that order; loads are issued 8 at a time (the slots were written by other CTAs: L2 loads).
template <class SlotFn>
__device__ __forceinline__ void sum_slots(const SegJob& j, int c4, int64_t n, SlotFn slot,
                                          D4& acc, double& acc2) {
  for (int64_t q0 = 0; q0 < n; q0 += 8) {
    double2 v[8][2];
    double p2[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u < n) {
        const int64_t sl = slot(q0 + u);
        const double2* pp = reinterpret_cast<const double2*>(j.part + sl * j.dim) + 2 * c4;
        v[u][0] = __ldcg(pp);
        v[u][1] = __ldcg(pp + 1);
        p2[u] = (c4 == 0 && j.rows2) ? __ldcg(j.part2 + sl) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u < n) {
        add4(acc, D4{v[u][0].x, v[u][0].y, v[u][1].x, v[u][1].y});
        acc2 += p2[u];
      }
    }
  }
}

// One CTA arrives with its piece of crossing segment s (window `chunk`; its partial is already
// in slot 2 chunk (head piece) or 2 chunk + 1 (the segment's first piece)).  Level 1: the pieces
// of s inside one block of kRunWin windows are summed, in window order, by the block's last
// arriver into the slot of the block's first piece.  Level 2: the last block to finish sums the
// block partials in block order and finishes the segment (table update or written sum).  Fixed
// order at both levels (R-16); arrival order only decides WHO adds, never the order.
template <int OPT, bool WR>
__device__ __forceinline__ void cross_arrive(const SegJob& j, uint32_t s, int64_t chunk,
                                          bool head_piece) {
  __shared__ int s_last;
  const int64_t c0 = j.seg_start[s] / j.chunk, c1 = (j.seg_start[s + 1] - 1) / j.chunk;
  const int64_t b = chunk / kRunWin;
  const int64_t w0 = max(c0, b * kRunWin), w1 = min(c1, b * kRunWin + kRunWin - 1);
  auto slot_of = [&](int64_t w) { return w == c0 ? 2 * w + 1 : 2 * w; };
  (void)head_piece;
  __syncthreads();  // this CTA's partial (all columns) is written
  if (threadIdx.x == 0) {
    __threadfence();
    // keyed by the run's first SLOT (a window can start one run and end another)
    const uint32_t need = (uint32_t)(w1 - w0 + 1);
    const int64_t key = slot_of(w0);
    const uint32_t old = atomicAdd(j.win_cnt + key, 1u);
    s_last = old + 1 == need;
    if (s_last) {
      j.win_cnt[key] = 0;
      __threadfence();
    }
  }
  __syncthreads();
  if (!s_last) return;
  const int n4 = j.dim >> 2;
  const int64_t first = slot_of(w0);
  const int64_t b0 = c0 / kRunWin, b1 = c1 / kRunWin;
  if (b0 == b1) {  // the segment lies in one block: level 1 finishes it (no second arrival)
    for (int c4 = threadIdx.x; c4 < n4; c4 += blockDim.x) {
      D4 acc = D4{0.0, 0.0, 0.0, 0.0};
      double acc2 = 0.0;
      sum_slots(j, c4, w1 - w0 + 1, [&](int64_t q) { return slot_of(w0 + q); }, acc, acc2);
      seg_finish_vec4<OPT, WR>(j, s, c4, acc, c4 == 0, acc2);
    }
    return;
  }
  for (int c4 = threadIdx.x; c4 < n4; c4 += blockDim.x) {  // level 1, window order
    D4 acc = D4{0.0, 0.0, 0.0, 0.0};
    double acc2 = 0.0;
    sum_slots(j, c4, w1 - w0 + 1, [&](int64_t q) { return slot_of(w0 + q); }, acc, acc2);
    reinterpret_cast<D4*>(j.part + first * j.dim)[c4] = acc;
    if (c4 == 0 && j.rows2) j.part2[first] = acc2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t old = atomicAdd(j.seg_cnt + s, 1u);
    s_last = old + 1 == (uint32_t)(b1 - b0 + 1);
    if (s_last) {
      j.seg_cnt[s] = 0;
      __threadfence();
    }
  }
  __syncthreads();
  if (!s_last) return;
  for (int c4 = threadIdx.x; c4 < n4; c4 += blockDim.x) {  // level 2, block order
    D4 acc = D4{0.0, 0.0, 0.0, 0.0};
    double acc2 = 0.0;
    sum_slots(j, c4, b1 - b0 + 1,
              [&](int64_t q) { return q == 0 ? 2 * c0 + 1 : 2 * (b0 + q) * kRunWin; }, acc, acc2);
    seg_finish_vec4<OPT, WR>(j, s, c4, acc, c4 == 0, acc2);
  }
}
static_assert(kChunk <= 32, "the window prologue maps row r of a window to lane r");
#ifndef TFS_WIN_MINB
#define TFS_WIN_MINB 4  // CTAs per SM the register budget must allow (128 regs at 4)
#endif
// WR: write mode (sort_reduce / route_reduce: sums written out, j.table == nullptr) or apply.
template <int OPT, bool WR>
__global__ void __launch_bounds__(128, TFS_WIN_MINB) seg_window_vec4_kernel(SegJob j) {
  pdl_enter();
  // The window's row program, built once by warp 0 (lane r = row r) and read by every column
  // thread as broadcast shared loads: the gradient row's float offset (-1: skipped row), its
  // companion offset, the table row's float offset when a whole segment ends at r (apply mode),
  // and the flags below.  The column loop then runs branch-uniform with no index arithmetic.
  enum : uint32_t { kReset = 1, kPieceEnd = 2, kWhole = 4, kHeadSlot = 8 };
  __shared__ int64_t s_off[32], s_off2[32], s_toff[32];  // one entry per lane of warp 0
  __shared__ uint32_t s_key[32], s_seg[32], s_fl[32];
  __shared__ int s_edge[2];
  const int64_t chunk = blockIdx.x;
  const int64_t base = chunk * j.chunk;
  const int cnt = (int)min((int64_t)j.chunk, j.n - base);
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    uint32_t key_l = 0xffffffffu, seg_l = 0, perm_l = 0;
    if (lane < cnt) {
      perm_l = j.perm[base + lane];
      key_l = j.keys[base + lane];
      seg_l = j.seg_of[base + lane];
    }
    uint32_t edge = 0;
    if (lane == 0 && base > 0) edge = j.keys[base - 1] == j.keys[base];
    if (lane == 1 && base + cnt < j.n) edge = j.keys[base + cnt] == j.keys[base + cnt - 1];
    const bool first_before = __shfl_sync(0xffffffffu, edge, 0) != 0;
    const bool last_after = __shfl_sync(0xffffffffu, edge, 1) != 0;
    const uint32_t key_prev = __shfl_up_sync(0xffffffffu, key_l, 1);
    const bool head_l = lane < cnt && (lane == 0 ? !first_before : key_l != key_prev);
    const uint32_t H = __ballot_sync(0xffffffffu, head_l);
    const bool valid_l = lane < cnt && key_l < j.invalid_key;
    // the piece holding row r starts at the last head <= r (row 0 if none: it started before)
    const uint32_t upto = H & ((2u << lane) - 1u);
    const bool starts_before = upto == 0;  // (implies first_before)
    const bool piece_end = lane < cnt && (lane == cnt - 1 || ((H >> (lane + 1)) & 1));
    const bool ends_after = lane == cnt - 1 && last_after;
    const bool whole = piece_end && !starts_before && !ends_after;
    uint32_t fl = 0;
    if (lane > 0 && lane < cnt && ((H >> lane) & 1)) fl |= kReset;
    if (valid_l && piece_end) fl |= kPieceEnd | (whole ? kWhole : 0) | (starts_before ? kHeadSlot : 0);
    s_fl[lane] = fl;
    s_key[lane] = key_l;
    s_seg[lane] = seg_l;
    s_off[lane] = valid_l ? row_off(j, perm_l) : -1;
    s_off2[lane] = (valid_l && j.rows2) ? row2_off(j, perm_l) : -1;
    s_toff[lane] = (!WR && valid_l && whole) ? (int64_t)key_l * j.dim : -1;
    if (lane == 0) {
      s_edge[0] = first_before;
      s_edge[1] = last_after;
    }
    // which segments own this window's two partial slots
    const uint32_t s_first = __shfl_sync(0xffffffffu, seg_l, 0);
    const uint32_t k_first = __shfl_sync(0xffffffffu, key_l, 0);
    const uint32_t s_last = __shfl_sync(0xffffffffu, seg_l, cnt - 1);
    const uint32_t k_last = __shfl_sync(0xffffffffu, key_l, cnt - 1);
    if (lane == 0) {
      const int head = (first_before && k_first < j.invalid_key) ? (int)s_first : -1;
      const int tail = (last_after && k_last < j.invalid_key && (int)s_last != head)
                           ? (int)s_last : -1;
      j.chunk_info[chunk] = make_int2(head, tail);
    }
  }
  __syncthreads();
  // Sorted keys put skipped entries (padding slots, bad ids: key >= invalid_key) last, so a
  // window whose first key is invalid has nothing to do, and no invalid row is ever loaded.
  if (s_key[0] >= j.invalid_key) return;
  const bool first_before = s_edge[0] != 0, last_after = s_edge[1] != 0;
  const int n4 = j.dim >> 2;
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c4 = tid; c4 < n4; c4 += blockDim.x) {
    const bool col0 = c4 == 0;
    D4 acc = D4{0.0, 0.0, 0.0, 0.0};
    double acc2 = 0.0;
    // Rows in half-batches of kHalf, software-pipelined: the loads of half-batch h + 1 (its
    // gradient rows and the table rows of the whole segments ending in it) are in flight while
    // half-batch h is summed and applied.
    constexpr int kHalf = kWinBatch / 2;
    float4 x[2][kHalf], t[2][kHalf];
    float r2v[2][kHalf];
    auto load_half = [&](int hb, int buf) {
#pragma unroll
      for (int q = 0; q < kHalf; ++q) {
        const int r = hb * kHalf + q;
        const int64_t o = s_off[r];
        x[buf][q] = o >= 0 ? __ldg(reinterpret_cast<const float4*>(j.rows + o) + c4) : z4;
        r2v[buf][q] = 0.f;
        if (col0) {
          const int64_t o2 = s_off2[r];
          if (o2 >= 0) r2v[buf][q] = __ldg(j.rows2 + o2);
        }
        if (!WR) {
          const int64_t to = s_toff[r];
          t[buf][q] = to >= 0 ? *(reinterpret_cast<const float4*>(j.table + to) + c4) : z4;
        }
      }
    };
    auto proc_half = [&](int hb, int buf) {
#pragma unroll
      for (int q = 0; q < kHalf; ++q) {
        const int r = hb * kHalf + q;
        if (r >= cnt) break;
        const uint32_t f = s_fl[r];
        if (f & kReset) {
          acc = D4{0.0, 0.0, 0.0, 0.0};
          acc2 = 0.0;
        }
        add4(acc, x[buf][q]);
        acc2 += r2v[buf][q];
        if (!(f & kPieceEnd)) continue;
        // ---- the piece ending at row r is complete
        if (f & kWhole) {  // whole segment: apply / write now
          const uint32_t kr = s_key[r];
          if (WR) {
            const OutPos op = seg_out_pos(j, s_seg[r], kr);
            if (op.row != nullptr) {
              reinterpret_cast<float4*>(op.row)[c4] = to_f4(acc);
              if (col0) {
                if (j.out_local) j.out_local[op.local] = (int64_t)(kr % (uint32_t)j.nloc);
                if (op.r2) *op.r2 = (float)acc2;
              }
            }
          } else {
            const float4 nv = opt_step4<OPT>(j, t[buf][q], acc, kr, c4);
            *(reinterpret_cast<float4*>(j.table + s_toff[r]) + c4) = nv;
            if (j.mirror)
              reinterpret_cast<uint2*>(j.mirror + s_toff[r])[c4] =
                  make_uint2(pack_bf16x2(nv.x, nv.y), pack_bf16x2(nv.z, nv.w));
            if (j.table2 && col0) opt_step2<OPT>(j, kr, acc2);
          }
        } else {
          const int64_t slot = (f & kHeadSlot) ? 2 * chunk : 2 * chunk + 1;
          reinterpret_cast<D4*>(j.part + slot * j.dim)[c4] = acc;
          if (col0 && j.rows2) j.part2[slot] = acc2;
        }
      }
    };
    const int nh = (cnt + kHalf - 1) / kHalf;
    load_half(0, 0);
    for (int hb = 0; hb < nh; hb += 2) {
      if (hb + 1 < nh) load_half(hb + 1, 1);
      proc_half(hb, 0);
      if (hb + 2 < nh) load_half(hb + 2, 0);
      if (hb + 1 < nh) proc_half(hb + 1, 1);
    }
  }
  // Pieces of segments crossing this window's edges (at most two: the one that started before
  // it and the one that continues after it): arrive, and the last arriver of a level sums it.
  const uint32_t kf = s_key[0], kl = s_key[cnt - 1];
  if (first_before && kf < j.invalid_key) cross_arrive<OPT, WR>(j, s_seg[0], chunk, true);
  if (last_after && kl < j.invalid_key && !(first_before && s_seg[cnt - 1] == s_seg[0]))
    cross_arrive<OPT, WR>(j, s_seg[cnt - 1], chunk, false);
}

// A segment whose pieces are all summed: T[key] = fl32(T - lr * g) (apply) or written out.
template <int OPT, bool WR>
__device__ __forceinline__ void seg_finish_vec4(const SegJob& j, uint32_t s, int c4, const D4& acc,
                                                bool col0, double acc2) {
  const uint32_t key = j.keys[j.seg_start[s]];
  if (key >= j.invalid_key) return;
  if (WR) {
    const OutPos op = seg_out_pos(j, s, key);
    if (op.row == nullptr) return;
    reinterpret_cast<float4*>(op.row)[c4] = to_f4(acc);
    if (col0) {
      if (j.out_local) j.out_local[op.local] = (int64_t)(key % (uint32_t)j.nloc);
      if (op.r2) *op.r2 = (float)acc2;
    }
  } else {
    float4* tp = reinterpret_cast<float4*>(j.table + (int64_t)key * j.dim) + c4;
    const float4 nv = opt_step4<OPT>(j, *tp, acc, key, c4);
    *tp = nv;
    if (j.mirror)
      reinterpret_cast<uint2*>(j.mirror + (int64_t)key * j.dim)[c4] =
          make_uint2(pack_bf16x2(nv.x, nv.y), pack_bf16x2(nv.z, nv.w));
    if (col0 && j.table2) opt_step2<OPT>(j, key, acc2);
  }
}

// Scalar columns (any dim): same structure, one column per lane per 32-column block.
__global__ void __launch_bounds__(256) seg_chunk_scalar_kernel(SegJob j) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t chunk = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t base = chunk * j.chunk;
  if (base >= j.n) return;
  const int cnt = (int)min((int64_t)j.chunk, j.n - base);
  uint32_t perm_l = 0, seg_l = 0, key_l = 0;
  float r2_l = 0.f;
  if (lane < cnt) {
    perm_l = j.perm[base + lane];
    seg_l = j.seg_of[base + lane];
    key_l = j.keys[base + lane];
    if (j.rows2) r2_l = j.rows2[row2_off(j, perm_l)];
  }
  uint32_t edge = 0;
  if (lane == 0 && base > 0) edge = j.keys[base - 1] == j.keys[base];
  if (lane == 1 && base + cnt < j.n) edge = j.keys[base + cnt] == j.keys[base + cnt - 1];
  const bool first_before = __shfl_sync(0xffffffffu, edge, 0) != 0;
  const bool last_after = __shfl_sync(0xffffffffu, edge, 1) != 0;
  const bool write_mode = j.table == nullptr;
  for (int c0 = 0; c0 < j.dim; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0, acc2 = 0.0;
    int r_start = 0;
    uint32_t cur = __shfl_sync(0xffffffffu, seg_l, 0);
    uint32_t cur_key = __shfl_sync(0xffffffffu, key_l, 0);
    auto flush = [&](int r_end) {
      if (cur_key >= j.invalid_key) return;
      const PieceDst dst = piece_dst(r_start == 0 && first_before, r_end == cnt && last_after,
                                     chunk);
      if (dst.kind == 0) {
        const OutPos op = write_mode ? seg_out_pos(j, cur, cur_key)
                                     : OutPos{j.sums + (int64_t)cur * j.dim,
                                              j.sums2 + cur, (int64_t)cur};
        if (op.row == nullptr) return;
        if (c < j.dim) op.row[c] = (float)acc;
        if (j.rows2 && op.r2 && lane == 0 && c0 == 0) *op.r2 = (float)acc2;
      } else {
        if (c < j.dim) j.part[dst.slot * j.dim + c] = acc;
        if (j.rows2 && lane == 0 && c0 == 0) j.part2[dst.slot] = acc2;
      }
    };
    for (int r = 0; r < cnt; ++r) {
      const uint32_t pr = __shfl_sync(0xffffffffu, perm_l, r);
      const uint32_t s = __shfl_sync(0xffffffffu, seg_l, r);
      const uint32_t k = __shfl_sync(0xffffffffu, key_l, r);
      const float r2 = __shfl_sync(0xffffffffu, r2_l, r);
      const float xv = c < j.dim ? j.rows[row_off(j, pr) + c] : 0.f;
      if (s != cur) {
        flush(r);
        cur = s;
        cur_key = k;
        r_start = r;
        acc = 0.0;
        acc2 = 0.0;
      }
      acc += xv;
      acc2 += r2;
    }
    flush(cnt);
  }
}

// One thread per (segment, column group): finish segments that cross chunk boundaries (their
// chunk partials added in chunk order) and, in apply mode, T[key] = fl32(T - lr * sum) for
// every segment; in write mode, out_local for every segment.  Fully parallel, coalesced.
template <bool VEC, int OPT>
__global__ void __launch_bounds__(256) seg_apply_kernel(SegJob j) {
  pdl_enter();
  const int64_t U = *j.num_unique;
  const int cols = VEC ? (j.dim >> 2) : j.dim;
  const int64_t total = U * cols;
  const bool write_mode = j.table == nullptr;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e / cols;
    const int c = (int)(e - u * cols);
    const uint32_t a = j.seg_start[u], b = j.seg_start[u + 1];
    const uint32_t key = j.keys[a];
    if (key >= j.invalid_key) continue;
    const OutPos op = write_mode ? seg_out_pos(j, u, key) : OutPos{j.table, nullptr, u};
    if (op.row == nullptr) continue;
    if (write_mode && c == 0 && j.out_local) j.out_local[op.local] = (int64_t)(key % (uint32_t)j.nloc);
    const int64_t c0 = a / j.chunk, c1 = (b - 1) / j.chunk;
    const bool cross = c0 != c1;
    if (write_mode && !cross) continue;  // the chunk kernel already wrote it
    if (VEC) {
      D4 acc;
      if (cross) {
        acc = reinterpret_cast<const D4*>(j.part + (2 * c0 + 1) * j.dim)[c];
#pragma unroll 4
        for (int64_t ch = c0 + 1; ch <= c1; ++ch)
          add4(acc, reinterpret_cast<const D4*>(j.part + (2 * ch) * j.dim)[c]);
      } else {
        const float4 s = reinterpret_cast<const float4*>(j.sums + u * j.dim)[c];
        acc = D4{s.x, s.y, s.z, s.w};
      }
      if (write_mode) {
        reinterpret_cast<float4*>(op.row)[c] = to_f4(acc);
      } else {
        float4* t = reinterpret_cast<float4*>(j.table + (int64_t)key * j.dim) + c;
        *t = opt_step4<OPT>(j, *t, acc, key, c);
      }
    } else {
      double acc;
      if (cross) {
        acc = j.part[(2 * c0 + 1) * j.dim + c];
#pragma unroll 4
        for (int64_t ch = c0 + 1; ch <= c1; ++ch) acc += j.part[(2 * ch) * j.dim + c];
      } else {
        acc = j.sums[u * j.dim + c];
      }
      if (write_mode) {
        op.row[c] = (float)acc;
      } else {
        float* t = j.table + (int64_t)key * j.dim + c;
        float sv = OPT ? j.slot[(int64_t)key * j.dim + c] : 0.f;
        *t = opt_step<OPT>(j, *t, acc, sv);
        if (OPT) j.slot[(int64_t)key * j.dim + c] = sv;
      }
    }
    if (c == 0 && j.rows2) {
      double acc2;
      if (cross) {
        acc2 = j.part2[2 * c0 + 1];
        for (int64_t ch = c0 + 1; ch <= c1; ++ch) acc2 += j.part2[2 * ch];
      } else {
        acc2 = write_mode ? 0.0 : j.sums2[u];
      }
      if (write_mode) {
        if (op.r2) *op.r2 = (float)acc2;
      } else if (j.table2) {
        opt_step2<OPT>(j, key, acc2);
      }
    }
  }
}

__global__ void owner_counts_kernel(const uint32_t* keys, const uint32_t* seg_start,
                                    const int64_t* num_unique, int32_t R, int64_t nloc,
                                    uint32_t invalid_key, int64_t* counts) {
  pdl_enter();
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

// Scratch of a segmented reduction, in two parts: the PLAN (sorted keys, permutation, segment
// structure -- a function of the ids only, so it can be built before the rows exist) and the
// APPLY scratch (partial sums of the segments that cross chunk boundaries).
struct SegScratch {
  // plan
  uint32_t *k0, *v0, *k1, *v1, *seg_start, *seg_of, *tile_cnt;
  int64_t* num_unique;
  void* sort_ws;
  size_t sort_ws_bytes;
  // apply
  double *part, *part2;
  float *sums, *sums2;
  uint32_t *cross_list, *cross_count;
  int2* chunk_info;
  uint32_t *win_cnt, *seg_cnt;
};

static void carve_plan(Carver& c, int64_t n, SegScratch& x) {
  const int64_t ntiles = cdiv(n, kSortTile);
  x.k0 = c.take<uint32_t>(n);
  x.v0 = c.take<uint32_t>(n);
  x.k1 = c.take<uint32_t>(n);
  x.v1 = c.take<uint32_t>(n);
  x.seg_start = c.take<uint32_t>(n + 1);
  x.seg_of = c.take<uint32_t>(n);
  x.tile_cnt = c.take<uint32_t>(ntiles + 1);
  x.num_unique = c.take<int64_t>(1);
  x.sort_ws_bytes = radix_sort_ws_bytes(n);
  x.sort_ws = c.take<char>(x.sort_ws_bytes);
}

static void carve_apply(Carver& c, int64_t n, int32_t dim, SegScratch& x) {
  const int64_t nchunks = cdiv(n, kChunkMin);
  x.part = c.take<double>((size_t)2 * nchunks * dim);
  x.part2 = c.take<double>((size_t)2 * nchunks);
  x.sums = c.take<float>((size_t)n * dim);
  x.sums2 = c.take<float>((size_t)n);
  x.cross_list = c.take<uint32_t>((size_t)nchunks + 1);
  x.cross_count = c.take<uint32_t>(1);
  x.chunk_info = c.take<int2>((size_t)nchunks);
  x.win_cnt = c.take<uint32_t>((size_t)2 * nchunks);
  x.seg_cnt = c.take<uint32_t>((size_t)n);
}

static size_t plan_scratch_bytes(int64_t n, SegScratch* s, void* ws, size_t cap) {
  Carver c(ws, cap);
  SegScratch x{};
  carve_plan(c, n, x);
  if (s) *s = x;
  return c.used + 256;
}

static size_t apply_scratch_bytes(int64_t n, int32_t dim, SegScratch* s, void* ws, size_t cap) {
  Carver c(ws, cap);
  SegScratch x{};
  carve_apply(c, n, dim, x);
  if (s) {
    s->part = x.part; s->part2 = x.part2; s->sums = x.sums; s->sums2 = x.sums2;
    s->cross_list = x.cross_list; s->cross_count = x.cross_count;
    s->chunk_info = x.chunk_info;
    s->win_cnt = x.win_cnt; s->seg_cnt = x.seg_cnt;
  }
  return c.used + 256;
}

static size_t seg_scratch_bytes(int64_t n, int32_t dim, SegScratch* s, void* ws, size_t cap) {
  Carver c(ws, cap);
  SegScratch x{};
  carve_plan(c, n, x);
  carve_apply(c, n, dim, x);
  if (s) *s = x;
  return c.used + 256;
}

// Single-CTA sort + segmentation for n <= kSmallMax (both plans of the X workload): keys are
// built, radix-sorted (8-bit LSD passes, stable) and segmented entirely in shared memory by
// one 1024-thread CTA -- one launch instead of nine.  Warp w owns the contiguous input range
// [w * per, (w + 1) * per); its digit counts are private (no per-round CTA barriers), and one
// CTA-wide exclusive scan over the (digit, warp) counters in digit-major order per pass makes
// the scatter stable (equal digits keep warp order, and lane order inside a warp).
constexpr int kSmallThreads = 1024;
constexpr int kSmallMax = 4096;  // above this the multi-CTA passes are faster (measured)
constexpr int kCntWords = 32 * 257;

__device__ __forceinline__ uint32_t cta1024_exclusive_scan(uint32_t v, uint32_t* wsum,
                                                           uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane], z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z - w;  // exclusive warp offsets
    if (lane == 31) wsum[32] = z;
  }
  __syncthreads();
  const uint32_t r = wsum[warp] + x - v;
  if (total) *total = wsum[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kSmallThreads, 1) sort_segment_small_kernel(
    IdsView ids, int n, int64_t limit, int32_t R, int64_t nloc, int composite, int passes,
    uint32_t* keys_out, uint32_t* perm_out, uint32_t* seg_start, uint32_t* seg_of,
    int64_t* num_unique, tfs_device_error* err) {
  pdl_enter();
  extern __shared__ uint32_t sm[];
  __shared__ uint32_t wsum[33];
  const int cap = (n + 31) & ~31;
  // counters: warp w, digit d at cnt[w * 257 + d] (pitch 257: conflict-free per-warp updates
  // and digit-major scans)
  uint32_t* cnt = sm;
  uint32_t* ka = cnt + kCntWords;
  uint32_t* kb = ka + cap;
  uint16_t* va = (uint16_t*)(kb + cap);
  uint16_t* vb = va + cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int i = tid; i < n; i += kSmallThreads) {
    const int64_t id = load_id(ids, i);
    uint32_t key;
    if (id < 0 || id >= limit) {
      if (id != -1) report_error(err, TFS_ERR_OUT_OF_RANGE, i);  // -1: padding, skipped
      key = composite ? (uint32_t)(R * nloc) : (uint32_t)limit;
    } else {
      key = composite ? (uint32_t)((id % R) * nloc + id / R) : (uint32_t)id;
    }
    ka[i] = key;
    va[i] = (uint16_t)i;
  }
  const int per = (((n + 31) / 32) + 31) & ~31;  // items per warp, a multiple of 32
  const int lo = min(n, warp * per), hi = min(n, lo + per);
  __syncthreads();
  for (int p = 0; p < passes; ++p) {
    const uint32_t* ks = ka;
    const uint16_t* vs = va;
    uint32_t* kd = kb;
    uint16_t* vd = vb;
    const int shift = 8 * p;
    for (int d = lane; d < 256; d += 32) cnt[warp * 257 + d] = 0;
    __syncwarp();
    for (int base = lo; base < hi; base += 32) {  // sweep 1: this warp's digit counts
      const int i = base + lane;
      const int dg = i < hi ? (int)((ks[i] >> shift) & 0xffu) : 256;
      const uint32_t peers = match_digit8(dg & 0xff, dg < 256);
      if (dg < 256 && lane == __ffs(peers) - 1) cnt[warp * 257 + dg] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {  // exclusive scan of the 8192 counters in (digit, warp) order; 8 per thread
      // entry e = d * 32 + w of the digit-major order lives at cnt[w * 257 + d]
      uint32_t c[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = tid * 8 + j;
        c[j] = cnt[(e & 31) * 257 + (e >> 5)];
        s += c[j];
      }
      uint32_t run = cta1024_exclusive_scan(s, wsum, nullptr);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int e = tid * 8 + j;
        cnt[(e & 31) * 257 + (e >> 5)] = run;
        run += c[j];
      }
    }
    __syncthreads();
    for (int base = lo; base < hi; base += 32) {  // sweep 2: stable scatter
      const int i = base + lane;
      const bool valid = i < hi;
      const uint32_t k = valid ? ks[i] : 0u;
      const int dg = valid ? (int)((k >> shift) & 0xffu) : 256;
      const uint32_t peers = match_digit8(dg & 0xff, valid);
      uint32_t off = 0;
      if (valid) {
        off = cnt[warp * 257 + dg];
        const uint32_t pos = off + __popc(peers & lanemask_lt());
        kd[pos] = k;
        vd[pos] = vs[i];
      }
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) cnt[warp * 257 + dg] = off + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    uint32_t* kt = ka; ka = kb; kb = kt;
    uint16_t* vt = va; va = vb; vb = vt;
  }
  // Segments of the sorted keys: heads, segment starts, segment of every position.
  const uint32_t* k = ka;
  const uint16_t* v = va;
  const int per_t = (n + kSmallThreads - 1) / kSmallThreads;
  const int t0 = min(n, tid * per_t), t1 = min(n, t0 + per_t);
  uint32_t h = 0;
  for (int i = t0; i < t1; ++i) h += (i == 0 || k[i] != k[i - 1]);
  uint32_t total;
  uint32_t pos = cta1024_exclusive_scan(h, wsum, &total);
  for (int i = t0; i < t1; ++i) {
    if (i == 0 || k[i] != k[i - 1]) seg_start[pos++] = (uint32_t)i;
    seg_of[i] = pos - 1;
    keys_out[i] = k[i];
    perm_out[i] = v[i];
  }
  if (tid == 0) {
    *num_unique = total;
    seg_start[total] = (uint32_t)n;
  }
}

static size_t small_sort_smem(int64_t n) {
  const int64_t cap = (n + 31) & ~31;
  return (size_t)(kCntWords * 4 + cap * 4 * 2 + cap * 2 * 2);
}

static int32_t sort_and_segment(IdsView ids, int64_t n, int64_t limit, int32_t R,
                                int64_t nloc, int composite, uint32_t key_max, SegScratch& s,
                                tfs_device_error* err, cudaStream_t st) {
  if (n <= kSmallMax) {
    const size_t smem = small_sort_smem(n);
    static bool attr = false;
    if (!attr) {
      TFS_CUDA_TRY(cudaFuncSetAttribute(sort_segment_small_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)small_sort_smem(kSmallMax)));
      attr = true;
    }
    const int bits = bits_for(key_max);
    const int passes = bits <= 8 ? 1 : (bits + 7) / 8;
    ::tfs::launch(sort_segment_small_kernel, 1, kSmallThreads, smem, st, 
        ids, (int)n, limit, R, nloc, composite, passes, s.k1, s.v1, s.seg_start, s.seg_of,
        s.num_unique, err);
    launched();
    TFS_LAUNCH_CHECK();
    return TFS_OK;
  }
  const int grid = (int)std::min<int64_t>(cdiv(n, 256), 4 * num_sms());
  ::tfs::launch(make_keys_kernel, grid, 256, 0, st, ids, n, limit, R, nloc, composite, s.k0, s.v0, err);
  launched();
  TFS_LAUNCH_CHECK();
  int32_t rc = radix_sort_pairs(s.k0, s.v0, s.k1, s.v1, n, bits_for(key_max), s.sort_ws,
                                s.sort_ws_bytes, st);
  if (rc != TFS_OK) return rc;
  const int ntiles = (int)cdiv(n, kSortTile);
  ::tfs::launch(heads_count_kernel, ntiles, kSortThreads, 0, st, s.k1, n, s.tile_cnt);
  launched();
  ::tfs::launch(heads_write_kernel, ntiles, kSortThreads, 0, st, s.k1, n, s.tile_cnt, ntiles, s.seg_start,
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
  j.sums = s.sums;
  j.sums2 = s.sums2;
  j.cross_list = s.cross_list;
  j.cross_count = s.cross_count;
  j.chunk_info = s.chunk_info;
  j.win_cnt = s.win_cnt;
  j.seg_cnt = s.seg_cnt;
}

static int32_t run_segments(SegJob& j, int64_t n, cudaStream_t st) {
  j.chunk = n >= TFS_SEG_SHORT_N ? kChunk : kChunkMin;
  const int64_t nchunks = cdiv(n, j.chunk);
  const int grid = (int)std::max<int64_t>(1, cdiv(nchunks, 8));
  // (inbox regions of out_tab are 16-byte aligned by construction: aligned bases, out_off % 4 == 0)
  const bool vec = (j.dim & 3) == 0 && ((uintptr_t)j.rows & 15) == 0 &&
                   (j.row_cap == 0 || j.row_stride % 4 == 0) &&
                   (j.table ? ((uintptr_t)j.table & 15) == 0
                            : (j.out_tab != nullptr || ((uintptr_t)j.out_rows & 15) == 0));
  if (!vec && j.mirror != nullptr) return TFS_ERR_INVALID_ARGUMENT;  // mirrors: vector path
  if (vec) {  // one launch: windows + the fused crossing reduction (cross_arrive)
    const int64_t n4 = j.dim >> 2;
    const int wthreads = (int)std::min<int64_t>(128, cdiv(n4, 32) * 32);
    const bool wr = j.table == nullptr;
    auto win_k = j.opt == 1   ? seg_window_vec4_kernel<1, false>
                 : j.opt == 2 ? seg_window_vec4_kernel<2, false>
                 : wr         ? seg_window_vec4_kernel<0, true>
                              : seg_window_vec4_kernel<0, false>;
    ::tfs::launch(win_k, (unsigned)nchunks, wthreads, 0, st, j);
    launched();
  } else {
    ::tfs::launch(seg_chunk_scalar_kernel, grid, 256, 0, st, j);
    launched();
    const int64_t work = n * j.dim;  // U <= n
    const int agrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(work, 256), 16 * num_sms()));
    auto apply_k = j.opt == 1 ? seg_apply_kernel<false, 1>
                              : (j.opt == 2 ? seg_apply_kernel<false, 2> : seg_apply_kernel<false, 0>);
    ::tfs::launch(apply_k, agrid, 256, 0, st, j);
    launched();
  }
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
  int32_t rc = sort_and_segment(IdsView{ids, 0, 0}, n, rows, 1, rows + 1, 0, (uint32_t)rows, s, err, st);
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

// ---- planned ScatterAdd-SGD: the id sort (plan) split from the row reduction (apply) ---------
extern "C" size_t tfs_scatter_plan_bytes(int64_t n) { return plan_scratch_bytes(n, nullptr, nullptr, 0); }

extern "C" int32_t tfs_scatter_plan(const int64_t* ids, int64_t n, int64_t rows, void* plan,
                                    size_t plan_bytes, tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 0 && rows >= 0 && rows < (1ll << 31) - 1 && n < (1ll << 31));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(ids && plan);
  TFS_SUPPORTED();
  SegScratch s;
  if (plan_bytes < plan_scratch_bytes(n, &s, plan, plan_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  return sort_and_segment(IdsView{ids, 0, 0}, n, rows, 1, rows + 1, 0, (uint32_t)rows, s, err, as_stream(stream));
}

extern "C" size_t tfs_scatter_apply_workspace_bytes(int64_t n, int32_t dim) {
  return apply_scratch_bytes(n, dim, nullptr, nullptr, 0);
}

extern "C" int32_t tfs_scatter_add_sgd_planned(float* table, int64_t rows, int32_t dim,
                                               const void* plan, size_t plan_bytes, int64_t n,
                                               const float* grad_rows, float lr, float* table2,
                                               const float* grad2, void* ws, size_t ws_bytes,
                                               void* stream) {
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0 && rows < (1ll << 31) - 1 && n < (1ll << 31));
  TFS_REQUIRE((table2 == nullptr) == (grad2 == nullptr));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && plan && grad_rows);
  TFS_REQUIRE(dim % 4 != 0 || ((uintptr_t)table & 15) == 0);
  TFS_SUPPORTED();
  SegScratch s;
  if (plan_bytes < plan_scratch_bytes(n, &s, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  if (ws_bytes < apply_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
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
  return run_segments(j, n, as_stream(stream));
}

// ---- fixed-capacity routing (R > 1): plan, unpack, reduce -----------------------------------
// A route plan is the composite-key (owner, local) sort plan of the requester's ids plus the
// per-owner segment bases: segment u of owner o travels in slot o * cap + (u - base[o]).  Only
// distinct ids travel (forward dedup); the reduced gradient rows use the same slots.
namespace tfs {

static size_t route_plan_bytes(int64_t n, int32_t R, SegScratch* s, int64_t** base, void* ws,
                               size_t cap) {
  Carver c(ws, cap);
  SegScratch x{};
  carve_plan(c, n, x);
  int64_t* b = c.take<int64_t>((size_t)R + 1);
  if (s) *s = x;
  if (base) *base = b;
  return c.used + 256;
}

// base[o] = first segment whose owner >= o (owner of an invalid key: R), o = 0..R: every
// segment u writes the bases of the owners in (owner(u-1), owner(u)], the last one those after
// it.  Fully parallel (no per-owner binary search).
__device__ __forceinline__ int64_t seg_owner(const uint32_t* keys, const uint32_t* seg_start,
                                             int64_t u, int32_t R, int64_t nloc,
                                             uint32_t invalid_key) {
  const uint32_t k = keys[seg_start[u]];
  return k >= invalid_key ? R : (int64_t)(k / (uint32_t)nloc);
}
__global__ void route_bases_kernel(const uint32_t* keys, const uint32_t* seg_start,
                                   const int64_t* num_unique, int64_t n, int32_t R, int64_t nloc,
                                   uint32_t invalid_key, int64_t* base) {
  pdl_enter();
  const int64_t U = *num_unique;
  if (U == 0) {
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o <= R;
         o += (int64_t)gridDim.x * blockDim.x)
      base[o] = 0;
    return;
  }
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ou = seg_owner(keys, seg_start, u, R, nloc, invalid_key);
    const int64_t op = u == 0 ? -1 : seg_owner(keys, seg_start, u - 1, R, nloc, invalid_key);
    for (int64_t o = op + 1; o <= ou; ++o) base[o] = u;
    if (u == U - 1)
      for (int64_t o = ou + 1; o <= R; ++o) base[o] = U;
  }
}

// Send ids go to send_local + o * stride (this GPU) or, with a pointer table, straight into
// owner o's inbox: dst_tab[o] + dst_off (one-sided NVLink stores).
__global__ void route_fill_kernel(const uint32_t* keys, const uint32_t* seg_start,
                                  const int64_t* base, int32_t R, int64_t cap, int64_t nloc,
                                  int64_t* send_local, int64_t stride,
                                  int64_t* const* dst_tab, int64_t dst_off, int64_t* counts,
                                  tfs_device_error* err) {
  pdl_enter();
  const int64_t total = (int64_t)R * cap;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = e / cap, jx = e - o * cap;
    if (jx == 0) {
      const int64_t c = base[o + 1] - base[o];
      if (counts) counts[o] = c;
      if (c > cap) report_error(err, TFS_ERR_CAPACITY, o);
    }
    const int64_t u = base[o] + jx;
    int64_t* dst = dst_tab ? dst_tab[o] + dst_off : send_local + o * stride;
    dst[jx] = u < base[o + 1] ? (int64_t)(keys[seg_start[u]] % (uint32_t)nloc) : -1;
  }
}

// out[t] = slots[o * cap + (u - base[o])] for every original position t (sorted position k:
// t = perm[k], u = seg_of[k], o = owner of keys[k]).
template <bool VEC>
__global__ void route_unpack_kernel(const uint32_t* keys, const uint32_t* perm,
                                    const uint32_t* seg_of, const int64_t* base, int64_t n,
                                    int32_t dim, int64_t cap, int64_t nloc, uint32_t invalid_key,
                                    const float* slots, int64_t stride, float* out) {
  pdl_enter();
  const int cols = VEC ? dim >> 2 : dim;
  const int64_t total = n * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / cols;
    const int c = (int)(e - k * cols);
    const uint32_t key = keys[k];
    if (key >= invalid_key) continue;
    const int64_t o = key / (uint32_t)nloc;
    const int64_t jx = (int64_t)seg_of[k] - base[o];
    if (jx >= cap) continue;
    const int64_t src = o * stride + jx * dim, dst = perm[k];  // float offset of the slot row
    if (VEC)
      reinterpret_cast<float4*>(out)[dst * cols + c] =
          __ldg(reinterpret_cast<const float4*>(slots + src) + c);
    else
      out[dst * dim + c] = __ldg(slots + src + c);
  }
}

}  // namespace tfs

extern "C" size_t tfs_route_plan_bytes(int64_t n, int32_t num_shards) {
  return route_plan_bytes(n, num_shards, nullptr, nullptr, nullptr, 0);
}

static int32_t route_plan_impl(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                               int64_t cap, void* plan, size_t plan_bytes, int64_t* out_send_local,
                               int64_t send_stride, int64_t* const* dst_tab, int64_t dst_off,
                               int64_t* out_counts, tfs_device_error* err, void* stream) {
  TFS_REQUIRE(n >= 1 && vocab >= 1 && num_shards >= 1 && num_shards <= 1024 && cap >= 1);
  TFS_REQUIRE(dst_tab != nullptr || send_stride >= cap);
  TFS_REQUIRE(n < (1ll << 31) && vocab + num_shards < (1ll << 32) - 1);
  TFS_REQUIRE(ids && plan && (out_send_local || dst_tab));
  TFS_SUPPORTED();
  SegScratch s;
  int64_t* base;
  if (plan_bytes < route_plan_bytes(n, num_shards, &s, &base, plan, plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  const int64_t nloc = cdiv(vocab, num_shards);
  const uint32_t invalid = (uint32_t)(num_shards * nloc);
  int32_t rc = sort_and_segment(IdsView{ids, 0, 0}, n, vocab, num_shards, nloc, 1, invalid, s, err, st);
  if (rc != TFS_OK) return rc;
  const int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4ll * num_sms()));
  ::tfs::launch(route_bases_kernel, bgrid, 256, 0, st, s.k1, s.seg_start, s.num_unique, n, num_shards, nloc,
                                            invalid, base);
  launched();
  const int64_t total = (int64_t)num_shards * cap;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 4ll * num_sms()));
  ::tfs::launch(route_fill_kernel, grid, 256, 0, st, s.k1, s.seg_start, base, num_shards, cap, nloc,
                                          out_send_local, send_stride, dst_tab, dst_off,
                                          out_counts, err);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" int32_t tfs_route_plan(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                                  int64_t cap, void* plan, size_t plan_bytes,
                                  int64_t* out_send_local, int64_t send_stride,
                                  int64_t* out_counts, tfs_device_error* err, void* stream) {
  return route_plan_impl(ids, n, vocab, num_shards, cap, plan, plan_bytes, out_send_local,
                         send_stride, nullptr, 0, out_counts, err, stream);
}

extern "C" int32_t tfs_route_plan_push(const int64_t* ids, int64_t n, int64_t vocab,
                                       int32_t num_shards, int64_t cap, void* plan,
                                       size_t plan_bytes, int64_t* const* dst_tab,
                                       int64_t dst_off, int64_t* out_counts,
                                       tfs_device_error* err, void* stream) {
  TFS_REQUIRE(dst_tab != nullptr && dst_off >= 0);
  return route_plan_impl(ids, n, vocab, num_shards, cap, plan, plan_bytes, nullptr, 0, dst_tab,
                         dst_off, out_counts, err, stream);
}

extern "C" int32_t tfs_route_unpack(const void* plan, size_t plan_bytes, int64_t n, int64_t vocab,
                                    int32_t num_shards, int64_t cap, const float* slots,
                                    int64_t slots_stride, int32_t dim, float* out, void* stream) {
  TFS_REQUIRE(n >= 1 && vocab >= 1 && num_shards >= 1 && num_shards <= 1024 && cap >= 1 &&
              dim >= 1 && slots_stride >= cap * dim);
  TFS_REQUIRE(plan && slots && out);
  TFS_SUPPORTED();
  SegScratch s;
  int64_t* base;
  if (plan_bytes < route_plan_bytes(n, num_shards, &s, &base, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  const int64_t nloc = cdiv(vocab, num_shards);
  const uint32_t invalid = (uint32_t)(num_shards * nloc);
  const bool vec = dim % 4 == 0 && slots_stride % 4 == 0 && ((uintptr_t)slots & 15) == 0 &&
                   ((uintptr_t)out & 15) == 0;
  const int64_t total = n * (vec ? dim / 4 : dim);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 8ll * num_sms()));
  if (vec)
    ::tfs::launch(route_unpack_kernel<true>, grid, 256, 0, st, s.k1, s.v1, s.seg_of, base, n, dim, cap, nloc,
                                                    invalid, slots, slots_stride, out);
  else
    ::tfs::launch(route_unpack_kernel<false>, grid, 256, 0, st, s.k1, s.v1, s.seg_of, base, n, dim, cap,
                                                     nloc, invalid, slots, slots_stride, out);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" size_t tfs_route_reduce_workspace_bytes(int64_t n, int32_t dim) {
  return apply_scratch_bytes(n, dim, nullptr, nullptr, 0);
}

extern "C" int32_t tfs_route_reduce(const void* plan, size_t plan_bytes, int64_t n, int64_t vocab,
                                    int32_t num_shards, int64_t cap, const float* rows,
                                    int32_t dim, const float* rows2, float* out_slots,
                                    int64_t out_stride, float* out_slots2, int64_t out2_stride,
                                    void* ws, size_t ws_bytes, void* stream) {
  TFS_REQUIRE(n >= 1 && vocab >= 1 && num_shards >= 1 && num_shards <= 1024 && cap >= 1 &&
              dim >= 1 && out_stride >= cap * dim);
  TFS_REQUIRE(plan && rows && out_slots);
  TFS_REQUIRE((rows2 == nullptr) == (out_slots2 == nullptr));
  TFS_REQUIRE(rows2 == nullptr || out2_stride >= cap);
  TFS_REQUIRE(dim % 4 != 0 || (((uintptr_t)out_slots & 15) == 0 && out_stride % 4 == 0));
  TFS_SUPPORTED();
  SegScratch s;
  int64_t* base;
  if (plan_bytes < route_plan_bytes(n, num_shards, &s, &base, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  if (ws_bytes < apply_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int64_t nloc = cdiv(vocab, num_shards);
  SegJob j{};
  bind(j, s, n);
  j.rows = rows;
  j.rows2 = rows2;
  j.dim = dim;
  j.invalid_key = (uint32_t)(num_shards * nloc);
  j.out_rows = out_slots;
  j.out_rows2 = out_slots2;
  j.nloc = nloc;
  j.slot_base = base;
  j.cap = cap;
  j.out_stride = out_stride;
  j.out2_stride = out2_stride;
  return run_segments(j, n, as_stream(stream));
}

// ---- merge of R ascending runs (owner side: every requester's distinct ids, ascending) -------
// Entry i = slot (o, s) of R runs of cap slots; a run is strictly ascending valid ids followed
// by -1 padding.  Sorted order = valid ids ascending, equal ids by run (requester) order, then
// the padding in entry order -- exactly the stable sort by key of the entries.  Every entry
// finds its place with R binary searches (one kernel instead of the radix passes).
__device__ __forceinline__ uint32_t run_key(const IdsView& v, int64_t o, int64_t s,
                                            int64_t limit) {
  const int64_t id = v.p[o * v.stride + s];
  return (id < 0 || id >= limit) ? 0xFFFFFFFFu : (uint32_t)id;
}
// number of entries of run o with key < x (strict) or <= x
__device__ __forceinline__ int64_t run_rank(const IdsView& v, int64_t o, int64_t cap,
                                            uint32_t x, bool inclusive, int64_t limit) {
  int64_t lo = 0, hi = cap;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const uint32_t k = run_key(v, o, mid, limit);
    if (inclusive ? k <= x : k < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__global__ void merge_runs_kernel(IdsView ids, int32_t R, int64_t cap, int64_t limit,
                                  uint32_t* keys_out, uint32_t* perm_out,
                                  tfs_device_error* err) {
  pdl_enter();
  const int64_t n = (int64_t)R * cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / cap, s = i - o * cap;
    const int64_t id = ids.p[o * ids.stride + s];
    const uint32_t k = run_key(ids, o, s, limit);
    if (id != -1 && k == 0xFFFFFFFFu) report_error(err, TFS_ERR_OUT_OF_RANGE, i);
    if (s + 1 < cap) {  // the promised layout: strictly ascending, padding only at the end
      const uint32_t kn = run_key(ids, o, s + 1, limit);
      if (kn != 0xFFFFFFFFu && kn <= k) report_error(err, TFS_ERR_INVALID_ARGUMENT, i);
    }
    int64_t pos;
    if (k != 0xFFFFFFFFu) {
      pos = s;
      for (int64_t q = 0; q < R; ++q)
        if (q != o) pos += run_rank(ids, q, cap, k, q < o, limit);
    } else {
      int64_t valid = 0, before = 0;
      for (int64_t q = 0; q < R; ++q) {
        const int64_t c = run_rank(ids, q, cap, 0xFFFFFFFEu, true, limit);
        valid += c;
        if (q < o) before += cap - c;
        else if (q == o) before += s - c;
      }
      pos = valid + before;
    }
    keys_out[pos] = k == 0xFFFFFFFFu ? (uint32_t)limit : k;
    perm_out[pos] = (uint32_t)i;
  }
}

extern "C" int32_t tfs_route_reduce_push(const void* plan, size_t plan_bytes, int64_t n,
                                         int64_t vocab, int32_t num_shards, int64_t cap,
                                         const float* rows, int32_t dim, const float* rows2,
                                         float* const* out_tab, int64_t out_off,
                                         float* const* out2_tab, int64_t out2_off, void* ws,
                                         size_t ws_bytes, void* stream) {
  TFS_REQUIRE(n >= 1 && vocab >= 1 && num_shards >= 1 && num_shards <= 1024 && cap >= 1 &&
              dim >= 1 && out_off >= 0 && out2_off >= 0);
  TFS_REQUIRE(plan && rows && out_tab);
  TFS_REQUIRE((rows2 == nullptr) == (out2_tab == nullptr));
  TFS_REQUIRE(dim % 4 != 0 || out_off % 4 == 0);
  TFS_SUPPORTED();
  SegScratch s;
  int64_t* base;
  if (plan_bytes < route_plan_bytes(n, num_shards, &s, &base, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  if (ws_bytes < apply_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  const int64_t nloc = cdiv(vocab, num_shards);
  SegJob j{};
  bind(j, s, n);
  j.rows = rows;
  j.rows2 = rows2;
  j.dim = dim;
  j.invalid_key = (uint32_t)(num_shards * nloc);
  j.nloc = nloc;
  j.slot_base = base;
  j.cap = cap;
  j.out_tab = out_tab;
  j.out2_tab = out2_tab;
  j.out_off = out_off;
  j.out2_off = out2_off;
  return run_segments(j, n, as_stream(stream));
}

// Same merge with every run staged in shared memory as 32-bit keys (R x cap x 4 bytes): the
// R binary searches per entry then cost shared-memory latency instead of L2 latency.
__device__ __forceinline__ int64_t smem_rank(const uint32_t* run, int64_t cap, uint32_t x,
                                             bool inclusive) {
  int64_t lo = 0, hi = cap;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const uint32_t k = run[mid];
    if (inclusive ? k <= x : k < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__global__ void __launch_bounds__(512) merge_runs_smem_kernel(IdsView ids, int32_t R, int64_t cap,
                                                              int64_t limit, uint32_t* keys_out,
                                                              uint32_t* perm_out,
                                                              tfs_device_error* err) {
  pdl_enter();
  extern __shared__ uint32_t runs[];  // [R][cap]
  const int64_t n = (int64_t)R * cap;
  for (int64_t i0 = threadIdx.x; i0 < n; i0 += 8 * (int64_t)blockDim.x) {  // 8 loads in flight
    uint32_t kk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * (int64_t)blockDim.x;
      kk[u] = i < n ? run_key(ids, i / cap, i - (i / cap) * cap, limit) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + u * (int64_t)blockDim.x;
      if (i < n) runs[i] = kk[u];
    }
  }
  __syncthreads();
  __shared__ int64_t valid_cnt[1024 + 1];  // R <= 1024: per-run valid counts, then the total
  for (int q = threadIdx.x; q < R; q += blockDim.x)
    valid_cnt[q] = smem_rank(runs + (int64_t)q * cap, cap, 0xFFFFFFFEu, true);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / cap, s = i - o * cap;
    const uint32_t k = runs[i];
    if (k == 0xFFFFFFFFu && ids.p[o * ids.stride + s] != -1)  // not padding: a bad id
      report_error(err, TFS_ERR_OUT_OF_RANGE, i);
    if (s + 1 < cap && runs[i + 1] != 0xFFFFFFFFu && runs[i + 1] <= k)
      report_error(err, TFS_ERR_INVALID_ARGUMENT, i);
    int64_t pos;
    if (k != 0xFFFFFFFFu) {
      pos = s;
      for (int64_t q = 0; q < R; ++q)
        if (q != o) pos += smem_rank(runs + q * cap, cap, k, q < o);
    } else {
      int64_t valid = 0, before = 0;
      for (int64_t q = 0; q < R; ++q) {
        const int64_t c = valid_cnt[q];
        valid += c;
        if (q < o) before += cap - c;
        else if (q == o) before += s - c;
      }
      pos = valid + before;
    }
    keys_out[pos] = k == 0xFFFFFFFFu ? (uint32_t)limit : k;
    perm_out[pos] = (uint32_t)i;
  }
}
constexpr size_t kMergeSmemMax = 200 * 1024;

// ---- planned ScatterAdd-SGD over ids / gradients received in slot layout (R x cap) ----------
extern "C" int32_t tfs_scatter_plan_slots(const int64_t* ids, int64_t ids_stride, int32_t R,
                                          int64_t cap, int64_t rows, int32_t sorted_runs,
                                          void* plan, size_t plan_bytes, tfs_device_error* err,
                                          void* stream) {
  TFS_REQUIRE(R >= 1 && cap >= 1 && ids_stride >= cap && rows >= 0 && rows < (1ll << 31) - 1);
  const int64_t n = (int64_t)R * cap;
  TFS_REQUIRE(n < (1ll << 31) && ids && plan);
  TFS_SUPPORTED();
  SegScratch s;
  if (plan_bytes < plan_scratch_bytes(n, &s, plan, plan_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  cudaStream_t st = as_stream(stream);
  if (!sorted_runs)
    return sort_and_segment(IdsView{ids, cap, ids_stride}, n, rows, 1, rows + 1, 0,
                            (uint32_t)rows, s, err, st);
  const size_t smem = (size_t)n * sizeof(uint32_t);
  if (smem <= kMergeSmemMax && R <= 1024) {
    static bool attr = false;
    if (!attr) {
      TFS_CUDA_TRY(cudaFuncSetAttribute(merge_runs_smem_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kMergeSmemMax));
      attr = true;
    }
    // every CTA stages all runs; few CTAs suffice (n ~ 1e4 entries)
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 512), num_sms()));
    ::tfs::launch(merge_runs_smem_kernel, grid, 512, smem, st, IdsView{ids, cap, ids_stride}, R, cap, rows,
                                                    s.k1, s.v1, err);
  } else {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8ll * num_sms()));
    ::tfs::launch(merge_runs_kernel, grid, 256, 0, st, IdsView{ids, cap, ids_stride}, R, cap, rows, s.k1,
                                            s.v1, err);
  }
  launched();
  const int ntiles = (int)cdiv(n, kSortTile);
  ::tfs::launch(heads_count_kernel, ntiles, kSortThreads, 0, st, s.k1, n, s.tile_cnt);
  launched();
  ::tfs::launch(heads_write_kernel, ntiles, kSortThreads, 0, st, s.k1, n, s.tile_cnt, ntiles, s.seg_start,
                                                      s.seg_of, s.num_unique);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

static int32_t planned_slots_impl(float* table, int64_t rows, int32_t dim, const void* plan,
                                  size_t plan_bytes, int32_t R, int64_t cap, const float* grad,
                                  int64_t grad_stride, float* table2, const float* grad2,
                                  int64_t grad2_stride, const tfs_sparse_opt* opt, void* ws,
                                  size_t ws_bytes, void* stream) {
  TFS_REQUIRE(R >= 1 && cap >= 1 && dim >= 1 && rows >= 0 && rows < (1ll << 31) - 1);
  TFS_REQUIRE(grad_stride >= cap * dim && (grad2 == nullptr || grad2_stride >= cap));
  TFS_REQUIRE((table2 == nullptr) == (grad2 == nullptr));
  TFS_REQUIRE(opt != nullptr && opt->kind >= 0 && opt->kind <= 2);
  TFS_REQUIRE(opt->kind == 0 || opt->slot != nullptr);
  TFS_REQUIRE(opt->kind == 0 || table2 == nullptr || opt->slot2 != nullptr);
  TFS_REQUIRE(opt->mirror == nullptr ||
              (dim % 8 == 0 && ((uintptr_t)opt->mirror & 15) == 0 && ((uintptr_t)table & 15) == 0));
  const int64_t n = (int64_t)R * cap;
  TFS_REQUIRE(table && plan && grad && n < (1ll << 31));
  TFS_REQUIRE(dim % 4 != 0 || (((uintptr_t)table & 15) == 0 && grad_stride % 4 == 0 &&
                               (opt->kind == 0 || ((uintptr_t)opt->slot & 15) == 0)));
  TFS_SUPPORTED();
  SegScratch s;
  if (plan_bytes < plan_scratch_bytes(n, &s, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  if (ws_bytes < apply_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  SegJob j{};
  bind(j, s, n);
  j.rows = grad;
  j.rows2 = grad2;
  j.dim = dim;
  j.invalid_key = (uint32_t)rows;
  j.table = table;
  j.table2 = table2;
  j.lr = opt->lr;
  j.opt = opt->kind;
  j.mu = (double)opt->mu;
  j.slot = opt->slot;
  j.slot2 = opt->slot2;
  j.mirror = opt->mirror;
  j.nloc = rows + 1;
  j.row_cap = cap;
  j.row_stride = grad_stride;
  j.row2_stride = grad2_stride;
  return run_segments(j, n, as_stream(stream));
}

extern "C" int32_t tfs_scatter_add_sgd_planned_slots(
    float* table, int64_t rows, int32_t dim, const void* plan, size_t plan_bytes, int32_t R,
    int64_t cap, const float* grad, int64_t grad_stride, float lr, float* table2,
    const float* grad2, int64_t grad2_stride, void* ws, size_t ws_bytes, void* stream) {
  const tfs_sparse_opt sgd{0, lr, 0.f, nullptr, nullptr};
  return planned_slots_impl(table, rows, dim, plan, plan_bytes, R, cap, grad, grad_stride, table2,
                            grad2, grad2_stride, &sgd, ws, ws_bytes, stream);
}

extern "C" int32_t tfs_scatter_opt_planned_slots(
    float* table, int64_t rows, int32_t dim, const void* plan, size_t plan_bytes, int32_t R,
    int64_t cap, const float* grad, int64_t grad_stride, float* table2, const float* grad2,
    int64_t grad2_stride, const tfs_sparse_opt* opt, void* ws, size_t ws_bytes, void* stream) {
  return planned_slots_impl(table, rows, dim, plan, plan_bytes, R, cap, grad, grad_stride, table2,
                            grad2, grad2_stride, opt, ws, ws_bytes, stream);
}

extern "C" int32_t tfs_scatter_opt_planned(float* table, int64_t rows, int32_t dim,
                                           const void* plan, size_t plan_bytes, int64_t n,
                                           const float* grad_rows, float* table2,
                                           const float* grad2, const tfs_sparse_opt* opt,
                                           void* ws, size_t ws_bytes, void* stream) {
  TFS_REQUIRE(opt != nullptr && opt->kind >= 0 && opt->kind <= 2);
  TFS_REQUIRE(n >= 0 && dim >= 1 && rows >= 0 && rows < (1ll << 31) - 1 && n < (1ll << 31));
  TFS_REQUIRE((table2 == nullptr) == (grad2 == nullptr));
  TFS_REQUIRE(opt->kind == 0 || opt->slot != nullptr);
  TFS_REQUIRE(opt->kind == 0 || table2 == nullptr || opt->slot2 != nullptr);
  TFS_REQUIRE(opt->mirror == nullptr ||
              (dim % 8 == 0 && ((uintptr_t)opt->mirror & 15) == 0 && ((uintptr_t)table & 15) == 0));
  if (n == 0) return TFS_OK;
  TFS_REQUIRE(table && plan && grad_rows);
  TFS_REQUIRE(dim % 4 != 0 || (((uintptr_t)table & 15) == 0 &&
                               (opt->kind == 0 || ((uintptr_t)opt->slot & 15) == 0)));
  TFS_SUPPORTED();
  SegScratch s;
  if (plan_bytes < plan_scratch_bytes(n, &s, const_cast<void*>(plan), plan_bytes))
    return TFS_ERR_WORKSPACE_TOO_SMALL;
  if (ws_bytes < apply_scratch_bytes(n, dim, &s, ws, ws_bytes)) return TFS_ERR_WORKSPACE_TOO_SMALL;
  SegJob j{};
  bind(j, s, n);
  j.rows = grad_rows;
  j.rows2 = grad2;
  j.dim = dim;
  j.invalid_key = (uint32_t)rows;
  j.table = table;
  j.table2 = table2;
  j.lr = opt->lr;
  j.opt = opt->kind;
  j.mu = (double)opt->mu;
  j.slot = opt->slot;
  j.slot2 = opt->slot2;
  j.mirror = opt->mirror;
  j.nloc = rows + 1;
  return run_segments(j, n, as_stream(stream));
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
  int32_t rc = sort_and_segment(IdsView{ids, 0, 0}, n, vocab, num_shards, nloc, 1, invalid, s, err, st);
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
  ::tfs::launch(owner_counts_kernel, 1, 1024, 0, st, s.k1, s.seg_start, s.num_unique, num_shards, nloc,
                                          invalid, out_counts);
  launched();
  TFS_LAUNCH_CHECK();
  // (With bad ids, U also counts their sentinel segment; outputs are unspecified then.)
  TFS_CUDA_TRY(cudaMemcpyAsync(out_num_unique, s.num_unique, sizeof(int64_t),
                               cudaMemcpyDeviceToDevice, st));
  return TFS_OK;
}
