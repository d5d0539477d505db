// step.cu -- the native step runtime of libtfs: the communicator (symmetric device heap +
// device barriers) and the stepper that composes the library's calls into one synchronous
// training step of the paper's large-vocabulary LM output path (include/tfs.h
// "The training step").  Every arithmetic step runs in the kernels of the other translation
// units; this file orders them on streams, moves nothing but ids / rows / gradients, and owns
// the buffers.
//
// One code path for both communicator modes: the step of one rank is a list of PHASES separated
// by barriers (each barrier names the stream it orders).  With one process per GPU the barrier
// is a one-block kernel on that stream (flags in the symmetric heap, P2P stores / loads); with
// all ranks simulated in one process on one GPU, phase k of every local rank is issued, then
// the barrier is stream ordering across the local ranks (events), then phase k + 1.  No kernel
// ever spins on another kernel of the same GPU.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "common.cuh"

#ifndef TFS_PRESAMPLE_LATE
#define TFS_PRESAMPLE_LATE 0  // A/B: R = 1 next-step draw forked after the softmax GEMMs
#endif
#ifndef TFS_SIDE_PRIO_HI
#define TFS_SIDE_PRIO_HI 1  // side / sampler streams at the highest priority (A/B switch)
#endif

namespace tfs {
namespace {

constexpr size_t kHeapHeader = 64 * 1024;  // barrier flags: [kChannels][kMaxRanks] uint32
#ifndef TFS_STEP_SM_RESERVE_R
#define TFS_STEP_SM_RESERVE_R 8  // SMs left free by the softmax GEMMs in the R > 1 step
#endif
#ifndef TFS_STEP_SM_RESERVE_1
#define TFS_STEP_SM_RESERVE_1 0  // ... and in the R = 1 step
#endif
constexpr int kChannels = 16;
constexpr int kMaxRanks = 64;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One block of >= R threads.  Thread i stores this barrier's epoch into slot (ch, rank) of rank
// i's flag area, then waits for slot (ch, i) of this rank's own area to reach the epoch.  The
// epoch lives in (local) device memory and advances by one per call, so a replayed CUDA graph
// keeps counting.  All prior work of the stream is complete when the kernel starts; the system
// fence + release store publish it to the peers, the acquire load orders what follows.
__global__ void barrier_kernel(const int64_t* bases, int R, int rank, int ch, uint32_t* epoch,
                               tfs_device_error* err, uint64_t timeout_ns) {
  pdl_enter();
  __shared__ uint32_t e;
  if (threadIdx.x == 0) {
    e = epoch[ch] + 1u;
    epoch[ch] = e;
  }
  __syncthreads();
  const int i = threadIdx.x;
  if (i < R) {
    __threadfence_system();
    uint32_t* peer = reinterpret_cast<uint32_t*>(bases[i]);
    st_release_sys(peer + ch * kMaxRanks + rank, e);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(bases[rank]) + ch * kMaxRanks + i;
    const uint64_t t0 = global_ns();
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
      if (global_ns() - t0 > timeout_ns) {
        report_error(err, TFS_ERR_COMM_TIMEOUT, i);
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void add_i64_kernel(int64_t* p, int64_t v) {
  pdl_enter(); *p += v; }

__global__ void next_counter_kernel(const int64_t* step, int64_t* next, int64_t add) {
  pdl_enter();
  *next = *step + add;
}

// Race detector (TFS_DEBUG_SIDE_DELAY_US, read at create; unset in production): a spin of that
// many microseconds at the head of every side-stream phase, so a missing cross-stream wait
// shows up as wrong results in the parity tests.  Results are unchanged -- only timing.
__global__ void delay_kernel(uint64_t ns) {
  pdl_enter();
  const uint64_t t0 = global_ns();
  while (global_ns() - t0 < ns) {
  }
}

// Index maps of the steps, computed once at create (nothing of them is left to the caller):
// mode 0: out[i] = i * mul + add (the candidate ids of a shard: j R + r; the full softmax's
// candidates 0..V-1); mode 1: out[g] = (g mod B) R + g div B (the all-gather order of the
// sharded full softmax: global token g = row g mod B of rank g div B, addressed as an id of the
// id-mod-R layout so that tfs_gather_peers can fetch it).
__global__ void index_map_kernel(int64_t* out, int64_t n, int mode, int64_t mul, int64_t add,
                                 int64_t B, int64_t R) {
  pdl_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = mode == 0 ? i * mul + add : (i % B) * R + i / B;
}

__global__ void fill_i64_kernel(int64_t* p, int64_t n, int64_t v) {
  pdl_enter();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void f32_to_bf16_kernel(const float* src, int64_t n, uint16_t* dst) {
  pdl_enter();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = f32_to_bf16_bits(src[i]);
}

inline int grid1d(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 65535)); }

}  // namespace
}  // namespace tfs

using namespace tfs;

// ================================================================================ communicator
struct tfs_comm {
  int32_t R = 0, first = 0, nlocal = 0, device = 0;
  size_t heap_bytes = 0;
  uint64_t timeout_ns = 0;
  std::vector<char*> heaps;            // nlocal local heaps
  std::vector<char*> bases;            // R heap bases as seen from this process
  std::vector<char> opened;            // bases[r] was IPC-opened (closed at destroy)
  std::vector<int64_t*> d_bases;       // per local rank: device int64[R]
  std::vector<uint32_t*> d_epoch;      // per local rank: device uint32[kChannels]
  std::vector<tfs_device_error*> d_err;
  bool connected = false;
};

namespace {
int32_t upload_bases(tfs_comm* c) {
  std::vector<int64_t> h(c->R);
  for (int r = 0; r < c->R; ++r) h[r] = (int64_t)(uintptr_t)c->bases[r];
  for (int l = 0; l < c->nlocal; ++l)
    TFS_CUDA_TRY(cudaMemcpy(c->d_bases[l], h.data(), sizeof(int64_t) * c->R,
                            cudaMemcpyHostToDevice));
  return TFS_OK;
}
}  // namespace

extern "C" int32_t tfs_comm_create(int32_t nranks, int32_t first_rank, int32_t nlocal,
                                   int32_t device, size_t heap_bytes, uint32_t timeout_ms,
                                   tfs_comm** out) {
  TFS_REQUIRE(out && nranks >= 1 && nranks <= kMaxRanks && nlocal >= 1);
  TFS_REQUIRE((nlocal == 1 && first_rank >= 0 && first_rank < nranks) ||
              (nlocal == nranks && first_rank == 0));
  TFS_CUDA_TRY(cudaSetDevice(device));
  TFS_SUPPORTED();
  tfs_comm* c = new tfs_comm();
  c->R = nranks;
  c->first = first_rank;
  c->nlocal = nlocal;
  c->device = device;
  c->heap_bytes = std::max(heap_bytes, kHeapHeader) ;
  c->heap_bytes = (c->heap_bytes + 4095) & ~size_t(4095);
  c->timeout_ns = (uint64_t)(timeout_ms ? timeout_ms : 10000) * 1000000ull;
  c->bases.assign(nranks, nullptr);
  c->opened.assign(nranks, 0);
  auto fail = [&](cudaError_t e, const char* what) {
    set_last_error(what, e);
    for (char* h : c->heaps) cudaFree(h);
    for (auto p : c->d_bases) cudaFree(p);
    delete c;
    return TFS_ERR_CUDA;
  };
  for (int l = 0; l < nlocal; ++l) {
    char* h = nullptr;
    cudaError_t e = cudaMalloc(&h, c->heap_bytes);
    if (e != cudaSuccess) return fail(e, "cudaMalloc(heap)");
    c->heaps.push_back(h);
    e = cudaMemset(h, 0, c->heap_bytes);
    if (e != cudaSuccess) return fail(e, "cudaMemset(heap)");
    c->bases[first_rank + l] = h;
    // small per-local-rank control block: bases [R] int64 | epochs [kChannels] u32 | error
    char* ctl = nullptr;
    e = cudaMalloc(&ctl, 1024);
    if (e != cudaSuccess) return fail(e, "cudaMalloc(ctl)");
    e = cudaMemset(ctl, 0, 1024);
    if (e != cudaSuccess) return fail(e, "cudaMemset(ctl)");
    c->d_bases.push_back(reinterpret_cast<int64_t*>(ctl));
    c->d_epoch.push_back(reinterpret_cast<uint32_t*>(ctl + 512));
    c->d_err.push_back(reinterpret_cast<tfs_device_error*>(ctl + 768));
    const tfs_device_error none{0, 0, INT64_MAX};
    e = cudaMemcpy(ctl + 768, &none, sizeof(none), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(e, "cudaMemcpy(err)");
  }
  if (nlocal == nranks) {  // simulated ranks: every heap is local
    if (upload_bases(c) != TFS_OK) return fail(cudaErrorUnknown, "upload_bases");
    c->connected = true;
  }
  *out = c;
  return TFS_OK;
}

extern "C" int32_t tfs_comm_export(tfs_comm* c, void* handle_out) {
  TFS_REQUIRE(c && handle_out && c->nlocal == 1);
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  TFS_CUDA_TRY(cudaSetDevice(c->device));
  TFS_CUDA_TRY(cudaIpcGetMemHandle(&h, c->heaps[0]));
  std::memcpy(handle_out, &h, 64);
  return TFS_OK;
}

extern "C" int32_t tfs_comm_connect(tfs_comm* c, const void* handles) {
  TFS_REQUIRE(c && handles && c->nlocal == 1 && !c->connected);
  TFS_CUDA_TRY(cudaSetDevice(c->device));
  for (int r = 0; r < c->R; ++r) {
    if (r == c->first) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, (const char*)handles + 64 * r, 64);
    void* p = nullptr;
    TFS_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->bases[r] = (char*)p;
    c->opened[r] = 1;
  }
  int32_t s = upload_bases(c);
  if (s != TFS_OK) return s;
  c->connected = true;
  return TFS_OK;
}

extern "C" int32_t tfs_comm_barrier(tfs_comm* c, int32_t channel, void* stream) {
  TFS_REQUIRE(c && c->nlocal == 1 && c->connected && channel >= 0 && channel < kChannels);
  ::tfs::launch(barrier_kernel, 1, 64, 0, as_stream(stream), c->d_bases[0], c->R, c->first, channel,
                                                 c->d_epoch[0], c->d_err[0], c->timeout_ns);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

extern "C" void* tfs_comm_heap(tfs_comm* c, int32_t local) {
  return (c && local >= 0 && local < c->nlocal) ? c->heaps[local] : nullptr;
}
extern "C" const int64_t* tfs_comm_peer_bases(tfs_comm* c, int32_t local) {
  return (c && local >= 0 && local < c->nlocal) ? c->d_bases[local] : nullptr;
}
extern "C" tfs_device_error* tfs_comm_error(tfs_comm* c, int32_t local) {
  return (c && local >= 0 && local < c->nlocal) ? c->d_err[local] : nullptr;
}

extern "C" int32_t tfs_comm_destroy(tfs_comm* c) {
  if (!c) return TFS_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < c->R; ++r)
    if (c->opened[r]) cudaIpcCloseMemHandle(c->bases[r]);
  for (char* h : c->heaps) cudaFree(h);
  for (auto p : c->d_bases) cudaFree(p);
  delete c;
  return TFS_OK;
}

// ===================================================================================== stepper
namespace {

struct Dims {
  int64_t V, B, S, Seff, M, shard_rows;
  int32_t d, R;
  bool full, sharded_full, bf16;
  int64_t cap_e, cap_w, istride, rstride, off_w, off_b;
};

Dims dims_of(const tfs_step_config* c) {
  Dims m{};
  m.V = c->vocab;
  m.d = c->dim;
  m.R = c->num_shards;
  m.B = c->tokens;
  m.S = c->num_sampled;
  m.full = c->num_sampled == 0;
  m.sharded_full = m.full && m.R > 1;
  m.Seff = m.full ? (m.R == 1 ? m.V : 0) : m.S;  // candidate rows gathered per replica
  m.M = m.R * m.B;
  m.shard_rows = cdiv(m.V, m.R);
  m.bf16 = c->operand_dtype == TFS_BF16;
  if (m.R > 1) {
    const int64_t ne = m.B, nw = m.sharded_full ? 0 : m.B + m.S;
    m.cap_e = c->cap_e > 0 ? std::min(c->cap_e, ne) : ne;
    m.cap_w = m.sharded_full ? 0 : (c->cap_w > 0 ? std::min(c->cap_w, nw) : nw);
    m.istride = m.cap_e + m.cap_w;
    m.off_w = m.cap_e * m.d;
    m.off_b = (m.cap_e + m.cap_w) * m.d;
    m.rstride = cdiv((m.cap_e + m.cap_w) * m.d + m.cap_w, 4) * 4;  // 16-byte aligned regions
  }
  return m;
}

// Symmetric heap layout (identical on every rank: it depends on the config only).
struct HeapLayout {
  size_t E, W, b, ids, grads, Wm, hsym, ysym, rowstats, dh_part, loss_part, total;
};
HeapLayout heap_layout(const Dims& m) {
  Carver c(nullptr, 0);
  c.take<char>(kHeapHeader);
  HeapLayout L{};
  auto off = [&](size_t bytes) {
    c.take<char>(0);
    const size_t o = (c.used + 255) & ~size_t(255);
    c.take<char>(bytes);
    return o;
  };
  L.E = off(sizeof(float) * m.shard_rows * m.d);
  L.W = off(sizeof(float) * m.shard_rows * m.d);
  L.b = off(sizeof(float) * m.shard_rows);
  L.ids = off(sizeof(int64_t) * m.R * std::max<int64_t>(m.istride, 1));
  L.grads = off(sizeof(float) * m.R * std::max<int64_t>(m.rstride, 4));
  // sampled softmax over R > 1 shards, bf16 operands: the bf16 mirror of W the requesters pull
  // (half the NVLink bytes of pulling fp32 rows; every owner update rewrites its rows)
  if (m.R > 1 && !m.sharded_full && m.bf16 && m.d % 8 == 0)
    L.Wm = off(sizeof(uint16_t) * m.shard_rows * m.d);
  if (m.sharded_full) {
    L.hsym = off(2 * m.B * m.d);
    L.ysym = off(sizeof(int64_t) * m.B);
    L.rowstats = off(sizeof(float) * 2 * m.M);
    L.dh_part = off(sizeof(float) * m.M * m.d);
    L.loss_part = off(16);
  }
  L.total = (c.used + 4095) & ~size_t(4095);
  return L;
}

struct BufInfo {
  void* p = nullptr;
  int64_t n = 0;
  int32_t t = 0;
};

enum Ev { kFork, kH, kQ, kPlanW, kOwn, kSsm, kRedE, kB2, kSideDone, kMainDone, kBar, kCommit,
          kSmp, kRows, kPushW, kNumEv };

struct Rank {
  int r = 0;           // global rank
  int64_t nloc = 0;    // rows of this shard
  cudaStream_t main = nullptr, side = nullptr;  // main: caller's stream (nlocal == 1) or own
  cudaStream_t smp = nullptr;                    // draws the NEXT step's candidates
  bool own_main = false;
  cudaEvent_t ev[kNumEv] = {};
  BufInfo buf[TFS_BUF_COUNT_];
  char* block = nullptr;  // one cudaMalloc of the non-symmetric buffers
  // tables
  float *E = nullptr, *W = nullptr, *b = nullptr, *sE = nullptr, *sW = nullptr, *sb = nullptr;
  // per step
  int64_t *x = nullptr, *y = nullptr, *qw = nullptr, *num_tries = nullptr, *step = nullptr;
  int64_t* counts = nullptr;
  float *les = nullptr, *ley = nullptr;
  void *h = nullptr, *w_rows = nullptr;
  float *b_rows = nullptr, *loss = nullptr, *lse = nullptr, *loss_sum = nullptr;
  float *dh = nullptr, *dw = nullptr, *db = nullptr;
  tfs_device_error* err = nullptr;
  void *smp_state = nullptr, *smp_ws = nullptr;
  int64_t *s_next = nullptr, *T_next = nullptr, *step_next = nullptr;  // drawn one step ahead
  float* les_next = nullptr;
  size_t smp_ws_b = 0;
  int64_t max_draws = 0;
  void* ws_ssm = nullptr;
  size_t ws_ssm_b = 0;
  // R = 1 plans
  void *plan_e = nullptr, *plan_w = nullptr, *apws_e = nullptr, *apws_w = nullptr;
  size_t plan_e_b = 0, plan_w_b = 0, apws_e_b = 0, apws_w_b = 0;
  // R > 1
  int64_t* recv_ids = nullptr;
  float* recv_grads = nullptr;
  uint16_t* Wm = nullptr;      // bf16 mirror of this shard's W (heap; R > 1 sampled path)
  int64_t* tab_Wm = nullptr;   // the owners' mirrors
  int64_t *tab_E = nullptr, *tab_W = nullptr, *tab_b = nullptr, *tab_ids = nullptr,
          *tab_grads = nullptr;
  void *rplan_e = nullptr, *rplan_w = nullptr, *rws_e = nullptr, *rws_w = nullptr;
  size_t rplan_e_b = 0, rplan_w_b = 0, rws_e_b = 0, rws_w_b = 0;
  void *oplan_e = nullptr, *oplan_w = nullptr, *ows_e = nullptr, *ows_w = nullptr;
  size_t oplan_e_b = 0, oplan_w_b = 0, ows_e_b = 0, ows_w_b = 0;
  // sharded full softmax
  uint16_t *hsym = nullptr, *h_all = nullptr, *W_bf = nullptr;
  int64_t *ysym = nullptr, *y_all = nullptr, *ag_ids = nullptr, *cand = nullptr;
  float *rowstats = nullptr, *lse_all = nullptr, *dh_part = nullptr, *dw_full = nullptr,
        *db_full = nullptr, *z_label = nullptr, *loss_part = nullptr;
  int64_t *tab_h = nullptr, *tab_y = nullptr, *tab_rowstats = nullptr, *tab_dh = nullptr;
  void* ws_full = nullptr;
  size_t ws_full_b = 0;
};

}  // namespace

struct tfs_stepper {
  tfs_step_config cfg{};
  Dims m{};
  tfs_comm* comm = nullptr;
  std::vector<Rank> ranks;
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int32_t status = TFS_OK;  // first failing call of the step being issued
  cudaEvent_t origin = nullptr;
  void* const* timing = nullptr;  // caller's instrumentation events of the step being issued
  uint64_t side_delay_ns = 0;     // TFS_DEBUG_SIDE_DELAY_US (race detector)
  int32_t sm_reserve = 0;         // SMs the softmax GEMMs leave to the side streams
};

namespace {

// issue-time status: the first failure of a step wins
#define STEP_CALL(st, expr)                  \
  do {                                       \
    int32_t _s = (expr);                     \
    if (_s != TFS_OK && (st)->status == TFS_OK) (st)->status = _s; \
  } while (0)

inline int32_t rec(cudaEvent_t e, cudaStream_t s) {
  TFS_CUDA_TRY(cudaEventRecord(e, s));
  return TFS_OK;
}
inline int32_t waitev(cudaStream_t s, cudaEvent_t e) {
  TFS_CUDA_TRY(cudaStreamWaitEvent(s, e, 0));
  return TFS_OK;
}
// s2 waits for everything issued so far on s1
inline int32_t join(cudaStream_t s2, cudaStream_t s1, cudaEvent_t e) {
  int32_t x = rec(e, s1);
  if (x != TFS_OK) return x;
  return waitev(s2, e);
}
// Fork the side stream from main (+ the race detector's delay).
void fork_side(tfs_stepper* st, Rank& k, cudaStream_t mn);

void set_buf(Rank& k, int which, void* p, int64_t n, int32_t t) {
  k.buf[which].p = p;
  k.buf[which].n = n;
  k.buf[which].t = t;
}

tfs_ssm_args ssm_args(const tfs_stepper* st, const Rank& k, void* const* events) {
  const Dims& m = st->m;
  tfs_ssm_args a{};
  const size_t es = m.bf16 ? 2 : 4;
  a.B = m.B;
  a.S = m.Seff;
  a.dim = m.d;
  a.operand_dtype = st->cfg.operand_dtype;
  a.flags = m.full ? TFS_REMOVE_ACCIDENTAL_HITS : st->cfg.flags;
  if (m.bf16) a.flags |= TFS_BF16_OPERANDS;
  a.grad_scale = 1.0f / (float)(m.R * m.B);
  a.h = (const float*)k.h;
  a.labels = k.y;
  a.w_true = (const float*)k.w_rows;
  a.b_true = k.b_rows;
  a.log_ec_true = k.ley;
  a.sampled = k.qw + m.B;
  a.w_s = (const float*)((const char*)k.w_rows + es * m.B * m.d);
  a.b_s = k.b_rows + m.B;
  a.log_ec_s = k.les;
  a.loss = k.loss;
  a.lse = k.lse;
  a.loss_sum = k.loss_sum;
  a.dh = k.dh;
  a.dw_true = k.dw;
  a.db_true = k.db;
  a.dw_s = k.dw + m.B * m.d;
  a.db_s = k.db + m.B;
  a.vocab = m.V;
  a.timing_events = events;
  a.sm_reserve = st->sm_reserve;
  return a;
}

tfs_ssm_args slice_args(const tfs_stepper* st, const Rank& k, bool backward) {
  const Dims& m = st->m;
  tfs_ssm_args a{};
  a.B = m.M;
  a.S = k.nloc;
  a.dim = m.d;
  a.operand_dtype = TFS_BF16;
  a.flags = TFS_LABEL_IN_CANDIDATES | TFS_BF16_OPERANDS;
  a.grad_scale = 1.0f / (float)(m.R * m.B);
  a.h = (const float*)k.h_all;
  a.labels = k.y_all;
  a.sampled = k.cand;
  a.w_s = (const float*)k.W_bf;
  a.b_s = k.b;
  a.vocab = m.V;
  a.sm_reserve = st->sm_reserve;
  if (backward) {
    a.lse = k.lse_all;
    a.dh = k.dh_part;
    a.dw_s = k.dw_full;
    a.db_s = k.db_full;
  }
  return a;
}

// The candidates of a step depend on (seed, step, replica) only (R-7, R-17), so each step draws
// the NEXT step's sample on its own stream, concurrently with its softmax, and commits the
// ahead-drawn sample at its start (tfs_sample_commit: copies + the labels' log expected counts).
// `add` = 1: draw for the step after the current counter (the pipelined case); 0: prime the
// pipeline for the current counter (create / set_counter / sync).
int32_t presample(tfs_stepper* st, Rank& k, cudaStream_t s, int64_t add) {
  const Dims& m = st->m;
  if (m.full) return TFS_OK;
  ::tfs::launch(next_counter_kernel, 1, 1, 0, s, k.step, k.step_next, add);
  launched();
  TFS_LAUNCH_CHECK();
  return tfs_log_uniform_sample(k.smp_state, m.V, (int32_t)m.S, st->cfg.unique, k.max_draws,
                                st->cfg.seed, 0, (const uint64_t*)k.step_next, (uint32_t)k.r,
                                nullptr, 0, k.s_next, k.les_next, nullptr, k.T_next, k.smp_ws,
                                k.smp_ws_b, k.err, s);
}

int32_t commit(tfs_stepper* st, Rank& k, cudaStream_t s) {
  const Dims& m = st->m;
  if (m.full) return TFS_OK;
  // also writes y into qw[0, B): the lookup ids y || s in one buffer (no separate copy)
  return tfs_sample_commit(m.V, (int32_t)m.S, st->cfg.unique, k.s_next, k.les_next, k.T_next,
                           k.y, m.B, k.qw + m.B, k.les, k.ley, k.num_tries, k.qw, k.err, s);
}

// At the start of a step: commit this step's sample, then fork the next step's draw.
void sample_phase(tfs_stepper* st, Rank& k, cudaStream_t mn) {
  if (st->m.full) return;
  STEP_CALL(st, commit(st, k, mn));
  STEP_CALL(st, join(k.smp, mn, k.ev[kCommit]));
  STEP_CALL(st, presample(st, k, k.smp, 1));
  STEP_CALL(st, rec(k.ev[kSmp], k.smp));
}
void sample_join(tfs_stepper* st, Rank& k, cudaStream_t mn) {
  if (!st->m.full) STEP_CALL(st, waitev(mn, k.ev[kSmp]));
}

int32_t apply_local(tfs_stepper* st, Rank& k, bool e_table, cudaStream_t s) {
  const Dims& m = st->m;
  const tfs_step_config& c = st->cfg;
  if (e_table) {
    if (c.optimizer == 0)
      return tfs_scatter_add_sgd_planned(k.E, m.V, m.d, k.plan_e, k.plan_e_b, m.B, k.dh, c.lr,
                                         nullptr, nullptr, k.apws_e, k.apws_e_b, s);
    const tfs_sparse_opt o{c.optimizer, c.lr, c.momentum, k.sE, nullptr};
    return tfs_scatter_opt_planned(k.E, m.V, m.d, k.plan_e, k.plan_e_b, m.B, k.dh, nullptr,
                                   nullptr, &o, k.apws_e, k.apws_e_b, s);
  }
  const int64_t n = m.B + m.Seff;
  if (c.optimizer == 0)
    return tfs_scatter_add_sgd_planned(k.W, m.V, m.d, k.plan_w, k.plan_w_b, n, k.dw, c.lr, k.b,
                                       k.db, k.apws_w, k.apws_w_b, s);
  const tfs_sparse_opt o{c.optimizer, c.lr, c.momentum, k.sW, k.sb};
  return tfs_scatter_opt_planned(k.W, m.V, m.d, k.plan_w, k.plan_w_b, n, k.dw, k.b, k.db, &o,
                                 k.apws_w, k.apws_w_b, s);
}

int32_t apply_owner(tfs_stepper* st, Rank& k, bool e_table, cudaStream_t s) {
  const Dims& m = st->m;
  const tfs_step_config& c = st->cfg;
  const tfs_sparse_opt o{c.optimizer, c.lr, c.momentum, e_table ? k.sE : k.sW,
                         e_table ? nullptr : k.sb, e_table ? nullptr : k.Wm};
  if (e_table)
    return tfs_scatter_opt_planned_slots(k.E, k.nloc, m.d, k.oplan_e, k.oplan_e_b, m.R, m.cap_e,
                                         k.recv_grads, m.rstride, nullptr, nullptr, 0, &o,
                                         k.ows_e, k.ows_e_b, s);
  return tfs_scatter_opt_planned_slots(k.W, k.nloc, m.d, k.oplan_w, k.oplan_w_b, m.R, m.cap_w,
                                       k.recv_grads + m.off_w, m.rstride, k.b,
                                       k.recv_grads + m.off_b, m.rstride, &o, k.ows_w, k.ows_w_b,
                                       s);
}

void fork_side(tfs_stepper* st, Rank& k, cudaStream_t mn) {
  STEP_CALL(st, join(k.side, mn, k.ev[kFork]));
  if (st->side_delay_ns) {
    ::tfs::launch(delay_kernel, 1, 1, 0, k.side, st->side_delay_ns);
    launched();
  }
}

// ---------------------------------------------------------------------------------- R = 1
// The embedding lookup (E) and the softmax-row lookup (W, b) are independent until the
// sampled softmax, and so are their updates afterwards: the E path runs on the side stream.
// With one shard Part / Stitch are identities (every Gather writes rows in their final
// place); the ScatterAdd plans (stable id sorts) depend on the ids only and are built on the
// side stream while the main stream samples, gathers and runs the softmax.
void local_step(tfs_stepper* st, Rank& k, cudaStream_t mn) {
  const Dims& m = st->m;
  cudaStream_t sd = k.side;
  const int32_t rdt = m.bf16 ? TFS_BF16 : TFS_F32;
  fork_side(st, k, mn);
  STEP_CALL(st, tfs_gather(k.E, m.V, m.d, TFS_F32, k.x, m.B, k.h, rdt, k.err, sd));
  STEP_CALL(st, rec(k.ev[kH], sd));
  STEP_CALL(st, tfs_scatter_plan(k.x, m.B, m.V, k.plan_e, k.plan_e_b, k.err, sd));
  if (m.full &&  // (the sampled path: the commit writes y into qw)
      cudaMemcpyAsync(k.qw, k.y, sizeof(int64_t) * m.B, cudaMemcpyDeviceToDevice, mn) != cudaSuccess)
    st->status = st->status ? st->status : TFS_ERR_CUDA;
  if (TFS_PRESAMPLE_LATE) {  // A/B: the next step's draw forked at rows-ready instead
    if (!m.full) STEP_CALL(st, commit(st, k, mn));
  } else {
    sample_phase(st, k, mn);
  }
  STEP_CALL(st, rec(k.ev[kQ], mn));
  STEP_CALL(st, waitev(sd, k.ev[kQ]));
  STEP_CALL(st, tfs_scatter_plan(k.qw, m.B + m.Seff, m.V, k.plan_w, k.plan_w_b, k.err, sd));
  STEP_CALL(st, rec(k.ev[kPlanW], sd));
  STEP_CALL(st, tfs_gather2(k.W, m.V, m.d, k.b, k.qw, m.B + m.Seff, k.w_rows, rdt, k.b_rows,
                            k.err, mn));
  STEP_CALL(st, waitev(mn, k.ev[kH]));
  tfs_ssm_args a = ssm_args(st, k, nullptr);
  // the softmax-row gradients are final before the call's last pass (the dh split-K
  // reduction): the W / b update starts then, on the side stream (after its plan), while the
  // main stream finishes dh and updates E (its plan was built on the side stream before W's)
  a.rows_ready_event = k.ev[kRows];
  STEP_CALL(st, tfs_sampled_softmax_fwd_bwd(&a, k.ws_ssm, k.ws_ssm_b, mn));
  STEP_CALL(st, waitev(sd, k.ev[kRows]));
  if (TFS_PRESAMPLE_LATE && !m.full) {
    STEP_CALL(st, waitev(k.smp, k.ev[kRows]));
    STEP_CALL(st, presample(st, k, k.smp, 1));
    STEP_CALL(st, rec(k.ev[kSmp], k.smp));
  }
  if (st->side_delay_ns) {  // race detector: the side-stream W update starts late too
    ::tfs::launch(delay_kernel, 1, 1, 0, sd, st->side_delay_ns);
    launched();
  }
  STEP_CALL(st, apply_local(st, k, false, sd));
  STEP_CALL(st, waitev(mn, k.ev[kPlanW]));
  STEP_CALL(st, apply_local(st, k, true, mn));
  STEP_CALL(st, join(mn, sd, k.ev[kSideDone]));
  sample_join(st, k, mn);
}

// The same step on one stream, its phases bracketed by the caller's events (instrumentation).
void local_step_serial(tfs_stepper* st, Rank& k, cudaStream_t mn, void* const* ev) {
  const Dims& m = st->m;
  const int32_t rdt = m.bf16 ? TFS_BF16 : TFS_F32;
  auto mark = [&](int i) {
    if (ev && ev[i]) STEP_CALL(st, rec((cudaEvent_t)ev[i], mn));
  };
  mark(0);
  if (m.full &&
      cudaMemcpyAsync(k.qw, k.y, sizeof(int64_t) * m.B, cudaMemcpyDeviceToDevice, mn) != cudaSuccess)
    st->status = st->status ? st->status : TFS_ERR_CUDA;
  STEP_CALL(st, commit(st, k, mn));       // this step's sample (drawn ahead) ...
  STEP_CALL(st, presample(st, k, mn, 1)); // ... and the next step's draw, inline here
  mark(1);
  STEP_CALL(st, tfs_gather(k.E, m.V, m.d, TFS_F32, k.x, m.B, k.h, rdt, k.err, mn));
  mark(2);
  STEP_CALL(st, tfs_gather2(k.W, m.V, m.d, k.b, k.qw, m.B + m.Seff, k.w_rows, rdt, k.b_rows,
                            k.err, mn));
  mark(3);
  tfs_ssm_args a = ssm_args(st, k, ev ? ev + 9 : nullptr);
  STEP_CALL(st, tfs_sampled_softmax_fwd_bwd(&a, k.ws_ssm, k.ws_ssm_b, mn));
  mark(4);
  STEP_CALL(st, tfs_scatter_plan(k.x, m.B, m.V, k.plan_e, k.plan_e_b, k.err, mn));
  mark(5);
  STEP_CALL(st, tfs_scatter_plan(k.qw, m.B + m.Seff, m.V, k.plan_w, k.plan_w_b, k.err, mn));
  mark(6);
  STEP_CALL(st, apply_local(st, k, true, mn));
  mark(7);
  STEP_CALL(st, apply_local(st, k, false, mn));
  mark(8);
}

void mark(tfs_stepper* st, int i, cudaStream_t s) {
  if (st->timing && st->timing[i]) STEP_CALL(st, rec((cudaEvent_t)st->timing[i], s));
}

// ------------------------------------------------------------------------------ R > 1 phases
// A phase issues rank k's work between two barriers; barrier[p] names the stream the barrier
// after phase p orders (0 = main, 1 = side).
struct PhasePlan {
  int nphase;
  int barrier_stream[8];
};

// Sampled softmax over one-sided NVLink:
//  phase 0: (nothing; B0 = previous updates done everywhere, inboxes free)
//  phase 1: pull h, W, b rows from the owners' shards (Part + route + owner Gather + Stitch in
//           one kernel); push the distinct ids into the owners' id inboxes     -> B1 (side)
//  phase 2: owners plan their inbox (merge of R ascending runs) on the side stream; softmax;
//           per-id gradient sums pushed into the owners' gradient inboxes      -> B2 (main)
//  phase 3: owners apply their planned ScatterAdd-SGD (E on the side stream, W + b on main)
const PhasePlan kP2P = {4, {0, 1, 0}};

void p2p_phase(tfs_stepper* st, Rank& k, int phase, cudaStream_t mn) {
  const Dims& m = st->m;
  cudaStream_t sd = k.side;
  const int R = m.R, rank = k.r;
  const int32_t rdt = m.bf16 ? TFS_BF16 : TFS_F32;
  const int64_t io = rank * m.istride, ro = rank * m.rstride;
  switch (phase) {
    case 0:
      mark(st, 0, mn);
      break;
    case 1:
      mark(st, 1, mn);  // B0 passed
      fork_side(st, k, mn);
      STEP_CALL(st, tfs_gather_peers((const float* const*)k.tab_E, m.shard_rows, m.d, k.x, m.B,
                                     m.V, R, k.h, rdt, k.err, sd));
      STEP_CALL(st, rec(k.ev[kH], sd));
      STEP_CALL(st, tfs_route_plan_push(k.x, m.B, m.V, R, m.cap_e, k.rplan_e, k.rplan_e_b,
                                        (int64_t* const*)k.tab_ids, io, k.counts, k.err, sd));
      if (m.full && cudaMemcpyAsync(k.qw, k.y, sizeof(int64_t) * m.B, cudaMemcpyDeviceToDevice,
                                    mn) != cudaSuccess)
        st->status = st->status ? st->status : TFS_ERR_CUDA;
      sample_phase(st, k, mn);
      mark(st, 2, mn);  // sample committed
      STEP_CALL(st, rec(k.ev[kQ], mn));
      STEP_CALL(st, waitev(sd, k.ev[kQ]));
      STEP_CALL(st, tfs_route_plan_push(k.qw, m.B + m.S, m.V, R, m.cap_w, k.rplan_w, k.rplan_w_b,
                                        (int64_t* const*)k.tab_ids, io + m.cap_e, k.counts + R,
                                        k.err, sd));
      STEP_CALL(st, rec(k.ev[kPlanW], sd));  // main's W gradient push reads this plan
      mark(st, 17, sd);  // side: pushes issued (before B1)
      break;
    case 2: {
      mark(st, 18, sd);  // side: B1 passed
      STEP_CALL(st, tfs_scatter_plan_slots(k.recv_ids, m.istride, R, m.cap_e, k.nloc, 1,
                                           k.oplan_e, k.oplan_e_b, k.err, sd));
      STEP_CALL(st, tfs_scatter_plan_slots(k.recv_ids + m.cap_e, m.istride, R, m.cap_w, k.nloc,
                                           1, k.oplan_w, k.oplan_w_b, k.err, sd));
      STEP_CALL(st, rec(k.ev[kOwn], sd));
      mark(st, 19, sd);  // side: owner plans built
      if (k.tab_Wm)  // bf16 rows straight from the owners' mirrors
        STEP_CALL(st, tfs_gather_peers2_bf16((const uint16_t* const*)k.tab_Wm, m.shard_rows,
                                             m.d, (const float* const*)k.tab_b, k.qw, m.B + m.S,
                                             m.V, R, (uint16_t*)k.w_rows, k.b_rows, k.err, mn));
      else
        STEP_CALL(st, tfs_gather_peers2((const float* const*)k.tab_W, m.shard_rows, m.d,
                                        (const float* const*)k.tab_b, k.qw, m.B + m.S, m.V, R,
                                        k.w_rows, rdt, k.b_rows, k.err, mn));
      mark(st, 3, mn);  // W rows pulled
      STEP_CALL(st, waitev(mn, k.ev[kH]));
      tfs_ssm_args a = ssm_args(st, k, st->timing ? st->timing + 9 : nullptr);
      // The W / b gradients are final before the softmax call's last pass (the dh split-K
      // reduction): outside instrumented steps their push runs on the sampler stream (idle by
      // then) from that point, overlapping dh's reduction and the E push on the main stream.
      // Both pushes stay off the side stream: B2 then does not wait for the side stream's owner
      // plans (which the persistent softmax GEMMs delay: they hold every SM).
      const bool split_push = st->timing == nullptr;
      if (split_push) a.rows_ready_event = k.ev[kRows];
      STEP_CALL(st, tfs_sampled_softmax_fwd_bwd(&a, k.ws_ssm, k.ws_ssm_b, mn));
      STEP_CALL(st, waitev(mn, k.ev[kPlanW]));  // the E and W route plans (side, phase 1)
      cudaStream_t ws = split_push ? k.smp : mn;
      if (split_push) {
        STEP_CALL(st, waitev(ws, k.ev[kRows]));
        STEP_CALL(st, waitev(ws, k.ev[kPlanW]));
        if (st->side_delay_ns) {  // race detector: the push starts late too
          ::tfs::launch(delay_kernel, 1, 1, 0, ws, st->side_delay_ns);
          launched();
        }
      }
      STEP_CALL(st, tfs_route_reduce_push(k.rplan_w, k.rplan_w_b, m.B + m.S, m.V, R, m.cap_w,
                                          k.dw, m.d, k.db, (float* const*)k.tab_grads,
                                          ro + m.off_w, (float* const*)k.tab_grads, ro + m.off_b,
                                          k.rws_w, k.rws_w_b, ws));
      if (split_push) STEP_CALL(st, rec(k.ev[kPushW], ws));
      mark(st, 4, mn);  // W gradients pushed
      STEP_CALL(st, tfs_route_reduce_push(k.rplan_e, k.rplan_e_b, m.B, m.V, R, m.cap_e, k.dh, m.d,
                                          nullptr, (float* const*)k.tab_grads, ro, nullptr, 0,
                                          k.rws_e, k.rws_e_b, mn));
      if (split_push) STEP_CALL(st, waitev(mn, k.ev[kPushW]));  // B2 orders both pushes
      mark(st, 20, mn);  // E gradients pushed
      break;
    }
    case 3:
      mark(st, 5, mn);  // B2 passed
      STEP_CALL(st, rec(k.ev[kB2], mn));
      STEP_CALL(st, waitev(sd, k.ev[kB2]));
      STEP_CALL(st, apply_owner(st, k, true, sd));
      STEP_CALL(st, waitev(mn, k.ev[kOwn]));
      STEP_CALL(st, apply_owner(st, k, false, mn));
      mark(st, 6, mn);  // W updated
      STEP_CALL(st, join(mn, sd, k.ev[kSideDone]));
      sample_join(st, k, mn);
      mark(st, 7, mn);  // E updated too (side joined)
      break;
  }
}

// Vocabulary-sharded full softmax ("the multiplication and gradient calculation are
// colocated with the shards"): W and b never move.
//  phase 0: (B0)
//  phase 1: pull h rows from the E owners (bf16); push the distinct x ids to them   -> B1
//  phase 2: owners plan the E inbox (side); all-gather h and y by peer loads into
//           [R B x d], [R B]; this shard's per-token (max, sum 2^x) pairs            -> B2
//  phase 3: lse of all R B tokens from the R pairs (rank order, the same everywhere);
//           G = c (p - onehot) on this shard's classes: its dh partial, dW / db of its
//           classes (dense SGD on the side stream), the loss of the labels it owns  -> B3
//  phase 4: pull and sum this rank's tokens' dh partials (rank order); per-id dh sums pushed
//           to the E owners                                                          -> B4
//  phase 5: E owners apply their planned ScatterAdd-SGD
const PhasePlan kFull = {6, {0, 0, 0, 0, 0}};

void full_phase(tfs_stepper* st, Rank& k, int phase, cudaStream_t mn) {
  const Dims& m = st->m;
  cudaStream_t sd = k.side;
  const int R = m.R, rank = k.r;
  const float lr = st->cfg.lr;
  switch (phase) {
    case 0:
      break;
    case 1:
      fork_side(st, k, mn);
      STEP_CALL(st, tfs_route_plan_push(k.x, m.B, m.V, R, m.cap_e, k.rplan_e, k.rplan_e_b,
                                        (int64_t* const*)k.tab_ids, rank * m.istride, k.counts,
                                        k.err, sd));
      STEP_CALL(st, rec(k.ev[kQ], sd));
      STEP_CALL(st, tfs_gather_peers((const float* const*)k.tab_E, m.shard_rows, m.d, k.x, m.B,
                                     m.V, R, k.hsym, TFS_BF16, k.err, mn));
      if (cudaMemcpyAsync(k.ysym, k.y, sizeof(int64_t) * m.B, cudaMemcpyDeviceToDevice, mn) !=
          cudaSuccess)
        st->status = st->status ? st->status : TFS_ERR_CUDA;
      STEP_CALL(st, waitev(mn, k.ev[kQ]));
      break;
    case 2: {
      STEP_CALL(st, join(sd, mn, k.ev[kH]));
      STEP_CALL(st, tfs_scatter_plan_slots(k.recv_ids, m.istride, R, m.cap_e, k.nloc, 1,
                                           k.oplan_e, k.oplan_e_b, k.err, sd));
      STEP_CALL(st, rec(k.ev[kOwn], sd));
      // all-gathers of h (bf16, as float words) and y (int64, as float pairs): bit copies
      STEP_CALL(st, tfs_gather_peers((const float* const*)k.tab_h, m.B, m.d / 2, k.ag_ids, m.M,
                                     m.M, R, k.h_all, TFS_F32, k.err, mn));
      STEP_CALL(st, tfs_gather_peers((const float* const*)k.tab_y, m.B, 2, k.ag_ids, m.M, m.M, R,
                                     k.y_all, TFS_F32, k.err, mn));
      tfs_ssm_args a = slice_args(st, k, false);
      mark(st, 9, mn);
      STEP_CALL(st, tfs_ssm_partial_stats(&a, k.rowstats, k.ws_full, k.ws_full_b, mn));
      mark(st, 10, mn);
      break;
    }
    case 3: {
      STEP_CALL(st, tfs_lse_combine_peers((const float* const*)k.tab_rowstats, R, m.M, k.lse_all,
                                          mn));
      tfs_ssm_args a = slice_args(st, k, true);
      mark(st, 11, mn);
      STEP_CALL(st, tfs_ssm_backward_from_lse(&a, k.z_label, k.ws_full, k.ws_full_b, mn));
      mark(st, 12, mn);
      STEP_CALL(st, tfs_label_loss_sum(k.lse_all, k.z_label, k.y_all, m.M, R, rank,
                                       1.0f / (float)(R * m.B), k.loss_part, mn));
      STEP_CALL(st, rec(k.ev[kSsm], mn));
      STEP_CALL(st, waitev(sd, k.ev[kSsm]));
      STEP_CALL(st, tfs_dense_sgd(k.W, k.dw_full, k.nloc * m.d, lr, k.W_bf, sd));
      STEP_CALL(st, tfs_dense_sgd(k.b, k.db_full, k.nloc, lr, nullptr, sd));
      break;
    }
    case 4:
      STEP_CALL(st, tfs_reduce_peers((const float* const*)k.tab_dh, R, (int64_t)rank * m.B * m.d,
                                     m.B * m.d, k.dh, mn));
      if (cudaMemcpyAsync(k.loss_sum, k.loss_part, sizeof(float), cudaMemcpyDeviceToDevice, mn) !=
          cudaSuccess)
        st->status = st->status ? st->status : TFS_ERR_CUDA;
      STEP_CALL(st, tfs_route_reduce_push(k.rplan_e, k.rplan_e_b, m.B, m.V, R, m.cap_e, k.dh, m.d,
                                          nullptr, (float* const*)k.tab_grads,
                                          rank * m.rstride, nullptr, 0, k.rws_e, k.rws_e_b, mn));
      break;
    case 5:
      STEP_CALL(st, waitev(mn, k.ev[kOwn]));
      STEP_CALL(st, apply_owner(st, k, true, mn));
      STEP_CALL(st, join(mn, sd, k.ev[kSideDone]));
      break;
  }
}

int32_t bump_step(Rank& k, cudaStream_t mn) {
  ::tfs::launch(add_i64_kernel, 1, 1, 0, mn, k.step, 1);
  launched();
  TFS_LAUNCH_CHECK();
  return TFS_OK;
}

// Barrier after a phase: a device barrier (one process per GPU) or stream ordering across the
// local ranks (simulated ranks on one GPU).
void barrier(tfs_stepper* st, int channel, int which_stream, std::vector<cudaStream_t>& mains) {
  tfs_comm* c = st->comm;
  const size_t nl = st->ranks.size();
  auto stream_of = [&](size_t l) { return which_stream ? st->ranks[l].side : mains[l]; };
  if (c->nlocal == 1) {
    Rank& k = st->ranks[0];
    ::tfs::launch(barrier_kernel, 1, 64, 0, stream_of(0), c->d_bases[0], c->R, k.r, channel, c->d_epoch[0],
                                               c->d_err[0], c->timeout_ns);
    launched();
    if (cudaGetLastError() != cudaSuccess && st->status == TFS_OK) st->status = TFS_ERR_CUDA;
    return;
  }
  for (size_t l = 0; l < nl; ++l) STEP_CALL(st, rec(st->ranks[l].ev[kBar], stream_of(l)));
  // every local rank's stream waits for every local rank's event
  for (size_t l = 0; l < nl; ++l)
    for (size_t q = 0; q < nl; ++q) STEP_CALL(st, waitev(stream_of(l), st->ranks[q].ev[kBar]));
}

// Issue one step of every local rank with `origin` as the caller's stream.
int32_t issue_step(tfs_stepper* st, cudaStream_t origin, void* const* timing) {
  st->status = TFS_OK;
  st->timing = timing;
  const Dims& m = st->m;
  const size_t nl = st->ranks.size();
  std::vector<cudaStream_t> mains(nl);
  if (nl == 1) {
    mains[0] = origin;
  } else {
    STEP_CALL(st, rec(st->origin, origin));
    for (size_t l = 0; l < nl; ++l) {
      mains[l] = st->ranks[l].main;
      STEP_CALL(st, waitev(mains[l], st->origin));
    }
  }
  if (m.R == 1) {
    Rank& k = st->ranks[0];
    if (timing) local_step_serial(st, k, mains[0], timing);
    else local_step(st, k, mains[0]);
    STEP_CALL(st, bump_step(k, mains[0]));
    return st->status;
  }
  const PhasePlan& P = m.sharded_full ? kFull : kP2P;
  for (int p = 0; p < P.nphase; ++p) {
    for (size_t l = 0; l < nl; ++l) {
      if (m.sharded_full) full_phase(st, st->ranks[l], p, mains[l]);
      else p2p_phase(st, st->ranks[l], p, mains[l]);
    }
    if (p + 1 < P.nphase) barrier(st, p, P.barrier_stream[p], mains);
  }
  for (size_t l = 0; l < nl; ++l) STEP_CALL(st, bump_step(st->ranks[l], mains[l]));
  if (nl > 1)
    for (size_t l = 0; l < nl; ++l) STEP_CALL(st, join(origin, mains[l], st->ranks[l].ev[kMainDone]));
  return st->status;
}

void free_rank(Rank& k) {
  for (int i = 0; i < kNumEv; ++i)
    if (k.ev[i]) cudaEventDestroy(k.ev[i]);
  if (k.side) cudaStreamDestroy(k.side);
  if (k.smp) cudaStreamDestroy(k.smp);
  if (k.own_main && k.main) cudaStreamDestroy(k.main);
  if (k.block) cudaFree(k.block);
}

}  // namespace

namespace {
// Draw the sample of the CURRENT step counter into the ahead buffers (create, set_counter,
// sync): the first step's commit then finds it there.
int32_t prime(tfs_stepper* st) {
  for (auto& k : st->ranks) {
    int32_t r = presample(st, k, k.smp, 0);
    if (r != TFS_OK) return r;
  }
  for (auto& k : st->ranks) TFS_CUDA_TRY(cudaStreamSynchronize(k.smp));
  return TFS_OK;
}
}  // namespace

extern "C" size_t tfs_step_heap_bytes(const tfs_step_config* cfg) {
  if (!cfg || cfg->num_shards < 1) return 0;
  return heap_layout(dims_of(cfg)).total;
}

extern "C" int32_t tfs_step_destroy(tfs_stepper* st) {
  if (!st) return TFS_OK;
  cudaDeviceSynchronize();
  if (st->exec) cudaGraphExecDestroy(st->exec);
  if (st->graph) cudaGraphDestroy(st->graph);
  if (st->cap_stream) cudaStreamDestroy(st->cap_stream);
  if (st->origin) cudaEventDestroy(st->origin);
  for (auto& k : st->ranks) free_rank(k);
  delete st;
  return TFS_OK;
}

extern "C" int32_t tfs_step_create(const tfs_step_config* cfg, tfs_comm* comm, tfs_stepper** out) {
  TFS_REQUIRE(cfg && out);
  const Dims m = dims_of(cfg);
  TFS_REQUIRE(m.V >= 1 && m.V < (1ll << 31) - 1 && m.d >= 1 && m.B >= 1 && m.S >= 0 && m.R >= 1);
  TFS_REQUIRE(cfg->operand_dtype == TFS_BF16 || cfg->operand_dtype == TFS_F32);
  TFS_REQUIRE(cfg->optimizer >= 0 && cfg->optimizer <= 2);
  TFS_REQUIRE(m.R == 1 || (comm && comm->R == m.R && comm->connected));
  TFS_REQUIRE(m.R == 1 || m.bf16);                       // the R > 1 paths pull bf16 rows
  TFS_REQUIRE(!m.sharded_full || (cfg->optimizer == 0 && m.d % 64 == 0));
  TFS_REQUIRE(!cfg->unique || m.full || m.S <= m.V);
  TFS_REQUIRE(m.R == 1 || comm->heap_bytes >= heap_layout(m).total);
  TFS_SUPPORTED();
  tfs_stepper* st = new tfs_stepper();
  st->cfg = *cfg;
  // The softmax's persistent GEMMs hold every SM they run on; leaving a few to the side
  // streams lets the plans / pushes / owner plans progress during the GEMMs (R > 1, where the
  // side work is on the critical path).  A tuning constant (A/B: profiles/r2_summary.md).
  st->sm_reserve = m.R > 1 ? TFS_STEP_SM_RESERVE_R : TFS_STEP_SM_RESERVE_1;
  if (const char* dly = std::getenv("TFS_DEBUG_SIDE_DELAY_US"))
    st->side_delay_ns = (uint64_t)std::strtoull(dly, nullptr, 10) * 1000ull;
  st->m = m;
  st->comm = comm;
  const int nl = (m.R == 1) ? 1 : comm->nlocal;
  st->ranks.resize(nl);
  const HeapLayout HL = heap_layout(m);
  auto bail = [&](int32_t s) {
    tfs_step_destroy(st);
    return s;
  };
  if (cudaStreamCreateWithFlags(&st->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&st->origin, cudaEventDisableTiming) != cudaSuccess)
    return bail(TFS_ERR_CUDA);
  const int32_t rdt_bytes = m.bf16 ? 2 : 4;
  const int64_t B = m.B, d = m.d, V = m.V, R = m.R;
  const int64_t nq = m.sharded_full ? B : B + m.Seff;  // ids looked up in W per replica
  for (int l = 0; l < nl; ++l) {
    Rank& k = st->ranks[l];
    k.r = (m.R == 1) ? 0 : comm->first + l;
    k.nloc = cdiv(V - k.r, R);
    // The side streams (plans, pushes, owner plans, the E path; the sampler ahead) get the
    // highest priority: the softmax's persistent GEMMs hold every SM while they run, so side
    // work only runs at the main stream's kernel boundaries -- where it should go first.
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    const int prio_side = TFS_SIDE_PRIO_HI ? prio_hi : prio_lo;
    if (cudaStreamCreateWithPriority(&k.side, cudaStreamNonBlocking, prio_side) != cudaSuccess ||
        cudaStreamCreateWithPriority(&k.smp, cudaStreamNonBlocking, prio_side) != cudaSuccess)
      return bail(TFS_ERR_CUDA);
    if (nl > 1) {
      if (cudaStreamCreateWithFlags(&k.main, cudaStreamNonBlocking) != cudaSuccess)
        return bail(TFS_ERR_CUDA);
      k.own_main = true;
    }
    for (int i = 0; i < kNumEv; ++i)
      if (cudaEventCreateWithFlags(&k.ev[i], cudaEventDisableTiming) != cudaSuccess)
        return bail(TFS_ERR_CUDA);
    // ---- sizes of the non-symmetric block
    int64_t md = 0;
    const size_t smp_state_b = m.full ? 0 : tfs_sampler_state_bytes(V);
    const size_t ssm_b = m.sharded_full ? 0 : tfs_ssm_workspace_bytes(B, m.Seff, (int32_t)d,
                                                                      cfg->operand_dtype, V);
    Carver c(nullptr, 0);
    auto plan_sizes = [&](Carver& cv, bool carve) {
      (void)carve;
      cv.take<char>(ssm_b);                         // ws_ssm (zeroed: candidate map head)
      cv.take<int64_t>(B);                          // x
      cv.take<int64_t>(B);                          // y
      cv.take<int64_t>(B + m.Seff);                 // qw
      cv.take<int64_t>(8);                          // num_tries, step, err(2)
      cv.take<int64_t>(2 * R);                      // counts
      cv.take<float>(std::max<int64_t>(m.Seff, 1)); // les
      cv.take<float>(B);                            // ley
      cv.take<char>(rdt_bytes * B * d);             // h
      cv.take<char>(rdt_bytes * (B + m.Seff) * d);  // w_rows
      cv.take<float>(B + m.Seff);                   // b_rows
      cv.take<float>(B);                            // loss
      cv.take<float>(B);                            // lse
      cv.take<float>(4);                            // loss_sum
      cv.take<float>(B * d);                        // dh
      cv.take<float>((B + m.Seff) * d);             // dw
      cv.take<float>(B + m.Seff);                   // db
      cv.take<char>(smp_state_b);
      cv.take<int64_t>(std::max<int64_t>(m.S, 1));  // s_next
      cv.take<float>(std::max<int64_t>(m.S, 1));    // les_next
      cv.take<int64_t>(4);                          // T_next, step_next
    };
    plan_sizes(c, false);
    // the rest is carved after the sizes of plans / workspaces are known
    k.max_draws = 0;
    size_t extra = 0;
    if (m.R == 1) {
      k.plan_e_b = tfs_scatter_plan_bytes(B);
      k.plan_w_b = tfs_scatter_plan_bytes(B + m.Seff);
      k.apws_e_b = tfs_scatter_apply_workspace_bytes(B, (int32_t)d);
      k.apws_w_b = tfs_scatter_apply_workspace_bytes(B + m.Seff, (int32_t)d);
      extra += k.plan_e_b + k.plan_w_b + k.apws_e_b + k.apws_w_b + 4 * 256;
      if (m.R == 1) {
        // tables (R = 1: plain device memory)
        extra += 2 * sizeof(float) * V * d + sizeof(float) * V + 3 * 256;
      }
    } else {
      k.rplan_e_b = tfs_route_plan_bytes(B, (int32_t)R);
      k.rws_e_b = tfs_route_reduce_workspace_bytes(B, (int32_t)d);
      k.oplan_e_b = tfs_scatter_plan_bytes(R * m.cap_e);
      k.ows_e_b = tfs_scatter_apply_workspace_bytes(R * m.cap_e, (int32_t)d);
      extra += k.rplan_e_b + k.rws_e_b + k.oplan_e_b + k.ows_e_b + 4 * 256;
      if (!m.sharded_full) {
        k.rplan_w_b = tfs_route_plan_bytes(B + m.S, (int32_t)R);
        k.rws_w_b = tfs_route_reduce_workspace_bytes(B + m.S, (int32_t)d);
        k.oplan_w_b = tfs_scatter_plan_bytes(R * m.cap_w);
        k.ows_w_b = tfs_scatter_apply_workspace_bytes(R * m.cap_w, (int32_t)d);
        extra += k.rplan_w_b + k.rws_w_b + k.oplan_w_b + k.ows_w_b + 4 * 256;
      }
      extra += 5 * sizeof(int64_t) * R + 5 * 256;  // peer tables
      if (m.sharded_full) {
        k.ws_full_b = tfs_ssm_workspace_bytes(m.M, k.nloc, (int32_t)d, TFS_BF16, V);
        extra += k.ws_full_b + 2 * m.M * d + sizeof(int64_t) * (2 * m.M + k.nloc) +
                 2 * k.nloc * d + sizeof(float) * (3 * m.M + k.nloc * d + k.nloc) +
                 4 * sizeof(int64_t) * R + 16 * 256;
      }
    }
    if (cfg->optimizer != 0) {
      const int64_t rows = (m.R == 1) ? V : k.nloc;
      extra += sizeof(float) * (2 * rows * d + rows) + 3 * 256;
    }
    const size_t total = c.used + extra + 4096;
    if (cudaMalloc(&k.block, total) != cudaSuccess) {
      set_last_error("cudaMalloc(step block)", cudaGetLastError());
      return bail(TFS_ERR_CUDA);
    }
    if (cudaMemset(k.block, 0, total) != cudaSuccess) return bail(TFS_ERR_CUDA);
    Carver cv(k.block, total);
    k.ws_ssm = cv.take<char>(ssm_b);
    k.ws_ssm_b = ssm_b;
    k.x = cv.take<int64_t>(B);
    k.y = cv.take<int64_t>(B);
    k.qw = cv.take<int64_t>(B + m.Seff);
    int64_t* misc = cv.take<int64_t>(8);
    k.num_tries = misc;
    k.step = misc + 1;
    k.err = reinterpret_cast<tfs_device_error*>(misc + 2);
    k.counts = cv.take<int64_t>(2 * R);
    k.les = cv.take<float>(std::max<int64_t>(m.Seff, 1));
    k.ley = cv.take<float>(B);
    k.h = cv.take<char>(rdt_bytes * B * d);
    k.w_rows = cv.take<char>(rdt_bytes * (B + m.Seff) * d);
    k.b_rows = cv.take<float>(B + m.Seff);
    k.loss = cv.take<float>(B);
    k.lse = cv.take<float>(B);
    k.loss_sum = cv.take<float>(4);
    k.dh = cv.take<float>(B * d);
    k.dw = cv.take<float>((B + m.Seff) * d);
    k.db = cv.take<float>(B + m.Seff);
    k.smp_state = smp_state_b ? (void*)cv.take<char>(smp_state_b) : nullptr;
    k.s_next = cv.take<int64_t>(std::max<int64_t>(m.S, 1));
    k.les_next = cv.take<float>(std::max<int64_t>(m.S, 1));
    k.T_next = cv.take<int64_t>(4);
    k.step_next = k.T_next + 1;
    if (m.R == 1) {
      k.plan_e = cv.take<char>(k.plan_e_b);
      k.plan_w = cv.take<char>(k.plan_w_b);
      k.apws_e = cv.take<char>(k.apws_e_b);
      k.apws_w = cv.take<char>(k.apws_w_b);
      k.E = cv.take<float>(V * d);
      k.W = cv.take<float>(V * d);
      k.b = cv.take<float>(V);
    } else {
      char* heap = comm->heaps[l];
      k.E = reinterpret_cast<float*>(heap + HL.E);
      k.W = reinterpret_cast<float*>(heap + HL.W);
      k.b = reinterpret_cast<float*>(heap + HL.b);
      k.recv_ids = reinterpret_cast<int64_t*>(heap + HL.ids);
      k.recv_grads = reinterpret_cast<float*>(heap + HL.grads);
      k.rplan_e = cv.take<char>(k.rplan_e_b);
      k.rws_e = cv.take<char>(k.rws_e_b);
      k.oplan_e = cv.take<char>(k.oplan_e_b);
      k.ows_e = cv.take<char>(k.ows_e_b);
      if (!m.sharded_full) {
        k.rplan_w = cv.take<char>(k.rplan_w_b);
        k.rws_w = cv.take<char>(k.rws_w_b);
        k.oplan_w = cv.take<char>(k.oplan_w_b);
        k.ows_w = cv.take<char>(k.ows_w_b);
      }
      // peer pointer tables: base[q] + offset of the buffer
      auto table = [&](size_t off) {
        int64_t* t = cv.take<int64_t>(R);
        std::vector<int64_t> h(R);
        for (int q = 0; q < R; ++q) h[q] = (int64_t)(uintptr_t)comm->bases[q] + (int64_t)off;
        cudaMemcpy(t, h.data(), sizeof(int64_t) * R, cudaMemcpyHostToDevice);
        return t;
      };
      k.tab_E = table(HL.E);
      k.tab_W = table(HL.W);
      if (HL.Wm) {
        k.Wm = reinterpret_cast<uint16_t*>(heap + HL.Wm);
        k.tab_Wm = table(HL.Wm);
      }
      k.tab_b = table(HL.b);
      k.tab_ids = table(HL.ids);
      k.tab_grads = table(HL.grads);
      if (m.sharded_full) {
        k.hsym = reinterpret_cast<uint16_t*>(heap + HL.hsym);
        k.ysym = reinterpret_cast<int64_t*>(heap + HL.ysym);
        k.rowstats = reinterpret_cast<float*>(heap + HL.rowstats);
        k.dh_part = reinterpret_cast<float*>(heap + HL.dh_part);
        k.loss_part = reinterpret_cast<float*>(heap + HL.loss_part);
        k.tab_h = table(HL.hsym);
        k.tab_y = table(HL.ysym);
        k.tab_rowstats = table(HL.rowstats);
        k.tab_dh = table(HL.dh_part);
        k.ws_full = cv.take<char>(k.ws_full_b);
        k.h_all = cv.take<uint16_t>(m.M * d);
        k.y_all = cv.take<int64_t>(m.M);
        k.ag_ids = cv.take<int64_t>(m.M);
        k.cand = cv.take<int64_t>(k.nloc);
        k.W_bf = cv.take<uint16_t>(k.nloc * d);
        k.lse_all = cv.take<float>(m.M);
        k.dw_full = cv.take<float>(k.nloc * d);
        k.db_full = cv.take<float>(k.nloc);
        k.z_label = cv.take<float>(m.M);
        ::tfs::launch(index_map_kernel, grid1d(m.M), 256, 0, 0, k.ag_ids, m.M, 1, 0, 0, B, R);
        ::tfs::launch(index_map_kernel, grid1d(k.nloc), 256, 0, 0, k.cand, k.nloc, 0, R, k.r, B, R);
        launched(2);
      }
    }
    if (cfg->optimizer != 0) {
      const int64_t rows = (m.R == 1) ? V : k.nloc;
      k.sE = cv.take<float>(rows * d);
      k.sW = cv.take<float>(rows * d);
      k.sb = cv.take<float>(rows);
    }
    if (!cv.fits()) return bail(TFS_ERR_INVALID_ARGUMENT);
    // ---- one-off initialisation
    const tfs_device_error none{0, 0, INT64_MAX};
    if (cudaMemcpy(k.err, &none, sizeof(none), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(TFS_ERR_CUDA);
    if (!m.full) {
      int32_t s = tfs_sampler_init(V, (int32_t)m.S, cfg->unique, k.smp_state, &md, nullptr);
      if (s != TFS_OK) return bail(s);
      k.max_draws = md;
      k.smp_ws_b = tfs_sampler_workspace_bytes(md);
      if (cudaMalloc(&k.smp_ws, k.smp_ws_b) != cudaSuccess) return bail(TFS_ERR_CUDA);
    } else if (m.R == 1) {  // candidates = all V classes, no correction (config F)
      ::tfs::launch(index_map_kernel, grid1d(V), 256, 0, 0, k.qw + B, V, 0, 1, 0, B, R);
      ::tfs::launch(fill_i64_kernel, 1, 1, 0, 0, k.num_tries, 1, V);
      launched(2);
    }
    if (cfg->optimizer == 2) {
      const int64_t rows = (m.R == 1) ? V : k.nloc;
      std::vector<float> init(1 << 20, cfg->adagrad_init);
      for (float* p : {k.sE, k.sW, k.sb}) {
        const int64_t n = (p == k.sb) ? rows : rows * d;
        for (int64_t o = 0; o < n; o += (int64_t)init.size())
          cudaMemcpy(p + o, init.data(), sizeof(float) * std::min<int64_t>(init.size(), n - o),
                     cudaMemcpyHostToDevice);
      }
    }
    // ---- named buffers
    const int32_t F = 0, BF = 1, I = 2;
    const int64_t rows = (m.R == 1) ? V : k.nloc;
    set_buf(k, TFS_BUF_E, k.E, rows * d, F);
    set_buf(k, TFS_BUF_W, k.W, rows * d, F);
    set_buf(k, TFS_BUF_B, k.b, rows, F);
    set_buf(k, TFS_BUF_SLOT_E, k.sE, k.sE ? rows * d : 0, F);
    set_buf(k, TFS_BUF_SLOT_W, k.sW, k.sW ? rows * d : 0, F);
    set_buf(k, TFS_BUF_SLOT_B, k.sb, k.sb ? rows : 0, F);
    set_buf(k, TFS_BUF_X, k.x, B, I);
    set_buf(k, TFS_BUF_Y, k.y, B, I);
    set_buf(k, TFS_BUF_QW, k.qw, B + m.Seff, I);
    set_buf(k, TFS_BUF_LOG_EC_S, k.les, m.Seff, F);
    set_buf(k, TFS_BUF_LOG_EC_Y, k.ley, B, F);
    set_buf(k, TFS_BUF_NUM_TRIES, k.num_tries, 1, I);
    set_buf(k, TFS_BUF_H, m.sharded_full ? (void*)k.hsym : k.h, B * d,
            m.sharded_full ? BF : (m.bf16 ? BF : F));
    set_buf(k, TFS_BUF_W_ROWS, k.w_rows, (B + m.Seff) * d, m.bf16 ? BF : F);
    set_buf(k, TFS_BUF_B_ROWS, k.b_rows, B + m.Seff, F);
    set_buf(k, TFS_BUF_LOSS, k.loss, B, F);
    set_buf(k, TFS_BUF_LSE, k.lse, B, F);
    set_buf(k, TFS_BUF_LOSS_SUM, k.loss_sum, 1, F);
    set_buf(k, TFS_BUF_DH, k.dh, B * d, F);
    set_buf(k, TFS_BUF_DW, k.dw, (B + m.Seff) * d, F);
    set_buf(k, TFS_BUF_DB, k.db, B + m.Seff, F);
    set_buf(k, TFS_BUF_ERR, k.err, 2, I);
    set_buf(k, TFS_BUF_STEP, k.step, 1, I);
    set_buf(k, TFS_BUF_COUNTS, k.counts, 2 * R, I);
    (void)nq;
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(TFS_ERR_CUDA);
  int32_t pr = prime(st);
  if (pr != TFS_OK) return bail(pr);
  *out = st;
  return TFS_OK;
}

extern "C" int32_t tfs_step_buffer(tfs_stepper* st, int32_t local, int32_t which, void** ptr,
                                   int64_t* numel, int32_t* elem_type) {
  TFS_REQUIRE(st && local >= 0 && local < (int32_t)st->ranks.size() && which >= 0 &&
              which < TFS_BUF_COUNT_);
  const BufInfo& b = st->ranks[local].buf[which];
  if (ptr) *ptr = b.p;
  if (numel) *numel = b.n;
  if (elem_type) *elem_type = b.t;
  return TFS_OK;
}

extern "C" int32_t tfs_step_sync(tfs_stepper* st) {
  TFS_REQUIRE(st);
  const tfs_device_error none{0, 0, INT64_MAX};
  for (auto& k : st->ranks) {
    if (k.W_bf) {
      ::tfs::launch(f32_to_bf16_kernel, grid1d(k.nloc * st->m.d), 256, 0, 0, k.W, k.nloc * st->m.d, k.W_bf);
      launched();
    }
    if (k.Wm) {
      ::tfs::launch(f32_to_bf16_kernel, grid1d(k.nloc * st->m.d), 256, 0, 0, k.W, k.nloc * st->m.d, k.Wm);
      launched();
    }
    TFS_CUDA_TRY(cudaMemcpy(k.err, &none, sizeof(none), cudaMemcpyHostToDevice));
  }
  if (st->comm)
    for (int l = 0; l < st->comm->nlocal; ++l)
      TFS_CUDA_TRY(cudaMemcpy(st->comm->d_err[l], &none, sizeof(none), cudaMemcpyHostToDevice));
  TFS_CUDA_TRY(cudaDeviceSynchronize());
  return prime(st);
}

extern "C" int32_t tfs_step_set_counter(tfs_stepper* st, int64_t value) {
  TFS_REQUIRE(st && value >= 0);
  TFS_CUDA_TRY(cudaDeviceSynchronize());
  for (auto& k : st->ranks)
    TFS_CUDA_TRY(cudaMemcpy(k.step, &value, sizeof(int64_t), cudaMemcpyHostToDevice));
  return prime(st);
}

extern "C" int32_t tfs_step_run(tfs_stepper* st, const tfs_step_io* io, void* stream) {
  TFS_REQUIRE(st);
  cudaStream_t s = as_stream(stream);
  const Dims& m = st->m;
  const size_t nl = st->ranks.size();
  void* const* timing = io ? io->timing_events : nullptr;
  TFS_REQUIRE(!timing || (nl == 1 && !st->exec));
  if (io && io->x && io->y) {
    const cudaMemcpyKind kind = io->host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    for (size_t l = 0; l < nl; ++l) {
      Rank& k = st->ranks[l];
      const int64_t* xs = io->x + l * m.B;
      const int64_t* ys = io->y + l * m.B;
      if (nl == 1 && ys == xs + m.B && k.y == k.x + m.B) {  // adjacent: one copy of x || y
        if (xs != k.x)
          TFS_CUDA_TRY(cudaMemcpyAsync(k.x, xs, 2 * sizeof(int64_t) * m.B, kind, s));
        continue;
      }
      if (xs != k.x) TFS_CUDA_TRY(cudaMemcpyAsync(k.x, xs, sizeof(int64_t) * m.B, kind, s));
      if (ys != k.y) TFS_CUDA_TRY(cudaMemcpyAsync(k.y, ys, sizeof(int64_t) * m.B, kind, s));
    }
  }
  if (st->exec) {
    TFS_CUDA_TRY(cudaGraphLaunch(st->exec, s));
  } else {
    int32_t r = issue_step(st, s, timing);
    if (r != TFS_OK) return r;
  }
  if (io && io->host && io->loss_host)
    for (size_t l = 0; l < nl; ++l)
      TFS_CUDA_TRY(cudaMemcpyAsync(io->loss_host + l, st->ranks[l].loss_sum, sizeof(float),
                                   cudaMemcpyDeviceToHost, s));
  return TFS_OK;
}

extern "C" int32_t tfs_step_capture(tfs_stepper* st) {
  TFS_REQUIRE(st);
  tfs_step_uncapture(st);
  TFS_CUDA_TRY(cudaDeviceSynchronize());
  TFS_CUDA_TRY(cudaStreamBeginCapture(st->cap_stream, cudaStreamCaptureModeRelaxed));
  int32_t r = issue_step(st, st->cap_stream, nullptr);
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(st->cap_stream, &g);
  if (r != TFS_OK) {
    if (g) cudaGraphDestroy(g);
    return r;
  }
  if (e != cudaSuccess) {
    set_last_error("cudaStreamEndCapture", e);
    return TFS_ERR_CUDA;
  }
  st->graph = g;
  TFS_CUDA_TRY(cudaGraphInstantiate(&st->exec, g, 0));
  return TFS_OK;
}

extern "C" int32_t tfs_step_uncapture(tfs_stepper* st) {
  TFS_REQUIRE(st);
  if (st->exec) cudaGraphExecDestroy(st->exec);
  if (st->graph) cudaGraphDestroy(st->graph);
  st->exec = nullptr;
  st->graph = nullptr;
  return TFS_OK;
}

extern "C" int64_t tfs_step_graph_kernels(tfs_stepper* st) {
  if (!st || !st->graph) return 0;
  size_t n = 0;
  if (cudaGraphGetNodes(st->graph, nullptr, &n) != cudaSuccess) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(st->graph, nodes.data(), &n) != cudaSuccess) return 0;
  int64_t k = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}
