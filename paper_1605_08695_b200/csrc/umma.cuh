// umma.cuh -- hand-written sm_100a tensor-core GEMM (tcgen05.mma + TMEM + TMA + mbarriers) with
// the sampled-softmax epilogues fused in.  C[m, n] = sum_k A(m, k) * B(n, k), bf16 operands,
// fp32 accumulation in TMEM.  Each operand is either K-major (row-major [rows x K]) or
// MN-major (row-major [K x rows]: the transposed view), selected per launch, so the softmax
// backward reads G, W_s and h in the layout they already have -- no transposed copies.
//
// Persistent over (problem, m-tile, n-tile, k-split) units, one CTA per SM (or one CTA pair per
// two SMs).  CTAs per tile (CT) is a template parameter chosen per launch kind: the logits
// (STATS) and gradient (GRAD) passes run one CTA per 128 x bn tile (cta_group::1); the grouped
// STORE GEMM runs CTA pairs (clusters of 2, cta_group::2): a pair owns a 256 x 256 tile, CTA r
// holding rows [128 r, +128) (its A half) and B rows [r N/2, +N/2), the leader's MMA thread
// multiplying across both CTAs' smem.  CTA = 12 warps:
//   warp 0      TMA producer (one lane): A 128 x 64 and B bn/CT x 64 tiles, 128-byte swizzle,
//               two k-blocks per stage of an mbarrier ring (as many stages as the launch's smem
//               allows); in pairs both CTAs' loads complete on the leader's full barrier.
//   warp 1      MMA issuer (one lane; the pair's leader): tcgen05.mma.cta_group::CT.kind::f16
//               (M = 128 CT, N <= 256, K = 16) into one of two 256-column TMEM accumulators;
//               tcgen05.commit releases stages / publishes the accumulator (to both CTAs).
//   warp 2      TMEM allocator (512 columns = both accumulators).
//   warps 4-11  epilogue: warp w reads TMEM lanes 32*(w%4).. (its 32 rows), columns
//               [128*((w-4)/4), +128) in 32-column tcgen05.ld chunks (double-buffered), applies
//               the fused epilogue and frees the accumulator, so the epilogue of tile i overlaps
//               the MMAs of tile i+1.  Results leave through per-warp swizzled smem slabs and
//               TMA bulk-tensor stores (full 64-byte row segments, clipped by the tensor map).
// Epilogue modes: STATS (row max / sum of 2^x of the corrected logits per half
// tile, log2 domain), GRAD (G = c exp(Z - lse) -> bf16 G), STORE (fp32 product or split-K
// partial, optional extra term g[m] * bf16(wt[m, n])).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace tfs {
namespace umma {

// CTAs per tile, per launch kind (the kernel's CT template parameter): the logits / gradient
// passes run one CTA per 128 x bn tile; the grouped STORE GEMM runs CTA pairs (cta_group::2,
// 256 x 256 tiles, each CTA loading half of B) -- measured round 2: STORE 53.2 -> 49.4 us at
// X and 1148 -> 963 us at Z with pairs, while pairs slow STATS / GRAD (31.2 -> 34.5 us at X).
#ifndef TFS_STORE_CTA
#define TFS_STORE_CTA 2
#endif
constexpr int kSoftmaxCta = 1, kStoreCta = TFS_STORE_CTA;
// Logits / gradient passes may run clusters of 2 single-CTA tiles sharing each B tile by TMA
// multicast (gemm_kernel's MC, chosen per launch by size in ssm.cu); 0: never.
#ifndef TFS_MCAST_B
#define TFS_MCAST_B 1
#endif

// TFS_SSM_ZPASS=1 builds (A/B only): the logits GEMM also stores the logits (fp32 Z, B x Spad)
// and G is formed from them in an elementwise pass instead of recomputing the logits on the
// tensor cores (the GRAD GEMM).  Measured round 2 (profiles/r2_ab_zpass.log): SLOWER -- X 186.7
// vs 184.9 us (STATS 33 -> 39 us with the store, the pass 39 us vs GRAD 36 us), Z 2691 vs 2454
// us (STATS 549 -> 724 us writing 2.2 GB, the pass 845 vs GRAD 772 us).  On B200 the recompute
// is cheaper than the logits' round trip through memory, so the product keeps it.
#ifndef TFS_SSM_ZPASS
#define TFS_SSM_ZPASS 0
#endif
static_assert(kStoreCta == 1 || kStoreCta == 2, "kStoreCta");
constexpr int BM = 128, BN = 256, BK = 64;      // BM: rows per CTA; BN: tile N
constexpr int STAGES = 4;                       // stages at the widest tile (BN); a launch with
constexpr int kMaxStages = 8;                   // narrower tiles / no staging fits more (Params)
// k-blocks per pipeline stage (one barrier pair each), per launch kind: the logits / gradient
// passes (K = d = 512: 8 k-blocks a tile) refill one k-block at a time (4-5 stages in flight),
// the long-K grouped STORE two (measured round 2, profiles/r2_ab_ksub.log).
#ifndef TFS_KSUB_SOFTMAX
#define TFS_KSUB_SOFTMAX 1
#endif
#ifndef TFS_KSUB_STORE
#define TFS_KSUB_STORE 2
#endif
__host__ __device__ constexpr int ksub_of(int mode) {
  return mode == 2 /* kStore */ ? TFS_KSUB_STORE : TFS_KSUB_SOFTMAX;
}
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + kEpiWarps * 32;  // 384
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int B_BYTES = BN * BK * 2;            // 32 KB (the widest single-CTA B stage)
constexpr int kMNBox = 64;                      // MN-major TMA box: 64 elements (128 B) x BK rows
constexpr int kMNBoxBytes = kMNBox * BK * 2;    // 8 KB
constexpr int kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// Epilogue staging: two 2 KB buffers per epilogue warp (32 rows x 64 B, 64-byte swizzle), the
// source of the TMA stores; and the column offsets cb of each (accumulator, half tile).
constexpr int kStageBytes = 2048;
constexpr int kEpiSmem = kEpiWarps * 2 * kStageBytes;  // 32 KB
constexpr int kCbSmem = 2 * 2 * 128 * 4;               // 2 KB
#ifndef TFS_URING
#define TFS_URING 3
#endif
constexpr int kURing = TFS_URING;  // unit-id ring of the dynamic schedule (scheduler -> the three roles)
constexpr int kBarBytes = 256;  // (2 kMaxStages + 4) mbarriers, the TMEM address slot, the unit ring
static_assert((2 * kMaxStages + 4) * 8 + 8 + kURing * 20 <= kBarBytes, "barrier area too small");
constexpr size_t kSmemBytes =
    (size_t)STAGES * (A_BYTES + B_BYTES) + kEpiSmem + kCbSmem + kBarBytes;  // 231680 B
static_assert(kSmemBytes <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");

// Instruction descriptor of tcgen05.mma.kind::f16: bf16 x bf16 -> f32, M = 256 (pair), N = n.
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int n, int m) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major (0 = K, 1 = MN)
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(n >> 3) << 17)    // N (multiple of 16)
         | ((uint32_t)(m >> 4) << 24);   // M (128 per CTA, 256 per pair)
}

enum Mode : int { kStats = 0, kGrad = 1, kStore = 2 };

struct EpiParams {
  // STATS / GRAD: corrected logit in log2 units  v = acc * log2(e) + cb[n], excluded (-> -inf)
  // when sid[n] == y[m].  cb / sid are padded to a multiple of BN (cb = -inf, sid = -1).
  // labels == nullptr: nothing is excluded.  Else the columns whose id equals the row's label
  // all lie in [lo, hi] from the candidate map (cmap[y] = {2^30 - lo, hi + 1}, {0, 0}: none;
  // without a map (vocab == 0) the range is every column), and the per-element id compare runs
  // only for chunks that intersect that range.
  CUtensorMap tG;      // GRAD: store map of bf16 G [M x ldG], box {32, 32}, 64-byte swizzle
  // STATS with zstore != 0: v (the corrected log2-unit logits, exclusions applied) is also
  // written to fp32 Z [M x ldz] through tZ (box {16, 32}), so the gradient pass can form G from
  // it instead of recomputing the logits GEMM (bit-identical G: same v, same arithmetic).
  CUtensorMap tZ;
  int zstore;
  const float* cb;
  const int32_t* sid;
  const int64_t* labels;
  const int2* cmap;
  int64_t vocab;
  int S_pad;
  float2* stats;       // STATS: [M x nparts] (max, sum of 2^(v - max)) per half tile
  int nparts;          // 2 * number of n-tiles
  const float* lse;    // GRAD: natural-log lse per row
  float c;             // GRAD: gradient scale
  // label_in != 0 (full softmax over a vocabulary slice): the label's column is NOT excluded;
  // STATS keeps it in the sums and GRAD writes c (p - 1) there instead of c p, and stores the
  // label's logit (natural units, bias included) to zlab[m].
  int label_in;
  float* zlab;
  // GRAD: column sums of each warp's 32-row slab of the stored (bf16) G, one fp32 partial per
  // (32-row slab, column): colpart[slab * colpart_ld + n] (slab = (m-tile * CT + rank) * 4 +
  // lane quarter); db_s = their fixed-order sum (a small finalize pass).  nullptr: no sums.
  float* colpart;
  int64_t colpart_ld;
  // Dynamic tile schedule (single-CTA tiles, no multicast; nullptr: static round robin):
  // sched[0] = claims made, sched[1] = CTAs done claiming; both zero before the launch, and
  // the last CTA done claiming zeroes them again (so a graph replays with them zero).
  unsigned* sched = nullptr;
};

// Division by a launch constant without the integer-divide sequence: the unit decode runs on
// the single producer / MMA threads at every tile boundary, where a ~40-instruction dependent
// divide chain showed as ~0.4 us per tile (role timeline, round 2).  q = (umulhi(n, mul) + n)
// >> shift, exact for n < 2^31 and 1 <= d < 2^31 (mul, shift from FastDiv::make on the host).
struct FastDiv {
  uint32_t d, mul, shift;
  static FastDiv make(uint32_t d) {
    FastDiv f{d, 0, 0};
    while ((1ull << f.shift) < d) ++f.shift;
    f.mul = (uint32_t)(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, mul) + n) >> shift);
  }
};

// One GEMM of a launch (a launch may carry two: the softmax backward runs dh and dW_s together
// so their tiles share the 148 SMs).  STORE epilogue: out[m, n] = acc (+ g[m] * bf16(wt[m, n]))
// when ksplit == 1; with K split `ksplit` ways each split writes its partial to
// part[ks][m][n] and a finalize pass adds them in split order (fixed order: deterministic).
struct Problem {
  CUtensorMap ta, tb;
  CUtensorMap to;   // STORE: fp32 out [M x ldo] (2D) or part [ksplit x M x N] (3D), box 16x32
  int M, N, K;
  int bn;  // tile width along N: a multiple of 32, <= BN (STATS / GRAD pick it to balance SMs)
  int num_m, num_n, ksplit, kb_per_split, kb_total, units;
  FastDiv fd_ks, fd_m, fd_n;  // by ksplit, num_m, num_n
  int a_mn, b_mn;
  int n_fast;       // unit order: n-tiles fastest (A larger than L2 can keep) or m-tiles fastest
  const float* g;   // optional row scale of the extra term (ksplit == 1 only)
  const void* wt;   // optional [M x ldw] matrix of the extra term: fp32 (bf16-rounded here)
  int64_t ldw;      //   or bf16 bits (wt_bf16)
  int wt_bf16;
};

// Shared-memory pipeline of a launch: `stages` ring slots of A (A_BYTES) and B (b_stride bytes:
// the widest B tile of the launch's problems, 1 KB aligned) -- as many as fit beside the
// epilogue staging (none for STATS), the column offsets and the barriers (stage_plan, host).
struct Params {
  Problem p[2];
  int nprob;
  int total_units;
  int stages;
  int b_stride;
  EpiParams ep;
};

// ---- role timeline (TFS_GEMM_TRACE builds only; results unchanged) ------------------------------
// clock64 stamps of CTA 0's roles per launch kind (tools/gemm_timeline.py prints them): slot 0
// setup done; 16+ producer stage ready; 128+ MMA tile start; 144+ MMA tile issued; 160+ MMA
// stage data arrived; 288+ / 304+ epilogue (warp 4) tile ready / done.
#ifdef TFS_GEMM_TRACE
__device__ unsigned long long g_trace[4][512];
// globaltimer (ns) of every CTA: kernel entry, setup done (after the PDL wait), exit
__device__ unsigned long long g_span[4][160][3];
#define SPAN(i)                                                                  \
  do {                                                                           \
    unsigned long long t_;                                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                       \
    if (threadIdx.x == 0 && blockIdx.x < 160) g_span[MODE][blockIdx.x][(i)] = t_; \
  } while (0)
#define TRACE(slot)                                                        \
  do {                                                                     \
    if (blockIdx.x == 0 && (slot) < 512) g_trace[MODE][(slot)] = clock64(); \
  } while (0)
#else
#define TRACE(slot) \
  do {              \
  } while (0)
#define SPAN(i) \
  do {          \
  } while (0)
#endif

// ---- PTX wrappers -----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// Pair variant: the completion goes to the LEADER CTA's mbarrier (peer bit cleared).
template <int CT>
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t leader_bar) {
  if constexpr (CT == 2) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(leader_bar)
        : "memory");
  }
}
// Multicast load: the box lands at the same smem offset in every CTA of ctaMask and each
// destination's mbarrier at offset `bar` receives the byte count.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1,
                                               uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
// Single-CTA MMAs' completion signalled on the mbarrier at this offset in every CTA of ctaMask.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
template <int CT>
__device__ __forceinline__ uint32_t cluster_ctarank() {
  if constexpr (CT == 1) return 0;
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <int CT>
__device__ __forceinline__ void cluster_sync_all() {  // both CTAs of a pair (else the CTA)
  if constexpr (CT == 2)
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  else
    __syncthreads();
}
// Arrive on the mbarrier at the same smem offset in the leader CTA (rank 0) of the pair.
template <int CT>
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  if constexpr (CT == 2) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(0));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                 : "memory");
  } else {
    mbar_arrive(bar);
  }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   (uint64_t)map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          (uint64_t)map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until at most N committed bulk stores of this thread still read their smem source.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {  // generic-proxy smem writes -> TMA
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Shared-memory matrix descriptor, 128-byte swizzle.  lbo / sbo in bytes:
//  K-major: 8-row core groups 1024 B apart (sbo); lbo unused (16 B).
//  MN-major: lbo = stride between 64-element MN blocks, sbo = stride between 8-row K groups.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t operand_desc(bool mn, uint32_t base, int k16) {
  // K advance of 16 elements: +32 B inside the swizzled row (K-major), +16 rows (MN-major).
  return mn ? desc_sw128(base + (uint32_t)k16 * 2048u, kMNBoxBytes, 1024)
            : desc_sw128(base + (uint32_t)k16 * 32u, 16, 1024);
}
template <int CT>
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::%5.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "n"(CT));
}
// Arrive (once MMAs issued so far complete) on the mbarrier at this offset (in both CTAs of a
// pair).
template <int CT>
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  if constexpr (CT == 2) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
  }
}
// tcgen05.ld of 32 consecutive accumulator columns of this warp's 32 lanes (no wait).
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
struct Unit {
  int pi, mt, nt, ks, kb0, kb1, nw;  // nw: MMA N of this tile (last n-tile may be narrower)
};
__device__ __forceinline__ Unit decode_unit(const Params& P, int u) {
  Unit r;
  r.pi = (P.nprob > 1 && u >= P.p[0].units) ? 1 : 0;
  const Problem& q = P.p[r.pi];
  const int v = r.pi ? u - P.p[0].units : u;
  // order: k-split fastest; then m-tiles (concurrent CTAs share the B tile: best while A and B
  // both stay in L2), or -- when A is too large for L2 (h and G at Z) -- n-tiles, so the
  // n-tiles of one A block run together and A comes from DRAM once (measured, round 2:
  // Z 2853 -> 2656 us per step; X 207 -> 216 us the other way round)
  const int t = (int)q.fd_ks.div((uint32_t)v);
  r.ks = v - t * q.ksplit;
  if (q.n_fast) {
    r.mt = (int)q.fd_n.div((uint32_t)t);
    r.nt = t - r.mt * q.num_n;
  } else {
    r.nt = (int)q.fd_m.div((uint32_t)t);
    r.mt = t - r.nt * q.num_m;  // m-pair index (PM rows)
  }
  r.kb0 = r.ks * q.kb_per_split;
  r.kb1 = min(q.kb_total, r.kb0 + q.kb_per_split);
  // whole 32-column chunks, so every epilogue chunk lies inside the MMA width
  r.nw = min(q.bn, (q.N - r.nt * q.bn + 31) & ~31);
  return r;
}

// One 32-row x 64-byte slab of this warp into a 64-byte-swizzled staging buffer (16-byte
// chunk k of row r lands at chunk k ^ ((r >> 1) & 3): conflict-free, the TMA SWIZZLE_64B layout).
__device__ __forceinline__ void stage_row64(uint8_t* buf, int lane, const uint4 (&x)[4]) {
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    *reinterpret_cast<uint4*>(buf + lane * 64 + ((k ^ sw) << 4)) = x[k];
}

// LAB: the label-in-candidates epilogue (EpiParams::label_in), a separate instantiation so the
// sampled-softmax kernels compile exactly as without it.
// MC = 2 (with CT = 1): clusters of two single-CTA tiles stacked along M share each B tile --
// CTA r loads B rows [r bn/2, +bn/2) and multicasts them into both CTAs' stage, so each CTA
// issues half of the B traffic; a stage is refilled once BOTH CTAs' MMAs have read it.
template <int MODE, bool LAB = false, int CT = 1, int MC = 1>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ Params P) {
  static_assert(MC == 1 || CT == 1, "multicast B is for single-CTA tiles");
  constexpr int CL = CT * MC;  // CTAs per cluster
  constexpr int PM = CL * BM;  // rows per unit
  extern __shared__ __align__(1024) uint8_t smem[];
  // PDL (common.cuh): this grid's setup (barriers, TMEM, descriptor prefetch) may overlap the
  // previous kernel's tail; its results are waited for below.
  if (TFS_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  SPAN(0);
  const int STAGES = P.stages;
  const int B_BYTES = P.b_stride;
  uint8_t* sA = smem;
  constexpr int KSUB = ksub_of(MODE);
  uint8_t* sB = smem + STAGES * KSUB * A_BYTES;
  uint8_t* sE = sB + STAGES * KSUB * B_BYTES;  // epilogue staging (STATS: only to store Z)
  float* sCb = reinterpret_cast<float*>(sE + (MODE == kStats && !TFS_SSM_ZPASS ? 0 : kEpiSmem));
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCb) + kCbSmem);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  uint64_t* ufull = tempty + 3;  // unit ring: claimed unit ids, producer -> MMA + epilogue
  uint64_t* uempty = ufull + kURing;
  volatile int* uslot = reinterpret_cast<volatile int*>(uempty + kURing);
  const EpiParams& ep = P.ep;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank<CL>();  // CT = 2: 0 = leader (issues the MMAs)
  const bool leader = CT == 1 || rank == 0;
  const int pair = blockIdx.x / CL, npairs = gridDim.x / CL;  // tile-owning CTA groups

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem) & 1023u) != 0) __trap();  // swizzled tiles need 1 KB alignment
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);   // leader: its expect_tx arrival + both CTAs' TMA bytes
      mbar_init(empty + s, MC);  // the leader's (multicast) commit; MC = 2: both CTAs' MMAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, CT * kEpiWarps);  // leader: epilogue warps of both CTAs
    }
    for (int r = 0; r < kURing; ++r) {
      mbar_init(ufull + r, 1);              // the producer's claim
      mbar_init(uempty + r, 2 + kEpiWarps);  // read by the producer, the MMA thread, every epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < P.nprob; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&P.p[i].ta) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&P.p[i].tb) : "memory");
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::%2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols), "n"(CT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::%0.sync.aligned;" ::"n"(CT));
  }
  tc_fence_before();
  cluster_sync_all<CL>();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous grid's outputs are visible
  // Unit sequence of this CTA.  Static: pair, pair + npairs, ...  Dynamic (CL == 1 and
  // ep.sched): the producer claims the next unit from the global counter when it needs one and
  // passes it through the ring, so CTAs that start late (SMs still held by side-stream kernels
  // when the GEMM launched) take fewer tiles instead of finishing last.
  const bool dyn = CL == 1 && ep.sched != nullptr;
  int u_next = pair, u_ring = 0;  // (u_next: the consumers' static sequence)
  uint32_t u_phase = 0;
  // The claims are made by a scheduler thread of its own (warp 3): the atomic's round trip
  // (~1 us with every CTA claiming at once) would otherwise stall the producer at each tile
  // boundary.  Its first unit is the CTA's index (no claim at the start), the next ones
  // npairs, npairs + 1, ... in claim order; the ring's depth bounds how far it claims ahead.
  auto take_unit = [&](bool warp_wide) -> int {  // producer / MMA thread, epilogue warp
    if (!dyn) {
      const int u = u_next;
      u_next += npairs;
      return u;
    }
    mbar_wait(ufull + u_ring, u_phase);
    const int u = uslot[u_ring];
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) mbar_arrive(uempty + u_ring);
    if (++u_ring == kURing) {
      u_ring = 0;
      u_phase ^= 1;
    }
    return u;
  };
  if (threadIdx.x == 0) TRACE(0);
  SPAN(1);

  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      int stage = 0;
      int tr_n = 0;  // (role timeline counter)
      (void)tr_n;
      uint32_t phase = 0;
      for (int u = take_unit(false); u < P.total_units; u = take_unit(false)) {
        const Unit t = decode_unit(P, u);
        const Problem& q = P.p[t.pi];
        const int nh = t.nw / CL;  // B rows this CTA loads (CT = 2: holds)
        const int bboxes = q.b_mn ? (nh + kMNBox - 1) / kMNBox : 0;
        const uint32_t bbytes = q.b_mn ? (uint32_t)(bboxes * kMNBoxBytes)
                                       : (uint32_t)((q.bn / CL) * BK * 2);  // box: bn/CL rows
        const int arow = t.mt * PM + (int)rank * BM;
        const int bcol = t.nt * q.bn + (int)rank * (MC == 2 ? q.bn / 2 : nh);
        for (int kb0 = t.kb0; kb0 < t.kb1; kb0 += KSUB) {
          const int ns = min(KSUB, t.kb1 - kb0);
          mbar_wait(empty + stage, phase ^ 1);
          TRACE(16 + tr_n++);
          // the leader's barrier (peer bit cleared)
          const uint32_t fb = smem_u32(full + stage) & (CT == 2 ? 0xFEFFFFFFu : 0xFFFFFFFFu);
          if (leader) mbar_expect_tx(full + stage, ns * (CT * A_BYTES + CL * bbytes));
          for (int sb = 0; sb < ns; ++sb) {
            const int kb = kb0 + sb;
            uint8_t* a = sA + (stage * KSUB + sb) * A_BYTES;
            uint8_t* b = sB + (stage * KSUB + sb) * B_BYTES;
            if (q.a_mn) {
#pragma unroll
              for (int i = 0; i < BM / kMNBox; ++i)
                tma_load_2d_pair<CT>(a + i * kMNBoxBytes, &q.ta, arow + i * kMNBox, kb * BK, fb);
            } else {
              tma_load_2d_pair<CT>(a, &q.ta, kb * BK, arow, fb);
            }
            if (MC == 2) {  // K-major B (STATS / GRAD): this CTA's half into both CTAs
              tma_load_2d_mc(b + (size_t)rank * (q.bn / 2) * (BK * 2), &q.tb, kb * BK, bcol,
                             full + stage, (uint16_t)3);
            } else if (q.b_mn) {
              for (int i = 0; i < bboxes; ++i)
                tma_load_2d_pair<CT>(b + i * kMNBoxBytes, &q.tb, bcol + i * kMNBox, kb * BK, fb);
            } else {
              tma_load_2d_pair<CT>(b, &q.tb, kb * BK, bcol, fb);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ==================================
    if (lane == 0 && leader) {
      int stage = 0, acc = 0;
      int tr_t = 0, tr_s = 0;  // (role timeline counters)
      (void)tr_t;
      (void)tr_s;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = take_unit(false); u < P.total_units; u = take_unit(false)) {
        const Unit t = decode_unit(P, u);
        const bool amn = P.p[t.pi].a_mn != 0, bmn = P.p[t.pi].b_mn != 0;
        const uint32_t idesc = make_idesc(amn, bmn, t.nw, CT * BM);
        mbar_wait(tempty + acc, acc_phase ^ 1);
        TRACE(128 + tr_t);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb0 = t.kb0; kb0 < t.kb1; kb0 += KSUB) {
          const int ns = min(KSUB, t.kb1 - kb0);
          mbar_wait(full + stage, phase);
          TRACE(160 + tr_s++);
          tc_fence_after();
          for (int sb = 0; sb < ns; ++sb) {
            const int kb = kb0 + sb;
            const uint32_t a0 = smem_u32(sA + (stage * KSUB + sb) * A_BYTES);
            const uint32_t b0 = smem_u32(sB + (stage * KSUB + sb) * B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16<CT>(d_tmem, operand_desc(amn, a0, k), operand_desc(bmn, b0, k), idesc,
                        (kb > t.kb0 || k > 0) ? 1u : 0u);
          }
          if (MC == 2)
            umma_commit_mc(empty + stage, (uint16_t)3);  // both CTAs may refill their halves
          else
            umma_commit_pair<CT>(empty + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair<CT>(tfull + acc);
        TRACE(144 + tr_t++);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp == 3) {
    // ============================ tile scheduler (dynamic) ========================
    if (dyn && lane == 0) {
      int r = 0;
      uint32_t ph = 0;
      for (int u = pair;; u = npairs + (int)atomicAdd(ep.sched, 1u)) {
        mbar_wait(uempty + r, ph ^ 1);
        uslot[r] = u;
        mbar_arrive(ufull + r);
        if (++r == kURing) {
          r = 0;
          ph ^= 1;
        }
        if (u >= P.total_units) break;
      }
      // this CTA's claims are all made: count it (release: after them); the last CTA to get
      // here resets the counters -- every claim of the launch is made by then, and the next
      // launch on them is ordered after this grid's completion
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                   : "=r"(prev)
                   : "l"(ep.sched + 1)
                   : "memory");
      if (prev == gridDim.x - 1) {
        atomicExch(ep.sched, 0u);
        atomicExch(ep.sched + 1, 0u);
      }
    }
  } else if (warp >= 4) {
    // ================================ Epilogue ====================================
    const int ew = warp - 4;       // 0..7
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;      // column half of the 256-wide tile
    uint8_t* stg = sE + ew * 2 * kStageBytes;
    uint32_t nst = 0;              // TMA stores issued by this warp (staging buffer parity)
    int acc = 0;
    int tr_e = 0;  // (role timeline counter)
    (void)tr_e;
    uint32_t acc_phase = 0;
    for (int u = take_unit(true); u < P.total_units; u = take_unit(true)) {
      const Unit t = decode_unit(P, u);
      const Problem& q = P.p[MODE == kStore ? t.pi : 0];
      const int M = q.M;
      const int row0 = t.mt * PM + (int)rank * BM + quarter * 32;  // this warp's 32-row slab
      const int row = row0 + lane;
      const bool row_ok = row < M;
      const int nw = t.nw;
      int32_t y = -2;
      int hlo = 1 << 30, hhi = -1;
      float goff = 0.f;  // GRAD: G = c 2^(v - lse log2 e) = 2^(v - goff)
      float* cbh = sCb + (acc * 2 + half) * 128;
      if (MODE != kStore) {
        // this half tile's 128 column offsets -> smem (each warp of the half loads 32); the
        // buffer of this accumulator was last read two tiles ago, before the previous barrier
        cbh[quarter * 32 + lane] =
            __ldg(ep.cb + t.nt * q.bn + half * 128 + quarter * 32 + lane);
        if (row_ok) {
          if (ep.labels != nullptr) {
            const int64_t yl = __ldg(ep.labels + row);
            y = (int32_t)yl;
            if (ep.cmap == nullptr) {
              hlo = 0;
              hhi = ep.S_pad;
            } else if (yl >= 0 && yl < ep.vocab) {
              const int2 m = __ldg(ep.cmap + yl);
              if (m.y > 0) {
                hlo = (1 << 30) - m.x;
                hhi = m.y - 1;
              }
            }
          }
          if (MODE == kGrad) goff = __ldg(ep.lse + row) * kLog2e - log2f(ep.c);
        }
        named_bar_sync(2 + half, 128);
      }
      float run_m = -INFINITY, run_s = 0.f;

      mbar_wait(tfull + acc, acc_phase);
      if (ew == 0 && lane == 0) TRACE(288 + tr_e);
      tc_fence_after();
      // Software-pipelined TMEM reads: chunk c+1 is in flight while chunk c is processed.
      const uint32_t tbase =
          tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + half * 128);
      uint32_t buf0[32], buf1[32];
      if (half * 128 < nw) tmem_ld32_nowait(tbase, buf0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ct = half * 128 + c * 32;  // column within the tile
        if (ct >= nw) break;                 // beyond a narrow tile's MMA width
        const int col0 = t.nt * q.bn + ct;
        const bool next = c + 1 < 4 && ct + 32 < nw;
        __syncwarp();  // tcgen05.ld / wait are .sync.aligned: the warp must be converged here
        tmem_wait_ld();
        float v[32];
        uint32_t labmask = 0;  // label_in: columns holding the row's label
        if (c & 1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(buf1[i]);
          if (next) tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), buf0);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(buf0[i]);
          if (next) tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), buf1);
        }
        if (MODE != kStore) {
          // corrected logits in log2 units; accidental hits (rare) -> -inf
          const float4* cb4 = reinterpret_cast<const float4*>(cbh + c * 32);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float4 cc = cb4[k];
            v[4 * k + 0] = fmaf(v[4 * k + 0], kLog2e, cc.x);
            v[4 * k + 1] = fmaf(v[4 * k + 1], kLog2e, cc.y);
            v[4 * k + 2] = fmaf(v[4 * k + 2], kLog2e, cc.z);
            v[4 * k + 3] = fmaf(v[4 * k + 3], kLog2e, cc.w);
          }
          const bool mine = hlo <= col0 + 31 && hhi >= col0;
          if (__any_sync(0xffffffffu, mine)) {
            if (mine) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i >= hlo && col0 + i <= hhi && __ldg(ep.sid + col0 + i) == y) {
                  if (LAB) {
                    labmask |= 1u << i;
                    if (MODE == kGrad) ep.zlab[row] = v[i] * kLn2;
                  } else {
                    v[i] = -INFINITY;
                  }
                }
            }
          }
        }
        if (MODE == kStats) {
          float m4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            m4[i] = fmaxf(fmaxf(fmaxf(v[i], v[i + 4]), fmaxf(v[i + 8], v[i + 12])),
                          fmaxf(fmaxf(v[i + 16], v[i + 20]), fmaxf(v[i + 24], v[i + 28])));
          const float cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          if (cm > -INFINITY) {
            const float nm = fmaxf(run_m, cm);
            float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < 32; ++i) s4[i & 3] += fast_exp2(v[i] - nm);
            run_s = run_s * fast_exp2(run_m - nm) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
            run_m = nm;
          }
          if (TFS_SSM_ZPASS && ep.zstore) {  // v -> Z (two 16-column halves via the slabs)
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
              uint4 x[4];
#pragma unroll
              for (int k = 0; k < 4; ++k)
                x[k] = make_uint4(__float_as_uint(v[16 * h2 + 4 * k]),
                                  __float_as_uint(v[16 * h2 + 4 * k + 1]),
                                  __float_as_uint(v[16 * h2 + 4 * k + 2]),
                                  __float_as_uint(v[16 * h2 + 4 * k + 3]));
              uint8_t* sb = stg + (nst & 1) * kStageBytes;
              if (lane == 0) bulk_wait_read<1>();
              __syncwarp();
              stage_row64(sb, lane, x);
              fence_proxy_async();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&ep.tZ, sb, col0 + 16 * h2, row0);
                bulk_commit();
              }
              ++nst;
            }
          }
        } else if (MODE == kGrad) {
          uint4 x[4];
          if (LAB) {  // G = c (p - 1) at the label's column
#pragma unroll
            for (int i = 0; i < 32; ++i)
              v[i] = fast_exp2(v[i] - goff) - (((labmask >> i) & 1u) ? ep.c : 0.f);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint32_t p[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                p[j] = pack_bf16x2(v[8 * k + 2 * j], v[8 * k + 2 * j + 1]);
              x[k] = make_uint4(p[0], p[1], p[2], p[3]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint32_t p[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                p[j] = pack_bf16x2(fast_exp2(v[8 * k + 2 * j] - goff),
                                   fast_exp2(v[8 * k + 2 * j + 1] - goff));
              x[k] = make_uint4(p[0], p[1], p[2], p[3]);
            }
          }
          uint8_t* sb = stg + (nst & 1) * kStageBytes;
          if (lane == 0) bulk_wait_read<1>();  // the store that last used this buffer has read it
          __syncwarp();
          stage_row64(sb, lane, x);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&ep.tG, sb, col0, row0);
            bulk_commit();
          }
          if (ep.colpart != nullptr && row0 < M) {  // db_s partial: column `lane` of the slab
            const int nrows = min(32, M - row0);
            const int k16 = lane >> 3, e2 = (lane & 7) * 2;
            float cs = 0.f;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const uint32_t gb =
                  *reinterpret_cast<const uint16_t*>(sb + r * 64 + ((k16 ^ ((r >> 1) & 3)) << 4) + e2);
              if (r < nrows) cs += __uint_as_float(gb << 16);
            }
            const int64_t slab = ((int64_t)t.mt * CL + rank) * 4 + quarter;
            ep.colpart[slab * ep.colpart_ld + col0 + lane] = cs;
          }
          ++nst;
        } else {
          if (q.g != nullptr && row_ok) {  // + g[row] * bf16(wt[row, col0 .. col0 + 31])
            const float gr = q.g[row];
            const int64_t w0 = (int64_t)row * q.ldw + col0;
            const int N = q.N;
            if (q.wt_bf16) {
              const uint16_t* w = static_cast<const uint16_t*>(q.wt) + w0;
              if (col0 + 32 <= N && (q.ldw & 7) == 0) {  // this row's 64 bytes: 4 vector loads
                uint4 u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) u[k] = __ldg(reinterpret_cast<const uint4*>(w) + k);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint32_t p[4] = {u[k].x, u[k].y, u[k].z, u[k].w};
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    v[8 * k + 2 * j] += gr * __uint_as_float(p[j] << 16);
                    v[8 * k + 2 * j + 1] += gr * __uint_as_float(p[j] & 0xffff0000u);
                  }
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < N) v[i] += gr * __uint_as_float((uint32_t)w[i] << 16);
              }
            } else {
              const float* w = static_cast<const float*>(q.wt) + w0;
              if (col0 + 32 <= N && (q.ldw & 3) == 0) {  // 128 bytes: 8 vector loads
                float4 f[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) f[k] = __ldg(reinterpret_cast<const float4*>(w) + k);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  v[4 * k] += gr * bf16_round(f[k].x);
                  v[4 * k + 1] += gr * bf16_round(f[k].y);
                  v[4 * k + 2] += gr * bf16_round(f[k].z);
                  v[4 * k + 3] += gr * bf16_round(f[k].w);
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (col0 + i < N) v[i] += gr * bf16_round(w[i]);
              }
            }
          }
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint4 x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              x[k] = make_uint4(__float_as_uint(v[16 * h2 + 4 * k]),
                                __float_as_uint(v[16 * h2 + 4 * k + 1]),
                                __float_as_uint(v[16 * h2 + 4 * k + 2]),
                                __float_as_uint(v[16 * h2 + 4 * k + 3]));
            uint8_t* sb = stg + (nst & 1) * kStageBytes;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            stage_row64(sb, lane, x);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (q.ksplit > 1)
                tma_store_3d(&q.to, sb, col0 + 16 * h2, row0, t.ks);
              else
                tma_store_2d(&q.to, sb, col0 + 16 * h2, row0);
              bulk_commit();
            }
            ++nst;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader<CT>(tempty + acc);  // the leader's barrier
      if (ew == 0 && lane == 0) TRACE(304 + tr_e);
      ++tr_e;
      if (MODE == kStats && row_ok)
        ep.stats[(int64_t)row * ep.nparts + t.nt * 2 + half] = make_float2(run_m, run_s);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait_read<0>();  // staging smem must outlive the last store's read
  }
  // Neither CTA may leave (or free TMEM) while its peer can still reach its smem / TMEM.
  tc_fence_before();
  cluster_sync_all<CL>();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::%2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols), "n"(CT));
  }
  SPAN(2);
}

// ---- host side ------------------------------------------------------------------------------------
// Operand view: base pointer, row stride `ld` (elements), and whether it is MN-major.  K-major:
// element (r, k) at base[r * ld + k]; MN-major: element (r, k) at base[k * ld + r].
struct Operand {
  const void* base;
  int64_t ld;
  bool mn;
};

// One GEMM to launch.  ksplit > 1 needs part (ksplit x M x N fp32).  N, ldo multiples of 4.
struct Gemm {
  Operand A, B;
  int M, N, K, ksplit;
  float* out;       // [M x ldo]
  int64_t ldo;
  float* part;
  const float* g;
  const void* wt;
  int64_t ldw;
  int wt_bf16;
};

// Scratch size (floats) of the split partials of a GEMM.
size_t part_floats(int M, int N, int ksplit);
int tiles_of(int M, int N, int ct);
int effective_split(int K, int ksplit);

// STATS / GRAD launch; for GRAD, G (bf16 [M x ldG], ldG % 8 == 0) receives the gradient.
// bn: tile width along N (pick_bn); cb / sid must be readable up to num_n * bn + 256 columns.
// STATS with ep.zstore: G / ldG are the fp32 logits buffer Z and its row stride instead.
int32_t launch_stats_or_grad(int mode, Operand A, Operand B, int M, int N, int K, int bn, int sms,
                             EpiParams ep, void* G, int64_t ldG, cudaStream_t st);
// Tile width for an M x N output of single-pass tiles: the multiple of 32 in [128, 256] that
// minimises the makespan (rounds of tiles over the CTA groups x tile width).
int pick_bn(int M, int N, int sms);
int32_t launch_store(const Gemm* g, int count, int sms, cudaStream_t st);

}  // namespace umma
}  // namespace tfs
