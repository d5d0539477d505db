// umma.cuh -- hand-written sm_100a tensor-core GEMM (tcgen05.mma + TMEM + TMA + mbarriers) with
// the sampled-softmax epilogues fused in.  C[m, n] = sum_k A(m, k) * B(n, k), bf16 operands,
// fp32 accumulation in TMEM.  Each operand is either K-major (row-major [rows x K]) or
// MN-major (row-major [K x rows]: the transposed view), selected per launch, so the softmax
// backward reads G, W_s and h in the layout they already have -- no transposed copies.
//
// CTA = 12 warps, persistent over (problem, m-tile, n-tile, k-split) units:
//   warp 0      TMA producer (one lane): A 128x64 and B 256x64 per stage, 128-byte swizzle,
//               4-stage smem ring guarded by full/empty mbarriers.
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma.kind::f16 (M=128, N=256, K=16) per stage
//               into one of two 256-column TMEM accumulators; tcgen05.commit frees the stage /
//               publishes the accumulator.
//   warp 2      TMEM allocator (512 columns = both accumulators).
//   warps 4-11  epilogue: warp w reads TMEM lanes 32*(w%4).. (its 32 rows), columns
//               [128*((w-4)/4), +128) in 32-column tcgen05.ld chunks, applies the fused epilogue
//               and frees the accumulator, so the epilogue of tile i overlaps the MMAs of i+1.
// Epilogue modes: STATS (row max / sum of 2^x of the corrected logits per half
// tile, log2 domain), GRAD (G = c exp(Z - lse) -> bf16 G), STORE (fp32 product; optional split
// partials, extra term and one extra column routed to its own vector -- db_s comes out of the
// dW_s GEMM as the product with a ones column appended to h).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"

namespace tfs {
namespace umma {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 128 + kEpiWarps * 32;  // 384
constexpr int A_BYTES = BM * BK * 2;            // 16 KB
constexpr int B_BYTES = BN * BK * 2;            // 32 KB
constexpr int kMNBox = 64;                      // MN-major TMA box: 64 elements (128 B) x BK rows
constexpr int kMNBoxBytes = kMNBox * BK * 2;    // 8 KB
constexpr int kTmemCols = 512;
constexpr float kLog2e = 1.4426950408889634f;
constexpr size_t kSmemBytes = 1024 /*align slack*/ + (size_t)STAGES * (A_BYTES + B_BYTES) +
                              256 /*barriers + flags*/;

__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, int n = BN) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major (0 = K, 1 = MN)
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(n >> 3) << 17)    // N (multiple of 16 for M = 128)
         | ((uint32_t)(BM >> 4) << 24);  // M
}

enum Mode : int { kStats = 0, kGrad = 1, kStore = 2 };



struct EpiParams {
  // STATS / GRAD: corrected logit in log2 units  v = acc * log2(e) + cb[n], excluded (-> -inf)
  // when sid[n] == y[m].  cb / sid are padded to a multiple of BN (cb = -inf, sid = -1).
  const float* cb;
  const int32_t* sid;
  const int32_t* y;
  float2* stats;     // STATS: [(2*num_n) x M] (max, sum of 2^(v - max)) per half tile
  const float* lse;  // GRAD: natural-log lse per row
  float c;           // GRAD: gradient scale
  uint16_t* G;       // GRAD: bf16 [M x ldG]
  int64_t ldG;
};

// One GEMM of a launch (a launch may carry two: the softmax backward runs dh and dW_s together
// so their tiles share the 148 SMs).  STORE epilogue: out[m, n] = acc (+ g[m] * bf16(wt[m, n]))
// when ksplit == 1; with K split `ksplit` ways each split writes its partial to
// part[ks][m][n] and a finalize pass adds them in split order (fixed order: deterministic).
struct Problem {
  CUtensorMap ta, tb;
  int M, N, K;
  int bn;  // tile width along N (multiple of 16, <= BN)
  int num_m, num_n, ksplit, kb_per_split, kb_total, units;
  int a_mn, b_mn;
  float* out;       // columns [0, N_out) of the product
  int64_t ldo;
  int N_out;
  float* col_out;   // optional: column col_idx of the product, one value per row
  int col_idx;
  float* part;      // [ksplit x M x N] fp32 (ksplit > 1)
  const float* g;   // optional row scale of the extra term
  const float* wt;  // optional [M x ldw] fp32 matrix of the extra term (bf16-rounded)
  int64_t ldw;
};

struct Params {
  Problem p[2];
  int nprob;
  int total_units;
  EpiParams ep;
};

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
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
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
__device__ __forceinline__ void epi_bar_sync() {  // the 8 epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
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
  r.ks = v % q.ksplit;
  const int t = v / q.ksplit;
  r.mt = t % q.num_m;
  r.nt = t / q.num_m;
  r.kb0 = r.ks * q.kb_per_split;
  r.kb1 = min(q.kb_total, r.kb0 + q.kb_per_split);
  r.nw = min(q.bn, (q.N - r.nt * q.bn + 15) & ~15);
  return r;
}

// Corrected logits of one 32-column chunk in log2 units (-inf where excluded).
__device__ __forceinline__ void corrected_logits(const EpiParams& ep, int col0, int32_t y,
                                                 float (&v)[32]) {
  const float4* cb4 = reinterpret_cast<const float4*>(ep.cb + col0);
  const int4* sid4 = reinterpret_cast<const int4*>(ep.sid + col0);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 c = __ldg(cb4 + q);
    const int4 s = __ldg(sid4 + q);
    v[4 * q + 0] = s.x == y ? -INFINITY : fmaf(v[4 * q + 0], kLog2e, c.x);
    v[4 * q + 1] = s.y == y ? -INFINITY : fmaf(v[4 * q + 1], kLog2e, c.y);
    v[4 * q + 2] = s.z == y ? -INFINITY : fmaf(v[4 * q + 2], kLog2e, c.z);
    v[4 * q + 3] = s.w == y ? -INFINITY : fmaf(v[4 * q + 3], kLog2e, c.w);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ Params P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + STAGES * (A_BYTES + B_BYTES));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const EpiParams& ep = P.ep;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < P.nprob; ++i) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&P.p[i].ta) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&P.p[i].tb) : "memory");
    }
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < P.total_units; u += gridDim.x) {
        const Unit t = decode_unit(P, u);
        const Problem& q = P.p[t.pi];
        const int bboxes = q.b_mn ? (t.nw + kMNBox - 1) / kMNBox : 0;
        const uint32_t bbytes =
            q.b_mn ? (uint32_t)(bboxes * kMNBoxBytes) : (uint32_t)(q.bn * BK * 2);
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
#ifdef TFS_EXP_NO_TMA
          mbar_expect_tx(full + stage, 0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
#endif
          mbar_expect_tx(full + stage, A_BYTES + bbytes);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * B_BYTES;
          if (q.a_mn) {
#pragma unroll
            for (int i = 0; i < BM / kMNBox; ++i)
              tma_load_2d(a + i * kMNBoxBytes, &q.ta, t.mt * BM + i * kMNBox, kb * BK, full + stage);
          } else {
            tma_load_2d(a, &q.ta, kb * BK, t.mt * BM, full + stage);
          }
          if (q.b_mn) {
            for (int i = 0; i < bboxes; ++i)
              tma_load_2d(b + i * kMNBoxBytes, &q.tb, t.nt * q.bn + i * kMNBox, kb * BK,
                          full + stage);
          } else {
            tma_load_2d(b, &q.tb, kb * BK, t.nt * q.bn, full + stage);
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
    if (lane == 0) {
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = blockIdx.x; u < P.total_units; u += gridDim.x) {
        const Unit t = decode_unit(P, u);
        const bool amn = P.p[t.pi].a_mn != 0, bmn = P.p[t.pi].b_mn != 0;
        const uint32_t idesc = make_idesc(amn, bmn, t.nw);
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = t.kb0; kb < t.kb1; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#ifndef TFS_EXP_NO_MMA
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, operand_desc(amn, a0, k), operand_desc(bmn, b0, k), idesc,
                      (kb > t.kb0 || k > 0) ? 1u : 0u);
#endif
          umma_commit(empty + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ================================ Epilogue ====================================
    const int ew = warp - 4;       // 0..7
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;      // column half of the 256-wide tile
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < P.total_units; u += gridDim.x) {
      const Unit t = decode_unit(P, u);
      const Problem& q = P.p[t.pi];
      const int rt = quarter * 32 + lane;  // row within the tile
      const int row = t.mt * BM + rt;
      const bool row_ok = row < q.M;
      int32_t y = -2;
      float goff = 0.f;  // GRAD: G = c 2^(v - lse log2 e) = 2^(v - goff)
      if (MODE != kStore && row_ok) y = ep.y[row];
      if (MODE == kGrad && row_ok) goff = ep.lse[row] * kLog2e - log2f(ep.c);
      float run_m = -INFINITY, run_s = 0.f;

      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
#ifdef TFS_EXP_NO_EPI
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
      continue;
#endif
      // Software-pipelined TMEM reads: chunk c+1 is in flight while chunk c is processed.
      const uint32_t tbase =
          tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + half * 128);
      uint32_t buf0[32], buf1[32];
      if (half * 128 < t.nw) tmem_ld32_nowait(tbase, buf0);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ct = half * 128 + c * 32;  // column within the tile
        const int col0 = t.nt * q.bn + ct;
        if (ct >= t.nw) break;               // beyond a narrow tile's MMA width
        // a 32-column chunk may run past this tile (bn % 32 != 0): those columns are stale TMEM
        const int nend = min(q.N, (t.nt + 1) * q.bn);
        const int nout = min(q.N_out, nend);
        const bool next = c + 1 < 4 && ct + 32 < t.nw;
        tmem_wait_ld();
        float v[32];
        if (c & 1) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(buf1[i]);
          if (next) tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), buf0);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(buf0[i]);
          if (next) tmem_ld32_nowait(tbase + (uint32_t)((c + 1) * 32), buf1);
        }
        if (MODE == kStats) {
          corrected_logits(ep, col0, y, v);
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
        } else if (MODE == kGrad) {
          corrected_logits(ep, col0, y, v);
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            packed[i] = pack_bf16x2(fast_exp2(v[2 * i] - goff), fast_exp2(v[2 * i + 1] - goff));
          if (row_ok) {
            uint16_t* gr = ep.G + (int64_t)row * ep.ldG + col0;
            if (col0 + 32 <= nend) {
              uint4* d4 = (uint4*)gr;
#pragma unroll
              for (int i = 0; i < 4; ++i)
                d4[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2],
                                   packed[4 * i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < nend)
                  gr[i] = (uint16_t)((i & 1) ? (packed[i >> 1] >> 16) : (packed[i >> 1] & 0xffffu));
            }
          }
        } else if (q.ksplit > 1) {
          // split partial, row-major [ksplit][M][N]; reduced (in split order) by a finalize pass
          if (row_ok) {
            float* o = q.part + ((int64_t)t.ks * q.M + row) * q.N + col0;
            if (col0 + 32 <= nend) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                ((float4*)o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < nend) o[i] = v[i];
            }
          }
        } else if (row_ok) {
          if (q.col_out != nullptr && q.col_idx >= col0 && q.col_idx < col0 + 32 &&
              q.col_idx < nend) {
            float xv = 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i == q.col_idx) xv = v[i];
            q.col_out[row] = xv;
          }
          if (q.g != nullptr) {
            const float gr = q.g[row];
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < nout) v[i] += gr * bf16_round(q.wt[(int64_t)row * q.ldw + col0 + i]);
          }
          float* o = q.out + (int64_t)row * q.ldo + col0;
          if (col0 + 32 <= nout) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              ((float4*)o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < nout) o[i] = v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (MODE == kStats && row_ok)
        ep.stats[(int64_t)(t.nt * 2 + half) * q.M + row] = make_float2(run_m, run_s);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---- host side ------------------------------------------------------------------------------------
// Operand view: base pointer, row stride `ld` (elements), and whether it is MN-major.  K-major:
// element (r, k) at base[r * ld + k]; MN-major: element (r, k) at base[k * ld + r].
struct Operand {
  const void* base;
  int64_t ld;
  bool mn;
};

// One GEMM to launch.  ksplit > 1 needs part (ksplit x M x N fp32).
struct Gemm {
  Operand A, B;
  int M, N, K, ksplit;
  int bn;           // tile width along N (0 = BN)
  float* out;       // columns [0, N_out)
  int64_t ldo;
  int N_out;
  float* col_out;   // optional column col_idx (one value per row)
  int col_idx;
  float* part;
  const float* g;
  const float* wt;
  int64_t ldw;
};

// Scratch size (floats) of the split partials of a GEMM.
size_t part_floats(int M, int N, int ksplit);
int tiles_of(int M, int N);
int effective_split(int K, int ksplit);

int32_t launch_stats_or_grad(int mode, Operand A, Operand B, int M, int N, int K,
                             const EpiParams& ep, cudaStream_t st);
int32_t launch_store(const Gemm* g, int count, cudaStream_t st);

}  // namespace umma
}  // namespace tfs
