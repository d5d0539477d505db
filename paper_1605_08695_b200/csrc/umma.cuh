// umma.cuh -- hand-written sm_100a tensor-core GEMM (tcgen05.mma + TMEM + TMA + mbarriers) with
// the sampled-softmax epilogues fused in.  C[m, n] = sum_k A(m, k) * B(n, k), bf16 operands,
// fp32 accumulation in TMEM.  Each operand is either K-major (row-major [rows x K]) or
// MN-major (row-major [K x rows]: the transposed view), selected per launch, so the softmax
// backward reads G, W_s and h in the layout they already have -- no transposed copies.
//
// CTA = 12 warps, persistent over (m-tile, n-tile, k-split) units:
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
// tile, log2 domain), GRAD (G = c exp(Z - lse) -> bf16 G + column sums for db), STORE (fp32).
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
                              256 /*barriers*/;

__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn) {
  return (1u << 4)                       // D format f32
         | (1u << 7)                     // A format bf16
         | (1u << 10)                    // B format bf16
         | ((a_mn ? 1u : 0u) << 15)      // A major (0 = K, 1 = MN)
         | ((b_mn ? 1u : 0u) << 16)      // B major
         | ((uint32_t)(BN >> 3) << 17)   // N
         | ((uint32_t)(BM >> 4) << 24);  // M
}

enum Mode : int { kStats = 0, kGrad = 1, kStore = 2 };

struct Shape {
  int M, N, K;
  int num_m, num_n, ksplit, kb_per_split, kb_total;
  int num_units;
};

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
  float* dbs_part;   // GRAD: [(4*num_m) x N] column sums of bf16(G)
  float* out;        // STORE: fp32, out[ks * split_stride + m * ldo + n]
  int64_t ldo;
  int64_t split_stride;
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
template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int k16) {
  // K advance of 16 elements: +32 B inside the swizzled row (K-major), +16 rows (MN-major).
  return MN ? desc_sw128(base + (uint32_t)k16 * 2048u, kMNBoxBytes, 1024)
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
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
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
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void decode_unit(const Shape& g, int u, int& mt, int& nt, int& ks,
                                            int& kb0, int& kb1) {
  ks = u % g.ksplit;
  const int r = u / g.ksplit;
  mt = r % g.num_m;
  nt = r / g.num_m;
  kb0 = ks * g.kb_per_split;
  kb1 = min(g.kb_total, kb0 + g.kb_per_split);
}

// Sum over the 32 lanes of v[i] for every i; afterwards lane l holds the sum for column l.
// Fixed butterfly order (deterministic): stage W halves the live values and the lane group.
template <int W>
__device__ __forceinline__ void transpose_reduce_stage(float (&v)[32], int lane) {
  const bool upper = (lane & W) != 0;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const float send = upper ? v[i] : v[i + W];
    const float keep = upper ? v[i + W] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, W);
  }
}
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
  transpose_reduce_stage<16>(v, lane);
  transpose_reduce_stage<8>(v, lane);
  transpose_reduce_stage<4>(v, lane);
  transpose_reduce_stage<2>(v, lane);
  transpose_reduce_stage<1>(v, lane);
  return v[0];
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

template <int MODE, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                Shape g, EpiParams ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + STAGES * (A_BYTES + B_BYTES));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

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
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
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
      for (int u = blockIdx.x; u < g.num_units; u += gridDim.x) {
        int mt, nt, ks, kb0, kb1;
        decode_unit(g, u, mt, nt, ks, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_expect_tx(full + stage, A_BYTES + B_BYTES);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * B_BYTES;
          if (A_MN) {
#pragma unroll
            for (int q = 0; q < BM / kMNBox; ++q)
              tma_load_2d(a + q * kMNBoxBytes, &tmA, mt * BM + q * kMNBox, kb * BK, full + stage);
          } else {
            tma_load_2d(a, &tmA, kb * BK, mt * BM, full + stage);
          }
          if (B_MN) {
#pragma unroll
            for (int q = 0; q < BN / kMNBox; ++q)
              tma_load_2d(b + q * kMNBoxBytes, &tmB, nt * BN + q * kMNBox, kb * BK, full + stage);
          } else {
            tma_load_2d(b, &tmB, kb * BK, nt * BN, full + stage);
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
      constexpr uint32_t idesc = make_idesc(A_MN, B_MN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = blockIdx.x; u < g.num_units; u += gridDim.x) {
        int mt, nt, ks, kb0, kb1;
        decode_unit(g, u, mt, nt, ks, kb0, kb1);
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, operand_desc<A_MN>(a0, k), operand_desc<B_MN>(b0, k), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
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
    for (int u = blockIdx.x; u < g.num_units; u += gridDim.x) {
      int mt, nt, ks, kb0, kb1;
      decode_unit(g, u, mt, nt, ks, kb0, kb1);
      const int row = mt * BM + quarter * 32 + lane;
      const bool row_ok = row < g.M;
      int32_t y = -2;
      float lse2 = 0.f;
      if (MODE != kStore && row_ok) y = ep.y[row];
      if (MODE == kGrad && row_ok) lse2 = ep.lse[row] * kLog2e;
      float run_m = -INFINITY, run_s = 0.f;

      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int ct = half * 128 + c * 32;  // column within the tile
        const int col0 = nt * BN + ct;
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + ct), v);
        if (MODE == kStats) {
          corrected_logits(ep, col0, y, v);
          float m4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            m4[q] = fmaxf(fmaxf(fmaxf(v[q], v[q + 4]), fmaxf(v[q + 8], v[q + 12])),
                          fmaxf(fmaxf(v[q + 16], v[q + 20]), fmaxf(v[q + 24], v[q + 28])));
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
          for (int i = 0; i < 16; ++i) {
            const float g0 = row_ok ? ep.c * fast_exp2(v[2 * i] - lse2) : 0.f;
            const float g1 = row_ok ? ep.c * fast_exp2(v[2 * i + 1] - lse2) : 0.f;
            packed[i] = pack_bf16x2(g0, g1);
            v[2 * i] = __uint_as_float(packed[i] << 16);              // bf16(g0) as fp32
            v[2 * i + 1] = __uint_as_float(packed[i] & 0xffff0000u);  // bf16(g1) as fp32
          }
          if (row_ok) {
            uint16_t* gr = ep.G + (int64_t)row * ep.ldG + col0;
            if (col0 + 32 <= g.N) {
              uint4* d4 = (uint4*)gr;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                d4[q] = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2],
                                   packed[4 * q + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < g.N)
                  gr[i] = (uint16_t)((i & 1) ? (packed[i >> 1] >> 16) : (packed[i >> 1] & 0xffffu));
            }
          }
          const float colsum = transpose_reduce32(v, lane);
          if (col0 + lane < g.N)
            ep.dbs_part[(int64_t)(mt * 4 + quarter) * g.N + col0 + lane] = colsum;
        } else {
          if (row_ok) {
            float* o = ep.out + (int64_t)ks * ep.split_stride + (int64_t)row * ep.ldo + col0;
            if (col0 + 32 <= g.N) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                ((float4*)o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (col0 + i < g.N) o[i] = v[i];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (MODE == kStats && row_ok)
        ep.stats[(int64_t)(nt * 2 + half) * g.M + row] = make_float2(run_m, run_s);
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

int32_t launch(int mode, Operand A, Operand B, int M, int N, int K, int ksplit,
               const EpiParams& ep, cudaStream_t st, int* ksplit_eff);

}  // namespace umma
}  // namespace tfs
