// common.cuh -- shared host/device helpers of libtfs (the CUDA product path).
// Nothing here is shared with oracle/ (the CPU oracle has its own code end to end).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stddef.h>

#include <utility>

#include "../../include/tfs.h"

namespace tfs {

constexpr int kNumSMsB200 = 148;

// ---- host-side error plumbing -----------------------------------------------------------------
void set_last_error(const char* where, cudaError_t e);
int32_t device_supported();  // TFS_OK on sm_100, else TFS_ERR_UNSUPPORTED (cached per device)
int num_sms();               // SM count of the current device (cached)
void launched(int n = 1);    // count kernel launches (tfs_debug_launch_count)

#define TFS_CUDA_TRY(expr)                                \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) {                              \
      ::tfs::set_last_error(#expr, _e);                   \
      return TFS_ERR_CUDA;                                \
    }                                                     \
  } while (0)

#define TFS_LAUNCH_CHECK()                                \
  do {                                                    \
    cudaError_t _e = cudaGetLastError();                  \
    if (_e != cudaSuccess) {                              \
      ::tfs::set_last_error("kernel launch", _e);         \
      return TFS_ERR_CUDA;                                \
    }                                                     \
  } while (0)

#define TFS_REQUIRE(cond)                                 \
  do {                                                    \
    if (!(cond)) return TFS_ERR_INVALID_ARGUMENT;         \
  } while (0)

#define TFS_SUPPORTED()                                   \
  do {                                                    \
    int32_t _s = ::tfs::device_supported();               \
    if (_s != TFS_OK) return _s;                          \
  } while (0)

// ---- workspace carving: 256-byte aligned slices of the caller's workspace ---------------------
struct Carver {
  char* base;
  size_t cap;
  size_t used = 0;
  Carver(void* b, size_t c) : base((char*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    return base ? (T*)(base + off) : nullptr;
  }
  bool fits() const { return used <= cap; }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__device__ __forceinline__ int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline cudaStream_t as_stream(void* s) { return (cudaStream_t)s; }

// ---- device helpers ----------------------------------------------------------------------------
__device__ __forceinline__ void report_error(tfs_device_error* err, int32_t code, int64_t index) {
  if (err == nullptr) return;
  atomicMin((unsigned long long*)&err->index, (unsigned long long)index);
  atomicCAS(&err->code, 0, code);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float x) {
  __nv_bfloat16 b = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&b);
}

__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // one cvt.rn.bf16x2.f32; lo in bits 0-15
  return *reinterpret_cast<uint32_t*>(&v);
}

// ---- programmatic dependent launch (PDL) ---------------------------------------------------------
// Every kernel of the library is launched with programmatic stream serialization and opens with
// pdl_enter(), which waits (griddepcontrol.wait) until the PREVIOUS grid on the stream has
// completed and its memory is visible before touching any data: results are those of plain
// stream order, and the next grid's launch is processed while the previous one drains (inside
// CUDA graphs too).  Measured round 2 (profiles/r2_ab_pdl.log): X step 192 -> 183 us, Z neutral.
// An explicit early trigger (griddepcontrol.launch_dependents at kernel start, TFS_PDL_TRIGGER=1
// builds) is SLOWER (X 215 us, Z +8 %): the early-scheduled CTAs sit on SMs while they wait and
// crowd out the side streams' kernels.  TFS_PDL=0 in the environment turns PDL off.
#ifndef TFS_PDL_TRIGGER
#define TFS_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_enter() {
  if (TFS_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- bulk (non-tensor) TMA copies into shared memory, completed on an mbarrier -----------------
// The row movers stage whole rows through a shared-memory ring with these: one elected lane
// issues cp.async.bulk for a row (global -> smem, bytes % 16 == 0, 16-byte aligned ends), the
// copy engine signals the slot's mbarrier with the byte count, the consumers wait on its phase.
// The bytes in flight then live in shared memory, not in registers.
namespace bulk {
__device__ __forceinline__ uint32_t s32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(count) : "memory");
}
// Make barrier initialisation visible to the async proxy (the copy engine).
__device__ __forceinline__ void fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Order this thread's generic-proxy accesses of shared memory before later async-proxy ones
// (a slot read by the consumers is about to be refilled by a bulk copy).
__device__ __forceinline__ void fence_proxy() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(s32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          s32(dst)),
      "l"(src), "r"(bytes), "r"(s32(bar))
      : "memory");
}
}  // namespace bulk

}  // namespace tfs

// ---- internal launchers shared between translation units --------------------------------------
namespace tfs {

// Stable digit sort engine (partition / radix).  See sort.cu.
enum DigitMode : int { kDigitMod = 0, kDigitAssign = 1, kDigitRadix = 2 };

// Stable LSD radix sort of (uint32 key, uint32 val) pairs; keys < 2^key_bits.  Result in
// keys_out/vals_out.  Scratch from the carver.
size_t radix_sort_ws_bytes(int64_t n);
int32_t radix_sort_pairs(const uint32_t* keys_in, const uint32_t* vals_in, uint32_t* keys_out,
                         uint32_t* vals_out, int64_t n, int key_bits, void* ws, size_t ws_bytes,
                         cudaStream_t st);

}  // namespace tfs
