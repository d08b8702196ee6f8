// Shared helpers for the STS sm_100a kernels: error plumbing for the C-ABI,
// order-preserving key transforms, and the PTX wrappers (cp.async, ldmatrix,
// mma.sync, movmatrix) the gather kernels use.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>

#include "../../include/sts_b200.h"

namespace sts {

// ---------------------------------------------------------------------------
// host-side error plumbing (thread-local message, status codes of the ABI)
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);

#define STS_REQUIRE(cond, code, ...)   \
  do {                                 \
    if (!(cond)) {                     \
      ::sts::set_error(__VA_ARGS__);   \
      return (code);                   \
    }                                  \
  } while (0)

#define STS_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::sts::set_error("CUDA error %s at %s:%d", cudaGetErrorString(_e),       \
                       __FILE__, __LINE__);                                    \
      return STS_ERR_CUDA;                                                     \
    }                                                                          \
  } while (0)

// every kernel launch of the library passes here (counted: sts_launch_count)
void count_launch();
#define STS_LAUNCH_CHECK()              \
  do {                                  \
    ::sts::count_launch();              \
    STS_CUDA_CHECK(cudaGetLastError()); \
  } while (0)

int num_sms();

// ---------------------------------------------------------------------------
// order-preserving keys: unsigned compare == reference rank order
// (-0.0 canonicalised to +0.0, NaN -> 0 i.e. below -inf)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t f32_key(float x) {
  // order-preserving: negatives -> ~bits, non-negatives -> bits | sign; -0 -> +0; NaN -> 0
  const uint32_t b = __float_as_uint(x + 0.0f);
  const uint32_t k = b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
  return x != x ? 0u : k;
}

__device__ __forceinline__ uint64_t f64_key(double x) {
  if (x != x) return 0ull;
  uint64_t b = (uint64_t)__double_as_longlong(x + 0.0);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

__device__ __forceinline__ void cp_async_16_zfill(uint32_t dst, const void* src, bool valid) {
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                            uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                                  uint32_t& r3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

__device__ __forceinline__ void ldmatrix_x2(uint32_t& r0, uint32_t& r1, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}

// D(16x8 f32) += A(16x16 bf16, row) * B(16x8 bf16, col)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4],
                                               const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// transpose an 8x8 b16 tile held in the standard fragment layout
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void set_status(int32_t* status, int bit) {
  if (status) atomicOr(status, bit);
}

}  // namespace sts
