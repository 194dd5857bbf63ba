#pragma once
// Element arithmetic shared by the forest kernels (fc_device.cuh) and the
// NVLS engine (fc_nvls.cu): accumulation type A, buffer element E, one
// round-to-nearest-even per hop (the arithmetic contract).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "fc_internal.h"

namespace {

// ---------------------------------------------------------------------------
// Element arithmetic.  Accumulation type A; buffer element E.
// ---------------------------------------------------------------------------
template <int DT>
struct Red;

template <>
struct Red<FC_FLOAT32> {
  using E = unsigned;
  using A = float;
  __device__ static A to(E x) { return __uint_as_float(x); }
  __device__ static E from(A a) { return __float_as_uint(a); }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
  __device__ static A mul(A a, float s) { return __fmul_rn(a, s); }
};

// bf16: fp32 accumulate, one round-to-nearest-even per hop with the hardware
// converter (cvt.rn.bf16x2.f32: denormals kept, NaN -> canonical 0x7FFF, as
// oracle/forest_oracle.py::f32_to_bf16).
template <>
struct Red<FC_BFLOAT16> {
  using E = unsigned short;
  using A = float;
  __device__ static A to(E x) { return __uint_as_float(((unsigned)x) << 16); }
  __device__ static E from(A a) {
    unsigned short r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(a));
    return r;
  }
  // two elements at once: lo -> bits 0..15, hi -> bits 16..31
  __device__ static unsigned from2(A lo, A hi) {
    unsigned r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
  __device__ static A mul(A a, float s) { return __fmul_rn(a, s); }
};

template <>
struct Red<FC_FLOAT16> {
  using E = unsigned short;
  using A = float;
  __device__ static A to(E x) { return __half2float(__ushort_as_half(x)); }
  __device__ static E from(A a) { return __half_as_ushort(__float2half_rn(a)); }
  __device__ static unsigned from2(A lo, A hi) {
    unsigned r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
  }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
  __device__ static A mul(A a, float s) { return __fmul_rn(a, s); }
};

template <>
struct Red<FC_INT32> {  // also uint32: wrapping two's-complement add
  using E = unsigned;
  using A = unsigned;
  __device__ static A to(E x) { return x; }
  __device__ static E from(A a) { return a; }
  __device__ static A add(A a, A b) { return a + b; }
  __device__ static A mul(A a, float) { return a; }  // AVG is rejected for integers
};

// 8-byte payload words of caller buffers at any alignment.  The LL / LL128
// paths are chosen from rank-uniform values only (size, dtype, plan,
// options), so a rank whose tensor view is not 8-byte aligned runs the same
// protocol as its peers and only its local loads / stores take this branch.
// Staging lines are always aligned.
__device__ __forceinline__ unsigned long long ld_u64_any(const char* p) {
  const uintptr_t a = (uintptr_t)p;
  if ((a & 7) == 0) return __ldcg(reinterpret_cast<const unsigned long long*>(p));
  if ((a & 3) == 0) {
    const unsigned* q = reinterpret_cast<const unsigned*>(p);
    return (unsigned long long)__ldcg(q) | ((unsigned long long)__ldcg(q + 1) << 32);
  }
  if ((a & 1) == 0) {
    const unsigned short* q = reinterpret_cast<const unsigned short*>(p);
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) v |= (unsigned long long)__ldcg(q + i) << (16 * i);
    return v;
  }
  unsigned long long v = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    v |= (unsigned long long)(unsigned char)__ldcg(reinterpret_cast<const signed char*>(p) + i) << (8 * i);
  return v;
}

__device__ __forceinline__ void st_u64_any(char* p, unsigned long long v) {
  const uintptr_t a = (uintptr_t)p;
  if ((a & 7) == 0) {
    *reinterpret_cast<unsigned long long*>(p) = v;
  } else if ((a & 3) == 0) {
    unsigned* q = reinterpret_cast<unsigned*>(p);
    q[0] = (unsigned)v;
    q[1] = (unsigned)(v >> 32);
  } else if ((a & 1) == 0) {
    unsigned short* q = reinterpret_cast<unsigned short*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = (unsigned short)(v >> (16 * i));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = (char)(v >> (8 * i));
  }
}

// The first n (< 8) bytes of an 8-byte payload word at the end of a buffer
// whose length is not a multiple of 8: loaded into the low bytes (the rest
// zero), stored back byte by byte.
__device__ __forceinline__ unsigned long long ld_tail(const char* p, long long n) {
  unsigned long long v = 0;
  for (long long i = 0; i < n; ++i)
    v |= (unsigned long long)(unsigned char)__ldcg(reinterpret_cast<const signed char*>(p) + i) << (8 * i);
  return v;
}
__device__ __forceinline__ void st_tail(char* p, unsigned long long v, long long n) {
  for (long long i = 0; i < n; ++i) p[i] = (char)(v >> (8 * i));
}

// Word at byte offset pb of an S-byte buffer: whole, tail, or absent (0).
__device__ __forceinline__ unsigned long long ld_word(const char* base, long long pb, long long S) {
  if (pb + 8 <= S) return ld_u64_any(base + pb);
  return pb < S ? ld_tail(base + pb, S - pb) : 0ull;
}
__device__ __forceinline__ void st_word(char* base, long long pb, long long S, unsigned long long v) {
  if (pb + 8 <= S) st_u64_any(base + pb, v);
  else if (pb < S) st_tail(base + pb, v, S - pb);
}

}  // namespace
