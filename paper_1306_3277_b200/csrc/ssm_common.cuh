// Shared device helpers for libssm_b200 (sm_100a).
#pragma once

#ifdef __CUDACC_RTC__  // NVRTC (generic-model kernels): no system headers
typedef unsigned int uint32_t;
typedef int int32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
#define CUDART_INF __longlong_as_double(0x7ff0000000000000ULL)
#define CUDART_NAN __longlong_as_double(0xfff8000000000000ULL)
#else
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#endif

#include "../../include/ssm_b200.h"

namespace ssm {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// Counter-based Philox4x32-10 (Salmon et al. 2011).  The device RNG of the
// fast path: a pure function of (key, counter) so draws are independent of
// launch geometry and of how filters are batched or sharded (the RngStream
// purity contract, rng.py:1-11).
// ---------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// two blocks under one key: the round-key schedule is computed once for both
__device__ __forceinline__ void philox4x32_10_x2(U4& a, U4& b, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t pa0 = static_cast<uint64_t>(0xD2511F53u) * a.x, pa1 = static_cast<uint64_t>(0xCD9E8D57u) * a.z;
    const uint64_t pb0 = static_cast<uint64_t>(0xD2511F53u) * b.x, pb1 = static_cast<uint64_t>(0xCD9E8D57u) * b.z;
    a = U4{static_cast<uint32_t>(pa1 >> 32) ^ a.y ^ k0, static_cast<uint32_t>(pa1),
           static_cast<uint32_t>(pa0 >> 32) ^ a.w ^ k1, static_cast<uint32_t>(pa0)};
    b = U4{static_cast<uint32_t>(pb1 >> 32) ^ b.y ^ k0, static_cast<uint32_t>(pb1),
           static_cast<uint32_t>(pb0 >> 32) ^ b.w ^ k1, static_cast<uint32_t>(pb0)};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// counter word 3 tags the purpose of a draw so streams never overlap
enum Purpose : uint32_t {
  kPurposeNoise = 1u,
  kPurposeResample = 2u,
  kPurposeInit = 3u,
  kPurposeSystematic = 4u,
  kPurposeSpacing = 5u,  // exponential spacings of the sorted multinomial
  kPurposeGen = 6u,      // generic-model draws (ssm_gen_rt.cuh); bits 8+ carry a retry index
};

// 53-bit uniform in [0,1) from two 32-bit words (same construction as numpy's
// random_standard_uniform: (raw64 >> 11) * 2^-53, rng.py:44-45)
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
  const uint64_t v = ((static_cast<uint64_t>(hi) << 32) | lo) >> 11;
  return static_cast<double>(v) * 0x1.0p-53;
}

// Box-Muller pair, float64: u1 in (0,1]
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                           double& z0, double& z1) {
  const double u1 = 1.0 - u53(a, b);  // (0, 1]
  const double u2 = u53(c, d);
  const double r = sqrt(-2.0 * log(u1));
  double s, co;
  sincospi(2.0 * u2, &s, &co);
  z0 = r * co;
  z1 = r * s;
}

// MUFU approximations with flush-to-zero: no denormal fix-up code around them
// (the arguments below are never denormal).
__device__ __forceinline__ float lg2_ftz(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_ftz(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Box-Muller pair, float32 (the device noise generator for both precisions).
// u1 = (a + 1/2) 2^-32 keeps 32 bits near 0, so |z| reaches 6.7 sigma; the
// radius and angle use the MUFU lg2 / sqrt / sin / cos (angle on [-pi, pi),
// |error| < 2^-21; a rotation by pi leaves the pair iid N(0,1)).  u1 >= 2^-33,
// so nothing here is denormal; the max() guards lg2's error near u1 = 1.
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  const float u1 = fmaf(static_cast<float>(a), 0x1.0p-32f, 0x1.0p-33f);  // (0, 1]
  const float th = fmaf(static_cast<float>(b >> 8), 6.28318530717958647692f * 0x1.0p-24f,
                        -3.14159265358979323846f);
  const float x = fmaxf(-1.38629436111989061883f * lg2_ftz(u1), 0.0f);  // -2 ln u1
  const float r = sqrt_ftz(x);
  float s, co;
  __sincosf(th, &s, &co);
  z0 = r * co;
  z1 = r * s;
}

// finite test on the exponent bits (integer pipe, keeps the FP64 pipe free)
__device__ __forceinline__ bool finite_bits(double v) {
  return (__double2hiint(v) & 0x7ff00000) != 0x7ff00000;
}
__device__ __forceinline__ bool finite_bits(float v) {
  return (__float_as_int(v) & 0x7f800000) != 0x7f800000;
}

// ---------------------------------------------------------------------------
// Arithmetic policy.  EXACT = the reference's op order with every operation
// individually rounded (no FMA contraction): bitwise-equal to numpy float64
// for the L96 RK4.  !EXACT lets nvcc contract into FMA.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT>
struct Ar;

template <>
struct Ar<double, true> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  // division by a constant b with host-computed reciprocal rb: exact mode divides,
  // fast mode multiplies (within 1 ulp more)
  static __device__ __forceinline__ double divc(double a, double b, double rb) { return __ddiv_rn(a, b); }
};
template <>
struct Ar<double, false> {
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  // division by a constant b with host-computed reciprocal rb: exact mode divides,
  // fast mode multiplies (within 1 ulp more)
  static __device__ __forceinline__ double divc(double a, double b, double rb) { return a * rb; }
};
template <>
struct Ar<float, true> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  // division by a constant b with host-computed reciprocal rb: exact mode divides,
  // fast mode multiplies (within 1 ulp more)
  static __device__ __forceinline__ float divc(float a, float b, float rb) { return __fdiv_rn(a, b); }
};
template <>
struct Ar<float, false> {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float div(float a, float b) { return a / b; }
  // division by a constant b with host-computed reciprocal rb: exact mode divides,
  // fast mode multiplies (within 1 ulp more)
  static __device__ __forceinline__ float divc(float a, float b, float rb) { return a * rb; }
};

// ---------------------------------------------------------------------------
// Log-sum-exp + ESS state with scipy-1.18 semantics (particle.py:127 calls
// scipy.special.logsumexp, which splits the maximal elements out of the sum):
//   the represented set has max m, c elements equal to m,
//   t  = sum_{a<m} exp(a - m),  s2 = sum_{a<m} exp(2(a - m)).
//   LSE = m + log1p(t / c) + log(c),  ESS = (c + t)^2 / (c + s2).
// Combination is deterministic for a fixed combination tree.
// ---------------------------------------------------------------------------
struct Lse {
  double m, c, t, s2;
};

__device__ __forceinline__ Lse lse_empty() { return Lse{-CUDART_INF, 0.0, 0.0, 0.0}; }

__device__ __forceinline__ void lse_push(Lse& s, double a) {
  if (a > s.m) {
    const double f = exp(s.m - a);
    s.t = (s.c + s.t) * f;
    s.s2 = (s.c + s.s2) * (f * f);
    s.c = 1.0;
    s.m = a;
  } else if (a == s.m) {
    s.c += 1.0;
  } else {
    const double e = exp(a - s.m);  // NaN propagates (degenerate)
    s.t += e;
    s.s2 += e * e;
  }
}

__device__ __forceinline__ Lse lse_combine(Lse a, Lse b) {
  if (b.m > a.m) {
    const Lse tmp = a;
    a = b;
    b = tmp;
  }
  if (b.m == a.m) return Lse{a.m, a.c + b.c, a.t + b.t, a.s2 + b.s2};
  if (b.c == 0.0 && b.t == 0.0) return a;  // empty (NaN t is not empty)
  if (a.c == 0.0 && a.t == 0.0 && a.m == -CUDART_INF) return b;
  const double f = exp(b.m - a.m);         // NaN m -> NaN result
  return Lse{a.m, a.c, a.t + (b.c + b.t) * f, a.s2 + (b.c + b.s2) * (f * f)};
}

__device__ __forceinline__ Lse lse_shfl_down(const Lse& s, int off) {
  return Lse{__shfl_down_sync(0xffffffffu, s.m, off), __shfl_down_sync(0xffffffffu, s.c, off),
             __shfl_down_sync(0xffffffffu, s.t, off), __shfl_down_sync(0xffffffffu, s.s2, off)};
}

// Block-wide deterministic reduction; result valid in thread 0.
template <int NT>
__device__ __forceinline__ Lse lse_block_reduce(Lse s, Lse* smem /* NT/32 entries */) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s = lse_combine(s, lse_shfl_down(s, off));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) smem[warp] = s;
  __syncthreads();
  if (warp == 0) {
    s = lane < NT / 32 ? smem[lane] : lse_empty();
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s = lse_combine(s, lse_shfl_down(s, off));
  }
  __syncthreads();
  return s;
}

// c > 0: scipy's log1p form (max elements split out); c == 0 (partials built
// from fixed-point tile totals relative to a reference >= max): m + log(t).
__device__ __forceinline__ double lse_value(const Lse& s) {
  if (s.c == 0.0) return s.t > 0.0 ? s.m + log(s.t) : (isnan(s.t) ? s.t : (s.t == 0.0 ? -CUDART_INF : s.m));
  return log1p(s.t / s.c) + log(s.c) + s.m;
}

__device__ __forceinline__ double lse_ess(const Lse& s) {
  const double sw = s.c + s.t;
  return sw * sw / (s.c + s.s2);
}

template <typename T>
__device__ __forceinline__ bool finite(T v) {
  return isfinite(v);
}

// cp.async (LDGSTS): an asynchronous global -> shared copy per thread that
// holds no register while in flight.  The fused kernel stages its ancestor
// gather through shared memory with it (thread-private slots: a thread only
// ever reads the copies it issued, so cp.async.wait_group alone orders them).
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Bulk (TMA) copies global -> shared completing on an mbarrier (sm_90+ async
// proxy): one thread arms the barrier with the byte count and issues the copies;
// consumers wait on the barrier's phase parity.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Programmatic dependent launch: the per-step kernels of the filter path are
// launched with programmatic stream serialization, so a kernel's launch and
// block scheduling overlap the tail of its predecessor; each such kernel calls
// pdl_wait() as its FIRST statement (before any early exit, so completion stays
// transitive along the chain).  A no-op when launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifndef __CUDACC_RTC__

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_smem(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                   Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#endif  // __CUDACC_RTC__

}  // namespace ssm

#ifndef __CUDACC_RTC__
// error reporting helper shared by the C-ABI entry points
extern "C" void ssm_set_last_error(cudaError_t e);
// generic models (ssm_gen.cu)
int ssm_gen_propagate_weight(const ssm_pw_args& A, cudaStream_t s);
int ssm_gen_nx(const void* handle);
#define SSM_CHECK_LAUNCH()                      \
  do {                                          \
    cudaError_t _e = cudaGetLastError();        \
    if (_e != cudaSuccess) {                    \
      ssm_set_last_error(_e);                   \
      return SSM_ERR_CUDA;                      \
    }                                           \
  } while (0)
#endif  // __CUDACC_RTC__
