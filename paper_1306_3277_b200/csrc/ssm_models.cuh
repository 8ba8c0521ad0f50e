// Per-particle model code of the two hand-written kernels (Lorenz '96, Windkessel):
// device noise, the transition (sub-steps of noise + RK4 / analytic update) and
// the initial draw.  Shared by the fused multi-kernel path (ssm_pw.cu), the
// trajectory replay and the persistent small-P kernel (ssm_small.cu), so every
// path computes the same bits.
#pragma once

#include "ssm_common.cuh"

namespace ssm {

// ----------------------------- noise ---------------------------------------

// Eight standard normals per particle and sub-step: two Philox4x32-10 blocks,
// float32 Box-Muller (MUFU-backed logf/sincospif), widened to T.  Keeping the
// transcendental work off the FP64 pipe is what lets the float64 filter stay
// memory-bound (profiles/r1_baseline_ncu.md).
template <typename T>
__device__ __forceinline__ void normals8(uint32_t k0, uint32_t k1, uint32_t p, uint32_t step,
                                         uint32_t sub, T z[8]) {
  U4 r[2] = {U4{p, step, sub << 8, kPurposeNoise}, U4{p, step, (sub << 8) | 1u, kPurposeNoise}};
  philox4x32_10_x2(r[0], r[1], k0, k1);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    float a, b, c, d;
    box_muller(r[g].x, r[g].y, a, b);
    box_muller(r[g].z, r[g].w, c, d);
    z[4 * g] = static_cast<T>(a);
    z[4 * g + 1] = static_cast<T>(b);
    z[4 * g + 2] = static_cast<T>(c);
    z[4 * g + 3] = static_cast<T>(d);
  }
}

// the same eight normals, kept in float (the SIMPLE fused kernel draws the next
// tile's noise while the current tile integrates)
__device__ __forceinline__ void normals8f(uint32_t k0, uint32_t k1, uint32_t p, uint32_t step, uint32_t sub,
                                          float (&z)[8]) {
  U4 r[2] = {U4{p, step, sub << 8, kPurposeNoise}, U4{p, step, (sub << 8) | 1u, kPurposeNoise}};
  philox4x32_10_x2(r[0], r[1], k0, k1);
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    box_muller(r[g].x, r[g].y, z[4 * g], z[4 * g + 1]);
    box_muller(r[g].z, r[g].w, z[4 * g + 2], z[4 * g + 3]);
  }
}

template <typename T>
__device__ __forceinline__ T normal1(uint32_t k0, uint32_t k1, uint32_t p, uint32_t step,
                                     uint32_t sub) {
  const U4 r = philox4x32_10(U4{p, step, sub << 8, kPurposeNoise}, k0, k1);
  float z0, z1;
  box_muller(r.x, r.y, z0, z1);
  return static_cast<T>(z0);
}

// ----------------------------- Lorenz '96 ----------------------------------
// Lorenz96.bi:27  dx[n]/dt = x[n-1]*(x[n+1] - x[n-2]) - x[n] + F + sqrt(sigma2)*deltaW[n]/h
// compiled (ir.py:188-214) as
//   ((((X[n-1] * (X[n+1] - X[n-2])) - X[n]) + F) + ((sqrt(sigma2) * W[n]) / 0.05))

template <typename T, bool E>
__device__ __forceinline__ void l96_deriv(const T x[8], T F, const T nt[8], T out[8]) {
  using O = Ar<T, E>;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    const T xm1 = x[(n + 7) & 7], xp1 = x[(n + 1) & 7], xm2 = x[(n + 6) & 7];
    out[n] = O::add(O::add(O::sub(O::mul(xm1, O::sub(xp1, xm2)), x[n]), F), nt[n]);
  }
}

// classic RK4, simulate.py:88-93 (evaluation order of the numpy expressions)
template <typename T, bool E>
__device__ __forceinline__ void l96_rk4(T x[8], T F, const T nt[8], T s) {
  using O = Ar<T, E>;
  T k[8], acc[8], st[8];
  const T hs = O::mul(T(0.5), s);  // `0.5 * s * k` == (0.5*s)*k
  l96_deriv<T, E>(x, F, nt, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = k[n];
    st[n] = O::add(x[n], O::mul(hs, k[n]));
  }
  l96_deriv<T, E>(st, F, nt, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = O::add(acc[n], O::mul(T(2.0), k[n]));
    st[n] = O::add(x[n], O::mul(hs, k[n]));
  }
  l96_deriv<T, E>(st, F, nt, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = O::add(acc[n], O::mul(T(2.0), k[n]));
    st[n] = O::add(x[n], O::mul(s, k[n]));
  }
  l96_deriv<T, E>(st, F, nt, k);
  const T s6 = O::div(s, T(6.0));
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = O::add(acc[n], k[n]);
    x[n] = O::add(x[n], O::mul(s6, acc[n]));
  }
}

// Fast (non-exact) float64 variant: same math, FMA-contracted and with the
// forcing and noise folded per sub-step (Fn = F + sqrt(sigma2) W / h); within
// 1e-12 norm-wise of the reference per step (tests/test_gpu_parity.py).
template <typename T>
__device__ __forceinline__ void l96_deriv_fast(const T x[8], const T Fn[8], T out[8]) {
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    const T xm1 = x[(n + 7) & 7], xp1 = x[(n + 1) & 7], xm2 = x[(n + 6) & 7];
    out[n] = fma(xm1, xp1 - xm2, -x[n]) + Fn[n];
  }
}

template <typename T>
__device__ __forceinline__ void l96_rk4_fast(T x[8], const T Fn[8], T s) {
  T k[8], acc[8], st[8];
  const T hs = T(0.5) * s;
  l96_deriv_fast<T>(x, Fn, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = k[n];
    st[n] = fma(hs, k[n], x[n]);
  }
  l96_deriv_fast<T>(st, Fn, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = fma(T(2.0), k[n], acc[n]);
    st[n] = fma(hs, k[n], x[n]);
  }
  l96_deriv_fast<T>(st, Fn, k);
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    acc[n] = fma(T(2.0), k[n], acc[n]);
    st[n] = fma(s, k[n], x[n]);
  }
  l96_deriv_fast<T>(st, Fn, k);
  const T s6 = s * T(1.0 / 6.0);
#pragma unroll
  for (int n = 0; n < 8; ++n) x[n] = fma(s6, acc[n] + k[n], x[n]);
}


// SIMPLE L96 step (one sub-step, one RK4 step) from standard normals z: the
// same arithmetic as transition_one's SIMPLE branch
template <typename T>
__device__ __forceinline__ void l96_simple_step(T (&x)[8], const float (&z)[8], T s_F, T s_c, T s_s) {
  T Fn[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) Fn[n] = fma(s_c, static_cast<T>(z[n]), s_F);  // F + sqrt(sigma2) sd z / h
  l96_rk4_fast<T>(x, Fn, s_s);
}

// One particle through one grid step (particle.py:110-111 / simulate.py:132-163):
// the sub-steps of noise + RK4 / windkessel update, in place on x.  Shared by
// the fused kernel and the trajectory replay, so both produce the same bits.
// SIMPLE (fast L96, one sub-step, one RK4 step) uses the hoisted constants
// s_F = F, s_c = sqrt(sigma2) / h * sqrt(d), s_s = RK4 step length.
template <int MODEL, typename T, bool E, bool INJ, bool SIMPLE>
__device__ __forceinline__ void transition_one(T (&x)[MODEL == SSM_MODEL_LORENZ96 ? 8 : 1], const double* th,
                                               const ssm_substep* subs, int n_sub, const T* noise, int P, int p,
                                               uint32_t k0, uint32_t k1, uint32_t pglob, uint32_t step, T s_F,
                                               T s_c, T s_s, bool check_finite, bool& bad, int& bad_sub) {
  using O = Ar<T, E>;
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  if constexpr (SIMPLE && MODEL == SSM_MODEL_LORENZ96 && !E && !INJ) {
    T z[8];
    normals8<T>(k0, k1, pglob, step, 0u, z);
    T Fn[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) Fn[n] = fma(s_c, z[n], s_F);  // F + sqrt(sigma2) sd z / h
    l96_rk4_fast<T>(x, Fn, s_s);
    if (check_finite && !bad) {
      bool ok = true;
#pragma unroll
      for (int n = 0; n < 8; ++n) ok &= finite_bits(x[n]);
      if (!ok) bad = true;  // bad_sub stays 0
    }
  } else {
  for (int k = 0; k < n_sub; ++k) {
    const ssm_substep& S = subs[k];
    if constexpr (MODEL == SSM_MODEL_LORENZ96) {
      T W[8];
      if constexpr (INJ) {
#pragma unroll
        for (int n = 0; n < 8; ++n) W[n] = noise[(static_cast<size_t>(k) * 8 + n) * P + p];
      } else {
        normals8<T>(k0, k1, pglob, step,
                    static_cast<uint32_t>(k), W);
        const T sd = static_cast<T>(S.sd);
#pragma unroll
        for (int n = 0; n < 8; ++n) W[n] = sd * W[n];
      }
      if constexpr (E) {
        const T F = static_cast<T>(th[0]);
        const T sq = static_cast<T>(th[1]);  // np.sqrt(sigma2), host-computed
        T nt[8];
#pragma unroll
        for (int n = 0; n < 8; ++n) nt[n] = O::div(O::mul(sq, W[n]), T(0.05));
        for (int m = 0; m < S.n_ode; ++m) l96_rk4<T, E>(x, F, nt, static_cast<T>(S.s[m]));
      } else {
        const T F = static_cast<T>(th[0]);
        const T sqh = static_cast<T>(th[1] * 20.0);  // sqrt(sigma2) / h
        T Fn[8];
#pragma unroll
        for (int n = 0; n < 8; ++n) Fn[n] = fma(sqh, W[n], F);
        for (int m = 0; m < S.n_ode; ++m) l96_rk4_fast<T>(x, Fn, static_cast<T>(S.s[m]));
      }
    } else {
      // Windkessel.bi:28-29, Pp <- exp(-h/(R*C))*Pp + R*(1 - exp(-h/(R*C)))*(F + xi)
      const T ca = static_cast<T>(th[0]), cb = static_cast<T>(th[1]);
      T xi;
      if constexpr (INJ) {
        xi = noise[static_cast<size_t>(k) * P + p];
      } else {
        xi = static_cast<T>(th[3]) * normal1<T>(k0, k1, pglob,
                                                step, static_cast<uint32_t>(k));
      }
      x[0] = O::add(O::mul(ca, x[0]), O::mul(cb, O::add(static_cast<T>(S.u_in), xi)));
    }
    if (check_finite && !bad) {
      bool ok = true;
#pragma unroll
      for (int n = 0; n < NX; ++n) ok &= finite_bits(x[n]);
      if (!ok) {
        bad = true;
        bad_sub = k;
      }
    }
  }
  }  // general sub-step loop
}

// initial state of global particle pg (sample_initial, simulate.py:111-129)
template <int MODEL, typename T>
__device__ __forceinline__ void init_one(T (&x)[MODEL == SSM_MODEL_LORENZ96 ? 8 : 1], uint32_t pg, uint32_t k0,
                                         uint32_t k1) {
  if constexpr (MODEL == SSM_MODEL_LORENZ96) {
    // x[n] ~ uniform(-1.0, 3.0): low + (high - low) * U  (Lorenz96.bi:21)
#pragma unroll
    for (uint32_t g = 0; g < 4; ++g) {
      const U4 r = philox4x32_10(U4{pg, 0u, g, kPurposeInit}, k0, k1);
      x[2 * g] = static_cast<T>(-1.0 + 4.0 * u53(r.x, r.y));
      x[2 * g + 1] = static_cast<T>(-1.0 + 4.0 * u53(r.z, r.w));
    }
  } else {
    // Pp ~ gaussian(90.0, 15.0)  (Windkessel.bi:24)
    const U4 r = philox4x32_10(U4{pg, 0u, 0u, kPurposeInit}, k0, k1);
    double z0, z1;
    box_muller(r.x, r.y, r.z, r.w, z0, z1);
    x[0] = static_cast<T>(90.0 + 15.0 * z0);
  }
}

}  // namespace ssm
