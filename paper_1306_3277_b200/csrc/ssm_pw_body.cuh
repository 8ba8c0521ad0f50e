// The fused propagate/weight step of one block of one filter (pw_body): the
// body of pw_kernel (ssm_pw.cu), shared with the persistent cooperative driver
// (ssm_resample.cu, ssm_advance_coop) which runs it on virtual blocks.
#pragma once

#include <climits>

#include "ssm_common.cuh"
#include "ssm_models.cuh"
#include "ssm_tile.cuh"

namespace ssm {

// ----------------------------- the kernel ----------------------------------
//
// Grid-stride over 256-particle block tiles; one particle per thread per tile.
// Per weighted WARP tile w (32 consecutive particles) the warp also produces,
// for the next step's resampling:
//   m_w     = max log-weight of the warp tile,
//   q_j     = round(exp(a_j - m_w) * 2^52)              (tile-local fixed point),
//   C_j     = inclusive prefix of q within the tile     -> cdf_local[j],
//   Q_w     = C_last                                    -> tile_rec[w] = {m_w, Q_w},
// and the tile's scipy-form LSE/ESS partial (max elements split out), folded
// in tile order into the warp / block partials for the fused finalize.

// SIMPLE: one sub-step with one RK4 step (the benchmark grid and the sparse
// SMC^2 grid) -- no runtime sub-step loops, sub-step constants hoisted out of
// the particle loop, observation slots selected by grid-uniform predicates.
// PEER (sharded filter): ancestors are global indices and the state is
// gathered from the rank that holds it through A.x_peer (NVLink P2P loads at
// the rank boundaries); the identity gather of a step without resampling reads
// this rank's own particles (global index p + p_offset).
// The fused step of block vb (of nvb) of filter b: the body of pw_kernel, also
// run by the persistent cooperative driver (ssm_coop.cu) on virtual blocks.
template <int MODEL, typename T, bool E, bool INJ, bool SIMPLE = false, bool PEER = false>
__device__ __forceinline__ void pw_body(const ssm_pw_args& A, int b, int vb, int nvb) {
  using O = Ar<T, E>;
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  const int P = A.P;
  const int ntiles = (P + kPwThreads - 1) / kPwThreads;
  ssm_filter_state* fs = A.fs + b;
  const int R = fs->resample_now;
  const bool uniform_in = R || fs->uniform;
  const double incr_prev = fs->incr;
  const size_t base = static_cast<size_t>(b) * NX * P;
  const int in_stride = A.x_in_stride > 0 ? A.x_in_stride : P;  // sharded filter: local + received states
  const T* __restrict__ xin = static_cast<const T*>(A.x_in) + static_cast<size_t>(b) * NX * in_stride;
  const int out_stride = A.x_out_stride > 0 ? A.x_out_stride : P;  // spill capacity for the sharded filter
  T* __restrict__ xout = static_cast<T*>(A.x_out) + static_cast<size_t>(b) * NX * out_stride;
  const int32_t* __restrict__ anc =
      (R && A.anc != nullptr) ? A.anc + static_cast<size_t>(b) * P : nullptr;
  const T* __restrict__ aprev =
      A.a_prev ? static_cast<const T*>(A.a_prev) + static_cast<size_t>(b) * P : nullptr;
  T* __restrict__ aout = A.a_out ? static_cast<T*>(A.a_out) + static_cast<size_t>(b) * P : nullptr;
  uint64_t* __restrict__ cloc =
      A.cdf_local ? static_cast<uint64_t*>(A.cdf_local) + static_cast<size_t>(b) * P : nullptr;
  ssm_tile_rec* __restrict__ trec =
      A.tile_rec ? static_cast<ssm_tile_rec*>(A.tile_rec) + static_cast<size_t>(b) * ((P + 31) >> 5) : nullptr;
  const T* __restrict__ noise =
      INJ ? static_cast<const T*>(A.noise) + static_cast<size_t>(b) * A.n_sub * NX * P : nullptr;
  const double* th = A.theta + 4 * b;
  const bool have_keys = !INJ && A.keys != nullptr;
  const uint32_t k0 = have_keys ? A.keys[2 * b] : 0u, k1 = have_keys ? A.keys[2 * b + 1] : 0u;
  const int has_obs = A.has_obs;
  const T logw0 = static_cast<T>(A.log_w0);
  const T obs_log_sd = static_cast<T>(A.obs_log_sd);
  const T lsp = static_cast<T>(A.log_sqrt_2pi);
  const int lane = threadIdx.x & 31;
  const bool want_ess = A.ess_rel >= 0.0;

  __shared__ double s_exp_tab[64];
  if (threadIdx.x < 64) s_exp_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
  __syncthreads();
  __shared__ ParkedTiles s_park[kPwThreads / 32];
  WarpTileAcc acc = warp_tile_acc(&s_park[threadIdx.x >> 5], lane);
  bool bad = false;
  int bad_sub = 0;

  // Staged ancestor gather (x = x[anc], particle.py:102): while the current
  // tile computes, each thread's cp.async copies of its NEXT tile's ancestor
  // state (NX words) are in flight into its own shared-memory slots, and the
  // ancestor index of the tile after that is loaded -- the anc -> x dependent
  // loads never stall an iteration and hold no registers (2-stage ring).
#ifndef SSM_STAGED_GATHER
#define SSM_STAGED_GATHER 0
#endif
  const int stride = nvb * kPwThreads;
  const int p0 = vb * kPwThreads + threadIdx.x;
#if SSM_STAGED_GATHER
  static_assert(!PEER, "the staged gather has no peer path");
  __shared__ __align__(16) T s_x[2][NX][kPwThreads];
  auto stage_x = [&](int st, int src) {
#pragma unroll
    for (int n = 0; n < NX; ++n) cp_async<sizeof(T)>(&s_x[st][n][threadIdx.x], xin + static_cast<size_t>(n) * in_stride + src);
  };
  if (p0 < P) stage_x(0, anc ? __ldg(anc + p0) : p0);
  cp_async_commit();
  int stage = 0;
#else
  // register prefetch: the next tile's gathered state is in flight in xn[]
  T xn[NX];
  auto load_x = [&](int src) {
    const T* base = xin;
    if constexpr (PEER) {  // global index -> owning rank's (peer-mapped) positions
      const int loc = src - A.p_offset;
      if (static_cast<unsigned>(loc) < static_cast<unsigned>(A.peer_n)) {
        src = loc;  // this rank's particle (all but the boundary ancestors)
      } else {
        const int o = src / A.peer_n;
        base = static_cast<const T*>(A.x_peer[o]) + static_cast<size_t>(b) * NX * in_stride;
        src -= o * A.peer_n;
      }
    }
#pragma unroll
    for (int n = 0; n < NX; ++n) xn[n] = base[static_cast<size_t>(n) * in_stride + src];
  };
  const int src_off = PEER ? A.p_offset : 0;  // identity gather: this rank's particle p (global p + offset)
  if (p0 < P) load_x(anc ? __ldg(anc + p0) : p0 + src_off);
#endif
  int anc_next = (anc && p0 + stride < P) ? __ldg(anc + p0 + stride) : p0 + stride + src_off;
  const T gconst = static_cast<T>(static_cast<double>(__popc(A.obs_mask)) * (A.obs_log_sd + A.log_sqrt_2pi));
  T s_F = T(0), s_c = T(0), s_s = T(0);
  // SIMPLE with every slot observed: the finite-state check rides on the observation sum
  const bool defer_finite = SIMPLE && MODEL == SSM_MODEL_LORENZ96 && !E && !INJ && has_obs &&
                            A.obs_mask == 0xFFu && A.check_finite != 0;
  if constexpr (SIMPLE) {
    s_F = static_cast<T>(th[0]);
    s_c = static_cast<T>(th[1] * 20.0 * A.subs[0].sd);  // sqrt(sigma2) / h * sqrt(d)
    s_s = static_cast<T>(A.subs[0].s[0]);
  }

#ifndef SSM_PIPE_NOISE
#define SSM_PIPE_NOISE 1
#endif
  // kPipeNoise: the next tile's draws issued during this tile's RK4 (8 more live
  // registers); kDrawNow: the tile's own draws at its start (fits 3 CTAs / SM)
  constexpr bool kPipeNoise = SSM_PIPE_NOISE && SIMPLE && MODEL == SSM_MODEL_LORENZ96 && !E && !INJ;
  constexpr bool kDrawNow = !SSM_PIPE_NOISE && SIMPLE && MODEL == SSM_MODEL_LORENZ96 && !E && !INJ;
  constexpr bool kPipeNoiseWK = SIMPLE && MODEL == SSM_MODEL_WINDKESSEL && !INJ;
  float zc[8], zn[8];  // (kPipeNoise*) this tile's and the next tile's standard normals
  if constexpr (kPipeNoise) {
    if (p0 < P) normals8f(k0, k1, static_cast<uint32_t>(p0 + A.p_offset), static_cast<uint32_t>(A.step), 0u, zc);
  }
  if constexpr (kPipeNoiseWK) {
    if (p0 < P) zc[0] = normal1<float>(k0, k1, static_cast<uint32_t>(p0 + A.p_offset), static_cast<uint32_t>(A.step), 0u);
  }
  // SIMPLE windkessel: the sub-step's input and the analytic-update constants hoisted
  const T wk_u = SIMPLE && MODEL == SSM_MODEL_WINDKESSEL ? static_cast<T>(A.subs[0].u_in) : T(0);

  for (int tile = vb; tile < ntiles; tile += nvb) {
    const int p = tile * kPwThreads + threadIdx.x;
    const bool act = p < P;
    double a_d = -CUDART_INF;
    T x[NX];
#if SSM_STAGED_GATHER
    {
      const int p2 = p + stride;
      if (p2 < P) stage_x(stage ^ 1, anc_next);
      cp_async_commit();  // (possibly empty) group per tile: uniform group accounting
      const int p3 = p2 + stride;
      anc_next = (anc && p3 < P) ? __ldg(anc + p3) : p3;
    }
    cp_async_wait<1>();  // this tile's copies have landed (the next tile's may be in flight)
#pragma unroll
    for (int n = 0; n < NX; ++n) x[n] = s_x[stage][n][threadIdx.x];
    stage ^= 1;
#else
#pragma unroll
    for (int n = 0; n < NX; ++n) x[n] = xn[n];
    {
      const int p2 = p + stride;
      if (p2 < P) load_x(anc_next);
      const int p3 = p2 + stride;
      anc_next = (anc && p3 < P) ? __ldg(anc + p3) : p3 + src_off;
    }
#endif
    if (act) {
      if constexpr (kPipeNoise) {
        // the next tile's draws do not depend on this tile: issuing them here gives the
        // scheduler integer / MUFU work to interleave with the FP64 RK4 chain
        const int pn = p + stride;
        if (pn < P) normals8f(k0, k1, static_cast<uint32_t>(pn + A.p_offset), static_cast<uint32_t>(A.step), 0u, zn);
        l96_simple_step<T>(reinterpret_cast<T(&)[8]>(x), zc, s_F, s_c, s_s);
        if (A.check_finite != 0 && !defer_finite && !bad) {
          bool ok = true;
#pragma unroll
          for (int n = 0; n < NX; ++n) ok &= finite_bits(x[n]);
          if (!ok) bad = true;
        }
#pragma unroll
        for (int n = 0; n < 8; ++n) zc[n] = zn[n];
      } else if constexpr (kDrawNow) {
        float z[8];
        normals8f(k0, k1, static_cast<uint32_t>(p + A.p_offset), static_cast<uint32_t>(A.step), 0u, z);
        l96_simple_step<T>(reinterpret_cast<T(&)[8]>(x), z, s_F, s_c, s_s);
        if (A.check_finite != 0 && !defer_finite && !bad) {
          bool ok = true;
#pragma unroll
          for (int n = 0; n < NX; ++n) ok &= finite_bits(x[n]);
          if (!ok) bad = true;
        }
      } else if constexpr (kPipeNoiseWK) {
        const int pn = p + stride;
        if (pn < P) zn[0] = normal1<float>(k0, k1, static_cast<uint32_t>(pn + A.p_offset), static_cast<uint32_t>(A.step), 0u);
        // Windkessel.bi:28-29 as transition_one: ca x + cb (F + xi), xi = h sqrt(sigma2) z
        using O = Ar<T, E>;
        const T xi = static_cast<T>(th[3]) * static_cast<T>(zc[0]);
        x[0] = O::add(O::mul(static_cast<T>(th[0]), x[0]), O::mul(static_cast<T>(th[1]), O::add(wk_u, xi)));
        if (A.check_finite != 0 && !bad && !finite_bits(x[0])) bad = true;
        zc[0] = zn[0];
      } else {
        transition_one<MODEL, T, E, INJ, SIMPLE>(x, th, A.subs, A.n_sub, noise, P, p, k0, k1,
                                                static_cast<uint32_t>(p + A.p_offset), static_cast<uint32_t>(A.step),
                                                s_F, s_c, s_s, A.check_finite != 0 && !defer_finite, bad, bad_sub);
      }
#pragma unroll
      for (int n = 0; n < NX; ++n) xout[static_cast<size_t>(n) * out_stride + p] = x[n];

      if (has_obs) {
        T g = T(0);
        if constexpr (MODEL == SSM_MODEL_LORENZ96) {
          if constexpr (E) {
#pragma unroll
            for (int n = 0; n < 8; ++n) {
              if (A.obs_mask & (1u << n)) {
                const T z = O::mul(O::sub(static_cast<T>(A.y[n]), x[n]), T(2.0));  // exact: / 0.5
                g = O::add(g, O::sub(O::sub(O::mul(O::mul(T(-0.5), z), z), obs_log_sd), lsp));
              }
            }
          } else {
            // sum of -z^2/2 with z = (y - x) / 0.5 = 2d, accumulated as -2 * sum(d^2):
            // every step differs from fma(-z/2, z, g) by a power-of-two scaling only,
            // so the two forms round identically (bitwise) with half the FP64 work
            T s = T(0);
            if constexpr (SIMPLE) {
              const uint32_t mask = A.obs_mask;  // grid-uniform: no divergence
              if (mask == 0xFFu) {
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                  const T d = static_cast<T>(A.y[n]) - x[n];
                  s = fma(d, d, s);
                }
                // deferred finite check: s is finite only if every x[n] is, so the
                // per-slot test runs only when s is not (overflow or a bad state)
                if (defer_finite && !bad && !(s < T(CUDART_INF))) {
                  bool ok = true;
#pragma unroll
                  for (int n = 0; n < 8; ++n) ok &= finite_bits(x[n]);
                  if (!ok) bad = true;  // bad_sub stays 0 (one sub-step)
                }
              } else {
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                  const T d = static_cast<T>(A.y[n]) - x[n];
                  if (mask & (1u << n)) s = fma(d, d, s);
                }
              }
            } else {
#pragma unroll
              for (int n = 0; n < 8; ++n) {
                if (A.obs_mask & (1u << n)) {
                  const T d = static_cast<T>(A.y[n]) - x[n];
                  s = fma(d, d, s);
                }
              }
            }
            g = fma(T(-2.0), s, -gconst);
          }
        } else {
          const T mean = O::add(x[0], O::mul(static_cast<T>(th[2]), static_cast<T>(A.u_obs)));
          const T z = O::mul(O::sub(static_cast<T>(A.y[0]), mean), T(0.5));  // exact: / 2.0
          g = O::add(g, O::sub(O::sub(O::mul(O::mul(T(-0.5), z), z), obs_log_sd), lsp));
        }
        const T lw = uniform_in ? logw0 : O::sub(aprev[p], static_cast<T>(incr_prev));
        const T a = O::add(lw, g);
        if (aout) aout[p] = a;
        a_d = static_cast<double>(a);
      }
    }
    if (!has_obs) continue;  // block-uniform

    warp_tile_weigh(acc, a_d, act, p, P, lane, s_exp_tab, cloc, trec, want_ess);
  }
  warp_tile_flush(acc, lane);

  if (bad) atomicMin(&fs->err_nonfinite, A.step * 64 + bad_sub);

  pw_block_finalize<kPwThreads>(A, fs, b, P, R, has_obs, acc.park->st, lane, kMaxPwBlocks, vb, nvb);
}


// The headline step (Lorenz '96, SIMPLE: one sub-step with one RK4 step, fast
// arithmetic, device noise, every slot observed, no ESS gate, one rank) with the
// warp-tile weighting of tile t issued in iteration t + 1: that weighting is a
// serial chain (REDUX, exp, fixed point, two shuffle scans) with nothing to
// overlap inside its own tile, but it is independent of the next tile's RK4 /
// Philox work, so in one basic block the scheduler interleaves the two.  Same
// arithmetic, stores and tile order as pw_body (bitwise the same filter).
template <typename T>
__device__ __forceinline__ void pw_body_lag(const ssm_pw_args& A, int b, int vb, int nvb) {
  constexpr int NX = 8;
  const int P = A.P;
  const int ntiles = (P + kPwThreads - 1) / kPwThreads;
  ssm_filter_state* fs = A.fs + b;
  const int R = fs->resample_now;
  const bool uniform_in = R || fs->uniform;
  const double incr_prev = fs->incr;
  const int in_stride = A.x_in_stride > 0 ? A.x_in_stride : P;
  const T* __restrict__ xin = static_cast<const T*>(A.x_in) + static_cast<size_t>(b) * NX * in_stride;
  const int out_stride = A.x_out_stride > 0 ? A.x_out_stride : P;
  T* __restrict__ xout = static_cast<T*>(A.x_out) + static_cast<size_t>(b) * NX * out_stride;
  const int32_t* __restrict__ anc = (R && A.anc != nullptr) ? A.anc + static_cast<size_t>(b) * P : nullptr;
  const T* __restrict__ aprev = A.a_prev ? static_cast<const T*>(A.a_prev) + static_cast<size_t>(b) * P : nullptr;
  T* __restrict__ aout = A.a_out ? static_cast<T*>(A.a_out) + static_cast<size_t>(b) * P : nullptr;
  uint64_t* __restrict__ cloc = static_cast<uint64_t*>(A.cdf_local) + static_cast<size_t>(b) * P;
  ssm_tile_rec* __restrict__ trec = static_cast<ssm_tile_rec*>(A.tile_rec) + static_cast<size_t>(b) * ((P + 31) >> 5);
  const double* th = A.theta + 4 * b;
  const uint32_t k0 = A.keys[2 * b], k1 = A.keys[2 * b + 1];
  const T logw0 = static_cast<T>(A.log_w0);
  const int lane = threadIdx.x & 31;

  __shared__ double s_exp_tab[64];
  if (threadIdx.x < 64) s_exp_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
  __syncthreads();
  __shared__ ParkedTiles s_park[kPwThreads / 32];
  WarpTileAcc acc = warp_tile_acc(&s_park[threadIdx.x >> 5], lane);
  bool bad = false;

  const int stride = nvb * kPwThreads;
  const int p0 = vb * kPwThreads + threadIdx.x;
  T xn[NX];
  auto load_x = [&](int src) {
#pragma unroll
    for (int n = 0; n < NX; ++n) xn[n] = xin[static_cast<size_t>(n) * in_stride + src];
  };
  if (p0 < P) load_x(anc ? __ldg(anc + p0) : p0);
  int anc_next = (anc && p0 + stride < P) ? __ldg(anc + p0 + stride) : p0 + stride;
  const T gconst = static_cast<T>(8.0 * (A.obs_log_sd + A.log_sqrt_2pi));
  const bool check = A.check_finite != 0;
  const T s_F = static_cast<T>(th[0]);
  const T s_c = static_cast<T>(th[1] * 20.0 * A.subs[0].sd);
  const T s_s = static_cast<T>(A.subs[0].s[0]);
  T yv[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) yv[n] = static_cast<T>(A.y[n]);
  float zc[8], zn[8];
  if (p0 < P) normals8f(k0, k1, static_cast<uint32_t>(p0 + A.p_offset), static_cast<uint32_t>(A.step), 0u, zc);

  double a_lag = -CUDART_INF;
  bool act_lag = false, real_lag = false;
  int p_lag = P;
  for (int tile = vb; tile < ntiles; tile += nvb) {
    const int p = tile * kPwThreads + threadIdx.x;
    const bool act = p < P;
    T x[NX];
#pragma unroll
    for (int n = 0; n < NX; ++n) x[n] = xn[n];
    {
      const int p2 = p + stride;
      if (p2 < P) load_x(anc_next);
      const int p3 = p2 + stride;
      anc_next = (anc && p3 < P) ? __ldg(anc + p3) : p3;
    }
    const int pn = p + stride;
    if (pn < P) normals8f(k0, k1, static_cast<uint32_t>(pn + A.p_offset), static_cast<uint32_t>(A.step), 0u, zn);
    l96_simple_step<T>(x, zc, s_F, s_c, s_s);
#pragma unroll
    for (int n = 0; n < 8; ++n) zc[n] = zn[n];
    if (act) {
#pragma unroll
      for (int n = 0; n < NX; ++n) xout[static_cast<size_t>(n) * out_stride + p] = x[n];
    }
    T sq = T(0);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const T d = yv[n] - x[n];
      sq = fma(d, d, sq);
    }
    const T g = fma(T(-2.0), sq, -gconst);
    const T lw = uniform_in ? logw0 : Ar<T, false>::sub(aprev[act ? p : 0], static_cast<T>(incr_prev));
    const T a = Ar<T, false>::add(lw, g);
    if (act && aout) aout[p] = a;
    // the previous tile's weighting (independent of this tile's work above)
    warp_tile_weigh_lag(acc, a_lag, act_lag, p_lag, P, lane, s_exp_tab, cloc, trec, real_lag);
    a_lag = act ? static_cast<double>(a) : -CUDART_INF;
    act_lag = act;
    p_lag = p;
    real_lag = true;
    // deferred finite check: sq is finite only if every x[n] is (as pw_body)
    if (check && act && !bad && !(sq < T(CUDART_INF))) {
      bool ok = true;
#pragma unroll
      for (int n = 0; n < 8; ++n) ok &= finite_bits(x[n]);
      if (!ok) bad = true;
    }
  }
  warp_tile_weigh_lag(acc, a_lag, act_lag, p_lag, P, lane, s_exp_tab, cloc, trec, real_lag);
  warp_tile_flush(acc, lane);

  if (bad) atomicMin(&fs->err_nonfinite, A.step * 64);
  pw_block_finalize<kPwThreads>(A, fs, b, P, R, 1, acc.park->st, lane, kMaxPwBlocks, vb, nvb);
}

// pw_body_lag with the ancestor gather staged through shared memory by TMA bulk
// copies: per warp tile, the ancestors of its 32 particles are non-decreasing
// (systematic / stratified / sorted multinomial, or the identity), so the tile
// reads one contiguous source range per state slot; lane 0 issues those 8 copies
// (cp.async.bulk, completing on the warp's mbarrier) one tile ahead, and every
// lane then reads its ancestor's state from shared memory.  Tiles whose source
// range exceeds the staging width fall back to direct loads.  Dynamic shared
// memory: [warps][2 stages][8 slots][kTmaW] of T.
constexpr int kTmaW = 64;
template <typename T>
__device__ __forceinline__ void pw_body_lag_tma(const ssm_pw_args& A, int b, int vb, int nvb) {
  constexpr int NX = 8;
  const int P = A.P;
  const int ntiles = (P + kPwThreads - 1) / kPwThreads;
  ssm_filter_state* fs = A.fs + b;
  const int R = fs->resample_now;
  const bool uniform_in = R || fs->uniform;
  const double incr_prev = fs->incr;
  const int in_stride = A.x_in_stride > 0 ? A.x_in_stride : P;
  const T* __restrict__ xin = static_cast<const T*>(A.x_in) + static_cast<size_t>(b) * NX * in_stride;
  const int out_stride = A.x_out_stride > 0 ? A.x_out_stride : P;
  T* __restrict__ xout = static_cast<T*>(A.x_out) + static_cast<size_t>(b) * NX * out_stride;
  const int32_t* __restrict__ anc = (R && A.anc != nullptr) ? A.anc + static_cast<size_t>(b) * P : nullptr;
  const T* __restrict__ aprev = A.a_prev ? static_cast<const T*>(A.a_prev) + static_cast<size_t>(b) * P : nullptr;
  T* __restrict__ aout = A.a_out ? static_cast<T*>(A.a_out) + static_cast<size_t>(b) * P : nullptr;
  uint64_t* __restrict__ cloc = static_cast<uint64_t*>(A.cdf_local) + static_cast<size_t>(b) * P;
  ssm_tile_rec* __restrict__ trec = static_cast<ssm_tile_rec*>(A.tile_rec) + static_cast<size_t>(b) * ((P + 31) >> 5);
  const double* th = A.theta + 4 * b;
  const uint32_t k0 = A.keys[2 * b], k1 = A.keys[2 * b + 1];
  const T logw0 = static_cast<T>(A.log_w0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  extern __shared__ __align__(16) unsigned char dyn_smem[];
  T* s_x = reinterpret_cast<T*>(dyn_smem) + static_cast<size_t>(warp) * 2 * NX * kTmaW;  // this warp's 2 stages
  __shared__ uint64_t s_bar[kPwThreads / 32][2];
  __shared__ double s_exp_tab[64];
  if (threadIdx.x < 64) s_exp_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
  if (lane == 0) {
    mbar_init(&s_bar[warp][0], 1u);
    mbar_init(&s_bar[warp][1], 1u);
    mbar_fence_init();
  }
  __syncthreads();
  __shared__ ParkedTiles s_park[kPwThreads / 32];
  WarpTileAcc acc = warp_tile_acc(&s_park[warp], lane);
  bool bad = false;

  const int stride = nvb * kPwThreads;
  const int p0 = vb * kPwThreads + threadIdx.x;
  auto anc_of = [&](int p) -> int { return anc ? __ldg(anc + min(p, P - 1)) : p; };
  // stage the source range of the warp tile whose lanes hold ancestors `a` (valid: p < P)
  // into stage st; returns the range start, or -1 (fallback: direct loads)
  auto issue = [&](int a, bool valid, int st) -> int {
    const int lo = __reduce_min_sync(0xffffffffu, valid ? a : INT_MAX);
    const int hi = __reduce_max_sync(0xffffffffu, valid ? a : -1);
    if (hi < 0) return -1;  // no particle in range
    constexpr int kAl = 16 / static_cast<int>(sizeof(T));  // elements per 16 bytes
    const int start = lo & ~(kAl - 1);
    const int count = (hi + kAl - start) & ~(kAl - 1);  // 16-byte aligned span covering [lo, hi]
    if (count > kTmaW || start + count > in_stride) return -1;
    __syncwarp();  // every lane is done reading this stage's previous tile
    if (lane == 0) {
      fence_proxy_async_smem();
      const uint32_t bytes = static_cast<uint32_t>(count * sizeof(T));
      mbar_expect_tx(&s_bar[warp][st], NX * bytes);
#pragma unroll
      for (int n = 0; n < NX; ++n)
        bulk_g2s(s_x + (st * NX + n) * kTmaW, xin + static_cast<size_t>(n) * in_stride + start, bytes,
                 &s_bar[warp][st]);
    }
    return start;
  };
  const T gconst = static_cast<T>(8.0 * (A.obs_log_sd + A.log_sqrt_2pi));
  const bool check = A.check_finite != 0;
  const T s_F = static_cast<T>(th[0]);
  const T s_c = static_cast<T>(th[1] * 20.0 * A.subs[0].sd);
  const T s_s = static_cast<T>(A.subs[0].s[0]);
  T yv[8];
#pragma unroll
  for (int n = 0; n < 8; ++n) yv[n] = static_cast<T>(A.y[n]);
  float zc[8], zn[8];
  if (p0 < P) normals8f(k0, k1, static_cast<uint32_t>(p0 + A.p_offset), static_cast<uint32_t>(A.step), 0u, zc);

  // a0: this tile's ancestor, a1: the next tile's (its copies are issued one tile ahead)
  int a0 = anc_of(p0), a1 = anc_of(p0 + stride);
  int st = 0;
  uint32_t phase[2] = {0u, 0u};
  int start0 = vb < ntiles ? issue(a0, p0 < P, 0) : -1;

  double a_lag = -CUDART_INF;
  bool act_lag = false, real_lag = false;
  int p_lag = P;
  for (int tile = vb; tile < ntiles; tile += nvb) {
    const int p = tile * kPwThreads + threadIdx.x;
    const bool act = p < P;
    const int pn = p + stride;
    const bool has_next = tile + nvb < ntiles;
    const int start1 = has_next ? issue(a1, pn < P, st ^ 1) : -1;
    const int a2 = anc_of(pn + stride);
    if (pn < P) normals8f(k0, k1, static_cast<uint32_t>(pn + A.p_offset), static_cast<uint32_t>(A.step), 0u, zn);
    T x[NX];
    if (start0 >= 0) {
      mbar_wait(&s_bar[warp][st], phase[st]);
      phase[st] ^= 1u;
      const int off = act ? a0 - start0 : 0;
#pragma unroll
      for (int n = 0; n < NX; ++n) x[n] = s_x[(st * NX + n) * kTmaW + off];
    } else {
#pragma unroll
      for (int n = 0; n < NX; ++n) x[n] = act ? xin[static_cast<size_t>(n) * in_stride + a0] : T(0);
    }
    l96_simple_step<T>(x, zc, s_F, s_c, s_s);
#pragma unroll
    for (int n = 0; n < 8; ++n) zc[n] = zn[n];
    if (act) {
#pragma unroll
      for (int n = 0; n < NX; ++n) xout[static_cast<size_t>(n) * out_stride + p] = x[n];
    }
    T sq = T(0);
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const T d = yv[n] - x[n];
      sq = fma(d, d, sq);
    }
    const T g = fma(T(-2.0), sq, -gconst);
    const T lw = uniform_in ? logw0 : Ar<T, false>::sub(aprev[act ? p : 0], static_cast<T>(incr_prev));
    const T a = Ar<T, false>::add(lw, g);
    if (act && aout) aout[p] = a;
    warp_tile_weigh_lag(acc, a_lag, act_lag, p_lag, P, lane, s_exp_tab, cloc, trec, real_lag);
    a_lag = act ? static_cast<double>(a) : -CUDART_INF;
    act_lag = act;
    p_lag = p;
    real_lag = true;
    if (check && act && !bad && !(sq < T(CUDART_INF))) {
      bool ok = true;
#pragma unroll
      for (int n = 0; n < 8; ++n) ok &= finite_bits(x[n]);
      if (!ok) bad = true;
    }
    a0 = a1;
    a1 = a2;
    start0 = start1;
    st ^= 1;
  }
  warp_tile_weigh_lag(acc, a_lag, act_lag, p_lag, P, lane, s_exp_tab, cloc, trec, real_lag);
  warp_tile_flush(acc, lane);

  if (bad) atomicMin(&fs->err_nonfinite, A.step * 64);
  pw_block_finalize<kPwThreads>(A, fs, b, P, R, 1, acc.park->st, lane, kMaxPwBlocks, vb, nvb);
}

}  // namespace ssm
