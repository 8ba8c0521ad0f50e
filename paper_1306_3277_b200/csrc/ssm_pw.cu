// K1/K2: fused ancestor-gather + propagate + weight + LSE/ESS finalize.
//
// One thread per particle, state in registers, SoA coalesced loads/stores.
// Replaces, for one grid step i of ParticleRun._step (particle.py:107-135):
//   x = x[anc]                                  particle.py:102
//   step_transition (sub-steps, noise, RK4)     simulate.py:132-163, 50-60, 71-93
//   observe_logpdf (Gaussian, present slots)    simulate.py:166-193, distributions.py:98-101
//   logw_new = logw + g; incr = logsumexp(...)  particle.py:125-127
//   degenerate check, loglik += incr            particle.py:128-133
//   ESS gate for the next step                  particle.py:99-100
// The LSE/ESS finalize runs in the last block to finish (completion counter),
// combining per-block partials in block order -> deterministic.

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
template <int MODEL, typename T, bool E, bool INJ, bool SIMPLE = false, bool PEER = false>
// NOTE: plain __launch_bounds__(kThreads).  An explicit minBlocks of 1 lets
// ptxas spend 172 registers on the SIMPLE f64 kernel (1 CTA/SM, 0.80 ms
// vs 0.63 ms at 119 registers / 2 CTAs); minBlocks 3 (<= 85) is also slower.
// resident CTAs per SM the register budget is sized for (SIMPLE L96: 3 x 256
// threads = 24 warps at <= 80 registers; profiles/ for the measured variants)
#ifndef SSM_PW_CTAS_SIMPLE
#define SSM_PW_CTAS_SIMPLE (2 * 256 / SSM_PW_THREADS)
#endif
__global__ void __launch_bounds__(kPwThreads, MODEL == SSM_MODEL_WINDKESSEL ? 4 * 256 / kPwThreads
                                              : (SIMPLE ? SSM_PW_CTAS_SIMPLE : 2 * 256 / kPwThreads))
    pw_kernel(const ssm_pw_args A) {
  pdl_wait();
  using O = Ar<T, E>;
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  const int b = blockIdx.y;
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
  const int stride = gridDim.x * kPwThreads;
  const int p0 = blockIdx.x * kPwThreads + threadIdx.x;
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

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
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

  pw_block_finalize<kPwThreads>(A, fs, b, P, R, has_obs, acc.park->st, lane, kMaxPwBlocks);
}

template <int MODEL, typename T, bool PEER>
static void launch_pw_impl(const ssm_pw_args& A, cudaStream_t s) {
  const dim3 grid(pw_grid_x(A.P), A.B);
  const bool inj = A.noise != nullptr;
  if constexpr (MODEL == SSM_MODEL_LORENZ96) {
    // host hint: one sub-step with one RK4 step (any observation mask)
    const bool simple = (A.hints & SSM_HINT_SINGLE_SUBSTEP) && A.n_sub == 1 && !A.exact && !inj;
    if (simple) {
      launch_pdl(pw_kernel<MODEL, T, false, false, true, PEER>, grid, dim3(kPwThreads), s, A);
      return;
    }
  } else {
    // windkessel with one sub-step per grid step (device noise): draws pipelined across tiles
    if ((A.hints & SSM_HINT_SINGLE_SUBSTEP) && A.n_sub == 1 && !inj) {
      if (A.exact)
        launch_pdl(pw_kernel<MODEL, T, true, false, true, PEER>, grid, dim3(kPwThreads), s, A);
      else
        launch_pdl(pw_kernel<MODEL, T, false, false, true, PEER>, grid, dim3(kPwThreads), s, A);
      return;
    }
  }
  if constexpr (PEER) {  // the sharded filter draws on the device
    if (A.exact)
      launch_pdl(pw_kernel<MODEL, T, true, false, false, true>, grid, dim3(kPwThreads), s, A);
    else
      launch_pdl(pw_kernel<MODEL, T, false, false, false, true>, grid, dim3(kPwThreads), s, A);
    return;
  }
  if (A.exact) {
    if (inj)
      launch_pdl(pw_kernel<MODEL, T, true, true>, grid, dim3(kPwThreads), s, A);
    else
      launch_pdl(pw_kernel<MODEL, T, true, false>, grid, dim3(kPwThreads), s, A);
  } else {
    if (inj)
      launch_pdl(pw_kernel<MODEL, T, false, true>, grid, dim3(kPwThreads), s, A);
    else
      launch_pdl(pw_kernel<MODEL, T, false, false>, grid, dim3(kPwThreads), s, A);
  }
}

template <int MODEL, typename T>
static void launch_pw(const ssm_pw_args& A, cudaStream_t s) {
  if (A.x_peer)
    launch_pw_impl<MODEL, T, true>(A, s);
  else
    launch_pw_impl<MODEL, T, false>(A, s);
}

// ----------------------------- K7: init ------------------------------------

template <int MODEL, typename T>
__global__ void __launch_bounds__(kThreads) init_kernel(int P, int p_offset, const uint32_t* keys, T* x) {
  const int b = blockIdx.y;
  const uint32_t k0 = keys[2 * b], k1 = keys[2 * b + 1];
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  T* xb = x + static_cast<size_t>(b) * NX * P;
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads) {
    T v[NX];
    init_one<MODEL, T>(v, static_cast<uint32_t>(p + p_offset), k0, k1);
#pragma unroll
    for (int n = 0; n < NX; ++n) xb[static_cast<size_t>(n) * P + p] = v[n];
  }
}

// ----------------------------- trajectory replay ---------------------------
// (ssm_replay_path) one thread per filter: ancestry walk, then the chosen
// line's states regenerated step by step with the fused kernel's transition.
template <int MODEL, typename T, bool E>
__global__ void replay_kernel(const ssm_replay_args R) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= R.B) return;
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  const int S = R.S;
  double* ob = R.out + static_cast<size_t>(b) * (S + 1) * NX;
  const int32_t* const* ab = R.ancs + static_cast<size_t>(b) * (S + 1);
  const uint32_t* kb = R.keys + static_cast<size_t>(b) * (S + 1) * 2;
  int j = R.j_final[b];
  ob[static_cast<size_t>(S) * NX] = static_cast<double>(j);
  for (int i = S; i > 0; --i) {
    const int32_t* a = ab[i];
    if (a) j = a[j];
    ob[static_cast<size_t>(i - 1) * NX] = static_cast<double>(j);
  }
  T x[NX];
  if (R.x0_flag && R.x0_flag[b]) {
#pragma unroll
    for (int n = 0; n < NX; ++n) x[n] = static_cast<T>(R.x0[static_cast<size_t>(b) * NX + n]);
  } else {
    init_one<MODEL, T>(x, static_cast<uint32_t>(j), kb[0], kb[1]);
  }
#pragma unroll
  for (int n = 0; n < NX; ++n) ob[n] = static_cast<double>(x[n]);
  const double* th = R.theta + 4 * b;
  for (int i = 1; i <= S; ++i) {
    const int ji = static_cast<int>(ob[static_cast<size_t>(i) * NX]);
    const ssm_step_desc& d = R.steps[i];
    const ssm_substep* subs = R.subs + d.subs_offset;
    bool bad = false;
    int bad_sub = 0;
    if constexpr (MODEL == SSM_MODEL_LORENZ96 && !E) {
      if ((d.hints & SSM_HINT_SINGLE_SUBSTEP) && d.n_sub == 1) {  // the fused kernel's SIMPLE choice
        const T s_F = static_cast<T>(th[0]);
        const T s_c = static_cast<T>(th[1] * 20.0 * subs[0].sd);
        const T s_s = static_cast<T>(subs[0].s[0]);
        transition_one<MODEL, T, false, false, true>(x, th, subs, d.n_sub, nullptr, R.P, ji, kb[2 * i],
                                                      kb[2 * i + 1], static_cast<uint32_t>(ji),
                                                      static_cast<uint32_t>(i), s_F, s_c, s_s, false, bad, bad_sub);
      } else {
        transition_one<MODEL, T, false, false, false>(x, th, subs, d.n_sub, nullptr, R.P, ji, kb[2 * i],
                                                       kb[2 * i + 1], static_cast<uint32_t>(ji),
                                                       static_cast<uint32_t>(i), T(0), T(0), T(0), false, bad,
                                                       bad_sub);
      }
    } else {
      transition_one<MODEL, T, E, false, false>(x, th, subs, d.n_sub, nullptr, R.P, ji, kb[2 * i], kb[2 * i + 1],
                                                static_cast<uint32_t>(ji), static_cast<uint32_t>(i), T(0), T(0),
                                                T(0), false, bad, bad_sub);
    }
#pragma unroll
    for (int n = 0; n < NX; ++n) ob[static_cast<size_t>(i) * NX + n] = static_cast<double>(x[n]);
  }
}

}  // namespace ssm

using namespace ssm;

extern "C" size_t ssm_pw_workspace_bytes(int B, int P) {
  (void)P;
  return static_cast<size_t>(B > 0 ? B : 1) * kMaxPwBlocks * sizeof(Lse);
}

extern "C" int ssm_propagate_weight(const ssm_pw_args* args, void* stream) {
  if (!args) return SSM_ERR_INVALID_ARG;
  const ssm_pw_args& A = *args;
  if (A.B <= 0 || A.P <= 0 || A.B > 65535 || A.n_sub < 0 || !A.x_in || !A.x_out || !A.theta ||
      (A.n_sub > 0 && !A.subs) || !A.fs || !A.workspace)
    return SSM_ERR_INVALID_ARG;
  // a_out may be omitted on the tile path (cdf_local set): ssm_advance skips it
  // when the next step resamples from the tile records
  if (A.has_obs && !A.a_out && !A.cdf_local) return SSM_ERR_INVALID_ARG;
  if (A.n_sub > 0 && !A.noise && !A.keys) return SSM_ERR_INVALID_ARG;
  if (A.x_peer && (A.noise || A.peer_n <= 0)) return SSM_ERR_INVALID_ARG;  // sharded: device noise only
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (A.model == SSM_MODEL_GENERIC) return ssm_gen_propagate_weight(A, s);
  if (A.model == SSM_MODEL_LORENZ96) {
    if (A.dtype == SSM_F64)
      launch_pw<SSM_MODEL_LORENZ96, double>(A, s);
    else if (A.dtype == SSM_F32)
      launch_pw<SSM_MODEL_LORENZ96, float>(A, s);
    else
      return SSM_ERR_INVALID_ARG;
  } else if (A.model == SSM_MODEL_WINDKESSEL) {
    if (A.dtype == SSM_F64)
      launch_pw<SSM_MODEL_WINDKESSEL, double>(A, s);
    else if (A.dtype == SSM_F32)
      launch_pw<SSM_MODEL_WINDKESSEL, float>(A, s);
    else
      return SSM_ERR_INVALID_ARG;
  } else {
    return SSM_ERR_UNSUPPORTED;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

template <int MODEL, typename T>
static void launch_replay(const ssm_replay_args& R, cudaStream_t s) {
  const int nt = 64;
  if (R.exact)
    replay_kernel<MODEL, T, true><<<(R.B + nt - 1) / nt, nt, 0, s>>>(R);
  else
    replay_kernel<MODEL, T, false><<<(R.B + nt - 1) / nt, nt, 0, s>>>(R);
}

extern "C" int ssm_replay_path(const ssm_replay_args* args, void* stream) {
  if (!args) return SSM_ERR_INVALID_ARG;
  const ssm_replay_args& R = *args;
  if (R.B <= 0 || R.P <= 0 || R.S < 0 || !R.theta || !R.steps || !R.subs || !R.keys || !R.ancs || !R.j_final ||
      !R.out || (R.x0_flag && !R.x0))
    return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (R.model == SSM_MODEL_LORENZ96) {
    if (R.dtype == SSM_F64)
      launch_replay<SSM_MODEL_LORENZ96, double>(R, s);
    else if (R.dtype == SSM_F32)
      launch_replay<SSM_MODEL_LORENZ96, float>(R, s);
    else
      return SSM_ERR_INVALID_ARG;
  } else if (R.model == SSM_MODEL_WINDKESSEL) {
    if (R.dtype == SSM_F64)
      launch_replay<SSM_MODEL_WINDKESSEL, double>(R, s);
    else if (R.dtype == SSM_F32)
      launch_replay<SSM_MODEL_WINDKESSEL, float>(R, s);
    else
      return SSM_ERR_INVALID_ARG;
  } else {
    return SSM_ERR_UNSUPPORTED;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_init_particles(int model, int dtype, int B, int P, int p_offset, const uint32_t* keys,
                                  void* x_out, void* stream) {
  if (B <= 0 || P <= 0 || B > 65535 || !keys || !x_out) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 grid(pw_grid_x(P), B);
  if (model == SSM_MODEL_LORENZ96) {
    if (dtype == SSM_F64)
      init_kernel<SSM_MODEL_LORENZ96, double><<<grid, kThreads, 0, s>>>(P, p_offset, keys, (double*)x_out);
    else
      init_kernel<SSM_MODEL_LORENZ96, float><<<grid, kThreads, 0, s>>>(P, p_offset, keys, (float*)x_out);
  } else if (model == SSM_MODEL_WINDKESSEL) {
    if (dtype == SSM_F64)
      init_kernel<SSM_MODEL_WINDKESSEL, double><<<grid, kThreads, 0, s>>>(P, p_offset, keys, (double*)x_out);
    else
      init_kernel<SSM_MODEL_WINDKESSEL, float><<<grid, kThreads, 0, s>>>(P, p_offset, keys, (float*)x_out);
  } else {
    return SSM_ERR_UNSUPPORTED;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// ----------------------------- device-noise export -------------------------

namespace ssm {
__global__ void __launch_bounds__(kThreads) normals_kernel(int model, int P, int p_offset, const uint32_t* keys,
                                                           int step, int sub, float* out) {
  const int b = blockIdx.y;
  const uint32_t k0 = keys[2 * b], k1 = keys[2 * b + 1];
  const int nx = model == SSM_MODEL_LORENZ96 ? 8 : 1;
  float* ob = out + static_cast<size_t>(b) * nx * P;
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads) {
    const uint32_t pg = static_cast<uint32_t>(p + p_offset);
    if (model == SSM_MODEL_LORENZ96) {
      float z[8];
      normals8f(k0, k1, pg, static_cast<uint32_t>(step), static_cast<uint32_t>(sub), z);
#pragma unroll
      for (int n = 0; n < 8; ++n) ob[static_cast<size_t>(n) * P + p] = z[n];
    } else {
      ob[p] = normal1<float>(k0, k1, pg, static_cast<uint32_t>(step), static_cast<uint32_t>(sub));
    }
  }
}
}  // namespace ssm

extern "C" int ssm_device_normals(int model, int B, int P, int p_offset, const uint32_t* keys, int step, int sub,
                                  float* out, void* stream) {
  if (B <= 0 || P <= 0 || B > 65535 || !keys || !out || sub < 0) return SSM_ERR_INVALID_ARG;
  if (model != SSM_MODEL_LORENZ96 && model != SSM_MODEL_WINDKESSEL) return SSM_ERR_UNSUPPORTED;
  const dim3 grid(pw_grid_x(P), B);
  ssm::normals_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(model, P, p_offset, keys, step, sub,
                                                                               out);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// ----------------------------- C1: cross-rank finalize ----------------------

namespace ssm {
__global__ void lse_combine_kernel(int W, int B, const double* parts, ssm_filter_state* fs, double ess_rel,
                                   double P_total, int step) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Lse acc = lse_empty();
  for (int r = 0; r < W; ++r) {  // rank order: deterministic
    const double* q = parts + (static_cast<size_t>(r) * B + b) * 4;
    acc = lse_combine(acc, Lse{q[0], q[1], q[2], q[3]});
  }
  ssm_filter_state* f = fs + b;
  const double incr = lse_value(acc);
  const double ess = lse_ess(acc);
  if (!isfinite(incr)) {
    f->err_degenerate = min(f->err_degenerate, step);
  } else {
    f->loglik += incr;
  }
  f->incr = incr;
  f->lse_raw = incr;
  f->ess = ess;
  f->uniform = 0;
  f->resample_now = (ess_rel < 0.0) ? 1 : (ess < ess_rel * P_total ? 1 : 0);
}
}  // namespace ssm

extern "C" int ssm_lse_combine(int W, int B, const double* parts, ssm_filter_state* fs, double ess_rel,
                               double P_total, int step, void* stream) {
  if (W <= 0 || B <= 0 || !parts || !fs) return SSM_ERR_INVALID_ARG;
  ssm::lse_combine_kernel<<<(B + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(W, B, parts, fs, ess_rel,
                                                                                          P_total, step);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}
