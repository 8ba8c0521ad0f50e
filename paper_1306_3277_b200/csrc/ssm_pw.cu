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


#include <cstdlib>

#include "ssm_pw_body.cuh"

namespace ssm {

// Resident CTAs per SM the register budget is sized for: 2 x 256 threads for
// L96 (an explicit minBlocks of 1 lets ptxas spend 172 registers on the SIMPLE
// f64 kernel: 0.80 ms vs 0.63 ms at 2 CTAs; 3 CTAs / SM (<= 80 registers)
// spills and is slower: profiles/r2_ab.txt), 4 for the windkessel.
#ifndef SSM_PW_CTAS_SIMPLE
#define SSM_PW_CTAS_SIMPLE (2 * 256 / SSM_PW_THREADS)
#endif
template <int MODEL, typename T, bool E, bool INJ, bool SIMPLE = false, bool PEER = false>
__global__ void __launch_bounds__(kPwThreads, MODEL == SSM_MODEL_WINDKESSEL ? 4 * 256 / kPwThreads
                                              : (SIMPLE ? SSM_PW_CTAS_SIMPLE : 2 * 256 / kPwThreads))
    pw_kernel(const ssm_pw_args A) {
  pdl_wait();
  pw_body<MODEL, T, E, INJ, SIMPLE, PEER>(A, blockIdx.y, blockIdx.x, gridDim.x);
}

// The headline step with the warp-tile weighting lagged one tile (pw_body_lag).
template <typename T>
__global__ void __launch_bounds__(kPwThreads, SSM_PW_CTAS_SIMPLE) pw_lag_kernel(const ssm_pw_args A) {
  pdl_wait();
  pw_body_lag<T>(A, blockIdx.y, blockIdx.x, gridDim.x);
}

// the lagged headline step with the TMA-staged gather (pw_body_lag_tma; A/B: SSM_PW_TMA=1)
template <typename T>
__global__ void __launch_bounds__(kPwThreads, SSM_PW_CTAS_SIMPLE) pw_lag_tma_kernel(const ssm_pw_args A) {
  pdl_wait();
  pw_body_lag_tma<T>(A, blockIdx.y, blockIdx.x, gridDim.x);
}

static bool pw_tma_enabled() {
  static const bool on = std::getenv("SSM_PW_TMA") != nullptr;
  return on;
}

template <typename T>
static cudaError_t launch_lag_tma(const ssm_pw_args& A, dim3 grid, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kPwThreads / 32) * 2 * 8 * kTmaW * sizeof(T);
  static bool attr = false;  // per T (one instantiation per static)
  if (!attr) {
    cudaFuncSetAttribute(pw_lag_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  return launch_pdl_smem(pw_lag_tma_kernel<T>, grid, dim3(kPwThreads), smem, s, A);
}

// SSM_NO_PW_LAG=1 in the environment selects pw_body for the headline step too (A/B)
static bool pw_lag_enabled() {
  static const bool on = std::getenv("SSM_NO_PW_LAG") == nullptr;
  return on;
}

template <int MODEL, typename T, bool PEER>
static void launch_pw_impl(const ssm_pw_args& A, cudaStream_t s) {
  const dim3 grid(pw_grid_x(A.P), A.B);
  const bool inj = A.noise != nullptr;
  if constexpr (MODEL == SSM_MODEL_LORENZ96) {
    // host hint: one sub-step with one RK4 step (any observation mask)
    const bool simple = (A.hints & SSM_HINT_SINGLE_SUBSTEP) && A.n_sub == 1 && !A.exact && !inj;
    if (simple) {
      if constexpr (!PEER) {
        if (A.has_obs && A.obs_mask == 0xFFu && A.ess_rel < 0.0 && A.cdf_local && A.tile_rec && A.keys &&
            pw_lag_enabled()) {
          const int in_stride = A.x_in_stride > 0 ? A.x_in_stride : A.P;
          if (pw_tma_enabled() && (in_stride % 4) == 0) {  // 16-byte aligned rows
            launch_lag_tma<T>(A, grid, s);
            return;
          }
          launch_pdl(pw_lag_kernel<T>, grid, dim3(kPwThreads), s, A);
          return;
        }
      }
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
