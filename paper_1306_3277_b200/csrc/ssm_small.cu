// Persistent small-P filter: ONE launch advances B filters through all their
// grid steps, one CTA per filter (device-noise mode).  For P <= 4096 the
// multi-kernel path is launch/latency bound (~5 small kernels per step); here
// the log-weights, the resampling CDF and the ancestors stay in shared memory,
// positions stream through global memory (the history, L2-resident at this
// size), and the step-to-step dependency is a __syncthreads.
//
// Semantics per step (particle.py:96-135), as in the multi-kernel path:
//   resample if fs.resample_now: cum_j = C_j / C_tot over an exact 64-bit
//   fixed-point block scan of w_j = exp(a_j - incr); ancestors by binary
//   search on the reference's float64 query values (resampling.py:28-36);
//   propagate / weight with the same device functions; scipy-form LSE/ESS
//   block reduction and finalize.  Ancestors are written for every step
//   (identity when no resampling happened, like the reference's arange).

#include "ssm_common.cuh"
#include "ssm_models.cuh"

namespace ssm {

constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxP = 4096;
constexpr double kFix61 = 2305843009213693952.0;  // 2^61

__device__ __forceinline__ double device_uniform_small(uint32_t k0, uint32_t k1, uint32_t k, uint32_t step,
                                                       uint32_t purpose) {
  const U4 r = philox4x32_10(U4{k, step, 0u, purpose}, k0, k1);  // same stream as the multi-kernel search
  return u53(r.x, r.y);
}

template <int MODEL, typename T, bool E>
__device__ __forceinline__ T small_obs(const T* x, const double* th, const ssm_step_desc& d, T obs_log_sd, T lsp) {
  using O = Ar<T, E>;
  T g = T(0);
  if constexpr (MODEL == SSM_MODEL_LORENZ96) {
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      if (d.obs_mask & (1u << n)) {
        const T z = O::mul(O::sub(static_cast<T>(d.y[n]), x[n]), T(2.0));
        g = O::add(g, O::sub(O::sub(O::mul(O::mul(T(-0.5), z), z), obs_log_sd), lsp));
      }
    }
  } else {
    const T mean = O::add(x[0], O::mul(static_cast<T>(th[2]), static_cast<T>(d.u_obs)));
    const T z = O::mul(O::sub(static_cast<T>(d.y[0]), mean), T(0.5));
    g = O::add(g, O::sub(O::sub(O::mul(O::mul(T(-0.5), z), z), obs_log_sd), lsp));
  }
  return g;
}

__device__ __forceinline__ uint64_t block_excl_scan_u64(uint64_t v, uint64_t* warp_tot, uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint64_t wex = 0, tot = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) {
    const uint64_t t = warp_tot[w];
    if (w < warp) wex += t;
    tot += t;
  }
  *total = tot;
  __syncthreads();
  return wex + incl - v;
}

// XS: positions double-buffered in shared memory (history still streamed to
// global memory); otherwise read back from the global history (L2).
template <int MODEL, typename T, bool E, bool XS>
__global__ void __launch_bounds__(kSmallThreads) small_filter_kernel(const ssm_small_args A) {
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  extern __shared__ __align__(16) unsigned char smem[];
  const int P = A.P;
  T* a_s = reinterpret_cast<T*>(smem);                                                       // [P]
  double* cum_s = reinterpret_cast<double*>(smem + ((sizeof(T) * P + 15) & ~size_t(15)));  // [P]
  int32_t* anc_s = reinterpret_cast<int32_t*>(cum_s + P);                                    // [P]
  T* xs0 = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(anc_s) + ((sizeof(int32_t) * P + 15) & ~size_t(15)));
  T* xs1 = xs0 + static_cast<size_t>(NX) * P;  // XS only: [NX][P] x 2
  __shared__ uint64_t warp_tot[kSmallThreads / 32];
  __shared__ Lse red[kSmallThreads / 32];
  __shared__ ssm_filter_state s_fs;  // the filter state lives in shared memory during the launch
  __shared__ double s_usys;

  const int b = blockIdx.x;
  ssm_filter_state* fs = A.fs + b;
  const double* th = A.theta + 4 * b;
  const uint32_t k0 = A.keys[2 * b], k1 = A.keys[2 * b + 1];
  const T obs_log_sd = static_cast<T>(A.obs_log_sd);
  const T lsp = static_cast<T>(A.log_sqrt_2pi);
  const T logw0 = static_cast<T>(A.log_w0);
  const int ipt = (P + blockDim.x - 1) / blockDim.x;  // contiguous chunk per thread for the scan
  const size_t xstride_b = static_cast<size_t>(NX) * P;

  if (threadIdx.x == 0) s_fs = *fs;
  if (A.a_prev) {
    const T* ap = static_cast<const T*>(A.a_prev) + static_cast<size_t>(b) * P;
    for (int p = threadIdx.x; p < P; p += blockDim.x) a_s[p] = ap[p];
  }
  const T* x_prev_g = static_cast<const T*>(A.x_in) + static_cast<size_t>(b) * xstride_b;
  if constexpr (XS) {
    for (int e = threadIdx.x; e < NX * P; e += blockDim.x) xs0[e] = x_prev_g[e];
  }
  T* xcur = xs0;
  T* xnext = xs1;
  bool bad = false;
  int bad_step = 0, bad_sub = 0;
  __syncthreads();

  for (int k = 0; k < A.n_steps; ++k) {
    const ssm_step_desc& d = A.steps[k];
    const int R = s_fs.resample_now;
    const double incr_prev = s_fs.incr;
    int32_t* anc_g = A.anc_arena + (static_cast<size_t>(k) * A.B + b) * P;
    if (R) {
      if (threadIdx.x == 0) s_usys = device_uniform_small(k0, k1, 0u, static_cast<uint32_t>(d.step), kPurposeSystematic);
      // exact 64-bit CDF of w = exp(a - incr) (resampling.py:26-27)
      const int j0 = threadIdx.x * ipt;
      uint64_t local = 0;
      for (int i = 0; i < ipt; ++i) {
        const int j = j0 + i;
        if (j < P) {
          const double w = exp(static_cast<double>(a_s[j]) - incr_prev);
          const uint64_t q = (w >= 0.0 && w <= 4.0) ? __double2ull_rn(w * kFix61) : 0ull;
          cum_s[j] = __longlong_as_double(static_cast<long long>(q));  // stash q
          local += q;
        }
      }
      uint64_t tot;
      uint64_t run = block_excl_scan_u64(local, warp_tot, &tot);
      const double inv_tot = 1.0 / static_cast<double>(tot);
      for (int i = 0; i < ipt; ++i) {
        const int j = j0 + i;
        if (j < P) {
          run += static_cast<uint64_t>(__double_as_longlong(cum_s[j]));
          cum_s[j] = j == P - 1 ? 1.0 : static_cast<double>(run) * inv_tot;  // cum[-1] = 1
        }
      }
      __syncthreads();
      // queries and searchsorted(cum, u, 'right').clip(0, P-1)  (resampling.py:28-36)
      const double u_sys = s_usys;
      for (int q = threadIdx.x; q < P; q += blockDim.x) {
        double u;
        if (A.scheme == SSM_SYSTEMATIC) {
          u = (static_cast<double>(q) + u_sys) / static_cast<double>(P);
        } else {
          const double U = device_uniform_small(k0, k1, static_cast<uint32_t>(q), static_cast<uint32_t>(d.step),
                                                kPurposeResample);
          u = A.scheme == SSM_STRATIFIED ? (static_cast<double>(q) + U) / static_cast<double>(P) : U;
        }
        int lo = 0, hi = P;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (cum_s[mid] <= u)
            lo = mid + 1;
          else
            hi = mid;
        }
        const int a_idx = lo < P ? lo : P - 1;
        anc_s[q] = a_idx;
        anc_g[q] = a_idx;
      }
    } else {
      for (int q = threadIdx.x; q < P; q += blockDim.x) anc_g[q] = q;  // identity (reference: arange)
    }
    __syncthreads();
    // propagate + weight
    T* x_out = static_cast<T*>(A.x_arena) + (static_cast<size_t>(k) * A.B + b) * xstride_b;
    const bool uni = R || s_fs.uniform;
    Lse st = lse_empty();
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      const int src = R ? anc_s[p] : p;
      T x[NX];
#pragma unroll
      for (int n = 0; n < NX; ++n) x[n] = XS ? xcur[n * P + src] : x_prev_g[static_cast<size_t>(n) * P + src];
      bool b_now = false;
      int bs = 0;
      // the fused kernel's general (non-SIMPLE) transition: the same draws and arithmetic
      transition_one<MODEL, T, E, false, false>(x, th, A.subs + d.subs_offset, d.n_sub, nullptr, P, p, k0, k1,
                                                static_cast<uint32_t>(p), static_cast<uint32_t>(d.step), T(0), T(0),
                                                T(0), A.check_finite != 0, b_now, bs);
      if (b_now && !bad) {
        bad = true;
        bad_step = d.step;
        bad_sub = bs;
      }
#pragma unroll
      for (int n = 0; n < NX; ++n) {
        x_out[static_cast<size_t>(n) * P + p] = x[n];
        if constexpr (XS) xnext[n * P + p] = x[n];
      }
      if (d.has_obs) {
        const T g = small_obs<MODEL, T, E>(x, th, d, obs_log_sd, lsp);
        const T lw = uni ? logw0 : Ar<T, E>::sub(a_s[p], static_cast<T>(incr_prev));
        const T a = Ar<T, E>::add(lw, g);
        a_s[p] = a;  // each thread owns its p: in-place is safe after the resample read above
        lse_push(st, static_cast<double>(a));
      }
    }
    if (d.has_obs) {
      const Lse r = lse_block_reduce<kSmallThreads>(st, red);
      if (threadIdx.x == 0) {
        const double incr = lse_value(r);
        const double ess = lse_ess(r);
        if (!isfinite(incr)) {
          s_fs.err_degenerate = min(s_fs.err_degenerate, d.step);
        } else {
          s_fs.loglik += incr;
        }
        s_fs.incr = incr;
        s_fs.lse_raw = incr;
        s_fs.ess = ess;
        s_fs.uniform = 0;
        s_fs.resample_now = (A.ess_rel < 0.0) ? 1 : (ess < A.ess_rel * static_cast<double>(P) ? 1 : 0);
      }
    } else if (threadIdx.x == 0 && R) {
      s_fs.uniform = 1;
      s_fs.resample_now = 0;
    }
    __syncthreads();
    if constexpr (XS) {
      T* t = xcur;
      xcur = xnext;
      xnext = t;
    } else {
      x_prev_g = x_out;
    }
  }
  if (bad) atomicMin(&s_fs.err_nonfinite, bad_step * 64 + bad_sub);
  __syncthreads();
  if (threadIdx.x == 0) *fs = s_fs;
  if (A.a_out) {
    T* ao = static_cast<T*>(A.a_out) + static_cast<size_t>(b) * P;
    for (int p = threadIdx.x; p < P; p += blockDim.x) ao[p] = a_s[p];
  }
}

template <int MODEL, typename T>
static int launch_small(const ssm_small_args& A, cudaStream_t s) {
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  const size_t base = ((sizeof(T) * A.P + 15) & ~size_t(15)) + sizeof(double) * A.P +
                      ((sizeof(int32_t) * A.P + 15) & ~size_t(15));
  const size_t with_x = base + 2 * sizeof(T) * NX * A.P;
  const bool xs = with_x <= 200 * 1024;
  const size_t sm = xs ? with_x : base;
  const int threads = kSmallThreads;  // block reductions assume a full block
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    kern<<<A.B, threads, sm, s>>>(A);
  };
  if (A.exact) {
    if (xs)
      go(small_filter_kernel<MODEL, T, true, true>);
    else
      go(small_filter_kernel<MODEL, T, true, false>);
  } else {
    if (xs)
      go(small_filter_kernel<MODEL, T, false, true>);
    else
      go(small_filter_kernel<MODEL, T, false, false>);
  }
  return SSM_OK;
}

}  // namespace ssm

using namespace ssm;

extern "C" int ssm_small_max_particles(void) { return kSmallMaxP; }

extern "C" int ssm_advance_small(const ssm_small_args* args, void* stream) {
  if (!args) return SSM_ERR_INVALID_ARG;
  const ssm_small_args& A = *args;
  if (A.B <= 0 || A.P < 2 || A.P > kSmallMaxP || A.n_steps < 0 || !A.x_in || !A.x_arena || !A.anc_arena ||
      !A.theta || !A.keys || !A.fs || !A.steps || !A.subs)
    return SSM_ERR_INVALID_ARG;
  if (A.scheme < SSM_MULTINOMIAL || A.scheme > SSM_SYSTEMATIC) return SSM_ERR_INVALID_ARG;
  if (A.n_steps == 0) return SSM_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (A.model == SSM_MODEL_LORENZ96) {
    if (A.dtype == SSM_F64)
      launch_small<SSM_MODEL_LORENZ96, double>(A, s);
    else
      launch_small<SSM_MODEL_LORENZ96, float>(A, s);
  } else if (A.model == SSM_MODEL_WINDKESSEL) {
    if (A.dtype == SSM_F64)
      launch_small<SSM_MODEL_WINDKESSEL, double>(A, s);
    else
      launch_small<SSM_MODEL_WINDKESSEL, float>(A, s);
  } else {
    return SSM_ERR_UNSUPPORTED;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}
