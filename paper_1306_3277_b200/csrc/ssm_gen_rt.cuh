// Generic-model kernels.  Compiled at run time by NVRTC
// (csrc/ssm_gen.cu) together with a generated `gen::Model`, which
// paper_1306_3277_b200/codegen.py lowers from a reference ModelIr
// (core/ir.py:83-121).  The generated model provides, per particle:
//
//   NX, NW, NWB (= max(NW, 1)), NU (inputs), KDRAW (draws per transition sub-step)
//   substep<T, E, INJ>(X, W, TH, U, d, draws, perr)  one transition sub-step
//        (simulate.py:132-163: the block's statements in order, sample /
//         assign / RK4 ode, with the reference's op order under E)
//   obs_logpdf<T, E>(X, W, TH, U, Y, mask, perr) sum over present obs slots
//        (simulate.py:166-193, distributions.py:94-123)
//   initial<T, E, INJ>(X, TH, draws, perr)       the initial block
//        (simulate.py:111-129)
//
// The kernels below are the generic counterparts of pw_kernel / init_kernel:
// the same ancestor gather, software pipeline, warp-tile weighting and fused
// LSE/ESS finalize (ssm_tile.cuh), so resampling downstream is shared.
#pragma once

#include "ssm_tile.cuh"

namespace ssm {

// np.mod on floats (numpy npy_divmod): the result takes the divisor's sign
template <typename T>
__device__ __forceinline__ T py_mod(T a, T b) {
  T m = fmod(a, b);
  if (b == T(0)) return m;
  if (m != T(0)) {
    if ((b < T(0)) != (m < T(0))) m += b;
  } else {
    m = copysign(T(0), b);
  }
  return m;
}

// Draws of one (particle, grid step, sub-step).  Device mode: Philox4x32-10
// blocks {particle, step, sub << 8 | block, kPurposeGen | retry << 8}; the
// generated code takes each block once and spends its four words on two
// Box-Muller pairs (four normals) or two 53-bit uniforms (codegen's draw plan).
// Injected mode (noise="host"): the reference's standard variates, [KDRAW][P]
// per sub-step, by draw index.
template <typename T>
struct GenDraws {
  uint32_t k0, k1, pg, step, sub;
  const T* inj;
  int P, p;

  __device__ __forceinline__ U4 block(int b, uint32_t retry = 0u) const {
    return philox4x32_10(U4{pg, step, (sub << 8) | static_cast<uint32_t>(b), kPurposeGen | (retry << 8)}, k0, k1);
  }
  // the injected variate of draw kd (INJ), else the device value
  template <bool INJ>
  __device__ __forceinline__ T pick(int kd, T device_value) const {
    if constexpr (INJ) return inj[static_cast<size_t>(kd) * P + p];
    else return device_value;
  }
  // standard gamma(shape) by Marsaglia-Tsang (device draws only, own counters:
  // block = draw index, retries 1..254, the shape < 1 boost uniform at 255);
  // shape < 1 through gamma(shape + 1) U^(1/shape)
  __device__ __forceinline__ double std_gamma(int kd, double shape) const {
    double boost = 1.0;
    if (shape < 1.0) {
      const U4 r = block(kd, 255u);
      boost = pow(1.0 - u53(r.z, r.w), 1.0 / shape);
      shape += 1.0;
    }
    const double dd = shape - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * dd);
    for (uint32_t it = 1; it < 255; ++it) {
      const U4 r = block(kd, it);
      float z0, z1;
      box_muller(r.x, r.y, z0, z1);
      const double z = z0;
      double v = 1.0 + c * z;
      if (v <= 0.0) continue;
      v = v * v * v;
      const double u = 1.0 - u53(r.z, r.w);
      if (log(u) < 0.5 * z * z + dd - dd * v + dd * log(v)) return dd * v * boost;
    }
    return dd * boost;  // not reached in practice (acceptance > 0.95 per try)
  }
};

// SIMPLE (host hint SSM_HINT_SINGLE_SUBSTEP, device draws, fast mode): one
// sub-step per grid step whose ode statements each take one RK4 step -- the
// sub-step loop and the RK4 step loops disappear and the sub-step record is
// read once per block.
template <class M, typename T, bool E, bool INJ, bool SIMPLE = false>
__global__ void __launch_bounds__(kPwThreads, 2) gen_pw_kernel(const ssm_pw_args A) {
  pdl_wait();
  constexpr int NX = M::NX;
  const int b = blockIdx.y;
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
  uint64_t* __restrict__ cloc =
      A.cdf_local ? static_cast<uint64_t*>(A.cdf_local) + static_cast<size_t>(b) * P : nullptr;
  ssm_tile_rec* __restrict__ trec =
      A.tile_rec ? static_cast<ssm_tile_rec*>(A.tile_rec) + static_cast<size_t>(b) * ((P + 31) >> 5) : nullptr;
  const T* __restrict__ noise =
      INJ ? static_cast<const T*>(A.noise) + static_cast<size_t>(b) * A.n_sub * M::KDRAW * P : nullptr;
  const double* th = A.theta + static_cast<size_t>(A.theta_stride) * b;
  const uint32_t k0 = (!INJ && A.keys) ? A.keys[2 * b] : 0u, k1 = (!INJ && A.keys) ? A.keys[2 * b + 1] : 0u;
  const int has_obs = A.has_obs;
  const T logw0 = static_cast<T>(A.log_w0);
  const int lane = threadIdx.x & 31;
  const bool want_ess = A.ess_rel >= 0.0;

  __shared__ double s_exp_tab[64];
  if (threadIdx.x < 64) s_exp_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
  __syncthreads();
  __shared__ ParkedTiles s_park[kPwThreads / 32];
  WarpTileAcc acc = warp_tile_acc(&s_park[threadIdx.x >> 5], lane);
  bool bad = false, perr = false;
  int bad_sub = 0, perr_sub = 0;

  // software pipeline as pw_kernel: next tile's gathered state in flight
  T xn[NX];
  const int stride = gridDim.x * kPwThreads;
  const int p0 = blockIdx.x * kPwThreads + threadIdx.x;
  // sharded filter (A.x_peer): global ancestor indices, gathered from the owning rank
  const bool peer = A.x_peer != nullptr;
  const int src_off = peer ? A.p_offset : 0;
  auto load_x = [&](int src) {
    const T* base = xin;
    if (peer) {
      const int loc = src - A.p_offset;
      if (static_cast<unsigned>(loc) < static_cast<unsigned>(A.peer_n)) {
        src = loc;
      } else {
        const int o = src / A.peer_n;
        base = static_cast<const T*>(A.x_peer[o]) + static_cast<size_t>(b) * NX * in_stride;
        src -= o * A.peer_n;
      }
    }
#pragma unroll
    for (int n = 0; n < NX; ++n) xn[n] = base[static_cast<size_t>(n) * in_stride + src];
  };
  if (p0 < P) load_x(anc ? __ldg(anc + p0) : p0 + src_off);
  int anc_next = (anc && p0 + stride < P) ? __ldg(anc + p0 + stride) : p0 + stride + src_off;

  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int p = tile * kPwThreads + threadIdx.x;
    const bool act = p < P;
    double a_d = -CUDART_INF;
    T x[NX];
#pragma unroll
    for (int n = 0; n < NX; ++n) x[n] = xn[n];
    {
      const int p2 = p + stride;
      if (p2 < P) load_x(anc_next);
      const int p3 = p2 + stride;
      anc_next = (anc && p3 < P) ? __ldg(anc + p3) : p3 + src_off;
    }
    if (act) {
      T w[M::NWB];  // the noise array of step_transition: zeros, then rewritten per sub-step
#pragma unroll
      for (int n = 0; n < M::NWB; ++n) w[n] = T(0);
      const int n_sub = SIMPLE ? 1 : A.n_sub;
      for (int k = 0; k < n_sub; ++k) {
        const ssm_substep& S = A.subs[k];
        const double* U = A.u_vec ? A.u_vec + static_cast<size_t>(k) * M::NU : &S.u_in;
        const GenDraws<T> dr{k0, k1, static_cast<uint32_t>(p + A.p_offset), static_cast<uint32_t>(A.step),
                             static_cast<uint32_t>(k), INJ ? noise + static_cast<size_t>(k) * M::KDRAW * P : nullptr,
                             P, p};
        bool pe = false;
        M::template substep<T, E, INJ, SIMPLE>(x, w, th, U, S.d, dr, pe);
        if (pe && !perr) {
          perr = true;
          perr_sub = k;
        }
        if (A.check_finite && !bad) {
          bool ok = true;
#pragma unroll
          for (int n = 0; n < NX; ++n) ok &= finite_bits(x[n]);
          if (!ok) {
            bad = true;
            bad_sub = k;
          }
        }
      }
#pragma unroll
      for (int n = 0; n < NX; ++n) xout[static_cast<size_t>(n) * out_stride + p] = x[n];
      if (has_obs) {
        T w0[M::NWB];  // observe_logpdf sees a zero noise array (simulate.py:181)
#pragma unroll
        for (int n = 0; n < M::NWB; ++n) w0[n] = T(0);
        const double* Uo = A.u_vec ? A.u_vec + static_cast<size_t>(A.n_sub) * M::NU : &A.u_obs;
        const double* Y = A.y_vec ? A.y_vec : A.y;
        bool pe = false;
        const T g = M::template obs_logpdf<T, E>(x, w0, th, Uo, Y, A.obs_mask, pe);
        if (pe && !perr) {
          perr = true;
          perr_sub = 63;  // the observation density at this step
        }
        const T lw = uniform_in ? logw0 : Ar<T, E>::sub(aprev[p], static_cast<T>(incr_prev));
        const T a = Ar<T, E>::add(lw, g);
        if (aout) aout[p] = a;
        a_d = static_cast<double>(a);
      }
    }
    if (!has_obs) continue;  // block-uniform
    warp_tile_weigh(acc, a_d, act, p, P, lane, s_exp_tab, cloc, trec, want_ess);
  }
  warp_tile_flush(acc, lane);

  if (bad) atomicMin(&fs->err_nonfinite, A.step * 64 + bad_sub);
  if (perr) atomicMin(&fs->err_param, A.step * 64 + perr_sub);
  pw_block_finalize<kPwThreads>(A, fs, b, P, R, has_obs, acc.park->st, lane, kMaxPwBlocks, blockIdx.x, gridDim.x);
}

// the model's initial block on the device (sample_initial, simulate.py:111-129)
template <class M, typename T>
__global__ void __launch_bounds__(kPwThreads)
    gen_init_kernel(int P, int p_offset, const uint32_t* keys, const double* theta, int theta_stride, T* x,
                    ssm_filter_state* fs) {
  constexpr int NX = M::NX;
  const int b = blockIdx.y;
  const uint32_t k0 = keys[2 * b], k1 = keys[2 * b + 1];
  const double* th = theta + static_cast<size_t>(theta_stride) * b;
  T* xb = x + static_cast<size_t>(b) * NX * P;
  bool perr = false;
  for (int p = blockIdx.x * kPwThreads + threadIdx.x; p < P; p += gridDim.x * kPwThreads) {
    T X[NX];
#pragma unroll
    for (int n = 0; n < NX; ++n) X[n] = T(0);
    const GenDraws<T> dr{k0, k1, static_cast<uint32_t>(p + p_offset), 0u, 0u, nullptr, P, p};
    bool pe = false;
    M::template initial<T, true, false>(X, th, dr, pe);
    perr |= pe;
#pragma unroll
    for (int n = 0; n < NX; ++n) xb[static_cast<size_t>(n) * P + p] = X[n];
  }
  if (perr && fs) atomicMin(&fs[b].err_param, 0);
}


// ---------------------------------------------------------------------------
// Theta-level blocks of a generated model (SURVEY 8f row 1 for generic models):
// the generated `M::Theta` walks proposal_parameter / proposal_initial (or the
// parameter / initial blocks when a proposal is absent) with the reference's
// sequential-overwrite semantics (simulate.py:264-299) and evaluates the
// priors (simulate.py:219-233); the kernel below strings them together like
// GenericModel.propose_batch / mcmc._propose (mcmc.py:138-148), one thread
// per chain.  ssm_theta_accept (ssm_theta.cu) applies the accept.
//
// Draws by index kd (the proposal walk's statements and slots in order, then
// the initial walk's): injected standard variates (u_in row: the uniform of a
// uniform / truncated-Gaussian draw, the standard normal of a Gaussian, the
// standard gamma of a (inverse-)gamma -- the reference's own numpy draws) or
// Philox blocks {kd, retry, step, kPurposeGenTheta} on the chain's key.
// All arithmetic is float64 with one rounding per operation (numpy order);
// log / lgamma / normcdf / normcdfinv are CUDA's (a few ulp from numpy/scipy).
constexpr uint32_t kPurposeGenTheta = 8u;
constexpr double kThLogSqrt2Pi = 0.91893853320467274178;  // distributions.py:15

struct ThetaDraws {
  const ssm_theta_args* A;
  int c;
  __device__ __forceinline__ U4 block(int kd, uint32_t retry) const {
    return philox4x32_10(U4{static_cast<uint32_t>(kd), retry, static_cast<uint32_t>(A->step), kPurposeGenTheta},
                         A->keys[2 * c], A->keys[2 * c + 1]);
  }
  __device__ __forceinline__ double injected(int kd) const {
    return A->u_in[static_cast<size_t>(c) * A->u_stride + kd];
  }
  __device__ double uniform(int kd) const {
    if (A->u_in) return injected(kd);
    const U4 r = block(kd, 0u);
    return u53(r.x, r.y);
  }
  __device__ double normal(int kd) const {
    if (A->u_in) return injected(kd);
    const U4 r = block(kd, 0u);
    double z0, z1;
    box_muller(r.x, r.y, r.z, r.w, z0, z1);
    return z0;
  }
  // standard gamma(shape): Marsaglia-Tsang, try `it` on blocks 2it+1 (normal) and
  // 2it+2 (uniform); shape < 1 through gamma(shape + 1) U^(1/shape) (block 0)
  __device__ double std_gamma(int kd, double shape) const {
    if (A->u_in) return injected(kd);
    if (!(shape > 0.0)) return CUDART_NAN;
    double boost = 1.0;
    if (shape < 1.0) {
      const U4 r = block(kd, 0u);
      boost = pow(1.0 - u53(r.x, r.y), 1.0 / shape);
      shape += 1.0;
    }
    const double dd = shape - 1.0 / 3.0, cc = 1.0 / sqrt(9.0 * dd);
    for (uint32_t it = 0; it < 1000u; ++it) {
      const U4 rz = block(kd, 2u * it + 1u), ru = block(kd, 2u * it + 2u);
      double z, z1;
      box_muller(rz.x, rz.y, rz.z, rz.w, z, z1);
      double v = 1.0 + cc * z;
      if (v <= 0.0) continue;
      v = v * v * v;
      const double u = 1.0 - u53(ru.x, ru.y);
      if (log(u) < 0.5 * z * z + dd - dd * v + dd * log(v)) return dd * v * boost;
    }
    return dd * boost;  // not reached in practice (acceptance > 0.95 per try)
  }
};

// distributions.sample (distributions.py:73-91) from a standard variate
__device__ __forceinline__ double th_sample_gaussian(const ThetaDraws& dr, int kd, const double* a, bool& perr) {
  if (!(a[1] > 0.0)) perr = true;
  return __dadd_rn(a[0], __dmul_rn(a[1], dr.normal(kd)));  // numpy: loc + scale * z
}
__device__ __forceinline__ double th_sample_uniform(const ThetaDraws& dr, int kd, const double* a, bool& perr) {
  if (!(a[0] < a[1])) perr = true;
  return __dadd_rn(a[0], __dmul_rn(__dsub_rn(a[1], a[0]), dr.uniform(kd)));  // low + (high - low) u
}
__device__ __forceinline__ double th_sample_truncated_gaussian(const ThetaDraws& dr, int kd, const double* a,
                                                               bool& perr) {
  const double fa = normcdf(__ddiv_rn(__dsub_rn(a[2], a[0]), a[1]));
  const double fb = normcdf(__ddiv_rn(__dsub_rn(a[3], a[0]), a[1]));
  if (!(a[1] > 0.0) || !(a[2] < a[3]) || !(__dsub_rn(fb, fa) > 0.0)) perr = true;
  const double q = __dadd_rn(fa, __dmul_rn(dr.uniform(kd), __dsub_rn(fb, fa)));
  return __dadd_rn(a[0], __dmul_rn(a[1], normcdfinv(q)));  // mean + sd ndtri(fa + u (fb - fa))
}
__device__ __forceinline__ double th_sample_gamma(const ThetaDraws& dr, int kd, const double* a, bool& perr) {
  if (!(a[0] > 0.0) || !(a[1] > 0.0)) perr = true;
  return __dmul_rn(a[1], dr.std_gamma(kd, a[0]));  // scale * standard_gamma(shape)
}
__device__ __forceinline__ double th_sample_inverse_gamma(const ThetaDraws& dr, int kd, const double* a,
                                                          bool& perr) {
  if (!(a[0] > 0.0) || !(a[1] > 0.0)) perr = true;
  return __ddiv_rn(1.0, __dmul_rn(__ddiv_rn(1.0, a[1]), dr.std_gamma(kd, a[0])));  // 1 / gamma(k, 1/s)
}

// distributions.logpdf (distributions.py:94-123), the reference's operation order
__device__ __forceinline__ double th_lp_gaussian(double x, const double* a, bool& perr) {
  if (!(a[1] > 0.0)) perr = true;
  const double z = __ddiv_rn(__dsub_rn(x, a[0]), a[1]);
  return __dsub_rn(__dsub_rn(__dmul_rn(__dmul_rn(-0.5, z), z), log(a[1])), kThLogSqrt2Pi);
}
__device__ __forceinline__ double th_lp_truncated_gaussian(double x, const double* a, bool& perr) {
  const double fa = normcdf(__ddiv_rn(__dsub_rn(a[2], a[0]), a[1]));
  const double fb = normcdf(__ddiv_rn(__dsub_rn(a[3], a[0]), a[1]));
  if (!(a[1] > 0.0) || !(a[2] < a[3]) || !(__dsub_rn(fb, fa) > 0.0)) perr = true;
  const double z = __ddiv_rn(__dsub_rn(x, a[0]), a[1]);
  const double core = __dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(__dmul_rn(-0.5, z), z), log(a[1])), kThLogSqrt2Pi),
                                log(__dsub_rn(fb, fa)));
  return (x >= a[2] && x <= a[3]) ? core : -CUDART_INF;
}
__device__ __forceinline__ double th_lp_gamma(double x, const double* a, bool& perr) {
  if (!(a[0] > 0.0) || !(a[1] > 0.0)) perr = true;
  if (!(x > 0.0)) return -CUDART_INF;
  const double t = __dsub_rn(__dmul_rn(__dsub_rn(a[0], 1.0), log(x)), __ddiv_rn(x, a[1]));
  return __dsub_rn(__dsub_rn(t, __dmul_rn(a[0], log(a[1]))), lgamma(a[0]));
}
__device__ __forceinline__ double th_lp_inverse_gamma(double x, const double* a, bool& perr) {
  if (!(a[0] > 0.0) || !(a[1] > 0.0)) perr = true;
  if (!(x > 0.0)) return -CUDART_INF;
  const double t = __dsub_rn(__dmul_rn(a[0], log(a[1])), lgamma(a[0]));
  return __dsub_rn(__dsub_rn(t, __dmul_rn(__dadd_rn(a[0], 1.0), log(x))), __ddiv_rn(a[1], x));
}
__device__ __forceinline__ double th_lp_uniform(double x, const double* a, bool& perr) {
  if (!(a[0] < a[1])) perr = true;
  return (x >= a[0] && x <= a[1]) ? -log(__dsub_rn(a[1], a[0])) : -CUDART_INF;
}

// One proposal per chain (GenericModel.propose_batch order): theta walk, its
// reverse density, then the x0 walk (new theta) + initial assigns, its reverse
// density (old theta), then the prior of the proposal.
template <class M>
__global__ void __launch_bounds__(128) gen_theta_propose_kernel(ssm_theta_args A) {
  using Th = typename M::Theta;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.n_chains) return;
  const ThetaDraws D{&A, c};
  const double* th = A.theta + static_cast<size_t>(c) * Th::NP;
  double* out = A.theta_new + static_cast<size_t>(c) * Th::NP;
  bool perr = false;
  double lq_f = 0.0, lq_r = 0.0;
  double tmp[Th::NPB];
  Th::param_walk(th, nullptr, out, D, lq_f, perr);
  Th::param_walk(out, th, tmp, D, lq_r, perr);
  double lp = Th::param_logpdf(out, perr);
  if (A.has_init) {
    const double* x0 = A.x0 + static_cast<size_t>(c) * Th::NX;
    double* x1 = A.x0_new + static_cast<size_t>(c) * Th::NX;
    double xn[Th::NXB], xt[Th::NXB];
    double lf = 0.0, lr = 0.0;
    Th::init_walk(out, x0, nullptr, xn, D, lf, perr);
    Th::init_assign(out, xn);
    Th::init_walk(th, xn, x0, xt, D, lr, perr);
    for (int n = 0; n < Th::NX; ++n) x1[n] = xn[n];
    lq_f = lq_f + lf;
    lq_r = lq_r + lr;
    lp = lp + Th::init_logpdf(out, xn, perr);
  }
  A.logq_fwd[c] = lq_f;
  A.logq_rev[c] = lq_r;
  A.log_prior_new[c] = lp;
  if (perr) atomicExch(A.err, 1);
}

}  // namespace ssm
