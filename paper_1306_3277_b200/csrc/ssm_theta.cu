// Device-side theta-level Metropolis-Hastings for the two hand-written models
// (SURVEY 8f row 1): the proposal walk (proposal_parameter / proposal_initial,
// simulate.py:272-352), its forward and reverse log-densities, the prior
// (parameter_logpdf + initial_logpdf, simulate.py:220-233) and the accept step
// (metropolis_accept, mcmc.py:28-33), one thread per chain.
//
// Draws are either device Philox (keyed per chain stream, purpose kPurposeTheta)
// or injected from the host (the reference's own numpy draws, for parity): the
// truncated-Gaussian uniforms, the gamma variate of the inverse-gamma statement
// (numpy gamma(2, 1/scale)) and the accept uniform.  Truncated Gaussians use the
// inverse-CDF sampler of distributions.py:78-84 with CUDA normcdf / normcdfinv
// for scipy's ndtr / ndtri (a few ulp apart, so device and host agree to ~1e-15
// relative rather than bitwise).
#include "ssm_common.cuh"

namespace ssm {
namespace {

constexpr uint32_t kPurposeTheta = 7u;
constexpr double kLogSqrt2Pi = 0.91893853320467274178;  // 0.5*log(2*pi), distributions.py:15

struct Draws {
  const ssm_theta_args* A;
  int c;
  // draw k of chain c: injected row or Philox block k/2 (two 53-bit uniforms per block)
  __device__ double uniform(int k) const {
    if (A->u_in) return A->u_in[static_cast<size_t>(c) * A->u_stride + k];
    const U4 r = philox4x32_10(U4{static_cast<uint32_t>(k >> 1), 0u, static_cast<uint32_t>(A->step), kPurposeTheta},
                               A->keys[2 * c], A->keys[2 * c + 1]);
    return (k & 1) ? u53(r.z, r.w) : u53(r.x, r.y);
  }
};

__device__ double tg_norm(double m, double sd, double lo, double hi, double* fa_out) {
  const double fa = normcdf((lo - m) / sd);
  const double fb = normcdf((hi - m) / sd);
  *fa_out = fa;
  return fb - fa;
}

// distributions.py:78-84: mean + sd*ndtri(fa + u*(fb-fa))
__device__ double tg_sample(double u, double m, double sd, double lo, double hi, int* err) {
  double fa;
  const double mass = tg_norm(m, sd, lo, hi, &fa);
  if (!(mass > 0.0)) *err = 1;
  return m + sd * normcdfinv(fa + u * mass);
}

// distributions.py:103-109
__device__ double tg_logpdf(double x, double m, double sd, double lo, double hi, int* err) {
  double fa;
  const double mass = tg_norm(m, sd, lo, hi, &fa);
  if (!(mass > 0.0)) *err = 1;
  const double z = (x - m) / sd;
  const double core = -0.5 * z * z - log(sd) - kLogSqrt2Pi - log(mass);
  return (x >= lo && x <= hi) ? core : -CUDART_INF;
}

__device__ double gamma_logpdf(double x, double a, double s) {
  return x > 0.0 ? (a - 1.0) * log(x) - x / s - a * log(s) - lgamma(a) : -CUDART_INF;
}

__device__ double invgamma_logpdf(double x, double a, double s) {
  return x > 0.0 ? a * log(s) - lgamma(a) - (a + 1.0) * log(x) - s / x : -CUDART_INF;
}

__device__ double uniform_logpdf(double x, double lo, double hi) {
  return (x >= lo && x <= hi) ? -log(hi - lo) : -CUDART_INF;
}

// Gamma(2, scale): injected numpy value, or scale * (E1 + E2) with E = -log(U), U in (0,1]
__device__ double gamma2(const Draws& D, int k, double scale) {
  if (D.A->g_in) return D.A->g_in[D.c];
  const double u1 = 1.0 - D.uniform(k), u2 = 1.0 - D.uniform(k + 1);
  return scale * (-log(u1) - log(u2));
}

__global__ void theta_propose_kernel(ssm_theta_args A) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.n_chains) return;
  const Draws D{&A, c};
  const int np = A.n_param;
  const double* th = A.theta + static_cast<size_t>(c) * np;
  double* out = A.theta_new + static_cast<size_t>(c) * np;
  int err = 0;
  double lq_f = 0.0, lq_r = 0.0, lp;
  // truncated-Gaussian statements (slot, sd, lower, upper) in block order, then the
  // inverse-gamma statement on slot ig; each reads the pre-statement value of its slot
  int n_tg, ig;
  double sd[3], lo[3], hi[3];
  if (A.model == SSM_MODEL_LORENZ96) {  // Lorenz96.bi:40-43
    n_tg = 1;
    ig = 1;
    sd[0] = 0.1, lo[0] = 8.0, hi[0] = 12.0;
  } else {  // Windkessel.bi:36-41
    n_tg = 3;
    ig = 3;
    sd[0] = 0.03, sd[1] = 0.1, sd[2] = 0.002;
    for (int k = 0; k < 3; ++k) lo[k] = 0.0, hi[k] = CUDART_INF;
  }
  for (int k = 0; k < n_tg; ++k) {
    const double v = tg_sample(D.uniform(k), th[k], sd[k], lo[k], hi[k], &err);
    out[k] = v;
    lq_f += tg_logpdf(v, th[k], sd[k], lo[k], hi[k], &err);
    lq_r += tg_logpdf(th[k], v, sd[k], lo[k], hi[k], &err);
  }
  const double s_f = 3.0 * th[ig];
  if (!(s_f > 0.0)) err = 1;
  const double g = gamma2(D, n_tg + (A.has_init ? A.nx : 0), 1.0 / s_f);
  const double v = 1.0 / g;
  out[ig] = v;
  lq_f += invgamma_logpdf(v, 2.0, s_f);
  lq_r += invgamma_logpdf(th[ig], 2.0, 3.0 * v);
  if (A.model == SSM_MODEL_LORENZ96) {  // Lorenz96.bi:16-19
    lp = (0.0 + uniform_logpdf(out[0], 8.0, 12.0)) + invgamma_logpdf(out[1], 2.0, 0.25);
  } else {  // Windkessel.bi:16-21
    lp = (((0.0 + gamma_logpdf(out[0], 2.0, 0.9)) + gamma_logpdf(out[1], 2.0, 1.5)) +
          gamma_logpdf(out[2], 2.0, 0.03)) + invgamma_logpdf(out[3], 2.0, 25.0);
  }
  if (A.has_init) {  // proposal_initial x[n] ~ truncated_gaussian(x[n], 0.1, -1, 3), Lorenz96.bi:46-48
    const double* x0 = A.x0 + static_cast<size_t>(c) * A.nx;
    double* x1 = A.x0_new + static_cast<size_t>(c) * A.nx;
    double lf = 0.0, lr = 0.0, li = 0.0;
    for (int n = 0; n < A.nx; ++n) {
      const double xn = tg_sample(D.uniform(n_tg + n), x0[n], 0.1, -1.0, 3.0, &err);
      x1[n] = xn;
      lf += tg_logpdf(xn, x0[n], 0.1, -1.0, 3.0, &err);
      lr += tg_logpdf(x0[n], xn, 0.1, -1.0, 3.0, &err);
      li += uniform_logpdf(xn, -1.0, 3.0);  // initial x[n] ~ uniform(-1, 3)
    }
    lq_f = lq_f + lf;
    lq_r = lq_r + lr;
    lp = lp + li;
  }
  A.logq_fwd[c] = lq_f;
  A.logq_rev[c] = lq_r;
  A.log_prior_new[c] = lp;
  if (err) atomicExch(A.err, 1);
}

// log_ratio = (ll' + lp' + lq_rev) - (ll + lp + lq_fwd); accept iff u <= exp(min(r, 0))
// (mcmc.py:28-33, 158-164).  Proposals outside the prior support were never filtered:
// their loglik_new is -inf and they reject without drawing.
__global__ void theta_accept_kernel(ssm_theta_args A) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= A.n_chains) return;
  const Draws D{&A, c};
  const double lp_new = A.log_prior_new[c];
  bool ok = false;
  if (lp_new != -CUDART_INF) {
    const double r = (A.loglik_new[c] + lp_new + A.logq_rev[c]) - (A.loglik[c] + A.log_prior[c] + A.logq_fwd[c]);
    if (!isnan(r) && r != -CUDART_INF) {
      const double u = A.u_acc_in ? A.u_acc_in[c] : D.uniform(A.u_stride - 1);
      ok = u <= exp(fmin(r, 0.0));
    }
  }
  A.accepted[c] = ok ? 1 : 0;
  if (!ok) return;
  for (int k = 0; k < A.n_param; ++k)
    A.theta[static_cast<size_t>(c) * A.n_param + k] = A.theta_new[static_cast<size_t>(c) * A.n_param + k];
  if (A.has_init)
    for (int n = 0; n < A.nx; ++n) A.x0[static_cast<size_t>(c) * A.nx + n] = A.x0_new[static_cast<size_t>(c) * A.nx + n];
  A.loglik[c] = A.loglik_new[c];
  A.log_prior[c] = lp_new;
}

int check_args(const ssm_theta_args* A) {
  if (!A || A->n_chains < 0) return SSM_ERR_INVALID_ARG;
  if (A->model == SSM_MODEL_LORENZ96) {
    if (A->n_param != 2 || A->nx != 8) return SSM_ERR_INVALID_ARG;
  } else if (A->model == SSM_MODEL_WINDKESSEL) {
    if (A->n_param != 4 || A->nx != 1 || A->has_init) return SSM_ERR_INVALID_ARG;
  } else if (A->model == SSM_MODEL_GENERIC) {  // accept only (the proposal is ssm_gen_theta_propose)
    if (A->n_param < 0 || A->nx < 0 || A->u_stride < 1) return SSM_ERR_INVALID_ARG;
  } else {
    return SSM_ERR_UNSUPPORTED;
  }
  if (!A->u_in && !A->keys) return SSM_ERR_INVALID_ARG;
  return SSM_OK;
}

}  // namespace
}  // namespace ssm

extern "C" int ssm_theta_draws(int model, int has_init) {
  if (model != SSM_MODEL_LORENZ96 && model != SSM_MODEL_WINDKESSEL) return -1;  // generic: ssm_gen_theta_draws
  const int n_tg = model == SSM_MODEL_LORENZ96 ? 1 : 3;
  const int nx = model == SSM_MODEL_LORENZ96 ? 8 : 1;
  return n_tg + (has_init ? nx : 0) + 2 + 1;  // tg uniforms, x0 uniforms, gamma(2) pair, accept
}

extern "C" int ssm_theta_propose(const ssm_theta_args* args, void* stream) {
  using namespace ssm;
  if (args && args->model == SSM_MODEL_GENERIC) return SSM_ERR_UNSUPPORTED;  // ssm_gen_theta_propose
  const int rc = check_args(args);
  if (rc != SSM_OK) return rc;
  if (args->n_chains == 0) return SSM_OK;
  if (!args->theta || !args->theta_new || !args->logq_fwd || !args->logq_rev || !args->log_prior_new || !args->err)
    return SSM_ERR_INVALID_ARG;
  if (args->has_init && (!args->x0 || !args->x0_new)) return SSM_ERR_INVALID_ARG;
  if (args->u_in && !args->g_in) return SSM_ERR_INVALID_ARG;
  const int nt = 128;
  theta_propose_kernel<<<(args->n_chains + nt - 1) / nt, nt, 0, static_cast<cudaStream_t>(stream)>>>(*args);
  return cudaGetLastError() == cudaSuccess ? SSM_OK : SSM_ERR_CUDA;
}

extern "C" int ssm_theta_accept(const ssm_theta_args* args, void* stream) {
  using namespace ssm;
  const int rc = check_args(args);
  if (rc != SSM_OK) return rc;
  if (args->n_chains == 0) return SSM_OK;
  if (!args->loglik_new || !args->loglik || !args->log_prior || !args->accepted || !args->theta ||
      !args->theta_new || (args->u_in && !args->u_acc_in))
    return SSM_ERR_INVALID_ARG;
  const int nt = 128;
  theta_accept_kernel<<<(args->n_chains + nt - 1) / nt, nt, 0, static_cast<cudaStream_t>(stream)>>>(*args);
  return cudaGetLastError() == cudaSuccess ? SSM_OK : SSM_ERR_CUDA;
}
