// Batched Kalman filter for linear-Gaussian models:
// the forward recursions of the reference's KalmanRun._step (kalman.py:57-96)
// for B systems at once, one thread per system (theta), sequential over grid
// steps, 32-thread blocks so a batch spreads over ceil(B / 32) SMs.  Covariance form: the reference carries upper-triangular square-root
// factors and re-factorizes; the filtered / predicted moments and the
// marginal likelihood are the same quantities (agreement to rounding).
//
//   predict:  mu^ = A mu + b,  P^ = A P A^T + Q                     (kalman.py:61-65)
//   update (present slots only, kalman.py:72-91):
//     S = H P^ H^T + diag(r^2) = L L^T,  e = y - (H mu^ + c),  v = L^-1 e
//     W = L^-1 H P^,  mu = mu^ + W^T v,  P = P^ - W^T W
//     loglik += -m/2 log(2 pi) - sum log L_jj - v.v/2
#include "ssm_common.cuh"

namespace ssm {
namespace {

constexpr int kKfMaxDim = 16;
constexpr double kLog2Pi = 1.83787706640934548356;

// N: compile-time bound on nx and ny (1, 2, 4, 8, 16): small models keep every array in registers
template <int N>
__global__ void __launch_bounds__(32) kalman_kernel(ssm_kalman_args A) {
  constexpr int kKfMax = N;
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= A.B) return;
  const int nx = A.nx, ny = A.ny, S = A.S;
  const size_t rec = static_cast<size_t>(f) * (S + 1);
  double mu[kKfMax], P[kKfMax * kKfMax], mh[kKfMax], Ph[kKfMax * kKfMax];
  double W[kKfMax * kKfMax], L[kKfMax * kKfMax], e[kKfMax], T[kKfMax * kKfMax];
  int slot[kKfMax];
  for (int i = 0; i < nx; ++i) mu[i] = A.mu[(rec + A.s0) * nx + i];
  for (int i = 0; i < nx * nx; ++i) P[i] = A.P[(rec + A.s0) * nx * nx + i];
  double ll = A.loglik[f];
  for (int s = A.s0 + 1; s <= A.s1; ++s) {
    const size_t tab = static_cast<size_t>(f) * S + (s - 1);
    // the tables are read-only for the whole launch: the non-coherent path lets these
    // loads issue ahead of the record stores below instead of behind them
    const double* __restrict__ Am = A.A + tab * nx * nx;
    const double* __restrict__ bv = A.b + tab * nx;
    const double* __restrict__ Qm = A.Q + tab * nx * nx;
    // predict
    for (int i = 0; i < nx; ++i) {
      double acc = __ldg(&bv[i]);
      for (int k = 0; k < nx; ++k) acc += __ldg(&Am[i * nx + k]) * mu[k];
      mh[i] = acc;
    }
    for (int i = 0; i < nx; ++i)  // T = A P
      for (int j = 0; j < nx; ++j) {
        double acc = 0.0;
        for (int k = 0; k < nx; ++k) acc += __ldg(&Am[i * nx + k]) * P[k * nx + j];
        T[i * nx + j] = acc;
      }
    for (int i = 0; i < nx; ++i)  // P^ = T A^T + Q, symmetric by construction
      for (int j = 0; j <= i; ++j) {
        double acc = __ldg(&Qm[i * nx + j]);
        for (int k = 0; k < nx; ++k) acc += T[i * nx + k] * __ldg(&Am[j * nx + k]);
        Ph[i * nx + j] = acc;
        Ph[j * nx + i] = acc;
      }
    for (int i = 0; i < nx; ++i) A.mu_p[(rec + s) * nx + i] = mh[i];
    for (int i = 0; i < nx * nx; ++i) A.P_p[(rec + s) * nx * nx + i] = Ph[i];
    // present slots in slot order
    int m = 0;
    for (int j = 0; j < ny; ++j)
      if (A.mask[static_cast<size_t>(s - 1) * ny + j]) slot[m++] = j;
    if (m == 0) {  // pure prediction (kalman.py:68-70)
      for (int i = 0; i < nx; ++i) mu[i] = mh[i];
      for (int i = 0; i < nx * nx; ++i) P[i] = Ph[i];
    } else {
      const double* __restrict__ Hm = A.H + tab * ny * nx;
      const double* __restrict__ cv = A.c + tab * ny;
      const double* __restrict__ rv = A.r_sd + tab * ny;
      const double* __restrict__ yv = A.y + static_cast<size_t>(s - 1) * ny;
      // W <- H P^ (m x nx), e <- y - H mu^ - c
      for (int a = 0; a < m; ++a) {
        const double* __restrict__ h = Hm + slot[a] * nx;
        double nu = __ldg(&cv[slot[a]]);
        for (int k = 0; k < nx; ++k) nu += __ldg(&h[k]) * mh[k];
        e[a] = __ldg(&yv[slot[a]]) - nu;
        for (int j = 0; j < nx; ++j) {
          double acc = 0.0;
          for (int k = 0; k < nx; ++k) acc += __ldg(&h[k]) * Ph[k * nx + j];
          W[a * nx + j] = acc;
        }
      }
      // S = (H P^) H^T + R, lower Cholesky in place in L
      bool bad = false;
      for (int a = 0; a < m; ++a)
        for (int bb = 0; bb <= a; ++bb) {
          const double* __restrict__ h = Hm + slot[bb] * nx;
          double acc = (a == bb) ? __ldg(&rv[slot[a]]) * __ldg(&rv[slot[a]]) : 0.0;
          for (int k = 0; k < nx; ++k) acc += W[a * nx + k] * __ldg(&h[k]);
          L[a * kKfMax + bb] = acc;
        }
      for (int j = 0; j < m; ++j) {
        double d = L[j * kKfMax + j];
        for (int k = 0; k < j; ++k) d -= L[j * kKfMax + k] * L[j * kKfMax + k];
        if (!(d > 0.0)) {
          bad = true;
          break;
        }
        d = sqrt(d);
        L[j * kKfMax + j] = d;
        for (int i = j + 1; i < m; ++i) {
          double v = L[i * kKfMax + j];
          for (int k = 0; k < j; ++k) v -= L[i * kKfMax + k] * L[j * kKfMax + k];
          L[i * kKfMax + j] = v / d;
        }
      }
      if (bad) {
        if (A.err[f] == 0) A.err[f] = s;
        ll = CUDART_NAN;
        break;
      }
      // forward solves: v = L^-1 e, W <- L^-1 W
      double vv = 0.0, logdet = 0.0;
      for (int a = 0; a < m; ++a) {
        double v = e[a];
        for (int k = 0; k < a; ++k) v -= L[a * kKfMax + k] * e[k];
        e[a] = v / L[a * kKfMax + a];
        vv += e[a] * e[a];
        logdet += log(L[a * kKfMax + a]);
        for (int j = 0; j < nx; ++j) {
          double w = W[a * nx + j];
          for (int k = 0; k < a; ++k) w -= L[a * kKfMax + k] * W[k * nx + j];
          W[a * nx + j] = w / L[a * kKfMax + a];
        }
      }
      for (int i = 0; i < nx; ++i) {
        double acc = mh[i];
        for (int a = 0; a < m; ++a) acc += W[a * nx + i] * e[a];
        mu[i] = acc;
      }
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j <= i; ++j) {
          double acc = Ph[i * nx + j];
          for (int a = 0; a < m; ++a) acc -= W[a * nx + i] * W[a * nx + j];
          P[i * nx + j] = acc;
          P[j * nx + i] = acc;
        }
      ll += -0.5 * kLog2Pi * m - logdet - 0.5 * vv;
    }
    for (int i = 0; i < nx; ++i) A.mu[(rec + s) * nx + i] = mu[i];
    for (int i = 0; i < nx * nx; ++i) A.P[(rec + s) * nx * nx + i] = P[i];
  }
  A.loglik[f] = ll;
}

// psd_cholesky_upper (kalman.py / linalg.py:21-50 pivot rule) in place on a
// symmetric n x n matrix S (row-major, stride ld): upper U with U^T U = S; a
// pivot within tol of zero leaves its row zero (the rest of the row must
// vanish too), one below -tol fails.  Returns false on failure.
template <int N>
__device__ __forceinline__ bool psd_chol_upper(const double* S, int n, double* U) {
  double dmax = 1.0, amax = 1.0;
  for (int i = 0; i < n; ++i) {
    dmax = fmax(dmax, fabs(S[i * N + i]));
    for (int j = 0; j < n; ++j) amax = fmax(amax, fabs(S[i * N + j]));
  }
  const double tol = 1e-12 * dmax, big = sqrt(tol) * amax;
  for (int i = 0; i < n; ++i) {
    double piv = S[i * N + i];
    for (int k = 0; k < i; ++k) piv -= U[k * N + i] * U[k * N + i];
    for (int j = 0; j < n; ++j)
      if (j != i) U[i * N + j] = 0.0;
    if (piv < -tol) return false;
    if (piv <= tol) {
      U[i * N + i] = 0.0;
      for (int j = i + 1; j < n; ++j) {
        double r = S[i * N + j];
        for (int k = 0; k < i; ++k) r -= U[k * N + i] * U[k * N + j];
        if (fabs(r) > big) return false;
      }
      continue;
    }
    const double d = sqrt(piv);
    U[i * N + i] = d;
    for (int j = i + 1; j < n; ++j) {
      double r = S[i * N + j];
      for (int k = 0; k < i; ++k) r -= U[k * N + i] * U[k * N + j];
      U[i * N + j] = r / d;
    }
  }
  return true;
}

// x = U^-T v (forward substitution on the lower factor U^T); zero pivots are
// absent directions (x_i = 0: the minimum-norm solution of a consistent system,
// the host path's pseudo-inverse)
template <int N>
__device__ __forceinline__ void solve_upper_t(const double* U, int n, const double* v, double* x) {
  for (int i = 0; i < n; ++i) {
    const double d = U[i * N + i];
    if (d == 0.0) {
      x[i] = 0.0;
      continue;
    }
    double r = v[i];
    for (int k = 0; k < i; ++k) r -= U[k * N + i] * x[k];
    x[i] = r / d;
  }
}

// Backward smoothing draw (kalman.py:98-114) for G runs, one thread each:
//   x_s = mu_s + chol(P_s)^T z_0
//   i = s-1..0:  Uh = chol(P^_{i+1}),  C = P_i A_i^T,  K = C Uh^-1,
//                omega = mu_i + K Uh^-T (x_{i+1} - mu^_{i+1}),
//                x_i = omega + chol(P_i - K K^T)^T z_{s-i}
// with the reference's standard normals z (host-drawn, each run's stream in its
// order) and the records of the device forward pass.
template <int N>
__global__ void __launch_bounds__(32) kalman_sample_kernel(ssm_kalman_sample_args A) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= A.G) return;
  const int nx = A.nx, s = A.s, S1 = A.S + 1;
  const size_t row = static_cast<size_t>(A.rows[g]);
  const double* mu = A.mu + row * S1 * nx;
  const double* P = A.P + row * S1 * nx * nx;
  const double* mu_p = A.mu_p + row * S1 * nx;
  const double* P_p = A.P_p + row * S1 * nx * nx;
  const double* Am = A.A + row * A.S * nx * nx;
  const double* z = A.z + static_cast<size_t>(g) * (s + 1) * nx;
  double* out = A.out + static_cast<size_t>(g) * (s + 1) * nx;
  double M[N * N], U[N * N], Uh[N * N], K[N * N], C[N * N], t[N], w[N], xn[N];
  auto load = [&](const double* src, double* dst) {  // nx x nx -> N-strided
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nx; ++j) dst[i * N + j] = src[i * nx + j];
  };
  load(P + static_cast<size_t>(s) * nx * nx, M);
  if (!psd_chol_upper<N>(M, nx, U)) {
    A.err[g] = s + 1;
    return;
  }
  for (int i = 0; i < nx; ++i) {
    double acc = mu[static_cast<size_t>(s) * nx + i];
    for (int k = 0; k <= i; ++k) acc += U[k * N + i] * z[k];
    xn[i] = acc;
    out[static_cast<size_t>(s) * nx + i] = acc;
  }
  for (int i = s - 1; i >= 0; --i) {
    load(P_p + static_cast<size_t>(i + 1) * nx * nx, M);
    if (!psd_chol_upper<N>(M, nx, Uh)) {
      A.err[g] = i + 1;
      return;
    }
    load(P + static_cast<size_t>(i) * nx * nx, M);  // P_i
    const double* Ai = Am + static_cast<size_t>(i) * nx * nx;
    for (int r = 0; r < nx; ++r)  // C = P_i A_i^T
      for (int c = 0; c < nx; ++c) {
        double acc = 0.0;
        for (int k = 0; k < nx; ++k) acc += M[r * N + k] * Ai[c * nx + k];
        C[r * N + c] = acc;
      }
    for (int r = 0; r < nx; ++r) {  // row r of K: Uh^-T C[r,:]^T
      for (int c = 0; c < nx; ++c) t[c] = C[r * N + c];
      solve_upper_t<N>(Uh, nx, t, w);
      for (int c = 0; c < nx; ++c) K[r * N + c] = w[c];
    }
    for (int c = 0; c < nx; ++c) t[c] = xn[c] - mu_p[static_cast<size_t>(i + 1) * nx + c];
    solve_upper_t<N>(Uh, nx, t, w);
    for (int r = 0; r < nx; ++r)  // M <- P_i - K K^T (symmetric)
      for (int c = 0; c < nx; ++c) {
        double acc = M[r * N + c];
        for (int k = 0; k < nx; ++k) acc -= K[r * N + k] * K[c * N + k];
        C[r * N + c] = acc;
      }
    if (!psd_chol_upper<N>(C, nx, U)) {
      A.err[g] = i + 1;
      return;
    }
    const double* zi = z + static_cast<size_t>(s - i) * nx;
    for (int r = 0; r < nx; ++r) {
      double acc = mu[static_cast<size_t>(i) * nx + r];
      for (int k = 0; k < nx; ++k) acc += K[r * N + k] * w[k];
      for (int k = 0; k <= r; ++k) acc += U[k * N + r] * zi[k];
      t[r] = acc;
    }
    for (int r = 0; r < nx; ++r) {
      xn[r] = t[r];
      out[static_cast<size_t>(i) * nx + r] = t[r];
    }
  }
}

}  // namespace
}  // namespace ssm

extern "C" int ssm_kalman_max_dim(void) { return ssm::kKfMaxDim; }

extern "C" int ssm_kalman_sample(const ssm_kalman_sample_args* args, void* stream) {
  using namespace ssm;
  if (!args || args->G < 0 || args->nx < 1 || args->nx > kKfMaxDim || args->s < 0 || args->s > args->S)
    return SSM_ERR_INVALID_ARG;
  if (args->G == 0) return SSM_OK;
  if (!args->rows || !args->A || !args->mu || !args->P || !args->mu_p || !args->P_p || !args->z || !args->out ||
      !args->err)
    return SSM_ERR_INVALID_ARG;
  const int nt = 32;
  const dim3 g((args->G + nt - 1) / nt);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n = args->nx;
  if (n <= 1)
    kalman_sample_kernel<1><<<g, nt, 0, st>>>(*args);
  else if (n <= 2)
    kalman_sample_kernel<2><<<g, nt, 0, st>>>(*args);
  else if (n <= 4)
    kalman_sample_kernel<4><<<g, nt, 0, st>>>(*args);
  else if (n <= 8)
    kalman_sample_kernel<8><<<g, nt, 0, st>>>(*args);
  else
    kalman_sample_kernel<16><<<g, nt, 0, st>>>(*args);
  return cudaGetLastError() == cudaSuccess ? SSM_OK : SSM_ERR_CUDA;
}

extern "C" int ssm_kalman_filter(const ssm_kalman_args* args, void* stream) {
  using namespace ssm;
  if (!args || args->B < 0 || args->nx < 1 || args->ny < 0 || args->nx > kKfMaxDim || args->ny > kKfMaxDim ||
      args->s0 < 0 || args->s1 < args->s0 || args->s1 > args->S)
    return SSM_ERR_INVALID_ARG;
  if (args->B == 0 || args->s1 == args->s0) return SSM_OK;
  if (!args->A || !args->b || !args->Q || !args->mu || !args->P || !args->mu_p || !args->P_p || !args->loglik ||
      !args->err || !args->mask || (args->ny > 0 && (!args->H || !args->c || !args->r_sd || !args->y)))
    return SSM_ERR_INVALID_ARG;
  // one thread per system, 32-thread blocks: B systems spread over ceil(B / 32) SMs
  const int nt = 32, n = args->nx > args->ny ? args->nx : args->ny;
  const dim3 g((args->B + nt - 1) / nt);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n <= 1)
    kalman_kernel<1><<<g, nt, 0, s>>>(*args);
  else if (n <= 2)
    kalman_kernel<2><<<g, nt, 0, s>>>(*args);
  else if (n <= 4)
    kalman_kernel<4><<<g, nt, 0, s>>>(*args);
  else if (n <= 8)
    kalman_kernel<8><<<g, nt, 0, s>>>(*args);
  else
    kalman_kernel<16><<<g, nt, 0, s>>>(*args);
  return cudaGetLastError() == cudaSuccess ? SSM_OK : SSM_ERR_CUDA;
}
