// Batched Kalman filter for linear-Gaussian models:
// the forward recursions of the reference's KalmanRun._step (kalman.py:57-96)
// for B systems at once, one thread per system (theta), sequential over grid
// steps.  Covariance form: the reference carries upper-triangular square-root
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
__global__ void __launch_bounds__(64) kalman_kernel(ssm_kalman_args A) {
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

}  // namespace
}  // namespace ssm

extern "C" int ssm_kalman_max_dim(void) { return ssm::kKfMaxDim; }

extern "C" int ssm_kalman_filter(const ssm_kalman_args* args, void* stream) {
  using namespace ssm;
  if (!args || args->B < 0 || args->nx < 1 || args->ny < 0 || args->nx > kKfMaxDim || args->ny > kKfMaxDim ||
      args->s0 < 0 || args->s1 < args->s0 || args->s1 > args->S)
    return SSM_ERR_INVALID_ARG;
  if (args->B == 0 || args->s1 == args->s0) return SSM_OK;
  if (!args->A || !args->b || !args->Q || !args->mu || !args->P || !args->mu_p || !args->P_p || !args->loglik ||
      !args->err || !args->mask || (args->ny > 0 && (!args->H || !args->c || !args->r_sd || !args->y)))
    return SSM_ERR_INVALID_ARG;
  const int nt = 64, n = args->nx > args->ny ? args->nx : args->ny;
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
