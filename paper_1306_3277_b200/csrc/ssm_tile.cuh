// Warp-tile weighting and the fused LSE/ESS finalize shared by the fused
// propagate/weight kernels (the hand-written pw_kernel and the NVRTC-compiled
// generic-model kernel).  Reference: particle.py:125-133 (logw + g, logsumexp,
// degenerate check, loglik), particle.py:83-85, 99-100 (ESS gate).
//
// Per weighted WARP tile w (32 consecutive particles) the warp produces, for the
// next step's resampling:
//   m_w     = max log-weight of the warp tile,
//   q_j     = round(exp(a_j - m_w) * 2^52)              (tile-local fixed point),
//   C_j     = inclusive prefix of q within the tile     -> cdf_local[j],
//   Q_w     = C_last                                    -> tile_rec[w] = {m_w, Q_w},
// and the tile's scipy-form LSE/ESS partial (max elements split out), folded
// in tile order into the warp / block partials for the fused finalize.
#pragma once

#include "ssm_common.cuh"

namespace ssm {

#ifndef SSM_PW_THREADS
#define SSM_PW_THREADS 256
#endif
constexpr int kPwThreads = SSM_PW_THREADS;  // fused-kernel block
constexpr int kMaxPwBlocks = 2048;  // per filter; a function of P only (determinism)

// Blocks per filter: >= 4 block tiles per block, so each warp folds several warp
// tiles per setup (matters at moderate P with many filters, e.g. PMMH 8 x 2^16).
// A function of P only, so the LSE fold order never depends on the batch.
#ifndef SSM_PW_TILES_PER_BLOCK
#define SSM_PW_TILES_PER_BLOCK 4
#endif
__host__ __device__ inline int pw_grid_x(int P) {
  const int tiles = (P + kPwThreads - 1) / kPwThreads;
  const int g = (tiles + SSM_PW_TILES_PER_BLOCK - 1) / SSM_PW_TILES_PER_BLOCK;
  return g < kMaxPwBlocks ? g : kMaxPwBlocks;
}

constexpr double kTileFix = 4503599627370496.0;  // 2^52

// exp(x) for x <= 0 (the tile weights e_j = exp(a_j - m_w)): 2^(j/64) table in
// shared memory + degree-6 polynomial on |r| <= ln2/128 (truncation < 3e-20,
// ~1-2 ulp overall); coefficients in the constant bank so the DFMAs take them
// as operands.  x < -40 -> 0 (round(e 2^52) is 0 below -36.7), NaN -> NaN.
__constant__ double c_exp_tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};
__constant__ double c_exp_poly[8] = {0x1.6c16c16c16c17p-10, 0x1.1111111111111p-7, 0x1.5555555555555p-5,
                                     0x1.5555555555555p-3, 0x1.0000000000000p-1, 0x1.71547652b82fep+6,
                                     0x1.62e42fefa39efp-7, 0x1.abc9e3b39803fp-62};

__device__ __forceinline__ double exp_tile(double x, const double* __restrict__ tab /* smem */) {
  if (!(x >= -40.0)) return x != x ? x : 0.0;
  const double t = fma(x, c_exp_poly[5], 0x1.8p52);  // round(x 64/ln2) in the low word
  const int n = __double2loint(t);
  const double nd = t - 0x1.8p52;
  double r = fma(nd, -c_exp_poly[6], x);
  r = fma(nd, -c_exp_poly[7], r);
  double p = fma(c_exp_poly[0], r, c_exp_poly[1]);
  p = fma(p, r, c_exp_poly[2]);
  p = fma(p, r, c_exp_poly[3]);
  p = fma(p, r, c_exp_poly[4]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double y = tab[n & 63] * p;  // in [0.99, 2.01)
  return __hiloint2double(__double2hiint(y) + ((n >> 6) << 20), __double2loint(y));  // * 2^(n >> 6)
}

// Fold up to 32 parked warp-tile partials (lane l holds tile l: m_l is a
// float-representable reference >= the tile's max, or -inf when empty) into
// the warp partial `st` (lane 0): one exp per lane and a fixed shuffle tree,
// so the result depends only on the tile layout (deterministic).
__device__ __forceinline__ Lse fold_tiles(Lse st, double m, double t, double s2, int lane) {
  const float mf = static_cast<float>(m);  // exact: m came from a float (or is +-inf / NaN)
  const int key = __float_as_int(mf) >= 0 ? __float_as_int(mf) : (__float_as_int(mf) ^ 0x7fffffff);
  const int kmax = __reduce_max_sync(0xffffffffu, key);
  const double M = static_cast<double>(__int_as_float(kmax >= 0 ? kmax : (kmax ^ 0x7fffffff)));
  if (M == -CUDART_INF) return st;  // warp-uniform: no particles in any parked tile
  const double f = exp(m - M);      // 0 for empty slots; NaN M propagates
  double T = t * f, S2 = s2 * (f * f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T += __shfl_down_sync(0xffffffffu, T, o);
    S2 += __shfl_down_sync(0xffffffffu, S2, o);
  }
  if (lane == 0) st = lse_combine(st, Lse{M, 0.0, T, S2});
  return st;
}

// Warp-tile partials parked until 32 have accumulated (one per slot, in tile
// order), and the warp partial they fold into (shared memory, not registers:
// the fused kernels run at 3 CTAs / SM on an 80-register budget).
struct ParkedTiles {
  double m[32], t[32], s2[32];
  Lse st;  // warp partial, groups of 32 warp tiles folded in order (lane 0 writes)
};

__device__ __forceinline__ void fold_parked(ParkedTiles* pk, bool valid, int lane) {
  const Lse st = lane == 0 ? pk->st : lse_empty();
  const Lse r = fold_tiles(st, valid ? pk->m[lane] : -CUDART_INF, valid ? pk->t[lane] : 0.0,
                           valid ? pk->s2[lane] : 0.0, lane);
  if (lane == 0) pk->st = r;
}

// Running state of a warp's weighted tiles (the warp partial lives in park->st).
struct WarpTileAcc {
  ParkedTiles* park;  // this warp's parking slots in shared memory
  int slot;           // parking slot of the current warp tile's {m_w, t_w, s2_w}
  int nparked;        // (lane 0) slots filled since the last fold: a prefix of the slots
};

__device__ __forceinline__ WarpTileAcc warp_tile_acc(ParkedTiles* park, int lane) {
  if (lane == 0) park->st = lse_empty();
  __syncwarp();
  return WarpTileAcc{park, 0, 0};
}

// One weighted warp tile: a_d = the particle's unnormalised log-weight (-inf
// when inactive).  Warp-uniform call (all 32 lanes).
__device__ __forceinline__ void warp_tile_weigh(WarpTileAcc& acc, double a_d, bool act, int p, int P, int lane,
                                                const double* __restrict__ s_exp_tab, uint64_t* __restrict__ cloc,
                                                ssm_tile_rec* __restrict__ trec, bool want_ess) {
  // reference max, fixed-point prefix, LSE/ESS partial: one REDUX + one ballot +
  // a 5-step split scan, no block barrier, so warps stay out of phase.
  // Reference m_w = float round-up of the tile max (>= every a_j, within 2^-24
  // relative), so every e_j = exp(a_j - m_w) <= 1.
  const float af = __double2float_ru(a_d);
  const int key = __float_as_int(af) >= 0 ? __float_as_int(af) : (__float_as_int(af) ^ 0x7fffffff);
  const int kmax = __reduce_max_sync(0xffffffffu, act ? key : (-2147483647 - 1));
  const int kb = kmax >= 0 ? kmax : (kmax ^ 0x7fffffff);
  const double mw = static_cast<double>(__int_as_float(kb));
  const bool any_nan = __any_sync(0xffffffffu, act && isnan(a_d));
  const double e = (!act || mw == -CUDART_INF) ? 0.0 : exp_tile(a_d - mw, s_exp_tab);
  const uint64_t q = (e >= 0.0 && e <= 1.0) ? __double2ull_rn(e * kTileFix) : 0ull;
  // inclusive prefix of q <= 2^52 over the tile as two 32-bit scans of its
  // 26-bit halves (each tile sum < 2^31): exact, half the shuffle work of a u64 scan
  uint32_t qh = static_cast<uint32_t>(q >> 26), ql = static_cast<uint32_t>(q) & 0x3ffffffu;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yh = __shfl_up_sync(0xffffffffu, qh, o);
    const uint32_t yl = __shfl_up_sync(0xffffffffu, ql, o);
    if (lane >= o) {
      qh += yh;
      ql += yl;
    }
  }
  const uint64_t qi = (static_cast<uint64_t>(qh) << 26) + ql;
  if (cloc && act) cloc[p] = qi;
  const uint64_t Qw = (static_cast<uint64_t>(__shfl_sync(0xffffffffu, qh, 31)) << 26) +
                      __shfl_sync(0xffffffffu, ql, 31);
  double s2_ = 0.0;
  if (want_ess) {  // block-uniform
    s2_ = e * e;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2_ += __shfl_xor_sync(0xffffffffu, s2_, o);
  }
  if (lane == 0 && trec && p < P) trec[p >> 5] = ssm_tile_rec{mw, Qw};
  // tile sum of exp(a - m_w) from the exact fixed-point total (|err| <= 32 * 2^-53),
  // parked in shared memory slot `slot` of the warp (the values are warp-uniform,
  // lane 0 stores); every 32 tiles the warp folds them in one pass
  if (lane == 0 && p - lane < P) {  // tiles past P stay empty (their m_w is a NaN sentinel)
    acc.park->m[acc.slot] = mw;
    acc.park->t[acc.slot] = any_nan ? CUDART_NAN : static_cast<double>(Qw) * (1.0 / kTileFix);
    acc.park->s2[acc.slot] = s2_;
    ++acc.nparked;
  }
  if (++acc.slot == 32) {
    __syncwarp();
    fold_parked(acc.park, lane < __shfl_sync(0xffffffffu, acc.nparked, 0), lane);
    __syncwarp();
    acc.slot = 0;
    acc.nparked = 0;
  }
}

// exp_tile without the early return: the same value for every x (the polynomial
// is evaluated and discarded for x < -40 / NaN), so a call site can keep it in
// the same basic block as independent work (pw_body_lag).
__device__ __forceinline__ double exp_tile_nb(double x, const double* __restrict__ tab /* smem */) {
  const double t = fma(x, c_exp_poly[5], 0x1.8p52);
  const int n = __double2loint(t);
  const double nd = t - 0x1.8p52;
  double r = fma(nd, -c_exp_poly[6], x);
  r = fma(nd, -c_exp_poly[7], r);
  double p = fma(c_exp_poly[0], r, c_exp_poly[1]);
  p = fma(p, r, c_exp_poly[2]);
  p = fma(p, r, c_exp_poly[3]);
  p = fma(p, r, c_exp_poly[4]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double y = tab[n & 63] * p;
  const double v = __hiloint2double(__double2hiint(y) + ((n >> 6) << 20), __double2loint(y));
  return x >= -40.0 ? v : (x != x ? x : 0.0);
}

// warp_tile_weigh for pw_body_lag: the same arithmetic, stores and parking, no
// ESS partial (the lagged kernel runs without an ESS gate) and no branches
// before the parking-slot fold.  `real` = false makes the call a no-op that
// still takes part in the warp collectives.
__device__ __forceinline__ void warp_tile_weigh_lag(WarpTileAcc& acc, double a_d, bool act, int p, int P, int lane,
                                                    const double* __restrict__ s_exp_tab,
                                                    uint64_t* __restrict__ cloc, ssm_tile_rec* __restrict__ trec,
                                                    bool real) {
  const float af = __double2float_ru(a_d);
  const int key = __float_as_int(af) >= 0 ? __float_as_int(af) : (__float_as_int(af) ^ 0x7fffffff);
  const int kmax = __reduce_max_sync(0xffffffffu, act ? key : (-2147483647 - 1));
  const int kb = kmax >= 0 ? kmax : (kmax ^ 0x7fffffff);
  const double mw = static_cast<double>(__int_as_float(kb));
  const bool any_nan = __any_sync(0xffffffffu, act && isnan(a_d));
  const double ex = exp_tile_nb(a_d - mw, s_exp_tab);
  const double e = (!act || mw == -CUDART_INF) ? 0.0 : ex;
  const uint64_t q = (e >= 0.0 && e <= 1.0) ? __double2ull_rn(e * kTileFix) : 0ull;
  uint32_t qh = static_cast<uint32_t>(q >> 26), ql = static_cast<uint32_t>(q) & 0x3ffffffu;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t yh = __shfl_up_sync(0xffffffffu, qh, o);
    const uint32_t yl = __shfl_up_sync(0xffffffffu, ql, o);
    if (lane >= o) {
      qh += yh;
      ql += yl;
    }
  }
  const uint64_t qi = (static_cast<uint64_t>(qh) << 26) + ql;
  if (real && act) cloc[p] = qi;
  const uint64_t Qw = (static_cast<uint64_t>(__shfl_sync(0xffffffffu, qh, 31)) << 26) +
                      __shfl_sync(0xffffffffu, ql, 31);
  if (real && lane == 0 && p < P) trec[p >> 5] = ssm_tile_rec{mw, Qw};
  if (real && lane == 0 && p - lane < P) {
    acc.park->m[acc.slot] = mw;
    acc.park->t[acc.slot] = any_nan ? CUDART_NAN : static_cast<double>(Qw) * (1.0 / kTileFix);
    acc.park->s2[acc.slot] = 0.0;
    ++acc.nparked;
  }
  acc.slot += real ? 1 : 0;
  if (acc.slot == 32) {
    __syncwarp();
    fold_parked(acc.park, lane < __shfl_sync(0xffffffffu, acc.nparked, 0), lane);
    __syncwarp();
    acc.slot = 0;
    acc.nparked = 0;
  }
}

// fold the partially filled parking slots after the last tile
__device__ __forceinline__ void warp_tile_flush(WarpTileAcc& acc, int lane) {
  if (acc.slot > 0) {
    __syncwarp();
    fold_parked(acc.park, lane < __shfl_sync(0xffffffffu, acc.nparked, 0), lane);
  }
  __syncwarp();
}

// Per-block partial + last-block finalize (completion counter): block partials
// are combined in block order, so the result is deterministic.  `R` = the
// filter resampled at this step; `max_blocks` = per-filter stride of the
// partials in A.workspace.
// (vb, nvb): this block's index among the filter's nvb blocks (blockIdx.x /
// gridDim.x of a plain launch; a virtual block of the persistent kernel).
template <int NT>
__device__ __forceinline__ void pw_block_finalize(const ssm_pw_args& A, ssm_filter_state* fs, int b, int P, int R,
                                                  int has_obs, Lse st, int lane, int max_blocks, int vb, int nvb) {
  // ---- per-block partial + last-block finalize ----
  __shared__ Lse red[NT / 32];
  __shared__ bool s_last;
  Lse* parts = reinterpret_cast<Lse*>(A.workspace) + static_cast<size_t>(b) * max_blocks;
  if (has_obs) {
    // lane 0 of each warp holds its warp's partial: fold the NT/32 warp partials in
    // warp 0 (the same combination tree lse_block_reduce applies, without its
    // intra-warp pass over empty lanes)
    const int warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = st;
    __syncthreads();
    if (warp == 0) {
      Lse r = lane < NT / 32 ? red[lane] : lse_empty();
#pragma unroll
      for (int off = NT / 64; off > 0; off >>= 1) r = lse_combine(r, lse_shfl_down(r, off));
      if (lane == 0) parts[vb] = r;
    }
  }
  // the last block reads only the partials thread 0 wrote (error flags are atomics),
  // so thread 0 alone fences before taking its ticket
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&fs->blocks_done, 1u) == static_cast<unsigned>(nvb - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  if (has_obs) {
    Lse acc = lse_empty();
    for (int i = threadIdx.x; i < nvb; i += NT) {
      const Lse q{__ldcg(&parts[i].m), __ldcg(&parts[i].c), __ldcg(&parts[i].t),
                  __ldcg(&parts[i].s2)};
      acc = lse_combine(acc, q);
    }
    acc = lse_block_reduce<NT>(acc, red);
    if (threadIdx.x == 0 && A.lse_out) {
      // sharded filter: hand the rank's partial to the cross-rank combine (C1)
      double* o = static_cast<double*>(A.lse_out) + 4 * b;
      o[0] = acc.m;
      o[1] = acc.c;
      o[2] = acc.t;
      o[3] = acc.s2;
    } else if (threadIdx.x == 0) {
      const double incr = lse_value(acc);
      const double ess = lse_ess(acc);
      if (!isfinite(incr)) {
        fs->err_degenerate = min(fs->err_degenerate, A.step);
      } else {
        fs->loglik += incr;
      }
      fs->incr = incr;
      fs->lse_raw = incr;
      fs->ess = ess;
      fs->uniform = 0;
      fs->resample_now = (A.ess_rel < 0.0) ? 1 : (ess < A.ess_rel * static_cast<double>(P) ? 1 : 0);
    }
  } else if (threadIdx.x == 0 && R) {
    fs->uniform = 1;  // resampled, no weighting at this step
    fs->resample_now = 0;
  }
  if (threadIdx.x == 0) fs->blocks_done = 0u;
}

}  // namespace ssm
