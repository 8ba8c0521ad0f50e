// K4 weight scan, K5 ancestor search, K6 gather, K8 trace, K3 standalone LSE,
// K9 theta-block gather.  Reference: inference/resampling.py:15-36,
// inference/particle.py:96-105 and 137-149, inference/smc.py:96-98.

#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <type_traits>

#include "ssm_common.cuh"
#include "ssm_tile.cuh"

namespace ssm {

// ===========================================================================
// K4: decoupled-look-back inclusive scan of 64-bit fixed-point weights.
//
// q_j = round(w_j * 2^61) with w normalised (sum ~ 1), so every partial sum
// stays < 2^62 and the top two bits of a tile-status word carry its state.
// Integer addition is associative, so the look-back result is exact and
// independent of timing: the CDF is bitwise deterministic,
// which a floating-point look-back is not.  cum_j = C_j / C_{P-1} reproduces
// cumsum(w / w.sum()) with cum[-1] = 1 (resampling.py:26-27).
// ===========================================================================

constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;  // 2048 weights per tile
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValueMask = (1ull << 62) - 1;
constexpr double kFix = 2305843009213693952.0;  // 2^61

__host__ __device__ inline int scan_tiles(int P) { return (P + kScanTile - 1) / kScanTile; }

struct ScanWs {
  uint32_t* counter;  // dynamic tile ticket
  uint32_t* done;     // [B] completion counters of the raw-weight pre-pass
  uint64_t* status;   // [B][tiles]
  double* scale;      // [B] raw-weight totals
  double* partial;    // [B][kRawBlocks] raw-weight block sums
};

constexpr int kRawBlocks = 1024;

__host__ __device__ inline size_t align256(size_t n) { return (n + 255) & ~size_t(255); }

// layout: [counter + done (zeroed per call)] [status (zeroed per call)] [scale] [partial]
__host__ inline size_t scan_ws_zero_bytes(int B, int P) {
  return align256(sizeof(uint32_t) * (1 + static_cast<size_t>(B))) +
         align256(sizeof(uint64_t) * static_cast<size_t>(B) * scan_tiles(P));
}

__host__ inline ScanWs scan_ws(void* base, int B, int P) {
  char* p = static_cast<char*>(base);
  ScanWs w;
  w.counter = reinterpret_cast<uint32_t*>(p);
  w.done = w.counter + 1;
  p += align256(sizeof(uint32_t) * (1 + static_cast<size_t>(B)));
  w.status = reinterpret_cast<uint64_t*>(p);
  p += align256(sizeof(uint64_t) * static_cast<size_t>(B) * scan_tiles(P));
  w.scale = reinterpret_cast<double*>(p);
  p += align256(sizeof(double) * B);
  w.partial = reinterpret_cast<double*>(p);
  return w;
}

__host__ inline size_t scan_ws_bytes(int B, int P) {
  return scan_ws_zero_bytes(B, P) + align256(sizeof(double) * B) +
         align256(sizeof(double) * static_cast<size_t>(B) * kRawBlocks);
}

__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  *reinterpret_cast<volatile uint64_t*>(p) = v;
}

// raw-weight pre-pass: validation + total (resampling.py:18-24), deterministic
__global__ void __launch_bounds__(kThreads)
raw_total_kernel(int P, const double* w, double* partial, uint32_t* done, double* scale,
                 uint32_t* flags) {
  const int b = blockIdx.y;
  const double* wb = w + static_cast<size_t>(b) * P;
  double s = 0.0;
  uint32_t f = 0;
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads) {
    const double v = wb[p];
    if (!(v >= 0.0) || !isfinite(v)) f |= SSM_FLAG_BAD_WEIGHT;
    s += v;
  }
  __shared__ double red[kThreads];
  __shared__ uint32_t fred;
  __shared__ bool last;
  if (threadIdx.x == 0) fred = 0;
  red[threadIdx.x] = s;
  __syncthreads();
  if (f) atomicOr(&fred, f);
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[static_cast<size_t>(b) * gridDim.x + blockIdx.x] = red[0];
    if (fred) atomicOr(&flags[b], fred);
    __threadfence();
    last = atomicAdd(&done[b], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) t += __ldcg(&partial[static_cast<size_t>(b) * gridDim.x + i]);
    scale[b] = t;
    if (!(t > 0.0)) atomicOr(&flags[b], SSM_FLAG_ZERO_TOTAL);
    done[b] = 0;
  }
}

template <typename T, bool IS_LOG>
__global__ void __launch_bounds__(kThreads)
scan_kernel(int B, int P, const T* __restrict__ a, const double* __restrict__ shift,
            const ssm_filter_state* __restrict__ fs, uint64_t* __restrict__ C, ScanWs ws,
            uint32_t* __restrict__ flags = nullptr) {
  __shared__ uint64_t sm[kScanTile + kScanTile / 8];  // padded: e -> e + e/8
  __shared__ uint64_t warp_tot[kThreads / 32];
  __shared__ uint64_t s_excl;
  __shared__ int s_tile;
  const int tiles = scan_tiles(P);
  if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(ws.counter, 1u));
  __syncthreads();
  const int ticket = s_tile;
  const int b = ticket / tiles;
  const int j = ticket % tiles;
  if (b >= B) return;
  if (fs && !fs[b].resample_now) return;  // whole filter skipped (uniform -> no resample)
  const size_t off = static_cast<size_t>(b) * P + static_cast<size_t>(j) * kScanTile;
  const int n = min(kScanTile, P - j * kScanTile);
  double sh = 0.0;
  if (IS_LOG) sh = shift ? shift[b] : fs[b].incr;
  const double total = IS_LOG ? 1.0 : ws.scale[b];

  // coalesced load -> fixed point -> padded smem
  bool over = false;  // normalisation precondition violated (is_log): reported, not wrapped
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    uint64_t q = 0;
    if (e < n) {
      double w;
      if (IS_LOG) {
        w = exp(static_cast<double>(a[off + e]) - sh);
      } else {
        w = static_cast<double>(a[off + e]) / total;
      }
      q = (w >= 0.0 && w <= 4.0) ? __double2ull_rn(w * kFix) : 0ull;
      if (IS_LOG && w > 1.0 + 0x1p-20) over = true;
    }
    sm[e + (e >> 3)] = q;
  }
  if (IS_LOG && flags && __syncthreads_or(over)) {
    if (threadIdx.x == 0) atomicOr(&flags[b], SSM_FLAG_UNNORMALISED);
  }
  __syncthreads();
  // thread-sequential 8 items
  uint64_t v[kScanItems];
  uint64_t run = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = threadIdx.x * kScanItems + i;
    run += sm[e + (e >> 3)];
    v[i] = run;
  }
  // block exclusive scan of thread totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint64_t warp_excl = 0, block_tot = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const uint64_t t = warp_tot[w];
    if (w < warp) warp_excl += t;
    block_tot += t;
  }
  const uint64_t thread_excl = warp_excl + incl - run;

  // decoupled look-back (warp 0)
  uint64_t* status = ws.status + static_cast<size_t>(b) * tiles;
  if (warp == 0) {
    uint64_t excl = 0;
    if (j == 0) {
      if (lane == 0) st_status(&status[0], kFlagPrefix | (block_tot & kValueMask));
    } else {
      if (lane == 0) st_status(&status[j], kFlagAgg | (block_tot & kValueMask));
      int look = j - 1;
      while (true) {
        const int idx = look - lane;
        uint64_t sv = idx >= 0 ? ld_status(&status[idx]) : kFlagPrefix;
        while (__any_sync(0xffffffffu, (sv >> 62) == 0)) {
          if ((sv >> 62) == 0) sv = ld_status(&status[idx]);
        }
        const bool is_prefix = (sv >> 62) == 2;
        const uint32_t pm = __ballot_sync(0xffffffffu, is_prefix);
        const int first = __ffs(pm) - 1;  // nearest predecessor holding a prefix (or -1)
        uint64_t contrib = (first < 0 || lane <= first) ? (sv & kValueMask) : 0ull;
        if (idx < 0) contrib = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_down_sync(0xffffffffu, contrib, o);
        excl += __shfl_sync(0xffffffffu, contrib, 0);
        if (first >= 0) break;
        look -= 32;
      }
      if (lane == 0) st_status(&status[j], kFlagPrefix | ((excl + block_tot) & kValueMask));
    }
    // a prefix at or above 2^62 would spill into the flag bits: report it
    if (lane == 0 && flags && excl + block_tot > kValueMask) atomicOr(&flags[b], SSM_FLAG_UNNORMALISED);
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  const uint64_t base = s_excl + thread_excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = threadIdx.x * kScanItems + i;
    sm[e + (e >> 3)] = base + v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    if (e < n) C[off + e] = sm[e + (e >> 3)];
  }
}

__global__ void fixed_to_cum_kernel(int P, const uint64_t* C, double* cum) {
  const int b = blockIdx.y;
  const uint64_t* cb = C + static_cast<size_t>(b) * P;
  const double tot = static_cast<double>(cb[P - 1]);
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads)
    cum[static_cast<size_t>(b) * P + p] = static_cast<double>(cb[p]) / tot;
}

// ===========================================================================
// K5: ancestor search.  anc_k = #{j : cum_j <= u_k} clipped to P_in - 1
// (searchsorted side='right', resampling.py:36).  All comparisons are done
// in float64 on the exact query values the reference forms:
//   systematic  u_k = (k + u) / P        resampling.py:33
//   stratified  u_k = (k + U_k) / P      resampling.py:31
//   multinomial u_k = U_k                resampling.py:29
// ===========================================================================

template <int KIND>
__device__ __forceinline__ double cum_at(const void* p, size_t off, double tot, int j) {
  if constexpr (KIND == 0) {
    return static_cast<const double*>(p)[off + j];
  } else {
    return static_cast<double>(__ldg(static_cast<const uint64_t*>(p) + off + j)) / tot;
  }
}

template <int KIND>
__device__ __forceinline__ double cum_total(const void* p, size_t off, int P_in) {
  if constexpr (KIND == 0) {
    return 1.0;
  } else {
    return static_cast<double>(static_cast<const uint64_t*>(p)[off + P_in - 1]);
  }
}

__device__ __forceinline__ double device_uniform(uint32_t k0, uint32_t k1, uint32_t k, uint32_t step,
                                                 uint32_t purpose) {
  const U4 r = philox4x32_10(U4{k, step, 0u, purpose}, k0, k1);
  return u53(r.x, r.y);
}

// query value u_k for SCHEME (stratified / systematic)
template <int SCHEME>
__device__ __forceinline__ double query(int k, int P_out, double u_sys, const double* uarr,
                                        uint32_t k0, uint32_t k1, int step) {
  if constexpr (SCHEME == SSM_SYSTEMATIC) {
    return (static_cast<double>(k) + u_sys) / static_cast<double>(P_out);
  } else {
    const double U = uarr ? uarr[k] : device_uniform(k0, k1, k, step, kPurposeResample);
    return (static_cast<double>(k) + U) / static_cast<double>(P_out);
  }
}

constexpr int kMergeItems = 8;

// ---------------------------------------------------------------------------
// Systematic / stratified: offspring boundaries + merge-path partition.
//
// The queries are sorted, so output k descends from particle j iff
//   c_{j-1} <= k < c_j,   c_j = #{k : u_k < cum_j}   (searchsorted 'right').
// c_j is computed exactly per particle (an estimate from cum_j * P, then the
// reference's own predicate on the exact float64 query values), so no
// binary search over the CDF is needed.  On the merge path of (c, outputs)
// particle j sits at diagonal j + c_j; the kernel that computes c_j also
// writes, for every diagonal tile boundary D it owns, split[D / kDiag] = j,
// which is the partition the expand kernel needs (no per-block searches).
// ---------------------------------------------------------------------------

constexpr int kDiag = 2048;  // merged-diagonal elements per expand block
constexpr int kShortRun = 32;    // offspring runs up to this length are written by the offspring kernel
constexpr int kRunChunk = 4096;  // long runs are filled in chunks of this many outputs
__host__ __device__ inline size_t long_runs_cap(int P_in, int P_out) {
  (void)P_in;  // a long run has > kShortRun outputs: at most P_out / kShortRun of them
  return static_cast<size_t>(P_out / kShortRun) + static_cast<size_t>(P_out / kRunChunk) + 4;
}

enum CumSrc { kCumDouble = 0, kCumFixed = 1, kCumLogw = 2, kCumTiles = 3 };

// layout of the kCumTiles prefix buffer: [B][nt] in-block tile prefixes, then [B][nblk] block prefixes
__host__ __device__ inline size_t B_total_tiles_offset(int nt, int B) { return static_cast<size_t>(B) * nt; }

constexpr double kTileScale = 512.0;  // 2^9: tile-local 2^52 fixed point -> global 2^61

__device__ __forceinline__ double sys_query(int k, double u, int P_out, double invP, bool pow2) {
  const double num = static_cast<double>(k) + u;
  return pow2 ? num * invP : num / static_cast<double>(P_out);  // exact scaling when P is 2^n
}

// c = #{k in [0, P_out) : u_k < cum}, u_k non-decreasing
template <int SCHEME>
__device__ __forceinline__ int offspring_bound(double cum, double u_sys, const double* U, uint32_t k0,
                                               uint32_t k1, int step, int P_out, double invP,
                                               bool pow2) {
  auto f = [&](int k) -> double {
    if constexpr (SCHEME == SSM_SYSTEMATIC) {
      return sys_query(k, u_sys, P_out, invP, pow2);
    } else {
      const double Uk = U ? U[k] : device_uniform(k0, k1, static_cast<uint32_t>(k), step, kPurposeResample);
      return sys_query(k, Uk, P_out, invP, pow2);
    }
  };
  if (!(cum > 0.0)) return 0;  // u_k >= 0
  if constexpr (SCHEME == SSM_SYSTEMATIC) {
    // Fast accept: query k satisfies fl(fl(k + u) / P) < cum  <=>  k < cum P - u
    // up to ~2^-27 absolute rounding (k < 2^25, P <= 2^30 checked below), so when
    // t = cum P - u lies more than 2^-20 from an integer, ceil(t) is the count
    // exactly; otherwise verify query by query as below.
    const double t = cum * static_cast<double>(P_out) - u_sys;
    const double e = ceil(t);
    if (e - t > 0x1p-20 && t - (e - 1.0) > 0x1p-20 && P_out <= (1 << 30))
      return t <= 0.0 ? 0 : (e >= static_cast<double>(P_out) ? P_out : static_cast<int>(e));
  }
  if constexpr (SCHEME == SSM_STRATIFIED) {
    // Stratified: query k is (k + U_k) / P, so with t = cum P every k < floor(t) is
    // counted and every k > floor(t) is not, up to the same ~2^-27 rounding; when t
    // lies more than 2^-20 from an integer only query floor(t) needs its uniform
    // (one Philox draw instead of the walk's two or three).
    const double t = cum * static_cast<double>(P_out);
    const double fl = floor(t);
    if (t - fl > 0x1p-20 && (fl + 1.0) - t > 0x1p-20 && P_out <= (1 << 30)) {
      if (fl >= static_cast<double>(P_out)) return P_out;
      const int k = static_cast<int>(fl);
      return f(k) < cum ? k + 1 : k;
    }
  }
  double est = SCHEME == SSM_SYSTEMATIC ? ceil(cum * P_out - u_sys) : floor(cum * P_out);
  est = est < 0.0 ? 0.0 : (est > P_out ? static_cast<double>(P_out) : est);
  int k = static_cast<int>(est);
  while (k > 0 && f(k - 1) >= cum) --k;
  while (k < P_out && f(k) < cum) ++k;
  return k;
}

// per-tile fixed-point sums of q_j = round(exp(a_j - shift) * 2^61)
template <typename T>
__global__ void __launch_bounds__(kThreads)
tile_sums_kernel(int P, const T* __restrict__ a, const double* __restrict__ shift,
                 const ssm_filter_state* __restrict__ fs, uint64_t* __restrict__ sums) {
  const int b = blockIdx.y, tile = blockIdx.x;
  if (fs && !fs[b].resample_now) return;
  const double sh = shift ? shift[b] : fs[b].incr;
  const T* ab = a + static_cast<size_t>(b) * P + static_cast<size_t>(tile) * kScanTile;
  const int n = min(kScanTile, P - tile * kScanTile);
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = i * kThreads + threadIdx.x;
    if (e < n) {
      const double w = exp(static_cast<double>(ab[e]) - sh);
      acc += (w >= 0.0 && w <= 4.0) ? __double2ull_rn(w * kFix) : 0ull;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ uint64_t red[kThreads / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    sums[static_cast<size_t>(b) * gridDim.x + tile] = t;
  }
}

// exclusive prefix of the tile sums, one 1024-thread block per filter
__global__ void __launch_bounds__(1024)
tile_prefix_kernel(int tiles, uint64_t* __restrict__ sums, uint64_t* __restrict__ totals,
                   const ssm_filter_state* __restrict__ fs) {
  const int b = blockIdx.x;
  if (fs && !fs[b].resample_now) return;
  uint64_t* sb = sums + static_cast<size_t>(b) * tiles;
  const int per = (tiles + 1023) / 1024;
  const int t0 = threadIdx.x * per;
  uint64_t local = 0;
  for (int t = t0; t < min(t0 + per, tiles); ++t) local += sb[t];
  __shared__ uint64_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint64_t wex = 0, tot = 0;
  for (int w = 0; w < 32; ++w) {
    if (w < warp) wex += wsum[w];
    tot += wsum[w];
  }
  uint64_t run = wex + incl - local;
  for (int t = t0; t < min(t0 + per, tiles); ++t) {
    const uint64_t v = sb[t];
    sb[t] = run;
    run += v;
  }
  if (threadIdx.x == 0) totals[b] = tot;
}

// Per-warp-tile global scale and exact exclusive prefix, from the pw kernel's
// tile records.  Q'_w = round(exp(m_w - incr) 2^9 Q_w) is exactly the value the
// offspring kernel reaches at the tile's last particle, so the global CDF is
// monotone and deterministic.  Two launches: per-block (2048 tiles) scan, then
// a 1-block scan of the block totals.
constexpr int kRecPerBlock = kThreads;  // 256 tile records per block (one per thread)

// per-filter constants of the tile-path offspring kernel (blk_prefix_kernel):
// 1 / total, P / total, the systematic uniform, 1 / P
struct OffspringConsts {
  double inv, tscale, u_sys, invP;
};

// Exclusive prefix of one filter's block totals in place, the filter total and
// (oc != nullptr) the offspring kernel's per-filter constants; one block of NT threads.
template <int NT>
__device__ __forceinline__ void filter_block_prefix(int nblk, uint64_t* __restrict__ bb, uint64_t* __restrict__ totals,
                                                    int b, OffspringConsts* __restrict__ oc, int P,
                                                    const double* __restrict__ u, const uint32_t* __restrict__ keys,
                                                    int step) {
  const int per = (nblk + NT - 1) / NT;
  const int t0 = threadIdx.x * per, t1 = min(t0 + per, nblk);
  uint64_t local = 0;
  for (int t = t0; t < t1; ++t) local += __ldcg(bb + t);
  __shared__ uint64_t wsum[NT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  uint64_t wex = 0, tot = 0;
  for (int w = 0; w < NT / 32; ++w) {
    if (w < warp) wex += wsum[w];
    tot += wsum[w];
  }
  uint64_t run = wex + incl - local;
  for (int t = t0; t < t1; ++t) {
    const uint64_t x = __ldcg(bb + t);
    bb[t] = run;
    run += x;
  }
  if (threadIdx.x == 0) {
    totals[b] = tot;
    if (oc) {  // the offspring kernel's per-filter constants, computed once
      const double inv = 1.0 / static_cast<double>(tot);
      const double Pd = static_cast<double>(P);
      const double us = u ? u[b] : (keys ? device_uniform(keys[2 * b], keys[2 * b + 1], 0u, step, kPurposeSystematic) : 0.0);
      oc[b] = OffspringConsts{inv, Pd * inv, us, 1.0 / Pd};
    }
  }
}

// Per-warp-tile scale and exclusive in-block prefix (one record per thread) and
// block totals.  With `fs_rw` (the filter path) the last block of each filter to
// finish (completion counter fs.prefix_done) also turns the block totals into
// exclusive block prefixes, so the offspring kernel follows directly.
// block blk (of nblk) of filter b (the persistent driver runs it on virtual blocks)
__device__ __forceinline__ void tile_scale_body(int b, int blk, int nblk, int ntiles, const ssm_tile_rec* __restrict__ rec,
                                                const ssm_filter_state* __restrict__ fs, double* __restrict__ scale,
                                                uint64_t* __restrict__ prel, uint64_t* __restrict__ blk_tot,
                                                uint32_t* __restrict__ long_count, int gate, ssm_filter_state* fs_rw,
                                                uint64_t* __restrict__ totals, OffspringConsts* __restrict__ oc, int P,
                                                const double* __restrict__ u, const uint32_t* __restrict__ keys,
                                                int step) {
  __shared__ uint64_t warp_tot[kThreads / 32];
  __shared__ bool s_last;
  const int e = blk * kRecPerBlock + threadIdx.x;
  const size_t off = static_cast<size_t>(b) * ntiles + e;
  // the record load is issued before the gate / incr loads so their latencies overlap
  ssm_tile_rec r{0.0, 0ull};
  if (e < ntiles) r = rec[off];
  const double incr = fs[b].incr;
  if (gate && !fs[b].resample_now) return;
  if (long_count && blk == 0 && threadIdx.x == 0) long_count[b] = 0u;  // long-run list of this resample
  uint64_t qg = 0;
  if (e < ntiles) {
    const double sc = r.m == -CUDART_INF ? 0.0 : exp(r.m - incr) * kTileScale;
    scale[off] = sc;
    const double v = sc * static_cast<double>(r.Q);
    qg = (v >= 0.0 && v < 4.0e18) ? __double2ull_rn(v) : 0ull;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t incl = qg;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  uint64_t wex = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) wex += warp_tot[w];
    tot += warp_tot[w];
  }
  if (e < ntiles) prel[off] = wex + incl - qg;  // exclusive, exact integer
  if (threadIdx.x == 0) blk_tot[static_cast<size_t>(b) * nblk + blk] = tot;
  if (!fs_rw) return;
  // only thread 0's block total is read by the last block (prel is read by the
  // next kernel), so only thread 0 fences before taking a ticket
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&fs_rw[b].prefix_done, 1u) == static_cast<unsigned>(nblk - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  filter_block_prefix<kThreads>(nblk, blk_tot + static_cast<size_t>(b) * nblk, totals, b, oc, P, u, keys, step);
  if (threadIdx.x == 0) fs_rw[b].prefix_done = 0u;
}

__global__ void __launch_bounds__(kThreads)
tile_scale_kernel(int ntiles, const ssm_tile_rec* __restrict__ rec, const ssm_filter_state* __restrict__ fs,
                  double* __restrict__ scale, uint64_t* __restrict__ prel, uint64_t* __restrict__ blk_tot,
                  uint32_t* __restrict__ long_count = nullptr, int gate = 1, ssm_filter_state* fs_rw = nullptr,
                  uint64_t* __restrict__ totals = nullptr, OffspringConsts* __restrict__ oc = nullptr, int P = 0,
                  const double* __restrict__ u = nullptr, const uint32_t* __restrict__ keys = nullptr,
                  int step = 0) {
  pdl_wait();
  tile_scale_body(blockIdx.y, blockIdx.x, gridDim.x, ntiles, rec, fs, scale, prel, blk_tot, long_count, gate, fs_rw,
                  totals, oc, P, u, keys, step);
}

__global__ void __launch_bounds__(1024)
blk_prefix_kernel(int nblk, uint64_t* __restrict__ blk, uint64_t* __restrict__ totals,
                  const ssm_filter_state* __restrict__ fs, OffspringConsts* __restrict__ oc = nullptr, int P = 0,
                  const double* __restrict__ u = nullptr, const uint32_t* __restrict__ keys = nullptr, int step = 0) {
  pdl_wait();
  const int b = blockIdx.x;
  if (fs && !fs[b].resample_now) return;
  filter_block_prefix<1024>(nblk, blk + static_cast<size_t>(b) * nblk, totals, b, oc, P, u, keys, step);
}

// c_j for every particle + merge-path partition entries
// g_off (nullable, sharded filter): global fixed-point offset of this rank's
// first particle; `totals` is then the global total and P_out the global
// particle count.  c_shift (nullable): subtracted from every stored c_j (the
// rank's first output), so partition and expand work on the rank's own outputs.
template <int SCHEME, int SRC, typename T>
__global__ void __launch_bounds__(kThreads)
offspring_kernel(int P_in, int P_out, const void* __restrict__ src, const double* __restrict__ shift,
                 const uint64_t* __restrict__ tile_prefix, const uint64_t* __restrict__ totals,
                 const double* __restrict__ u, const uint32_t* __restrict__ keys, int step,
                 const ssm_filter_state* __restrict__ fs, int32_t* __restrict__ cnt,
                 int32_t* __restrict__ split, int ndiag, const uint64_t* __restrict__ g_off = nullptr,
                 const int32_t* __restrict__ c_shift = nullptr) {
  __shared__ __align__(16) uint64_t sm[kScanTile + kScanTile / 8];
  __shared__ uint64_t warp_tot[kThreads / 32];
  const int b = blockIdx.y, tile = blockIdx.x;
  if (fs && !fs[b].resample_now) return;
  const int tiles = gridDim.x;
  const int j0 = tile * kScanTile;
  const int n = min(kScanTile, P_in - j0);
  const bool pow2 = (P_out & (P_out - 1)) == 0;
  const double invP = 1.0 / static_cast<double>(P_out);
  const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
  double u_sys = 0.0;
  if constexpr (SCHEME == SSM_SYSTEMATIC) {
    if (u) {
      u_sys = u[b];
    } else {  // one Philox draw per block, not per thread
      __shared__ double s_u;
      if (threadIdx.x == 0) s_u = device_uniform(k0, k1, 0u, step, kPurposeSystematic);
      __syncthreads();
      u_sys = s_u;
    }
  }
  const double* U = (SCHEME == SSM_STRATIFIED && u) ? u + static_cast<size_t>(b) * P_out : nullptr;
  int32_t* cb = cnt + static_cast<size_t>(b) * P_in;
  int32_t* sp = split + static_cast<size_t>(b) * (ndiag + 1);

  // cum_j for the thread's kScanItems consecutive particles, and cum_{j-1}
  double cum[kScanItems];
  double cum_prev;
  const int jt = j0 + threadIdx.x * kScanItems;
  if constexpr (SRC == kCumDouble) {
    const double* cd = static_cast<const double*>(src) + static_cast<size_t>(b) * P_in;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) cum[i] = jt + i < P_in ? cd[jt + i] : 2.0;
    cum_prev = (jt > 0 && jt <= P_in) ? cd[jt - 1] : 0.0;  // threads past P_in return below
  } else if constexpr (SRC == kCumTiles) {
    // src = cdf_local (u64 [B][P]); `shift` = per-warp-tile scale exp(m_w - incr) 2^9
    // [B][nt]; tile_prefix = per-tile exclusive prefix within its 2048-tile block
    // [B][nt] followed by the block prefixes [B][nblk].
    const int nt = (P_in + 31) / 32;
    const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
    const uint64_t* cl = static_cast<const uint64_t*>(src) + static_cast<size_t>(b) * P_in;
    const int tw = jt >> 5;  // kScanItems consecutive particles share one warp tile
    const bool ok = tw < nt;
    const double sc = ok ? shift[static_cast<size_t>(b) * nt + tw] : 0.0;
    const uint64_t* blk_pre = tile_prefix + static_cast<size_t>(B_total_tiles_offset(nt, gridDim.y));
    const uint64_t goff = g_off ? g_off[b] : 0ull;
    const uint64_t pre = goff + (ok ? tile_prefix[static_cast<size_t>(b) * nt + tw] +
                                          blk_pre[static_cast<size_t>(b) * nblk + tw / kRecPerBlock]
                                    : 0ull);
    const double inv = 1.0 / static_cast<double>(totals[b]);
    uint64_t lv[kScanItems];
    if (jt + kScanItems <= P_in && (P_in & 7) == 0) {  // 4 x 16-byte vector loads, aligned
      const ulonglong2* v2 = reinterpret_cast<const ulonglong2*>(cl + jt);
#pragma unroll
      for (int i = 0; i < kScanItems / 2; ++i) {
        const ulonglong2 t2 = __ldg(v2 + i);
        lv[2 * i] = t2.x;
        lv[2 * i + 1] = t2.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kScanItems; ++i) lv[i] = jt + i < P_in ? cl[jt + i] : 0ull;
    }
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int j = jt + i;
      cum[i] = j < P_in ? static_cast<double>(pre + __double2ull_rn(sc * static_cast<double>(lv[i]))) * inv : 2.0;
      if (j == P_in - 1 && (!g_off || goff + blk_pre[static_cast<size_t>(b) * nblk + nblk - 1] +
                                              tile_prefix[static_cast<size_t>(b) * nt + nt - 1] +
                                              __double2ull_rn(shift[static_cast<size_t>(b) * nt + nt - 1] *
                                                              static_cast<double>(cl[P_in - 1])) == totals[b]))
        cum[i] = 1.0;  // cum[-1] = 1.0 (resampling.py:27)
    }
    cum_prev = jt == 0 ? static_cast<double>(goff) * inv
               : ((jt & 31) == 0 || jt > P_in  // (threads past P_in return below)
                      ? static_cast<double>(pre) * inv
                      : static_cast<double>(pre + __double2ull_rn(sc * static_cast<double>(cl[jt - 1]))) * inv);
  } else {
    const size_t off = static_cast<size_t>(b) * P_in + j0;
    double sh = 0.0;
    if constexpr (SRC == kCumLogw) sh = shift ? shift[b] : fs[b].incr;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      const int e = i * kThreads + threadIdx.x;
      uint64_t q = 0;
      if (e < n) {
        if constexpr (SRC == kCumLogw) {
          const double w = exp(static_cast<double>(static_cast<const T*>(src)[off + e]) - sh);
          q = (w >= 0.0 && w <= 4.0) ? __double2ull_rn(w * kFix) : 0ull;
        } else {
          q = static_cast<const uint64_t*>(src)[off + e];  // inclusive C_j already
        }
      }
      sm[e + (e >> 3)] = q;
    }
    __syncthreads();
    double tot;
    uint64_t Cv[kScanItems];
    uint64_t Cprev;
    if constexpr (SRC == kCumLogw) {
      uint64_t run = 0;
#pragma unroll
      for (int i = 0; i < kScanItems; ++i) {
        const int e = threadIdx.x * kScanItems + i;
        run += sm[e + (e >> 3)];
        Cv[i] = run;
      }
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      uint64_t incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) warp_tot[warp] = incl;
      __syncthreads();
      uint64_t wex = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w)
        if (w < warp) wex += warp_tot[w];
      const uint64_t base = tile_prefix[static_cast<size_t>(b) * tiles + tile] + wex + incl - run;
#pragma unroll
      for (int i = 0; i < kScanItems; ++i) Cv[i] += base;
      Cprev = base;
      tot = static_cast<double>(totals[b]);
    } else {
      const uint64_t* Cb = static_cast<const uint64_t*>(src) + static_cast<size_t>(b) * P_in;
#pragma unroll
      for (int i = 0; i < kScanItems; ++i) {
        const int e = threadIdx.x * kScanItems + i;
        Cv[i] = sm[e + (e >> 3)];
      }
      Cprev = (jt > 0 && jt <= P_in) ? Cb[jt - 1] : 0ull;  // threads past P_in return below
      tot = static_cast<double>(Cb[P_in - 1]);
    }
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      cum[i] = jt + i < P_in ? static_cast<double>(Cv[i]) / tot : 2.0;
    cum_prev = jt > 0 ? static_cast<double>(Cprev) / tot : 0.0;
  }

  const int cshift = c_shift ? c_shift[b] : 0;
  if (jt >= P_in) return;
  int c_prev = (jt > 0 || g_off) ? offspring_bound<SCHEME>(cum_prev, u_sys, U, k0, k1, step, P_out, invP, pow2) - cshift
                                 : 0;
  const int total = P_in + P_out;
  int32_t cvals[kScanItems];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int j = jt + i;
    if (j >= P_in) break;
    const int c = offspring_bound<SCHEME>(cum[i], u_sys, U, k0, k1, step, P_out, invP, pow2) - cshift;
    cvals[i] = c;
    // diagonal boundaries D in (j-1 + c_prev, j + c] are split at particle j
    const int lo = j - 1 + c_prev, hi = j + c;
    for (int t = lo / kDiag + 1; t * kDiag <= hi && t <= ndiag; ++t) sp[t] = j;
    if (j == P_in - 1) {
      for (int t = hi / kDiag + 1; t <= ndiag; ++t) sp[t] = P_in;  // tail outputs, and D = total
    }
    if (j == 0) sp[0] = 0;
    c_prev = c;
  }
  (void)total;
  if (jt + kScanItems <= P_in && (P_in & 7) == 0) {  // two 16-byte vector stores, aligned
    int4* c4 = reinterpret_cast<int4*>(cb + jt);
    c4[0] = make_int4(cvals[0], cvals[1], cvals[2], cvals[3]);
    c4[1] = make_int4(cvals[4], cvals[5], cvals[6], cvals[7]);
  } else {
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
      if (jt + i < P_in) cb[jt + i] = cvals[i];
  }
}

// Long offspring runs (> kShortRun outputs of one particle, e.g. degenerate
// weights): one block per run, grid-stride over runs.
// Where an output's ancestor goes: this filter's own array (LocalStore), or --
// sharded filter -- the array of the rank that owns output slot k, through
// that rank's peer-mapped pointer (PeerStore: a P2P store over NVLink when the
// owner is another GPU); `base` turns a local particle index into a global one.
struct LocalStore {
  int32_t* anc;  // [B][P]
  int P;
  __device__ __forceinline__ void operator()(int b, int k, int v) const { anc[static_cast<size_t>(b) * P + k] = v; }
};
struct PeerStore {
  int32_t* const* tab;  // [W] owners' ancestor arrays for this step (peer-mapped)
  int P_loc;
  int base;             // global index of this rank's particle 0
  __device__ __forceinline__ void operator()(int, int k, int v) const {
    const int o = k / P_loc;
    tab[o][k - o * P_loc] = v + base;
  }
};

template <typename Store>
__device__ __forceinline__ void long_runs_body(int b, int r0, int rstride, int P_in, int P_out,
                                               const int4* __restrict__ runs, const uint32_t* __restrict__ count,
                                               const ssm_filter_state* __restrict__ fs, const Store& st) {
  if (fs && !fs[b].resample_now) return;
  const uint32_t n = count[b];
  const int4* rb = runs + static_cast<size_t>(b) * long_runs_cap(P_in, P_out);
  for (uint32_t r = r0; r < n; r += rstride) {
    const int4 q = rb[r];
    for (int k = q.y + threadIdx.x; k < q.z; k += kThreads) st(b, k, q.x);
  }
}

template <typename Store = LocalStore>
__global__ void __launch_bounds__(kThreads)
long_runs_kernel(int P_in, int P_out, const int4* __restrict__ runs, const uint32_t* __restrict__ count,
                 const ssm_filter_state* __restrict__ fs, Store st) {
  pdl_wait();
  long_runs_body(blockIdx.y, blockIdx.x, gridDim.x, P_in, P_out, runs, count, fs, st);
  if constexpr (!std::is_same<Store, LocalStore>::value) __threadfence_system();  // peer stores
}

// Filter-path offspring + ancestors from the fused kernel's tile records
// (ssm_resample_from_tiles).  Lane = particle: each warp walks 8 consecutive
// 32-particle tiles (its tile's prefix and scale are warp-uniform, cdf_local
// loads are coalesced), c_{j-1} comes from the neighbouring lane.  The block's
// output window [c_{j0-1}, c_{j0+2047}) is then filled in shared memory: run
// starts are marked with their particle and an inclusive max-scan propagates
// them; blocks whose window exceeds the staging buffer (degenerate weights)
// write short runs directly and defer long ones to long_runs_kernel.
// Counts are c_j = #{k : u_k < C_j / total} exactly (systematic fast accept when
// C_j P / total - u is not within 2^-20 of an integer, query-by-query otherwise);
// the last particle's run ends at P (cum[-1] = 1.0, resampling.py:27 + clip).
// Shared-memory window of a block's outputs (see offspring_tiles_kernel).
constexpr int kRunIt = kScanTile / kThreads;  // 32-particle tiles per warp (8)
struct RunWindow {
  int32_t out[4096 + 4096 / 32];
  int lo, hi;
  int wmax[kThreads / 32];
};

// Writes anc for a block's particles [jw, jw + 256) per warp (lane = particle,
// cv / pv = c_j / c_{j-1} for the warp's 8 tiles).  sm.lo = c_{j0-1} must be
// set by the caller before the call; the last thread's cv is the window end.
// Windows up to 4096 outputs are filled in shared memory (run-start marks +
// max-scan) and stored coalesced; larger ones (degenerate weights) write short
// runs directly and defer long runs to long_runs_kernel.
template <typename Store>
__device__ __forceinline__ void fill_run_window(RunWindow& sm, int b, int P, int jw, const int (&cv)[kRunIt],
                                                const int (&pv)[kRunIt], const Store& st,
                                                int4* __restrict__ long_runs, uint32_t* __restrict__ long_count) {
  constexpr int kOutBuf = 4096;
  constexpr int kPer = kOutBuf / kThreads;
  constexpr int kIt = kRunIt;
  static_assert(kPer == 16 && kIt == 8, "layout");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == kThreads - 1) sm.hi = cv[kIt - 1];
  for (int e = threadIdx.x; e < (kOutBuf + kOutBuf / 32) / 4; e += kThreads)
    reinterpret_cast<int4*>(sm.out)[e] = make_int4(-1, -1, -1, -1);
  __syncthreads();
  const int lo_blk = sm.lo, n_out = sm.hi - lo_blk;
  if (n_out <= kOutBuf) {
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int e = pv[it] - lo_blk;
      if (cv[it] > pv[it]) sm.out[e + (e >> 5)] = jw + it * 32 + lane;
    }
    __syncthreads();
    int32_t* sv = sm.out + threadIdx.x * kPer + (threadIdx.x >> 1);  // pad(t*16 + i) = t*16 + i + t/2
    int v[kPer];
    int run = -1;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      run = max(run, sv[i]);
      v[i] = run;
    }
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl = max(incl, y);
    }
    int cin = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) cin = -1;
    if (lane == 31) sm.wmax[warp] = incl;
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w)
      if (w < warp) cin = max(cin, sm.wmax[w]);
#pragma unroll
    for (int i = 0; i < kPer; ++i) sv[i] = max(cin, v[i]);
    __syncthreads();
    for (int e = threadIdx.x; e < n_out; e += kThreads) st(b, lo_blk + e, sm.out[e + (e >> 5)]);
  } else {
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int j = jw + it * 32 + lane, lo = pv[it], hi = cv[it];
      if (hi - lo <= kShortRun) {
        for (int k = lo; k < hi; ++k) st(b, k, j);
      } else {
        const int nchunk = (hi - lo + kRunChunk - 1) / kRunChunk;
        const uint32_t slot = atomicAdd(long_count + b, static_cast<uint32_t>(nchunk));
        int4* rb = long_runs + static_cast<size_t>(b) * long_runs_cap(P, P);
        for (int q = 0; q < nchunk; ++q) {
          const int lo_q = lo + q * kRunChunk;
          rb[slot + q] = make_int4(j, lo_q, min(lo_q + kRunChunk, hi), 0);
        }
      }
    }
  }
}


// Sharded filter (one rank of W): this rank's particles are global indices
// [base, base + P), its fixed-point CDF starts at the global offset g_off, the
// queries run over P_glob global outputs and the ancestors land in the owners'
// arrays (PeerStore).  Single filter: base 0, g_off 0, P_glob = P, LocalStore.
struct ShardSpan {
  const uint64_t* g_off;  // [B] global fixed-point offset of particle 0, or nullptr
  int P_glob;
  int base;
};

// block blk of filter b (of B filters): the body of offspring_tiles_kernel, also run
// by the persistent cooperative driver on virtual blocks
template <int SCHEME, typename Store>
__device__ __forceinline__ void offspring_tiles_body(int b, int blk, int B, int P, const uint64_t* __restrict__ cdf_local,
                                                     const double* __restrict__ scale, const uint64_t* __restrict__ pref,
                                                     const double* __restrict__ u, const uint32_t* __restrict__ keys,
                                                     int step, const ssm_filter_state* __restrict__ fs, const Store& st,
                                                     int4* __restrict__ long_runs, uint32_t* __restrict__ long_count,
                                                     const OffspringConsts* __restrict__ oc, const ShardSpan& span) {
  constexpr int kIt = kRunIt;
  constexpr bool kLocal = std::is_same<Store, LocalStore>::value;
  __shared__ __align__(16) RunWindow sm;
  struct __align__(16) TileInfo {
    uint64_t pre;
    double sc;
  };
  __shared__ TileInfo s_tile[kThreads / 32][kIt];
  const int Pg = kLocal ? P : span.P_glob;  // outputs (global for a sharded filter)
  const uint64_t goff = kLocal ? 0ull : span.g_off[b];
  if (fs && !fs[b].resample_now) {  // ESS gate held (particle.py:99-100): the history records identity
    const int k1 = min(P, (blk + 1) * kScanTile);
    for (int k = blk * kScanTile + threadIdx.x; k < k1; k += kThreads) st(b, k + (kLocal ? 0 : span.base), k);
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = (P + 31) >> 5;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  const uint64_t* tp = pref + static_cast<size_t>(b) * nt;
  const uint64_t* bp = pref + B_total_tiles_offset(nt, B) + static_cast<size_t>(b) * nblk;
  const double* scb = scale + static_cast<size_t>(b) * nt;
  const uint64_t* cl = cdf_local + static_cast<size_t>(b) * P;
  const int jw = blk * kScanTile + warp * (kScanTile / (kThreads / 32));  // warp's first particle
  const int tw0 = jw >> 5;
  // issue every load of the warp's 8 tiles first: cdf_local per lane, and the
  // tiles' prefix / scale one per lane (broadcast by shuffle below).  The last
  // GLOBAL particle's run ends at P_glob; a rank's last local particle is not special.
  const int jlast = kLocal || span.base + P == Pg ? P - 1 : P;
  uint64_t qv[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int j = jw + it * 32 + lane;
    qv[it] = j < jlast ? __ldg(cl + j) : 0ull;
  }
  // the warp's 8 tiles' prefix / scale, one per lane, broadcast through shared memory
  if (lane < kIt) {
    TileInfo ti{goff, 0.0};
    if (tw0 + lane < nt) ti = TileInfo{goff + tp[tw0 + lane] + bp[(tw0 + lane) / kRecPerBlock], scb[tw0 + lane]};
    s_tile[warp][lane] = ti;
  }
  const OffspringConsts K = oc[b];  // 1 / total, P / total, u, 1 / P (blk_prefix_kernel / shard_consts_kernel)
  const double inv = K.inv, tscale = K.tscale, invP = K.invP;
  const bool pow2 = (Pg & (Pg - 1)) == 0;
  const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
  const double u_sys = SCHEME == SSM_SYSTEMATIC ? K.u_sys : 0.0;
  __syncwarp();
  const double* U = (SCHEME == SSM_STRATIFIED && u) ? u + static_cast<size_t>(b) * Pg : nullptr;
  const auto count = [&](uint64_t C) -> int {
    const double Cd = static_cast<double>(C);
    if constexpr (SCHEME == SSM_SYSTEMATIC) {
      const double t = fma(Cd, tscale, -u_sys);
      const double e = ceil(t);
      const double d = e - t;  // in [0, 1), within 2^-53
      if (d > 0x1p-20 && d < 1.0 - 0x1p-20 && Pg <= (1 << 30))
        return min(max(__double2int_rz(e), 0), Pg);
    }
    return offspring_bound<SCHEME>(Cd * inv, u_sys, U, k0, k1, step, Pg, invP, pow2);
  };

  // c_{jw-1}: particle jw-1 closes tile tw0-1, so its C is tile tw0's exclusive prefix
  // (for a sharded rank's particle 0: the previous rank's last particle, C = g_off)
  const uint64_t pre0 = s_tile[warp][0].pre;
  // F: the count of every particle >= jlast (the last global particle's run ends
  // at P_glob; a non-last rank's padding lanes repeat its last particle's count)
  int F = Pg;
  if (!kLocal && jlast == P)
    F = count(goff + tp[nt - 1] + bp[(nt - 1) / kRecPerBlock] + __double2ull_rn(scb[nt - 1] * static_cast<double>(cl[P - 1])));
  int carry = 0;
  if ((jw > 0 || (!kLocal && span.base > 0)) && jw < P) carry = count(pre0);
  else if (jw >= P) carry = F;
  if (warp == 0 && lane == 0) sm.lo = carry;
  int cv[kIt], pv[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int j = jw + it * 32 + lane;
    const TileInfo ti = s_tile[warp][it];
    const uint64_t pre = ti.pre;
    const double sc = ti.sc;
    // the last (global) particle's run ends at P_glob, later lanes are empty
    const int c = j < jlast ? count(pre + __double2ull_rn(sc * static_cast<double>(qv[it]))) : F;
    const int up = __shfl_up_sync(0xffffffffu, c, 1);
    pv[it] = lane == 0 ? carry : up;
    cv[it] = c;
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
  fill_run_window(sm, b, Pg, jw, cv, pv, st, long_runs, long_count);
}

template <int SCHEME, typename Store = LocalStore>
#ifndef SSM_OFFSPRING_MINB
#define SSM_OFFSPRING_MINB 6  // <= 42 registers: 6 CTAs / SM (4 at the default 64); 2^24 resample 99 -> 96 us
#endif
__global__ void __launch_bounds__(kThreads, SSM_OFFSPRING_MINB)
offspring_tiles_kernel(int P, const uint64_t* __restrict__ cdf_local, const double* __restrict__ scale,
                       const uint64_t* __restrict__ pref, const uint64_t* __restrict__ totals,
                       const double* __restrict__ u, const uint32_t* __restrict__ keys, int step,
                       const ssm_filter_state* __restrict__ fs, Store st,
                       int4* __restrict__ long_runs, uint32_t* __restrict__ long_count,
                       const OffspringConsts* __restrict__ oc, ShardSpan span = ShardSpan{nullptr, 0, 0}) {
  pdl_wait();
  (void)totals;
  offspring_tiles_body<SCHEME, Store>(blockIdx.y, blockIdx.x, gridDim.y, P, cdf_local, scale, pref, u, keys, step, fs,
                                      st, long_runs, long_count, oc, span);
  if constexpr (!std::is_same<Store, LocalStore>::value) __threadfence_system();  // peer stores before the barrier
}

// ---------------------------------------------------------------------------
// Fused filter-path resample (systematic / stratified): tile scale, global
// prefix and offspring + ancestors in ONE kernel.  Each block owns 2048
// particles = 64 warp tiles: it scales its tiles' records (Q'_w =
// round(exp(m_w - incr) 2^9 Q_w)), scans them, and obtains its exclusive prefix
// from its predecessors by a decoupled look-back over exact 64-bit integer
// aggregates (associative: the same prefix on every run, whatever the timing).
// The CDF is normalised by the nominal total 2^61 = exp(LSE) on the 2^61 fixed
// point instead of the exact sum of the Q'_w (which would need a second pass
// over all tiles): C_j / 2^61 differs from C_j / sum_w Q'_w by the rounding of
// the LSE (~1e-15 relative), far below the fixed-point CDF's own distance to
// the reference's float64 cumsum.  The last particle's
// run still ends at P (cum[-1] = 1.0, resampling.py:27) and counts clamp at P.
// Look-back status words and the long-run counters are double-buffered by
// `parity`: each launch clears the other parity's words for the next one (whose
// previous user completed before this kernel passed griddepcontrol.wait).
// ---------------------------------------------------------------------------
constexpr int kFusedTiles = kScanTile / 32;  // 64 warp tiles per block
constexpr double kNominalTotal = 2305843009213693952.0;  // 2^61

struct FusedWs {
  uint64_t* status;      // [2][B][nb]
  uint32_t* long_count;  // [2][B]
};

__host__ __device__ inline size_t fused_ws_words(int B, int P) {
  return 2 * static_cast<size_t>(B) * scan_tiles(P) + static_cast<size_t>(B) + 1;
}

__host__ __device__ inline FusedWs fused_ws(uint64_t* base, int B, int P) {
  return FusedWs{base, reinterpret_cast<uint32_t*>(base + 2 * static_cast<size_t>(B) * scan_tiles(P))};
}

template <int SCHEME>
__global__ void __launch_bounds__(kThreads)
resample_fused_kernel(int P, const uint64_t* __restrict__ cdf_local, const ssm_tile_rec* __restrict__ rec,
                      const ssm_filter_state* __restrict__ fs, const double* __restrict__ u,
                      const uint32_t* __restrict__ keys, int step, int32_t* __restrict__ anc,
                      int4* __restrict__ long_runs, FusedWs ws, int parity) {
  pdl_wait();
  constexpr int kIt = kRunIt;
  __shared__ __align__(16) RunWindow sm;
  __shared__ uint64_t s_pre[kFusedTiles];
  __shared__ double s_sc[kFusedTiles];
  __shared__ uint64_t s_wtot[2];
  __shared__ uint64_t s_excl;
  __shared__ double s_usys;
  const int b = blockIdx.y, blk = blockIdx.x, nb = gridDim.x, B = gridDim.y;
  uint64_t* st = ws.status + (static_cast<size_t>(parity) * B + b) * nb;
  uint32_t* long_count = ws.long_count + static_cast<size_t>(parity) * B;
  if (threadIdx.x == 0) {  // the other parity's words, for the next launch
    ws.status[(static_cast<size_t>(parity ^ 1) * B + b) * nb + blk] = 0ull;
    if (blk == 0) ws.long_count[static_cast<size_t>(parity ^ 1) * B + b] = 0u;
  }
  if (fs && !fs[b].resample_now) {  // ESS gate held (particle.py:99-100): the history records identity
    int32_t* ab = anc + static_cast<size_t>(b) * P;
    const int k1 = min(P, (blk + 1) * kScanTile);
    for (int k = blk * kScanTile + threadIdx.x; k < k1; k += kThreads) ab[k] = k;
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nt = (P + 31) >> 5;
  const double incr = fs[b].incr;
  // (1) this block's 64 warp tiles: global scale and in-block exclusive prefix
  uint64_t q = 0, incl = 0;
  if (threadIdx.x < kFusedTiles) {
    const int w = blk * kFusedTiles + threadIdx.x;
    double sc = 0.0;
    if (w < nt) {
      const ssm_tile_rec r = rec[static_cast<size_t>(b) * nt + w];
      sc = r.m == -CUDART_INF ? 0.0 : exp(r.m - incr) * kTileScale;
      const double v = sc * static_cast<double>(r.Q);
      q = (v >= 0.0 && v < 4.0e18) ? __double2ull_rn(v) : 0ull;
    }
    s_sc[threadIdx.x] = sc;
    incl = q;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wtot[warp] = incl;
  }
  if (threadIdx.x == kThreads - 1) {
    const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
    s_usys = SCHEME == SSM_SYSTEMATIC ? (u ? u[b] : device_uniform(k0, k1, 0u, step, kPurposeSystematic)) : 0.0;
  }
  __syncthreads();
  // (2) decoupled look-back for the block's exclusive prefix (warp 0)
  if (warp == 0) {
    const uint64_t btot = s_wtot[0] + s_wtot[1];
    uint64_t excl = 0;
    if (blk == 0) {
      if (lane == 0) st_status(&st[0], kFlagPrefix | (btot & kValueMask));
    } else {
      if (lane == 0) st_status(&st[blk], kFlagAgg | (btot & kValueMask));
      int look = blk - 1;
      while (true) {
        const int idx = look - lane;
        uint64_t sv = idx >= 0 ? ld_status(&st[idx]) : kFlagPrefix;
        while (__any_sync(0xffffffffu, (sv >> 62) == 0)) {
          if ((sv >> 62) == 0) sv = ld_status(&st[idx]);
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
        const int first = __ffs(pm) - 1;  // nearest predecessor holding a prefix
        uint64_t contrib = (first < 0 || lane <= first) ? (sv & kValueMask) : 0ull;
        if (idx < 0) contrib = 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) contrib += __shfl_down_sync(0xffffffffu, contrib, o);
        excl += __shfl_sync(0xffffffffu, contrib, 0);
        if (first >= 0) break;
        look -= 32;
      }
      if (lane == 0) st_status(&st[blk], kFlagPrefix | ((excl + btot) & kValueMask));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  if (threadIdx.x < kFusedTiles) s_pre[threadIdx.x] = s_excl + (warp == 1 ? s_wtot[0] : 0ull) + incl - q;
  __syncthreads();
  // (3) offspring counts per particle (lane = particle, 8 tiles per warp) -> window fill
  const uint64_t* cl = cdf_local + static_cast<size_t>(b) * P;
  const int jw = blk * kScanTile + warp * (kScanTile / (kThreads / 32));
  uint64_t qv[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int j = jw + it * 32 + lane;
    qv[it] = j < P - 1 ? __ldg(cl + j) : 0ull;
  }
  const double inv = 1.0 / kNominalTotal, Pd = static_cast<double>(P);
  const double tscale = Pd * inv, invP = 1.0 / Pd;
  const bool pow2 = (P & (P - 1)) == 0;
  const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
  const double u_sys = s_usys;
  const double* U = (SCHEME == SSM_STRATIFIED && u) ? u + static_cast<size_t>(b) * P : nullptr;
  const auto count = [&](uint64_t C) -> int {
    const double Cd = static_cast<double>(C);
    if constexpr (SCHEME == SSM_SYSTEMATIC) {
      const double t = fma(Cd, tscale, -u_sys);
      const double e = ceil(t);
      const double d = e - t;  // in [0, 1), within 2^-53
      if (d > 0x1p-20 && d < 1.0 - 0x1p-20 && P <= (1 << 30)) return min(max(__double2int_rz(e), 0), P);
    }
    return offspring_bound<SCHEME>(Cd * inv, u_sys, U, k0, k1, step, P, invP, pow2);
  };
  const int tw = warp * kIt;  // the warp's first tile within the block
  int carry = 0;
  if (jw > 0 && jw < P) carry = count(s_pre[tw]);
  else if (jw >= P) carry = P;
  if (warp == 0 && lane == 0) sm.lo = carry;
  int cv[kIt], pv[kIt];
#pragma unroll
  for (int it = 0; it < kIt; ++it) {
    const int j = jw + it * 32 + lane;
    const int c = j < P - 1 ? count(s_pre[tw + it] + __double2ull_rn(s_sc[tw + it] * static_cast<double>(qv[it]))) : P;
    const int up = __shfl_up_sync(0xffffffffu, c, 1);
    pv[it] = lane == 0 ? carry : up;
    cv[it] = c;
    carry = __shfl_sync(0xffffffffu, c, 31);
  }
  fill_run_window(sm, b, P, jw, cv, pv, LocalStore{anc, P}, long_runs, long_count);
}

// ---------------------------------------------------------------------------
// Sorted multinomial via exponential spacings: with E_1..E_{P+1} iid Exp(1) and
// S_k = E_1 + ... + E_k, (S_1, ..., S_P) / S_{P+1} has the law of P sorted iid
// U(0,1) draws, so searchsorted(cum, U_(k)) is a multinomial sample with the
// ancestors already ascending.  Each 2048-output block rebuilds its U_(k) in
// shared memory (the block's spacing sums come from spacing_sums_kernel and a
// one-block prefix, all in a fixed summation order: deterministic), finds its
// first and last ancestor by binary search, and fills its outputs from the
// particles in between (count of U_(k) < cum_j per particle, run-start marks,
// max-scan).  Replaces P random-access searches of the unsorted draw.
// ---------------------------------------------------------------------------
// spacings 2m and 2m + 1 from one Philox block (words x,y and z,w)
__device__ __forceinline__ void spacing_pair(uint32_t k0, uint32_t k1, uint32_t m, uint32_t step, double& e0,
                                             double& e1) {
  const U4 r = philox4x32_10(U4{m, step, 0u, kPurposeSpacing}, k0, k1);
  e0 = -log(1.0 - u53(r.x, r.y));  // 1 - u in (0, 1], exact
  e1 = -log(1.0 - u53(r.z, r.w));
}

// inclusive prefix of the block's 2048 spacings (thread t: items 8t..8t+7), fixed order;
// returns the thread's 8 inclusive values and the block total (all threads)
__device__ __forceinline__ double spacing_block_scan(uint32_t k0, uint32_t k1, int step, int kbase, int n_valid,
                                                     double (&v)[kScanItems], double* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double run = 0.0;
  static_assert(kScanItems % 2 == 0 && kScanTile % 2 == 0, "spacing pairs");
#pragma unroll
  for (int i = 0; i < kScanItems; i += 2) {
    const int kl = threadIdx.x * kScanItems + i;  // even: the pair (kl, kl + 1) shares a block
    double e0 = 0.0, e1 = 0.0;
    if (kl < n_valid)
      spacing_pair(k0, k1, static_cast<uint32_t>((kbase + kl) >> 1), static_cast<uint32_t>(step), e0, e1);
    run += e0;
    v[i] = run;
    run += kl + 1 < n_valid ? e1 : 0.0;
    v[i + 1] = run;
  }
  double incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  double wex = 0.0, tot = 0.0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    if (w < warp) wex += s_warp[w];
    tot += s_warp[w];
  }
  const double base = wex + (incl - run);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) v[i] += base;
  __syncthreads();
  return tot;
}

// block totals of the P + 1 spacings (outputs k = 0..P; k = P is the extra E_{P+1})
__global__ void __launch_bounds__(kThreads)
spacing_sums_kernel(int P, const uint32_t* __restrict__ keys, int step, const ssm_filter_state* __restrict__ fs,
                    double* __restrict__ blk, double* __restrict__ spc) {
  __shared__ double s_warp[kThreads / 32];
  const int b = blockIdx.y;
  if (fs && !fs[b].resample_now) return;
  const int kbase = blockIdx.x * kScanTile;
  double v[kScanItems];
  const double tot = spacing_block_scan(keys[2 * b], keys[2 * b + 1], step, kbase, min(kScanTile, P + 1 - kbase), v, s_warp);
  if (threadIdx.x == 0) blk[static_cast<size_t>(b) * gridDim.x + blockIdx.x] = tot;
  // block-local inclusive prefixes for the merge pass (thread-contiguous, 4 x 16-byte stores)
  double2* dst = reinterpret_cast<double2*>(spc + static_cast<size_t>(b) * gridDim.x * kScanTile + kbase +
                                            threadIdx.x * kScanItems);
#pragma unroll
  for (int i = 0; i < kScanItems / 2; ++i) dst[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

// exclusive prefix of the block totals in place (fixed order), grand total -> tot[b]
__global__ void __launch_bounds__(1024)
spacing_prefix_kernel(int nblk, double* __restrict__ blk, double* __restrict__ tot,
                      const ssm_filter_state* __restrict__ fs) {
  __shared__ double wsum[32];
  const int b = blockIdx.x;
  if (fs && !fs[b].resample_now) return;
  double* bb = blk + static_cast<size_t>(b) * nblk;
  const int per = (nblk + 1023) / 1024;
  const int t0 = threadIdx.x * per, t1 = min(t0 + per, nblk);
  double local = 0.0;
  for (int t = t0; t < t1; ++t) local += bb[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  double wex = 0.0, all = 0.0;
  for (int w = 0; w < 32; ++w) {
    if (w < warp) wex += wsum[w];
    all += wsum[w];
  }
  double run = wex + incl - local;
  for (int t = t0; t < t1; ++t) {
    const double x = bb[t];
    bb[t] = run;
    run += x;
  }
  if (threadIdx.x == 0) tot[b] = all;
}

// CDF accessors for the sorted multinomial: cum_j = C_j / C_tot from an
// inclusive u64 array (scan of the log-weights) or from the fused kernel's
// tile records (C_j = tile prefix + round(scale_w * cdf_local_j), as the
// systematic offspring kernel; the last particle's C is the total: cum = 1)
// The sorted multinomial's CDF accessors scale by a precomputed 1 / total (its
// draws are device noise: consistency between its two sources is what matters);
// the trajectory pick keeps the division (CumTileRecs), which the host-draw
// parity runs compare against the reference.
struct CumFixedArr {
  const uint64_t* C;
  double inv;
  __device__ __forceinline__ double operator()(int j) const { return static_cast<double>(__ldg(C + j)) * inv; }
};
struct CumTileRecsMul {
  const uint64_t* cl;
  const double* sc;
  const uint64_t* tp;
  const uint64_t* bp;
  double inv;
  __device__ __forceinline__ double operator()(int j) const {
    const int tw = j >> 5;
    const uint64_t C = tp[tw] + bp[tw / kRecPerBlock] + __double2ull_rn(sc[tw] * static_cast<double>(__ldg(cl + j)));
    return static_cast<double>(C) * inv;
  }
};
struct CumTileRecs {
  const uint64_t* cl;
  const double* sc;
  const uint64_t* tp;
  const uint64_t* bp;
  double tot;
  __device__ __forceinline__ double operator()(int j) const {
    const int tw = j >> 5;
    const uint64_t C = tp[tw] + bp[tw / kRecPerBlock] + __double2ull_rn(sc[tw] * static_cast<double>(__ldg(cl + j)));
    return static_cast<double>(C) / tot;
  }
};

// searchsorted(cum, q, 'right') by one warp: 32 probes per round (5 rounds
// for 2^24 entries instead of 24 dependent loads); all lanes return the answer
template <typename Cum>
__device__ __forceinline__ int warp_search_right(const Cum& cum_at, int P, double q, int lane) {
  int lo = 0, hi = P;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int p = min(lo + (lane + 1) * step - 1, hi - 1);
    const unsigned m = __ballot_sync(0xffffffffu, cum_at(p) <= q);
    const int cnt = __popc(m);  // probes are ascending: the true ones are a prefix
    const int p_last = __shfl_sync(0xffffffffu, p, cnt > 0 ? cnt - 1 : 0);
    const int p_next = __shfl_sync(0xffffffffu, p, cnt < 32 ? cnt : 31);
    if (cnt > 0) lo = p_last + 1;
    if (cnt < 32) hi = p_next;
  }
  const int p = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, p < hi && cum_at(p) <= q);
  return lo + __popc(m);
}

// warp_search_right starting from a window of 32 x 1024 entries around `guess`
// (output k's ancestor is near k unless the weights are very uneven): one round
// places q inside the window -- or outside it, and the full search runs --, then
// two rounds finish instead of five.  Same answer as warp_search_right.
template <typename Cum>
__device__ __forceinline__ int warp_search_right_near(const Cum& cum_at, int P, double q, int lane, int guess) {
  constexpr int kW = 32 * 1024;
  if (P > 4 * kW) {
    const int wlo = max(0, min(guess - kW / 2, P - kW));
    const int step = kW / 32;
    const int p = wlo + (lane + 1) * step - 1;
    const bool below_ok = wlo == 0 || cum_at(wlo - 1) <= q;  // every lane: the same probe (cached)
    const unsigned m = __ballot_sync(0xffffffffu, cum_at(p) <= q);
    const int cnt = __popc(m);
    if (below_ok && cnt < 32) {  // answer in [wlo, wlo + kW)
      int lo = cnt > 0 ? wlo + cnt * step : wlo;
      int hi = wlo + (cnt + 1) * step - 1;
      while (hi - lo > 32) {
        const int st = (hi - lo + 31) / 32;
        const int pp = min(lo + (lane + 1) * st - 1, hi - 1);
        const unsigned mm = __ballot_sync(0xffffffffu, cum_at(pp) <= q);
        const int c2 = __popc(mm);
        const int p_last = __shfl_sync(0xffffffffu, pp, c2 > 0 ? c2 - 1 : 0);
        const int p_next = __shfl_sync(0xffffffffu, pp, c2 < 32 ? c2 : 31);
        if (c2 > 0) lo = p_last + 1;
        if (c2 < 32) hi = p_next;
      }
      const int pf = lo + lane;
      const unsigned mf = __ballot_sync(0xffffffffu, pf < hi && cum_at(pf) <= q);
      return lo + __popc(mf);
    }
  }
  return warp_search_right(cum_at, P, q, lane);
}

// SRC 0: cum = inclusive u64 array `C` ([B][P]); SRC 1: tile records (cdf_local,
// scale [B][nt], tile prefixes [B][nt] then block prefixes [B][nblk], totals)
template <int SRC>
__global__ void __launch_bounds__(kThreads)
spacing_merge_kernel(int P, const uint64_t* __restrict__ C, const uint64_t* __restrict__ cdf_local,
                     const double* __restrict__ scale, const uint64_t* __restrict__ pref,
                     const uint64_t* __restrict__ totals, const double* __restrict__ spc,
                     const double* __restrict__ blk, const double* __restrict__ tot,
                     const ssm_filter_state* __restrict__ fs, int32_t* __restrict__ anc) {
  __shared__ double sU[kScanTile];
  __shared__ __align__(16) int32_t sOut[kScanTile + kScanTile / 32];
  __shared__ double s_warp[kThreads / 32];
  __shared__ int s_wmax[kThreads / 32];
  __shared__ int s_j[2];
  __shared__ int s_carry[kThreads / 32];
  __shared__ int s_prev;
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* ab = anc + static_cast<size_t>(b) * P;
  const int k0 = blockIdx.x * kScanTile, n_out = min(kScanTile, P - k0);
  if (fs && !fs[b].resample_now) {  // ESS gate held: identity ancestors
    for (int k = threadIdx.x; k < n_out; k += kThreads) ab[k0 + k] = k0 + k;
    return;
  }
  const int nsb = gridDim.x + (P % kScanTile == 0 ? 1 : 0);  // spacing blocks cover P + 1 outputs
  const double off = blk[static_cast<size_t>(b) * nsb + blockIdx.x];
  const double inv = 1.0 / tot[b];
  const double* spb = spc + static_cast<size_t>(b) * nsb * kScanTile + k0;
  (void)s_warp;
  const size_t coff = static_cast<size_t>(b) * P;
  using Cum = typename std::conditional<SRC == 0, CumFixedArr, CumTileRecsMul>::type;
  Cum cum_at;
  if constexpr (SRC == 0) {
    cum_at = CumFixedArr{C + coff, 1.0 / static_cast<double>(C[coff + P - 1])};
  } else {
    const int nt = (P + 31) >> 5;
    const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
    cum_at = CumTileRecsMul{cdf_local + coff, scale + static_cast<size_t>(b) * nt, pref + static_cast<size_t>(b) * nt,
                         pref + B_total_tiles_offset(nt, gridDim.y) + static_cast<size_t>(b) * nblk,
                         1.0 / static_cast<double>(totals[b])};
  }
  // first / last ancestor: searchsorted(cum, U, 'right'), clipped -- warps 0 and 1
  // search (their U from the spacing prefixes directly) while warps 2-7 build the
  // block's U_(k0+k) = (S_{k0} + local inclusive sum) / S_{P+1} and clear the marks
  if (warp < 2) {  // warp 0: first output, warp 1: last output
    const int kq = warp == 0 ? 0 : n_out - 1;
    const int j = warp_search_right_near(cum_at, P, (off + spb[kq]) * inv, lane, k0 + kq);
    if (lane == 0) s_j[warp] = j < P ? j : P - 1;
  } else {
    const int t = threadIdx.x - 64;
    constexpr int kBuilders = kThreads - 64;
    const double2* src = reinterpret_cast<const double2*>(spb);
    for (int e = t; e < kScanTile / 2; e += kBuilders) {
      const double2 v = src[e];
      sU[2 * e] = (off + v.x) * inv;
      sU[2 * e + 1] = (off + v.y) * inv;
    }
    for (int e = t; e < (kScanTile + kScanTile / 32) / 4; e += kBuilders)
      reinterpret_cast<int4*>(sOut)[e] = make_int4(-1, -1, -1, -1);
  }
  __syncthreads();
  const int jlo = s_j[0], jhi = s_j[1];
  if (jhi - jlo > 8 * kScanTile) {
    // degenerate weights: the tile's outputs span a long stretch of (near-)zero-weight
    // particles; one binary search per output instead of a walk over every particle.
    // searchsorted(cum, U, 'right') within [jlo, jhi] (jhi already clipped to P - 1)
    for (int e = threadIdx.x; e < n_out; e += kThreads) {
      const double u = sU[e];
      int lo = jlo, hi = jhi;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cum_at(mid) <= u)
          lo = mid + 1;
        else
          hi = mid;
      }
      ab[k0 + e] = lo;
    }
    return;
  }
  // local count of U < cum_j (the last particle takes every remaining output: clip rule)
  auto cnt_lt = [&](int j) -> int {
    if (j < jlo) return 0;
    if (j >= P - 1 || j >= jhi) return n_out;
    const double c = cum_at(j);
    int lo = 0, hi = n_out;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (sU[mid] < c)
        lo = mid + 1;
      else
        hi = mid;
    }
    return lo;
  };
  // the same count continued from particle j - 1's (cum is non-decreasing, so every
  // U below c_{j-1} is below cum_j): a short linear walk, then a binary search
  auto cnt_from = [&](int j, int c) -> int {
    if (j >= P - 1 || j >= jhi) return n_out;
    const double cj = cum_at(j);
    int lim = min(c + 16, n_out);
    while (c < lim && sU[c] < cj) ++c;
    if (c < lim || c == n_out) return c;
    int hi = n_out;
    while (c < hi) {
      const int mid = (c + hi) >> 1;
      if (sU[mid] < cj)
        c = mid + 1;
      else
        hi = mid;
    }
    return c;
  };
  // chunks of 2048 particles, 8 consecutive per thread: one binary search for the
  // thread's first particle, the next seven continue from it (merge walk)
  for (int j0 = jlo; j0 <= jhi; j0 += kScanTile) {
    const int jt = j0 + threadIdx.x * kScanItems;
    int cv[kScanItems];
    int c = jt <= jhi ? cnt_lt(jt) : n_out;
    cv[0] = c;
#pragma unroll
    for (int i = 1; i < kScanItems; ++i) {
      c = jt + i <= jhi ? cnt_from(jt + i, c) : n_out;
      cv[i] = c;
    }
    const int up = __shfl_up_sync(0xffffffffu, c, 1);
    if (lane == 31) s_carry[warp] = c;
    __syncthreads();
    int a = lane > 0 ? up : (warp > 0 ? s_carry[warp - 1] : (j0 == jlo ? cnt_lt(jlo - 1) : s_prev));
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (jt + i <= jhi && cv[i] > a) sOut[a + (a >> 5)] = jt + i;
      a = cv[i];
    }
    __syncthreads();
    if (threadIdx.x == kThreads - 1) s_prev = c;
  }
  __syncthreads();
  // inclusive max-scan of the marks (all outputs have an owner: position 0 is jlo's)
  constexpr int kPer = kScanTile / kThreads;  // 8
  int vv[kPer];
  int run = -1;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = threadIdx.x * kPer + i;
    run = max(run, sOut[e + (e >> 5)]);
    vv[i] = run;
  }
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = max(incl, y);
  }
  int cin = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) cin = -1;
  if (lane == 31) s_wmax[warp] = incl;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w)
    if (w < warp) cin = max(cin, s_wmax[w]);
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = threadIdx.x * kPer + i;
    sOut[e + (e >> 5)] = max(cin, vv[i]);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n_out; e += kThreads) ab[k0 + e] = sOut[e + (e >> 5)];
}

// anc_k = #{j : c_j <= k}, clipped to P_in - 1, from the precomputed partition.
// Balanced without searches: the block's particles [i0, i1] each mark the first
// output of their offspring run inside [kb0, kb1); an inclusive max-scan of
// the marks then assigns every output its owner.  Work per thread: kScanItems
// particles + kScanItems outputs.
__global__ void __launch_bounds__(kThreads)
expand_kernel(int P_in, int P_out, const int32_t* __restrict__ cnt, const int32_t* __restrict__ split,
              int ndiag, const ssm_filter_state* __restrict__ fs, int32_t* __restrict__ anc) {
  __shared__ int32_t sMark[kDiag + kDiag / 8];  // padded: e -> e + e/8 (conflict-free sequential scan)
  __shared__ int32_t warp_max[kThreads / 32];
  const int b = blockIdx.y, t = blockIdx.x;
  int32_t* ab = anc + static_cast<size_t>(b) * P_out;
  const int total = P_in + P_out;
  const int D0 = t * kDiag, D1 = min(D0 + kDiag, total);
  if (fs && !fs[b].resample_now) {
    // identity ancestors (ESS gate held, particle.py:99-100); block t covers outputs [D0/2, D1/2)
    const int ka = D0 >> 1, kb = t == ndiag - 1 ? P_out : min(D1 >> 1, P_out);
    for (int k = ka + threadIdx.x; k < kb; k += kThreads) ab[k] = k;
    return;
  }
  const int32_t* sp = split + static_cast<size_t>(b) * (ndiag + 1);
  const int32_t* cb = cnt + static_cast<size_t>(b) * P_in;
  const int i0 = sp[t], i1 = sp[t + 1];
  const int kb0 = D0 - i0, kb1 = D1 - i1;
  const int nb = kb1 - kb0;  // outputs of this block (<= kDiag)
  if (nb <= 0) return;
  for (int q = threadIdx.x; q < nb; q += kThreads) sMark[q + (q >> 3)] = -1;
  __syncthreads();
  // particles i0 .. min(i1, P_in - 1): mark run starts clamped into the block
  const int jlast = i1 < P_in ? i1 : P_in - 1;
  for (int j = i0 + threadIdx.x; j <= jlast; j += kThreads) {
    const int c_lo = j > 0 ? __ldg(cb + j - 1) : 0;
    const int c_hi = __ldg(cb + j);
    const int st = c_lo > kb0 ? c_lo : kb0;
    const int en = c_hi < kb1 ? c_hi : kb1;
    if (st < en) sMark[(st - kb0) + ((st - kb0) >> 3)] = j;
  }
  // outputs past the last particle's run belong to P_in -> clipped to P_in - 1
  if (threadIdx.x == 0 && i1 >= P_in) {
    const int c_last = __ldg(cb + P_in - 1);
    const int st = c_last > kb0 ? c_last : kb0;
    const int q = st - kb0;
    if (st < kb1 && sMark[q + (q >> 3)] < 0) sMark[q + (q >> 3)] = P_in - 1;
  }
  __syncthreads();
  // block inclusive max-scan over the marks (kScanItems consecutive per thread)
  int v[kScanItems];
  int run = -1;
  const int e0 = threadIdx.x * kScanItems;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = e0 + i;
    const int m = e < nb ? sMark[e + (e >> 3)] : -1;
    run = m > run ? m : run;
    v[i] = run;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = y > incl ? y : incl;
  }
  if (lane == 31) warp_max[warp] = incl;
  int excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = -1;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w)
    if (w < warp) excl = warp_max[w] > excl ? warp_max[w] : excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int e = e0 + i;
    if (e < nb) {
      const int a_idx = v[i] > excl ? v[i] : excl;
      sMark[e + (e >> 3)] = a_idx < P_in ? a_idx : P_in - 1;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nb; q += kThreads) ab[kb0 + q] = sMark[q + (q >> 3)];
}


template <int KIND>
__global__ void __launch_bounds__(kThreads)
binary_search_kernel(int P_in, int P_out, const void* __restrict__ cum, const double* __restrict__ u,
                     const uint32_t* __restrict__ keys, int step,
                     const ssm_filter_state* __restrict__ fs, int32_t* __restrict__ anc) {
  const int b = blockIdx.y;
  int32_t* ancb = anc + static_cast<size_t>(b) * P_out;
  const bool skip = fs && !fs[b].resample_now;
  const size_t coff = static_cast<size_t>(b) * P_in;
  const double tot = skip ? 1.0 : cum_total<KIND>(cum, coff, P_in);
  const double* ub = u ? u + static_cast<size_t>(b) * P_out : nullptr;
  const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
  for (int k = blockIdx.x * kThreads + threadIdx.x; k < P_out; k += gridDim.x * kThreads) {
    if (skip) {
      ancb[k] = k;
      continue;
    }
    const double q = ub ? ub[k] : device_uniform(k0, k1, k, step, kPurposeResample);
    int lo = 0, hi = P_in;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cum_at<KIND>(cum, coff, tot, mid) <= q)
        lo = mid + 1;
      else
        hi = mid;
    }
    ancb[k] = lo < P_in ? lo : P_in - 1;
  }
}

// ===========================================================================
// K6 gather, K8 trace, K9 block gather
// ===========================================================================

template <typename T>
__global__ void __launch_bounds__(kThreads)
gather_kernel(int nx, int P, const T* __restrict__ x, const int32_t* __restrict__ anc,
              T* __restrict__ out) {
  const int b = blockIdx.y;
  const size_t base = static_cast<size_t>(b) * nx * P;
  const int32_t* ab = anc + static_cast<size_t>(b) * P;
  for (int k = blockIdx.x * kThreads + threadIdx.x; k < P; k += gridDim.x * kThreads) {
    const int src = ab[k];
    for (int n = 0; n < nx; ++n) out[base + static_cast<size_t>(n) * P + k] = x[base + static_cast<size_t>(n) * P + src];
  }
}

// out[n][k] = x[n][idx[k]]: x rows of length in_stride, out rows of length n_out
template <typename T>
__global__ void __launch_bounds__(kThreads)
gather_cols_kernel(int nx, int n_out, int in_stride, const T* __restrict__ x, const int32_t* __restrict__ idx,
                   T* __restrict__ out) {
  for (int k = blockIdx.x * kThreads + threadIdx.x; k < n_out; k += gridDim.x * kThreads) {
    const int src = idx[k];
    for (int n = 0; n < nx; ++n)
      out[static_cast<size_t>(n) * n_out + k] = x[static_cast<size_t>(n) * in_stride + src];
  }
}

// One block per filter.  Thread 0 walks the ancestry chain j_S -> j_0 (the
// only serial part: one dependent load per step; the per-step pointer loads
// are independent and run ahead) and parks j_i in out[i][0]; then the block
// gathers the (S+1) x nx states in parallel.
template <typename T>
__global__ void __launch_bounds__(128)
trace_kernel(int B, int S, int nx, int P, const void* const* __restrict__ xs,
             const int32_t* const* __restrict__ ancs, const int32_t* __restrict__ j_final,
             double* __restrict__ out) {
  const int b = blockIdx.x;
  const size_t row = static_cast<size_t>(b) * (S + 1);
  if (threadIdx.x == 0) {
    int j = j_final[b];
    out[(row + S) * nx] = static_cast<double>(j);
#pragma unroll 8
    for (int i = S; i > 0; --i) {
      const int32_t* a = ancs[row + i];
      if (a) j = __ldcg(a + j);
      out[(row + i - 1) * nx] = static_cast<double>(j);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= S; i += blockDim.x) {
    const int j = static_cast<int>(out[(row + i) * nx]);
    const T* xi = static_cast<const T*>(xs[row + i]);
    for (int n = 0; n < nx; ++n)
      out[(row + i) * nx + n] = static_cast<double>(xi[static_cast<size_t>(n) * P + j]);
  }
}

__global__ void block_gather_kernel(size_t words, const uint4* __restrict__ src,
                                    const int32_t* __restrict__ idx, uint4* __restrict__ dst) {
  const int jb = blockIdx.y;
  const uint4* s = src + static_cast<size_t>(idx[jb]) * words;
  uint4* d = dst + static_cast<size_t>(jb) * words;
  for (size_t w = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<size_t>(gridDim.x) * blockDim.x)
    d[w] = s[w];
}

// ===========================================================================
// K3 standalone LSE + ESS
// ===========================================================================
constexpr int kMaxLseBlocks = 1024;

template <typename T>
__global__ void __launch_bounds__(kThreads)
lse_kernel(int P, const T* __restrict__ a, Lse* parts, uint32_t* done, double* out_lse,
           double* out_ess) {
  const int b = blockIdx.y;
  const T* ab = a + static_cast<size_t>(b) * P;
  Lse st = lse_empty();
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads)
    lse_push(st, static_cast<double>(ab[p]));
  __shared__ Lse red[kThreads / 32];
  __shared__ bool last;
  const Lse r = lse_block_reduce<kThreads>(st, red);
  Lse* pb = parts + static_cast<size_t>(b) * kMaxLseBlocks;
  if (threadIdx.x == 0) {
    pb[blockIdx.x] = r;
    __threadfence();
    last = atomicAdd(&done[b], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  Lse acc = lse_empty();
  for (int i = threadIdx.x; i < static_cast<int>(gridDim.x); i += kThreads) {
    const Lse q{__ldcg(&pb[i].m), __ldcg(&pb[i].c), __ldcg(&pb[i].t), __ldcg(&pb[i].s2)};
    acc = lse_combine(acc, q);
  }
  acc = lse_block_reduce<kThreads>(acc, red);
  if (threadIdx.x == 0) {
    out_lse[b] = lse_value(acc);
    if (out_ess) out_ess[b] = lse_ess(acc);
    done[b] = 0;
  }
}

static inline int grid_for(int n, int per, int cap) {
  int g = (n + per - 1) / per;
  if (g < 1) g = 1;
  return g < cap ? g : cap;
}

}  // namespace ssm

using namespace ssm;

// ------------------------------- C ABI --------------------------------------

static thread_local cudaError_t g_last_err = cudaSuccess;
extern "C" void ssm_set_last_error(cudaError_t e) { g_last_err = e; }
extern "C" const char* ssm_last_cuda_error(void) { return cudaGetErrorString(g_last_err); }
extern "C" const char* ssm_version(void) { return "ssm_b200 0.1.0 (sm_100a)"; }
extern "C" const char* ssm_status_string(int s) {
  switch (s) {
    case SSM_OK: return "ok";
    case SSM_ERR_INVALID_ARG: return "invalid argument";
    case SSM_ERR_CUDA: return "CUDA error";
    case SSM_ERR_UNSUPPORTED: return "unsupported";
    default: return "unknown status";
  }
}
extern "C" int ssm_sm_count(int device, int* out) {
  if (!out) return SSM_ERR_INVALID_ARG;
  cudaError_t e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

extern "C" size_t ssm_scan_workspace_bytes(int B, int P) { return scan_ws_bytes(B, P); }

extern "C" int ssm_weights_scan(int B, int P, int dtype, const void* a, int is_log,
                                const double* shift, const ssm_filter_state* fs, uint64_t* C,
                                uint32_t* flags, void* workspace, void* stream) {
  if (B <= 0 || P <= 0 || !a || !C || !workspace) return SSM_ERR_INVALID_ARG;
  if (is_log && !shift && !fs) return SSM_ERR_INVALID_ARG;
  if (!is_log && (dtype != SSM_F64 || !flags)) return SSM_ERR_INVALID_ARG;
  if (static_cast<long long>(B) * scan_tiles(P) > 0x7fffffffLL) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ScanWs ws = scan_ws(workspace, B, P);
  cudaError_t e = cudaMemsetAsync(workspace, 0, scan_ws_zero_bytes(B, P), s);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  const int tiles = scan_tiles(P);
  if (!is_log) {
    const dim3 g(grid_for(P, kThreads, kRawBlocks), B);
    raw_total_kernel<<<g, kThreads, 0, s>>>(P, static_cast<const double*>(a), ws.partial, ws.done,
                                            ws.scale, flags);
    SSM_CHECK_LAUNCH();
    scan_kernel<double, false><<<B * tiles, kThreads, 0, s>>>(B, P, static_cast<const double*>(a),
                                                             nullptr, fs, C, ws, flags);
  } else if (dtype == SSM_F64) {
    scan_kernel<double, true><<<B * tiles, kThreads, 0, s>>>(B, P, static_cast<const double*>(a),
                                                            shift, fs, C, ws, flags);
  } else if (dtype == SSM_F32) {
    scan_kernel<float, true><<<B * tiles, kThreads, 0, s>>>(B, P, static_cast<const float*>(a),
                                                           shift, fs, C, ws, flags);
  } else {
    return SSM_ERR_INVALID_ARG;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_fixed_to_cum(int B, int P, const uint64_t* C, double* cum, void* stream) {
  if (B <= 0 || P <= 0 || !C || !cum) return SSM_ERR_INVALID_ARG;
  fixed_to_cum_kernel<<<dim3(grid_for(P, kThreads, 4096), B), kThreads, 0,
                        static_cast<cudaStream_t>(stream)>>>(P, C, cum);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// workspace: [tile sums B*tiles u64][totals B u64][cnt B*P_in i32][split B*(ndiag+1) i32]
//            [+ look-back scan workspace for multinomial from log-weights]
static inline int ndiag_of(int P_in, int P_out) {
  return static_cast<int>((static_cast<long long>(P_in) + P_out + kDiag - 1) / kDiag);
}

struct SearchWs {
  uint64_t* sums;
  uint64_t* totals;
  int32_t* cnt;
  int32_t* split;
  void* scan;
  uint64_t* C;
  double* spc;  // sorted multinomial: block-local inclusive spacing sums, [B][nsb * 2048]
  uint64_t* lb;  // fused tile resample: double-buffered look-back status + long-run counts (fused_ws)
  uint64_t* lt_cdf;       // ssm_resample_from_logw's tile path: cdf_local [B][P_in]
  ssm_tile_rec* lt_rec;   // ... its warp-tile records [B][nt]
  ssm_filter_state* lt_fs;  // ... and per-filter states {incr = shift, resample_now}
};

static inline size_t search_ws_layout(int B, int P_in, int P_out, void* base, SearchWs* w) {
  const int tiles = scan_tiles(P_in);
  const int nd = ndiag_of(P_in, P_out);
  size_t off = 0;
  char* p = static_cast<char*>(base);
  auto take = [&](size_t bytes) {
    char* r = p ? p + off : nullptr;
    off += align256(bytes);
    return r;
  };
  SearchWs tmp;
  // regions that depend on P_out (the partition) go last, so the offsets of
  // the others are the same for every P_out (the sharded phases rely on it)
  // sums: tile sums, or the sorted multinomial's (P + 1)-spacing block sums (tiles + 1 per filter)
  tmp.sums = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * static_cast<size_t>(B) * (tiles + 1)));
  // totals, long-run counts, spacing totals, then OffspringConsts (4 words) per filter
  tmp.totals = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 7 * static_cast<size_t>(B)));
  // C doubles as the tile path's [scale | in-block prefix | block prefix] (2 nt + nblk per filter)
  const size_t nt = (static_cast<size_t>(P_in) + 31) / 32;
  const size_t tile_words = 2 * nt + (nt + kRecPerBlock - 1) / kRecPerBlock;
  const size_t c_words = static_cast<size_t>(P_in) > tile_words ? static_cast<size_t>(P_in) : tile_words;
  tmp.C = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * static_cast<size_t>(B) * c_words));
  tmp.spc = reinterpret_cast<double*>(
      take(sizeof(double) * static_cast<size_t>(B) * ((P_in + 1 + kScanTile - 1) / kScanTile) * kScanTile));
  tmp.scan = take(scan_ws_bytes(B, P_in));
  tmp.lb = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * fused_ws_words(B, P_in)));
  // cnt doubles as the long-run list of the direct ancestor writer (int4 per run, P_out/32 + ... per filter);
  // it and split depend on P_out, so they come last (the sharded phases share the other offsets)
  const size_t cnt_bytes = sizeof(int32_t) * static_cast<size_t>(B) * P_in;
  const size_t runs_bytes = sizeof(int4) * static_cast<size_t>(B) * long_runs_cap(P_in, P_out);
  tmp.cnt = reinterpret_cast<int32_t*>(take(cnt_bytes > runs_bytes ? cnt_bytes : runs_bytes));
  tmp.split = reinterpret_cast<int32_t*>(take(sizeof(int32_t) * static_cast<size_t>(B) * (nd + 1)));
  tmp.lt_cdf = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * static_cast<size_t>(B) * P_in));
  tmp.lt_rec = reinterpret_cast<ssm_tile_rec*>(take(sizeof(ssm_tile_rec) * static_cast<size_t>(B) * nt));
  tmp.lt_fs = reinterpret_cast<ssm_filter_state*>(take(sizeof(ssm_filter_state) * static_cast<size_t>(B)));
  if (w) *w = tmp;
  return off;
}

template <int SRC, typename T>
static void launch_offspring_expand(int scheme, int B, int P_in, int P_out, const void* src,
                                    const double* shift, const SearchWs& w, const double* u,
                                    const uint32_t* keys, int step, const ssm_filter_state* fs,
                                    int32_t* anc, cudaStream_t s) {
  const int tiles = scan_tiles(P_in);
  const int nd = ndiag_of(P_in, P_out);
  const dim3 g(tiles, B);
  if (scheme == SSM_SYSTEMATIC)
    offspring_kernel<SSM_SYSTEMATIC, SRC, T><<<g, kThreads, 0, s>>>(
        P_in, P_out, src, shift, w.sums, w.totals, u, keys, step, fs, w.cnt, w.split, nd);
  else
    offspring_kernel<SSM_STRATIFIED, SRC, T><<<g, kThreads, 0, s>>>(
        P_in, P_out, src, shift, w.sums, w.totals, u, keys, step, fs, w.cnt, w.split, nd);
  expand_kernel<<<dim3(nd, B), kThreads, 0, s>>>(P_in, P_out, w.cnt, w.split, nd, fs, anc);
}

extern "C" size_t ssm_search_workspace_bytes(int B, int P_in, int P_out) {
  if (B <= 0 || P_in <= 0 || P_out <= 0) return 0;
  return search_ws_layout(B, P_in, P_out, nullptr, nullptr);
}

extern "C" int ssm_resample_search(int B, int P_in, int P_out, int scheme, int cum_kind,
                                   const void* cum, const double* u, const uint32_t* keys, int step,
                                   const ssm_filter_state* fs, int32_t* anc, void* workspace,
                                   void* stream) {
  if (B <= 0 || B > 65535 || P_in <= 0 || P_out <= 0 || !cum || !anc) return SSM_ERR_INVALID_ARG;
  if (!u && !keys) return SSM_ERR_INVALID_ARG;
  if (fs && P_in != P_out) return SSM_ERR_INVALID_ARG;
  if (static_cast<long long>(P_in) + P_out > 0x7fffffffLL) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (scheme == SSM_MULTINOMIAL) {
    const dim3 g(grid_for(P_out, kThreads, 65535), B);
    if (cum_kind == 0)
      binary_search_kernel<0><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
    else
      binary_search_kernel<1><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
  } else if (scheme == SSM_STRATIFIED || scheme == SSM_SYSTEMATIC) {
    if (!workspace) return SSM_ERR_INVALID_ARG;
    SearchWs w;
    search_ws_layout(B, P_in, P_out, workspace, &w);
    if (cum_kind == 0)
      launch_offspring_expand<kCumDouble, double>(scheme, B, P_in, P_out, cum, nullptr, w, u, keys,
                                                  step, fs, anc, s);
    else
      launch_offspring_expand<kCumFixed, double>(scheme, B, P_in, P_out, cum, nullptr, w, u, keys,
                                                 step, fs, anc, s);
  } else {
    return SSM_ERR_INVALID_ARG;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_resample_from_tiles(int B, int P, int scheme, const void* cdf_local,
                                       const void* tile_rec, const ssm_filter_state* fs,
                                       const double* u, const uint32_t* keys, int step, int32_t* anc,
                                       void* workspace, void* stream) {
  return ssm_resample_tiles_step(B, P, scheme, cdf_local, tile_rec, fs, u, keys, step, anc, workspace, 0, 1,
                                 stream);
}

extern "C" int ssm_resample_tiles_step(int B, int P, int scheme, const void* cdf_local, const void* tile_rec,
                                       const ssm_filter_state* fs, const double* u, const uint32_t* keys, int step,
                                       int32_t* anc, void* workspace, int parity, int zero_state, void* stream) {
  if (B <= 0 || B > 65535 || P <= 0 || !cdf_local || !tile_rec || !fs || !anc || !workspace)
    return SSM_ERR_INVALID_ARG;
  if (!u && !keys) return SSM_ERR_INVALID_ARG;
  if (scheme != SSM_SYSTEMATIC && scheme != SSM_STRATIFIED && scheme != SSM_MULTINOMIAL_SORTED)
    return SSM_ERR_INVALID_ARG;
  if (scheme == SSM_MULTINOMIAL_SORTED && (u || !keys)) return SSM_ERR_INVALID_ARG;
  if (parity != 0 && parity != 1) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SearchWs w;
  search_ws_layout(B, P, P, workspace, &w);
#ifndef SSM_RESAMPLE_FUSED
#define SSM_RESAMPLE_FUSED 0  // measured slower: 0.176 vs 0.103 ms per 2^24 resample (profiles/r2_ab.txt)
#endif
  if (SSM_RESAMPLE_FUSED && scheme != SSM_MULTINOMIAL_SORTED) {  // one fused kernel + long-run fill
    if (zero_state) {
      const cudaError_t e = cudaMemsetAsync(w.lb, 0, sizeof(uint64_t) * fused_ws_words(B, P), s);
      if (e != cudaSuccess) {
        ssm_set_last_error(e);
        return SSM_ERR_CUDA;
      }
    }
    const FusedWs fw = fused_ws(w.lb, B, P);
    const dim3 g(scan_tiles(P), B);
    const auto* cl = static_cast<const uint64_t*>(cdf_local);
    const auto* rec = static_cast<const ssm_tile_rec*>(tile_rec);
    int4* long_runs = reinterpret_cast<int4*>(w.cnt);
    if (scheme == SSM_SYSTEMATIC)
      launch_pdl(resample_fused_kernel<SSM_SYSTEMATIC>, g, dim3(kThreads), s, P, cl, rec, fs, u, keys, step, anc,
                 long_runs, fw, parity);
    else
      launch_pdl(resample_fused_kernel<SSM_STRATIFIED>, g, dim3(kThreads), s, P, cl, rec, fs, u, keys, step, anc,
                 long_runs, fw, parity);
    const int gx = std::max(1, std::min(1184 / B, P / kRunChunk + 1));
    launch_pdl(long_runs_kernel<LocalStore>, dim3(gx, B), dim3(kThreads), s, P, P, static_cast<const int4*>(long_runs),
               static_cast<const uint32_t*>(fw.long_count + static_cast<size_t>(parity) * B), fs, LocalStore{anc, P});
    SSM_CHECK_LAUNCH();
    return SSM_OK;
  }
  const int nt = (P + 31) / 32;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  // reuse w.C (B*P u64): [scale B*nt doubles][in-block prefixes B*nt][block prefixes B*nblk]
  double* scale = reinterpret_cast<double*>(w.C);
  uint64_t* pref = reinterpret_cast<uint64_t*>(w.C) + static_cast<size_t>(B) * nt;
  uint64_t* blk = pref + B_total_tiles_offset(nt, B);
  // the offspring kernel writes the ancestors itself; long runs of degenerate
  // blocks go to a list (w.cnt region reused, count zeroed by tile_scale)
  // filled by long_runs_kernel.  All four are programmatic dependent launches.
  uint32_t* long_count = reinterpret_cast<uint32_t*>(w.totals) + 2 * static_cast<size_t>(B);  // after totals
  int4* long_runs = reinterpret_cast<int4*>(w.cnt);
  // per-filter offspring constants after the totals / long-run counts / spacing totals
  OffspringConsts* oc = reinterpret_cast<OffspringConsts*>(w.totals + 3 * static_cast<size_t>(B));
  // tile scale + in-block prefix, and (last block per filter) the block prefix and constants
  launch_pdl(tile_scale_kernel, dim3(nblk, B), dim3(kThreads), s, nt, static_cast<const ssm_tile_rec*>(tile_rec), fs,
             scale, pref, blk, long_count, 1, const_cast<ssm_filter_state*>(fs), w.totals, oc, P, u, keys, step);
  const dim3 g(scan_tiles(P), B);
  if (scheme == SSM_MULTINOMIAL_SORTED) {  // spacing sums in w.sums (doubles), totals after the u64 totals
    const int nsb = (P + 1 + kScanTile - 1) / kScanTile;
    double* blkE = reinterpret_cast<double*>(w.sums);
    double* totE = reinterpret_cast<double*>(w.totals) + 2 * static_cast<size_t>(B);  // free slots
    spacing_sums_kernel<<<dim3(nsb, B), kThreads, 0, s>>>(P, keys, step, fs, blkE, w.spc);
    spacing_prefix_kernel<<<B, 1024, 0, s>>>(nsb, blkE, totE, fs);
    spacing_merge_kernel<1><<<g, kThreads, 0, s>>>(P, nullptr, static_cast<const uint64_t*>(cdf_local), scale, pref,
                                                   w.totals, w.spc, blkE, totE, fs, anc);
    SSM_CHECK_LAUNCH();
    return SSM_OK;
  }
  const uint64_t* cl = static_cast<const uint64_t*>(cdf_local);
  if (scheme == SSM_SYSTEMATIC)
    launch_pdl(offspring_tiles_kernel<SSM_SYSTEMATIC>, g, dim3(kThreads), s, P, cl, scale, pref, w.totals, u, keys,
               step, fs, LocalStore{anc, P}, long_runs, long_count, static_cast<const OffspringConsts*>(oc),
               ShardSpan{nullptr, P, 0});
  else
    launch_pdl(offspring_tiles_kernel<SSM_STRATIFIED>, g, dim3(kThreads), s, P, cl, scale, pref, w.totals, u, keys,
               step, fs, LocalStore{anc, P}, long_runs, long_count, static_cast<const OffspringConsts*>(oc),
               ShardSpan{nullptr, P, 0});
  const int gx = std::max(1, std::min(1184 / B, P / kRunChunk + 1));
  launch_pdl(long_runs_kernel<LocalStore>, dim3(gx, B), dim3(kThreads), s, P, P, static_cast<const int4*>(long_runs),
             static_cast<const uint32_t*>(long_count), fs, LocalStore{anc, P});
  (void)expand_kernel;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// ---------------------------------------------------------------------------
// Sharded single filter (config 5): the three resampling phases around the
// host-side collectives.
// ---------------------------------------------------------------------------

// Per-rank constants of the sharded resample from the all-gathered rank totals:
// this rank's global fixed-point offset (sum of the lower ranks' totals, rank
// order: exact integers, the same on every rank), the offspring constants on
// the global total, and a zeroed long-run list.
__global__ void shard_consts_kernel(int W, int rank, int P_global, const uint64_t* __restrict__ totals_all,
                                    const double* __restrict__ u, const uint32_t* __restrict__ keys, int step,
                                    uint64_t* __restrict__ g_off, OffspringConsts* __restrict__ oc,
                                    uint32_t* __restrict__ long_count) {
  if (threadIdx.x != 0) return;
  uint64_t off = 0, tot = 0;
  for (int d = 0; d < W; ++d) {
    if (d < rank) off += totals_all[d];
    tot += totals_all[d];
  }
  g_off[0] = off;
  const double inv = 1.0 / static_cast<double>(tot), Pd = static_cast<double>(P_global);
  const double us = u ? u[0] : (keys ? device_uniform(keys[0], keys[1], 0u, step, kPurposeSystematic) : 0.0);
  oc[0] = OffspringConsts{inv, Pd * inv, us, 1.0 / Pd};
  long_count[0] = 0u;
}

// Trajectory of the sharded filter (particle.py:137-149): one thread walks the
// ancestry through every rank's peer-mapped history -- x_tab[r] / anc_tab[r]
// are rank r's position / ancestor arenas ([S+1][nx][P_loc], [S][P_loc] global
// indices, steps without a resample flagged 0 in has_anc: identity) -- so
// every rank obtains the same trajectory without a per-step exchange.
template <typename T>
__global__ void trace_peer_kernel(int S, int nx, int P_loc, const void* const* __restrict__ x_tab,
                                  const int32_t* const* __restrict__ anc_tab, const int32_t* __restrict__ has_anc,
                                  const int32_t* __restrict__ j_final, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int j = j_final[0];
  for (int i = S; i >= 0; --i) {
    const int o = j / P_loc, l = j - o * P_loc;
    const T* x = static_cast<const T*>(x_tab[o]) + static_cast<size_t>(i) * nx * P_loc;
    for (int n = 0; n < nx; ++n) out[static_cast<size_t>(i) * nx + n] = static_cast<double>(x[static_cast<size_t>(n) * P_loc + l]);
    if (i > 0 && has_anc[i]) j = anc_tab[o][static_cast<size_t>(i - 1) * P_loc + l];
  }
}

// Final multinomial pick across ranks (resample(exp(logw), "multinomial", size=1)):
// the rank whose global CDF range holds u writes its global particle index,
// the others -1 (the host takes the max over ranks).
__global__ void pick_shard_kernel(int W, int rank, int P_loc, const uint64_t* __restrict__ cdf_local,
                                  const double* __restrict__ scale, const uint64_t* __restrict__ pref,
                                  const uint64_t* __restrict__ totals_all, const double* __restrict__ u,
                                  int32_t* __restrict__ j_out) {
  uint64_t off = 0, tot = 0;
  for (int d = 0; d < W; ++d) {
    if (d < rank) off += totals_all[d];
    tot += totals_all[d];
  }
  const double q = u[0];
  const double totd = static_cast<double>(tot);
  const bool mine = static_cast<double>(off) / totd <= q &&
                    (rank == W - 1 || q < static_cast<double>(off + totals_all[rank]) / totd);
  if (!mine) {
    if (threadIdx.x == 0) j_out[0] = -1;
    return;
  }
  const int nt = (P_loc + 31) >> 5;
  struct Cum {
    const uint64_t *cl, *tp, *bp;
    const double* sc;
    uint64_t off;
    double tot;
    __device__ __forceinline__ double operator()(int j) const {
      const int tw = j >> 5;
      return static_cast<double>(off + tp[tw] + bp[tw / kRecPerBlock] +
                                 __double2ull_rn(sc[tw] * static_cast<double>(__ldg(cl + j)))) / tot;
    }
  } cum{cdf_local, pref, pref + nt, scale, off, totd};
  const int j = warp_search_right(cum, P_loc, q, threadIdx.x);
  if (threadIdx.x == 0) j_out[0] = rank * P_loc + (j < P_loc ? j : P_loc - 1);
}

extern "C" int ssm_tiles_total(int B, int P, const void* tile_rec, const ssm_filter_state* fs,
                               uint64_t* total_out, void* workspace, void* stream) {
  if (B <= 0 || P <= 0 || !tile_rec || !fs || !total_out || !workspace) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SearchWs w;
  search_ws_layout(B, P, P, workspace, &w);
  const int nt = (P + 31) / 32;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  double* scale = reinterpret_cast<double*>(w.C);
  uint64_t* pref = reinterpret_cast<uint64_t*>(w.C) + static_cast<size_t>(B) * nt;
  uint64_t* blk = pref + B_total_tiles_offset(nt, B);
  // not gated on fs.resample_now: the trajectory pick needs the totals after an ESS-held step too
  tile_scale_kernel<<<dim3(nblk, B), kThreads, 0, s>>>(nt, static_cast<const ssm_tile_rec*>(tile_rec), fs, scale,
                                                      pref, blk, nullptr, 0);
  blk_prefix_kernel<<<B, 1024, 0, s>>>(nblk, blk, total_out, nullptr);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_offspring_push(int P, int P_global, int W, int rank, int scheme, const void* cdf_local,
                                  const uint64_t* totals_all, const double* u, const uint32_t* keys, int step,
                                  const ssm_filter_state* fs, int32_t* const* anc_tab, void* workspace, void* stream) {
  if (P <= 0 || W <= 0 || rank < 0 || rank >= W || P_global != P * W || !cdf_local || !totals_all || !fs ||
      !anc_tab || !workspace)
    return SSM_ERR_INVALID_ARG;
  if (!u && !keys) return SSM_ERR_INVALID_ARG;
  if (scheme != SSM_SYSTEMATIC && scheme != SSM_STRATIFIED) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SearchWs w;
  search_ws_layout(1, P, P_global, workspace, &w);
  const int nt = (P + 31) / 32;
  double* scale = reinterpret_cast<double*>(w.C);
  uint64_t* pref = reinterpret_cast<uint64_t*>(w.C) + nt;
  uint64_t* g_off = w.totals + 1;
  uint32_t* long_count = reinterpret_cast<uint32_t*>(w.totals + 2);
  OffspringConsts* oc = reinterpret_cast<OffspringConsts*>(w.totals + 3);
  int4* long_runs = reinterpret_cast<int4*>(w.cnt);
  shard_consts_kernel<<<1, 32, 0, s>>>(W, rank, P_global, totals_all, u, keys, step, g_off, oc, long_count);
  const PeerStore st{anc_tab, P, rank * P};
  const ShardSpan span{g_off, P_global, rank * P};
  const dim3 g(scan_tiles(P), 1);
  if (scheme == SSM_SYSTEMATIC)
    offspring_tiles_kernel<SSM_SYSTEMATIC, PeerStore><<<g, kThreads, 0, s>>>(
        P, static_cast<const uint64_t*>(cdf_local), scale, pref, w.totals, u, keys, step, fs, st, long_runs, long_count,
        oc, span);
  else
    offspring_tiles_kernel<SSM_STRATIFIED, PeerStore><<<g, kThreads, 0, s>>>(
        P, static_cast<const uint64_t*>(cdf_local), scale, pref, w.totals, u, keys, step, fs, st, long_runs, long_count,
        oc, span);
  const int gx = std::max(1, std::min(1184, P_global / kRunChunk + 1));
  long_runs_kernel<PeerStore><<<dim3(gx, 1), kThreads, 0, s>>>(P, P_global, long_runs, long_count, fs, st);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_pick_sharded(int P, int W, int rank, const void* cdf_local, const uint64_t* totals_all,
                                const double* u, int32_t* j_out, void* workspace, void* stream) {
  if (P <= 0 || W <= 0 || rank < 0 || rank >= W || !cdf_local || !totals_all || !u || !j_out || !workspace)
    return SSM_ERR_INVALID_ARG;
  SearchWs w;
  search_ws_layout(1, P, P * W, workspace, &w);
  const int nt = (P + 31) / 32;
  pick_shard_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      W, rank, P, static_cast<const uint64_t*>(cdf_local), reinterpret_cast<const double*>(w.C),
      reinterpret_cast<const uint64_t*>(w.C) + nt, totals_all, u, j_out);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_trace_peer(int dtype, int S, int nx, int P, const void* const* x_tab, const int32_t* const* anc_tab,
                              const int32_t* has_anc, const int32_t* j_final, double* out, void* stream) {
  if (S < 0 || nx <= 0 || P <= 0 || !x_tab || !anc_tab || !has_anc || !j_final || !out) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == SSM_F64)
    trace_peer_kernel<double><<<1, 32, 0, s>>>(S, nx, P, x_tab, anc_tab, has_anc, j_final, out);
  else if (dtype == SSM_F32)
    trace_peer_kernel<float><<<1, 32, 0, s>>>(S, nx, P, x_tab, anc_tab, has_anc, j_final, out);
  else
    return SSM_ERR_INVALID_ARG;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_ipc_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return SSM_ERR_INVALID_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

extern "C" int ssm_ipc_close(void* ptr) {
  if (!ptr) return SSM_ERR_INVALID_ARG;
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

extern "C" size_t ssm_sharded_workspace_bytes(int B, int P, int P_global) {
  return search_ws_layout(B, P, P_global, nullptr, nullptr);
}

extern "C" size_t ssm_resample_workspace_bytes(int B, int P) {
  return ssm_search_workspace_bytes(B, P, P);
}

// Log-weights -> the fused kernel's warp-tile records (the weighting half of
// pw_kernel's warp_tile_weigh, standalone): per 32-particle tile m_w = float
// round-up of the tile max, q_j = round(exp(a_j - m_w) 2^52), cdf_local = the
// tile-inclusive prefix of q, {m_w, Q_w}; and per filter a state with
// incr = shift (the weights' log-sum-exp) for the tile-path resample that
// follows.  One warp per tile, grid-stride.
template <typename T>
__global__ void __launch_bounds__(kThreads)
logw_tiles_kernel(int P, const T* __restrict__ a, const double* __restrict__ shift,
                  const ssm_filter_state* __restrict__ fs_in, uint64_t* __restrict__ cloc,
                  ssm_tile_rec* __restrict__ trec, ssm_filter_state* __restrict__ fs_out) {
  __shared__ double s_exp_tab[64];
  if (threadIdx.x < 64) s_exp_tab[threadIdx.x] = c_exp_tab[threadIdx.x];
  __syncthreads();
  const int b = blockIdx.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ssm_filter_state f = {};
    f.incr = shift ? shift[b] : fs_in[b].incr;
    f.resample_now = fs_in ? fs_in[b].resample_now : 1;
    f.err_nonfinite = f.err_degenerate = f.err_param = INT_MAX;
    fs_out[b] = f;
  }
  const int lane = threadIdx.x & 31;
  const int nt = (P + 31) >> 5;
  const T* ab = a + static_cast<size_t>(b) * P;
  uint64_t* cl = cloc + static_cast<size_t>(b) * P;
  ssm_tile_rec* tr = trec + static_cast<size_t>(b) * nt;
  const int nwarps = gridDim.x * (kThreads / 32);
  for (int w = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); w < nt; w += nwarps) {
    const int p = w * 32 + lane;
    const bool act = p < P;
    const double a_d = act ? static_cast<double>(__ldg(ab + p)) : -CUDART_INF;
    const float af = __double2float_ru(a_d);
    const int key = __float_as_int(af) >= 0 ? __float_as_int(af) : (__float_as_int(af) ^ 0x7fffffff);
    const int kmax = __reduce_max_sync(0xffffffffu, act ? key : (-2147483647 - 1));
    const int kb = kmax >= 0 ? kmax : (kmax ^ 0x7fffffff);
    const double mw = static_cast<double>(__int_as_float(kb));
    const double e = (!act || mw == -CUDART_INF) ? 0.0 : exp_tile(a_d - mw, s_exp_tab);
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
    if (act) cl[p] = (static_cast<uint64_t>(qh) << 26) + ql;
    if (lane == 31) tr[w] = ssm_tile_rec{mw, (static_cast<uint64_t>(qh) << 26) + ql};
  }
}

extern "C" int ssm_resample_from_logw(int B, int P, int dtype, int scheme, const void* a,
                                      const double* shift, const ssm_filter_state* fs,
                                      const double* u, const uint32_t* keys, int step, int32_t* anc,
                                      void* workspace, void* stream) {
  if (B <= 0 || B > 65535 || P <= 0 || !a || !anc || !workspace) return SSM_ERR_INVALID_ARG;
  if (!shift && !fs) return SSM_ERR_INVALID_ARG;
  if (!u && !keys) return SSM_ERR_INVALID_ARG;
  if (dtype != SSM_F64 && dtype != SSM_F32) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SearchWs w;
  search_ws_layout(B, P, P, workspace, &w);
  const int tiles = scan_tiles(P);
  if (scheme == SSM_MULTINOMIAL) {
    int st = ssm_weights_scan(B, P, dtype, a, 1, shift, fs, w.C, nullptr, w.scan, stream);
    if (st != SSM_OK) return st;
    const dim3 g(grid_for(P, kThreads, 65535), B);
    binary_search_kernel<1><<<g, kThreads, 0, s>>>(P, P, w.C, u, keys, step, fs, anc);
#ifndef SSM_LOGW_VIA_TILES
#define SSM_LOGW_VIA_TILES 1  // 0: the log-weight scan paths below (A/B)
#endif
  } else if (SSM_LOGW_VIA_TILES &&
             (scheme == SSM_MULTINOMIAL_SORTED || scheme == SSM_SYSTEMATIC || scheme == SSM_STRATIFIED)) {
    // the filter path's resampler on tile records built from the log-weights (one
    // pass: read a, write cdf_local + records), then tile scale -> offspring
    // (ancestors written directly) -> long-run fill / the sorted-multinomial merge
    if (scheme == SSM_MULTINOMIAL_SORTED && (u || !keys)) return SSM_ERR_INVALID_ARG;  // device draws only
    const int nt = (P + 31) / 32;
    const dim3 g(std::max(1, std::min((nt + kThreads / 32 - 1) / (kThreads / 32), 8192)), B);
    if (dtype == SSM_F64)
      logw_tiles_kernel<double><<<g, kThreads, 0, s>>>(P, static_cast<const double*>(a), shift, fs, w.lt_cdf, w.lt_rec,
                                                       w.lt_fs);
    else
      logw_tiles_kernel<float><<<g, kThreads, 0, s>>>(P, static_cast<const float*>(a), shift, fs, w.lt_cdf, w.lt_rec,
                                                      w.lt_fs);
    SSM_CHECK_LAUNCH();
    return ssm_resample_tiles_step(B, P, scheme, w.lt_cdf, w.lt_rec, w.lt_fs, u, keys, step, anc, workspace, 0, 1,
                                   stream);
  } else if (scheme == SSM_MULTINOMIAL_SORTED) {  // log-weight scan + spacing merge
    if (u || !keys) return SSM_ERR_INVALID_ARG;  // device draws only
    int st = ssm_weights_scan(B, P, dtype, a, 1, shift, fs, w.C, nullptr, w.scan, stream);
    if (st != SSM_OK) return st;
    // spacing block sums over P + 1 outputs in w.sums (as doubles), total in w.totals
    const int nsb = (P + 1 + kScanTile - 1) / kScanTile;
    double* blkE = reinterpret_cast<double*>(w.sums);
    double* totE = reinterpret_cast<double*>(w.totals);
    spacing_sums_kernel<<<dim3(nsb, B), kThreads, 0, s>>>(P, keys, step, fs, blkE, w.spc);
    spacing_prefix_kernel<<<B, 1024, 0, s>>>(nsb, blkE, totE, fs);
    spacing_merge_kernel<0><<<dim3(tiles, B), kThreads, 0, s>>>(P, w.C, nullptr, nullptr, nullptr, nullptr, w.spc,
                                                                blkE, totE, fs, anc);
    } else if (scheme == SSM_SYSTEMATIC || scheme == SSM_STRATIFIED) {
    if (dtype == SSM_F64) {
      tile_sums_kernel<double><<<dim3(tiles, B), kThreads, 0, s>>>(P, static_cast<const double*>(a), shift, fs, w.sums);
      tile_prefix_kernel<<<B, 1024, 0, s>>>(tiles, w.sums, w.totals, fs);
      launch_offspring_expand<kCumLogw, double>(scheme, B, P, P, a, shift, w, u, keys, step, fs, anc, s);
    } else {
      tile_sums_kernel<float><<<dim3(tiles, B), kThreads, 0, s>>>(P, static_cast<const float*>(a), shift, fs, w.sums);
      tile_prefix_kernel<<<B, 1024, 0, s>>>(tiles, w.sums, w.totals, fs);
      launch_offspring_expand<kCumLogw, float>(scheme, B, P, P, a, shift, w, u, keys, step, fs, anc, s);
    }
  } else {
    return SSM_ERR_INVALID_ARG;
  }
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_gather(int dtype, int B, int nx, int P, const void* x_in, const int32_t* anc,
                          void* x_out, void* stream) {
  if (B <= 0 || B > 65535 || nx <= 0 || P <= 0 || !x_in || !anc || !x_out) return SSM_ERR_INVALID_ARG;
  const dim3 g(grid_for(P, kThreads, 8192), B);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == SSM_F64)
    gather_kernel<double><<<g, kThreads, 0, s>>>(nx, P, (const double*)x_in, anc, (double*)x_out);
  else if (dtype == SSM_F32)
    gather_kernel<float><<<g, kThreads, 0, s>>>(nx, P, (const float*)x_in, anc, (float*)x_out);
  else
    return SSM_ERR_INVALID_ARG;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_gather_cols(int dtype, int nx, int n_out, int in_stride, const void* x_in, const int32_t* idx,
                               void* x_out, void* stream) {
  if (nx <= 0 || n_out < 0 || in_stride <= 0 || !x_in || !idx || !x_out) return SSM_ERR_INVALID_ARG;
  if (n_out == 0) return SSM_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int g = grid_for(n_out, kThreads, 8192);
  if (dtype == SSM_F64)
    gather_cols_kernel<double><<<g, kThreads, 0, s>>>(nx, n_out, in_stride, (const double*)x_in, idx, (double*)x_out);
  else if (dtype == SSM_F32)
    gather_cols_kernel<float><<<g, kThreads, 0, s>>>(nx, n_out, in_stride, (const float*)x_in, idx, (float*)x_out);
  else
    return SSM_ERR_INVALID_ARG;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// Trajectory pick (sample_trajectory's one multinomial draw, particle.py:140-141)
// from the fused kernel's tile records: one warp per filter searches the
// global fixed-point CDF for u_b (no full scan of the weights).
__global__ void __launch_bounds__(32)
pick_tiles_kernel(int P, const uint64_t* __restrict__ cdf_local, const double* __restrict__ scale,
                  const uint64_t* __restrict__ pref, const uint64_t* __restrict__ totals,
                  const double* __restrict__ u, int32_t* __restrict__ j_out) {
  const int b = blockIdx.x;
  const int nt = (P + 31) >> 5;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  const CumTileRecs cum{cdf_local + static_cast<size_t>(b) * P, scale + static_cast<size_t>(b) * nt,
                        pref + static_cast<size_t>(b) * nt,
                        pref + B_total_tiles_offset(nt, gridDim.x) + static_cast<size_t>(b) * nblk,
                        static_cast<double>(totals[b])};
  const int j = warp_search_right(cum, P, u[b], threadIdx.x);
  if (threadIdx.x == 0) j_out[b] = j < P ? j : P - 1;
}

extern "C" int ssm_pick_from_tiles(int B, int P, const void* cdf_local, const void* tile_rec,
                                   const ssm_filter_state* fs, const double* u, int32_t* j_out, void* workspace,
                                   void* stream) {
  if (B <= 0 || B > 65535 || P <= 0 || !cdf_local || !tile_rec || !fs || !u || !j_out || !workspace)
    return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SearchWs w;
  search_ws_layout(B, P, P, workspace, &w);
  const int nt = (P + 31) / 32;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  double* scale = reinterpret_cast<double*>(w.C);
  uint64_t* pref = reinterpret_cast<uint64_t*>(w.C) + static_cast<size_t>(B) * nt;
  uint64_t* blk = pref + B_total_tiles_offset(nt, B);
  tile_scale_kernel<<<dim3(nblk, B), kThreads, 0, s>>>(nt, static_cast<const ssm_tile_rec*>(tile_rec), fs, scale,
                                                      pref, blk, nullptr, 0);
  blk_prefix_kernel<<<B, 1024, 0, s>>>(nblk, blk, w.totals, nullptr);
  pick_tiles_kernel<<<B, 32, 0, s>>>(P, static_cast<const uint64_t*>(cdf_local), scale, pref, w.totals, u, j_out);
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_trace(int dtype, int B, int S, int nx, int P, const void* const* xs,
                         const int32_t* const* ancs, const int32_t* j_final, double* out,
                         void* stream) {
  if (B <= 0 || S < 0 || nx <= 0 || P <= 0 || !xs || !ancs || !j_final || !out)
    return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == SSM_F64)
    trace_kernel<double><<<B, 128, 0, s>>>(B, S, nx, P, xs, ancs, j_final, out);
  else if (dtype == SSM_F32)
    trace_kernel<float><<<B, 128, 0, s>>>(B, S, nx, P, xs, ancs, j_final, out);
  else
    return SSM_ERR_INVALID_ARG;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" size_t ssm_lse_workspace_bytes(int B, int P) {
  (void)P;
  return static_cast<size_t>(B) * kMaxLseBlocks * sizeof(Lse) + 256 + sizeof(uint32_t) * B;
}

extern "C" int ssm_logsumexp(int dtype, int B, int P, const void* a, double* out_lse,
                             double* out_ess, void* workspace, void* stream) {
  if (B <= 0 || B > 65535 || P <= 0 || !a || !out_lse || !workspace) return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Lse* parts = static_cast<Lse*>(workspace);
  uint32_t* done = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(workspace) +
                                               static_cast<size_t>(B) * kMaxLseBlocks * sizeof(Lse) + 256);
  cudaError_t e = cudaMemsetAsync(done, 0, sizeof(uint32_t) * B, s);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  const dim3 g(grid_for(P, kThreads, kMaxLseBlocks), B);
  if (dtype == SSM_F64)
    lse_kernel<double><<<g, kThreads, 0, s>>>(P, (const double*)a, parts, done, out_lse, out_ess);
  else if (dtype == SSM_F32)
    lse_kernel<float><<<g, kThreads, 0, s>>>(P, (const float*)a, parts, done, out_lse, out_ess);
  else
    return SSM_ERR_INVALID_ARG;
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

extern "C" int ssm_block_gather(int J, size_t block_bytes, const void* src, const int32_t* idx,
                                void* dst, void* stream) {
  if (J <= 0 || J > 65535 || block_bytes == 0 || (block_bytes % 16) != 0 || !src || !idx || !dst)
    return SSM_ERR_INVALID_ARG;
  const size_t words = block_bytes / 16;
  const dim3 g(grid_for(static_cast<int>(words < 0x7fffffff ? words : 0x7fffffff), kThreads, 1024), J);
  block_gather_kernel<<<g, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      words, static_cast<const uint4*>(src), idx, static_cast<uint4*>(dst));
  SSM_CHECK_LAUNCH();
  return SSM_OK;
}

// ===========================================================================
// Persistent cooperative driver (ssm_advance_coop): the whole grid loop of
// ssm_advance in ONE cooperative launch for moderate particle counts (PMMH
// chains, SMC^2 theta-particles: a few 10^5 - 10^6 particles per launch, where
// the per-step kernels are latency-bound).  Every phase runs the multi-kernel
// path's device bodies on virtual blocks -- tile scale with the filter prefix
// in its last block, offspring + window fill, long runs, the fused
// propagate/weight step with its last-block finalize -- separated by grid-wide
// barriers, so the results are bitwise those of ssm_advance.
// ===========================================================================

#include <cooperative_groups.h>

#include "ssm_pw_body.cuh"

namespace ssm {

struct CoopArgs {
  ssm_advance_args A;          // as ssm_advance (host fields unused)
  const ssm_step_desc* steps;  // device [n_steps]
  SearchWs w;                  // A.resample_ws as laid out by search_ws_layout(B, P, P)
};

template <int MODEL, typename T, bool E, bool SIMPLE, int SCHEME>
__global__ void __launch_bounds__(kThreads, MODEL == SSM_MODEL_WINDKESSEL ? 3 : 2) advance_coop_kernel(const CoopArgs C) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const ssm_advance_args& A = C.A;
  constexpr int NX = MODEL == SSM_MODEL_LORENZ96 ? 8 : 1;
  const int B = A.pw.B, P = A.pw.P;
  const size_t esz = sizeof(T);
  const size_t xstep = static_cast<size_t>(B) * NX * P * esz, astep = static_cast<size_t>(B) * P * esz;
  const SearchWs& w = C.w;  // the resample workspace, laid out as ssm_resample_from_tiles
  const int nt = (P + 31) / 32;
  const int nblk = (nt + kRecPerBlock - 1) / kRecPerBlock;
  double* scale = reinterpret_cast<double*>(w.C);
  uint64_t* pref = reinterpret_cast<uint64_t*>(w.C) + static_cast<size_t>(B) * nt;
  uint64_t* blk = pref + B_total_tiles_offset(nt, B);
  uint32_t* long_count = reinterpret_cast<uint32_t*>(w.totals) + 2 * static_cast<size_t>(B);
  int4* long_runs = reinterpret_cast<int4*>(w.cnt);
  OffspringConsts* oc = reinterpret_cast<OffspringConsts*>(w.totals + 3 * static_cast<size_t>(B));
  const int nob = scan_tiles(P);  // offspring blocks per filter
  const int nvb = pw_grid_x(P);   // fused-step blocks per filter
  const int gx_long = max(1, min(1184 / B, P / kRunChunk + 1));

  __shared__ ssm_pw_args s_args;  // this step's arguments (built by thread 0)
  const void* x_prev = A.x_in;
  const void* a_last = A.a_prev;
  int maybe = A.maybe_nonuniform, slot = 0, last_obs = -1;
  for (int k = 0; k < A.n_steps; ++k)
    if (C.steps[k].has_obs) last_obs = k;
  const bool skip_a = !A.ess_gate;
  for (int k = 0; k < A.n_steps; ++k) {
    const ssm_step_desc d = C.steps[k];
    int32_t* anc = nullptr;
    if (maybe) {
      anc = A.anc_arena + static_cast<size_t>(k) * B * P;
      // (1) tile scale + in-block prefix; the last block of each filter the block prefix and constants
      for (int it = blockIdx.x; it < B * nblk; it += gridDim.x) {
        __syncthreads();
        tile_scale_body(it / nblk, it % nblk, nblk, nt, static_cast<const ssm_tile_rec*>(A.tile_rec), A.pw.fs, scale,
                        pref, blk, long_count, 1, A.pw.fs, w.totals, oc, P, nullptr, A.pw.keys, d.step);
      }
      grid.sync();
      // (2) offspring counts + window fill
      const LocalStore st{anc, P};
      for (int it = blockIdx.x; it < B * nob; it += gridDim.x) {
        __syncthreads();
        offspring_tiles_body<SCHEME, LocalStore>(it / nob, it % nob, B, P, static_cast<const uint64_t*>(A.cdf_local),
                                                 scale, pref, nullptr, A.pw.keys, d.step, A.pw.fs, st, long_runs,
                                                 long_count, oc, ShardSpan{nullptr, P, 0});
      }
      grid.sync();
      // (3) long offspring runs (degenerate weights only)
      bool any_long = false;
      for (int b = 0; b < B; ++b) any_long |= A.pw.fs[b].resample_now && long_count[b] > 0;
      if (any_long) {
        for (int it = blockIdx.x; it < B * gx_long; it += gridDim.x) {
          __syncthreads();
          long_runs_body(it / gx_long, it % gx_long, gx_long, P, P, long_runs, long_count, A.pw.fs, st);
        }
        grid.sync();
      }
    }
    // (4) the fused propagate / weight step, finalize in the last virtual block of each filter
    const int slot_x = A.x_ring > 0 ? k % A.x_ring : k;
    void* x_out = static_cast<char*>(A.x_arena) + static_cast<size_t>(slot_x) * xstep;
    void* a_out = nullptr;
    const int a_slot = A.a_ring > 0 ? slot % A.a_ring : slot;
    if (d.has_obs && !(skip_a && k != last_obs)) a_out = static_cast<char*>(A.a_arena) + static_cast<size_t>(a_slot) * astep;
    __syncthreads();
    if (threadIdx.x == 0) {
      s_args = A.pw;
      s_args.step = d.step;
      s_args.n_sub = d.n_sub;
      s_args.hints = static_cast<uint32_t>(d.hints);
      s_args.subs = A.subs_table + d.subs_offset;
      s_args.x_in = x_prev;
      s_args.x_out = x_out;
      s_args.anc = anc;
      s_args.a_prev = a_last;
      s_args.has_obs = d.has_obs;
      s_args.obs_mask = d.obs_mask;
      for (int n = 0; n < 8; ++n) s_args.y[n] = d.y[n];
      s_args.u_obs = d.u_obs;
      s_args.a_out = a_out;
      s_args.cdf_local = d.has_obs ? A.cdf_local : nullptr;
      s_args.tile_rec = d.has_obs ? A.tile_rec : nullptr;
    }
    __syncthreads();
    const bool simple = SIMPLE && (d.hints & SSM_HINT_SINGLE_SUBSTEP) && d.n_sub == 1;
    for (int it = blockIdx.x; it < B * nvb; it += gridDim.x) {
      __syncthreads();
      if (simple)
        pw_body<MODEL, T, E, false, SIMPLE>(s_args, it / nvb, it % nvb, nvb);
      else
        pw_body<MODEL, T, E, false, false>(s_args, it / nvb, it % nvb, nvb);
    }
    grid.sync();
    x_prev = x_out;
    if (d.has_obs) {
      if (a_out) a_last = a_out;
      ++slot;
      maybe = 1;
    } else if (maybe && !A.ess_gate) {
      maybe = 0;
    }
  }
}

template <int MODEL, typename T, bool E, bool SIMPLE, int SCHEME>
static int launch_coop(const CoopArgs& C, cudaStream_t s) {
  auto kern = advance_coop_kernel<MODEL, T, E, SIMPLE, SCHEME>;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
  if (per_sm < 1) return SSM_ERR_UNSUPPORTED;
  const int B = C.A.pw.B, P = C.A.pw.P;
  const int want = B * std::max(pw_grid_x(P), scan_tiles(P));
  const int grid = std::max(1, std::min(sms * per_sm, want));
  void* params[] = {const_cast<CoopArgs*>(&C)};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(kThreads),
                                                    params, 0, s);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

template <int MODEL, typename T, bool E>
static int launch_coop_scheme(const CoopArgs& C, bool simple, cudaStream_t s) {
  (void)simple;
  if (C.A.scheme == SSM_SYSTEMATIC) return launch_coop<MODEL, T, E, true, SSM_SYSTEMATIC>(C, s);
  return launch_coop<MODEL, T, E, true, SSM_STRATIFIED>(C, s);
}

}  // namespace ssm

extern "C" int ssm_advance_coop(ssm_advance_args* A, const ssm_step_desc* steps_dev, void* stream) {
  using namespace ssm;
  if (!A || !A->steps || !steps_dev || A->n_steps < 0 || !A->x_in || !A->x_arena || !A->anc_used ||
      !A->resample_ws || !A->cdf_local || !A->tile_rec)
    return SSM_ERR_INVALID_ARG;
  if (A->pw.noise != nullptr || !A->pw.keys || !A->tiles) return SSM_ERR_INVALID_ARG;
  if (A->scheme != SSM_SYSTEMATIC && A->scheme != SSM_STRATIFIED) return SSM_ERR_UNSUPPORTED;
  if (A->pw.model != SSM_MODEL_LORENZ96 && A->pw.model != SSM_MODEL_WINDKESSEL) return SSM_ERR_UNSUPPORTED;
  if (A->n_steps == 0) return SSM_OK;
  // the host-side bookkeeping of ssm_advance: which steps resample, the last weighted slot
  const int maybe0 = A->maybe_nonuniform;
  int maybe = maybe0, slot = 0, last_obs = -1;
  for (int k = 0; k < A->n_steps; ++k)
    if (A->steps[k].has_obs) last_obs = k;
  A->a_last_index = -1;
  bool all_single = true;
  for (int k = 0; k < A->n_steps; ++k) {
    const ssm_step_desc& d = A->steps[k];
    A->anc_used[k] = maybe ? 1 : 0;
    all_single &= (d.hints & SSM_HINT_SINGLE_SUBSTEP) && d.n_sub == 1;
    if (d.has_obs) {
      const int a_slot = A->a_ring > 0 ? slot % A->a_ring : slot;
      if (A->ess_gate || k == last_obs) A->a_last_index = a_slot;
      ++slot;
      maybe = 1;
    } else if (maybe && !A->ess_gate) {
      maybe = 0;
    }
  }
  (void)all_single;
  for (int k = 0; k < A->n_steps; ++k)
    if (A->anc_used[k] && !A->anc_arena) return SSM_ERR_INVALID_ARG;
  if (A->pw.exact) return SSM_ERR_UNSUPPORTED;  // the FMA (fast) arithmetic only; exact runs take ssm_advance
  CoopArgs C{*A, steps_dev, SearchWs{}};  // carries the START state (maybe_nonuniform = maybe0)
  search_ws_layout(A->pw.B, A->pw.P, A->pw.P, A->resample_ws, &C.w);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // SIMPLE instances carry both paths (steps without the hint take the general body)
  int st;
  if (A->pw.model == SSM_MODEL_LORENZ96)
    st = A->pw.dtype == SSM_F64 ? launch_coop_scheme<SSM_MODEL_LORENZ96, double, false>(C, true, s)
                                : launch_coop_scheme<SSM_MODEL_LORENZ96, float, false>(C, true, s);
  else
    st = A->pw.dtype == SSM_F64 ? launch_coop_scheme<SSM_MODEL_WINDKESSEL, double, false>(C, true, s)
                                : launch_coop_scheme<SSM_MODEL_WINDKESSEL, float, false>(C, true, s);
  if (st == SSM_OK) A->maybe_nonuniform = maybe;  // unchanged on failure: the caller may fall back to ssm_advance
  (void)maybe0;
  return st;
}
