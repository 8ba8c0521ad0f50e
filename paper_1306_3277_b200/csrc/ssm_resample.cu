// K4 weight scan, K5 ancestor search, K6 gather, K8 trace, K3 standalone LSE,
// K9 theta-block gather.  Reference: inference/resampling.py:15-36,
// inference/particle.py:96-105 and 137-149, inference/smc.py:96-98.

#include <stdio.h>

#include "ssm_common.cuh"

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
            const ssm_filter_state* __restrict__ fs, uint64_t* __restrict__ C, ScanWs ws) {
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
    }
    sm[e + (e >> 3)] = q;
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
      if (lane == 0) st_status(&status[0], kFlagPrefix | block_tot);
    } else {
      if (lane == 0) st_status(&status[j], kFlagAgg | block_tot);
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
      if (lane == 0) st_status(&status[j], kFlagPrefix | (excl + block_tot));
    }
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
constexpr int kMergeTile = kThreads * kMergeItems;  // merged-diagonal elements per block

// merge-path split: number of cum elements among the first d merged elements
// (cum_j precedes u_k iff cum_j <= u_k)
template <typename FA, typename FB>
__device__ __forceinline__ int merge_split(int d, int na, int nb, FA A, FB Bq) {
  int lo = d > nb ? d - nb : 0;
  int hi = d < na ? d : na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A(mid) <= Bq(d - 1 - mid))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <int SCHEME, int KIND>
__global__ void __launch_bounds__(kThreads)
merge_search_kernel(int P_in, int P_out, const void* __restrict__ cum, const double* __restrict__ u,
                    const uint32_t* __restrict__ keys, int step,
                    const ssm_filter_state* __restrict__ fs, int32_t* __restrict__ anc) {
  __shared__ double sA[kMergeTile];
  __shared__ double sB[kMergeTile];
  __shared__ int32_t sOut[kMergeTile];
  __shared__ int s_split[2];
  const int b = blockIdx.y;
  int32_t* ancb = anc + static_cast<size_t>(b) * P_out;
  const int total = P_in + P_out;
  const int d0 = blockIdx.x * kMergeTile;
  if (d0 >= total) return;
  const int d1 = min(d0 + kMergeTile, total);
  if (fs && !fs[b].resample_now) {
    // identity ancestors (ESS gate held, particle.py:99-100)
    const int k0 = d0 >> 1, k1 = min(d1 >> 1, P_out);
    for (int k = k0 + threadIdx.x; k < k1; k += kThreads) ancb[k] = k;
    if (blockIdx.x == gridDim.x - 1)
      for (int k = k1 + threadIdx.x; k < P_out; k += kThreads) ancb[k] = k;
    return;
  }
  const size_t coff = static_cast<size_t>(b) * P_in;
  const double tot = cum_total<KIND>(cum, coff, P_in);
  const double u_sys =
      SCHEME == SSM_SYSTEMATIC
          ? (u ? u[b] : device_uniform(keys[2 * b], keys[2 * b + 1], 0u, step, kPurposeSystematic))
          : 0.0;
  const double* ub = (SCHEME == SSM_STRATIFIED && u) ? u + static_cast<size_t>(b) * P_out : nullptr;
  const uint32_t k0 = keys ? keys[2 * b] : 0u, k1 = keys ? keys[2 * b + 1] : 0u;
  auto A = [&](int j) { return cum_at<KIND>(cum, coff, tot, j); };
  auto Bq = [&](int k) { return query<SCHEME>(k, P_out, u_sys, ub, k0, k1, step); };
  if (threadIdx.x < 2) {
    const int d = threadIdx.x == 0 ? d0 : d1;
    s_split[threadIdx.x] = merge_split(d, P_in, P_out, A, Bq);
  }
  __syncthreads();
  const int i0 = s_split[0], i1 = s_split[1];
  const int kb0 = d0 - i0, kb1 = d1 - i1;
  const int na = i1 - i0, nb = kb1 - kb0;
  for (int t = threadIdx.x; t < na; t += kThreads) sA[t] = A(i0 + t);
  for (int t = threadIdx.x; t < nb; t += kThreads) sB[t] = Bq(kb0 + t);
  __syncthreads();
  // per-thread merge of kMergeItems diagonal elements
  const int dl = threadIdx.x * kMergeItems;
  if (dl < na + nb) {
    int ia = merge_split(dl, na, nb, [&](int j) { return sA[j]; }, [&](int k) { return sB[k]; });
    int kb = dl - ia;
    const int lim = min(dl + kMergeItems, na + nb);
    for (int e = dl; e < lim; ++e) {
      if (ia < na && (kb >= nb || sA[ia] <= sB[kb])) {
        ++ia;
      } else {
        const int a_idx = i0 + ia;
        sOut[kb] = a_idx < P_in ? a_idx : P_in - 1;  // .clip(0, P-1)
        ++kb;
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nb; t += kThreads) ancb[kb0 + t] = sOut[t];
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

template <typename T>
__global__ void trace_kernel(int B, int S, int nx, int P, const void* const* xs,
                             const int32_t* const* ancs, const int32_t* j_final, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  int j = j_final[b];
  const size_t row = static_cast<size_t>(b) * (S + 1);
  for (int i = S; i >= 0; --i) {
    const T* xi = static_cast<const T*>(xs[row + i]);
    for (int n = 0; n < nx; ++n)
      out[(row + i) * nx + n] = static_cast<double>(xi[static_cast<size_t>(n) * P + j]);
    if (i > 0) {
      const int32_t* a = ancs[row + i];
      if (a) j = a[j];
    }
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
                                                             nullptr, fs, C, ws);
  } else if (dtype == SSM_F64) {
    scan_kernel<double, true><<<B * tiles, kThreads, 0, s>>>(B, P, static_cast<const double*>(a),
                                                            shift, fs, C, ws);
  } else if (dtype == SSM_F32) {
    scan_kernel<float, true><<<B * tiles, kThreads, 0, s>>>(B, P, static_cast<const float*>(a),
                                                           shift, fs, C, ws);
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

extern "C" int ssm_resample_search(int B, int P_in, int P_out, int scheme, int cum_kind,
                                   const void* cum, const double* u, const uint32_t* keys, int step,
                                   const ssm_filter_state* fs, int32_t* anc, void* stream) {
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
    const long long total = static_cast<long long>(P_in) + P_out;
    const dim3 g(static_cast<unsigned>((total + kMergeTile - 1) / kMergeTile), B);
    if (scheme == SSM_STRATIFIED) {
      if (cum_kind == 0)
        merge_search_kernel<SSM_STRATIFIED, 0><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
      else
        merge_search_kernel<SSM_STRATIFIED, 1><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
    } else {
      if (cum_kind == 0)
        merge_search_kernel<SSM_SYSTEMATIC, 0><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
      else
        merge_search_kernel<SSM_SYSTEMATIC, 1><<<g, kThreads, 0, s>>>(P_in, P_out, cum, u, keys, step, fs, anc);
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

extern "C" int ssm_trace(int dtype, int B, int S, int nx, int P, const void* const* xs,
                         const int32_t* const* ancs, const int32_t* j_final, double* out,
                         void* stream) {
  if (B <= 0 || S < 0 || nx <= 0 || P <= 0 || !xs || !ancs || !j_final || !out)
    return SSM_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nt = 128;
  if (dtype == SSM_F64)
    trace_kernel<double><<<(B + nt - 1) / nt, nt, 0, s>>>(B, S, nx, P, xs, ancs, j_final, out);
  else if (dtype == SSM_F32)
    trace_kernel<float><<<(B + nt - 1) / nt, nt, 0, s>>>(B, S, nx, P, xs, ancs, j_final, out);
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
