/*
 * ssm_b200.h -- C ABI of libssm_b200.so, the sm_100a implementation of the
 * bootstrap-particle-filter hot path of the LibBi paper (arXiv 1306.3277),
 * as restated by the reference package `ssmkit`.
 *
 * All reference citations are file:line under /root/reference/pkg/src/ssmkit.
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless stated otherwise.
 *   - Every entry point is stream-ordered on `stream` (a cudaStream_t passed
 *     as void*; NULL = legacy default stream), reentrant, and keeps no global
 *     mutable state.  The library never allocates: scratch space comes from
 *     the caller through `workspace` pointers sized by the *_workspace_bytes()
 *     queries.
 *   - Particle state is SoA: x[b][slot][p] for filter b of a batch of B
 *     filters, P particles each, nx state slots (L96: 8, windkessel: 1).
 *   - `dtype` selects the arithmetic type of states and log-weights:
 *     SSM_F64 (the reference's float64) or SSM_F32.  Log-likelihood
 *     accumulators, LSE/ESS reductions and resampling CDFs are always float64
 *     (CDF: exact 64-bit fixed point, see ssm_weights_scan).
 *   - Return value: ssm_status.  Data-dependent failures that the reference
 *     raises as exceptions (NonFiniteStateError simulate.py:158-162,
 *     DegenerateEnsembleError particle.py:128-131 / resampling.py:23-24,
 *     ValueError resampling.py:20-21) are recorded on the device in
 *     ssm_filter_state / an int flag word and mapped to the same exception
 *     classes (with time=) by the host layer.
 */
#ifndef SSM_B200_H
#define SSM_B200_H

#ifndef __CUDACC_RTC__ /* the NVRTC-compiled generic-model kernels include this header too */
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SSM_OK = 0,
  SSM_ERR_INVALID_ARG = 1,
  SSM_ERR_CUDA = 2,
  SSM_ERR_UNSUPPORTED = 3
} ssm_status;

typedef enum { SSM_F32 = 0, SSM_F64 = 1 } ssm_dtype;

/* model ids: the two hand-written model kernels, and any other model lowered
 * from a reference ModelIr and compiled at run time (ssm_gen_compile) */
typedef enum {
  SSM_MODEL_LORENZ96 = 0,   /* Lorenz96.bi  (8 slots, RK4, Wiener noise) */
  SSM_MODEL_WINDKESSEL = 1, /* Windkessel.bi (1 slot, analytic update, input F) */
  SSM_MODEL_GENERIC = 2     /* ssm_pw_args.gen: a handle from ssm_gen_compile */
} ssm_model;

/* resampling schemes, resampling.py:12 SCHEMES */
typedef enum {
  SSM_MULTINOMIAL = 0,
  SSM_STRATIFIED = 1,
  SSM_SYSTEMATIC = 2,
  /* multinomial with device draws, ancestors in ascending order: searchsorted(cum,
   * U_(k)) with U_(k) = S_k / S_{P+1} the order statistics of P iid uniforms from
   * exponential spacings (the law of resampling.py:28-36's multinomial draw, slot
   * order sorted).  ssm_resample_from_logw / ssm_advance with device keys only. */
  SSM_MULTINOMIAL_SORTED = 3
} ssm_scheme;

/* flag bits written by ssm_weights_scan for raw (non-log) weights,
 * resampling.py:18-24 */
#define SSM_FLAG_BAD_WEIGHT 1u  /* negative or non-finite weight -> ValueError */
#define SSM_FLAG_ZERO_TOTAL 2u  /* all weights zero -> DegenerateEnsembleError */
/* (is_log = 1, flags != NULL) the normalisation precondition sum exp(a - shift) = 1
 * is violated: a weight above 1 + 2^-20 or a fixed-point prefix reaching 2^62
 * (the look-back flag bits).  The CDF is then not meaningful -> ValueError. */
#define SSM_FLAG_UNNORMALISED 4u

/* One transition sub-step, built on the host from substep_schedule
 * (simulate.py:28-38) and the RK4 step split (simulate.py:85-87). */
typedef struct ssm_substep {
  double d;      /* sub-step duration */
  double sd;     /* sqrt(d): sd of the wiener() increment, simulate.py:54 */
  double u_in;   /* model input at the sub-step start (windkessel F(t_k)), simulate.py:150 */
  double s[4];   /* RK4 step lengths s_k = min(h, d - k h), simulate.py:85-87 */
  int32_t n_ode; /* number of RK4 steps (<= 4) */
  int32_t pad;
} ssm_substep;

/* Per-filter device state: the scalar part of ParticleRun (particle.py:47-59).
 * Zero-initialise, then set uniform = 1 (ParticleRun.init, particle.py:69-70),
 * err_* = INT32_MAX. */
typedef struct ssm_filter_state {
  double loglik;          /* ParticleRun.loglik */
  double incr;            /* LSE of the last weighted step (log-weights are a - incr) */
  double ess;             /* ESS of the current weights (particle.py:83-85) */
  double lse_raw;         /* scratch */
  int32_t uniform;        /* ParticleRun.weights_uniform */
  int32_t resample_now;   /* resample at the start of the next step (particle.py:96-100) */
  int32_t err_nonfinite;  /* min(step*64 + sub-step) with a non-finite state, else INT32_MAX */
  int32_t err_degenerate; /* min(step) with a non-finite LSE increment, else INT32_MAX */
  uint32_t blocks_done;   /* completion counter for the fused finalize (reset by the kernel) */
  int32_t err_param;      /* generic models: min(step*64 + sub-step) where a distribution
                             argument was invalid (DistributionParameterError,
                             distributions.py:53-69), else INT32_MAX */
  uint32_t prefix_done;   /* completion counter of the resample's tile-prefix pass (reset by the kernel) */
  int32_t pad;
} ssm_filter_state;

/* Arguments of the fused propagate + weight step (kernels K1/K2).
 * Replaces, per grid step i, ParticleRun._step after resampling
 * (particle.py:107-135): the ancestor gather x = x[anc] (particle.py:102),
 * simulate.step_transition (simulate.py:132-163), simulate.observe_logpdf
 * (simulate.py:166-193), logw + g, scipy logsumexp (particle.py:127), the
 * degenerate check (128-131), loglik += incr (132) and, when ess_rel >= 0,
 * the ESS gate for the next step (particle.py:99-100). */
typedef struct ssm_pw_args {
  int32_t model;        /* ssm_model */
  int32_t dtype;        /* ssm_dtype */
  int32_t B, P;         /* filters, particles per filter */
  int32_t step;         /* grid index i (RNG counter and error location) */
  int32_t n_sub;        /* number of sub-steps in subs[] */
  int32_t exact;        /* 1: reference op order, no FMA contraction (bitwise FP64) */
  int32_t check_finite; /* simulate.py:158 */
  int32_t has_obs;      /* grid.obs_at(i) is not None (timegrid.py:44-49) */
  uint32_t obs_mask;    /* bit n = obs slot n present */
  double y[8];          /* observation values by obs slot */
  double u_obs;         /* model input at the observation time (windkessel F(t_i)) */
  double log_w0;        /* -log(P): the uniform log-weight (particle.py:68, 103) */
  double obs_log_sd;    /* log(obs sd): log(0.5) L96, log(2.0) windkessel */
  double log_sqrt_2pi;  /* distributions.py:15 */
  double ess_rel;       /* < 0: no ESS gate (always resample after weighting) */
  const void* x_in;     /* [B][nx][P] positions at grid index i-1 */
  void* x_out;          /* [B][nx][P] positions at grid index i */
  const int32_t* anc;   /* [B][P] ancestors for step i (used iff fs.resample_now) or NULL */
  const void* a_prev;   /* [B][P] unnormalised log-weights of the last weighted step, or NULL */
  void* a_out;          /* [B][P] unnormalised log-weights logw + g (iff has_obs; may be NULL when
                           cdf_local is set and the next step resamples from the tile records) */
  const double* theta;  /* [B][4] derived per-filter constants */
  const ssm_substep* subs; /* [n_sub] */
  const void* noise;    /* injected noise-variable values [B][n_sub][n_noise][P], or NULL */
  const uint32_t* keys; /* [B][2] Philox4x32 keys, used when noise == NULL */
  ssm_filter_state* fs; /* [B] */
  void* workspace;      /* ssm_pw_workspace_bytes(B, P) bytes */
  void* cdf_local;      /* [B][P] uint64 tile-local fixed-point CDF for the next resample, or NULL */
  void* tile_rec;       /* [B][ceil(P/32)] ssm_tile_rec (one per warp tile), or NULL */
  uint32_t hints;       /* SSM_HINT_* bits the host guarantees */
  int32_t p_offset;     /* global index of particle 0 (device RNG counters; sharded filter) */
  int32_t x_in_stride;  /* row stride of x_in in particles (0: P) */
  int32_t x_out_stride; /* row stride of x_out in particles (0: P) */
  void* lse_out;        /* [B][4] doubles or NULL: if set, the finalize writes the LSE/ESS partial
                           (m, c, t, s2) here instead of updating fs (cross-rank combine) */
  const void* gen;      /* SSM_MODEL_GENERIC: the ssm_gen_compile handle, else NULL */
  int32_t theta_stride; /* doubles per filter in theta (0: 4, the hand-written kernels) */
  int32_t gen_pad;
  const double* y_vec;  /* generic models, nullable: observation values [n_obs] (<= 32) of this step
                           (device); NULL: y[] */
  const double* u_vec;  /* generic models, nullable: inputs [n_sub + 1][n_input] (device): one row per
                           sub-step start (simulate.py:150), then the observation time; NULL: u_in / u_obs */
  const void* const* x_peer; /* sharded filter, nullable (device): [W] every rank's x_in (peer-mapped, row
                                stride x_in_stride); anc then holds GLOBAL indices, rank = idx / peer_n */
  int32_t peer_n;            /* particles per rank */
  int32_t peer_pad;
} ssm_pw_args;

/* hint: subs[0] is the only sub-step and holds exactly one RK4 step (n_ode == 1) */
#define SSM_HINT_SINGLE_SUBSTEP 1u

/* Per 32-particle (warp) tile of a weighted step (written by ssm_propagate_weight):
 * the tile's max log-weight and its fixed-point weight total
 * Q = sum_j round(exp(a_j - m) * 2^52).  The tile-local inclusive prefix of the
 * same q_j is cdf_local.  ssm_resample_from_tiles turns them into exact
 * global 64-bit CDF offsets once the step's LSE is known. */
typedef struct ssm_tile_rec {
  double m;
  uint64_t Q;
} ssm_tile_rec;

const char* ssm_version(void);
const char* ssm_status_string(int status);
const char* ssm_last_cuda_error(void);
int ssm_sm_count(int device, int* out);

/* K1/K2 fused propagate + weight (+ gather, + LSE/ESS finalize).  Kernel choice
 * (same results): SIMPLE specialisations when SSM_HINT_SINGLE_SUBSTEP holds; for
 * Lorenz '96 with device noise, fast arithmetic, every slot observed, no ESS gate
 * and tile records requested, the variant that weighs each warp tile one tile
 * late (overlapping that chain with the next tile's RK4; SSM_NO_PW_LAG=1 in the
 * environment disables it). */
size_t ssm_pw_workspace_bytes(int B, int P);
int ssm_propagate_weight(const ssm_pw_args* args, void* stream);

/* Generic models: any reference ModelIr within the limits
 * below, lowered on the host (paper_1306_3277_b200/codegen.py) to a CUDA
 * source that defines `gen::Model` and includes csrc/ssm_gen_rt.cuh, then
 * compiled here for sm_100a with NVRTC and loaded into the current context
 * (ir.py:83-121 ModelIr, simulate.py:50-193 block semantics).
 *   ssm_gen_compile: source -> handle (`out`); `include_dir` = the csrc
 *     directory; `log` (HOST, nullable) receives the NVRTC log.  Compiles
 *     the float64 / FMA / device-noise fused kernel now (errors surface
 *     here); every other variant compiles on its first launch.
 *   ssm_gen_check: compile every variant only (no device needed; CPU tests).
 * The handle is used through ssm_pw_args.gen (model = SSM_MODEL_GENERIC) by
 * ssm_propagate_weight / ssm_advance, and by ssm_gen_init_particles (the
 * model's `initial` block on the device).  Limits: n_state <= 32,
 * n_obs <= 32, n_input <= 16 (vectors through ssm_pw_args.y_vec / u_vec),
 * <= 255 Philox blocks per sub-step. */
int ssm_gen_compile(const char* source, const char* include_dir, void** out, char* log, size_t log_len);
int ssm_gen_check(const char* source, const char* include_dir, char* log, size_t log_len);
int ssm_gen_destroy(void* handle);
int ssm_gen_info(const void* handle, int* n_state, int* n_draws);
int ssm_gen_init_particles(const void* handle, int dtype, int B, int P, int p_offset, const uint32_t* keys,
                           const double* theta, int theta_stride, void* x_out, ssm_filter_state* fs,
                           void* stream);

/* K7: initial particles (simulate.sample_initial, simulate.py:111-129) drawn
 * on the device: L96 x ~ U(-1,3) (Lorenz96.bi:21), windkessel Pp ~ N(90,15)
 * (Windkessel.bi:24).  keys: [B][2]. */
int ssm_init_particles(int model, int dtype, int B, int P, int p_offset, const uint32_t* keys,
                       void* x_out, void* stream);

/* Validation export of the device noise: the float32 standard normals the
 * fused kernels draw for particles [p_offset, p_offset + P) at grid step `step`,
 * sub-step `sub` (Philox4x32-10 + float32 Box-Muller, ssm_common.cuh).  L96:
 * out [B][8][P] (slot-major, the draws of Lorenz96.bi:25 before the sqrt(d)
 * scaling); windkessel: out [B][P].  Lets the tests feed the oracle the exact
 * draws the benchmark kernel consumed and test the generator's law. */
int ssm_device_normals(int model, int B, int P, int p_offset, const uint32_t* keys, int step, int sub,
                       float* out, void* stream);

/* Cross-rank finalize of a weighted step for a filter sharded over W ranks
 * (C1): combines the W per-rank partials (m, c, t, s2) in rank order and
 * performs the finalize of ssm_propagate_weight (loglik, degenerate flag, ESS
 * gate against P_total) on fs. parts: [W][B][4] doubles. */
int ssm_lse_combine(int W, int B, const double* parts, ssm_filter_state* fs, double ess_rel,
                    double P_total, int step, void* stream);

/* K4: per-filter CDF of the resampling weights as an exact, deterministic
 * 64-bit fixed-point inclusive scan (decoupled look-back), replacing
 * cumsum(w / w.sum()) with cum[-1] = 1 (resampling.py:22-27):
 *   cum[j] = (double)C[j] / (double)C[P-1].
 * is_log = 1: w = exp(a - shift[b]) with a of `dtype` (ParticleRun passes its
 * unnormalised log-weights and the last LSE, particle.py:101, 133); with
 * shift == NULL the shift is fs[b].incr.
 * is_log = 0: w = a (float64 raw weights); validated as in resampling.py:18-24
 * with failures OR-ed into flags[b] (SSM_FLAG_*).  flags is required for
 * is_log = 0 and optional for is_log = 1 (SSM_FLAG_UNNORMALISED).
 * fs (nullable): filters with fs[b].resample_now == 0 are skipped. */
size_t ssm_scan_workspace_bytes(int B, int P);
int ssm_weights_scan(int B, int P, int dtype, const void* a, int is_log, const double* shift,
                     const ssm_filter_state* fs, uint64_t* C, uint32_t* flags, void* workspace,
                     void* stream);
/* cum[b][j] = C[b][j] / C[b][P-1] as float64 (for inspection / parity tests) */
int ssm_fixed_to_cum(int B, int P, const uint64_t* C, double* cum, void* stream);

/* K5: ancestor search, searchsorted(cum, u, 'right').clip(0, P-1)
 * (resampling.py:28-36), exact in float64 on the reference's query values.
 *   systematic / stratified (sorted queries): per-particle offspring bounds
 *     c_j = #{k : u_k < cum_j} plus the merge-path partition they imply, then
 *     a search-free expand (anc_k = #{j : c_j <= k});
 *   multinomial: per-query binary search (query order kept).
 *   cum_kind 0: cum is float64 [B][P_in] (injected CDF, exact parity mode)
 *   cum_kind 1: cum is the uint64 fixed-point output of ssm_weights_scan
 * Queries: u != NULL -> injected uniforms, [B][P_out] (multinomial,
 * stratified) or [B][1] (systematic), exactly the draws resampling.py:28-33
 * consumes; u == NULL -> drawn on the device from keys[b] at counter `step`.
 * fs (nullable): filters with fs[b].resample_now == 0 get identity ancestors.
 * workspace: ssm_search_workspace_bytes(B, P_in, P_out) (unused for multinomial). */
size_t ssm_search_workspace_bytes(int B, int P_in, int P_out);
int ssm_resample_search(int B, int P_in, int P_out, int scheme, int cum_kind, const void* cum,
                        const double* u, const uint32_t* keys, int step,
                        const ssm_filter_state* fs, int32_t* anc, void* workspace, void* stream);

/* K4+K5 for the filter (particle.py:96-105): ancestors straight from the
 * unnormalised log-weights a (w = exp(a - shift[b]), shift NULL -> fs[b].incr).
 * shift must be the log-sum-exp of a[b] (the weights sum to 1): the exact
 * fixed-point CDF has 2^52 units per unit of weight and no headroom beyond 1.
 * systematic / stratified / sorted multinomial: one pass builds the fused
 * kernel's warp-tile records from a (tile-local 2^52 fixed point + {m_w, Q_w},
 * in the workspace), then the filter path's tile resampler (ssm_resample_tiles_step:
 * tile scale -> offspring counts writing the ancestors -> long-run fill, or the
 * spacing merge); multinomial (reference query order): look-back scan + binary
 * search. */
size_t ssm_resample_workspace_bytes(int B, int P);
/* Filter fast path: ancestors from the tile records + cdf_local written by the
 * weighted ssm_propagate_weight (systematic / stratified; sorted multinomial
 * with device keys): tile scale + in-block prefix, with the exact block prefix
 * done by the last block of each filter (fs.prefix_done) -> offspring counts
 * that write the ancestors (window fill in shared memory) -> long-run fill.
 * Global CDF: C_j = prefix_b + round(exp(m_b - incr) 2^9 cdf_local_j). */
int ssm_resample_from_tiles(int B, int P, int scheme, const void* cdf_local, const void* tile_rec,
                            const ssm_filter_state* fs, const double* u, const uint32_t* keys,
                            int step, int32_t* anc, void* workspace, void* stream);
/* ssm_resample_from_tiles as the native driver calls it once per grid step.
 * `parity` / `zero_state` carry the state of the single-kernel variant (built
 * with -DSSM_RESAMPLE_FUSED=1: tile scale + decoupled look-back prefix +
 * offspring + window fill in one kernel, look-back state double-buffered by
 * parity, cleared when zero_state != 0); the default build runs the two-kernel
 * path (tile scale with the block prefix in its last block, then offspring +
 * window fill), which measured faster.  ssm_resample_from_tiles = parity 0,
 * zero_state 1. */
int ssm_resample_tiles_step(int B, int P, int scheme, const void* cdf_local, const void* tile_rec,
                            const ssm_filter_state* fs, const double* u, const uint32_t* keys, int step,
                            int32_t* anc, void* workspace, int parity, int zero_state, void* stream);
int ssm_resample_from_logw(int B, int P, int dtype, int scheme, const void* a, const double* shift,
                           const ssm_filter_state* fs, const double* u, const uint32_t* keys,
                           int step, int32_t* anc, void* workspace, void* stream);

/* Native driver for ParticleRun.advance_to (particle.py:87-94), device-noise
 * mode: one call enqueues, for each grid step, the resample kernels (when the
 * previous step weighted, particle.py:96-105) and ssm_propagate_weight, with
 * the host-side weighting state machine.  No synchronisation. */
typedef struct ssm_step_desc {
  int32_t step;         /* grid index i */
  int32_t n_sub;
  int64_t subs_offset;  /* index of the step's first record in subs_table */
  int32_t has_obs;
  uint32_t obs_mask;
  int32_t hints;        /* SSM_HINT_* */
  int32_t pad;
  double y[8];
  double u_obs;
  int64_t y_off;        /* offset (doubles) of the step's y_vec in ssm_advance_args.y_table, or -1 */
  int64_t u_off;        /* offset (doubles) of the step's u_vec in ssm_advance_args.u_table, or -1 */
} ssm_step_desc;

typedef struct ssm_advance_args {
  ssm_pw_args pw;       /* per-run constants (model, dtype, B, P, exact, ..., theta, keys, fs,
                           workspace); per-step fields are filled by ssm_advance */
  const ssm_substep* subs_table;  /* device */
  const ssm_step_desc* steps;     /* HOST [n_steps] */
  int32_t n_steps;
  int32_t scheme;
  int32_t tiles;             /* 1: resample from the fused kernel's tile CDF (systematic/stratified) */
  int32_t maybe_nonuniform;  /* in: before the first step; out: after the last */
  int32_t ess_gate;          /* ess_rel >= 0 */
  int32_t x_ring;            /* 0: x_arena has n_steps slots (history kept); r > 0: step k writes
                                slot k % r (history-free runs: positions are replayed on demand) */
  const void* x_in;          /* [B][nx][P] */
  void* x_arena;             /* [n_steps or x_ring][B][nx][P] positions written per step */
  int32_t* anc_arena;        /* [n_steps][B][P]; slot k valid iff anc_used[k] */
  const void* a_prev;        /* unnormalised log-weights of the last weighted step, or NULL */
  void* a_arena;             /* [n_weighted or a_ring][B][P] */
  void* cdf_local;           /* [B][P] uint64 */
  void* tile_rec;            /* [B][ceil(P/32)] ssm_tile_rec */
  void* resample_ws;         /* ssm_resample_workspace_bytes(B, P) */
  int32_t* anc_used;         /* HOST out [n_steps] */
  int32_t a_last_index;      /* out: a_arena slot of the last weighted step (-1: a_prev) */
  int32_t a_ring;            /* 0: a_arena has a slot per weighted step; r > 0: weighted step w writes
                                slot w % r (only the last weighted step's log-weights are read later) */
  void* const* events;       /* HOST, nullable: 4 cudaEvent_t per step (resample start/end, pw start/end) */
  const double* y_table;     /* device, nullable: per-step observation vectors (ssm_step_desc.y_off) */
  const double* u_table;     /* device, nullable: per-step input rows (ssm_step_desc.u_off) */
} ssm_advance_args;

int ssm_advance(ssm_advance_args* args, void* stream);
/* ssm_advance as ONE persistent cooperative launch (moderate particle counts:
 * PMMH chains, SMC^2 theta-particles), hand-written models, device noise, the
 * tile path with systematic / stratified resampling: the same device bodies
 * on virtual blocks separated by grid-wide barriers (bitwise ssm_advance).
 * steps_dev: the same [n_steps] descriptors in device memory.  `events` is
 * ignored; SSM_ERR_UNSUPPORTED when the kernel cannot be co-resident. */
int ssm_advance_coop(ssm_advance_args* args, const ssm_step_desc* steps_dev, void* stream);
int ssm_event_create(void** out);
int ssm_event_destroy(void* event);
int ssm_event_elapsed_ms(void* start, void* end, float* ms);

/* Single filter sharded over W ranks (config 5).  Rank r holds
 * the P consecutive particles [rP, (r+1)P) of a P_global = W P filter and owns
 * the output slots of the same range.  Every rank maps every other rank's
 * position and ancestor arenas (CUDA IPC, ssm_ipc_open: NVLink peer memory),
 * so no particle state is ever exchanged through the host:
 *   pw:   ssm_propagate_weight with x_peer set gathers each ancestor from the
 *         rank that holds it (P2P loads at the rank boundaries) and writes the
 *         rank's LSE partial to lse_out -> all-gather (C1) -> ssm_lse_combine;
 *   1. ssm_tiles_total: this rank's fixed-point weight total -> all-gather (C1');
 *   2. ssm_offspring_push: the global offspring counts of the local particles
 *      (global query indices, offset = the lower ranks' totals) and the window
 *      fill, storing each ancestor (a global index) straight into the array of
 *      the rank that owns the output slot (P2P stores) -> rank barrier (C2);
 *   trajectory: ssm_tiles_total + all-gather, ssm_pick_sharded on every rank
 *      (the owner writes the global index, max over ranks), ssm_trace_peer walks
 *      the ancestry through the peer-mapped arenas.
 * Draws use global indices, so the result does not depend on the rank count
 * beyond the association of the LSE partials. */
size_t ssm_sharded_workspace_bytes(int B, int P, int P_global);
int ssm_tiles_total(int B, int P, const void* tile_rec, const ssm_filter_state* fs, uint64_t* total_out,
                    void* workspace, void* stream);
int ssm_offspring_push(int P, int P_global, int W, int rank, int scheme, const void* cdf_local,
                       const uint64_t* totals_all, const double* u, const uint32_t* keys, int step,
                       const ssm_filter_state* fs, int32_t* const* anc_tab, void* workspace, void* stream);
int ssm_pick_sharded(int P, int W, int rank, const void* cdf_local, const uint64_t* totals_all, const double* u,
                     int32_t* j_out, void* workspace, void* stream);
int ssm_trace_peer(int dtype, int S, int nx, int P, const void* const* x_tab, const int32_t* const* anc_tab,
                   const int32_t* has_anc, const int32_t* j_final, double* out, void* stream);
/* CUDA IPC: map a peer allocation (64-byte cudaIpcMemHandle_t from its owner)
 * into this process with lazy peer access; unmap. */
int ssm_ipc_open(const void* handle, void** ptr);
int ssm_ipc_close(void* ptr);

/* Persistent small-P filter (P <= ssm_small_max_particles()): one CTA per
 * filter runs all n_steps grid steps in ONE launch (device noise).  Same
 * semantics as ssm_advance; log-weights, CDF and ancestors stay in shared
 * memory; ancestors are written for every step (identity when not resampled). */
typedef struct ssm_small_args {
  int32_t model, dtype, B, P, scheme, exact, check_finite, n_steps;
  double log_w0, obs_log_sd, log_sqrt_2pi, ess_rel;
  const double* theta;         /* [B][4] */
  const uint32_t* keys;        /* [B][2] */
  ssm_filter_state* fs;        /* [B] */
  const ssm_substep* subs;     /* device sub-step table */
  const ssm_step_desc* steps;  /* DEVICE [n_steps] */
  const void* x_in;            /* [B][nx][P] */
  void* x_arena;               /* [n_steps][B][nx][P] */
  int32_t* anc_arena;          /* [n_steps][B][P] */
  const void* a_prev;          /* [B][P] or NULL */
  void* a_out;                 /* [B][P] final unnormalised log-weights, or NULL */
} ssm_small_args;

int ssm_small_max_particles(void);
int ssm_advance_small(const ssm_small_args* args, void* stream);

/* K6: ancestor gather x_out[b][s][k] = x_in[b][s][anc[b][k]] (particle.py:102). */
int ssm_gather(int dtype, int B, int nx, int P, const void* x_in, const int32_t* anc,
               void* x_out, void* stream);

/* Strided gather out[s][k] = x_in[s][idx[k]] (x_in rows of in_stride particles,
 * out rows of n_out): the cross-rank spill of the sharded filter. */
int ssm_gather_cols(int dtype, int nx, int n_out, int in_stride, const void* x_in, const int32_t* idx,
                    void* x_out, void* stream);

/* K8: ancestry trace (ParticleRun.sample_trajectory, particle.py:137-149).
 * xs[b*(S+1) + i] points at history position array x_i of filter b
 * ([nx][P] SoA), ancs[b*(S+1) + i] at the ancestors of step i (NULL =
 * identity; index 0 unused).  j_final[b] is the drawn final particle.
 * out: [B][S+1][nx] float64. */
/* sample_trajectory's final-weight pick (particle.py:140-141) from the tile
 * records of the last weighted ssm_propagate_weight: j_out[b] =
 * searchsorted(cum_b, u[b], 'right') clipped, cum from the exact fixed-point
 * CDF (same as ssm_resample_from_tiles); workspace = ssm_resample_workspace_bytes. */
/* Trajectory of history-free runs (device noise).  With counter-based noise a
 * particle's state at grid step i is a function of its ancestor's state at
 * i - 1, its slot j_i and step i only, so sample_trajectory's output
 * (particle.py:137-149) is recomputed along the chosen ancestry: walk j_S ->
 * j_0 through the stored ancestors, regenerate x_0[j_0] (ssm_init_particles'
 * draw or the fixed initial state), then apply each grid step's transition
 * with slot j_i's draws -- the fused kernel's own transition code, so the
 * result is bitwise the stored-history trajectory.  One thread per filter. */
typedef struct ssm_replay_args {
  int32_t model, dtype, B, P, S, exact;
  const double* theta;            /* [B][4] derived parameters (as ssm_pw_args.theta) */
  const ssm_substep* subs;        /* device sub-step table */
  const ssm_step_desc* steps;     /* device [S + 1]; entry i describes grid step i (i >= 1) */
  const uint32_t* keys;           /* device [B][S + 1][2]: Philox key of grid step i; entry 0 = init key */
  const double* x0;               /* device [B][nx]: fixed initial state rows (used where x0_flag[b]) */
  const int32_t* x0_flag;         /* device [B] or NULL: 1 = start from x0[b], 0 = init draw */
  const int32_t* const* ancs;     /* device [B][S + 1] ancestor rows of each step (NULL: identity) */
  const int32_t* j_final;         /* device [B]: picked final particle */
  double* out;                    /* device [B][S + 1][nx] */
} ssm_replay_args;
int ssm_replay_path(const ssm_replay_args* args, void* stream);

int ssm_pick_from_tiles(int B, int P, const void* cdf_local, const void* tile_rec, const ssm_filter_state* fs,
                        const double* u, int32_t* j_out, void* workspace, void* stream);
int ssm_trace(int dtype, int B, int S, int nx, int P, const void* const* xs,
              const int32_t* const* ancs, const int32_t* j_final, double* out, void* stream);

/* K3 standalone: scipy-1.18 logsumexp and ESS of B log-weight vectors
 * (particle.py:83-85, 127).  out_lse/out_ess: [B] float64. */
size_t ssm_lse_workspace_bytes(int B, int P);
int ssm_logsumexp(int dtype, int B, int P, const void* a, double* out_lse, double* out_ess,
                  void* workspace, void* stream);

/* K9: theta-block gather for SMC^2 theta-resampling (smc.py:96-98):
 * dst[j] = src[idx[j]] for J blocks of `block_bytes` bytes each. */
int ssm_block_gather(int J, size_t block_bytes, const void* src, const int32_t* idx, void* dst,
                     void* stream);

/* K10: theta-level marginal MH on the device for the hand-written models.
 * ssm_theta_propose replaces the proposal walk and its densities
 * (simulate.py:272-352 propose_parameters / proposal_parameter_logpdf / propose_initial /
 * proposal_initial_logpdf) and the prior of the proposal (simulate.py:220-233), as called
 * from mcmc.py:_propose (138-148).  ssm_theta_accept replaces the accept step
 * (mcmc.py:28-33, 155-164): accepted chains copy theta_new / x0_new / loglik_new /
 * log_prior_new into the current state in place.  One thread per chain.
 * Draws: device Philox keyed by keys[c] and `step` (u_in == NULL), or injected
 * reference draws: u_in [C][u_stride] standard uniforms (truncated-Gaussian statements in
 * block order, then proposal_initial slots), g_in [C] the numpy gamma(2, 1/scale) variate
 * of the inverse-gamma statement, u_acc_in [C] the accept uniform.  u_stride must be
 * ssm_theta_draws(model, has_init).  *err is set to 1 when a distribution parameter is
 * invalid (DistributionParameterError on the host). */
typedef struct {
  int32_t model;                 /* SSM_MODEL_LORENZ96 or SSM_MODEL_WINDKESSEL */
  int32_t n_chains;
  int32_t n_param;               /* 2 (L96) / 4 (WK) */
  int32_t nx;                    /* 8 / 1 */
  int32_t has_init;              /* L96 proposal_initial: chains carry x0 */
  int32_t u_stride;
  uint64_t step;                 /* device-draw counter word (MH step index) */
  const uint32_t* keys;          /* device [C][2] Philox keys of the chain streams */
  double* theta;                 /* device [C][n_param] current (updated by accept) */
  double* x0;                    /* device [C][nx] current initial state or NULL */
  double* theta_new;             /* device [C][n_param] */
  double* x0_new;                /* device [C][nx] or NULL */
  double* logq_fwd;              /* device [C] */
  double* logq_rev;              /* device [C] */
  double* log_prior_new;         /* device [C] parameter_logpdf (+ initial_logpdf) of the proposal */
  double* loglik;                /* device [C] current loglik (accept) */
  double* log_prior;             /* device [C] current log prior (accept) */
  const double* loglik_new;      /* device [C] filter loglik at the proposal (-inf: not run) */
  int32_t* accepted;             /* device [C] */
  int32_t* err;                  /* device [1] */
  const double* u_in;            /* injected draws or NULL */
  const double* g_in;
  const double* u_acc_in;
} ssm_theta_args;
/* K11: batched Kalman filter for linear-Gaussian models, replacing the
 * forward pass of KalmanRun (kalman.py:53-96) for B systems per launch (one thread each).
 * The system of filter f comes from lineargauss.extract_linear_gaussian (lineargauss.py:292-316)
 * in the form x_s = A x_{s-1} + b + N(0, Q), y_s = H x_s + c + N(0, diag(r_sd^2)).
 * Records: entry 0 of mu / P is the initial state (input); entries s0+1..s1 are written
 * (filtered moments in mu / P, predicted in mu_p / P_p).  err[f] = first step whose
 * innovation covariance is not positive definite (CholeskyError on the host). */
typedef struct {
  int32_t B, nx, ny, S;          /* S = grid steps in the tables */
  int32_t s0, s1;                /* advance over steps s0+1..s1 */
  const double* A;               /* [B][S][nx][nx] */
  const double* b;               /* [B][S][nx] */
  const double* Q;               /* [B][S][nx][nx] */
  const double* H;               /* [B][S][ny][nx] */
  const double* c;               /* [B][S][ny] */
  const double* r_sd;            /* [B][S][ny] */
  const double* y;               /* [S][ny] */
  const uint8_t* mask;           /* [S][ny] present slots */
  double* mu;                    /* [B][S+1][nx] */
  double* P;                     /* [B][S+1][nx][nx] */
  double* mu_p;                  /* [B][S+1][nx] */
  double* P_p;                   /* [B][S+1][nx][nx] */
  double* loglik;                /* [B] accumulated in place */
  int32_t* err;                  /* [B] */
} ssm_kalman_args;
int ssm_kalman_max_dim(void);
int ssm_kalman_filter(const ssm_kalman_args* args, void* stream);

/* Backward smoothing draws (KalmanRun.sample_trajectory, kalman.py:98-114) of
 * G runs on the device, one thread per run, from the records of
 * ssm_kalman_filter: rows[g] selects the batch row, s the run position, z the
 * reference's standard normals [G][s+1][nx] (row q = the draw for step s-q,
 * drawn on the host from each run's stream in the reference's order); out
 * [G][s+1][nx].  Covariance-form algebra with the reference's PSD pivot rule;
 * err[g] = failing grid index + 1 (CholeskyError), else untouched. */
typedef struct ssm_kalman_sample_args {
  int32_t G, nx, S, s;
  const int32_t* rows;
  const double *A, *mu, *P, *mu_p, *P_p; /* batch records, as ssm_kalman_args */
  const double* z;
  double* out;
  int32_t* err;
} ssm_kalman_sample_args;
int ssm_kalman_sample(const ssm_kalman_sample_args* args, void* stream);
/* Host helper: numpy SeedSequence(entropy).generate_state(n_words, uint32) for
 * n streams (the RngStream key derivation, rng.py:16-34) -- entropy [n][L]
 * 32-bit words (run entropy padded to 4 words, then the spawn key), out
 * [n][n_words].  Bit-exact with numpy; no device work. */
int ssm_seedseq_state(int n, int L, const uint32_t* entropy, int n_words, uint32_t* out);
int ssm_theta_draws(int model, int has_init);
int ssm_theta_propose(const ssm_theta_args* args, void* stream);
int ssm_theta_accept(const ssm_theta_args* args, void* stream);
/* The theta-level proposal of a GENERATED model (model = SSM_MODEL_GENERIC, handle from
 * ssm_gen_compile): the walk of proposal_parameter (else parameter) and, with has_init,
 * of proposal_initial (else initial) plus the initial block's assigns, both proposal
 * log-densities and parameter_logpdf + initial_logpdf of the proposal (simulate.py:219-352,
 * in GenericModel.propose_batch / mcmc._propose order, mcmc.py:138-148), one thread per
 * chain.  u_in rows carry the reference's standard variates by draw index (uniform of a
 * uniform / truncated-Gaussian statement, standard normal of a Gaussian, standard gamma
 * of a gamma / inverse-gamma), the accept uniform last; g_in is unused.  u_stride must be
 * ssm_gen_theta_draws(handle, has_init).  ssm_theta_accept takes the same args. */
int ssm_gen_theta_draws(const void* handle, int has_init);
int ssm_gen_theta_propose(const void* handle, const ssm_theta_args* args, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SSM_B200_H */
