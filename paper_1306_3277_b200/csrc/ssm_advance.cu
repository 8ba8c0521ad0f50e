// Native filter driver: the ParticleRun.advance_to host loop (particle.py:87-94)
// as one C-ABI call.  For every grid step it enqueues the resample kernels
// (when the previous step weighted) and the fused propagate/weight kernel on
// the caller's stream, with the same host-side state machine as
// paper_1306_3277_b200.inference.particle.advance_runs (device-noise mode).
// Nothing synchronises; the device state machine lives in ssm_filter_state.

#include "ssm_common.cuh"

extern "C" int ssm_advance(ssm_advance_args* A, void* stream) {
  if (!A || !A->steps || A->n_steps < 0 || !A->x_in || !A->x_arena || !A->anc_used) return SSM_ERR_INVALID_ARG;
  if (A->pw.noise != nullptr || !A->pw.keys) return SSM_ERR_INVALID_ARG;  // device noise only
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int B = A->pw.B, P = A->pw.P;
  const size_t esz = A->pw.dtype == SSM_F64 ? 8 : 4;
  const int nx = A->pw.model == SSM_MODEL_GENERIC ? ssm_gen_nx(A->pw.gen)
                 : (A->pw.model == SSM_MODEL_LORENZ96 ? 8 : 1);
  if (nx <= 0) return SSM_ERR_INVALID_ARG;
  const size_t xstep = static_cast<size_t>(B) * nx * P * esz;
  const size_t astep = static_cast<size_t>(B) * P * esz;
  const size_t ancstep = static_cast<size_t>(B) * P;
  const void* x_prev = A->x_in;
  const void* a_last = A->a_prev;
  int maybe = A->maybe_nonuniform;
  int slot = 0;
  A->a_last_index = -1;
  // On the tile path without an ESS gate every weighted step is resampled from
  // its tile records, so the unnormalised log-weights of a weighted step are read
  // again only when it is the call's LAST weighted step (ParticleRun.logw / ess,
  // a resumed advance): the others are not written (8 B / particle / step less).
  int last_obs = -1;
  for (int k = 0; k < A->n_steps; ++k)
    if (A->steps[k].has_obs) last_obs = k;
  const bool skip_a = A->tiles && !A->ess_gate;
  int n_resample = 0;  // fused resample: look-back state parity
  cudaEvent_t* ev = reinterpret_cast<cudaEvent_t*>(const_cast<void**>(A->events));
  for (int k = 0; k < A->n_steps; ++k) {
    const ssm_step_desc& d = A->steps[k];
    int32_t* anc = nullptr;
    if (maybe) {
      anc = A->anc_arena + static_cast<size_t>(k) * ancstep;
      A->anc_used[k] = 1;
      if (ev && ev[4 * k + 0]) cudaEventRecord(ev[4 * k + 0], s);
      int st;
      if (A->tiles) {
        st = ssm_resample_tiles_step(B, P, A->scheme, A->cdf_local, A->tile_rec, A->pw.fs, nullptr, A->pw.keys,
                                     d.step, anc, A->resample_ws, n_resample & 1, n_resample == 0, stream);
        ++n_resample;
      } else {
        st = ssm_resample_from_logw(B, P, A->pw.dtype, A->scheme, a_last, nullptr, A->pw.fs, nullptr,
                                    A->pw.keys, d.step, anc, A->resample_ws, stream);
      }
      if (ev && ev[4 * k + 1]) cudaEventRecord(ev[4 * k + 1], s);
      if (st != SSM_OK) return st;
    } else {
      A->anc_used[k] = 0;
    }
    ssm_pw_args pw = A->pw;
    pw.step = d.step;
    pw.n_sub = d.n_sub;
    pw.hints = static_cast<uint32_t>(d.hints);
    pw.subs = A->subs_table + d.subs_offset;
    pw.x_in = x_prev;
    const int slot_x = A->x_ring > 0 ? k % A->x_ring : k;
    void* x_out = static_cast<char*>(A->x_arena) + static_cast<size_t>(slot_x) * xstep;
    pw.x_out = x_out;
    pw.anc = anc;
    pw.a_prev = a_last;
    pw.has_obs = d.has_obs;
    pw.obs_mask = d.obs_mask;
    for (int n = 0; n < 8; ++n) pw.y[n] = d.y[n];
    pw.u_obs = d.u_obs;
    pw.y_vec = (A->y_table && d.y_off >= 0) ? A->y_table + d.y_off : nullptr;
    pw.u_vec = (A->u_table && d.u_off >= 0) ? A->u_table + d.u_off : nullptr;
    void* a_out = nullptr;
    const int a_slot = A->a_ring > 0 ? slot % A->a_ring : slot;
    if (d.has_obs && !(skip_a && k != last_obs)) a_out = static_cast<char*>(A->a_arena) + static_cast<size_t>(a_slot) * astep;
    pw.a_out = a_out;
    pw.cdf_local = (A->tiles && d.has_obs) ? A->cdf_local : nullptr;
    pw.tile_rec = (A->tiles && d.has_obs) ? A->tile_rec : nullptr;
    if (ev && ev[4 * k + 2]) cudaEventRecord(ev[4 * k + 2], s);
    const int st = ssm_propagate_weight(&pw, stream);
    if (ev && ev[4 * k + 3]) cudaEventRecord(ev[4 * k + 3], s);
    if (st != SSM_OK) return st;
    x_prev = x_out;
    if (d.has_obs) {
      a_last = a_out;
      A->a_last_index = a_slot;
      ++slot;
      maybe = 1;
    } else if (maybe && !A->ess_gate) {
      maybe = 0;  // resampled at this step and no new weights (particle.py:103-104)
    }
  }
  A->maybe_nonuniform = maybe;
  return SSM_OK;
}

extern "C" int ssm_event_create(void** out) {
  if (!out) return SSM_ERR_INVALID_ARG;
  cudaEvent_t e;
  const cudaError_t r = cudaEventCreate(&e);
  if (r != cudaSuccess) {
    ssm_set_last_error(r);
    return SSM_ERR_CUDA;
  }
  *out = e;
  return SSM_OK;
}

extern "C" int ssm_event_destroy(void* e) {
  return cudaEventDestroy(static_cast<cudaEvent_t>(e)) == cudaSuccess ? SSM_OK : SSM_ERR_CUDA;
}

extern "C" int ssm_event_elapsed_ms(void* start, void* end, float* ms) {
  if (!ms) return SSM_ERR_INVALID_ARG;
  const cudaError_t r = cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(end));
  if (r != cudaSuccess) {
    ssm_set_last_error(r);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}
