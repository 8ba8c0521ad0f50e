// Run-time compilation of generic models: the CUDA source
// that paper_1306_3277_b200/codegen.py generates from a reference ModelIr
// (a `gen::Model` + #include "ssm_gen_rt.cuh") is compiled for sm_100a with
// NVRTC, loaded with the runtime library API (cudaLibraryLoadData) and
// launched like the hand-written kernels (programmatic dependent launches on
// the caller's stream).  Each kernel variant (dtype x exact x injected noise,
// init) is compiled on first use; the handle owns the loaded libraries.

#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ssm_common.cuh"
#include "ssm_tile.cuh"

namespace {

// kernel instantiations: pw[dtype][exact][injected] = variant dtype * 4 + exact * 2 + injected,
// init[dtype] = variant 8 + dtype (dtype 0 float, 1 double), theta proposal = variant 10,
// SIMPLE pw (fast, device draws) = variant 11 + dtype
constexpr int kVariants = 13;
constexpr int kThetaVariant = 10;
constexpr int kSimpleVariant = 11;
const char* kVariantNames[kVariants] = {
    "ssm::gen_pw_kernel<gen::Model, float, false, false>",  "ssm::gen_pw_kernel<gen::Model, float, false, true>",
    "ssm::gen_pw_kernel<gen::Model, float, true, false>",   "ssm::gen_pw_kernel<gen::Model, float, true, true>",
    "ssm::gen_pw_kernel<gen::Model, double, false, false>", "ssm::gen_pw_kernel<gen::Model, double, false, true>",
    "ssm::gen_pw_kernel<gen::Model, double, true, false>",  "ssm::gen_pw_kernel<gen::Model, double, true, true>",
    "ssm::gen_init_kernel<gen::Model, float>",              "ssm::gen_init_kernel<gen::Model, double>",
    "ssm::gen_theta_propose_kernel<gen::Model>",
    "ssm::gen_pw_kernel<gen::Model, float, false, false, true>",
    "ssm::gen_pw_kernel<gen::Model, double, false, false, true>"};
const char* kInfoName = "ssm_gen_model_info";  // extern "C" __device__ int[4] = {NX, KDRAW, KP, KI}

// One handle per model: the source, and each kernel variant compiled (NVRTC)
// and loaded on first use, so a model pays only for the variants it runs.
struct GenModel {
  std::string src, inc;
  std::mutex mu;
  cudaLibrary_t lib[kVariants] = {};
  cudaKernel_t kernel[kVariants] = {};
  int nx = 0, kdraw = 0;
  int kp = 0, ki = 0;  // theta-level draws: parameter walk, initial walk
};

int pw_variant(int dtype, int exact, int injected) {
  return (dtype == SSM_F64 ? 4 : 0) + (exact ? 2 : 0) + (injected ? 1 : 0);
}

void copy_log(const std::string& s, char* log, size_t log_len) {
  if (!log || log_len == 0) return;
  const size_t n = s.size() < log_len - 1 ? s.size() : log_len - 1;
  std::memcpy(log, s.data(), n);
  log[n] = '\0';
}

// NVRTC: source -> sm_100a cubin for the given instantiations (+ their lowered names)
int compile(const char* source, const char* include_dir, const std::vector<const char*>& names,
            std::vector<char>* cubin, std::vector<std::string>* lowered, char* log, size_t log_len) {
  if (!source || !include_dir) return SSM_ERR_INVALID_ARG;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source, "ssm_gen_model.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return SSM_ERR_INVALID_ARG;
  for (const char* n : names) nvrtcAddNameExpression(prog, n);
  const std::string inc = std::string("--include-path=") + include_dir;
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device", "-lineinfo",
                        "--extra-device-vectorization", inc.c_str()};
  const nvrtcResult r = nvrtcCompileProgram(prog, sizeof(opts) / sizeof(opts[0]), opts);
  size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  std::string lg(ls, '\0');
  if (ls) nvrtcGetProgramLog(prog, &lg[0]);
  copy_log(lg, log, log_len);
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return SSM_ERR_INVALID_ARG;
  }
  if (cubin) {
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin->resize(n);
    nvrtcGetCUBIN(prog, cubin->data());
  }
  if (lowered) {
    for (const char* n : names) {
      const char* low = nullptr;
      nvrtcGetLoweredName(prog, n, &low);
      lowered->push_back(low ? low : "");
    }
  }
  nvrtcDestroyProgram(&prog);
  return SSM_OK;
}

// compile + load one variant (caller holds g->mu); also reads the model sizes
int load_variant(GenModel* g, int v, char* log, size_t log_len) {
  if (g->kernel[v]) return SSM_OK;
  std::vector<char> cubin;
  std::vector<std::string> low;
  const int st = compile(g->src.c_str(), g->inc.c_str(), {kVariantNames[v]}, &cubin, &low, log, log_len);
  if (st != SSM_OK) return st;
  cudaFree(nullptr);  // the primary context (the one torch uses) is current
  cudaLibrary_t lib;
  cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  cudaKernel_t k = nullptr;
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&k, lib, low[0].c_str());
  if (e == cudaSuccess && g->nx == 0) {  // model sizes from ssm_gen_model_info (NX, KDRAW, KP, KI)
    int info[4] = {0, 0, 0, 0};
    void* dptr = nullptr;
    size_t bytes = 0;
    e = cudaLibraryGetGlobal(&dptr, &bytes, lib, kInfoName);
    if (e == cudaSuccess && bytes >= sizeof(info)) e = cudaMemcpy(info, dptr, sizeof(info), cudaMemcpyDeviceToHost);
    g->nx = info[0];
    g->kdraw = info[1];
    g->kp = info[2];
    g->ki = info[3];
  }
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  g->lib[v] = lib;
  g->kernel[v] = k;
  return SSM_OK;
}

cudaKernel_t get_kernel(const void* handle, int v) {
  GenModel* g = static_cast<GenModel*>(const_cast<void*>(handle));
  std::lock_guard<std::mutex> lock(g->mu);
  return load_variant(g, v, nullptr, 0) == SSM_OK ? g->kernel[v] : nullptr;
}

}  // namespace

extern "C" int ssm_gen_check(const char* source, const char* include_dir, char* log, size_t log_len) {
  std::vector<const char*> all(kVariantNames, kVariantNames + kVariants);
  return compile(source, include_dir, all, nullptr, nullptr, log, log_len);
}

extern "C" int ssm_gen_compile(const char* source, const char* include_dir, void** out, char* log,
                               size_t log_len) {
  if (!out || !source || !include_dir) return SSM_ERR_INVALID_ARG;
  *out = nullptr;
  GenModel* g = new GenModel();
  g->src = source;
  g->inc = include_dir;
  // the filter's default variant (float64, FMA, device draws) now: reports compile
  // errors here and reads the model sizes; the others compile on first use
  int st;
  {
    std::lock_guard<std::mutex> lock(g->mu);
    st = load_variant(g, pw_variant(SSM_F64, 0, 0), log, log_len);
  }
  if (st != SSM_OK) {
    delete g;
    return st;
  }
  *out = g;
  return SSM_OK;
}

extern "C" int ssm_gen_destroy(void* handle) {
  if (!handle) return SSM_OK;
  GenModel* g = static_cast<GenModel*>(handle);
  for (int v = 0; v < kVariants; ++v)
    if (g->lib[v]) cudaLibraryUnload(g->lib[v]);
  delete g;
  return SSM_OK;
}

extern "C" int ssm_gen_info(const void* handle, int* n_state, int* n_draws) {
  if (!handle) return SSM_ERR_INVALID_ARG;
  const GenModel* g = static_cast<const GenModel*>(handle);
  if (n_state) *n_state = g->nx;
  if (n_draws) *n_draws = g->kdraw;
  return SSM_OK;
}

// called by ssm_propagate_weight for SSM_MODEL_GENERIC
int ssm_gen_propagate_weight(const ssm_pw_args& A, cudaStream_t s) {
  if (!A.gen || A.theta_stride <= 0) return SSM_ERR_INVALID_ARG;
  if (A.dtype != SSM_F64 && A.dtype != SSM_F32) return SSM_ERR_INVALID_ARG;
  const bool simple = (A.hints & SSM_HINT_SINGLE_SUBSTEP) && A.n_sub == 1 && !A.exact && A.noise == nullptr;
  cudaKernel_t k = get_kernel(A.gen, simple ? kSimpleVariant + (A.dtype == SSM_F64 ? 1 : 0)
                                            : pw_variant(A.dtype, A.exact, A.noise != nullptr));
  if (!k) return SSM_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ssm::pw_grid_x(A.P), A.B);
  cfg.blockDim = dim3(ssm::kPwThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  void* params[] = {const_cast<ssm_pw_args*>(&A)};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), params);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

int ssm_gen_nx(const void* handle) { return handle ? static_cast<const GenModel*>(handle)->nx : 0; }

extern "C" int ssm_gen_init_particles(const void* handle, int dtype, int B, int P, int p_offset,
                                      const uint32_t* keys, const double* theta, int theta_stride, void* x_out,
                                      ssm_filter_state* fs, void* stream) {
  if (!handle || B <= 0 || P <= 0 || B > 65535 || !keys || !theta || theta_stride <= 0 || !x_out)
    return SSM_ERR_INVALID_ARG;
  if (dtype != SSM_F64 && dtype != SSM_F32) return SSM_ERR_INVALID_ARG;
  cudaKernel_t k = get_kernel(handle, 8 + (dtype == SSM_F64 ? 1 : 0));
  if (!k) return SSM_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ssm::pw_grid_x(P), B);
  cfg.blockDim = dim3(ssm::kPwThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  void* params[] = {&P, &p_offset, const_cast<uint32_t**>(&keys), const_cast<double**>(&theta), &theta_stride,
                    &x_out, &fs};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), params);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}

extern "C" int ssm_gen_theta_draws(const void* handle, int has_init) {
  if (!handle) return -1;
  const GenModel* g = static_cast<const GenModel*>(handle);
  return g->kp + (has_init ? g->ki : 0) + 1;  // walk draws, then the accept uniform
}

extern "C" int ssm_gen_theta_propose(const void* handle, const ssm_theta_args* A, void* stream) {
  if (!handle || !A || A->model != SSM_MODEL_GENERIC || A->n_chains < 0) return SSM_ERR_INVALID_ARG;
  const GenModel* g = static_cast<const GenModel*>(handle);
  if (A->nx != g->nx || A->u_stride != ssm_gen_theta_draws(handle, A->has_init)) return SSM_ERR_INVALID_ARG;
  if (A->n_chains == 0) return SSM_OK;
  if (!A->theta || !A->theta_new || !A->logq_fwd || !A->logq_rev || !A->log_prior_new || !A->err)
    return SSM_ERR_INVALID_ARG;
  if (A->has_init && (!A->x0 || !A->x0_new)) return SSM_ERR_INVALID_ARG;
  if (!A->u_in && !A->keys) return SSM_ERR_INVALID_ARG;
  cudaKernel_t k = get_kernel(handle, kThetaVariant);
  if (!k) return SSM_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((A->n_chains + 127) / 128);
  cfg.blockDim = dim3(128);
  cfg.stream = static_cast<cudaStream_t>(stream);
  void* params[] = {const_cast<ssm_theta_args*>(A)};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), params);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}
