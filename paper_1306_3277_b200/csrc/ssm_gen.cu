// Run-time compilation of generic models: the CUDA source
// that paper_1306_3277_b200/codegen.py generates from a reference ModelIr
// (a `gen::Model` + #include "ssm_gen_rt.cuh") is compiled for sm_100a with
// NVRTC, loaded with the runtime library API (cudaLibraryLoadData) and
// launched like the hand-written kernels (programmatic dependent launches on
// the caller's stream).  The handle owns the loaded library; no other state.

#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ssm_common.cuh"
#include "ssm_tile.cuh"

namespace {

// kernel instantiations, in handle order: pw[dtype][exact][injected], init[dtype]
const char* kPwNames[2][2][2] = {
    {{"ssm::gen_pw_kernel<gen::Model, float, false, false>", "ssm::gen_pw_kernel<gen::Model, float, false, true>"},
     {"ssm::gen_pw_kernel<gen::Model, float, true, false>", "ssm::gen_pw_kernel<gen::Model, float, true, true>"}},
    {{"ssm::gen_pw_kernel<gen::Model, double, false, false>", "ssm::gen_pw_kernel<gen::Model, double, false, true>"},
     {"ssm::gen_pw_kernel<gen::Model, double, true, false>", "ssm::gen_pw_kernel<gen::Model, double, true, true>"}}};
const char* kInitNames[2] = {"ssm::gen_init_kernel<gen::Model, float>", "ssm::gen_init_kernel<gen::Model, double>"};
const char* kInfoName = "ssm_gen_model_info";  // extern "C" __device__ int[2] = {NX, KDRAW}

struct GenModel {
  cudaLibrary_t lib;
  cudaKernel_t pw[2][2][2];
  cudaKernel_t init[2];
  int nx, kdraw;
};

void copy_log(const std::string& s, char* log, size_t log_len) {
  if (!log || log_len == 0) return;
  const size_t n = s.size() < log_len - 1 ? s.size() : log_len - 1;
  std::memcpy(log, s.data(), n);
  log[n] = '\0';
}

// NVRTC: source -> sm_100a cubin (+ lowered kernel names)
int compile(const char* source, const char* include_dir, std::vector<char>* cubin,
            std::vector<std::string>* lowered, char* log, size_t log_len) {
  if (!source || !include_dir) return SSM_ERR_INVALID_ARG;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source, "ssm_gen_model.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    return SSM_ERR_INVALID_ARG;
  std::vector<const char*> names;
  for (int t = 0; t < 2; ++t)
    for (int e = 0; e < 2; ++e)
      for (int i = 0; i < 2; ++i) names.push_back(kPwNames[t][e][i]);
  names.push_back(kInitNames[0]);
  names.push_back(kInitNames[1]);
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

}  // namespace

extern "C" int ssm_gen_check(const char* source, const char* include_dir, char* log, size_t log_len) {
  return compile(source, include_dir, nullptr, nullptr, log, log_len);
}

extern "C" int ssm_gen_compile(const char* source, const char* include_dir, void** out, char* log,
                               size_t log_len) {
  if (!out) return SSM_ERR_INVALID_ARG;
  *out = nullptr;
  std::vector<char> cubin;
  std::vector<std::string> low;
  const int st = compile(source, include_dir, &cubin, &low, log, log_len);
  if (st != SSM_OK) return st;
  cudaFree(nullptr);  // the primary context (the one torch uses) is current
  GenModel* g = new GenModel();
  cudaError_t e = cudaLibraryLoadData(&g->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) {
    delete g;
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  int k = 0;
  for (int t = 0; t < 2; ++t)
    for (int x = 0; x < 2; ++x)
      for (int i = 0; i < 2; ++i, ++k)
        if (e == cudaSuccess) e = cudaLibraryGetKernel(&g->pw[t][x][i], g->lib, low[k].c_str());
  for (int t = 0; t < 2; ++t, ++k)
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&g->init[t], g->lib, low[k].c_str());
  // model sizes from the module's ssm_gen_model_info (NX, KDRAW)
  int info[2] = {0, 0};
  if (e == cudaSuccess) {
    void* dptr = nullptr;
    size_t bytes = 0;
    e = cudaLibraryGetGlobal(&dptr, &bytes, g->lib, kInfoName);
    if (e == cudaSuccess && bytes >= sizeof(info)) e = cudaMemcpy(info, dptr, sizeof(info), cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) {
    cudaLibraryUnload(g->lib);
    delete g;
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  g->nx = info[0];
  g->kdraw = info[1];
  *out = g;
  return SSM_OK;
}

extern "C" int ssm_gen_destroy(void* handle) {
  if (!handle) return SSM_OK;
  GenModel* g = static_cast<GenModel*>(handle);
  cudaLibraryUnload(g->lib);
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
  const GenModel* g = static_cast<const GenModel*>(A.gen);
  if (!g || A.theta_stride <= 0) return SSM_ERR_INVALID_ARG;
  if (A.dtype != SSM_F64 && A.dtype != SSM_F32) return SSM_ERR_INVALID_ARG;
  const int t = A.dtype == SSM_F64 ? 1 : 0;
  cudaKernel_t k = g->pw[t][A.exact ? 1 : 0][A.noise ? 1 : 0];
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
  const GenModel* g = static_cast<const GenModel*>(handle);
  if (!g || B <= 0 || P <= 0 || B > 65535 || !keys || !theta || theta_stride <= 0 || !x_out)
    return SSM_ERR_INVALID_ARG;
  if (dtype != SSM_F64 && dtype != SSM_F32) return SSM_ERR_INVALID_ARG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ssm::pw_grid_x(P), B);
  cfg.blockDim = dim3(ssm::kPwThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  void* params[] = {&P, &p_offset, const_cast<uint32_t**>(&keys), const_cast<double**>(&theta), &theta_stride,
                    &x_out, &fs};
  const cudaError_t e =
      cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(g->init[dtype == SSM_F64 ? 1 : 0]), params);
  if (e != cudaSuccess) {
    ssm_set_last_error(e);
    return SSM_ERR_CUDA;
  }
  return SSM_OK;
}
