// cusolver_dyn.hpp -- cuSOLVER resolved at run time (dlopen), for the deterministic baselines
// only (t_hosvd / st_hosvd / hooi, tucker.cpp:242-316: SVDs of full unfoldings, off the
// randomized hot path).  The randomized algorithms never load it.
#pragma once
#include <cusolverDn.h>
#include <dlfcn.h>

#include <mutex>
#include <stdexcept>
#include <string>

namespace lmra_host {

struct CusolverApi {
  decltype(&cusolverDnCreate) Create = nullptr;
  decltype(&cusolverDnDestroy) Destroy = nullptr;
  decltype(&cusolverDnSetStream) SetStream = nullptr;
  decltype(&cusolverDnDgeqrf_bufferSize) Dgeqrf_bufferSize = nullptr;
  decltype(&cusolverDnDgeqrf) Dgeqrf = nullptr;
  decltype(&cusolverDnDgesvd_bufferSize) Dgesvd_bufferSize = nullptr;
  decltype(&cusolverDnDgesvd) Dgesvd = nullptr;
  cusolverStatus_t (*SetDeterministicMode)(cusolverDnHandle_t, cusolverDeterministicMode_t) = nullptr;
};

inline const CusolverApi& cusolver() {
  static CusolverApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libcusolver: ") + dlerror();
      return;
    }
#define LMRA_CUSOLVER_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    LMRA_CUSOLVER_SYM(Create, "cusolverDnCreate");
    LMRA_CUSOLVER_SYM(Destroy, "cusolverDnDestroy");
    LMRA_CUSOLVER_SYM(SetStream, "cusolverDnSetStream");
    LMRA_CUSOLVER_SYM(Dgeqrf_bufferSize, "cusolverDnDgeqrf_bufferSize");
    LMRA_CUSOLVER_SYM(Dgeqrf, "cusolverDnDgeqrf");
    LMRA_CUSOLVER_SYM(Dgesvd_bufferSize, "cusolverDnDgesvd_bufferSize");
    LMRA_CUSOLVER_SYM(Dgesvd, "cusolverDnDgesvd");
    LMRA_CUSOLVER_SYM(SetDeterministicMode, "cusolverDnSetDeterministicMode");
#undef LMRA_CUSOLVER_SYM
    if (!api.Create || !api.SetStream || !api.Dgeqrf || !api.Dgesvd || !api.Dgeqrf_bufferSize ||
        !api.Dgesvd_bufferSize)
      err = "libcusolver lacks required symbols";
  });
  if (!err.empty()) throw std::runtime_error(err);
  return api;
}

}  // namespace lmra_host
