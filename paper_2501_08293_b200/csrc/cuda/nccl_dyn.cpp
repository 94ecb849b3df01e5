// Run-time binding of NCCL (nccl_dyn.hpp).
#include "nccl_dyn.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

namespace dopf::cuda::nccl {

namespace {

struct Loaded {
  Api api{};
  std::string where, error;
  int version = 0;
  bool ok = false;
};

template <typename F>
bool bind(void* h, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  return fn != nullptr;
}

Loaded load() {
  Loaded L;
  void* h = nullptr;
  if (const char* env = std::getenv("DOPF_NCCL_SO"); env && *env) {
    h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    L.where = env;
  }
  if (!h) {  // an NCCL this process already holds (e.g. PyTorch's)
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    L.where = "libnccl.so.2 (already loaded)";
  }
  if (!h) {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    L.where = "libnccl.so.2";
  }
  if (!h) {
    const char* e = dlerror();
    L.error = std::string("NCCL not available: ") + (e ? e : "dlopen(libnccl.so.2) failed");
    return L;
  }
  Api& a = L.api;
  const bool ok = bind(h, "ncclGetVersion", a.GetVersion) && bind(h, "ncclGetUniqueId", a.GetUniqueId) &&
                  bind(h, "ncclCommInitRank", a.CommInitRank) && bind(h, "ncclCommInitAll", a.CommInitAll) &&
                  bind(h, "ncclCommDestroy", a.CommDestroy) && bind(h, "ncclCommAbort", a.CommAbort) &&
                  bind(h, "ncclCommGetAsyncError", a.CommGetAsyncError) && bind(h, "ncclAllGather", a.AllGather) &&
                  bind(h, "ncclAllReduce", a.AllReduce) && bind(h, "ncclGetErrorString", a.GetErrorString);
  if (!ok) {
    L.error = "NCCL at " + L.where + " lacks a required symbol";
    return L;
  }
  a.GetVersion(&L.version);
  L.ok = true;
  return L;
}

const Loaded& loaded() {
  static std::once_flag once;
  static Loaded L;
  std::call_once(once, [] { L = load(); });
  return L;
}

}  // namespace

const Api& api() {
  const Loaded& L = loaded();
  if (!L.ok) throw NcclFailure(L.error);
  return L.api;
}

std::string describe() {
  const Loaded& L = loaded();
  return L.ok ? L.where + " version " + std::to_string(L.version) : L.error;
}

void check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  throw NcclFailure(std::string(what) + ": " + api().GetErrorString(r));
}

}  // namespace dopf::cuda::nccl
