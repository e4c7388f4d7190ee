// NCCL loader and the in-place all-gather of the multi-GPU path (nccl_comm.hpp).
#include "nccl_comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <map>
#include <mutex>

#include "cltk_b200.hpp"

namespace cltk {
namespace b200 {

namespace {

struct Nccl {
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
  const char* (*errstr)(ncclResult_t) = nullptr;
  std::string why;
  int version = 0;
  bool ok = false;
};

Nccl loadNccl() {
  Nccl n;
  void* h = nullptr;
  // the copy torch already loaded (same soname) is reused; else the system one
  for (const char* name : {"libnccl.so.2", "libnccl.so", "/usr/lib/x86_64-linux-gnu/libnccl.so.2"}) {
    h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    n.why = "libnccl.so.2 not loadable";
    return n;
  }
  auto sym = [&](const char* s) { return dlsym(h, s); };
  n.commInitAll = reinterpret_cast<decltype(n.commInitAll)>(sym("ncclCommInitAll"));
  n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
  n.allGather = reinterpret_cast<decltype(n.allGather)>(sym("ncclAllGather"));
  n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
  n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
  n.getVersion = reinterpret_cast<decltype(n.getVersion)>(sym("ncclGetVersion"));
  n.errstr = reinterpret_cast<decltype(n.errstr)>(sym("ncclGetErrorString"));
  n.ok = n.commInitAll && n.commDestroy && n.allGather && n.groupStart && n.groupEnd &&
         n.getVersion && n.errstr;
  if (!n.ok) {
    n.why = "libnccl lacks the collective API";
    return n;
  }
  n.getVersion(&n.version);
  return n;
}

Nccl& nccl() {
  static Nccl n = loadNccl();
  return n;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw DeviceError(std::string("nccl: ") + what + ": " + nccl().errstr(r));
}

}  // namespace

struct NcclClique {
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;
};

bool ncclAvailable(std::string* info) {
  Nccl& n = nccl();
  if (info) *info = n.ok ? "nccl " + std::to_string(n.version) : n.why;
  return n.ok;
}

std::shared_ptr<NcclClique> ncclClique(const std::vector<int>& devices) {
  static std::mutex mu;
  // never destroyed: communicators live until the process exits (tearing them
  // down from a static destructor would race the CUDA runtime's own teardown)
  static auto& cache = *new std::map<std::vector<int>, std::shared_ptr<NcclClique>>();
  Nccl& n = nccl();
  if (!n.ok) throw UnsupportedError("multi-GPU: " + n.why);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(devices);
  if (it != cache.end()) return it->second;
  auto c = std::make_shared<NcclClique>();
  c->devices = devices;
  c->comms.assign(devices.size(), nullptr);
  int cur = 0;
  cudaGetDevice(&cur);
  nck(n.commInitAll(c->comms.data(), static_cast<int>(devices.size()), devices.data()),
      "ncclCommInitAll");
  cudaSetDevice(cur);
  cache.emplace(devices, c);
  return c;
}

void ncclAllGatherInPlace(NcclClique& c, const std::vector<double*>& bufs, size_t count,
                          const std::vector<cudaStream_t>& streams) {
  Nccl& n = nccl();
  int cur = 0;
  cudaGetDevice(&cur);
  nck(n.groupStart(), "ncclGroupStart");
  for (size_t g = 0; g < c.comms.size(); ++g) {
    cudaSetDevice(c.devices[g]);
    // in place: rank g's send buffer is its own slice of the receive buffer
    const ncclResult_t r = n.allGather(bufs[g] + g * count, bufs[g], count, ncclDouble,
                                       c.comms[g], streams[g]);
    if (r != ncclSuccess) {
      n.groupEnd();
      cudaSetDevice(cur);
      nck(r, "ncclAllGather");
    }
  }
  const ncclResult_t r = n.groupEnd();
  cudaSetDevice(cur);
  nck(r, "ncclGroupEnd");
}

}  // namespace b200
}  // namespace cltk
