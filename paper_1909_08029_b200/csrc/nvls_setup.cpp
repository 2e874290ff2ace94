// Multicast objects for the NVLS P-Reduce (nvls.cu).
//
// The paper caches one NCCL communicator per group (at most 64). On an NVSwitch
// node the analog is a multicast object per GPU subset: created once, its handle shared
// with the other GPUs of the subset as a POSIX file descriptor, every GPU binds its own
// physical memory to it and maps both the multicast address (stores and reductions that
// the switch fans out / combines) and its own copy (unicast address).
//
// One process per GPU: the creator of a subset's object is its lowest GPU; the descriptor
// travels over a Unix-domain socket (SCM_RIGHTS) in the abstract namespace, named after
// the creator's pid (exchanged by rp_peer_export / rp_peer_import). Phases, separated by
// the caller's collective barrier:
//   1  creators: cuMulticastCreate, export the descriptor, listen
//   2  members connect; creators accept and send; members import; every member
//      cuMulticastAddDevice(own device)
//   3  every member: cuMemCreate on its GPU, cuMulticastBindMem, map uc + mc, zero flags
// Driver entry points are resolved through cudaGetDriverEntryPoint (no link-time libcuda).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rp_internal.h"

namespace rp {

namespace {

struct Drv {
  PFN_cuDeviceGetAttribute_v2000 DeviceGetAttribute = nullptr;
  PFN_cuDeviceGet_v2000 DeviceGet = nullptr;
  PFN_cuMulticastCreate_v12010 MulticastCreate = nullptr;
  PFN_cuMulticastGetGranularity_v12010 MulticastGetGranularity = nullptr;
  PFN_cuMulticastAddDevice_v12010 MulticastAddDevice = nullptr;
  PFN_cuMulticastBindMem_v12010 MulticastBindMem = nullptr;
  PFN_cuMulticastUnbind_v12010 MulticastUnbind = nullptr;
  PFN_cuMemCreate_v10020 MemCreate = nullptr;
  PFN_cuMemRelease_v10020 MemRelease = nullptr;
  PFN_cuMemAddressReserve_v10020 MemAddressReserve = nullptr;
  PFN_cuMemAddressFree_v10020 MemAddressFree = nullptr;
  PFN_cuMemMap_v10020 MemMap = nullptr;
  PFN_cuMemUnmap_v10020 MemUnmap = nullptr;
  PFN_cuMemSetAccess_v10020 MemSetAccess = nullptr;
  PFN_cuMemExportToShareableHandle_v10020 MemExportToShareableHandle = nullptr;
  PFN_cuMemImportFromShareableHandle_v10020 MemImportFromShareableHandle = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 MemGetAllocationGranularity = nullptr;
  bool ok = false;
};

template <typename F>
bool resolve(const char* name, F* fn) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || !f) return false;
  *fn = reinterpret_cast<F>(f);
  return true;
}

const Drv& drv() {
  static Drv d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    d.ok = resolve("cuDeviceGetAttribute", &d.DeviceGetAttribute) && resolve("cuDeviceGet", &d.DeviceGet) &&
           resolve("cuMulticastCreate", &d.MulticastCreate) &&
           resolve("cuMulticastGetGranularity", &d.MulticastGetGranularity) &&
           resolve("cuMulticastAddDevice", &d.MulticastAddDevice) &&
           resolve("cuMulticastBindMem", &d.MulticastBindMem) && resolve("cuMulticastUnbind", &d.MulticastUnbind) &&
           resolve("cuMemCreate", &d.MemCreate) && resolve("cuMemRelease", &d.MemRelease) &&
           resolve("cuMemAddressReserve", &d.MemAddressReserve) && resolve("cuMemAddressFree", &d.MemAddressFree) &&
           resolve("cuMemMap", &d.MemMap) && resolve("cuMemUnmap", &d.MemUnmap) &&
           resolve("cuMemSetAccess", &d.MemSetAccess) &&
           resolve("cuMemExportToShareableHandle", &d.MemExportToShareableHandle) &&
           resolve("cuMemImportFromShareableHandle", &d.MemImportFromShareableHandle) &&
           resolve("cuMemGetAllocationGranularity", &d.MemGetAllocationGranularity);
  }
  return d;
}

std::string cu_str(CUresult r) { return "CUresult " + std::to_string(static_cast<int>(r)); }

#define CU_TRY(expr, what)                                          \
  do {                                                              \
    const CUresult _r = (expr);                                     \
    if (_r != CUDA_SUCCESS) {                                       \
      *err = std::string(what) + ": " + cu_str(_r);                 \
      return RP_ECUDA;                                              \
    }                                                               \
  } while (0)

int popcount(uint32_t m) { return __builtin_popcount(m); }

// abstract-namespace socket name of (creator pid, subset)
void sock_addr(int pid, uint32_t mask, sockaddr_un* a, socklen_t* len) {
  std::memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  const std::string name = "rp-nvls-" + std::to_string(pid) + "-" + std::to_string(mask);
  std::memcpy(a->sun_path + 1, name.data(), name.size());  // sun_path[0] = 0: abstract
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + name.size());
}

int send_fd(int sock, int fd) {
  char byte = 'f';
  iovec iov{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctrl;
  msg.msg_controllen = sizeof(ctrl);
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  cm->cmsg_level = SOL_SOCKET;
  cm->cmsg_type = SCM_RIGHTS;
  cm->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(cm), &fd, sizeof(int));
  return sendmsg(sock, &msg, 0) == 1 ? 0 : -1;
}

int recv_fd(int sock) {
  char byte = 0;
  iovec iov{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr msg{};
  msg.msg_iov = &iov;
  msg.msg_iovlen = 1;
  msg.msg_control = ctrl;
  msg.msg_controllen = sizeof(ctrl);
  if (recvmsg(sock, &msg, 0) != 1) return -1;
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  if (!cm || cm->cmsg_type != SCM_RIGHTS) return -1;
  int fd = -1;
  std::memcpy(&fd, CMSG_DATA(cm), sizeof(int));
  return fd;
}

struct Pending {
  NvlsObj obj;
  int listen_fd = -1;  // creator
  int share_fd = -1;   // exported / received descriptor
  int conn_fd = -1;    // member's connection to the creator
};

void close_fd(int* fd) {
  if (*fd >= 0) close(*fd);
  *fd = -1;
}

}  // namespace

int nvls_supported(int device, int* out) {
  *out = 0;
  const Drv& d = drv();
  if (!d.ok) return RP_OK;
  CUdevice dev;
  if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return RP_OK;
  int v = 0;
  if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return RP_OK;
  *out = v ? 1 : 0;
  return RP_OK;
}

NvlsObj* nvls_find(NvlsState* s, uint32_t mask) {
  for (auto& o : s->objs)
    if (o.mask == mask) return &o;
  return nullptr;
}

void nvls_teardown(NvlsState* s) {
  const Drv& d = drv();
  if (!d.ok) return;
  for (auto& o : s->objs) {
    if (o.mc_va) {
      d.MemUnmap(o.mc_va, o.size);
      d.MemAddressFree(o.mc_va, o.size);
    }
    if (o.uc_va) {
      d.MemUnmap(o.uc_va, o.size);
      d.MemAddressFree(o.uc_va, o.size);
    }
    if (o.mc_handle && o.mem_handle) {
      CUdevice dev;
      int cur = 0;
      cudaGetDevice(&cur);
      if (d.DeviceGet(&dev, cur) == CUDA_SUCCESS) d.MulticastUnbind(o.mc_handle, dev, 0, o.size);
    }
    if (o.mem_handle) d.MemRelease(o.mem_handle);
    if (o.mc_handle) d.MemRelease(o.mc_handle);
  }
  s->objs.clear();
  s->min_gpus = 0;
}

int nvls_setup(NvlsState* s, int rank, int n_gpus, int device, int wpg, int64_t n, int min_gpus,
               const int32_t* peer_pids, rp_barrier_fn barrier, void* user, std::string* err) {
  const Drv& d = drv();
  if (!d.ok) {
    *err = "nvls: driver multicast entry points unavailable";
    return RP_ENODEV;
  }
  CUdevice dev;
  CU_TRY(d.DeviceGet(&dev, device), "cuDeviceGet");
  // geometry shared by every object
  const int64_t CH = nvls_chunk_f4();
  const int64_t n4 = n / 4;
  const int64_t nch = std::max<int64_t>(1, (n4 + CH - 1) / CH);
  const int64_t data_bytes = (n * 4 + 255) / 256 * 256;
  const int64_t slot_bytes = (data_bytes + nch * kNvlsFlagStride * 8 + 255) / 256 * 256;
  std::vector<Pending> mine;  // subsets containing this GPU
  for (uint32_t mask = 1; mask < (1u << n_gpus); ++mask) {
    if (popcount(mask) < min_gpus || !((mask >> rank) & 1)) continue;
    Pending p;
    p.obj.mask = mask;
    p.obj.kp = popcount(mask);
    p.obj.me = popcount(mask & ((1u << rank) - 1));
    p.obj.slots = wpg;
    p.obj.slot_bytes = slot_bytes;
    p.obj.data_bytes = data_bytes;
    p.obj.nch = nch;
    p.obj.CH = CH;
    mine.push_back(p);
  }
  int rc = RP_OK;
  auto cleanup = [&]() {
    for (auto& p : mine) {
      close_fd(&p.listen_fd);
      close_fd(&p.share_fd);
      close_fd(&p.conn_fd);
    }
  };
  // ---- phase 1: creators create, export and listen
  for (auto& p : mine) {
    if (rc != RP_OK) break;
    if (__builtin_ctz(p.obj.mask) != rank) continue;
    CUmulticastObjectProp prop{};
    prop.numDevices = static_cast<unsigned int>(p.obj.kp);
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = static_cast<size_t>(slot_bytes) * p.obj.slots;
    size_t gran = 0;
    CUresult r = d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM);
    if (r != CUDA_SUCCESS) {
      *err = "cuMulticastGetGranularity: " + cu_str(r);
      rc = RP_ECUDA;
      break;
    }
    prop.size = (prop.size + gran - 1) / gran * gran;
    CUmemGenericAllocationHandle h;
    if ((r = d.MulticastCreate(&h, &prop)) != CUDA_SUCCESS) {
      *err = "cuMulticastCreate: " + cu_str(r);
      rc = RP_ECUDA;
      break;
    }
    p.obj.mc_handle = h;
    p.obj.size = prop.size;
    int fd = -1;
    if ((r = d.MemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS) {
      *err = "cuMemExportToShareableHandle: " + cu_str(r);
      rc = RP_ECUDA;
      break;
    }
    p.share_fd = fd;
    p.listen_fd = socket(AF_UNIX, SOCK_STREAM, 0);
    sockaddr_un a;
    socklen_t len;
    sock_addr(static_cast<int>(getpid()), p.obj.mask, &a, &len);
    if (p.listen_fd < 0 || bind(p.listen_fd, reinterpret_cast<sockaddr*>(&a), len) != 0 ||
        listen(p.listen_fd, 16) != 0) {
      *err = "nvls: cannot listen on the descriptor socket";
      rc = RP_ECUDA;
      break;
    }
  }
  // every rank reaches every barrier, errors included (the others would hang)
  if (barrier(user, rc) != 0 && rc == RP_OK) {
    *err = "nvls: another rank failed (phase 1)";
    rc = RP_ECUDA;
  }
  // ---- phase 2: members connect (never blocks: the creator listens with a backlog),
  // creators accept + send, members receive + import, everyone adds its device
  if (rc == RP_OK) {
    for (auto& p : mine) {
      const int creator = __builtin_ctz(p.obj.mask);
      if (creator == rank) continue;
      p.conn_fd = socket(AF_UNIX, SOCK_STREAM, 0);
      sockaddr_un a;
      socklen_t len;
      sock_addr(peer_pids[creator], p.obj.mask, &a, &len);
      bool ok = false;
      for (int t = 0; t < 2000 && p.conn_fd >= 0; ++t) {
        if (connect(p.conn_fd, reinterpret_cast<sockaddr*>(&a), len) == 0) {
          ok = true;
          break;
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(5));
      }
      if (!ok) {
        *err = "nvls: cannot connect to the creator of GPU subset " + std::to_string(p.obj.mask);
        rc = RP_ECUDA;
        break;
      }
    }
  }
  if (rc == RP_OK) {
    for (auto& p : mine) {
      if (__builtin_ctz(p.obj.mask) != rank) continue;
      for (int i = 1; i < p.obj.kp; ++i) {
        const int cfd = accept(p.listen_fd, nullptr, nullptr);
        if (cfd < 0 || send_fd(cfd, p.share_fd) != 0) {
          if (cfd >= 0) close(cfd);
          *err = "nvls: cannot hand the multicast descriptor to a member";
          rc = RP_ECUDA;
          break;
        }
        close(cfd);
      }
      if (rc != RP_OK) break;
    }
  }
  if (rc == RP_OK) {
    for (auto& p : mine) {
      if (__builtin_ctz(p.obj.mask) == rank) continue;
      p.share_fd = recv_fd(p.conn_fd);
      if (p.share_fd < 0) {
        *err = "nvls: no multicast descriptor received";
        rc = RP_ECUDA;
        break;
      }
      CUmemGenericAllocationHandle h;
      const CUresult r = d.MemImportFromShareableHandle(
          &h, reinterpret_cast<void*>(static_cast<uintptr_t>(p.share_fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      if (r != CUDA_SUCCESS) {
        *err = "cuMemImportFromShareableHandle: " + cu_str(r);
        rc = RP_ECUDA;
        break;
      }
      p.obj.mc_handle = h;
      CUmulticastObjectProp prop{};
      prop.numDevices = static_cast<unsigned int>(p.obj.kp);
      prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      prop.size = static_cast<size_t>(slot_bytes) * p.obj.slots;
      size_t gran = 0;
      if (d.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) {
        *err = "cuMulticastGetGranularity";
        rc = RP_ECUDA;
        break;
      }
      p.obj.size = (prop.size + gran - 1) / gran * gran;
    }
  }
  if (rc == RP_OK) {
    for (auto& p : mine) {
      const CUresult r = d.MulticastAddDevice(p.obj.mc_handle, dev);
      if (r != CUDA_SUCCESS) {
        *err = "cuMulticastAddDevice: " + cu_str(r);
        rc = RP_ECUDA;
        break;
      }
    }
  }
  if (barrier(user, rc) != 0 && rc == RP_OK) {
    *err = "nvls: another rank failed (phase 2)";
    rc = RP_ECUDA;
  }
  // ---- phase 3: bind physical memory on this GPU, map multicast + unicast, zero
  if (rc == RP_OK) {
    for (auto& p : mine) {
      CUmemAllocationProp ap{};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = device;
      ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      CUmemGenericAllocationHandle mh;
      CUresult r = d.MemCreate(&mh, p.obj.size, &ap, 0);
      if (r != CUDA_SUCCESS) {
        *err = "cuMemCreate (" + std::to_string(p.obj.size) + " bytes): " + cu_str(r);
        rc = r == CUDA_ERROR_OUT_OF_MEMORY ? RP_ENOMEM : RP_ECUDA;
        break;
      }
      p.obj.mem_handle = mh;
      if ((r = d.MulticastBindMem(p.obj.mc_handle, 0, mh, 0, p.obj.size, 0)) != CUDA_SUCCESS) {
        *err = "cuMulticastBindMem: " + cu_str(r);
        rc = RP_ECUDA;
        break;
      }
      CUmemAccessDesc ad{};
      ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ad.location.id = device;
      ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      CUdeviceptr uc = 0, mc = 0;
      if ((r = d.MemAddressReserve(&uc, p.obj.size, 0, 0, 0)) != CUDA_SUCCESS ||
          (r = d.MemMap(uc, p.obj.size, 0, mh, 0)) != CUDA_SUCCESS ||
          (r = d.MemSetAccess(uc, p.obj.size, &ad, 1)) != CUDA_SUCCESS) {
        *err = "nvls unicast mapping: " + cu_str(r);
        rc = RP_ECUDA;
        break;
      }
      p.obj.uc_va = uc;
      if ((r = d.MemAddressReserve(&mc, p.obj.size, 0, 0, 0)) != CUDA_SUCCESS ||
          (r = d.MemMap(mc, p.obj.size, 0, p.obj.mc_handle, 0)) != CUDA_SUCCESS ||
          (r = d.MemSetAccess(mc, p.obj.size, &ad, 1)) != CUDA_SUCCESS) {
        *err = "nvls multicast mapping: " + cu_str(r);
        rc = RP_ECUDA;
        break;
      }
      p.obj.mc_va = mc;
      const cudaError_t e = cudaMemset(reinterpret_cast<void*>(uc), 0, p.obj.size);
      if (e != cudaSuccess) {
        *err = std::string("nvls: zeroing the slots: ") + cudaGetErrorString(e);
        rc = RP_ECUDA;
        break;
      }
    }
    if (rc == RP_OK && cudaDeviceSynchronize() != cudaSuccess) {
      *err = "nvls: device synchronize after setup";
      rc = RP_ECUDA;
    }
  }
  if (barrier(user, rc) != 0 && rc == RP_OK) {
    *err = "nvls: another rank failed (phase 3)";
    rc = RP_ECUDA;
  }
  cleanup();
  for (auto& p : mine) s->objs.push_back(p.obj);
  if (rc != RP_OK) {
    nvls_teardown(s);
    return rc;
  }
  s->min_gpus = min_gpus;
  return RP_OK;
}

}  // namespace rp
