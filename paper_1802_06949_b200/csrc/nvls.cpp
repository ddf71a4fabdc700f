// nvls.cpp -- see nvls.hpp.
#include "nvls.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <thread>

#include "common.hpp"
#include "ledger.hpp"

namespace csb {

namespace {

template <typename F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
  CSB_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  if (!p || q != cudaDriverEntryPointSuccess) throw CudaError(std::string("driver entry point missing: ") + name);
  return reinterpret_cast<F>(p);
}

struct Driver {
  decltype(&cuDeviceGet) deviceGet;
  decltype(&cuDeviceGetAttribute) deviceGetAttribute;
  decltype(&cuGetErrorString) getErrorString;
  decltype(&cuMulticastCreate) mcCreate;
  decltype(&cuMulticastAddDevice) mcAddDevice;
  decltype(&cuMulticastBindMem) mcBindMem;
  decltype(&cuMulticastUnbind) mcUnbind;
  decltype(&cuMulticastGetGranularity) mcGetGranularity;
  decltype(&cuMemCreate) memCreate;
  decltype(&cuMemRelease) memRelease;
  decltype(&cuMemGetAllocationGranularity) memGetAllocationGranularity;
  decltype(&cuMemExportToShareableHandle) memExport;
  decltype(&cuMemImportFromShareableHandle) memImport;
  decltype(&cuMemAddressReserve) addressReserve;
  decltype(&cuMemAddressFree) addressFree;
  decltype(&cuMemMap) memMap;
  decltype(&cuMemUnmap) memUnmap;
  decltype(&cuMemSetAccess) memSetAccess;
};

const Driver& drv() {
  static const Driver d = [] {
    Driver x;
    x.deviceGet = entry<decltype(x.deviceGet)>("cuDeviceGet");
    x.deviceGetAttribute = entry<decltype(x.deviceGetAttribute)>("cuDeviceGetAttribute");
    x.getErrorString = entry<decltype(x.getErrorString)>("cuGetErrorString");
    x.mcCreate = entry<decltype(x.mcCreate)>("cuMulticastCreate");
    x.mcAddDevice = entry<decltype(x.mcAddDevice)>("cuMulticastAddDevice");
    x.mcBindMem = entry<decltype(x.mcBindMem)>("cuMulticastBindMem");
    x.mcUnbind = entry<decltype(x.mcUnbind)>("cuMulticastUnbind");
    x.mcGetGranularity = entry<decltype(x.mcGetGranularity)>("cuMulticastGetGranularity");
    x.memCreate = entry<decltype(x.memCreate)>("cuMemCreate");
    x.memRelease = entry<decltype(x.memRelease)>("cuMemRelease");
    x.memGetAllocationGranularity = entry<decltype(x.memGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    x.memExport = entry<decltype(x.memExport)>("cuMemExportToShareableHandle");
    x.memImport = entry<decltype(x.memImport)>("cuMemImportFromShareableHandle");
    x.addressReserve = entry<decltype(x.addressReserve)>("cuMemAddressReserve");
    x.addressFree = entry<decltype(x.addressFree)>("cuMemAddressFree");
    x.memMap = entry<decltype(x.memMap)>("cuMemMap");
    x.memUnmap = entry<decltype(x.memUnmap)>("cuMemUnmap");
    x.memSetAccess = entry<decltype(x.memSetAccess)>("cuMemSetAccess");
    return x;
  }();
  return d;
}

void cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  drv().getErrorString(r, &s);
  throw CudaError(std::string(what) + ": " + (s ? s : "unknown driver error"));
}

sockaddr_un abstract_addr(const std::string& name, socklen_t* len) {
  sockaddr_un a{};
  a.sun_family = AF_UNIX;
  const std::string n = name.substr(0, sizeof(a.sun_path) - 2);
  a.sun_path[0] = '\0';  // abstract namespace: nothing on disk
  std::memcpy(a.sun_path + 1, n.data(), n.size());
  *len = static_cast<socklen_t>(offsetof(sockaddr_un, sun_path) + 1 + n.size());
  return a;
}

void send_fd(int sock, int fd) {
  char byte = 'x';
  iovec io{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  c->cmsg_level = SOL_SOCKET;
  c->cmsg_type = SCM_RIGHTS;
  c->cmsg_len = CMSG_LEN(sizeof(int));
  std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
  if (sendmsg(sock, &m, 0) != 1) throw ConfigError("nvls: sendmsg(SCM_RIGHTS) failed");
}

int recv_fd(int sock) {
  char byte = 0;
  iovec io{&byte, 1};
  char ctrl[CMSG_SPACE(sizeof(int))] = {};
  msghdr m{};
  m.msg_iov = &io;
  m.msg_iovlen = 1;
  m.msg_control = ctrl;
  m.msg_controllen = sizeof(ctrl);
  if (recvmsg(sock, &m, 0) != 1) throw ConfigError("nvls: recvmsg(SCM_RIGHTS) failed");
  cmsghdr* c = CMSG_FIRSTHDR(&m);
  if (!c || c->cmsg_type != SCM_RIGHTS) throw ConfigError("nvls: no descriptor received");
  int fd = -1;
  std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
  return fd;
}

void ledger_barrier(Ledger& L, int slot, int rank, int nranks) {
  const int32_t one = 1;
  L.post_rank_blob(slot, rank, &one, sizeof(one));
  for (int r = 0; r < nranks; ++r) {
    int32_t v = 0;
    L.read_rank_blob(slot, r, &v, sizeof(v));
  }
}

}  // namespace

bool nvls_device_supported(int device) {
  try {
    CUdevice dev;
    cu(drv().deviceGet(&dev, device), "cuDeviceGet");
    int v = 0;
    cu(drv().deviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev), "cuDeviceGetAttribute");
    return v != 0;
  } catch (...) {
    return false;
  }
}

NvlsBuffer nvls_alloc(Ledger& L, int rank, int nranks, int device, size_t bytes, const std::string& tag,
                      int slot) {
  const Driver& d = drv();
  CSB_CUDA(cudaSetDevice(device));
  CSB_CUDA(cudaFree(nullptr));  // primary context current
  CUdevice dev;
  cu(d.deviceGet(&dev, device), "cuDeviceGet");

  CUmulticastObjectProp mp{};
  mp.numDevices = static_cast<unsigned>(nranks);
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t mgran = 0, agran = 0;
  cu(d.mcGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // multicast-bindable
  cu(d.memGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED),
     "cuMemGetAllocationGranularity");
  const size_t gran = std::max(mgran, agran);
  const size_t size = (bytes + gran - 1) / gran * gran;
  mp.size = size;

  NvlsBuffer b;
  b.bytes = size;
  b.device = device;
  CUmemGenericAllocationHandle mc = 0;
  const std::string sock_name = "csb-nvls-" + tag + "-" + std::to_string(slot);
  if (rank == 0) {
    cu(d.mcCreate(&mc, &mp), "cuMulticastCreate");
    int fd = -1;
    cu(d.memExport(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
    int s = socket(AF_UNIX, SOCK_STREAM, 0);
    socklen_t len = 0;
    sockaddr_un a = abstract_addr(sock_name, &len);
    if (s < 0 || bind(s, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(s, nranks) != 0)
      throw ConfigError("nvls: cannot listen on abstract socket " + sock_name);
    for (int i = 1; i < nranks; ++i) {
      int c = accept(s, nullptr, nullptr);
      if (c < 0) throw ConfigError("nvls: accept failed");
      send_fd(c, fd);
      close(c);
    }
    close(s);
    close(fd);
  } else {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::seconds(120);
    int fd = -1;
    for (;;) {
      int s = socket(AF_UNIX, SOCK_STREAM, 0);
      socklen_t len = 0;
      sockaddr_un a = abstract_addr(sock_name, &len);
      if (s >= 0 && connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0) {
        fd = recv_fd(s);
        close(s);
        break;
      }
      if (s >= 0) close(s);
      if (std::chrono::steady_clock::now() > deadline) throw DeadlockTimeout("nvls: rank 0 never served " + sock_name);
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    cu(d.memImport(&mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
       "cuMemImportFromShareableHandle");
    close(fd);
  }
  cu(d.mcAddDevice(mc, dev), "cuMulticastAddDevice");
  ledger_barrier(L, slot, rank, nranks);  // every device added before any bind

  CUmemGenericAllocationHandle mem = 0;
  cu(d.memCreate(&mem, size, &ap, 0), "cuMemCreate");
  cu(d.mcBindMem(mc, 0, mem, 0, size, 0), "cuMulticastBindMem");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc = 0, mcva = 0;
  cu(d.addressReserve(&uc, size, gran, 0, 0), "cuMemAddressReserve");
  cu(d.memMap(uc, size, 0, mem, 0), "cuMemMap");
  cu(d.memSetAccess(uc, size, &acc, 1), "cuMemSetAccess");
  cu(d.addressReserve(&mcva, size, gran, 0, 0), "cuMemAddressReserve(mc)");
  cu(d.memMap(mcva, size, 0, mc, 0), "cuMemMap(mc)");
  cu(d.memSetAccess(mcva, size, &acc, 1), "cuMemSetAccess(mc)");
  CSB_CUDA(cudaMemset(reinterpret_cast<void*>(uc), 0, size));
  CSB_CUDA(cudaDeviceSynchronize());
  ledger_barrier(L, slot + 1, rank, nranks);  // every rank bound before any multicast access

  b.uc = reinterpret_cast<void*>(uc);
  b.mc = reinterpret_cast<void*>(mcva);
  b.mc_handle = mc;
  b.mem_handle = mem;
  return b;
}

void nvls_free(NvlsBuffer& b) {
  if (!b.uc) return;
  const Driver& d = drv();
  cudaSetDevice(b.device);
  cudaDeviceSynchronize();
  CUdevice dev;
  d.deviceGet(&dev, b.device);
  d.memUnmap(reinterpret_cast<CUdeviceptr>(b.mc), b.bytes);
  d.addressFree(reinterpret_cast<CUdeviceptr>(b.mc), b.bytes);
  d.memUnmap(reinterpret_cast<CUdeviceptr>(b.uc), b.bytes);
  d.addressFree(reinterpret_cast<CUdeviceptr>(b.uc), b.bytes);
  d.mcUnbind(b.mc_handle, dev, 0, b.bytes);
  d.memRelease(b.mem_handle);
  d.memRelease(b.mc_handle);
  b = NvlsBuffer{};
}

}  // namespace csb
