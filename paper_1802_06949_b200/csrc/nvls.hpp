// nvls.hpp -- NVLink SHARP (NVSwitch multicast + in-switch reduction) buffers
// for the fused peer-memory collective.
//
// A multicast object spans the same-size physical allocation on every rank's
// GPU.  Through its multicast VA, `multimem.ld_reduce` returns the sum of all
// ranks' copies (the reduction runs in the NVSwitch) and `multimem.st`
// writes every rank's copy, so an allreduce moves ~(1 + 1/N) x the bucket
// per GPU per direction instead of ring's 2(N-1)/N.  Setup is a collective
// (one process per GPU): rank 0 creates the object and passes its POSIX file
// descriptor to the peers over an abstract Unix socket (SCM_RIGHTS); every
// rank adds its device, binds its own cuMemCreate allocation, maps a unicast
// and a multicast VA.  Driver entry points come from cudaGetDriverEntryPoint,
// so the library never links libcuda (it still loads on a GPU-less host).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

namespace csb {

class Ledger;

struct NvlsBuffer {
  void* uc = nullptr;  // this rank's copy (unicast VA)
  void* mc = nullptr;  // multicast VA (all ranks)
  size_t bytes = 0;
  // driver handles (opaque here)
  unsigned long long mc_handle = 0, mem_handle = 0;
  int device = -1;
};

// True when this device supports multicast objects (driver attribute).
bool nvls_device_supported(int device);
// Collective over `ledger` ranks; `tag` makes the socket name unique.
NvlsBuffer nvls_alloc(Ledger& ledger, int rank, int nranks, int device, size_t bytes,
                      const std::string& tag, int slot);
void nvls_free(NvlsBuffer& b);

}  // namespace csb
