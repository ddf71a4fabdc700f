// kernels.hpp -- host launchers of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "collsim_b200.h"

namespace csb {

void pack(const cs_copy_entry* entries, int n, int src_dt, int dst_dt, cudaStream_t s);
void sum_buffers(const void* const* in, int m, void* const* out, int nout, uint64_t n, int dt,
                 cudaStream_t s);
void sgd_update(const cs_update_entry* entries, int n, int w_dt, int g_dt, double lr,
                double rescale, double momentum, cudaStream_t s);
void synth_backward(const void* src, void* dst, uint64_t n, int dt, uint64_t spin_ns, int ctas,
                    cudaStream_t s);
void checksum(const void* x, uint64_t n, int dt, double* out, cudaStream_t s);

// A kernel table kept resident in HBM for repeated launches over the same
// keys (a KvStore bucket): the launch passes a pointer instead of a
// parameter block of up to 21 KB, and the table is re-uploaded only when an
// entry changes (stream-ordered cudaMallocAsync / copy / cudaFreeAsync, so
// earlier launches on the same stream keep reading the old copy).  Every
// launch through one DeviceTable must use the same stream.
class DeviceTable {
 public:
  DeviceTable() = default;
  ~DeviceTable();
  DeviceTable(const DeviceTable&) = delete;
  DeviceTable& operator=(const DeviceTable&) = delete;
  void pack(const cs_copy_entry* es, int n, int src_dt, int dst_dt, cudaStream_t s);
  void sgd(const cs_update_entry* es, int n, int w_dt, int g_dt, double lr, double rescale,
           double momentum, cudaStream_t s);
  // Kernel (a) fused with kernel (c) when the collective between them is the
  // identity (one rank): every entry's gradient (g_dt) is staged into its
  // comm-bucket slot (c_dt, the copy of kvstore.cpp:109) and, from the same
  // registers, the weights are updated with the staged value -- one pass
  // instead of a pack launch plus an update launch that re-reads the bucket.
  // es[i]: g = gradient, mom, w = weights, bucket = the key's comm slot
  // (may equal g: an in-place bucket view, nothing to stage).
  struct PackUpdate {
    const void* g;
    void* bucket;
    void* w;
    void* mom;
    uint64_t n;
  };
  static bool pack_sgd_supported(int g_dt, int c_dt, int w_dt);
  void pack_sgd(const std::vector<PackUpdate>& es, int g_dt, int c_dt, int w_dt, double lr, double rescale,
                double momentum, cudaStream_t s);
  uint64_t uploads() const { return uploads_; }

  struct Entry {  // 56 B; a/b/c/d per kernel: pack a=src c=dst; sgd a=g b=mom c=w;
                  // pack_sgd a=g b=mom c=w d=comm-bucket slot
    const void* a;
    const void* b;
    void* c;
    uint64_t n;
    uint64_t gstart, gend;
    void* d = nullptr;
  };
  // Keeps `es` resident (uploading on change) and returns the device copy.
  const Entry* resident(const std::vector<Entry>& es, cudaStream_t s);

 private:
  void sync(uint64_t chunk_groups, cudaStream_t s);
  std::vector<Entry> host_;
  std::vector<uint32_t> first_;  // first entry of every chunk (+ the last entry)
  std::vector<uint8_t> vec_;
  uint64_t groups_ = 0;
  int grid_ = 0;
  void* dev_ = nullptr;
  int dev_device_ = -1;
  std::vector<unsigned char> shadow_;  // what dev_ holds
  std::vector<Entry> last_host_;       // entries / flags / chunk of the last sync
  std::vector<uint8_t> last_vec_;
  uint64_t chunk_ = ~0ull;
  uint64_t uploads_ = 0;
};

// Fused allreduce (+ SGD) over NVLink peer memory (kernels.cu): `bufs` /
// `flags` hold every rank's bucket base and flag region (UVA / IPC-mapped),
// `tab` the update entries in bucket-group coordinates (gstart = slot offset
// / 8), sorted; nullptr / update=false reduces only.
struct P2PArgs {
  void* bufs[CS_MAX_RANKS];
  uint32_t* flags[CS_MAX_RANKS];
  void* mc = nullptr;  // NVLS multicast VA of the bucket: in-switch reduction instead of peer loads
  int nranks = 0, rank = 0;
  uint64_t count = 0;  // bucket elements, multiple of 8
  int cdt = CS_F32, wdt = CS_F32;
  uint32_t epoch = 0;  // identical on every rank for the same op (ledger seq + 1)
  const DeviceTable::Entry* tab = nullptr;
  int n_entries = 0;
  bool update = false;
  bool shard_only = false;  // phase 1 stores only the own shard; the update reads the owners' buckets
  // stage the gradients (entry d, the comm dtype) into this rank's bucket
  // slots (entry a) inside the kernel, before barrier 0 (kernel (a) folded in)
  bool pack = false;
  // ZeRO-1: master-weight shards of every rank and this rank's momentum shard
  // (shard-local layout, p2p_shard_elems each); weights all-gathered after the update
  bool zero = false;
  void* wm[CS_MAX_RANKS] = {};
  void* mom_b = nullptr;
  // direct: phase 1 reads every rank's gradients in place (entry d = this
  // rank's copy; rank r's = gbase[r] + (d - gbase[rank])) -- registered
  // regions with the same layout on every rank; nothing is staged
  bool direct = false;
  void* gbase[CS_MAX_RANKS] = {};
  double lr = 0, rescale = 0, momentum = 0;
  // every rank's grid on the SAME device (local peer transport): cap each
  // grid so all `nranks` grids are co-resident, plain (non-cooperative) launch
  bool colocated = false;
  // peer launches that may run at the same time on this device (ConCom's
  // communicators): every grid is capped to 1/concurrent of the device's
  // resident CTAs and launched plainly, so all of them can be resident at
  // once on every GPU whatever order they start in -- none can hold the SMs
  // a peer-waiting grid of another communicator needs
  int concurrent = 1;
  // host-mapped abort word (device address): [0] code, [1..3] where.  The
  // pair barriers poll it while waiting and give up (no __trap) once it is
  // set, or set it themselves after `timeout_ns` without the peer.
  uint32_t* abort_word = nullptr;
  uint64_t timeout_ns = 0;
  // CSB_P2P_TRACE: per-CTA phase stamps of this launch (device address of
  // kP2PMaxCtas x 5 host-mapped uint64), null = off
  uint64_t* stamps = nullptr;
};
// Abort codes in abort_word[0]
enum : uint32_t { kAbortNone = 0, kAbortHost = 1, kAbortDeviceTimeout = 2 };
size_t p2p_flag_bytes();
// elements of the largest shard of a `count`-element bucket (a multiple of 8)
uint64_t p2p_shard_elems(uint64_t count, int nranks);
int p2p_grid(uint64_t groups, int nranks, bool colocated = false, int concurrent = 1);
void p2p_allreduce(const P2PArgs& args, cudaStream_t s);
// CSB_P2P_TIMEOUT_MS (default 30000): a pair barrier waiting longer than this
// for a peer CTA records kAbortDeviceTimeout and the kernel returns
uint64_t p2p_timeout_ns();

// Launch accounting and optional per-launch CUDA-event timing (roofline).
enum KernelKind {
  kKernPack = 0, kKernSum = 1, kKernSgd = 2, kKernSynth = 3, kKernChecksum = 4, kKernPackSgd = 5, kKernKinds = 6
};
struct KernelStats {
  uint64_t launches = 0;
  double total_ms = 0.0;  // summed CUDA-event durations (profiling on only)
  double bytes = 0.0;     // algorithmic bytes moved by those launches
};
uint64_t launch_count();
void profile_enable(bool on);
KernelStats profile_collect(int kind);  // synchronizes pending timing events
void profile_reset();

}  // namespace csb
