// transport.hpp -- collectives over device memory.
//
// Reference interface: R/core/include/collsim/collective.hpp:36-61
// (Transport{num_ranks, world, new_communicator, allreduce_sum, broadcast,
// barrier, set_inject_latency}).  Every call first goes through the matching
// Ledger (issue order, signature, watchdog, latch); only a matched call
// touches the device, stream-ordered on the caller's stream:
//
//   Backend::Local  in-process rank threads (one GPU or several, UVA peers).
//                   The last arriver waits on every rank's ready event and
//                   runs kernel (b) over all R buffers in fixed rank order,
//                   writing the sum to every buffer -- the reference's
//                   "last arriver reduces" (collective.cpp:228-243) on HBM,
//                   bit-identical to it.  The others make their stream wait
//                   on the reducer's done event.  With `peer` (create_local
//                   (..., true)) the rank threads instead run the fused
//                   peer-memory kernels on each other's buffers (plain device
//                   pointers, every rank's grid capped so all R grids are
//                   co-resident on one GPU): the same kernels, barriers and
//                   epochs as across GPUs, testable on one device.
//   Backend::Nccl   one process per GPU; ledger in POSIX shm; data over NCCL
//                   (NVLink 5 / NVSwitch).  One ncclComm_t per communicator
//                   (world + ConCom's extra communicators, ncclCommSplit).
//   Backend::LedgerOnly  matching only (CPU tests of the host logic).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "ledger.hpp"
#include "nvls.hpp"

namespace csb {

class Transport {
 public:
  enum class Backend { Local, Nccl, LedgerOnly };

  static std::unique_ptr<Transport> create_local(int nranks, std::chrono::milliseconds watchdog,
                                                 TraceSink* trace, bool peer = false);
  static std::unique_ptr<Transport> create_nccl(const std::string& name, int nranks, int rank,
                                                int device, std::chrono::milliseconds watchdog,
                                                TraceSink* trace);
  static std::unique_ptr<Transport> create_ledger_only(const std::string& name, int nranks,
                                                       int rank, std::chrono::milliseconds watchdog,
                                                       TraceSink* trace);
  ~Transport();

  int num_ranks() const { return ledger_->num_ranks(); }
  static constexpr int world() { return 0; }
  Backend backend() const { return backend_; }
  int local_rank() const { return rank_; }

  int new_communicator();
  int num_communicators() const { return ledger_->num_communicators(); }

  void allreduce_sum(int comm, int rank, void* buf, uint64_t count, int dtype, int trace_key,
                     cudaStream_t stream, int bucket = -1);
  void broadcast(int comm, int rank, int root, void* buf, uint64_t count, int dtype,
                 int trace_key, cudaStream_t stream);
  void barrier(int comm, int rank, int trace_key, cudaStream_t stream);

  void set_inject_latency(std::chrono::microseconds us);
  std::chrono::microseconds inject_latency() const;
  void abort(const std::string& why);
  Ledger& ledger() { return *ledger_; }

  // ---- peer-memory path (one process per GPU, NVLink) --------------------
  // True for the NCCL backend with >= 2 ranks on peer-capable devices, and
  // for a local transport created with `peer` (>= 2 rank threads).
  bool p2p_capable() const {
    return num_ranks() > 1 && ((backend_ == Backend::Nccl && p2p_ok_) || (backend_ == Backend::Local && local_peer_));
  }
  bool colocated() const { return backend_ == Backend::Local; }
  // Setup-phase collective: every rank passes the base of one cudaMalloc
  // allocation, in the same order; returns every rank's mapping of its peer
  // (CUDA IPC handles exchanged through the ledger; local peer mode: the
  // rank threads' pointers), own entry = base.  `rank` is required for the
  // local transport (one object serves every rank thread).
  std::vector<void*> share_buffer(void* base, int rank = -1);
  // Closes this rank's mappings of the peers' buffers returned by
  // share_buffer (before the owner of `ptrs` frees its own buffer, so the
  // same addresses can be shared again later).
  void unshare_buffer(const std::vector<void*>& ptrs);
  // Device abort word of the peer kernels (host-mapped): 0 while healthy;
  // set by abort() / the engine watchdog, or by a kernel whose pair barrier
  // timed out.  Returns the failure description when one was recorded.
  std::string device_failure() const;
  // device_failure(), or an NCCL asynchronous error (ncclCommGetAsyncError)
  std::string async_failure();
  struct P2PUpdate {
    const DeviceTable::Entry* tab = nullptr;  // bucket-group coordinates, sorted
    int n_entries = 0;
    bool update = true;  // false: a plain allreduce (the table only locates direct-read gradients)
    int wdt = CS_F32;
    double lr = 0, rescale = 0, momentum = 0;
    bool shard_only = false;  // the bucket keeps only this rank's shard (update reads owners)
    bool pack = false;        // entries' d = gradients: the kernel stages them first (kernel (a) folded in)
    const void* const* wm = nullptr;  // ZeRO-1: every rank's master shard; null = replicated update
    void* mom_b = nullptr;            // ZeRO-1: this rank's momentum shard
    // direct gradient reads: every rank's registered gradient region (entries'
    // d = this rank's gradients inside it); `layout` hashes the (key, offset)
    // list, matched across ranks like the rest of the signature
    const void* const* gbase = nullptr;
    uint64_t layout = 0;
  };
  // Allreduce of one bucket through peer memory, matched by the ledger like
  // allreduce_sum; with `upd`, fused with the SGD / momentum update of the
  // keys in the bucket (kernels.cu p2p_allreduce_kernel).
  // `concurrent`: peer launches of other communicators that may run at the
  // same time on this device (ConCom), see P2PArgs::concurrent.
  void allreduce_p2p(int comm, int rank, void* const* peer_bufs, uint64_t count, int dtype,
                     int trace_key, cudaStream_t stream, int bucket, const P2PUpdate* upd,
                     void* mc = nullptr, int concurrent = 1);
  // CSB_P2P_TRACE=1: the last peer launch's per-CTA phase stamps of `rank`
  // (%globaltimer ns; CTA-major, 5 per CTA: start, past barrier 0, own shard
  // done, past barrier 1, end); empty when tracing is off.
  std::vector<uint64_t> p2p_stamps(int rank) const;
  // NVLink SHARP: every rank's device supports multicast objects.
  bool nvls_capable() const { return p2p_capable() && nvls_ok_; }
  // Setup-phase collective: a multicast-bound allocation (nvls.hpp).
  NvlsBuffer alloc_nvls(size_t bytes);

 private:
  Transport() = default;
  struct SlotDev;  // per (comm, ring slot) payload of the local backend
  void run(int comm, int rank, const CallSig& sig, void* buf, int trace_key, cudaStream_t stream,
           int bucket);
  void local_data(const Ledger::Ticket& t, const CallSig& sig, void* buf, cudaStream_t stream);
  void nccl_data(int comm, const CallSig& sig, void* buf, cudaStream_t stream);
  void device_latency(cudaStream_t stream);

  Backend backend_ = Backend::LedgerOnly;
  int rank_ = -1;
  int device_ = -1;
  std::unique_ptr<Ledger> ledger_;
  std::vector<ncclComm_t> comms_;  // nccl: index = communicator id
  std::vector<std::unique_ptr<SlotDev>> slots_;  // local: comm * kLedgerSlots + slot
  std::mutex mu_;
  // peer-memory path
  void setup_flags();  // one flag region per communicator, shared
  void ensure_local_flags(int comm);  // local peer mode: R regions per communicator
  void setup_abort();
  void serialize_launch(int comm, int rank, cudaStream_t s, bool after);
  void wait_colocated(int comm, int rank);
  bool local_peer_ = false;
  std::vector<int> local_share_next_;  // local peer mode: next mailbox slot per rank
  int flags_device_ = -1;
  struct LaunchOrder {
    cudaStream_t stream = nullptr;
    cudaEvent_t ev = nullptr;
    int dev = -1;
  };
  std::vector<LaunchOrder> launch_order_;  // comm * kLedgerMaxRanks + rank
  uint32_t* abort_host_ = nullptr;         // [0] abort code, [1..3] where (host-mapped)
  uint32_t* abort_dev_ = nullptr;
  // CSB_P2P_TRACE=1: per-rank phase stamps of the last peer launch (host-mapped)
  uint64_t* stamps_host_ = nullptr;
  uint64_t* stamps_dev_ = nullptr;
  int watch_id_ = -1;
  bool p2p_ok_ = false;
  bool nvls_ok_ = false;
  std::string name_;
  int share_slots_ = 0;
  std::vector<std::pair<void*, void*>> ipc_opened_;  // (opened allocation base, pointer handed out)
  std::vector<void*> own_flags_;
  std::vector<std::vector<void*>> flags_;  // comm -> every rank's flag region
};

}  // namespace csb
