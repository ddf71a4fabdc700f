// transport.cpp -- see transport.hpp.
#include "transport.hpp"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "hostprof.hpp"
#include "kernels.hpp"
#include "watch.hpp"

namespace csb {

namespace {
constexpr size_t kStampsPerRank = 1184 * 5;  // kP2PMaxCtas x the peer kernels' phase stamps
}  // namespace

namespace {

[[noreturn]] void throw_nccl(ncclResult_t r, const char* what, ncclComm_t comm) {
  std::string msg = std::string(what) + ": " + ncclGetErrorString(r);
  const char* last = ncclGetLastError(comm);
  if (last && last[0]) msg += std::string(" (") + last + ")";
  throw NcclError(msg);
}

#define CSB_NCCL(call, comm)                                \
  do {                                                      \
    ncclResult_t csb_r_ = (call);                           \
    if (csb_r_ != ncclSuccess) throw_nccl(csb_r_, #call, comm); \
  } while (0)

ncclDataType_t nccl_type(int dt) {
  switch (dt) {
    case CS_F64: return ncclFloat64;
    case CS_F32: return ncclFloat32;
    case CS_BF16: return ncclBfloat16;
  }
  throw UsageError("collective: unknown dtype");
}

int current_device() {
  int d = 0;
  CSB_CUDA(cudaGetDevice(&d));
  return d;
}

// (Re)creates `ev` on the calling thread's device when needed.
void ensure_event(cudaEvent_t& ev, int& ev_dev) {
  const int d = current_device();
  if (ev && ev_dev == d) return;
  if (ev) {
    int prev = d;
    cudaSetDevice(ev_dev);
    cudaEventDestroy(ev);
    cudaSetDevice(prev);
  }
  CSB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  ev_dev = d;
}

}  // namespace

struct Transport::SlotDev {
  void* bufs[kLedgerMaxRanks] = {};
  cudaEvent_t ready[kLedgerMaxRanks] = {};
  int ready_dev[kLedgerMaxRanks] = {};
  cudaEvent_t done = nullptr;
  int done_dev = -1;
  ~SlotDev() {
    for (int r = 0; r < kLedgerMaxRanks; ++r)
      if (ready[r]) {
        cudaSetDevice(ready_dev[r]);
        cudaEventDestroy(ready[r]);
      }
    if (done) {
      cudaSetDevice(done_dev);
      cudaEventDestroy(done);
    }
  }
};

std::unique_ptr<Transport> Transport::create_local(int nranks, std::chrono::milliseconds watchdog,
                                                   TraceSink* trace, bool peer) {
  std::unique_ptr<Transport> t(new Transport());
  t->backend_ = Backend::Local;
  t->ledger_ = Ledger::create_local(nranks, watchdog, trace);
  t->slots_.resize(static_cast<size_t>(kLedgerMaxComms) * kLedgerSlots);
  t->local_peer_ = peer;
  t->local_share_next_.assign(static_cast<size_t>(nranks), 0);
  if (peer) t->setup_abort();
  return t;
}

std::unique_ptr<Transport> Transport::create_ledger_only(const std::string& name, int nranks,
                                                         int rank,
                                                         std::chrono::milliseconds watchdog,
                                                         TraceSink* trace) {
  std::unique_ptr<Transport> t(new Transport());
  t->backend_ = Backend::LedgerOnly;
  if (name.empty()) {
    t->ledger_ = Ledger::create_local(nranks, watchdog, trace);
  } else {
    t->ledger_ = Ledger::create_shm(name, nranks, rank, watchdog, trace);
    t->rank_ = rank;
  }
  return t;
}

std::unique_ptr<Transport> Transport::create_nccl(const std::string& name, int nranks, int rank,
                                                  int device, std::chrono::milliseconds watchdog,
                                                  TraceSink* trace) {
  std::unique_ptr<Transport> t(new Transport());
  t->backend_ = Backend::Nccl;
  t->rank_ = rank;
  t->device_ = device;
  t->ledger_ = Ledger::create_shm(name, nranks, rank, watchdog, trace);
  CSB_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  if (rank == 0) {
    CSB_NCCL(ncclGetUniqueId(&id), nullptr);
    t->ledger_->post_blob(0, &id, sizeof(id));
  } else {
    t->ledger_->read_blob(0, &id, sizeof(id));
  }
  ncclComm_t world = nullptr;
  CSB_NCCL(ncclCommInitRank(&world, nranks, id, rank), nullptr);
  t->comms_.push_back(world);
  if (nranks > 1) {
    int ndev = 0;
    CSB_CUDA(cudaGetDeviceCount(&ndev));
    bool ok = ndev >= nranks;
    for (int d = 0; ok && d < ndev; ++d) {
      if (d == device) continue;
      int can = 0;
      CSB_CUDA(cudaDeviceCanAccessPeer(&can, device, d));
      ok = ok && can;
    }
    // every rank must agree, or the shared setup below would not match
    const int32_t mine = (ok ? 1 : 0) | (nvls_device_supported(device) ? 2 : 0);
    t->ledger_->post_rank_blob(kLedgerRankBlobSlots - 1, rank, &mine, sizeof(mine));
    bool nvls = true;
    for (int r = 0; r < nranks; ++r) {
      int32_t v = 0;
      t->ledger_->read_rank_blob(kLedgerRankBlobSlots - 1, r, &v, sizeof(v));
      ok = ok && (v & 1);
      nvls = nvls && (v & 2);
    }
    t->p2p_ok_ = ok;
    t->nvls_ok_ = ok && nvls;
    t->name_ = name;
    if (ok) t->setup_flags();
  }
  t->setup_abort();
  return t;
}

// Host-mapped abort word of the peer kernels + registration with the
// process-wide watch (watch.hpp): the Engine's device waits poll it for
// asynchronous failures and abort every transport on a timeout.
void Transport::setup_abort() {
  CSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&abort_host_), 4 * sizeof(uint32_t),
                         cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(abort_host_, 0, 4 * sizeof(uint32_t));
  CSB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&abort_dev_), abort_host_, 0));
  if (const char* e = std::getenv("CSB_P2P_TRACE"); e && std::string(e) == "1") {
    const size_t bytes = sizeof(uint64_t) * kStampsPerRank * kLedgerMaxRanks;
    CSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stamps_host_), bytes, cudaHostAllocMapped));
    std::memset(stamps_host_, 0, bytes);
    CSB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&stamps_dev_), stamps_host_, 0));
  }
  watch_id_ = watch::add([this] { return async_failure(); }, [this](const std::string& why) { abort(why); });
}

std::string Transport::device_failure() const {
  if (!abort_host_) return {};
  const uint32_t code = reinterpret_cast<volatile uint32_t*>(abort_host_)[0];
  if (code != kAbortDeviceTimeout) return {};
  const volatile uint32_t* w = abort_host_;
  return "peer-memory kernel: rank " + std::to_string(w[1]) + " CTA " + std::to_string(w[3]) +
         " waited more than " + std::to_string(p2p_timeout_ns() / 1000000) + " ms at pair barrier phase " +
         std::to_string(w[2] & 0xff) + " for rank " + std::to_string(w[2] >> 8) +
         " (the peer never launched its half of the collective)";
}

std::string Transport::async_failure() {
  std::string m = device_failure();
  if (!m.empty()) return m;
  if (backend_ != Backend::Nccl) return {};
  std::lock_guard<std::mutex> lock(mu_);
  for (ncclComm_t c : comms_) {
    if (!c) continue;
    ncclResult_t r = ncclSuccess;
    if (ncclCommGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
      return std::string("NCCL asynchronous error: ") + ncclGetErrorString(r);
  }
  return {};
}

std::vector<void*> Transport::share_buffer(void* base, int rank) {
  if (!p2p_capable()) throw UsageError("Transport: peer-memory path needs the NCCL backend on peer-capable GPUs");
  if (backend_ == Backend::Local) {
    // rank threads of one process: exchange plain device pointers through
    // the ledger's per-rank mailbox (same call order on every rank thread)
    if (rank < 0 || rank >= num_ranks()) throw UsageError("Transport: share_buffer needs the caller's rank");
    int slot;
    {
      std::lock_guard<std::mutex> lock(mu_);
      slot = local_share_next_[static_cast<size_t>(rank)]++;
    }
    if (slot >= kLedgerRankBlobSlots) throw ConfigError("Transport: too many shared buffers");
    const uint64_t mine = reinterpret_cast<uintptr_t>(base);
    ledger_->post_rank_blob(slot, rank, &mine, sizeof(mine));
    std::vector<void*> ptrs(static_cast<size_t>(num_ranks()), nullptr);
    for (int r = 0; r < num_ranks(); ++r) {
      uint64_t v = 0;
      ledger_->read_rank_blob(slot, r, &v, sizeof(v));
      ptrs[static_cast<size_t>(r)] = reinterpret_cast<void*>(static_cast<uintptr_t>(v));
    }
    return ptrs;
  }
  if (rank >= 0 && rank != rank_) throw UsageError("Transport: share_buffer rank differs from this process's rank");
  std::lock_guard<std::mutex> lock(mu_);
  if (share_slots_ >= kLedgerRankBlobSlots - 1) throw ConfigError("Transport: too many shared buffers");
  const int slot = share_slots_++;
  CSB_CUDA(cudaSetDevice(device_));
  // an IPC handle names the whole allocation (a peer's mapping starts at its
  // base), so `base` may be an interior pointer: post the handle together
  // with base's offset inside its allocation
  struct Blob {
    cudaIpcMemHandle_t h;
    uint64_t offset;
  } blob{};
  static_assert(sizeof(Blob) <= kRankBlobLen, "IPC handle does not fit the mailbox");
  CSB_CUDA(cudaIpcGetMemHandle(&blob.h, base));
  {
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = [] {
      void* fp = nullptr;
      cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
      CSB_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q));
      if (!fp || q != cudaDriverEntryPointSuccess) throw CudaError("driver entry point missing: cuMemGetAddressRange");
      return reinterpret_cast<GetRange>(fp);
    }();
    CUdeviceptr alloc = 0;
    size_t alloc_bytes = 0;
    if (get_range(&alloc, &alloc_bytes, reinterpret_cast<CUdeviceptr>(base)) != CUDA_SUCCESS)
      throw UsageError("Transport: share_buffer of memory that is not a device allocation");
    blob.offset = reinterpret_cast<CUdeviceptr>(base) - alloc;
  }
  ledger_->post_rank_blob(slot, rank_, &blob, sizeof(blob));
  std::vector<void*> ptrs(static_cast<size_t>(num_ranks()), nullptr);
  for (int r = 0; r < num_ranks(); ++r) {
    if (r == rank_) {
      ptrs[r] = base;
      continue;
    }
    Blob pb{};
    ledger_->read_rank_blob(slot, r, &pb, sizeof(pb));
    void* p = nullptr;
    CSB_CUDA(cudaIpcOpenMemHandle(&p, pb.h, cudaIpcMemLazyEnablePeerAccess));
    ptrs[r] = static_cast<char*>(p) + pb.offset;
    ipc_opened_.push_back({p, ptrs[r]});
  }
  return ptrs;
}

void Transport::unshare_buffer(const std::vector<void*>& ptrs) {
  if (backend_ != Backend::Nccl) return;  // local peers are plain pointers
  std::lock_guard<std::mutex> lock(mu_);
  cudaSetDevice(device_);
  for (size_t r = 0; r < ptrs.size(); ++r) {
    if (static_cast<int>(r) == rank_ || !ptrs[r]) continue;
    auto it = std::find_if(ipc_opened_.begin(), ipc_opened_.end(),
                           [&](const std::pair<void*, void*>& o) { return o.second == ptrs[r]; });
    if (it == ipc_opened_.end()) continue;
    cudaIpcCloseMemHandle(it->first);
    ipc_opened_.erase(it);
  }
}

NvlsBuffer Transport::alloc_nvls(size_t bytes) {
  if (!nvls_capable()) throw UsageError("Transport: NVLS multicast unavailable on these devices");
  int slot;
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (share_slots_ + 2 > kLedgerRankBlobSlots - 1) throw ConfigError("Transport: too many shared buffers");
    slot = share_slots_;
    share_slots_ += 2;
  }
  std::string tag = name_;
  for (char& c : tag)
    if (c == '/') c = '_';
  return nvls_alloc(*ledger_, rank_, num_ranks(), device_, bytes, tag, slot);
}

void Transport::setup_flags() {
  void* f = nullptr;
  CSB_CUDA(cudaSetDevice(device_));
  CSB_CUDA(cudaMalloc(&f, p2p_flag_bytes()));
  CSB_CUDA(cudaMemset(f, 0, p2p_flag_bytes()));
  CSB_CUDA(cudaDeviceSynchronize());
  own_flags_.push_back(f);
  flags_.push_back(share_buffer(f));
}

// Local peer mode: one flag region per rank thread for `comm`, on the
// calling rank's device, zeroed on a private stream (no device-wide sync:
// other ranks' kernels may already be running).
void Transport::ensure_local_flags(int comm) {
  std::lock_guard<std::mutex> lock(mu_);
  if (comm < 0 || comm >= kLedgerMaxComms) throw UsageError("collective: unknown communicator");
  if (static_cast<int>(flags_.size()) <= comm) flags_.resize(static_cast<size_t>(comm) + 1);
  auto& f = flags_[static_cast<size_t>(comm)];
  if (!f.empty()) return;
  const int R = num_ranks();
  const size_t bytes = p2p_flag_bytes();
  char* base = nullptr;
  CSB_CUDA(cudaMalloc(&base, bytes * static_cast<size_t>(R)));
  cudaStream_t z;
  CSB_CUDA(cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking));
  CSB_CUDA(cudaMemsetAsync(base, 0, bytes * static_cast<size_t>(R), z));
  CSB_CUDA(cudaStreamSynchronize(z));
  CSB_CUDA(cudaStreamDestroy(z));
  CSB_CUDA(cudaGetDevice(&flags_device_));
  own_flags_.push_back(base);
  for (int r = 0; r < R; ++r) f.push_back(base + bytes * static_cast<size_t>(r));
}

// Peer kernels of one (communicator, rank) share a flag region, so they must
// run one after another: a launch on a different stream than the previous
// one first waits for it (the KvStore uses one ordered lane anyway).
void Transport::serialize_launch(int comm, int rank, cudaStream_t s, bool after) {
  std::lock_guard<std::mutex> lock(mu_);
  const size_t idx = static_cast<size_t>(comm) * kLedgerMaxRanks + static_cast<size_t>(rank);
  if (launch_order_.size() <= idx) launch_order_.resize(static_cast<size_t>(kLedgerMaxComms) * kLedgerMaxRanks);
  LaunchOrder& lo = launch_order_[idx];
  if (!after) {
    if (lo.ev && lo.stream != s) CSB_CUDA(cudaStreamWaitEvent(s, lo.ev, 0));
    return;
  }
  if (!lo.ev) {
    CSB_CUDA(cudaGetDevice(&lo.dev));
    CSB_CUDA(cudaEventCreateWithFlags(&lo.ev, cudaEventDisableTiming));
  }
  CSB_CUDA(cudaEventRecord(lo.ev, s));
  lo.stream = s;
}

void Transport::allreduce_p2p(int comm, int rank, void* const* peer_bufs, uint64_t count, int dtype,
                              int trace_key, cudaStream_t stream, int bucket, const P2PUpdate* upd,
                              void* mc, int concurrent) {
  if (!p2p_capable()) throw UsageError("Transport: peer-memory path unavailable");
  if (count == 0) throw UsageError("allreduce_sum: empty buffer");
  if (rank < 0 || rank >= num_ranks()) throw UsageError("collective: rank out of range");
  if (abort_host_ && reinterpret_cast<volatile uint32_t*>(abort_host_)[0] != kAbortNone) {
    // a previous peer launch timed out or the transport was aborted: latch
    const std::string m = device_failure();
    ledger_->abort(m.empty() ? "Transport: aborted" : m);
    throw DeadlockTimeout(m.empty() ? "Transport: aborted (peer-memory collectives disabled)" : m);
  }
  if (backend_ == Backend::Local) ensure_local_flags(comm);
  // a launch with no update entries is a plain reduce (kernel without phase 2)
  if (upd && (!upd->tab || upd->n_entries == 0)) upd = nullptr;
  CallSig sig;
  sig.kind = CollKind::AllreduceSum;
  sig.dtype = dtype;
  sig.count = static_cast<int64_t>(count);
  // every rank must run the same barrier protocol (a shard_only
  // rank would wait at a phase-2 barrier its peers never reach)
  const bool fused = upd && upd->update;
  sig.variant = kVarP2P | (mc ? kVarNvls : 0) | (fused ? kVarUpdate : 0) |
                (fused && upd->shard_only && !mc ? kVarShardOnly : 0) | (fused && upd->wm ? kVarZero : 0) |
                (upd && upd->gbase && !mc ? kVarDirect : 0);
  if (sig.variant & kVarDirect) sig.layout = upd->layout;
  Ledger::Ticket t;
  {
    hostprof::Scope prof(hostprof::kLedger);
    t = ledger_->arrive(comm, rank, sig, trace_key, bucket);
  }
  if (t.last) ledger_->finish(t);
  P2PArgs a;
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (comm < 0 || comm >= static_cast<int>(flags_.size())) throw UsageError("collective: unknown communicator");
    for (int r = 0; r < num_ranks(); ++r) {
      a.bufs[r] = peer_bufs[r];
      a.flags[r] = static_cast<uint32_t*>(flags_[static_cast<size_t>(comm)][static_cast<size_t>(r)]);
    }
  }
  a.mc = mc;
  a.nranks = num_ranks();
  a.rank = rank;
  a.colocated = colocated();
  a.concurrent = concurrent;
  a.abort_word = abort_dev_;
  if (stamps_dev_) a.stamps = stamps_dev_ + static_cast<size_t>(rank) * kStampsPerRank;
  a.count = count;
  a.cdt = dtype;
  a.epoch = static_cast<uint32_t>(t.seq + 1);  // same matched sequence on every rank
  if (upd) {
    a.update = upd->update;
    a.tab = upd->tab;
    a.n_entries = upd->n_entries;
    a.wdt = upd->wdt;
    a.lr = upd->lr;
    a.rescale = upd->rescale;
    a.momentum = upd->momentum;
    a.shard_only = upd->shard_only && !mc;
    a.pack = upd->pack && !mc;
    if (upd->gbase && !mc) {
      a.direct = true;
      for (int r = 0; r < num_ranks(); ++r) a.gbase[r] = const_cast<void*>(upd->gbase[r]);
    }
    if (upd->wm) {
      a.zero = true;
      for (int r = 0; r < num_ranks(); ++r) a.wm[r] = const_cast<void*>(upd->wm[r]);
      a.mom_b = upd->mom_b;
    }
  }
  device_latency(stream);
  serialize_launch(comm, rank, stream, false);
  p2p_allreduce(a, stream);
  serialize_launch(comm, rank, stream, true);
  ledger_->depart(t, trace_key, bucket);
  if (colocated()) wait_colocated(comm, rank);
}

// Colocated ranks share one device, so their streams share its hardware
// work queues (CUDA_DEVICE_MAX_CONNECTIONS).  A queue entry that waits on
// this kernel's completion, submitted after it, could then sit in front of
// a peer's launch of the same collective in a shared queue -- a false
// dependency that deadlocks the pair barriers.  So a colocated rank returns
// only once its peer kernel has completed: nothing it submits afterwards
// waits on an unfinished peer kernel, and every entry queued ahead of a
// launch depends only on that rank's own, finite work.
void Transport::wait_colocated(int comm, int rank) {
  cudaEvent_t ev;
  {
    std::lock_guard<std::mutex> lock(mu_);
    ev = launch_order_[static_cast<size_t>(comm) * kLedgerMaxRanks + static_cast<size_t>(rank)].ev;
  }
  int spins = 0;
  for (;;) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) CSB_CUDA(e);
    if (++spins < 256) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  if (reinterpret_cast<volatile uint32_t*>(abort_host_)[0] != kAbortNone) {
    const std::string m = device_failure();
    ledger_->abort(m.empty() ? "Transport: aborted" : m);
    throw DeadlockTimeout(m.empty() ? "Transport: peer-memory collective aborted while waiting for a peer" : m);
  }
}

std::vector<uint64_t> Transport::p2p_stamps(int rank) const {
  if (!stamps_host_ || rank < 0 || rank >= kLedgerMaxRanks) return {};
  const volatile uint64_t* p = stamps_host_ + static_cast<size_t>(rank) * kStampsPerRank;
  return std::vector<uint64_t>(p, p + kStampsPerRank);
}

Transport::~Transport() {
  if (watch_id_ >= 0) watch::remove(watch_id_);
  for (LaunchOrder& lo : launch_order_)
    if (lo.ev) {
      cudaSetDevice(lo.dev);
      cudaEventDestroy(lo.ev);
    }
  if (backend_ == Backend::Local && !own_flags_.empty()) {
    cudaSetDevice(flags_device_);
    for (void* p : own_flags_) cudaFree(p);
  }
  if (abort_host_) cudaFreeHost(abort_host_);
  if (stamps_host_) cudaFreeHost(stamps_host_);
  if (backend_ == Backend::Nccl) {
    const bool aborted = ledger_ && ledger_->latched();
    cudaSetDevice(device_);
    for (const auto& o : ipc_opened_) cudaIpcCloseMemHandle(o.first);
    for (void* p : own_flags_) cudaFree(p);
    for (ncclComm_t c : comms_) {
      if (!c) continue;
      if (aborted) ncclCommAbort(c);
      else ncclCommDestroy(c);
    }
  }
}

int Transport::new_communicator() {
  const int id = ledger_->new_communicator();
  if (backend_ == Backend::Nccl) {
    std::lock_guard<std::mutex> lock(mu_);
    CSB_CUDA(cudaSetDevice(device_));
    ncclComm_t c = nullptr;
    // ConCom's communicators run concurrently on one GPU: cap each one's
    // CTAs so all of them stay resident together (a communicator whose
    // channels cannot all be scheduled would wait on peers that wait on it)
    static const int max_ctas = [] {
      const char* e = std::getenv("CSB_CONCOM_MAX_CTAS");
      return std::max(1, e ? std::atoi(e) : 16);
    }();
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.maxCTAs = max_ctas;
    cfg.minCTAs = std::min(cfg.maxCTAs, 4);
    CSB_NCCL(ncclCommSplit(comms_[0], 0, rank_, &c, &cfg), comms_[0]);
    if (static_cast<int>(comms_.size()) != id) throw UsageError("Transport: communicator ids diverged");
    comms_.push_back(c);
  }
  if (backend_ == Backend::Nccl && p2p_capable()) setup_flags();  // every comm gets its own flag region
  return id;
}

void Transport::set_inject_latency(std::chrono::microseconds us) { ledger_->set_inject_latency(us); }
std::chrono::microseconds Transport::inject_latency() const { return ledger_->inject_latency(); }

void Transport::abort(const std::string& why) {
  // release every peer kernel still waiting in a pair barrier (they poll
  // the host-mapped word and return), then latch and abort NCCL
  if (abort_host_) {
    volatile uint32_t* w = abort_host_;
    if (w[0] == kAbortNone) w[0] = kAbortHost;
  }
  ledger_->abort(why);
  if (backend_ == Backend::Nccl) {
    std::lock_guard<std::mutex> lock(mu_);
    for (ncclComm_t& c : comms_) {
      if (c) ncclCommAbort(c);
      c = nullptr;
    }
  }
}

void Transport::allreduce_sum(int comm, int rank, void* buf, uint64_t count, int dtype,
                              int trace_key, cudaStream_t stream, int bucket) {
  if (count == 0) throw UsageError("allreduce_sum: empty buffer");  // collective.cpp:63-69
  CallSig sig;
  sig.kind = CollKind::AllreduceSum;
  sig.dtype = dtype;
  sig.count = static_cast<int64_t>(count);
  run(comm, rank, sig, buf, trace_key, stream, bucket);
}

void Transport::broadcast(int comm, int rank, int root, void* buf, uint64_t count, int dtype,
                          int trace_key, cudaStream_t stream) {
  if (root < 0 || root >= num_ranks()) throw UsageError("broadcast: root out of range");
  CallSig sig;
  sig.kind = CollKind::Broadcast;
  sig.dtype = dtype;
  sig.count = static_cast<int64_t>(count);
  sig.root = root;
  run(comm, rank, sig, buf, trace_key, stream, -1);
}

void Transport::barrier(int comm, int rank, int trace_key, cudaStream_t stream) {
  CallSig sig;
  sig.kind = CollKind::Barrier;
  run(comm, rank, sig, nullptr, trace_key, stream, -1);
}

void Transport::device_latency(cudaStream_t stream) {
  const auto lat = ledger_->inject_latency();
  if (lat.count() > 0 && stream)
    synth_backward(nullptr, nullptr, 0, CS_F32, static_cast<uint64_t>(lat.count()) * 1000, 1, stream);
}

void Transport::run(int comm, int rank, const CallSig& sig, void* buf, int trace_key,
                    cudaStream_t stream, int bucket) {
  if (backend_ != Backend::LedgerOnly && sig.kind != CollKind::Barrier && sig.count > 0 && !buf)
    throw UsageError("collective: null buffer");
  std::function<void(const Ledger::Ticket&)> publish;
  if (backend_ == Backend::Local && sig.kind != CollKind::Barrier) {
    publish = [&](const Ledger::Ticket& t) {
      SlotDev* sd;
      {
        std::lock_guard<std::mutex> lock(mu_);
        auto& p = slots_[ledger_->slot_uid(t)];
        if (!p) p = std::make_unique<SlotDev>();
        sd = p.get();
      }
      sd->bufs[rank] = buf;
      ensure_event(sd->ready[rank], sd->ready_dev[rank]);
      CSB_CUDA(cudaEventRecord(sd->ready[rank], stream));
    };
  }
  Ledger::Ticket t;
  {
    hostprof::Scope prof(hostprof::kLedger);
    t = ledger_->arrive(comm, rank, sig, trace_key, bucket, publish);
  }
  if (t.last) {
    try {
      if (backend_ == Backend::Local && sig.kind != CollKind::Barrier) local_data(t, sig, buf, stream);
    } catch (...) {
      ledger_->abort("collective: reducer failed to enqueue");
      ledger_->finish(t);
      throw;
    }
    ledger_->finish(t);
  } else if (backend_ == Backend::Local && sig.kind != CollKind::Barrier && sig.count > 0) {
    SlotDev* sd;
    {
      std::lock_guard<std::mutex> lock(mu_);
      sd = slots_[ledger_->slot_uid(t)].get();
    }
    CSB_CUDA(cudaStreamWaitEvent(stream, sd->done, 0));
  }
  // one rank: the matched call is the identity (collective.cpp:228-243 with
  // R = 1), nothing to move
  if (backend_ == Backend::Nccl && sig.kind != CollKind::Barrier && sig.count > 0 && num_ranks() > 1) {
    device_latency(stream);
    nccl_data(comm, sig, buf, stream);
  }
  ledger_->depart(t, trace_key, bucket);
}

// Last arriver of an in-process rendezvous: fixed rank-order reduction of
// every rank's buffer by kernel (b), result written to all of them
// (collective.cpp:228-236), or root -> everyone copy (collective.cpp:237-243).
void Transport::local_data(const Ledger::Ticket& t, const CallSig& sig, void* buf,
                           cudaStream_t stream) {
  SlotDev* sd;
  {
    std::lock_guard<std::mutex> lock(mu_);
    sd = slots_[ledger_->slot_uid(t)].get();
  }
  const int R = num_ranks();
  for (int r = 0; r < R; ++r)
    if (r != t.rank) CSB_CUDA(cudaStreamWaitEvent(stream, sd->ready[r], 0));
  if (sig.count > 0) {
    device_latency(stream);
    if (sig.kind == CollKind::AllreduceSum) {
      if (R > 1) sum_buffers(sd->bufs, R, sd->bufs, R, static_cast<uint64_t>(sig.count), sig.dtype, stream);
    } else {
      const void* src[1] = {sd->bufs[sig.root]};
      void* dst[kLedgerMaxRanks];
      int nd = 0;
      for (int r = 0; r < R; ++r)
        if (r != sig.root) dst[nd++] = sd->bufs[r];
      if (nd > 0) sum_buffers(src, 1, dst, nd, static_cast<uint64_t>(sig.count), sig.dtype, stream);
    }
  }
  (void)buf;
  ensure_event(sd->done, sd->done_dev);
  CSB_CUDA(cudaEventRecord(sd->done, stream));
}

void Transport::nccl_data(int comm, const CallSig& sig, void* buf, cudaStream_t stream) {
  ncclComm_t c;
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (comm < 0 || comm >= static_cast<int>(comms_.size()) || !comms_[comm])
      throw UsageError("collective: communicator not available");
    c = comms_[comm];
  }
  const ncclDataType_t ty = nccl_type(sig.dtype);
  if (sig.kind == CollKind::AllreduceSum) {
    CSB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(sig.count), ty, ncclSum, c, stream), c);
  } else if (sig.kind == CollKind::Broadcast) {
    CSB_NCCL(ncclBroadcast(buf, buf, static_cast<size_t>(sig.count), ty, sig.root, c, stream), c);
  }
}

}  // namespace csb
