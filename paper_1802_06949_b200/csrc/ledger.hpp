// ledger.hpp -- cross-rank collective matching ledger.
//
// Host-side restatement of the reference Transport's rendezvous
// (R/core/src/collective.cpp:136-290) that runs BEFORE any device work is
// enqueued: the k-th call a rank issues on a communicator takes sequence
// index k (collective.cpp:151-152) and is paired with every other rank's
// k-th call; signatures {kind, count, root, dtype} must agree
// (collective.cpp:192-204) or every participant raises MismatchError; a
// rendezvous still incomplete after the watchdog raises DeadlockTimeout with
// a per-rank pending-call report (collective.cpp:114-134, 249-264); any
// failure latches for the whole run (collective.cpp:92-105).  Because NCCL
// kernels are only enqueued after a complete, matched rendezvous, a
// misordered schedule (the paper's naive hazard) surfaces as an exception
// instead of hanging NVLink kernels.
//
// Storage is either process memory (in-process rank threads) or a POSIX
// shared-memory segment (one process per GPU on one box); both use
// process-shared pthread mutex/condvar, so the code path is identical.
#pragma once

#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "trace.hpp"

namespace csb {

enum class CollKind : int32_t { AllreduceSum = 0, Broadcast = 1, Barrier = 2 };
const char* coll_kind_name(CollKind k);

struct CallSig {
  CollKind kind = CollKind::Barrier;
  int32_t dtype = -1;
  int64_t count = 0;
  int32_t root = -1;
  // B200 extension: peer-memory kernels pair CTAs across ranks, so every rank
  // must launch the same barrier protocol (CallVariant bits); 0 = plain call
  int32_t variant = 0;
  // kVarDirect: hash of the gradients' (key, offset in the registered region)
  // layout, which must be identical on every rank (peers address each other's
  // gradients by this rank's offsets)
  uint64_t layout = 0;
  bool operator==(const CallSig& o) const {
    return kind == o.kind && count == o.count && root == o.root && dtype == o.dtype && variant == o.variant &&
           layout == o.layout;
  }
};

// CallSig::variant bits of a peer-memory allreduce (kernels.cu p2p kernels)
enum CallVariant : int32_t {
  kVarP2P = 1,        // fused peer-memory kernel (pair barriers)
  kVarUpdate = 2,     // fused SGD / momentum update
  kVarShardOnly = 4,  // update reads the owners' shards; trailing barrier
  kVarZero = 8,       // ZeRO-1 form
  kVarNvls = 16,      // NVSwitch multicast reduction
  kVarDirect = 32,    // phase 1 reads every rank's gradients in place (registered region, no staging)
};

std::string describe_call(const CallSig& sig);

constexpr int kLedgerMaxRanks = 16;
constexpr int kLedgerMaxComms = 17;  // world + up to 16 extra communicators
constexpr int kLedgerSlots = 256;    // ring of in-flight sequence indices per comm
constexpr int kLedgerRankBlobSlots = 64;  // per-rank setup mailbox slots
constexpr int kRankBlobLen = 80;          // >= sizeof(cudaIpcMemHandle_t) + metadata

struct LedgerShared;  // layout in ledger.cpp

class Ledger {
 public:
  struct Ticket {
    int comm = -1;
    int rank = -1;
    uint64_t seq = 0;
    int slot = -1;
    bool last = false;  // this rank completed the rendezvous
    int inflight = -1;
  };

  // In-process ledger for `nranks` rank threads.
  static std::unique_ptr<Ledger> create_local(int nranks, std::chrono::milliseconds watchdog,
                                              TraceSink* trace);
  // Shared-memory ledger: rank 0 creates segment `name`, all ranks attach,
  // then the name is unlinked.  Blocks until every rank attached.
  static std::unique_ptr<Ledger> create_shm(const std::string& name, int nranks, int rank,
                                            std::chrono::milliseconds watchdog, TraceSink* trace);
  ~Ledger();

  int num_ranks() const { return nranks_; }
  bool shared_memory() const { return shm_; }

  // Setup-phase only (collective.cpp:44-51).  In shm mode every rank calls
  // it in the same order; returns the new communicator id.
  int new_communicator();
  int num_communicators() const;

  // Takes the next sequence index of `rank` on `comm`, checks the signature
  // against the ranks already there and blocks until all ranks arrived.
  // The last arriver returns with ticket.last = true and must call
  // finish(); everyone else returns once the last arriver has finished.
  // Throws MismatchError / DeadlockTimeout / UsageError.
  // on_matched_slot (optional) runs under the ledger lock once this rank's
  // sequence index, ring slot and signature check are settled, before the
  // wait: the local backend publishes its buffer and ready event there.
  Ticket arrive(int comm, int rank, const CallSig& sig, int trace_key, int bucket = -1,
                const std::function<void(const Ticket&)>& on_matched_slot = {});
  // Last arriver: releases the waiting ranks (after the optional injected
  // latency, collective.cpp:222-227).
  void finish(const Ticket& t);
  // Every participant, after its own enqueue: emits coll_done, frees the slot
  // once all ranks departed.
  void depart(const Ticket& t, int trace_key, int bucket = -1);

  void set_inject_latency(std::chrono::microseconds us);
  std::chrono::microseconds inject_latency() const;
  // Latches an abort (every current and future call fails fast).
  void abort(const std::string& why);
  bool latched() const;

  // Setup mailbox for NCCL unique ids (shm mode): rank 0 posts, others wait.
  void post_blob(int index, const void* data, size_t n);
  void read_blob(int index, void* data, size_t n);
  // Per-rank setup mailbox (CUDA IPC handles of peer-shared buffers).
  void post_rank_blob(int slot, int rank, const void* data, size_t n);
  void read_rank_blob(int slot, int rank, void* data, size_t n);

  uint64_t slot_uid(const Ticket& t) const { return static_cast<uint64_t>(t.comm) * kLedgerSlots + t.slot; }

 private:
  Ledger() = default;
  void init_storage(bool creator);
  [[noreturn]] void throw_latched() const;
  [[noreturn]] void fail_slot(int comm, int slot, Error::Kind kind, const std::string& msg);
  std::string deadlock_report(int comm, uint64_t seq) const;
  void emit(const char* event, int rank, int key, int comm, uint64_t seq, CollKind kind, int bucket);

  int nranks_ = 0;
  int rank_ = -1;  // shm mode: the owning rank; local: -1 (all)
  bool shm_ = false;
  std::string name_;
  size_t bytes_ = 0;
  LedgerShared* s_ = nullptr;
  std::chrono::milliseconds watchdog_{5000};
  TraceSink* trace_ = nullptr;
};

}  // namespace csb
