// ledger.cpp -- see ledger.hpp.
#include "ledger.hpp"

#include <errno.h>
#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <thread>

namespace csb {

namespace {
constexpr uint64_t kFree = ~0ull;
constexpr int kInflightPerRank = 32;
constexpr int kMsgLen = 512;
constexpr int kDescLen = 96;  // room for the p2p variant and the direct layout hash
constexpr int kBlobLen = 256;
}  // namespace

const char* coll_kind_name(CollKind k) {
  switch (k) {
    case CollKind::AllreduceSum: return "allreduce";
    case CollKind::Broadcast: return "broadcast";
    case CollKind::Barrier: return "barrier";
  }
  return "unknown";
}

// collective.cpp:23-33 (describe): "allreduce(count=6)", "broadcast(count=4, root=0)", "barrier"
std::string describe_call(const CallSig& sig) {
  std::ostringstream os;
  os << coll_kind_name(sig.kind);
  if (sig.kind == CollKind::AllreduceSum) {
    os << "(count=" << sig.count;
    if (sig.variant & kVarP2P) {
      os << ", " << ((sig.variant & kVarNvls) ? "nvls" : "p2p");
      if (sig.variant & kVarUpdate) os << "+update";
      if (sig.variant & kVarShardOnly) os << "+shard_only";
      if (sig.variant & kVarZero) os << "+zero";
      if (sig.variant & kVarDirect) os << "+direct(layout " << std::hex << sig.layout << std::dec << ")";
    }
    os << ")";
  } else if (sig.kind == CollKind::Broadcast) {
    os << "(count=" << sig.count << ", root=" << sig.root << ")";
  }
  return os.str();
}

struct SlotRec {
  uint64_t seq;
  int32_t arrived, returned, all_arrived, done, failed, fail_kind;
  CallSig sig;
  char desc[kLedgerMaxRanks][kDescLen];
  char fail_msg[kMsgLen];
};

struct InflightRec {
  int32_t used;
  int32_t rank;
  uint64_t order;
  char desc[96];
};

struct LedgerShared {
  std::atomic<uint64_t> magic;
  int32_t nranks;
  int32_t ncomms;
  int32_t attached;
  int32_t started;
  int32_t latched;
  int32_t latch_kind;
  int64_t latency_us;
  uint64_t inflight_order;
  char latch_msg[kMsgLen];
  pthread_mutex_t mu;
  pthread_cond_t cv;
  int32_t comms_by_rank[kLedgerMaxRanks];
  int32_t started_by_rank[kLedgerMaxRanks];
  uint64_t next_seq[kLedgerMaxComms][kLedgerMaxRanks];
  InflightRec inflight[kLedgerMaxRanks * kInflightPerRank];
  int32_t blob_ready[kLedgerMaxComms];
  char blob[kLedgerMaxComms][kBlobLen];
  int32_t rblob_ready[kLedgerRankBlobSlots][kLedgerMaxRanks];
  char rblob[kLedgerRankBlobSlots][kLedgerMaxRanks][kRankBlobLen];
  SlotRec slots[kLedgerMaxComms][kLedgerSlots];
};

namespace {

constexpr uint64_t kMagic = 0xC0115B200ull ^ (static_cast<uint64_t>(sizeof(LedgerShared)) << 20);

struct Lock {
  LedgerShared* s;
  explicit Lock(LedgerShared* sh) : s(sh) {
    int rc = pthread_mutex_lock(&s->mu);
    if (rc == EOWNERDEAD) pthread_mutex_consistent(&s->mu);
  }
  ~Lock() { pthread_mutex_unlock(&s->mu); }
};

timespec abs_deadline(std::chrono::steady_clock::time_point dl) {
  // steady_clock == CLOCK_MONOTONIC on Linux/glibc
  auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(dl.time_since_epoch()).count();
  timespec ts;
  ts.tv_sec = static_cast<time_t>(ns / 1000000000LL);
  ts.tv_nsec = static_cast<long>(ns % 1000000000LL);
  return ts;
}

// true on timeout
bool timed_wait(LedgerShared* s, std::chrono::steady_clock::time_point dl) {
  timespec ts = abs_deadline(dl);
  int rc = pthread_cond_timedwait(&s->cv, &s->mu, &ts);
  if (rc == EOWNERDEAD) pthread_mutex_consistent(&s->mu);
  return rc == ETIMEDOUT;
}

void plain_wait(LedgerShared* s) {
  int rc = pthread_cond_wait(&s->cv, &s->mu);
  if (rc == EOWNERDEAD) pthread_mutex_consistent(&s->mu);
}

void copy_str(char* dst, size_t cap, const std::string& src) {
  size_t n = std::min(cap - 1, src.size());
  std::memcpy(dst, src.data(), n);
  dst[n] = '\0';
}

void init_sync(LedgerShared* s) {
  pthread_mutexattr_t ma;
  pthread_mutexattr_init(&ma);
  pthread_mutexattr_setpshared(&ma, PTHREAD_PROCESS_SHARED);
  pthread_mutexattr_setrobust(&ma, PTHREAD_MUTEX_ROBUST);
  pthread_mutex_init(&s->mu, &ma);
  pthread_mutexattr_destroy(&ma);
  pthread_condattr_t ca;
  pthread_condattr_init(&ca);
  pthread_condattr_setpshared(&ca, PTHREAD_PROCESS_SHARED);
  pthread_condattr_setclock(&ca, CLOCK_MONOTONIC);
  pthread_cond_init(&s->cv, &ca);
  pthread_condattr_destroy(&ca);
}

void init_slots(LedgerShared* s) {
  for (int c = 0; c < kLedgerMaxComms; ++c)
    for (int i = 0; i < kLedgerSlots; ++i) s->slots[c][i].seq = kFree;
}

}  // namespace

std::unique_ptr<Ledger> Ledger::create_local(int nranks, std::chrono::milliseconds watchdog,
                                             TraceSink* trace) {
  if (nranks < 1) throw ConfigError("Transport: num_ranks must be >= 1");
  if (nranks > kLedgerMaxRanks) throw ConfigError("Transport: at most 16 ranks");
  if (watchdog.count() <= 0) throw ConfigError("Transport: watchdog duration must be positive");
  std::unique_ptr<Ledger> l(new Ledger());
  l->nranks_ = nranks;
  l->watchdog_ = watchdog;
  l->trace_ = trace;
  l->bytes_ = sizeof(LedgerShared);
  void* mem = mmap(nullptr, l->bytes_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (mem == MAP_FAILED) throw ConfigError("Transport: ledger allocation failed");
  l->s_ = static_cast<LedgerShared*>(mem);  // zero-filled by the kernel
  init_sync(l->s_);
  init_slots(l->s_);
  l->s_->nranks = nranks;
  l->s_->ncomms = 1;
  l->s_->attached = nranks;
  l->s_->magic.store(kMagic);
  return l;
}

std::unique_ptr<Ledger> Ledger::create_shm(const std::string& name_in, int nranks, int rank,
                                           std::chrono::milliseconds watchdog, TraceSink* trace) {
  if (nranks < 1) throw ConfigError("Transport: num_ranks must be >= 1");
  if (nranks > kLedgerMaxRanks) throw ConfigError("Transport: at most 16 ranks");
  if (rank < 0 || rank >= nranks) throw ConfigError("Transport: rank out of range");
  if (watchdog.count() <= 0) throw ConfigError("Transport: watchdog duration must be positive");
  if (name_in.empty()) throw ConfigError("Transport: shared-memory ledger needs a name");
  std::string name = name_in[0] == '/' ? name_in : "/" + name_in;
  std::unique_ptr<Ledger> l(new Ledger());
  l->nranks_ = nranks;
  l->rank_ = rank;
  l->shm_ = true;
  l->name_ = name;
  l->watchdog_ = watchdog;
  l->trace_ = trace;
  l->bytes_ = sizeof(LedgerShared);
  const auto attach_deadline =
      std::chrono::steady_clock::now() + std::max(watchdog, std::chrono::milliseconds(120000));
  if (rank == 0) {
    shm_unlink(name.c_str());
    int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw ConfigError("Transport: shm_open(" + name + ") failed: " + strerror(errno));
    if (ftruncate(fd, static_cast<off_t>(l->bytes_)) != 0) {
      close(fd);
      throw ConfigError("Transport: ftruncate of the ledger failed");
    }
    void* mem = mmap(nullptr, l->bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mem == MAP_FAILED) throw ConfigError("Transport: mmap of the ledger failed");
    l->s_ = static_cast<LedgerShared*>(mem);
    init_sync(l->s_);
    init_slots(l->s_);
    l->s_->nranks = nranks;
    l->s_->ncomms = 1;
    l->s_->magic.store(kMagic, std::memory_order_release);
  } else {
    for (;;) {
      int fd = shm_open(name.c_str(), O_RDWR, 0600);
      if (fd >= 0) {
        struct stat st;
        if (fstat(fd, &st) == 0 && static_cast<size_t>(st.st_size) == l->bytes_) {
          void* mem = mmap(nullptr, l->bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
          close(fd);
          if (mem != MAP_FAILED) {
            auto* s = static_cast<LedgerShared*>(mem);
            if (s->magic.load(std::memory_order_acquire) == kMagic && s->nranks == nranks) {
              l->s_ = s;
              break;
            }
            munmap(mem, l->bytes_);
          }
        } else {
          close(fd);
        }
      }
      if (std::chrono::steady_clock::now() > attach_deadline)
        throw DeadlockTimeout("Transport: rank " + std::to_string(rank) +
                              " could not attach to ledger " + name);
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  {
    Lock lk(l->s_);
    l->s_->attached++;
    pthread_cond_broadcast(&l->s_->cv);
    while (l->s_->attached < nranks) {
      if (timed_wait(l->s_, attach_deadline) && l->s_->attached < nranks)
        throw DeadlockTimeout("Transport: only " + std::to_string(l->s_->attached) + " of " +
                              std::to_string(nranks) + " ranks attached to ledger " + name);
    }
  }
  if (rank == 0) shm_unlink(name.c_str());  // mapping persists; nothing left in /dev/shm
  return l;
}

Ledger::~Ledger() {
  if (s_) munmap(s_, bytes_);
}

int Ledger::new_communicator() {
  Lock lk(s_);
  // setup-phase only (collective.cpp:44-51); with one process per rank the
  // phase is per process: this rank must not have issued a collective yet
  if (shm_ ? s_->started_by_rank[rank_] : s_->started)
    throw UsageError(
        "Transport: communicators must be created before workers start issuing collectives");
  if (shm_) {
    int id = ++s_->comms_by_rank[rank_];
    if (id >= kLedgerMaxComms) throw ConfigError("Transport: too many communicators");
    if (id + 1 > s_->ncomms) s_->ncomms = id + 1;
    return id;
  }
  if (s_->ncomms >= kLedgerMaxComms) throw ConfigError("Transport: too many communicators");
  return s_->ncomms++;
}

int Ledger::num_communicators() const {
  Lock lk(s_);
  return s_->ncomms;
}

void Ledger::set_inject_latency(std::chrono::microseconds us) {
  Lock lk(s_);
  s_->latency_us = us.count();
}

std::chrono::microseconds Ledger::inject_latency() const {
  Lock lk(s_);
  return std::chrono::microseconds(s_->latency_us);
}

bool Ledger::latched() const {
  Lock lk(s_);
  return s_->latched != 0;
}

void Ledger::abort(const std::string& why) {
  Lock lk(s_);
  if (!s_->latched) {
    s_->latched = 1;
    s_->latch_kind = static_cast<int32_t>(Error::Kind::DeadlockTimeout);
    copy_str(s_->latch_msg, kMsgLen, why);
  }
  pthread_cond_broadcast(&s_->cv);
}

void Ledger::throw_latched() const {
  const std::string msg(s_->latch_msg);
  if (s_->latch_kind == static_cast<int32_t>(Error::Kind::DeadlockTimeout)) throw DeadlockTimeout(msg);
  throw MismatchError(msg);
}

void Ledger::fail_slot(int comm, int slot, Error::Kind kind, const std::string& msg) {
  SlotRec& sr = s_->slots[comm][slot];
  sr.failed = 1;
  sr.fail_kind = static_cast<int32_t>(kind);
  copy_str(sr.fail_msg, kMsgLen, msg);
  if (!shm_ && trace_) trace_->gauges().collective_closed();
  // collective failures are unrecoverable for the run (collective.cpp:92-105)
  s_->latched = 1;
  s_->latch_kind = static_cast<int32_t>(kind);
  copy_str(s_->latch_msg, kMsgLen, msg);
  pthread_cond_broadcast(&s_->cv);
  if (kind == Error::Kind::DeadlockTimeout) throw DeadlockTimeout(msg);
  throw MismatchError(msg);
}

// collective.cpp:114-134
std::string Ledger::deadlock_report(int comm, uint64_t seq) const {
  std::ostringstream os;
  os << "rendezvous on comm " << comm << " seq " << seq << " incomplete after "
     << watchdog_.count() << " ms;";
  for (int r = 0; r < nranks_; ++r) {
    os << " rank " << r << ": ";
    // in registration order
    std::vector<const InflightRec*> mine;
    for (const InflightRec& f : s_->inflight)
      if (f.used && f.rank == r) mine.push_back(&f);
    std::sort(mine.begin(), mine.end(),
              [](const InflightRec* a, const InflightRec* b) { return a->order < b->order; });
    bool any = false;
    for (const InflightRec* f : mine) {
      if (any) os << ", ";
      os << f->desc;
      any = true;
    }
    if (!any) os << "no call issued";
    if (r + 1 < nranks_) os << ";";
  }
  return os.str();
}

void Ledger::emit(const char* event, int rank, int key, int comm, uint64_t seq, CollKind kind,
                  int bucket) {
  if (!trace_) return;
  TraceEvent ev;
  ev.rank = rank;
  ev.event = event;
  ev.key = key;
  ev.comm = comm;
  ev.seq = static_cast<int64_t>(seq);
  ev.kind = coll_kind_name(kind);
  ev.bucket = bucket;
  trace_->emit(std::move(ev));
}

Ledger::Ticket Ledger::arrive(int comm, int rank, const CallSig& sig, int trace_key, int bucket,
                              const std::function<void(const Ticket&)>& on_matched_slot) {
  Lock lk(s_);
  if (rank < 0 || rank >= nranks_) throw UsageError("collective: rank out of range");
  if (shm_ && rank != rank_) throw UsageError("collective: rank differs from this process's rank");
  if (comm < 0 || comm >= s_->ncomms) throw UsageError("collective: unknown communicator");
  if (s_->latched) throw_latched();
  s_->started = 1;
  s_->started_by_rank[rank] = 1;

  const uint64_t seq = s_->next_seq[comm][rank]++;
  const int slot = static_cast<int>(seq % kLedgerSlots);
  const auto deadline = std::chrono::steady_clock::now() + watchdog_;
  const std::string call_desc = describe_call(sig);

  // register as in flight (deadlock report)
  int token = -1;
  for (int i = rank * kInflightPerRank; i < (rank + 1) * kInflightPerRank; ++i) {
    if (!s_->inflight[i].used) {
      token = i;
      break;
    }
  }
  if (token < 0) throw UsageError("collective: too many in-flight calls on one rank");
  {
    InflightRec& f = s_->inflight[token];
    f.used = 1;
    f.rank = rank;
    f.order = s_->inflight_order++;
    std::ostringstream os;
    os << call_desc << " on comm " << comm << " seq " << seq;
    copy_str(f.desc, sizeof(f.desc), os.str());
  }
  auto drop = [&] { s_->inflight[token].used = 0; };

  emit("coll_enqueued", rank, trace_key, comm, seq, sig.kind, bucket);

  // claim the ring slot (an older sequence may still be draining)
  for (;;) {
    SlotRec& sr = s_->slots[comm][slot];
    if (sr.seq == seq) break;
    if (sr.seq == kFree) {
      sr.seq = seq;
      sr.arrived = sr.returned = sr.all_arrived = sr.done = sr.failed = 0;
      sr.fail_kind = 0;
      std::memset(sr.desc, 0, sizeof(sr.desc));
      sr.fail_msg[0] = '\0';
      break;
    }
    if (s_->latched) {
      drop();
      throw_latched();
    }
    if (timed_wait(s_, deadline) && s_->slots[comm][slot].seq != seq &&
        s_->slots[comm][slot].seq != kFree) {
      const std::string report = deadlock_report(comm, s_->slots[comm][slot].seq);
      drop();
      fail_slot(comm, slot, Error::Kind::DeadlockTimeout, report);
    }
  }
  SlotRec& sr = s_->slots[comm][slot];
  if (sr.failed) {
    drop();
    if (sr.fail_kind == static_cast<int32_t>(Error::Kind::DeadlockTimeout))
      throw DeadlockTimeout(sr.fail_msg);
    throw MismatchError(sr.fail_msg);
  }
  if (sr.arrived == 0) {
    sr.sig = sig;
    if (!shm_ && trace_) trace_->gauges().collective_opened();
  } else if (!(sr.sig == sig)) {
    copy_str(sr.desc[rank], kDescLen, call_desc);
    std::ostringstream os;
    os << "collective signature mismatch on comm " << comm << " seq " << seq << ":";
    for (int r = 0; r < nranks_; ++r)
      if (sr.desc[r][0]) os << " rank " << r << ": " << sr.desc[r] << ";";
    drop();
    fail_slot(comm, slot, Error::Kind::Mismatch, os.str());
  }
  copy_str(sr.desc[rank], kDescLen, call_desc);

  Ticket t;
  t.comm = comm;
  t.rank = rank;
  t.seq = seq;
  t.slot = slot;
  t.inflight = token;
  if (on_matched_slot) {
    try {
      on_matched_slot(t);
    } catch (...) {
      drop();
      throw;
    }
  }
  sr.arrived++;
  if (sr.arrived == nranks_) {
    sr.all_arrived = 1;
    emit("coll_matched", rank, trace_key, comm, seq, sig.kind, bucket);
    pthread_cond_broadcast(&s_->cv);
    t.last = true;
    return t;
  }
  // Ranks usually arrive within microseconds of each other: poll the slot
  // with the lock released before sleeping on the (process-shared) condvar.
  // A futex wake-up from an idle core can take hundreds of microseconds, and
  // a rank that sleeps wakes late and makes the others wait at the next
  // collective -- measured as a bimodal 0.6 / 1.6 ms step at 4 GPUs with a
  // 100 us spin.  CSB_LEDGER_SPIN_US (default 2000).
  {
    static const long spin_us = [] {
      const char* e = std::getenv("CSB_LEDGER_SPIN_US");
      return e ? std::atol(e) : 2000L;
    }();
    pthread_mutex_unlock(&s_->mu);
    const auto spin_end = std::chrono::steady_clock::now() + std::chrono::microseconds(spin_us);
    while (!__atomic_load_n(&sr.done, __ATOMIC_ACQUIRE) && !__atomic_load_n(&sr.failed, __ATOMIC_ACQUIRE) &&
           !__atomic_load_n(&s_->latched, __ATOMIC_ACQUIRE) && std::chrono::steady_clock::now() < spin_end) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
    const int rc = pthread_mutex_lock(&s_->mu);
    if (rc == EOWNERDEAD) pthread_mutex_consistent(&s_->mu);
  }
  // wait for completion; the watchdog only applies before full arrival
  // (collective.cpp:249-264)
  for (;;) {
    if (sr.done || sr.failed) break;
    if (sr.all_arrived) {
      plain_wait(s_);
      continue;
    }
    if (s_->latched) break;
    if (timed_wait(s_, deadline) && !(sr.done || sr.failed || sr.all_arrived || s_->latched)) {
      const std::string report = deadlock_report(comm, seq);  // includes this call
      drop();
      fail_slot(comm, slot, Error::Kind::DeadlockTimeout, report);
    }
  }
  if (sr.failed) {
    drop();
    if (sr.fail_kind == static_cast<int32_t>(Error::Kind::DeadlockTimeout))
      throw DeadlockTimeout(sr.fail_msg);
    throw MismatchError(sr.fail_msg);
  }
  if (!sr.done && s_->latched) {
    drop();
    throw_latched();
  }
  return t;
}

void Ledger::finish(const Ticket& t) {
  int64_t lat = 0;
  {
    Lock lk(s_);
    lat = s_->latency_us;
  }
  if (lat > 0) std::this_thread::sleep_for(std::chrono::microseconds(lat));
  Lock lk(s_);
  SlotRec& sr = s_->slots[t.comm][t.slot];
  sr.done = 1;
  if (!shm_ && trace_) trace_->gauges().collective_closed();
  pthread_cond_broadcast(&s_->cv);
}

void Ledger::depart(const Ticket& t, int trace_key, int bucket) {
  Lock lk(s_);
  if (t.inflight >= 0) s_->inflight[t.inflight].used = 0;
  SlotRec& sr = s_->slots[t.comm][t.slot];
  emit("coll_done", t.rank, trace_key, t.comm, t.seq, sr.sig.kind, bucket);
  sr.returned++;
  if (sr.returned == nranks_) {
    sr.seq = kFree;
    pthread_cond_broadcast(&s_->cv);
  }
}

void Ledger::post_blob(int index, const void* data, size_t n) {
  if (index < 0 || index >= kLedgerMaxComms || n > kBlobLen) throw UsageError("ledger blob index");
  Lock lk(s_);
  std::memcpy(s_->blob[index], data, n);
  s_->blob_ready[index] = 1;
  pthread_cond_broadcast(&s_->cv);
}

void Ledger::post_rank_blob(int slot, int rank, const void* data, size_t n) {
  if (slot < 0 || slot >= kLedgerRankBlobSlots || rank < 0 || rank >= nranks_ || n > kRankBlobLen)
    throw UsageError("ledger: rank blob slot out of range");
  Lock lk(s_);
  std::memcpy(s_->rblob[slot][rank], data, n);
  s_->rblob_ready[slot][rank] = 1;
  pthread_cond_broadcast(&s_->cv);
}

void Ledger::read_rank_blob(int slot, int rank, void* data, size_t n) {
  if (slot < 0 || slot >= kLedgerRankBlobSlots || rank < 0 || rank >= nranks_ || n > kRankBlobLen)
    throw UsageError("ledger: rank blob slot out of range");
  const auto deadline =
      std::chrono::steady_clock::now() + std::max(watchdog_, std::chrono::milliseconds(120000));
  Lock lk(s_);
  while (!s_->rblob_ready[slot][rank]) {
    if (timed_wait(s_, deadline) && !s_->rblob_ready[slot][rank])
      throw DeadlockTimeout("Transport: rank " + std::to_string(rank) + " never posted setup blob " +
                            std::to_string(slot));
  }
  std::memcpy(data, s_->rblob[slot][rank], n);
}

void Ledger::read_blob(int index, void* data, size_t n) {
  if (index < 0 || index >= kLedgerMaxComms || n > kBlobLen) throw UsageError("ledger blob index");
  const auto deadline =
      std::chrono::steady_clock::now() + std::max(watchdog_, std::chrono::milliseconds(120000));
  Lock lk(s_);
  while (!s_->blob_ready[index]) {
    if (timed_wait(s_, deadline) && !s_->blob_ready[index])
      throw DeadlockTimeout("Transport: setup blob " + std::to_string(index) + " never posted");
  }
  std::memcpy(data, s_->blob[index], n);
}

}  // namespace csb
