// engine.cpp -- see engine.hpp.  Reference behaviour mirrored:
//   push validation / enqueue      R/core/src/engine.cpp:52-111
//   grant_head (write / read run)  R/core/src/engine.cpp:113-133
//   decrement_pending / complete   R/core/src/engine.cpp:135-161
//   worker loop, poison            R/core/src/engine.cpp:163-215
//   wait_for / wait_all / shutdown R/core/src/engine.cpp:217-246
#include "engine.hpp"
#include "watch.hpp"

#include "hostprof.hpp"

#include <algorithm>
#include <array>
#include <cstdlib>

namespace csb {

namespace {
std::atomic<uint64_t> g_engine_ids{1};
constexpr int kMaxLanes = 64;
}  // namespace

const char* op_kind_name(OpKind kind) {
  switch (kind) {
    case OpKind::Compute: return "compute";
    case OpKind::Copy: return "copy";
    case OpKind::Collective: return "collective";
    case OpKind::Other: return "other";
  }
  return "other";
}

// Recycles CUDA events (creation is a driver call; an aggregation step
// records one per op).  Shared with every EventRef so it outlives them.
struct EventPool {
  int device = -1;
  std::mutex mu;
  std::vector<cudaEvent_t> free;
  std::vector<cudaEvent_t> all;
  ~EventPool() {
    if (device < 0) return;
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    cudaSetDevice(device);
    for (cudaEvent_t e : all) cudaEventDestroy(e);
    cudaSetDevice(prev);
  }
};

Engine::Engine(int num_worker_threads, int rank, TraceSink* trace, int device)
    : engine_id_(g_engine_ids.fetch_add(1)), rank_(rank), trace_(trace), device_(device) {
  if (num_worker_threads < 1) throw ConfigError("Engine: worker pool size must be >= 1");
  pool_ = std::make_shared<EventPool>();
  pool_->device = device;
  if (const char* s = std::getenv("CSB_ENGINE_SPIN_US")) spin_ = std::chrono::microseconds(std::atoll(s));
  lanes_.reserve(kMaxLanes);
  lane_seq_.assign(kMaxLanes, 0);
  if (device_ >= 0) {
    int count = 0;
    CSB_CUDA(cudaGetDeviceCount(&count));
    if (device_ >= count) throw ConfigError("Engine: device index out of range");
    bind_device();
    cudaStream_t s;
    CSB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    lanes_.push_back(s);
  }
  workers_.reserve(static_cast<size_t>(num_worker_threads));
  for (int i = 0; i < num_worker_threads; ++i) workers_.emplace_back([this, i] { worker_loop(i); });
}

Engine::~Engine() {
  shutdown();
  if (device_ >= 0) {
    try {
      sync_lanes();
    } catch (...) {
    }
  }
  {
    std::lock_guard<std::mutex> lock(mu_);
    vars_.clear();
    live_.clear();
  }
  if (device_ >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device_);
    for (cudaStream_t s : lanes_) cudaStreamDestroy(s);
    cudaSetDevice(prev);
  }
}

void Engine::bind_device() const {
  if (device_ < 0) return;
  int cur = -1;
  CSB_CUDA(cudaGetDevice(&cur));
  if (cur != device_) CSB_CUDA(cudaSetDevice(device_));
}

int Engine::new_lane(int priority) {
  if (device_ < 0) throw UsageError("Engine: host-only engine has no stream lanes");
  std::lock_guard<std::mutex> lock(lanes_mu_);
  if (static_cast<int>(lanes_.size()) >= kMaxLanes) throw ConfigError("Engine: too many lanes");
  bind_device();
  int lo = 0, hi = 0;
  CSB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const int prio = std::max(hi, std::min(lo, priority));
  cudaStream_t s;
  CSB_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio));
  lanes_.push_back(s);
  return static_cast<int>(lanes_.size()) - 1;
}

cudaStream_t Engine::lane_stream(int lane) const {
  std::lock_guard<std::mutex> lock(lanes_mu_);
  if (lane < 0 || lane >= static_cast<int>(lanes_.size())) throw UsageError("Engine: unknown lane");
  return lanes_[static_cast<size_t>(lane)];
}

int Engine::num_lanes() const {
  std::lock_guard<std::mutex> lock(lanes_mu_);
  return static_cast<int>(lanes_.size());
}

Tag Engine::new_variable() {
  std::lock_guard<std::mutex> lock(mu_);
  uint64_t id = next_tag_++;
  vars_.emplace(id, VarRecord{});
  return Tag{id, engine_id_};
}

Engine::VarRecord& Engine::var_for(const Tag& tag) {
  if (tag.engine_id != engine_id_) throw UsageError("Engine: tag belongs to a different engine");
  auto it = vars_.find(tag.id);
  if (it == vars_.end()) throw UsageError("Engine: unknown tag");
  return it->second;
}

OpId Engine::push(std::function<void()> body, const std::vector<Tag>& reads,
                  const std::vector<Tag>& mutates, OpKind kind, int key) {
  auto op = std::make_unique<Operation>();
  op->host_body = std::move(body);
  op->kind = kind;
  op->key = key;
  op->dispatch = Dispatch::Host;
  return enqueue(std::move(op), reads, mutates);
}

OpId Engine::push_stream(std::function<void(cudaStream_t)> body, const std::vector<Tag>& reads,
                         const std::vector<Tag>& mutates, OpKind kind, int key, int lane,
                         Dispatch dispatch) {
  if (device_ < 0) throw UsageError("Engine: stream op pushed to a host-only engine");
  if (dispatch == Dispatch::Host) throw UsageError("Engine: stream ops dispatch Inline or Pool");
  if (lane < 0 || lane >= num_lanes()) throw UsageError("Engine: unknown lane");
  auto op = std::make_unique<Operation>();
  op->stream_body = std::move(body);
  op->kind = kind;
  op->key = key;
  op->lane = lane;
  op->dispatch = dispatch;
  return enqueue(std::move(op), reads, mutates);
}

OpId Engine::enqueue(std::unique_ptr<Operation> op, const std::vector<Tag>& reads,
                     const std::vector<Tag>& mutates) {
  OpId id;
  {
    hostprof::Scope prof(hostprof::kEnqueue);
    std::lock_guard<std::mutex> lock(mu_);
    if (shut_down_ || stopping_) throw UsageError("Engine: push after shutdown");
    if (!reads.empty() && !mutates.empty()) {
      std::vector<uint64_t> r;
      r.reserve(reads.size());
      for (const Tag& t : reads) r.push_back(t.id);
      std::sort(r.begin(), r.end());
      for (const Tag& m : mutates)
        if (std::binary_search(r.begin(), r.end(), m.id))
          throw UsageError("Engine: a tag may not appear in both reads and mutates");
    }
    for (const Tag& t : reads) var_for(t);
    for (const Tag& t : mutates) var_for(t);

    id = next_op_++;
    op->id = id;
    for (const Tag& t : reads) op->reads.push_back(t.id);
    for (const Tag& t : mutates) op->mutates.push_back(t.id);
    op->pending = static_cast<int>(op->reads.size() + op->mutates.size());
    Operation* raw = op.get();
    live_.emplace(id, std::move(op));

    if (trace_) {
      TraceEvent ev;
      ev.rank = rank_;
      ev.event = "op_pushed";
      ev.op = static_cast<int64_t>(id);
      ev.key = raw->key;
      ev.kind = op_kind_name(raw->kind);
      trace_->emit(std::move(ev));
    }

    if (raw->pending == 0) {
      raw->pending = 1;
      decrement_pending(raw);
    } else {
      for (uint64_t t : raw->reads) vars_[t].queue.push_back(QueueEntry{raw, false});
      for (uint64_t t : raw->mutates) {
        VarRecord& var = vars_[t];
        var.queue.push_back(QueueEntry{raw, true});
        var.writes_pushed++;
      }
      for (uint64_t t : raw->reads) grant_head(vars_[t]);
      for (uint64_t t : raw->mutates) grant_head(vars_[t]);
    }
  }
  drain_inline();
  return id;
}

// A grant hands the op the events it must wait on for this tag: the last
// dispatched write (reads), or that write plus every read dispatched since
// (writes).  Nothing conflicting can be dispatched on the tag until the
// granted op completes, so the snapshot stays exact.
void Engine::grant_head(VarRecord& var) {
  auto it = var.queue.begin();
  if (it == var.queue.end()) return;
  if (it->write) {
    if (!it->granted) {
      it->granted = true;
      if (var.last_write) it->op->deps.push_back(var.last_write);
      for (const EventRef& r : var.readers) it->op->deps.push_back(r);
      decrement_pending(it->op);
    }
    return;
  }
  for (; it != var.queue.end() && !it->write; ++it) {
    if (!it->granted) {
      it->granted = true;
      if (var.last_write) it->op->deps.push_back(var.last_write);
      decrement_pending(it->op);
    }
  }
}

void Engine::decrement_pending(Operation* op) {
  if (--op->pending == 0) {
    if (op->dispatch == Dispatch::Inline) {
      inline_ready_.push_back(op);
    } else {
      ready_.push_back(op);
      ready_count_.fetch_add(1, std::memory_order_release);
      if (sleepers_ > 0) work_cv_.notify_one();
    }
  }
}

void Engine::complete(Operation* op, EventRef done, std::exception_ptr failure) {
  if (failure && !poisoned_) {
    poisoned_ = true;
    first_failure_ = failure;
  }
  for (uint64_t t : op->reads) {
    VarRecord& var = vars_[t];
    auto it = std::find_if(var.queue.begin(), var.queue.end(),
                           [op](const QueueEntry& e) { return e.op == op && !e.write; });
    var.queue.erase(it);
    if (done) {
      // events on one lane complete in order: keep only the newest per lane,
      // so a tag that is read every step but rarely written stays O(lanes)
      auto same = std::find_if(var.readers.begin(), var.readers.end(),
                               [&](const EventRef& r) { return r->lane == done->lane; });
      if (same != var.readers.end()) *same = done;
      else var.readers.push_back(done);
    }
    grant_head(var);
  }
  for (uint64_t t : op->mutates) {
    VarRecord& var = vars_[t];
    auto it = std::find_if(var.queue.begin(), var.queue.end(),
                           [op](const QueueEntry& e) { return e.op == op && e.write; });
    var.queue.erase(it);
    var.writes_done++;
    var.last_write = done;
    var.readers.clear();
    grant_head(var);
  }
  live_.erase(op->id);
  ops_done_++;
  control_cv_.notify_all();
}

std::vector<const EventObj*> Engine::latest_per_lane(const std::vector<EventRef>& deps, int skip_lane) {
  std::vector<const EventObj*> out;
  for (const EventRef& d : deps) {
    if (!d || d->lane == skip_lane) continue;
    auto it = std::find_if(out.begin(), out.end(), [&](const EventObj* e) { return e->lane == d->lane; });
    if (it == out.end()) out.push_back(d.get());
    else if (d->seq > (*it)->seq) *it = d.get();
  }
  return out;
}

EventRef Engine::acquire_event(int lane) {
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> lock(pool_->mu);
    if (!pool_->free.empty()) {
      ev = pool_->free.back();
      pool_->free.pop_back();
    }
  }
  if (!ev) {
    CSB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    std::lock_guard<std::mutex> lock(pool_->mu);
    pool_->all.push_back(ev);
  }
  std::shared_ptr<EventPool> pool = pool_;
  EventRef ref(new EventObj{ev, lane}, [pool](EventObj* e) {
    {
      std::lock_guard<std::mutex> lock(pool->mu);
      pool->free.push_back(e->ev);
    }
    delete e;
  });
  return ref;
}

// Device waits double as the failure detector of device-side collectives
// (watch.hpp): every ~50 ms of waiting they poll the registered transports
// (NCCL asynchronous errors, a peer kernel's device timeout); on a failure
// or on this engine's watchdog every transport is aborted -- peer kernels
// leave their pair barriers, NCCL communicators are aborted, the ledgers
// latch -- before the error is thrown, so the device work drains instead of
// hanging the GPU (collective.cpp:92-105, 249-264: timeout -> report -> latch).
void Engine::device_wait_tick(std::chrono::steady_clock::time_point deadline,
                              std::chrono::steady_clock::time_point& next_poll, const char* what) {
  const auto now = std::chrono::steady_clock::now();
  if (now >= next_poll) {
    next_poll = now + std::chrono::milliseconds(50);
    const std::string m = watch::poll();
    if (!m.empty()) {
      watch::abort_all(m);
      throw DeadlockTimeout("Engine: device collective failed while waiting (" + std::string(what) + "): " + m);
    }
  }
  if (now > deadline) {
    const std::string m = std::string("Engine: device work not complete after ") +
                          std::to_string(watchdog_.count()) + " ms (" + what + ")";
    watch::abort_all(m);
    throw DeadlockTimeout(m);
  }
}

void Engine::sync_event(const EventRef& ev, const char* what) {
  if (!ev) return;
  const auto deadline = std::chrono::steady_clock::now() + watchdog_;
  auto next_poll = std::chrono::steady_clock::now() + std::chrono::milliseconds(50);
  // spin (yielding) for the engine's spin budget before sleeping: a sleep
  // overshoots by the kernel's timer slack (~50 us), which a synchronous
  // funnel pays once per collective
  const auto spin_until = std::chrono::steady_clock::now() + spin_;
  for (;;) {
    cudaError_t e = cudaEventQuery(ev->ev);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) throw_cuda(e, what, __FILE__, __LINE__);
    device_wait_tick(deadline, next_poll, what);
    if (std::chrono::steady_clock::now() < spin_until) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void Engine::sync_lanes() {
  if (device_ < 0) return;
  bind_device();
  std::vector<cudaStream_t> lanes;
  {
    std::lock_guard<std::mutex> lock(lanes_mu_);
    lanes = lanes_;
  }
  const auto deadline = std::chrono::steady_clock::now() + watchdog_;
  auto next_poll = std::chrono::steady_clock::now() + std::chrono::milliseconds(50);
  const auto spin_until = std::chrono::steady_clock::now() + spin_;
  for (cudaStream_t s : lanes) {
    for (;;) {
      cudaError_t e = cudaStreamQuery(s);
      if (e == cudaSuccess) break;
      if (e != cudaErrorNotReady) throw_cuda(e, "cudaStreamQuery", __FILE__, __LINE__);
      device_wait_tick(deadline, next_poll, "lane work");
      if (std::chrono::steady_clock::now() < spin_until) std::this_thread::yield();
      else std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
}

void Engine::run_op(Operation* op) {
  std::exception_ptr failure;
  EventRef done;
  auto emit = [&](const char* name) {
    if (!trace_) return;
    TraceEvent ev;
    ev.rank = rank_;
    ev.event = name;
    ev.op = static_cast<int64_t>(op->id);
    ev.key = op->key;
    ev.kind = op_kind_name(op->kind);
    trace_->emit(std::move(ev));
  };
  ConcurrencyGauges* gauges = trace_ ? &trace_->gauges() : nullptr;

  if (op->dispatch == Dispatch::Host) {
    try {
      for (const EventRef& d : op->deps) sync_event(d, "host op dependency");
    } catch (...) {
      failure = std::current_exception();
    }
    op->deps.clear();
    emit("op_started");
    if (gauges && op->kind == OpKind::Compute) gauges->compute_started();
    if (!failure) {
      try {
        op->host_body();
      } catch (...) {
        failure = std::current_exception();
      }
    }
    if (gauges && op->kind == OpKind::Compute) gauges->compute_finished();
    emit("op_finished");
  } else {
    cudaStream_t stream = nullptr;
    try {
      bind_device();
      stream = lane_stream(op->lane);
      // one wait per other lane -- its latest event; same-lane events are
      // already ordered (a DepCha pull over 161 keys would otherwise wait on
      // 161 events of the producer lane, ~0.2 us of host time each)
      const std::vector<const EventObj*> waits = latest_per_lane(op->deps, op->lane);
      hostprof::Scope prof(hostprof::kDispatchWait);
      for (const EventObj* d : waits) CSB_CUDA(cudaStreamWaitEvent(stream, d->ev, 0));
    } catch (...) {
      failure = std::current_exception();
    }
    op->deps.clear();
    emit("op_started");
    if (!failure) {
      hostprof::Scope prof(hostprof::kDispatchBody);
      try {
        op->stream_body(stream);
      } catch (...) {
        failure = std::current_exception();
      }
    }
    try {
      hostprof::Scope prof(hostprof::kDispatchRecord);
      if (stream) {
        done = acquire_event(op->lane);
        std::lock_guard<std::mutex> rec(rec_mu_);
        done->seq = ++lane_seq_[static_cast<size_t>(op->lane)];
        CSB_CUDA(cudaEventRecord(done->ev, stream));
      }
    } catch (...) {
      if (!failure) failure = std::current_exception();
      done.reset();
    }
    emit("op_finished");
  }
  hostprof::Scope prof(hostprof::kComplete);
  std::lock_guard<std::mutex> lock(mu_);
  complete(op, std::move(done), failure);
}

void Engine::drain_inline() {
  for (;;) {
    Operation* op = nullptr;
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (inline_ready_.empty()) return;
      op = inline_ready_.front();
      inline_ready_.pop_front();
    }
    run_op(op);
  }
}

// Worker 0 spins on the ready counter for a short while before blocking: a
// blocked thread takes tens of microseconds to wake, and every DepCha /
// ConCom collective is handed to the pool, so wake-up latency would
// otherwise serialize into the step (CSB_ENGINE_SPIN_US, default 1000).  The
// other workers block at once, so N ranks x T workers never oversubscribe
// the host cores (a rank's collectives become ready one at a time anyway).
void Engine::worker_loop(int index) {
  for (;;) {
    const auto spin_until = std::chrono::steady_clock::now() + (index == 0 ? spin_ : std::chrono::microseconds(0));
    while (ready_count_.load(std::memory_order_acquire) == 0 &&
           !stop_flag_.load(std::memory_order_relaxed) &&
           std::chrono::steady_clock::now() < spin_until) {
#if defined(__x86_64__)
      __builtin_ia32_pause();
#endif
    }
    Operation* op = nullptr;
    {
      std::unique_lock<std::mutex> lock(mu_);
      ++sleepers_;
      work_cv_.wait(lock, [this] { return stopping_ || !ready_.empty(); });
      --sleepers_;
      if (ready_.empty()) return;  // stopping and drained
      op = ready_.front();
      ready_.pop_front();
      ready_count_.fetch_sub(1, std::memory_order_relaxed);
    }
    run_op(op);
    drain_inline();
  }
}

void Engine::wait_for(const Tag& tag) {
  EventRef ev;
  {
    std::unique_lock<std::mutex> lock(mu_);
    VarRecord& var = var_for(tag);
    const uint64_t target = var.writes_pushed;
    control_cv_.wait(lock, [&var, target] { return var.writes_done >= target; });
    ev = var.last_write;
  }
  if (ev) {
    bind_device();
    sync_event(ev, "wait_for");
  }
}

OpId Engine::import_event(cudaEvent_t ev, const std::vector<Tag>& mutates, int key, int lane) {
  if (!ev) throw UsageError("Engine::import_event: null event");
  return push_stream([ev](cudaStream_t s) { CSB_CUDA(cudaStreamWaitEvent(s, ev, 0)); }, {}, mutates,
                     OpKind::Other, key, lane, Dispatch::Inline);
}

void Engine::stream_wait(const std::vector<Tag>& tags, cudaStream_t stream) {
  std::vector<EventRef> evs;
  {
    std::unique_lock<std::mutex> lock(mu_);
    for (const Tag& tag : tags) {
      VarRecord& var = var_for(tag);
      control_cv_.wait(lock, [&var] { return var.queue.empty(); });
      if (var.last_write) evs.push_back(var.last_write);
      for (const EventRef& r : var.readers) evs.push_back(r);
    }
  }
  const std::vector<const EventObj*> waits = latest_per_lane(evs, -1);
  if (waits.empty()) return;
  bind_device();
  for (const EventObj* e : waits) CSB_CUDA(cudaStreamWaitEvent(stream, e->ev, 0));
}

void Engine::wait_all() {
  {
    std::unique_lock<std::mutex> lock(mu_);
    const uint64_t target = next_op_;
    control_cv_.wait(lock, [this, target] { return ops_done_ >= target; });
  }
  sync_lanes();
  std::lock_guard<std::mutex> lock(mu_);
  if (poisoned_) std::rethrow_exception(first_failure_);
}

void Engine::shutdown() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (shut_down_) return;
    stopping_ = true;
    shut_down_ = true;
    stop_flag_.store(true);
    work_cv_.notify_all();
  }
  for (std::thread& t : workers_) t.join();
}

uint64_t Engine::ops_pushed() const { return next_op_.load(std::memory_order_acquire); }

uint64_t Engine::ops_completed() const { return ops_done_.load(std::memory_order_acquire); }

}  // namespace csb
