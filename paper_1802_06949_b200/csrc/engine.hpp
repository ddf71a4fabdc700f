// engine.hpp -- dependency engine mapped onto CUDA streams and events.
//
// Keeps the reference Engine API (R/core/include/collsim/engine.hpp:41-74):
// tags, push(body, reads, mutates, kind, key), wait_for, wait_all, shutdown,
// and its grant rules (engine.cpp:113-133): per tag a FIFO; the head write is
// granted exclusively; a maximal head run of reads is granted together;
// writes to a tag are therefore issued in push order.
//
// What changes on the B200 is what "granted" and "complete" mean:
//   * a *stream op* (push_stream) is dispatched once every conflicting earlier
//     op has been DISPATCHED -- not finished.  Dispatch makes the op's lane
//     stream wait (cudaStreamWaitEvent) on the CUDA events those ops recorded
//     (last write for a read; last write + reads since for a write), runs the
//     body to enqueue device work, and records the op's own event.  Device
//     dependencies are resolved by the GPU; the host never blocks on them.
//   * Dispatch::Inline ops are dispatched by whichever thread grants them
//     (normally the control thread inside push), with no pool hand-off.
//     Dispatch::Pool ops run on the worker pool because their body may block
//     on the host (a collective's cross-rank matching rendezvous).
//   * a *host op* (push with a void() body, the reference signature) runs on
//     the pool after its dependencies have COMPLETED on the device
//     (cudaEventSynchronize), exactly the reference semantics.
// wait_for / wait_all wait for dispatch, then for the device events, under a
// watchdog; wait_all rethrows the first body failure (engine.cpp:224-231).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "trace.hpp"

namespace csb {

struct Tag {
  uint64_t id = 0;
  uint64_t engine_id = 0;
};

using OpId = uint64_t;

enum class OpKind { Compute, Copy, Collective, Other };
enum class Dispatch { Inline, Pool, Host };

const char* op_kind_name(OpKind kind);

class Engine;

// A recorded CUDA event, returned to its engine's pool when the last
// reference (tag state or pending dependency) drops.
struct EventObj {
  cudaEvent_t ev = nullptr;
  int lane = -1;
  // position in its lane's record order: a wait for the latest event of a
  // lane covers every earlier one (stream order), so dependency lists keep
  // one event per lane
  uint64_t seq = 0;
};
using EventRef = std::shared_ptr<EventObj>;

class Engine {
 public:
  // device < 0: host-only engine (no CUDA calls; stream ops rejected).
  Engine(int num_worker_threads, int rank = 0, TraceSink* trace = nullptr, int device = -1);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  Tag new_variable();

  // Reference signature (engine.hpp:57-58): host body on the pool.
  OpId push(std::function<void()> body, const std::vector<Tag>& reads,
            const std::vector<Tag>& mutates, OpKind kind = OpKind::Other, int key = -1);

  // Stream body: enqueues device work on lane's stream.
  OpId push_stream(std::function<void(cudaStream_t)> body, const std::vector<Tag>& reads,
                   const std::vector<Tag>& mutates, OpKind kind = OpKind::Other, int key = -1,
                   int lane = 0, Dispatch dispatch = Dispatch::Inline);

  void wait_for(const Tag& tag);
  void wait_all();

  // Interop with an external CUDA stream (a framework's compute stream).
  // import_event: a stream op on `lane` that waits on `ev` and mutates
  // `mutates` -- the external producer's writes (recorded by `ev`) become the
  // tags' latest writes.  stream_wait: blocks the host until every op pushed
  // so far on `tags` is dispatched, then makes `stream` wait on their last
  // write and the reads since, so the external stream may read or write them.
  OpId import_event(cudaEvent_t ev, const std::vector<Tag>& mutates, int key = -1, int lane = 0);
  void stream_wait(const std::vector<Tag>& tags, cudaStream_t stream);
  void shutdown();

  // Lane 0 exists from construction (the compute lane).  priority follows
  // cudaStreamCreateWithPriority (lower = higher priority, <= 0).
  int new_lane(int priority = 0);
  cudaStream_t lane_stream(int lane) const;
  int num_lanes() const;
  int device() const { return device_; }
  int rank() const { return rank_; }
  uint64_t engine_id() const { return engine_id_; }
  Tag tag_of(uint64_t id) const { return Tag{id, engine_id_}; }
  int num_threads() const { return static_cast<int>(workers_.size()); }
  uint64_t ops_pushed() const;
  uint64_t ops_completed() const;
  void set_watchdog(std::chrono::milliseconds ms) { watchdog_ = ms; }
  std::chrono::milliseconds watchdog() const { return watchdog_; }
  TraceSink* trace() const { return trace_; }

  // Makes the calling thread's current device the engine's device.
  void bind_device() const;

 private:
  struct Operation {
    std::function<void()> host_body;
    std::function<void(cudaStream_t)> stream_body;
    std::vector<uint64_t> reads;
    std::vector<uint64_t> mutates;
    std::vector<EventRef> deps;
    int pending = 0;
    OpId id = 0;
    OpKind kind = OpKind::Other;
    int key = -1;
    int lane = 0;
    Dispatch dispatch = Dispatch::Host;
  };
  struct QueueEntry {
    Operation* op;
    bool write;
    bool granted = false;
  };
  struct VarRecord {
    std::deque<QueueEntry> queue;
    uint64_t writes_pushed = 0;
    uint64_t writes_done = 0;  // dispatched (stream ops) / finished (host ops)
    EventRef last_write;       // null: no device write outstanding
    std::vector<EventRef> readers;
  };

  OpId enqueue(std::unique_ptr<Operation> op, const std::vector<Tag>& reads,
               const std::vector<Tag>& mutates);
  void worker_loop(int index);
  void run_op(Operation* op);         // no lock held
  void grant_head(VarRecord& var);    // mu_ held
  void decrement_pending(Operation* op);  // mu_ held
  void complete(Operation* op, EventRef done, std::exception_ptr failure);  // mu_ held
  void drain_inline();                // no lock held
  VarRecord& var_for(const Tag& tag); // mu_ held
  EventRef acquire_event(int lane);
  static std::vector<const EventObj*> latest_per_lane(const std::vector<EventRef>& deps, int skip_lane);
  void sync_event(const EventRef& ev, const char* what);
  void sync_lanes();
  void device_wait_tick(std::chrono::steady_clock::time_point deadline,
                        std::chrono::steady_clock::time_point& next_poll, const char* what);

  const uint64_t engine_id_;
  const int rank_;
  TraceSink* trace_;
  const int device_;
  std::chrono::milliseconds watchdog_{600000};

  mutable std::mutex mu_;
  std::condition_variable work_cv_;
  std::condition_variable control_cv_;
  std::unordered_map<uint64_t, VarRecord> vars_;
  std::deque<Operation*> ready_;         // pool / host dispatch
  std::deque<Operation*> inline_ready_;  // dispatched by the granting thread
  std::unordered_map<OpId, std::unique_ptr<Operation>> live_;
  uint64_t next_tag_ = 0;
  std::atomic<OpId> next_op_{0};      // written under mu_, read lock-free
  std::atomic<uint64_t> ops_done_{0};  // written under mu_, read lock-free
  bool stopping_ = false;
  bool shut_down_ = false;
  bool poisoned_ = false;
  std::exception_ptr first_failure_;
  std::vector<std::thread> workers_;
  std::atomic<int> ready_count_{0};
  std::atomic<bool> stop_flag_{false};
  int sleepers_ = 0;  // mu_
  std::chrono::microseconds spin_{1000};

  std::vector<cudaStream_t> lanes_;
  mutable std::mutex lanes_mu_;
  std::mutex rec_mu_;  // seq assignment and cudaEventRecord in one step (same order)
  std::vector<uint64_t> lane_seq_;  // per lane, sized at construction

  std::shared_ptr<struct EventPool> pool_;
};

}  // namespace csb
