// trainer.hpp -- synthetic training step driving the KvStore with the
// reference trainer's loop shapes (R/core/src/trainer.cpp:89-151).
//
// The reference's forward/backward of a toy MLP is out of scope;
// here a synthetic backward replaces it: one producer op per key, in
// descending key order (backward produces the last layer first,
// trainer.cpp:64-71), writing the key's gradient and holding the device for
// a calibrated time.  Gradients are the reference's synthetic inputs:
// random_uniform(n_k, 1000 + r*K + k) (test_kvstore.cpp:304), weights
// random_uniform(n_k, mix_seed(7, k)) on rank 0, broadcast at init
// (kvstore.cpp:95).  Generated on the host with std::mt19937_64, the same
// generator the reference uses (tensor.cpp:28-38).
#pragma once

#include <vector>

#include "kvstore.hpp"

namespace csb {

struct SynthConfig {
  KvMode mode = KvMode::DepCha;
  std::vector<uint64_t> sizes;
  int wdt = CS_F32;
  int gdt = CS_F32;
  int cdt = CS_F32;
  uint64_t bucket_bytes = 0;
  int issue_order = 0;
  int outstanding = 1;
  double lr = 0.1;
  double rescale = 1.0;
  double momentum = 0.0;
  uint64_t backward_ns = 0;  // total synthetic backward device time per step
  int backward_ctas = 0;     // 0: one CTA per SM
  bool fused = true;         // pull_update (kernel (c) on the reduced bucket)
  int comm_priority = 0;
  bool host_source = false;  // gradients arrive from pinned host memory (e2e)
  int p2p = 0;               // NVLink peer-memory collectives (KvConfig::p2p)
  bool grad_views = false;   // produce gradients in place in the comm buckets (KvStore::bucket_view)
  int zero = 0;              // ZeRO-1 sharded update (KvConfig::zero)
  bool direct_grads = false; // register the gradient arena (KvStore::register_grads): in-place peer reads
  int order_seed = 0;        // != 0: per-rank random gradient-ready order (deadlock stress)
  uint64_t seed_base = 1000;
  // Measured gradient-ready time of every key from the start of a real
  // backward (tools/calibrate_backward.py).  When set, producers run in
  // ready order and key k holds the device for ready[k] - ready[previous],
  // replacing the size-proportional split of backward_ns.
  std::vector<double> ready_ms;
};

enum SynthFlags {
  kStepBackward = 1,     // producer ops (synthetic backward or H2D copies)
  kStepComm = 2,         // kvstore push / pull(+update) per mode loop
  kStepLocalUpdate = 4,  // no kvstore: local SGD from the local gradient
  kStepChecksum = 8,     // weight checksum -> 8-byte D2H read of the result
};

class SynthModel {
 public:
  SynthModel(Engine& engine, Transport& transport, int rank, int nranks, SynthConfig cfg,
             std::vector<int> concom_comms);
  ~SynthModel();
  void init();
  void enqueue_step(int flags);
  // Device time of `steps` steps (CUDA events spanning every lane).
  double run(int steps, int flags);
  // Wall-clock of `steps` steps, each ending with the host reading the result.
  double run_e2e(int steps, int flags);
  double checksum();
  // Every key's weights, concatenated without padding, into host memory
  // (bytes = sum n_k * sizeof(wdt)); waits for this rank's work first.
  void read_weights(void* host, uint64_t bytes);
  // host time the last run() spent enqueueing (dispatching every op)
  double last_host_ms() const { return last_host_ms_; }
  uint64_t grad_bytes() const;
  uint64_t h2d_bytes_per_step() const;
  int num_buckets() { return static_cast<int>(kv_.bucket_groups().size()); }
  KvStore& store() { return kv_; }

 private:
  Engine& engine_;
  Transport& transport_;
  const int rank_, nranks_;
  SynthConfig cfg_;
  KvStore kv_;
  std::vector<void*> w_, g_, src_;
  std::vector<Tag> wt_, gt_;
  std::vector<uint64_t> spin_ns_;
  std::vector<int> produce_order_;  // producer order (descending keys or measured ready order)
  char* w_arena_ = nullptr;
  uint64_t w_arena_elems_ = 0;
  char* g_arena_ = nullptr;
  uint64_t g_arena_bytes_ = 0;
  char* src_arena_ = nullptr;  // device (synthetic) or pinned host (e2e)
  void* h2d_dst_ = nullptr;    // e2e upload target: the gradient arena, or the bucket arena (views)
  // two checksum slots, so the host can read step t's result while step t+1
  // is already queued (run_e2e)
  double* sum_dev_ = nullptr;
  double* sum_host_ = nullptr;
  Tag sum_tag_[2];
  int sum_next_ = 0;  // slot of the next checksum
  int sum_last_ = 0;  // slot of the last enqueued checksum
  std::vector<std::vector<int>> groups_;
  std::vector<void*> mom_local_;  // momentum of the no-kvstore update path
  double last_host_ms_ = 0.0;
  DeviceTable local_tab_;  // the no-kvstore update's resident kernel table
};

}  // namespace csb
