// kvstore.hpp -- per-rank init/push/pull/barrier facade (reference:
// R/core/include/collsim/kvstore.hpp:13-96, R/core/src/kvstore.cpp).
//
// Schedules (kvstore.hpp:39-53 of the reference), B200 treatment:
//   funnel  push stages the gradient and issues the allreduce from the
//           control thread onto ONE ordered comm stream; collectives carry
//           a funnel ordering tag so they are issued in push order.
//   depcha  push only stages; pull issues one op {allreduce; unpack/update}
//           that also mutates the shared dummy tag, so the engine's in-order
//           write rule chains the collectives: every rank issues them in
//           the same order, and the GPU sees a cudaStreamWaitEvent chain.
//   concom  push stages, then hands the allreduce to the pool on
//           comms[bucket % outstanding], one NCCL communicator and one
//           CUDA stream each; barrier() drains the in-flight counter and
//           runs a world barrier.
//   naive   depcha without the dummy tag (deliberately broken; the ledger
//           turns the misordering into MismatchError / DeadlockTimeout).
// Extensions: comm buffers in any dtype (fp32 grads -> bf16 buckets),
// fusion buckets (keys grouped in issue order, one collective per bucket),
// list push/pull (MXNet KVStore key lists), and pull fused with the SGD /
// momentum update (kernel (c) reads the reduced bucket, the copy-back of
// kvstore.cpp:160/170 disappears).
#pragma once

#include <atomic>
#include <vector>

#include "engine.hpp"
#include "kernels.hpp"
#include "transport.hpp"

namespace csb {

enum class KvMode { Funnel = 0, DepCha = 1, ConCom = 2, Naive = 3 };
const char* kv_mode_name(KvMode m);
KvMode parse_kv_mode(const std::string& name);

struct KvConfig {
  KvMode mode = KvMode::Funnel;
  int outstanding = 1;
  int num_keys = 0;
  int comm_dtype = -1;        // -1: dtype of the init weights
  uint64_t bucket_bytes = 0;  // 0: one buffer per key (reference map)
  int issue_order = 0;        // bucket grouping order: 0 ascending, 1 descending
  int comm_priority = 0;      // CUDA stream priority of the comm lanes
  // Peer-memory collectives over NVLink instead of NCCL (needs fusion
  // buckets and a peer-capable NCCL transport): bit-exact rank-order sums,
  // and DepCha's pull_update becomes ONE fused allreduce+update kernel.
  int p2p = 0;
  // ZeRO-1 over the fused kernel (p2p == 1): master weights + momentum of the
  // own shard only; the kernel all-gathers the updated weights.
  int zero = 0;
};

// Non-owning device view + engine tag (kvstore.hpp:16-19).
struct TensorSlot {
  void* data = nullptr;
  int dtype = CS_F32;
  uint64_t numel = 0;
  Tag tag;
};

struct SgdConfig {
  double lr = 0.1;
  double rescale = 1.0;
  double momentum = 0.0;
};

std::vector<int> create_communicators(Transport& transport, int count);

class KvStore {
 public:
  KvStore(Engine& engine, Transport& transport, int rank, KvConfig config,
          std::vector<int> concom_comms = {});
  ~KvStore();
  KvStore(const KvStore&) = delete;
  KvStore& operator=(const KvStore&) = delete;

  // kvstore.cpp:76-97: keys densely in order; rank 0's weights broadcast.
  void init(int key, TensorSlot weights);
  // kvstore.cpp:99-143 / 145-183, one key (the reference calls) or a list
  // (one pack / one collective per fusion bucket).
  void push(int key, TensorSlot grad) { push(std::vector<int>{key}, std::vector<TensorSlot>{grad}); }
  void pull(int key, TensorSlot out) { pull(std::vector<int>{key}, std::vector<TensorSlot>{out}); }
  void push(const std::vector<int>& keys, const std::vector<TensorSlot>& grads);
  void pull(const std::vector<int>& keys, const std::vector<TensorSlot>& outs);
  // pull fused with sgd_update (model.cpp:17-27; + momentum): the update reads
  // the reduced bucket directly; with p2p, DepCha does the allreduce and the
  // update in ONE kernel (ZeRO-1 with cfg.zero).
  void pull_update(const std::vector<int>& keys, const std::vector<TensorSlot>& weights,
                   const SgdConfig& sgd);
  // kvstore.cpp:185-193 (ConCom: drain the window, then a world barrier).
  void barrier();

  int rank() const { return rank_; }
  const KvConfig& config() const { return cfg_; }
  int outstanding_in_flight() const { return outstanding_.load(); }
  // Synchronizes the key's comm buffer and copies it to host memory.
  void comm_buf(int key, void* host_out);
  int comm_dtype() const { return comm_dt_; }
  uint64_t key_numel(int key) const;
  // Builds the fusion buckets first when every key is initialized (a
  // setup-phase collective with the peer-memory path: call it on every rank).
  void key_map(int key, int* bucket, uint64_t* offset);
  int num_buckets() const { return static_cast<int>(buckets_.size()); }
  int bucket_lane(int b) const;
  // Keys of every comm bucket, buckets in issue order (builds the map).
  std::vector<std::vector<int>> bucket_groups();
  // Bucket views (DDP's gradient-as-bucket-view): the device address of the
  // key's slot in its comm bucket, in the comm dtype.  A gradient produced
  // there and pushed with that address is not copied (push only orders it);
  // the collective then rewrites it in place.  Builds the buckets.
  void* bucket_view(int key);
  // Setup collective: register the allocation holding this rank's gradients
  // (same layout on every rank) so the fused kernels read them in place
  // instead of staging them into the buckets (N > 1: over NVLink from every
  // peer; one rank: the fused pack+update kernel skips the staging store).
  void register_grads(void* base, uint64_t bytes);
  // The fusion-bucket arena (one allocation holding every bucket).
  void arena(void** base, uint64_t* bytes);

 private:
  struct KeyState {
    uint64_t numel = 0;
    int wdtype = -1;
    bool initialized = false;
    bool pushed = false;
    int bucket = -1;
    uint64_t offset = 0;  // elements into the bucket buffer
    void* mom = nullptr;  // momentum state (lazy)
  };
  struct Bucket {
    std::vector<int> keys;  // in bucket order
    uint64_t count = 0;     // elements in the collective (incl. alignment padding)
    void* base = nullptr;
    int pushed = 0;
    int pulled = 0;
    bool issued = false;  // collective issued this iteration
    int comm = 0;
    int lane = 0;
    Tag tag;  // engine tag of the whole comm buffer
    std::shared_ptr<DeviceTable> pack_tab, upd_tab, unpack_tab, p2p_tab;  // resident kernel tables
    std::vector<void*> peer_bufs;  // p2p: this bucket on every rank (IPC-mapped)
    void* mc = nullptr;            // nvls: this bucket's multicast VA
    // tags of pushed gradients that ARE this bucket's slots (bucket views):
    // the collective mutates them and the copy-out / update reads them, so a
    // producer's next write waits for both
    std::vector<Tag> view_tags;
    // ZeRO-1: every rank's master-weight shard of this bucket, this rank's
    // momentum shard (shard-local layout), filled from the weights at the
    // first pull_update
    std::vector<const void*> wm_peers;
    void* mom_b = nullptr;
    bool master_ready = false;
    // One rank (the allreduce is the identity): DepCha's staging copy is
    // deferred from push to the pull_update and fused with the update in one
    // kernel (DeviceTable::pack_sgd); any other use of the bucket flushes it
    // as the ordinary pack op first.
    std::vector<std::pair<int, cs_copy_entry>> deferred;  // (key, staging copy)
    std::vector<Tag> deferred_reads;                      // the pushed gradients' tags
    int deferred_dt = -1;
    std::shared_ptr<DeviceTable> fused_tab;
  };

  void check_key(int key, bool must_be_initialized) const;
  void build_buckets();
  std::vector<std::pair<int, std::vector<int>>> group_by_bucket(const std::vector<int>& keys) const;
  void issue_collective(int b, const std::vector<Tag>& extra_reads);
  void pull_impl(const std::vector<int>& keys, const std::vector<TensorSlot>& outs,
                 const SgdConfig* sgd);
  void* key_ptr(int key) const;
  void ensure_momentum(int key, int wdt);
  bool use_p2p() const { return p2p_active_; }
  // DepCha collectives: the dummy tag already fixes their order, so they can
  // be dispatched by the granting thread (no pool hand-off per collective);
  // naive keeps the pool (its hazard comes from racing pool threads).
  // CSB_DEPCHA_DISPATCH=pool restores the reference's pool dispatch.
  Dispatch depcha_dispatch() const;
  void collective_body(const Bucket& B, int bucket_id, cudaStream_t s, const Transport::P2PUpdate* upd);
  void zero_fill_master(Bucket& B, const std::vector<DeviceTable::Entry>& es, int wdt, cudaStream_t s);
  void push_pack_op(Bucket& B, const std::vector<cs_copy_entry>& entries, const std::vector<Tag>& reads, int src_dt,
                    int key0);
  void flush_deferred(Bucket& B);
  void clear_deferred(Bucket& B);
  // key -> staging source of its deferred pack (nullptr: none), kept in step
  // with every bucket's `deferred` list: O(1) lookups in pull
  std::vector<const void*> defer_src_;
  // register_grads(): this rank's region and every rank's mapping of theirs
  void* greg_base_ = nullptr;
  uint64_t greg_bytes_ = 0;
  std::vector<const void*> greg_peers_;
  bool deferred_in_region(const Bucket& B) const;
  const void* deferred_src(int k) const {
    return static_cast<size_t>(k) < defer_src_.size() ? defer_src_[static_cast<size_t>(k)] : nullptr;
  }

  Engine& engine_;
  Transport& transport_;
  const int rank_;
  const KvConfig cfg_;
  std::vector<int> comms_;
  int comm_dt_ = -1;
  std::vector<KeyState> keys_;
  std::vector<Bucket> buckets_;
  std::vector<void*> allocations_;
  int world_lane_ = 0;
  int pack_lane_ = 0;
  int update_lane_ = 0;
  std::vector<int> comm_lanes_;  // concom: lane per extra communicator
  std::vector<Tag> comm_order_tags_;  // concom: per-communicator issue-order chain
  Tag init_order_tag_;
  Tag dummy_tag_;
  Tag funnel_tag_;
  int initialized_count_ = 0;
  bool built_ = false;
  bool p2p_active_ = false;
  NvlsBuffer nvls_;  // p2p == 2: the multicast-bound comm arena
  void* arena_ = nullptr;
  uint64_t arena_bytes_ = 0;
  bool zero_active_ = false;  // ZeRO-1 (cfg_.zero over an active peer-memory path)
  bool defer_pack_ = false;   // one rank, DepCha / naive: pack fused into the pull_update (CSB_N1_FUSE=0: off)
  std::vector<std::vector<void*>> shared_;  // share_buffer results, unmapped at destruction
  int zero_wdt_ = -1;
  std::vector<uint32_t> seen_;  // duplicate-key detection in one call
  uint32_t stamp_ = 0;
  uint32_t next_stamp() {
    if (seen_.size() != keys_.size()) seen_.assign(keys_.size(), 0);
    return ++stamp_;
  }
  std::atomic<int> outstanding_{0};
};

}  // namespace csb
