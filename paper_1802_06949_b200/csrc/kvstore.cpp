// kvstore.cpp -- see kvstore.hpp.  Reference anchors (R/core/src/kvstore.cpp):
//   construction / config checks   34-60
//   init (rank-0 world broadcast)  76-97
//   push (stage + per-mode comm)   99-143
//   pull (copy-out / depcha op)    145-183
//   barrier (drain + world)        185-193
#include "kvstore.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "hostprof.hpp"
#include "kernels.hpp"

namespace csb {

const char* kv_mode_name(KvMode m) {
  switch (m) {
    case KvMode::Funnel: return "funnel";
    case KvMode::DepCha: return "depcha";
    case KvMode::ConCom: return "concom";
    case KvMode::Naive: return "naive";
  }
  return "unknown";
}

KvMode parse_kv_mode(const std::string& name) {
  if (name == "funnel") return KvMode::Funnel;
  if (name == "depcha") return KvMode::DepCha;
  if (name == "concom") return KvMode::ConCom;
  if (name == "naive") return KvMode::Naive;
  throw ConfigError("unknown kvstore mode: " + name);
}

std::vector<int> create_communicators(Transport& transport, int count) {
  std::vector<int> comms;
  for (int i = 0; i < count; ++i) comms.push_back(transport.new_communicator());
  return comms;
}

namespace {
constexpr uint64_t kAlignBytes = 256;  // comm-slot alignment inside a fusion bucket

void* device_alloc_zeroed(size_t bytes) {
  void* p = nullptr;
  CSB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
  CSB_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 256)));
  return p;
}
}  // namespace

KvStore::KvStore(Engine& engine, Transport& transport, int rank, KvConfig config,
                 std::vector<int> concom_comms)
    : engine_(engine),
      transport_(transport),
      rank_(rank),
      cfg_(config),
      comms_(std::move(concom_comms)) {
  if (cfg_.num_keys < 1) throw ConfigError("KvStore: num_keys must be >= 1");
  if (cfg_.mode == KvMode::ConCom) {
    if (cfg_.outstanding < 1) throw ConfigError("KvStore: concom requires outstanding >= 1");
    if (static_cast<int>(comms_.size()) != cfg_.outstanding)
      throw ConfigError("KvStore: concom requires exactly `outstanding` communicators");
  }
  if (cfg_.comm_dtype >= 0) dtype_size(cfg_.comm_dtype);  // validates
  comm_dt_ = cfg_.comm_dtype;
  if (cfg_.p2p && cfg_.bucket_bytes == 0)
    throw ConfigError("KvStore: the peer-memory path needs fusion buckets (bucket_bytes > 0)");
  // Peer kernels pair CTAs across GPUs.  ConCom runs up to `outstanding` of
  // them concurrently (one per communicator stream): each grid is capped to
  // 1/outstanding of the device's resident CTAs and launched plainly, so all
  // of them are resident together and none can hold the SMs that another
  // communicator's peer-waiting grid needs (P2PArgs::concurrent).
  if (cfg_.p2p == 2 && cfg_.mode == KvMode::ConCom)
    throw ConfigError("KvStore: NVLS runs on one ordered comm stream (funnel/depcha)");
  // ZeRO-1 lives in DepCha's fused pull (Funnel/ConCom issue the collective
  // at push, before the weights are known)
  if (cfg_.zero && (cfg_.p2p != 1 || cfg_.mode != KvMode::DepCha))
    throw ConfigError("KvStore: ZeRO-1 runs on the peer-memory path (p2p = 1) under depcha");
  // one rank: nothing crosses NVLink, the collectives are the identity
  p2p_active_ = cfg_.p2p != 0 && transport_.p2p_capable();
  zero_active_ = p2p_active_ && cfg_.zero;
  static const bool n1_fuse = [] {
    const char* e = std::getenv("CSB_N1_FUSE");
    return !(e && std::string(e) == "0");
  }();
  // and across GPUs: DepCha's whole-bucket fused peer kernel stages the
  // gradients itself (CTA c packs the column its peers read after barrier 0)
  static const bool p2p_fuse = [] {
    const char* e = std::getenv("CSB_P2P_FUSE_PACK");
    return !(e && std::string(e) == "0");
  }();
  defer_pack_ = (n1_fuse && transport_.num_ranks() == 1 &&
                 (cfg_.mode == KvMode::DepCha || cfg_.mode == KvMode::Naive)) ||
                (p2p_fuse && p2p_active_ && cfg_.mode == KvMode::DepCha && cfg_.p2p == 1);
  if (engine_.device() < 0) throw ConfigError("KvStore: the engine must be bound to a CUDA device");
  keys_.resize(static_cast<size_t>(cfg_.num_keys));
  init_order_tag_ = engine_.new_variable();
  if (cfg_.mode == KvMode::DepCha) dummy_tag_ = engine_.new_variable();
  if (cfg_.mode == KvMode::Funnel) funnel_tag_ = engine_.new_variable();
  // Lanes: packs, collectives (one ordered stream per communicator) and
  // unpack/update run on separate CUDA streams, so bucket b's update
  // overlaps bucket b+1's collective; the engine's events order each key.
  world_lane_ = engine_.new_lane(cfg_.comm_priority);
  if (cfg_.mode == KvMode::ConCom)
    for (int i = 0; i < cfg_.outstanding; ++i) {
      comm_lanes_.push_back(engine_.new_lane(cfg_.comm_priority));
      comm_order_tags_.push_back(engine_.new_variable());
    }
  pack_lane_ = engine_.new_lane(cfg_.comm_priority);
  update_lane_ = engine_.new_lane(0);
  // CSB_KV_LANES=1: packs, world collectives and updates share one stream
  // (no cross-stream event hops; buckets then no longer overlap each other)
  static const bool one_lane = [] {
    const char* e = std::getenv("CSB_KV_LANES");
    return e && std::string(e) == "1";
  }();
  if (one_lane && cfg_.mode != KvMode::ConCom) pack_lane_ = update_lane_ = world_lane_;
}

KvStore::~KvStore() {
  try {
    engine_.wait_all();
  } catch (...) {
  }
  engine_.bind_device();
  for (const auto& peers : shared_) transport_.unshare_buffer(peers);
  for (KeyState& k : keys_)
    if (k.mom) cudaFree(k.mom);
  for (void* p : allocations_) cudaFree(p);
  nvls_free(nvls_);
}

void KvStore::check_key(int key, bool must_be_initialized) const {
  if (key < 0 || key >= cfg_.num_keys) throw UsageError("KvStore: key out of range");
  if (must_be_initialized && !keys_[static_cast<size_t>(key)].initialized)
    throw UsageError("KvStore: key not initialized");
}

uint64_t KvStore::key_numel(int key) const {
  check_key(key, true);
  return keys_[static_cast<size_t>(key)].numel;
}

void KvStore::key_map(int key, int* bucket, uint64_t* offset) {
  check_key(key, true);
  const KeyState& k = keys_[static_cast<size_t>(key)];
  if (k.bucket < 0) build_buckets();  // UsageError until every key is initialized
  *bucket = k.bucket;
  *offset = k.offset;
}

int KvStore::bucket_lane(int b) const {
  if (b < 0 || b >= num_buckets()) throw UsageError("KvStore: bucket out of range");
  return buckets_[static_cast<size_t>(b)].lane;
}

// ZeRO-1: the first fused op of a bucket seeds this rank's master shard from
// its (broadcast, identical) weights, on the op's stream before the kernel.
void KvStore::zero_fill_master(Bucket& B, const std::vector<DeviceTable::Entry>& es, int wdt, cudaStream_t s) {
  const int N = transport_.num_ranks();
  const uint64_t T = B.count / 8, s0 = T * rank_ / N, s1 = T * (rank_ + 1) / N;
  const uint64_t ws = dtype_size(wdt);
  char* master = static_cast<char*>(const_cast<void*>(B.wm_peers[static_cast<size_t>(rank_)]));
  std::vector<cs_copy_entry> copies;
  for (const DeviceTable::Entry& e : es) {
    const uint64_t g0 = std::max(e.gstart, s0), g1 = std::min(e.gend, s1);
    if (g0 >= g1) continue;
    const uint64_t e0 = (g0 - e.gstart) * 8, e1 = std::min<uint64_t>(e.n, (g1 - e.gstart) * 8);
    if (e0 >= e1) continue;
    copies.push_back(cs_copy_entry{static_cast<char*>(e.c) + e0 * ws, master + (g0 - s0) * 8 * ws, e1 - e0});
  }
  if (!copies.empty()) pack(copies.data(), static_cast<int>(copies.size()), wdt, wdt, s);
  B.master_ready = true;
}

void* KvStore::bucket_view(int key) {
  check_key(key, true);
  build_buckets();
  return key_ptr(key);
}

void KvStore::arena(void** base, uint64_t* bytes) {
  build_buckets();
  if (!arena_) throw UsageError("KvStore: no fusion-bucket arena (bucket_bytes = 0 keeps one buffer per key)");
  *base = arena_;
  *bytes = arena_bytes_;
}

std::vector<std::vector<int>> KvStore::bucket_groups() {
  build_buckets();
  std::vector<std::vector<int>> g;
  for (const Bucket& b : buckets_) g.push_back(b.keys);
  if (cfg_.bucket_bytes == 0 && cfg_.issue_order) std::reverse(g.begin(), g.end());
  return g;
}

void* KvStore::key_ptr(int key) const {
  const KeyState& k = keys_[static_cast<size_t>(key)];
  const Bucket& b = buckets_[static_cast<size_t>(k.bucket)];
  return static_cast<char*>(b.base) + k.offset * dtype_size(comm_dt_);
}

void KvStore::init(int key, TensorSlot weights) {
  check_key(key, false);
  KeyState& ks = keys_[static_cast<size_t>(key)];
  if (ks.initialized) throw UsageError("KvStore: duplicate init for key");
  if (key != initialized_count_) throw UsageError("KvStore: keys must be initialized densely, in order");
  if (weights.numel == 0) throw UsageError("Shape: extents must be >= 1");
  if (comm_dt_ < 0) comm_dt_ = weights.dtype;
  dtype_size(weights.dtype);
  ks.numel = weights.numel;
  ks.wdtype = weights.dtype;
  ks.initialized = true;
  ++initialized_count_;

  if (cfg_.bucket_bytes == 0) {
    // reference map: comm_buf[key] 1:1 with the key (kvstore.cpp:84)
    engine_.bind_device();
    Bucket b;
    b.keys = {key};
    b.tag = engine_.new_variable();
    b.count = ks.numel;
    b.base = device_alloc_zeroed(ks.numel * dtype_size(comm_dt_));
    allocations_.push_back(b.base);
    if (cfg_.mode == KvMode::ConCom) {
      b.comm = comms_[static_cast<size_t>(key % cfg_.outstanding)];  // kvstore.cpp:119
      b.lane = comm_lanes_[static_cast<size_t>(key % cfg_.outstanding)];
    } else {
      b.comm = Transport::world();
      b.lane = world_lane_;
    }
    ks.bucket = static_cast<int>(buckets_.size());
    ks.offset = 0;
    buckets_.push_back(b);
    built_ = (initialized_count_ == cfg_.num_keys);
  }

  // Rank 0's weights reach everyone through a world broadcast; the op
  // mutates the weights plus a store-wide ordering tag so each rank issues
  // its broadcasts in key order (kvstore.cpp:186-195).
  Transport* tr = &transport_;
  const int rank = rank_;
  void* data = weights.data;
  const uint64_t n = weights.numel;
  const int dt = weights.dtype;
  engine_.push_stream(
      [tr, rank, data, n, dt, key](cudaStream_t s) {
        tr->broadcast(Transport::world(), rank, 0, data, n, dt, key, s);
      },
      {}, {weights.tag, init_order_tag_}, OpKind::Collective, key, world_lane_, Dispatch::Pool);
}

// Fusion buckets: keys grouped greedily in issue order into buffers of at
// most bucket_bytes (a larger key gets its own bucket); every key slot is
// aligned to 256 B inside one zero-filled arena, so 16-byte vector access
// holds for every key and the padding sums to zero.
void KvStore::build_buckets() {
  if (built_) return;
  if (initialized_count_ != cfg_.num_keys)
    throw UsageError("KvStore: fusion buckets need every key initialized before the first push");
  const uint64_t es = dtype_size(comm_dt_);
  const uint64_t align = kAlignBytes / es;
  std::vector<int> order(static_cast<size_t>(cfg_.num_keys));
  for (int k = 0; k < cfg_.num_keys; ++k)
    order[static_cast<size_t>(k)] = cfg_.issue_order ? cfg_.num_keys - 1 - k : k;
  std::vector<Bucket> bs;
  Bucket cur;
  uint64_t cur_bytes = 0;
  for (int k : order) {
    const uint64_t bytes = keys_[static_cast<size_t>(k)].numel * es;
    if (!cur.keys.empty() && cur_bytes + bytes > cfg_.bucket_bytes) {
      bs.push_back(cur);
      cur = Bucket();
      cur_bytes = 0;
    }
    KeyState& ks = keys_[static_cast<size_t>(k)];
    ks.bucket = static_cast<int>(bs.size());
    ks.offset = cur.count;
    cur.keys.push_back(k);
    cur.count = (cur.count + ks.numel + align - 1) / align * align;
    cur_bytes += bytes;
  }
  if (!cur.keys.empty()) bs.push_back(cur);
  uint64_t total = 0;
  for (Bucket& b : bs) total += b.count;
  engine_.bind_device();
  char* arena = nullptr;
  if (p2p_active_ && cfg_.p2p == 2 && transport_.nvls_capable()) {
    // NVLink SHARP: the arena is bound to a multicast object on every rank
    nvls_ = transport_.alloc_nvls(total * es);
    arena = static_cast<char*>(nvls_.uc);
  } else {
    arena = static_cast<char*>(device_alloc_zeroed(total * es));
    allocations_.push_back(arena);
  }
  arena_ = arena;
  arena_bytes_ = total * es;
  uint64_t off = 0;
  for (size_t i = 0; i < bs.size(); ++i) {
    Bucket& b = bs[i];
    b.tag = engine_.new_variable();
    b.base = arena + off * es;
    off += b.count;
    if (cfg_.mode == KvMode::ConCom) {
      b.comm = comms_[i % static_cast<size_t>(cfg_.outstanding)];
      b.lane = comm_lanes_[i % static_cast<size_t>(cfg_.outstanding)];
    } else {
      b.comm = Transport::world();
      b.lane = world_lane_;
    }
  }
  if (p2p_active_ && nvls_.mc) {
    for (Bucket& b : bs) {
      const uint64_t boff = static_cast<uint64_t>(static_cast<char*>(b.base) - arena);
      b.mc = static_cast<char*>(nvls_.mc) + boff;
      b.peer_bufs.assign(static_cast<size_t>(transport_.num_ranks()), nullptr);
      b.peer_bufs[static_cast<size_t>(rank_)] = b.base;
    }
  } else if (p2p_active_) {
    // setup-phase collective: every rank maps every peer's arena (CUDA IPC)
    const std::vector<void*> peers = transport_.share_buffer(arena, rank_);
    shared_.push_back(peers);
    for (Bucket& b : bs) {
      const uint64_t boff = static_cast<uint64_t>(static_cast<char*>(b.base) - arena);
      for (void* p : peers) b.peer_bufs.push_back(static_cast<char*>(p) + boff);
    }
  }
  if (zero_active_) {
    // ZeRO-1 shards: master weights (IPC-shared: peers all-gather from them)
    // and momentum, each 1/N of the bucket, in shard-local layout
    zero_wdt_ = keys_[0].wdtype;
    for (const KeyState& k : keys_)
      if (k.wdtype != zero_wdt_) throw UsageError("KvStore: ZeRO-1 needs one weight dtype for every key");
    const uint64_t ws = dtype_size(zero_wdt_), ms = zero_wdt_ == CS_F64 ? 8 : 4;
    const int N = transport_.num_ranks();
    uint64_t shard_total = 0;
    for (const Bucket& b : bs) shard_total += p2p_shard_elems(b.count, N);
    void* master = device_alloc_zeroed(shard_total * ws);
    void* mom = device_alloc_zeroed(shard_total * ms);
    allocations_.push_back(master);
    allocations_.push_back(mom);
    const std::vector<void*> peers = transport_.share_buffer(master, rank_);
    shared_.push_back(peers);
    uint64_t soff = 0;
    for (Bucket& b : bs) {
      for (void* p : peers) b.wm_peers.push_back(static_cast<char*>(p) + soff * ws);
      b.mom_b = static_cast<char*>(mom) + soff * ms;
      soff += p2p_shard_elems(b.count, N);
    }
  }
  buckets_ = std::move(bs);
  built_ = true;
}

std::vector<std::pair<int, std::vector<int>>> KvStore::group_by_bucket(
    const std::vector<int>& keys) const {
  std::vector<std::pair<int, std::vector<int>>> groups;
  for (size_t i = 0; i < keys.size(); ++i) {
    const int b = keys_[static_cast<size_t>(keys[i])].bucket;
    auto it = std::find_if(groups.begin(), groups.end(), [b](const auto& g) { return g.first == b; });
    if (it == groups.end()) groups.push_back({b, {static_cast<int>(i)}});
    else it->second.push_back(static_cast<int>(i));
  }
  return groups;
}

void KvStore::push(const std::vector<int>& keys, const std::vector<TensorSlot>& grads) {
  hostprof::Scope prof(hostprof::kKvPush);
  if (keys.size() != grads.size()) throw UsageError("KvStore: keys and values differ in length");
  const uint32_t stamp = next_stamp();
  for (size_t i = 0; i < keys.size(); ++i) {
    check_key(keys[i], true);
    const KeyState& ks = keys_[static_cast<size_t>(keys[i])];
    if (grads[i].numel != ks.numel)
      throw UsageError("KvStore: pushed gradient shape differs from init shape");
    if (ks.pushed) throw UsageError("KvStore: key pushed twice without a pull");
    if (seen_[static_cast<size_t>(keys[i])] == stamp) throw UsageError("KvStore: duplicate key in one push");
    seen_[static_cast<size_t>(keys[i])] = stamp;
  }
  build_buckets();

  for (const auto& [b, idxs] : group_by_bucket(keys)) {
    Bucket& B = buckets_[static_cast<size_t>(b)];
    // stage every gradient of this call into its bucket slot: kernel (a),
    // one launch per bucket (kvstore.cpp:109 `copy(g, comm_buf)`)
    std::vector<cs_copy_entry> entries;
    std::vector<Tag> reads, muts;
    int src_dt = -1;
    for (int i : idxs) {
      const int k = keys[static_cast<size_t>(i)];
      const TensorSlot& g = grads[static_cast<size_t>(i)];
      if (src_dt < 0) src_dt = g.dtype;
      if (g.dtype != src_dt) throw UsageError("KvStore: one push mixes gradient dtypes in a bucket");
      if (g.data == key_ptr(k) && g.dtype == comm_dt_) B.view_tags.push_back(g.tag);  // in place
      else entries.push_back(cs_copy_entry{g.data, key_ptr(k), g.numel});
      reads.push_back(g.tag);
      keys_[static_cast<size_t>(k)].pushed = true;
    }
    const int key0 = keys[static_cast<size_t>(idxs[0])];
    // Funnel over peer memory with registered gradients: defer too -- the
    // bucket's collective reads the gradients in place if they all lie in
    // the region (issue_collective), else flushes the pack first
    const bool funnel_direct = p2p_active_ && cfg_.mode == KvMode::Funnel && !greg_peers_.empty();
    if ((defer_pack_ || funnel_direct) && (B.deferred_dt < 0 || B.deferred_dt == src_dt)) {
      // one rank: stage at the pull_update, fused with the update (or flushed
      // as this very pack op by any other use of the bucket)
      size_t j = 0;
      for (int i : idxs) {
        const int k = keys[static_cast<size_t>(i)];
        const TensorSlot& g = grads[static_cast<size_t>(i)];
        if (g.data == key_ptr(k) && g.dtype == comm_dt_) continue;  // a bucket view
        if (defer_src_.size() != keys_.size()) defer_src_.assign(keys_.size(), nullptr);
        defer_src_[static_cast<size_t>(k)] = entries[j].src;
        B.deferred.push_back({k, entries[j++]});
      }
      B.deferred_reads.insert(B.deferred_reads.end(), reads.begin(), reads.end());
      B.deferred_dt = src_dt;
    } else {
      flush_deferred(B);
      push_pack_op(B, entries, reads, src_dt, key0);
    }
    B.pushed += static_cast<int>(idxs.size());

    if (B.pushed == static_cast<int>(B.keys.size()) &&
        (cfg_.mode == KvMode::Funnel || cfg_.mode == KvMode::ConCom))
      issue_collective(b, reads);
  }
}

// kernel (a): stage the listed gradients into their bucket slots, one launch
// (kvstore.cpp:109 `copy(g, comm_buf)`), ordered after the gradients' writes
void KvStore::push_pack_op(Bucket& B, const std::vector<cs_copy_entry>& entries, const std::vector<Tag>& reads,
                           int src_dt, int key0) {
  const int dst_dt = comm_dt_;
  if (!B.pack_tab) B.pack_tab = std::make_shared<DeviceTable>();
  DeviceTable* tab = B.pack_tab.get();  // resident table; all its launches on pack_lane_
  engine_.push_stream(
      [entries, src_dt, dst_dt, tab](cudaStream_t s) {
        if (!entries.empty()) tab->pack(entries.data(), static_cast<int>(entries.size()), src_dt, dst_dt, s);
      },
      reads, {B.tag}, OpKind::Copy, key0, pack_lane_, Dispatch::Inline);
}

void KvStore::clear_deferred(Bucket& B) {
  for (const auto& [k, e] : B.deferred) defer_src_[static_cast<size_t>(k)] = nullptr;
  B.deferred.clear();
  B.deferred_reads.clear();
  B.deferred_dt = -1;
}

void KvStore::flush_deferred(Bucket& B) {
  if (B.deferred.empty() && B.deferred_reads.empty()) return;
  std::vector<cs_copy_entry> entries;
  for (const auto& [k, e] : B.deferred) entries.push_back(e);
  push_pack_op(B, entries, B.deferred_reads, B.deferred_dt, B.deferred.empty() ? B.keys[0] : B.deferred[0].first);
  clear_deferred(B);
}

void KvStore::issue_collective(int b, const std::vector<Tag>& extra_reads) {
  Bucket& B = buckets_[static_cast<size_t>(b)];
  std::vector<Tag> muts{B.tag};
  for (const Tag& t : B.view_tags) muts.push_back(t);  // rewritten in place
  const int key0 = B.keys[0];
  B.issued = true;
  KvStore* self = this;
  if (cfg_.mode == KvMode::Funnel) {
    // control-thread collective on the single ordered comm stream
    // (kvstore.cpp:112-116); the funnel tag keeps issue order = push order
    muts.push_back(funnel_tag_);
    // registered gradients: the peer kernel reads every rank's gradients in
    // place and writes the sums into every bucket -- no pack (§7.2)
    const bool direct = p2p_active_ && B.view_tags.empty() && B.deferred.size() == B.keys.size() &&
                        (B.deferred_dt < 0 || B.deferred_dt == comm_dt_) && deferred_in_region(B);
    if (!direct) flush_deferred(B);
    if (direct) {
      std::vector<DeviceTable::Entry> es;
      for (const auto& [k, e] : B.deferred) {
        const KeyState& ks = keys_[static_cast<size_t>(k)];
        const uint64_t g0 = ks.offset / 8;
        DeviceTable::Entry en{key_ptr(k), nullptr, nullptr, e.n, g0, g0 + (e.n + 7) / 8};
        en.d = const_cast<void*>(e.src);
        es.push_back(en);
      }
      std::sort(es.begin(), es.end(), [](const auto& x, const auto& y) { return x.gstart < y.gstart; });
      uint64_t layout = 1469598103934665603ull;  // FNV-1a of (slot, region offset), as the fused pull
      for (const auto& e : es)
        for (uint64_t v : {e.gstart, static_cast<uint64_t>(static_cast<const char*>(e.d) -
                                                           static_cast<const char*>(greg_base_))}) {
          layout ^= v;
          layout *= 1099511628211ull;
        }
      std::vector<Tag> reads = B.deferred_reads;
      clear_deferred(B);
      if (!B.p2p_tab) B.p2p_tab = std::make_shared<DeviceTable>();
      DeviceTable* ptab = B.p2p_tab.get();
      engine_.push_stream(
          [self, b, es, ptab, layout](cudaStream_t s) {
            Transport::P2PUpdate u;
            u.update = false;  // a plain allreduce of the in-place gradients into the buckets
            u.tab = ptab->resident(es, s);
            u.n_entries = static_cast<int>(es.size());
            u.gbase = self->greg_peers_.data();
            u.layout = layout;
            self->collective_body(self->buckets_[b], b, s, &u);
          },
          reads, muts, OpKind::Collective, key0, B.lane, Dispatch::Inline);
    } else {
      engine_.push_stream([self, b](cudaStream_t s) { self->collective_body(self->buckets_[b], b, s, nullptr); },
                          {}, muts, OpKind::Collective, key0, B.lane, Dispatch::Inline);
    }
    // The funnel: ONE thread performs every collective, synchronously.  The
    // reference's push waits for the gradient and runs the allreduce on the
    // calling (control) thread (kvstore.cpp:112-116), so nothing after it --
    // the next key, the next iteration's forward -- is issued before the
    // collective is done.  Same here: the control thread waits until this
    // bucket's collective has completed on the device.  (CSB_FUNNEL_ASYNC=1
    // only enqueues it, the stream order alone keeping the funnel order.)
    static const bool async = [] {
      const char* e = std::getenv("CSB_FUNNEL_ASYNC");
      return e && std::string(e) == "1";
    }();
    if (!async) engine_.wait_for(B.tag);
  } else {
    // offloaded collective on comms[b % outstanding] (kvstore.cpp:117-136).
    // Collectives of one communicator are chained in push order through the
    // communicator's order tag: two pool threads of one rank must not reach
    // the ledger out of order, or it would pair one key's buffer with
    // another's on the peers (equal counts match).  The reference leaves that
    // to the caller's barrier window (one call in flight per comm);
    // here a pushed-ahead window stays correct, and the communicators still
    // run concurrently with each other.
    for (size_t i = 0; i < comm_lanes_.size(); ++i)
      if (comm_lanes_[i] == B.lane) muts.push_back(comm_order_tags_[i]);
    std::atomic<int>* outstanding = &outstanding_;
    outstanding_.fetch_add(1);
    std::vector<Tag> reads;
    for (const Tag& t : extra_reads)
      if (std::none_of(B.view_tags.begin(), B.view_tags.end(), [&](const Tag& v) { return v.id == t.id; }))
        reads.push_back(t);
    engine_.push_stream(
        [self, b, outstanding](cudaStream_t s) {
          struct Drain {
            std::atomic<int>* c;
            ~Drain() {
              c->fetch_sub(1);
              c->notify_all();
            }
          } drain{outstanding};
          self->collective_body(self->buckets_[b], b, s, nullptr);
        },
        reads, muts, OpKind::Collective, key0, B.lane, Dispatch::Pool);
  }
}

Dispatch KvStore::depcha_dispatch() const {
  static const bool pool = [] {
    const char* e = std::getenv("CSB_DEPCHA_DISPATCH");
    return e && std::string(e) == "pool";
  }();
  if (cfg_.mode == KvMode::Naive || pool) return Dispatch::Pool;
  // an injected latency makes every collective block its dispatching host
  // thread (the reference's blocking MPI call, collective.cpp:249): then the
  // collectives belong on the pool, as in the reference (kvstore.cpp:163-179),
  // so the control thread keeps issuing the next step (acceptance 7)
  if (transport_.inject_latency().count() > 0) return Dispatch::Pool;
  return Dispatch::Inline;
}

// One bucket's allreduce on its communicator: NCCL (or the local rank-order
// kernel) by default, the peer-memory kernel when p2p is active (optionally
// fused with the update of the keys in `upd`).
void KvStore::collective_body(const Bucket& B, int b, cudaStream_t s, const Transport::P2PUpdate* upd) {
  const int bid = cfg_.bucket_bytes ? b : -1;
  if (p2p_active_) {
    transport_.allreduce_p2p(B.comm, rank_, B.peer_bufs.data(), B.count, comm_dt_, B.keys[0], s, bid, upd,
                             B.mc, cfg_.mode == KvMode::ConCom ? cfg_.outstanding : 1);
  } else {
    transport_.allreduce_sum(B.comm, rank_, B.base, B.count, comm_dt_, B.keys[0], s, bid);
  }
}

void KvStore::pull(const std::vector<int>& keys, const std::vector<TensorSlot>& outs) {
  pull_impl(keys, outs, nullptr);
}

void KvStore::pull_update(const std::vector<int>& keys, const std::vector<TensorSlot>& weights,
                          const SgdConfig& sgd) {
  pull_impl(keys, weights, &sgd);
}

void KvStore::ensure_momentum(int key, int wdt) {
  KeyState& ks = keys_[static_cast<size_t>(key)];
  if (ks.mom) return;
  engine_.bind_device();
  const size_t es = (wdt == CS_F64) ? 8 : 4;
  CSB_CUDA(cudaMalloc(&ks.mom, std::max<size_t>(ks.numel * es, 256)));
  CSB_CUDA(cudaMemset(ks.mom, 0, std::max<size_t>(ks.numel * es, 256)));
  // one-time: zeroed before any lane touches it (the legacy stream only: a
  // device-wide sync would wait on colocated ranks' peer kernels)
  CSB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

void KvStore::pull_impl(const std::vector<int>& keys, const std::vector<TensorSlot>& outs,
                        const SgdConfig* sgd) {
  hostprof::Scope prof(hostprof::kKvPull);
  if (keys.size() != outs.size()) throw UsageError("KvStore: keys and values differ in length");
  const uint32_t stamp = next_stamp();
  for (size_t i = 0; i < keys.size(); ++i) {
    check_key(keys[i], true);
    const KeyState& ks = keys_[static_cast<size_t>(keys[i])];
    if (!ks.pushed) throw UsageError("KvStore: pull without a preceding push this iteration");
    if (outs[i].numel != ks.numel) throw UsageError("KvStore: pull output shape differs from init shape");
    if (seen_[static_cast<size_t>(keys[i])] == stamp) throw UsageError("KvStore: duplicate key in one pull");
    seen_[static_cast<size_t>(keys[i])] = stamp;
  }
  const bool momentum = sgd && sgd->momentum != 0.0;

  for (const auto& [b, idxs] : group_by_bucket(keys)) {
    Bucket& B = buckets_[static_cast<size_t>(b)];
    if (B.pushed != static_cast<int>(B.keys.size()))
      throw UsageError("KvStore: pull of a fusion bucket before all of its keys were pushed");
    // one rank: a whole-bucket pull_update (into the comm dtype's supported
    // weights) stages and updates in one kernel; anything else packs first
    const bool whole_upd = sgd && !B.issued && B.pulled == 0 && idxs.size() == B.keys.size();
    const bool deferred = !B.deferred_reads.empty();
    const bool fuse = deferred && whole_upd && !p2p_active_ &&
                      DeviceTable::pack_sgd_supported(B.deferred_dt < 0 ? comm_dt_ : B.deferred_dt, comm_dt_,
                                                      outs[static_cast<size_t>(idxs[0])].dtype);
    const bool fuse_p2p = deferred && whole_upd && p2p_active_ && (B.deferred_dt < 0 || B.deferred_dt == comm_dt_);
    if (!fuse && !fuse_p2p) flush_deferred(B);
    std::vector<Tag> buf_tags{B.tag}, out_tags;
    for (const Tag& t : B.view_tags) buf_tags.push_back(t);
    std::vector<cs_copy_entry> copies;
    std::vector<cs_update_entry> updates;
    int out_dt = -1;
    for (int i : idxs) {
      const int k = keys[static_cast<size_t>(i)];
      const TensorSlot& o = outs[static_cast<size_t>(i)];
      if (out_dt < 0) out_dt = o.dtype;
      if (o.dtype != out_dt) throw UsageError("KvStore: one pull mixes output dtypes in a bucket");
      if (!sgd && o.data == key_ptr(k) && o.dtype == comm_dt_) continue;  // a bucket view: already in place
      out_tags.push_back(o.tag);
      if (sgd) {
        if (momentum && !zero_active_) ensure_momentum(k, o.dtype);  // ZeRO-1 keeps a momentum shard
        updates.push_back(cs_update_entry{o.data, key_ptr(k), keys_[static_cast<size_t>(k)].mom, o.numel});
      } else {
        copies.push_back(cs_copy_entry{key_ptr(k), o.data, o.numel});
      }
    }
    const int cdt = comm_dt_;
    const SgdConfig opt = sgd ? *sgd : SgdConfig{};
    const bool upd = sgd != nullptr;
    // unpack (kvstore.cpp:160/170 copy) or the fused SGD update, kernel (a)/(c),
    // through the bucket's resident tables (all launched on update_lane_)
    if (!B.upd_tab) B.upd_tab = std::make_shared<DeviceTable>();
    if (!B.unpack_tab) B.unpack_tab = std::make_shared<DeviceTable>();
    DeviceTable* utab = B.upd_tab.get();
    DeviceTable* ctab = B.unpack_tab.get();
    auto finish = [copies, updates, cdt, out_dt, opt, upd, utab, ctab](cudaStream_t s) {
      if (upd) utab->sgd(updates.data(), static_cast<int>(updates.size()), out_dt, cdt, opt.lr,
                         opt.rescale, opt.momentum, s);
      else if (!copies.empty()) ctab->pack(copies.data(), static_cast<int>(copies.size()), cdt, out_dt, s);
    };
    const int key0 = keys[static_cast<size_t>(idxs[0])];

    if ((cfg_.mode == KvMode::DepCha || cfg_.mode == KvMode::Naive) && !B.issued) {
      // the reference pushes one op {allreduce; copy-out} mutating {out,
      // dummy} (kvstore.cpp:163-179).  Here the collective is its own op on
      // the ordered comm stream -- it rewrites the comm buffer, so it is
      // modelled as a write (the reference holds only a read grant there) --
      // and carries the dummy tag, so collectives stay chained in push order;
      // the copy-out / update follows as an op on the update lane.
      // this op updates every key of the bucket, so nothing reads the
      // bucket afterwards: keep only the own shard of the sum locally.
      // Validated before any bucket / key state changes (a rejected call
      // leaves the bucket as it was).
      const bool whole = B.pulled == 0 && idxs.size() == B.keys.size();
      if (p2p_active_ && upd && zero_active_ && (!whole || out_dt != zero_wdt_))
        throw UsageError("KvStore: ZeRO-1 needs pull_update of whole fusion buckets into the init weights' dtype");
      std::vector<Tag> muts{B.tag};
      for (const Tag& t : B.view_tags) muts.push_back(t);  // rewritten in place
      if (cfg_.mode == KvMode::DepCha) muts.push_back(dummy_tag_);
      const int ckey = B.keys[0];
      B.issued = true;
      KvStore* self = this;
      const int bi = b;
      if (p2p_active_ && upd) {
        // peer-memory path: ONE kernel does the NVLink allreduce of the
        // bucket and the SGD / momentum update of these keys (phase 2 reads
        // the reduced gradient from the local bucket), mutating the weights
        std::vector<DeviceTable::Entry> es;
        for (size_t j = 0; j < updates.size(); ++j) {
          const int k = keys[static_cast<size_t>(idxs[j])];
          const KeyState& ks = keys_[static_cast<size_t>(k)];
          const uint64_t g0 = ks.offset / 8;
          es.push_back(DeviceTable::Entry{updates[j].g, updates[j].mom, updates[j].w, updates[j].n, g0,
                                          g0 + (updates[j].n + 7) / 8});
          if (fuse_p2p)  // the kernel stages this key's gradient (d) into its slot (a)
            if (const void* src = deferred_src(k)) es.back().d = const_cast<void*>(src);
        }
        std::vector<Tag> p2p_reads;
        if (fuse_p2p) {
          // the pushed gradients; bucket views are already among the writes
          for (const Tag& t : B.deferred_reads)
            if (std::none_of(B.view_tags.begin(), B.view_tags.end(), [&](const Tag& v) { return v.id == t.id; }))
              p2p_reads.push_back(t);
          clear_deferred(B);
        }
        std::sort(es.begin(), es.end(), [](const auto& x, const auto& y) { return x.gstart < y.gstart; });
        // direct: every staged gradient lies in the registered region -> the
        // kernel reads all ranks' copies in place and stages nothing.  The
        // (slot, offset) layout is hashed into the ledger signature, so ranks
        // whose regions are laid out differently fail with MismatchError
        // before any launch instead of reading wrong addresses.
        bool direct = fuse_p2p && !greg_peers_.empty();
        uint64_t layout = 1469598103934665603ull;  // FNV-1a
        for (const auto& e : es) {
          if (!direct) break;
          const char* d = static_cast<const char*>(e.d);
          const char* base = static_cast<const char*>(greg_base_);
          if (!d || d == e.a || d < base || d + e.n * dtype_size(comm_dt_) > base + greg_bytes_ ||
              (reinterpret_cast<uintptr_t>(d) & 15u) != 0) {
            direct = false;
            break;
          }
          for (uint64_t v : {e.gstart, static_cast<uint64_t>(d - base)}) {
            layout ^= v;
            layout *= 1099511628211ull;
          }
        }
        if (!B.p2p_tab) B.p2p_tab = std::make_shared<DeviceTable>();
        DeviceTable* ptab = B.p2p_tab.get();  // all its uploads on B.lane
        for (const Tag& t : out_tags) muts.push_back(t);
        const bool zero = zero_active_;
        engine_.push_stream(
            [self, bi, es, ptab, out_dt, opt, whole, zero, fuse_p2p, direct, layout](cudaStream_t s) {
              Bucket& Bk = self->buckets_[bi];
              Transport::P2PUpdate u;
              u.tab = ptab->resident(es, s);
              u.n_entries = static_cast<int>(es.size());
              u.wdt = out_dt;
              u.lr = opt.lr;
              u.rescale = opt.rescale;
              u.momentum = opt.momentum;
              u.shard_only = whole;
              u.pack = fuse_p2p && !direct;
              if (direct) {
                u.gbase = self->greg_peers_.data();
                u.layout = layout;
              }
              if (zero) {
                if (!Bk.master_ready) self->zero_fill_master(Bk, es, out_dt, s);
                u.wm = Bk.wm_peers.data();
                u.mom_b = Bk.mom_b;
              }
              self->collective_body(Bk, bi, s, &u);
            },
            p2p_reads, muts, OpKind::Collective, ckey, B.lane, depcha_dispatch());
        for (int i : idxs) keys_[static_cast<size_t>(keys[static_cast<size_t>(i)])].pushed = false;
        B.pulled += static_cast<int>(idxs.size());
        if (B.pulled == static_cast<int>(B.keys.size())) {
          B.pushed = 0;
          B.pulled = 0;
          B.issued = false;
          B.view_tags.clear();
        }
        continue;
      }
      engine_.push_stream([self, bi](cudaStream_t s) { self->collective_body(self->buckets_[bi], bi, s, nullptr); },
                          {}, muts, OpKind::Collective, ckey, B.lane, depcha_dispatch());
    }
    if (fuse) {
      // (a)+(c) in one op after the (identity) collective: reads the pushed
      // gradients, writes the bucket and the weights.  Registered gradients
      // (register_grads) are read in place and not staged into the bucket
      // either -- the one-rank twin of the peer kernels' direct reads: the
      // bucket then keeps no copy of this step's gradients (as under ZeRO-1).
      const bool in_place = deferred_in_region(B);
      std::vector<DeviceTable::PackUpdate> pu;
      for (int i : idxs) {
        const int k = keys[static_cast<size_t>(i)];
        const TensorSlot& o = outs[static_cast<size_t>(i)];
        const void* g = key_ptr(k);  // a bucket view: already in place
        if (const void* src = deferred_src(k)) g = src;
        void* slot = in_place ? const_cast<void*>(g) : key_ptr(k);  // slot == g: no staging store
        pu.push_back(DeviceTable::PackUpdate{g, slot, o.data, keys_[static_cast<size_t>(k)].mom, o.numel});
      }
      std::vector<Tag> reads;
      for (const Tag& t : B.deferred_reads)
        if (std::none_of(B.view_tags.begin(), B.view_tags.end(), [&](const Tag& v) { return v.id == t.id; }))
          reads.push_back(t);
      for (const Tag& t : B.view_tags) reads.push_back(t);
      std::vector<Tag> fmuts{B.tag};
      for (const Tag& t : out_tags) fmuts.push_back(t);
      if (!B.fused_tab) B.fused_tab = std::make_shared<DeviceTable>();
      DeviceTable* ftab = B.fused_tab.get();  // resident table, update lane only
      const int gdt = B.deferred_dt < 0 ? comm_dt_ : B.deferred_dt;
      engine_.push_stream(
          [pu, gdt, cdt, out_dt, opt, ftab](cudaStream_t s) {
            ftab->pack_sgd(pu, gdt, cdt, out_dt, opt.lr, opt.rescale, opt.momentum, s);
          },
          reads, fmuts, OpKind::Compute, key0, update_lane_, Dispatch::Inline);
      clear_deferred(B);
    } else {
      engine_.push_stream(finish, buf_tags, out_tags, upd ? OpKind::Compute : OpKind::Copy, key0,
                          update_lane_, Dispatch::Inline);
    }
    for (int i : idxs) keys_[static_cast<size_t>(keys[static_cast<size_t>(i)])].pushed = false;
    B.pulled += static_cast<int>(idxs.size());
    if (B.pulled == static_cast<int>(B.keys.size())) {
      B.pushed = 0;
      B.pulled = 0;
      B.issued = false;
      B.view_tags.clear();
    }
  }
}

// Setup collective (every rank, same order): the region holding this rank's
// gradients, mapped into every peer.  Whole-bucket pull_updates whose pushed
// gradients all lie inside it then let the fused peer kernel read every
// rank's gradients in place: push stages nothing (kvstore.cpp:109's copy is
// skipped; the gradients' tags are read by the collective op, so they stay
// unmodified until every rank has read them).
void KvStore::register_grads(void* base, uint64_t bytes) {
  if (!base || bytes == 0) throw UsageError("KvStore: empty gradient region");
  if (greg_base_) throw UsageError("KvStore: a gradient region is already registered");
  greg_base_ = base;
  greg_bytes_ = bytes;
  if (!p2p_active_) return;  // one rank: the fused pull reads the region in place (no peers to map)
  engine_.bind_device();
  std::vector<void*> peers = transport_.share_buffer(base, rank_);
  shared_.push_back(peers);
  greg_peers_.assign(peers.begin(), peers.end());
}

// every deferred gradient of B lies in the registered region (16-B aligned)
bool KvStore::deferred_in_region(const Bucket& B) const {
  if (!greg_base_ || B.deferred.empty()) return false;
  const char* base = static_cast<const char*>(greg_base_);
  const size_t es = dtype_size(B.deferred_dt < 0 ? comm_dt_ : B.deferred_dt);
  for (const auto& [k, e] : B.deferred) {
    const char* d = static_cast<const char*>(e.src);
    if (d < base || d + e.n * es > base + greg_bytes_ || (reinterpret_cast<uintptr_t>(d) & 15u) != 0) return false;
  }
  return true;
}

// kvstore.cpp:185-193: drain the in-flight counter, then a world barrier.
void KvStore::barrier() {
  if (cfg_.mode != KvMode::ConCom) return;
  for (int v = outstanding_.load(); v != 0; v = outstanding_.load()) outstanding_.wait(v);
  engine_.bind_device();
  transport_.barrier(Transport::world(), rank_, -1, engine_.lane_stream(world_lane_));
}

void KvStore::comm_buf(int key, void* host_out) {
  check_key(key, true);
  const KeyState& ks = keys_[static_cast<size_t>(key)];
  if (ks.bucket < 0) throw UsageError("KvStore: comm buffer not allocated yet");
  flush_deferred(buckets_[static_cast<size_t>(ks.bucket)]);
  engine_.wait_for(buckets_[static_cast<size_t>(ks.bucket)].tag);
  engine_.bind_device();
  CSB_CUDA(cudaMemcpy(host_out, key_ptr(key), ks.numel * dtype_size(comm_dt_), cudaMemcpyDeviceToHost));
}

}  // namespace csb
