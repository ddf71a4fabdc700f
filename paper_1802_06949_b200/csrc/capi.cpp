// capi.cpp -- the extern "C" boundary (include/collsim_b200.h).  Every entry
// point converts C++ exceptions into a status code + thread-local message;
// nothing throws across the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "collsim_b200.h"
#include "engine.hpp"
#include "hostprof.hpp"
#include "kernels.hpp"
#include "kvstore.hpp"
#include "trainer.hpp"
#include "transport.hpp"

using namespace csb;

struct cs_trace {
  TraceSink sink;
};
struct cs_engine {
  std::unique_ptr<Engine> e;
};
struct cs_transport {
  std::unique_ptr<Transport> t;
};
struct cs_kvstore {
  std::unique_ptr<KvStore> kv;
  Engine* engine;
};
struct cs_synth {
  std::unique_ptr<SynthModel> m;
};

namespace {
thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return CS_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CS_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return CS_ERR_INTERNAL;
  }
}

std::vector<Tag> tags_of(const Engine& e, const uint64_t* ids, int n) {
  if (n < 0 || (n > 0 && !ids)) throw UsageError("Engine: bad tag list");
  std::vector<Tag> v;
  v.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v.push_back(e.tag_of(ids[i]));
  return v;
}

OpKind kind_of(int k) {
  switch (k) {
    case CS_OP_COMPUTE: return OpKind::Compute;
    case CS_OP_COPY: return OpKind::Copy;
    case CS_OP_COLLECTIVE: return OpKind::Collective;
    case CS_OP_OTHER: return OpKind::Other;
  }
  throw UsageError("Engine: unknown op kind");
}

TensorSlot slot_of(const Engine& e, const cs_slot& s) {
  TensorSlot t;
  t.data = s.data;
  t.dtype = s.dtype;
  t.numel = s.numel;
  t.tag = e.tag_of(s.tag);
  dtype_size(s.dtype);
  if (s.numel > 0 && !s.data) throw UsageError("KvStore: null tensor data");
  return t;
}

#define CHECK_HANDLE(h) \
  if (!(h)) throw UsageError("null handle")
}  // namespace

extern "C" {

const char* cs_last_error(void) { return g_last_error.c_str(); }

const char* cs_status_name(int status) {
  switch (status) {
    case CS_OK: return "OK";
    case CS_ERR_CONFIG: return "ConfigError";
    case CS_ERR_USAGE: return "UsageError";
    case CS_ERR_MISMATCH: return "MismatchError";
    case CS_ERR_DEADLOCK: return "DeadlockTimeout";
    case CS_ERR_ENGINE: return "EngineError";
    case CS_ERR_CUDA: return "CudaError";
    case CS_ERR_NCCL: return "NcclError";
  }
  return "InternalError";
}

int cs_version(void) { return 10000; }

int cs_device_count(int* out) {
  return guard([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
      cudaGetLastError();
      n = 0;
    } else if (e != cudaSuccess) {
      throw_cuda(e, "cudaGetDeviceCount", __FILE__, __LINE__);
    }
    *out = n;
  });
}

// ------------------------------------------------------------ kernels
int cs_pack(const cs_copy_entry* entries, int n_entries, cs_dtype src_dt, cs_dtype dst_dt,
            cs_stream_t stream) {
  return guard([&] { pack(entries, n_entries, src_dt, dst_dt, reinterpret_cast<cudaStream_t>(stream)); });
}

int cs_sum_buffers(const void* const* in, int m, void* const* out, int nout, uint64_t n,
                   cs_dtype dt, cs_stream_t stream) {
  return guard([&] { sum_buffers(in, m, out, nout, n, dt, reinterpret_cast<cudaStream_t>(stream)); });
}

int cs_sgd_update(const cs_update_entry* entries, int n_entries, cs_dtype w_dt, cs_dtype g_dt,
                  double lr, double rescale, double momentum, cs_stream_t stream) {
  return guard([&] {
    sgd_update(entries, n_entries, w_dt, g_dt, lr, rescale, momentum,
               reinterpret_cast<cudaStream_t>(stream));
  });
}

int cs_synth_backward(const void* src, void* dst, uint64_t n, cs_dtype dt, uint64_t spin_ns,
                      int ctas, cs_stream_t stream) {
  return guard([&] {
    synth_backward(src, dst, n, dt, spin_ns, ctas, reinterpret_cast<cudaStream_t>(stream));
  });
}

int cs_checksum(const void* x, uint64_t n, cs_dtype dt, double* out_dev, cs_stream_t stream) {
  return guard([&] { checksum(x, n, dt, out_dev, reinterpret_cast<cudaStream_t>(stream)); });
}

// -------------------------------------------------------------- trace
int cs_trace_create(cs_trace_t* out) {
  return guard([&] { *out = new cs_trace(); });
}
int cs_trace_destroy(cs_trace_t t) {
  return guard([&] { delete t; });
}
int cs_trace_count(cs_trace_t t, uint64_t* out) {
  return guard([&] {
    CHECK_HANDLE(t);
    *out = t->sink.count();
  });
}
int cs_trace_write_jsonl(cs_trace_t t, const char* path) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->sink.write_jsonl(path);
  });
}
int cs_trace_gauges(cs_trace_t t, int* max_open, int* overlap) {
  return guard([&] {
    CHECK_HANDLE(t);
    *max_open = t->sink.gauges().max_open_collectives();
    *overlap = t->sink.gauges().compute_overlap() ? 1 : 0;
  });
}

// ------------------------------------------------------------- engine
int cs_engine_create(int num_worker_threads, int rank, int device, cs_trace_t trace,
                     cs_engine_t* out) {
  return guard([&] {
    auto h = std::make_unique<cs_engine>();
    h->e = std::make_unique<Engine>(num_worker_threads, rank, trace ? &trace->sink : nullptr, device);
    *out = h.release();
  });
}
int cs_engine_destroy(cs_engine_t e) {
  return guard([&] { delete e; });
}
int cs_engine_new_variable(cs_engine_t e, uint64_t* tag) {
  return guard([&] {
    CHECK_HANDLE(e);
    *tag = e->e->new_variable().id;
  });
}
int cs_engine_push_host(cs_engine_t e, cs_host_fn fn, void* arg, const uint64_t* reads, int n_reads,
                        const uint64_t* mutates, int n_mutates, int kind, int key, uint64_t* op_id) {
  return guard([&] {
    CHECK_HANDLE(e);
    if (!fn) throw UsageError("Engine: null body");
    OpId id = e->e->push([fn, arg] { if (fn(arg) != 0) throw EngineError("host op body failed"); }, tags_of(*e->e, reads, n_reads),
                         tags_of(*e->e, mutates, n_mutates), kind_of(kind), key);
    if (op_id) *op_id = id;
  });
}
int cs_engine_push_stream(cs_engine_t e, cs_stream_fn fn, void* arg, const uint64_t* reads,
                          int n_reads, const uint64_t* mutates, int n_mutates, int kind, int key,
                          int lane, int dispatch, uint64_t* op_id) {
  return guard([&] {
    CHECK_HANDLE(e);
    if (!fn) throw UsageError("Engine: null body");
    if (dispatch != CS_DISPATCH_INLINE && dispatch != CS_DISPATCH_POOL)
      throw UsageError("Engine: stream ops dispatch inline or on the pool");
    OpId id = e->e->push_stream(
        [fn, arg](cudaStream_t s) { if (fn(arg, reinterpret_cast<cs_stream_t>(s)) != 0) throw EngineError("stream op body failed"); },
        tags_of(*e->e, reads, n_reads), tags_of(*e->e, mutates, n_mutates), kind_of(kind), key,
        lane, dispatch == CS_DISPATCH_POOL ? Dispatch::Pool : Dispatch::Inline);
    if (op_id) *op_id = id;
  });
}
int cs_engine_wait_for(cs_engine_t e, uint64_t tag) {
  return guard([&] {
    CHECK_HANDLE(e);
    e->e->wait_for(e->e->tag_of(tag));
  });
}
int cs_engine_import_event(cs_engine_t e, void* cuda_event, const uint64_t* mutates, int n_mutates,
                           int key, int lane, uint64_t* op_id) {
  return guard([&] {
    CHECK_HANDLE(e);
    OpId id = e->e->import_event(static_cast<cudaEvent_t>(cuda_event), tags_of(*e->e, mutates, n_mutates),
                                 key, lane);
    if (op_id) *op_id = id;
  });
}
int cs_engine_stream_wait(cs_engine_t e, const uint64_t* tags, int n_tags, cs_stream_t stream) {
  return guard([&] {
    CHECK_HANDLE(e);
    e->e->stream_wait(tags_of(*e->e, tags, n_tags), reinterpret_cast<cudaStream_t>(stream));
  });
}
int cs_engine_wait_all(cs_engine_t e) {
  return guard([&] {
    CHECK_HANDLE(e);
    e->e->wait_all();
  });
}
int cs_engine_shutdown(cs_engine_t e) {
  return guard([&] {
    CHECK_HANDLE(e);
    e->e->shutdown();
  });
}
int cs_engine_new_lane(cs_engine_t e, int priority, int* lane) {
  return guard([&] {
    CHECK_HANDLE(e);
    *lane = e->e->new_lane(priority);
  });
}
int cs_engine_lane_stream(cs_engine_t e, int lane, cs_stream_t* out) {
  return guard([&] {
    CHECK_HANDLE(e);
    *out = reinterpret_cast<cs_stream_t>(e->e->lane_stream(lane));
  });
}
int cs_engine_stats(cs_engine_t e, uint64_t* pushed, uint64_t* completed) {
  return guard([&] {
    CHECK_HANDLE(e);
    *pushed = e->e->ops_pushed();
    *completed = e->e->ops_completed();
  });
}
int cs_engine_set_watchdog(cs_engine_t e, int64_t ms) {
  return guard([&] {
    CHECK_HANDLE(e);
    if (ms < 1) throw UsageError("Engine: watchdog must be >= 1 ms");
    e->e->set_watchdog(std::chrono::milliseconds(ms));
  });
}
int cs_engine_num_threads(cs_engine_t e, int* out) {
  return guard([&] {
    CHECK_HANDLE(e);
    *out = e->e->num_threads();
  });
}

// ---------------------------------------------------------- transport
int cs_transport_create_local(int num_ranks, int watchdog_ms, cs_trace_t trace, cs_transport_t* out) {
  return guard([&] {
    auto h = std::make_unique<cs_transport>();
    h->t = Transport::create_local(num_ranks, std::chrono::milliseconds(watchdog_ms),
                                   trace ? &trace->sink : nullptr);
    *out = h.release();
  });
}
int cs_transport_create_local_peer(int num_ranks, int watchdog_ms, cs_trace_t trace, cs_transport_t* out) {
  return guard([&] {
    auto h = std::make_unique<cs_transport>();
    h->t = Transport::create_local(num_ranks, std::chrono::milliseconds(watchdog_ms),
                                   trace ? &trace->sink : nullptr, true);
    *out = h.release();
  });
}
int cs_transport_create_nccl(const char* name, int num_ranks, int rank, int device, int watchdog_ms,
                             cs_trace_t trace, cs_transport_t* out) {
  return guard([&] {
    auto h = std::make_unique<cs_transport>();
    h->t = Transport::create_nccl(name ? name : "", num_ranks, rank, device,
                                  std::chrono::milliseconds(watchdog_ms),
                                  trace ? &trace->sink : nullptr);
    *out = h.release();
  });
}
int cs_transport_create_ledger_only(const char* name, int num_ranks, int rank, int watchdog_ms,
                                    cs_trace_t trace, cs_transport_t* out) {
  return guard([&] {
    auto h = std::make_unique<cs_transport>();
    h->t = Transport::create_ledger_only(name ? name : "", num_ranks, rank,
                                         std::chrono::milliseconds(watchdog_ms),
                                         trace ? &trace->sink : nullptr);
    *out = h.release();
  });
}
int cs_transport_destroy(cs_transport_t t) {
  return guard([&] { delete t; });
}
int cs_transport_num_ranks(cs_transport_t t, int* out) {
  return guard([&] {
    CHECK_HANDLE(t);
    *out = t->t->num_ranks();
  });
}
int cs_transport_num_communicators(cs_transport_t t, int* out) {
  return guard([&] {
    CHECK_HANDLE(t);
    *out = t->t->num_communicators();
  });
}
int cs_transport_new_communicator(cs_transport_t t, int* comm) {
  return guard([&] {
    CHECK_HANDLE(t);
    *comm = t->t->new_communicator();
  });
}
int cs_transport_set_inject_latency(cs_transport_t t, int64_t us) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->t->set_inject_latency(std::chrono::microseconds(us));
  });
}
int cs_transport_abort(cs_transport_t t) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->t->abort("Transport: aborted by the caller");
  });
}
int cs_allreduce_sum(cs_transport_t t, int comm, int rank, void* buf, uint64_t n, cs_dtype dt,
                     int trace_key, cs_stream_t stream) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->t->allreduce_sum(comm, rank, buf, n, dt, trace_key, reinterpret_cast<cudaStream_t>(stream));
  });
}
int cs_broadcast(cs_transport_t t, int comm, int rank, int root, void* buf, uint64_t n, cs_dtype dt,
                 int trace_key, cs_stream_t stream) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->t->broadcast(comm, rank, root, buf, n, dt, trace_key, reinterpret_cast<cudaStream_t>(stream));
  });
}
int cs_barrier(cs_transport_t t, int comm, int rank, int trace_key, cs_stream_t stream) {
  return guard([&] {
    CHECK_HANDLE(t);
    t->t->barrier(comm, rank, trace_key, reinterpret_cast<cudaStream_t>(stream));
  });
}

int cs_transport_p2p_capable(cs_transport_t t, int* out) {
  return guard([&] {
    CHECK_HANDLE(t);
    *out = t->t->p2p_capable() ? 1 : 0;
  });
}
int cs_transport_share_buffer(cs_transport_t t, void* base, void** ptrs_out) {
  return guard([&] {
    CHECK_HANDLE(t);
    std::vector<void*> p = t->t->share_buffer(base);
    for (size_t i = 0; i < p.size(); ++i) ptrs_out[i] = p[i];
  });
}
int cs_transport_share_buffer_rank(cs_transport_t t, int rank, void* base, void** ptrs_out) {
  return guard([&] {
    CHECK_HANDLE(t);
    std::vector<void*> p = t->t->share_buffer(base, rank);
    for (size_t i = 0; i < p.size(); ++i) ptrs_out[i] = p[i];
  });
}
int cs_transport_device_failure(cs_transport_t t, char* buf, int cap) {
  return guard([&] {
    CHECK_HANDLE(t);
    const std::string m = t->t->async_failure();
    if (cap > 0) {
      const size_t n = std::min<size_t>(m.size(), static_cast<size_t>(cap) - 1);
      std::memcpy(buf, m.data(), n);
      buf[n] = '\0';
    }
  });
}
int cs_transport_p2p_stamps(cs_transport_t t, int rank, uint64_t* out, int cap, int* n) {
  return guard([&] {
    CHECK_HANDLE(t);
    const std::vector<uint64_t> v = t->t->p2p_stamps(rank);
    const int m = std::min(cap, static_cast<int>(v.size()));
    if (m > 0) std::memcpy(out, v.data(), sizeof(uint64_t) * static_cast<size_t>(m));
    if (n) *n = static_cast<int>(v.size());
  });
}
namespace {
struct P2PTables {  // resident tables of the C-ABI p2p entry point, per stream
  std::mutex mu;
  std::unordered_map<cudaStream_t, std::unique_ptr<DeviceTable>> by_stream;
};
P2PTables& p2p_tables() {
  static P2PTables t;
  return t;
}
}  // namespace
namespace {
void p2p_call(cs_transport_t t, int comm, int rank, void* const* peer_bufs, void* mc, uint64_t n, cs_dtype dt,
              int trace_key, const cs_p2p_update* upd, cs_stream_t stream);
}
int cs_transport_nvls_capable(cs_transport_t t, int* out) {
  return guard([&] {
    CHECK_HANDLE(t);
    *out = t->t->nvls_capable() ? 1 : 0;
  });
}
int cs_transport_alloc_nvls(cs_transport_t t, uint64_t bytes, void** uc, void** mc) {
  return guard([&] {
    CHECK_HANDLE(t);
    NvlsBuffer b = t->t->alloc_nvls(bytes);  // lives as long as the process (bench / tests)
    *uc = b.uc;
    *mc = b.mc;
  });
}
int cs_allreduce_nvls(cs_transport_t t, int comm, int rank, void* uc, void* mc, uint64_t n, cs_dtype dt,
                      int trace_key, const cs_p2p_update* upd, cs_stream_t stream) {
  return guard([&] {
    CHECK_HANDLE(t);
    std::vector<void*> bufs(static_cast<size_t>(t->t->num_ranks()), nullptr);
    bufs[static_cast<size_t>(rank)] = uc;
    p2p_call(t, comm, rank, bufs.data(), mc, n, dt, trace_key, upd, stream);
  });
}
int cs_allreduce_p2p(cs_transport_t t, int comm, int rank, void* const* peer_bufs, uint64_t n, cs_dtype dt,
                     int trace_key, const cs_p2p_update* upd, cs_stream_t stream) {
  return guard([&] { p2p_call(t, comm, rank, peer_bufs, nullptr, n, dt, trace_key, upd, stream); });
}
namespace {
void p2p_call(cs_transport_t t, int comm, int rank, void* const* peer_bufs, void* mc, uint64_t n, cs_dtype dt,
              int trace_key, const cs_p2p_update* upd, cs_stream_t stream) {
  {
    CHECK_HANDLE(t);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!upd) {
      t->t->allreduce_p2p(comm, rank, peer_bufs, n, dt, trace_key, s, -1, nullptr, mc);
      return;
    }
    const size_t esz = dtype_size(dt);
    const char* base = static_cast<const char*>(peer_bufs[rank]);
    std::vector<DeviceTable::Entry> es;
    for (int i = 0; i < upd->n_entries; ++i) {
      const cs_update_entry& e = upd->entries[i];
      const uint64_t off = static_cast<uint64_t>(static_cast<const char*>(e.g) - base) / esz;
      if (off % 8 || off + e.n > n) throw UsageError("cs_allreduce_p2p: entry outside the bucket or misaligned");
      es.push_back(DeviceTable::Entry{e.g, e.mom, e.w, e.n, off / 8, off / 8 + (e.n + 7) / 8});
    }
    std::sort(es.begin(), es.end(), [](const auto& x, const auto& y) { return x.gstart < y.gstart; });
    DeviceTable* tab;
    {
      auto& reg = p2p_tables();
      std::lock_guard<std::mutex> lock(reg.mu);
      auto& p = reg.by_stream[s];
      if (!p) p = std::make_unique<DeviceTable>();
      tab = p.get();
    }
    Transport::P2PUpdate u;
    u.tab = tab->resident(es, s);
    u.n_entries = static_cast<int>(es.size());
    u.wdt = upd->w_dtype;
    u.lr = upd->lr;
    u.rescale = upd->rescale;
    u.momentum = upd->momentum;
    u.shard_only = upd->shard_only != 0;
    t->t->allreduce_p2p(comm, rank, peer_bufs, n, dt, trace_key, s, -1, &u, mc);
  }
}
}  // namespace

// ------------------------------------------------------------ kvstore
int cs_create_communicators(cs_transport_t t, int count, int* comms_out) {
  return guard([&] {
    CHECK_HANDLE(t);
    std::vector<int> c = create_communicators(*t->t, count);
    for (int i = 0; i < count; ++i) comms_out[i] = c[static_cast<size_t>(i)];
  });
}
int cs_kv_create(cs_engine_t e, cs_transport_t t, int rank, const cs_kv_config* cfg,
                 const int* concom_comms, int n_comms, cs_kvstore_t* out) {
  return guard([&] {
    CHECK_HANDLE(e);
    CHECK_HANDLE(t);
    CHECK_HANDLE(cfg);
    KvConfig c;
    if (cfg->mode < 0 || cfg->mode > 3) throw ConfigError("unknown kvstore mode");
    c.mode = static_cast<KvMode>(cfg->mode);
    c.outstanding = cfg->outstanding;
    c.num_keys = cfg->num_keys;
    c.comm_dtype = cfg->comm_dtype;
    c.bucket_bytes = cfg->bucket_bytes;
    c.issue_order = cfg->issue_order;
    c.comm_priority = cfg->comm_priority;
    c.p2p = cfg->p2p;
    c.zero = cfg->zero;
    std::vector<int> comms;
    for (int i = 0; i < n_comms; ++i) comms.push_back(concom_comms[i]);
    auto h = std::make_unique<cs_kvstore>();
    h->engine = e->e.get();
    h->kv = std::make_unique<KvStore>(*e->e, *t->t, rank, c, comms);
    *out = h.release();
  });
}
int cs_kv_destroy(cs_kvstore_t kv) {
  return guard([&] { delete kv; });
}
int cs_kv_init(cs_kvstore_t kv, int key, cs_slot w) {
  return guard([&] {
    CHECK_HANDLE(kv);
    kv->kv->init(key, slot_of(*kv->engine, w));
  });
}
int cs_kv_push(cs_kvstore_t kv, const int* keys, const cs_slot* grads, int n) {
  return guard([&] {
    CHECK_HANDLE(kv);
    std::vector<int> k(keys, keys + n);
    std::vector<TensorSlot> s;
    for (int i = 0; i < n; ++i) s.push_back(slot_of(*kv->engine, grads[i]));
    kv->kv->push(k, s);
  });
}
int cs_kv_pull(cs_kvstore_t kv, const int* keys, const cs_slot* outs, int n) {
  return guard([&] {
    CHECK_HANDLE(kv);
    std::vector<int> k(keys, keys + n);
    std::vector<TensorSlot> s;
    for (int i = 0; i < n; ++i) s.push_back(slot_of(*kv->engine, outs[i]));
    kv->kv->pull(k, s);
  });
}
int cs_kv_pull_update(cs_kvstore_t kv, const int* keys, const cs_slot* weights, int n,
                      const cs_sgd* sgd) {
  return guard([&] {
    CHECK_HANDLE(kv);
    CHECK_HANDLE(sgd);
    std::vector<int> k(keys, keys + n);
    std::vector<TensorSlot> s;
    for (int i = 0; i < n; ++i) s.push_back(slot_of(*kv->engine, weights[i]));
    kv->kv->pull_update(k, s, SgdConfig{sgd->lr, sgd->rescale, sgd->momentum});
  });
}
int cs_kv_barrier(cs_kvstore_t kv) {
  return guard([&] {
    CHECK_HANDLE(kv);
    kv->kv->barrier();
  });
}
int cs_kv_outstanding_in_flight(cs_kvstore_t kv, int* out) {
  return guard([&] {
    CHECK_HANDLE(kv);
    *out = kv->kv->outstanding_in_flight();
  });
}
int cs_kv_comm_buf(cs_kvstore_t kv, int key, void* host_out, uint64_t* numel, int* dtype) {
  return guard([&] {
    CHECK_HANDLE(kv);
    if (numel) *numel = kv->kv->key_numel(key);
    if (dtype) *dtype = kv->kv->comm_dtype();
    if (host_out) kv->kv->comm_buf(key, host_out);
  });
}
int cs_kv_key_map(cs_kvstore_t kv, int key, int* bucket, uint64_t* offset_elems) {
  return guard([&] {
    CHECK_HANDLE(kv);
    kv->kv->key_map(key, bucket, offset_elems);
  });
}
int cs_kv_bucket_view(cs_kvstore_t kv, int key, void** ptr) {
  return guard([&] {
    CHECK_HANDLE(kv);
    *ptr = kv->kv->bucket_view(key);
  });
}
int cs_kv_arena(cs_kvstore_t kv, void** base, uint64_t* bytes) {
  return guard([&] {
    CHECK_HANDLE(kv);
    kv->kv->arena(base, bytes);
  });
}
int cs_kv_register_grads(cs_kvstore_t kv, void* base, uint64_t bytes) {
  return guard([&] {
    CHECK_HANDLE(kv);
    kv->kv->register_grads(base, bytes);
  });
}
int cs_kv_num_buckets(cs_kvstore_t kv, int* out) {
  return guard([&] {
    CHECK_HANDLE(kv);
    *out = kv->kv->num_buckets();
  });
}
int cs_kv_bucket_lane(cs_kvstore_t kv, int bucket, int* lane) {
  return guard([&] {
    CHECK_HANDLE(kv);
    *lane = kv->kv->bucket_lane(bucket);
  });
}

// -------------------------------------------------------------- synth
int cs_synth_create(cs_engine_t e, cs_transport_t t, int rank, int nranks, const cs_synth_config* cfg,
                    const uint64_t* sizes, int num_keys, const int* concom_comms, int n_comms,
                    cs_synth_t* out) {
  return guard([&] {
    CHECK_HANDLE(e);
    CHECK_HANDLE(t);
    CHECK_HANDLE(cfg);
    if (num_keys < 1 || !sizes) throw ConfigError("synth: no keys");
    if (cfg->mode < 0 || cfg->mode > 3) throw ConfigError("unknown kvstore mode");
    SynthConfig c;
    c.mode = static_cast<KvMode>(cfg->mode);
    c.sizes.assign(sizes, sizes + num_keys);
    c.wdt = cfg->w_dtype;
    c.gdt = cfg->g_dtype;
    c.cdt = cfg->comm_dtype;
    c.bucket_bytes = cfg->bucket_bytes;
    c.issue_order = cfg->issue_order;
    c.outstanding = cfg->outstanding;
    c.lr = cfg->lr;
    c.rescale = cfg->rescale;
    c.momentum = cfg->momentum;
    c.backward_ns = cfg->backward_ns;
    c.backward_ctas = cfg->backward_ctas;
    c.fused = cfg->fused_update != 0;
    c.comm_priority = cfg->comm_priority;
    c.host_source = cfg->host_source != 0;
    c.p2p = cfg->p2p;
    c.grad_views = cfg->grad_views != 0;
    c.zero = cfg->zero;
    c.order_seed = cfg->order_seed;
    c.direct_grads = cfg->direct_grads != 0;
    std::vector<int> comms(concom_comms, concom_comms + std::max(0, n_comms));
    auto h = std::make_unique<cs_synth>();
    h->m = std::make_unique<SynthModel>(*e->e, *t->t, rank, nranks, c, comms);
    *out = h.release();
  });
}
int cs_synth_create_profiled(cs_engine_t e, cs_transport_t t, int rank, int nranks,
                             const cs_synth_config* cfg, const uint64_t* sizes, const double* ready_ms,
                             int num_keys, const int* concom_comms, int n_comms, cs_synth_t* out) {
  return guard([&] {
    CHECK_HANDLE(e);
    CHECK_HANDLE(t);
    CHECK_HANDLE(cfg);
    if (num_keys < 1 || !sizes) throw ConfigError("synth: no keys");
    if (cfg->mode < 0 || cfg->mode > 3) throw ConfigError("unknown kvstore mode");
    SynthConfig c;
    c.mode = static_cast<KvMode>(cfg->mode);
    c.sizes.assign(sizes, sizes + num_keys);
    if (ready_ms) c.ready_ms.assign(ready_ms, ready_ms + num_keys);
    c.wdt = cfg->w_dtype;
    c.gdt = cfg->g_dtype;
    c.cdt = cfg->comm_dtype;
    c.bucket_bytes = cfg->bucket_bytes;
    c.issue_order = cfg->issue_order;
    c.outstanding = cfg->outstanding;
    c.lr = cfg->lr;
    c.rescale = cfg->rescale;
    c.momentum = cfg->momentum;
    c.backward_ns = cfg->backward_ns;
    c.backward_ctas = cfg->backward_ctas;
    c.fused = cfg->fused_update != 0;
    c.comm_priority = cfg->comm_priority;
    c.host_source = cfg->host_source != 0;
    c.p2p = cfg->p2p;
    c.grad_views = cfg->grad_views != 0;
    c.zero = cfg->zero;
    c.order_seed = cfg->order_seed;
    c.direct_grads = cfg->direct_grads != 0;
    std::vector<int> comms(concom_comms, concom_comms + std::max(0, n_comms));
    auto h = std::make_unique<cs_synth>();
    h->m = std::make_unique<SynthModel>(*e->e, *t->t, rank, nranks, c, comms);
    *out = h.release();
  });
}
int cs_synth_destroy(cs_synth_t s) {
  return guard([&] { delete s; });
}
int cs_synth_init(cs_synth_t s) {
  return guard([&] {
    CHECK_HANDLE(s);
    s->m->init();
  });
}
int cs_synth_step(cs_synth_t s, int flags) {
  return guard([&] {
    CHECK_HANDLE(s);
    s->m->enqueue_step(flags);
  });
}
int cs_synth_run(cs_synth_t s, int steps, int flags, double* device_ms) {
  return guard([&] {
    CHECK_HANDLE(s);
    *device_ms = s->m->run(steps, flags);
  });
}
int cs_synth_run_e2e(cs_synth_t s, int steps, int flags, double* wall_ms) {
  return guard([&] {
    CHECK_HANDLE(s);
    *wall_ms = s->m->run_e2e(steps, flags);
  });
}
int cs_synth_checksum(cs_synth_t s, double* out) {
  return guard([&] {
    CHECK_HANDLE(s);
    *out = s->m->checksum();
  });
}
int cs_synth_read_weights(cs_synth_t s, void* host, uint64_t bytes) {
  return guard([&] {
    CHECK_HANDLE(s);
    s->m->read_weights(host, bytes);
  });
}
int cs_synth_info(cs_synth_t s, uint64_t* grad_bytes, uint64_t* h2d, int* num_buckets) {
  return guard([&] {
    CHECK_HANDLE(s);
    if (grad_bytes) *grad_bytes = s->m->grad_bytes();
    if (h2d) *h2d = s->m->h2d_bytes_per_step();
    if (num_buckets) *num_buckets = s->m->num_buckets();
  });
}
int cs_synth_last_host_ms(cs_synth_t s, double* out) {
  return guard([&] {
    CHECK_HANDLE(s);
    *out = s->m->last_host_ms();
  });
}

// ---------------------------------------------------- launch accounting
int cs_launch_count(uint64_t* out) {
  return guard([&] { *out = launch_count(); });
}
int cs_profile_enable(int on) {
  return guard([&] { profile_enable(on != 0); });
}
int cs_profile_collect(int kind, uint64_t* launches, double* total_ms, double* bytes) {
  return guard([&] {
    KernelStats st = profile_collect(kind);
    if (launches) *launches = st.launches;
    if (total_ms) *total_ms = st.total_ms;
    if (bytes) *bytes = st.bytes;
  });
}
int cs_profile_reset(void) {
  return guard([&] { profile_reset(); });
}
int cs_host_profile(char* buf, int cap, int reset) {
  return guard([&] {
    const std::string s = hostprof::report_json();
    if (buf && cap > 0) {
      const size_t n = std::min(static_cast<size_t>(cap - 1), s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
    if (reset) hostprof::reset();
  });
}

}  // extern "C"
