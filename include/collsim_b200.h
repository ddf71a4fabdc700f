/*
 * collsim_b200.h -- C ABI of the B200-native gradient-aggregation hot path
 * (KvStore init/push/pull/barrier -> dependency engine -> collectives ->
 * SGD update) of arXiv 1802.06949, as modelled by the reference simulator
 * `collsim` (R = /root/reference/proj).
 *
 * Conventions
 *   - Every entry point returns an int status: 0 = ok, negative = error.
 *     Codes -1..-5 mirror collsim::Error::Kind (R/core/include/collsim/error.hpp:10-31);
 *     cs_last_error() returns the thread-local message of the last failure.
 *     No C++ exception ever crosses this boundary.
 *   - The caller owns every data pointer.  Device work is stream-ordered on
 *     the cs_stream_t given (a cudaStream_t) or on an engine lane stream.
 *   - Tags, ops and communicators are plain integers, as in the reference.
 *
 * Reference interfaces each group replaces (drop-in map):
 *   kernels   <- tensor.cpp:61-64 copy (a), collective.cpp:228-236 rank-order
 *                sum (b), model.cpp:17-27 sgd_update (c)
 *   engine    <- engine.hpp:46-69  Engine{new_variable,push,wait_for,wait_all,shutdown}
 *   transport <- collective.hpp:38-59 Transport{new_communicator,allreduce_sum,broadcast,barrier,set_inject_latency}
 *   kvstore   <- kvstore.hpp:35-78 create_communicators, KvStore{init,push,pull,barrier,comm_buf,outstanding_in_flight}
 *   trace     <- trace.hpp:14-78 TraceSink{emit,snapshot,write_jsonl}
 *   trainer   <- trainer.cpp:89-151 train_epoch loop shapes (synthetic producer)
 */
#ifndef COLLSIM_B200_H_
#define COLLSIM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cs_stream_t; /* == cudaStream_t */

/* ------------------------------------------------------------ status */
enum {
  CS_OK = 0,
  CS_ERR_CONFIG = -1,   /* collsim::ConfigError   */
  CS_ERR_USAGE = -2,    /* collsim::UsageError    */
  CS_ERR_MISMATCH = -3, /* collsim::MismatchError */
  CS_ERR_DEADLOCK = -4, /* collsim::DeadlockTimeout */
  CS_ERR_ENGINE = -5,   /* collsim::EngineError   */
  CS_ERR_CUDA = -6,
  CS_ERR_NCCL = -7,
  CS_ERR_INTERNAL = -8
};

typedef enum cs_dtype { CS_F64 = 0, CS_F32 = 1, CS_BF16 = 2 } cs_dtype;

const char* cs_last_error(void);
const char* cs_status_name(int status); /* "ConfigError", ... (error.hpp:19-28) */
int cs_version(void);
int cs_device_count(int* out);

/* ------------------------------------------------ kernels (a) (b) (c) */

/* (a) pack / cast: dst[i] = (dst_dt) src[i] for every entry.  Used for the
 * gradient -> comm-bucket staging copy (kvstore.cpp:109 `copy(g, comm_buf)`)
 * and for the pull copy-out (kvstore.cpp:160/170). One launch per table. */
typedef struct cs_copy_entry {
  const void* src;
  void* dst;
  uint64_t n; /* elements */
} cs_copy_entry;
int cs_pack(const cs_copy_entry* entries, int n_entries, cs_dtype src_dt, cs_dtype dst_dt,
            cs_stream_t stream);

/* (b) multi-buffer rank-order sum: every out[j][i] = ((in[0][i] + in[1][i]) + ...) + in[m-1][i]
 * (collective.cpp:228-236).  out[j] may alias in[j] (in-place allreduce).
 * m, nout <= CS_MAX_RANKS.  Pointers may be peer (UVA) addresses. */
#define CS_MAX_RANKS 16
int cs_sum_buffers(const void* const* in, int m, void* const* out, int nout, uint64_t n,
                   cs_dtype dt, cs_stream_t stream);

/* (c) fused SGD / momentum update reading the reduced gradient directly:
 *   momentum == 0: w[i] -= (lr*rescale) * g[i]              (model.cpp:17-27)
 *   momentum  > 0: v = mu*v - (lr*rescale)*g; w += v        (MXNet form, new)
 * w_dt in {F64,F32,BF16}; g_dt the comm dtype; mom has w's compute type
 * (f64 for F64 weights, f32 otherwise) and may be NULL when momentum == 0. */
typedef struct cs_update_entry {
  void* w;
  const void* g;
  void* mom;
  uint64_t n;
} cs_update_entry;
int cs_sgd_update(const cs_update_entry* entries, int n_entries, cs_dtype w_dt, cs_dtype g_dt,
                  double lr, double rescale, double momentum, cs_stream_t stream);

/* synthetic backward producer: dst = src (cast), then the kernel is held for
 * at least spin_ns on the device (models per-key backward compute). */
int cs_synth_backward(const void* src, void* dst, uint64_t n, cs_dtype dt, uint64_t spin_ns,
                      int ctas, cs_stream_t stream);

/* deterministic fp64 checksum sum_i x[i] of a buffer into *out_dev (device f64). */
int cs_checksum(const void* x, uint64_t n, cs_dtype dt, double* out_dev, cs_stream_t stream);

/* ------------------------------------------------------------- trace */
typedef struct cs_trace* cs_trace_t;
int cs_trace_create(cs_trace_t* out);
int cs_trace_destroy(cs_trace_t t);
int cs_trace_count(cs_trace_t t, uint64_t* out);
int cs_trace_write_jsonl(cs_trace_t t, const char* path);
/* gauges (trace.hpp:29-55): max_open_collectives, compute_overlap */
int cs_trace_gauges(cs_trace_t t, int* max_open_collectives, int* compute_overlap);

/* ------------------------------------------------------------ engine */
typedef struct cs_engine* cs_engine_t;
enum { CS_OP_COMPUTE = 0, CS_OP_COPY = 1, CS_OP_COLLECTIVE = 2, CS_OP_OTHER = 3 }; /* engine.hpp:30 */
enum { CS_DISPATCH_INLINE = 0, CS_DISPATCH_POOL = 1, CS_DISPATCH_HOST = 2 };
typedef int (*cs_host_fn)(void* arg); /* non-zero return = body failure */
typedef int (*cs_stream_fn)(void* arg, cs_stream_t stream);

/* device < 0: host-only engine (host ops only; no CUDA calls). */
int cs_engine_create(int num_worker_threads, int rank, int device, cs_trace_t trace,
                     cs_engine_t* out);
int cs_engine_destroy(cs_engine_t e);
int cs_engine_new_variable(cs_engine_t e, uint64_t* tag);
/* Reference semantics (engine.hpp:57-58): body runs once every earlier
 * conflicting op on its tags has completed (device work included). */
int cs_engine_push_host(cs_engine_t e, cs_host_fn fn, void* arg, const uint64_t* reads, int n_reads,
                        const uint64_t* mutates, int n_mutates, int kind, int key, uint64_t* op_id);
/* Stream op: body enqueues device work on `lane`'s stream after the engine
 * has made that stream wait for the CUDA events of every conflicting op. */
int cs_engine_push_stream(cs_engine_t e, cs_stream_fn fn, void* arg, const uint64_t* reads,
                          int n_reads, const uint64_t* mutates, int n_mutates, int kind, int key,
                          int lane, int dispatch, uint64_t* op_id);
int cs_engine_wait_for(cs_engine_t e, uint64_t tag);
int cs_engine_wait_all(cs_engine_t e);
/* Interop with a framework's own CUDA stream (no reference counterpart: the
 * reference's producers are engine ops, trainer.cpp:36-72).
 * import_event: stream op on `lane` that waits on `cuda_event` (a cudaEvent_t
 * the caller recorded after producing the tensors) and mutates `mutates`; the
 * event may be re-recorded once the op is dispatched (inline, normally inside
 * this call).  stream_wait: waits on the host until every op pushed so far on
 * `tags` is dispatched, then makes `stream` wait on their last write and the
 * reads since (the external stream may then read or overwrite the tensors). */
int cs_engine_import_event(cs_engine_t e, void* cuda_event, const uint64_t* mutates, int n_mutates,
                           int key, int lane, uint64_t* op_id);
int cs_engine_stream_wait(cs_engine_t e, const uint64_t* tags, int n_tags, cs_stream_t stream);
int cs_engine_shutdown(cs_engine_t e);
int cs_engine_new_lane(cs_engine_t e, int priority, int* lane);
int cs_engine_lane_stream(cs_engine_t e, int lane, cs_stream_t* out);
int cs_engine_stats(cs_engine_t e, uint64_t* pushed, uint64_t* completed);
int cs_engine_num_threads(cs_engine_t e, int* out);
/* Device waits (wait_for / wait_all) give up after `ms` (default 600 s): every
 * transport is aborted first -- peer kernels leave their pair barriers, NCCL
 * communicators are aborted, ledgers latch -- then CS_ERR_DEADLOCK is
 * returned (collective.cpp:249-264 watchdog -> report -> latch).  The same
 * waits poll for asynchronous failures (ncclCommGetAsyncError, a peer
 * kernel's device timeout) every ~50 ms. */
int cs_engine_set_watchdog(cs_engine_t e, int64_t ms);

/* --------------------------------------------------------- transport */
typedef struct cs_transport* cs_transport_t;
/* In-process ranks (threads), buffers on one or several local GPUs; the last
 * arriver reduces with kernel (b) in rank order (collective.cpp:228-236). */
int cs_transport_create_local(int num_ranks, int watchdog_ms, cs_trace_t trace,
                              cs_transport_t* out);
/* Same, but the rank threads run the fused peer-memory kernels (the path the
 * NCCL transport takes across GPUs) directly on each other's buffers: plain
 * device pointers, every rank's grid capped so all grids are co-resident on
 * one GPU.  Exercises the cross-GPU kernels, barriers and epochs on one device. */
int cs_transport_create_local_peer(int num_ranks, int watchdog_ms, cs_trace_t trace,
                                   cs_transport_t* out);
/* One process per GPU: matching ledger in POSIX shared memory `name`
 * (rank 0 creates it), data over NCCL (NVLink / NVSwitch). */
int cs_transport_create_nccl(const char* name, int num_ranks, int rank, int device,
                             int watchdog_ms, cs_trace_t trace, cs_transport_t* out);
/* Host-only matching ledger (no data movement) for CPU tests of the
 * matching / watchdog logic: in-process when name is NULL or "", else shm. */
int cs_transport_create_ledger_only(const char* name, int num_ranks, int rank, int watchdog_ms,
                                    cs_trace_t trace, cs_transport_t* out);
int cs_transport_destroy(cs_transport_t t);
int cs_transport_num_ranks(cs_transport_t t, int* out);
int cs_transport_num_communicators(cs_transport_t t, int* out);
int cs_transport_new_communicator(cs_transport_t t, int* comm);
int cs_transport_set_inject_latency(cs_transport_t t, int64_t us);
int cs_transport_abort(cs_transport_t t);
int cs_allreduce_sum(cs_transport_t t, int comm, int rank, void* buf, uint64_t n, cs_dtype dt,
                     int trace_key, cs_stream_t stream);
int cs_broadcast(cs_transport_t t, int comm, int rank, int root, void* buf, uint64_t n,
                 cs_dtype dt, int trace_key, cs_stream_t stream);
int cs_barrier(cs_transport_t t, int comm, int rank, int trace_key, cs_stream_t stream);
/* NVLink peer-memory path (NCCL transport, >= 2 peer-capable ranks):
 * setup-phase collective mapping every rank's allocation `base` (CUDA IPC);
 * ptrs_out[r] = rank r's buffer as seen from this process. */
int cs_transport_p2p_capable(cs_transport_t t, int* out);
int cs_transport_share_buffer(cs_transport_t t, void* base, void** ptrs_out);
/* same, naming the calling rank (required by a local peer transport, whose
 * one object serves every rank thread) */
int cs_transport_share_buffer_rank(cs_transport_t t, int rank, void* base, void** ptrs_out);
/* a peer kernel's device timeout (CSB_P2P_TIMEOUT_MS, default 30 s: the pair
 * barrier records where it waited and the kernel returns -- no __trap) or an
 * NCCL asynchronous error, as text into buf ("" when healthy) */
int cs_transport_device_failure(cs_transport_t t, char* buf, int cap);
/* CSB_P2P_TRACE=1 (set before the transport is created): the last peer
 * launch of `rank` stamps %globaltimer per CTA at 5 points -- start, past
 * the arrival barrier, own shard done, past barrier 1, end -- into
 * host-mapped memory; copies up to `cap` values (CTA-major) into out, *n =
 * the total (0 when tracing is off).  A diagnostic for the peer kernels,
 * which ncu cannot replay (their CTAs wait on other GPUs). */
int cs_transport_p2p_stamps(cs_transport_t t, int rank, uint64_t* out, int cap, int* n);
/* allreduce of peer_bufs[*] (n elements, multiple of 8) in rank order, every
 * rank ends with the sum.  Launches of one (comm, rank) run in call order even
 * on different streams (they share the comm's flag region); every rank must
 * pass the same update / shard_only choice (else CS_ERR_MISMATCH); with upd != NULL fused with the SGD / momentum
 * update of the listed weights (entries address the bucket by element
 * offset: entry.g = &bucket[offset], offset a multiple of 8). */
typedef struct cs_p2p_update {
  const cs_update_entry* entries; /* g points into this rank's bucket */
  int n_entries;
  int w_dtype;
  double lr, rescale, momentum;
  int shard_only; /* 1: on return the bucket holds only this rank's shard of the sum (the update
                     read the other shards from their owners' buckets: less NVLink and HBM traffic);
                     0: the whole sum, as without an update.  Ignored by cs_allreduce_nvls. */
} cs_p2p_update;
int cs_allreduce_p2p(cs_transport_t t, int comm, int rank, void* const* peer_bufs, uint64_t n,
                     cs_dtype dt, int trace_key, const cs_p2p_update* upd, cs_stream_t stream);
/* NVLink SHARP: setup-phase collective allocating `bytes` bound to an NVSwitch
 * multicast object on every rank; *uc = this rank's copy, *mc = multicast VA.
 * cs_allreduce_nvls reduces in the switch (multimem.ld_reduce / multimem.st),
 * optionally fused with the update as cs_allreduce_p2p (f32 / bf16). */
int cs_transport_nvls_capable(cs_transport_t t, int* out);
int cs_transport_alloc_nvls(cs_transport_t t, uint64_t bytes, void** uc, void** mc);
int cs_allreduce_nvls(cs_transport_t t, int comm, int rank, void* uc, void* mc, uint64_t n, cs_dtype dt,
                      int trace_key, const cs_p2p_update* upd, cs_stream_t stream);

/* ----------------------------------------------------------- kvstore */
typedef struct cs_kvstore* cs_kvstore_t;
enum { CS_KV_FUNNEL = 0, CS_KV_DEPCHA = 1, CS_KV_CONCOM = 2, CS_KV_NAIVE = 3 }; /* kvstore.hpp:21 */
typedef struct cs_kv_config {
  int mode;              /* CS_KV_* */
  int outstanding;       /* concom window / number of extra communicators */
  int num_keys;
  int comm_dtype;        /* cs_dtype of the comm buffers (-1: dtype of the init weights) */
  uint64_t bucket_bytes; /* 0: one comm buffer per key (reference 1:1 map, kvstore.cpp:84) */
  int issue_order;       /* bucket grouping order: 0 ascending keys, 1 descending */
  int comm_priority;     /* CUDA stream priority of the comm lanes (<=0, lower = higher prio) */
  int p2p;               /* 1: NVLink peer-memory collectives (needs bucket_bytes > 0 and a
                            peer-capable NCCL transport); DepCha pull_update becomes one fused
                            allreduce+update kernel per bucket, rank-order (bit-exact) sums;
                            ConCom runs one peer-memory allreduce per communicator concurrently,
                            each grid capped to 1/outstanding of the device so all co-reside.
                            2: NVSwitch multicast (NVLS, funnel/depcha only) */
  int zero;              /* 1 (DepCha, p2p = 1): ZeRO-1 -- each rank keeps master weights and momentum of
                            its shard only; the fused kernel reduce-scatters, updates the shard and
                            all-gathers the weights.  pull_update must cover whole buckets. */
} cs_kv_config;
typedef struct cs_slot { /* TensorSlot (kvstore.hpp:16-19): non-owning device view + tag */
  void* data;
  int dtype;
  uint64_t numel;
  uint64_t tag;
} cs_slot;
typedef struct cs_sgd {
  double lr;
  double rescale;
  double momentum;
} cs_sgd;
int cs_create_communicators(cs_transport_t t, int count, int* comms_out); /* kvstore.hpp:35 */
int cs_kv_create(cs_engine_t e, cs_transport_t t, int rank, const cs_kv_config* cfg,
                 const int* concom_comms, int n_comms, cs_kvstore_t* out);
int cs_kv_destroy(cs_kvstore_t kv);
int cs_kv_init(cs_kvstore_t kv, int key, cs_slot weights);
/* list forms (MXNet KVStore push/pull of key lists; n == 1 is the reference call) */
int cs_kv_push(cs_kvstore_t kv, const int* keys, const cs_slot* grads, int n);
int cs_kv_pull(cs_kvstore_t kv, const int* keys, const cs_slot* outs, int n);
/* pull fused with the SGD update: weights <- sgd(weights, aggregated grad) */
int cs_kv_pull_update(cs_kvstore_t kv, const int* keys, const cs_slot* weights, int n,
                      const cs_sgd* sgd);
int cs_kv_barrier(cs_kvstore_t kv);
int cs_kv_outstanding_in_flight(cs_kvstore_t kv, int* out);
/* synchronizes the key's comm buffer and copies it to host memory (comm dtype) */
int cs_kv_comm_buf(cs_kvstore_t kv, int key, void* host_out, uint64_t* numel, int* dtype);
/* key -> (fusion bucket, element offset); builds the buckets once every key is
 * initialized (with the peer-memory path a setup collective: all ranks call it) */
int cs_kv_key_map(cs_kvstore_t kv, int key, int* bucket, uint64_t* offset_elems);
/* Bucket views (gradient-as-bucket-view): the device address of the key's slot
 * in its comm bucket (comm dtype).  A gradient written there and pushed with
 * that address is not copied; the collective rewrites it in place (the whole
 * sum after a pull, only this rank's shard after a shard_only fused update).
 * cs_kv_arena: the one allocation holding every fusion bucket (to zero it). */
int cs_kv_bucket_view(cs_kvstore_t kv, int key, void** ptr);
int cs_kv_arena(cs_kvstore_t kv, void** base, uint64_t* bytes);
/* Setup collective (every rank, same order): the allocation holding this
 * rank's gradients -- any device pointer into it, keys at the same offsets
 * on every rank.  A whole-bucket cs_kv_pull_update whose pushed gradients all
 * lie inside it reads them in place and stages nothing into the buckets
 * (replaces the kvstore.cpp:109 copy): at N > 1 the fused peer kernel reads
 * every rank's gradients over NVLink, at one rank the fused pack + update
 * kernel skips the staging store.  The buckets then hold no copy of those
 * gradients afterwards (cs_kv_comm_buf), as under ZeRO-1.  Ranks whose
 * layouts differ fail with CS_ERR_MISMATCH before any launch. */
int cs_kv_register_grads(cs_kvstore_t kv, void* base, uint64_t bytes);
int cs_kv_num_buckets(cs_kvstore_t kv, int* out);
int cs_kv_bucket_lane(cs_kvstore_t kv, int bucket, int* lane);

/* ------------------------------------------ synthetic training step */
/* The reference trainer's loop shapes (trainer.cpp:112-141) over a key set,
 * with a synthetic backward (one producer op per key, descending keys). */
typedef struct cs_synth* cs_synth_t;
typedef struct cs_synth_config {
  int mode;               /* CS_KV_* */
  int w_dtype, g_dtype, comm_dtype;
  uint64_t bucket_bytes;
  int issue_order;        /* 0 ascending keys, 1 descending (gradient-ready order) */
  int outstanding;
  double lr, rescale, momentum;
  uint64_t backward_ns;   /* total synthetic backward device time per step */
  int backward_ctas;      /* 0: one CTA per SM */
  int fused_update;       /* 1: pull_update (kernel (c) on the reduced bucket) */
  int comm_priority;
  int host_source;        /* 1: gradients copied from pinned host memory each step */
  int p2p;                /* as cs_kv_config.p2p */
  int grad_views;         /* 1: gradients are produced in place in the comm buckets (cs_kv_bucket_view) */
  int zero;               /* as cs_kv_config.zero */
  int order_seed;         /* != 0: this rank's gradients become ready in a random order (seeded per
                             rank) -- the deadlock-stress producer of SURVEY §8d config 5 */
  int direct_grads;       /* 1: the gradient arena is registered (cs_kv_register_grads): at N > 1 the
                             fused peer kernel reads every rank's gradients in place, no staging */
} cs_synth_config;
enum { CS_STEP_BACKWARD = 1, CS_STEP_COMM = 2, CS_STEP_LOCAL_UPDATE = 4, CS_STEP_CHECKSUM = 8 };
int cs_synth_create(cs_engine_t e, cs_transport_t t, int rank, int nranks, const cs_synth_config* cfg,
                    const uint64_t* sizes, int num_keys, const int* concom_comms, int n_comms,
                    cs_synth_t* out);
/* same, with the measured gradient-ready time of every key (ms from the start
 * of a real backward, tools/calibrate_backward.py) driving the producers */
int cs_synth_create_profiled(cs_engine_t e, cs_transport_t t, int rank, int nranks,
                             const cs_synth_config* cfg, const uint64_t* sizes, const double* ready_ms,
                             int num_keys, const int* concom_comms, int n_comms, cs_synth_t* out);
int cs_synth_destroy(cs_synth_t s);
int cs_synth_init(cs_synth_t s);
int cs_synth_step(cs_synth_t s, int flags);
/* device time (CUDA events spanning every lane) of `steps` steps */
int cs_synth_run(cs_synth_t s, int steps, int flags, double* device_ms);
/* host wall time of `steps` steps, each ending with the result on the host */
int cs_synth_run_e2e(cs_synth_t s, int steps, int flags, double* wall_ms);
int cs_synth_checksum(cs_synth_t s, double* out);
/* every key's weights, concatenated without padding, into host memory
 * (bytes = sum n_k * sizeof(w_dtype)); waits for this rank's work first */
int cs_synth_read_weights(cs_synth_t s, void* host, uint64_t bytes);
int cs_synth_info(cs_synth_t s, uint64_t* grad_bytes, uint64_t* h2d_bytes_per_step, int* num_buckets);
/* host time the last cs_synth_run spent dispatching (enqueue-bound check) */
int cs_synth_last_host_ms(cs_synth_t s, double* out);

/* ------------------------------------------------ launch accounting */
enum {
  CS_KERNEL_PACK = 0, CS_KERNEL_SUM = 1, CS_KERNEL_SGD = 2, CS_KERNEL_SYNTH = 3, CS_KERNEL_CHECKSUM = 4,
  CS_KERNEL_PACK_SGD = 5 /* (a)+(c) fused: one rank, the collective between them is the identity */
};
int cs_launch_count(uint64_t* out); /* kernels of this library launched so far */
int cs_profile_enable(int on);      /* per-launch CUDA-event timing on the launch stream */
int cs_profile_collect(int kind, uint64_t* launches, double* total_ms, double* bytes);
int cs_profile_reset(void);
/* host-side section timers (enabled by CSB_HOST_PROFILE=1): JSON into buf */
int cs_host_profile(char* buf, int cap, int reset);

#ifdef __cplusplus
}
#endif
#endif /* COLLSIM_B200_H_ */
