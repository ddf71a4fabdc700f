// trainer.cpp -- see trainer.hpp.  Loop shapes: R/core/src/trainer.cpp:112-141.
#include "trainer.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <random>
#include <thread>

#include "kernels.hpp"

namespace csb {

namespace {

constexpr uint64_t kAlign = 256;

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// SplitMix64 step, as R/core/src/tensor.cpp:76-81.
uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint16_t bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// uniform [-1, 1) from std::mt19937_64's top 53 bits, written in dtype `dt`.
void fill_uniform(void* out, uint64_t n, uint64_t seed, int dt) {
  std::mt19937_64 gen(seed);
  for (uint64_t i = 0; i < n; ++i) {
    const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const double v = 2.0 * u - 1.0;
    if (dt == CS_F64) static_cast<double*>(out)[i] = v;
    else if (dt == CS_F32) static_cast<float*>(out)[i] = static_cast<float>(v);
    else static_cast<uint16_t*>(out)[i] = bf16_rne(static_cast<float>(v));
  }
}

template <typename F>
void parallel_for(int n, F f) {
  const int T = std::max(1, std::min<int>(n, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  for (int t = 0; t < T; ++t)
    th.emplace_back([&] {
      for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) f(i);
    });
  for (auto& x : th) x.join();
}

KvConfig kv_config(const SynthConfig& c) {
  KvConfig k;
  k.mode = c.mode;
  k.outstanding = c.outstanding;
  k.num_keys = static_cast<int>(c.sizes.size());
  k.comm_dtype = c.cdt;
  k.bucket_bytes = c.bucket_bytes;
  k.issue_order = c.issue_order;
  k.comm_priority = c.comm_priority;
  k.p2p = c.p2p;
  k.zero = c.zero;
  return k;
}

}  // namespace

SynthModel::SynthModel(Engine& engine, Transport& transport, int rank, int nranks, SynthConfig cfg,
                       std::vector<int> concom_comms)
    : engine_(engine),
      transport_(transport),
      rank_(rank),
      nranks_(nranks),
      cfg_(std::move(cfg)),
      kv_(engine, transport, rank, kv_config(cfg_), std::move(concom_comms)) {
  if (cfg_.sizes.empty()) throw ConfigError("SynthModel: no keys");
}

SynthModel::~SynthModel() {
  try {
    engine_.wait_all();
  } catch (...) {
  }
  engine_.bind_device();
  if (w_arena_) cudaFree(w_arena_);
  if (g_arena_) cudaFree(g_arena_);
  if (src_arena_) {
    if (cfg_.host_source) cudaFreeHost(src_arena_);
    else cudaFree(src_arena_);
  }
  if (sum_dev_) cudaFree(sum_dev_);
  if (sum_host_) cudaFreeHost(sum_host_);
  for (void* p : mom_local_) cudaFree(p);
}

uint64_t SynthModel::grad_bytes() const {
  uint64_t b = 0;
  for (uint64_t n : cfg_.sizes) b += n * dtype_size(cfg_.gdt);
  return b;
}

uint64_t SynthModel::h2d_bytes_per_step() const { return cfg_.host_source ? g_arena_bytes_ : 0; }

void SynthModel::init() {
  const int K = static_cast<int>(cfg_.sizes.size());
  const uint64_t ws = dtype_size(cfg_.wdt), gs = dtype_size(cfg_.gdt);
  std::vector<uint64_t> woff(K), goff(K);
  uint64_t wtot = 0, gtot = 0;
  for (int k = 0; k < K; ++k) {
    woff[k] = wtot;
    goff[k] = gtot;
    wtot += round_up(cfg_.sizes[k] * ws, kAlign);
    gtot += round_up(cfg_.sizes[k] * gs, kAlign);
  }
  // host staging, generated in parallel over keys
  std::vector<char> wh(wtot, 0), gh(gtot, 0);
  parallel_for(K, [&](int k) {
    if (rank_ == 0) fill_uniform(wh.data() + woff[k], cfg_.sizes[k], mix_seed(7, k), cfg_.wdt);
    fill_uniform(gh.data() + goff[k], cfg_.sizes[k],
                 cfg_.seed_base + static_cast<uint64_t>(rank_) * K + k, cfg_.gdt);
  });
  engine_.bind_device();
  CSB_CUDA(cudaMalloc(&w_arena_, wtot));
  CSB_CUDA(cudaMalloc(&g_arena_, gtot));
  CSB_CUDA(cudaMemcpy(w_arena_, wh.data(), wtot, cudaMemcpyHostToDevice));
  CSB_CUDA(cudaMemset(g_arena_, 0, gtot));
  if (cfg_.host_source) {
    CSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&src_arena_), gtot, cudaHostAllocDefault));
    std::memcpy(src_arena_, gh.data(), gtot);
  } else {
    CSB_CUDA(cudaMalloc(&src_arena_, gtot));
    CSB_CUDA(cudaMemcpy(src_arena_, gh.data(), gtot, cudaMemcpyHostToDevice));
  }
  CSB_CUDA(cudaMalloc(&sum_dev_, 2 * sizeof(double)));
  CSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&sum_host_), 2 * sizeof(double), cudaHostAllocDefault));
  w_arena_elems_ = wtot / ws;
  g_arena_bytes_ = gtot;

  // synthetic backward time split over keys in proportion to their size
  // (with a 2 us floor per key), as stated in DESIGN.md
  uint64_t total = 0;
  for (uint64_t n : cfg_.sizes) total += n;
  spin_ns_.resize(K);
  produce_order_.resize(K);
  for (int k = 0; k < K; ++k) produce_order_[k] = K - 1 - k;  // backward: last layer first
  if (static_cast<int>(cfg_.ready_ms.size()) == K) {
    std::stable_sort(produce_order_.begin(), produce_order_.end(),
                     [&](int a, int b) { return cfg_.ready_ms[a] < cfg_.ready_ms[b]; });
    double prev = 0.0;
    for (int k : produce_order_) {
      spin_ns_[k] = static_cast<uint64_t>(std::max(0.0, cfg_.ready_ms[k] - prev) * 1e6);
      prev = std::max(prev, cfg_.ready_ms[k]);
    }
  } else {
    if (cfg_.order_seed != 0) {
      // deadlock stress: every rank produces its gradients in its own random
      // order (the schedules must still issue identical collective sequences)
      std::mt19937_64 g(mix_seed(static_cast<uint64_t>(cfg_.order_seed), static_cast<uint64_t>(rank_)));
      std::shuffle(produce_order_.begin(), produce_order_.end(), g);
    }
    for (int k = 0; k < K; ++k)
      spin_ns_[k] = cfg_.backward_ns == 0
                        ? 0
                        : std::max<uint64_t>(2000, static_cast<uint64_t>(static_cast<double>(cfg_.backward_ns) *
                                                                         cfg_.sizes[k] / total));
  }
  for (int k = 0; k < K; ++k) {
    w_.push_back(w_arena_ + woff[k]);
    g_.push_back(g_arena_ + goff[k]);
    src_.push_back(src_arena_ + goff[k]);
    wt_.push_back(engine_.new_variable());
    gt_.push_back(engine_.new_variable());
  }
  sum_tag_[0] = engine_.new_variable();
  sum_tag_[1] = engine_.new_variable();
  for (int k = 0; k < K; ++k)
    kv_.init(k, TensorSlot{w_[k], cfg_.wdt, cfg_.sizes[k], wt_[k]});
  engine_.wait_all();
  groups_ = kv_.bucket_groups();
  h2d_dst_ = g_arena_;
  if (cfg_.direct_grads && !cfg_.grad_views) kv_.register_grads(g_arena_, gtot);  // any N
  if (cfg_.grad_views) {
    if (cfg_.bucket_bytes == 0) throw ConfigError("synth: bucket views need fusion buckets");
    if (kv_.comm_dtype() != cfg_.gdt) throw ConfigError("synth: bucket views need comm dtype == gradient dtype");
    void* base = nullptr;
    uint64_t bytes = 0;
    kv_.arena(&base, &bytes);
    for (int k = 0; k < K; ++k) g_[k] = kv_.bucket_view(k);
    if (cfg_.host_source) {
      // the pinned source in bucket layout: one H2D copy fills every view
      char* h = nullptr;
      CSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h), bytes, cudaHostAllocDefault));
      std::memset(h, 0, bytes);
      for (int k = 0; k < K; ++k)
        std::memcpy(h + (static_cast<char*>(g_[k]) - static_cast<char*>(base)), src_arena_ + goff[k],
                    cfg_.sizes[k] * gs);
      cudaFreeHost(src_arena_);
      src_arena_ = h;
      g_arena_bytes_ = bytes;
    }
    h2d_dst_ = base;
    cudaFree(g_arena_);
    g_arena_ = nullptr;
  }
}

void SynthModel::enqueue_step(int flags) {
  const int K = static_cast<int>(cfg_.sizes.size());
  const int gdt = cfg_.gdt;
  const std::vector<void*>& G = g_;
  const std::vector<Tag>& GT = gt_;
  if ((flags & kStepBackward) && cfg_.host_source) {
    // e2e input upload: the step's gradients arrive from pinned host memory
    // in one H2D copy of the contiguous gradient arena
    void* dst = h2d_dst_;
    const void* src = src_arena_;
    const size_t bytes = g_arena_bytes_;
    engine_.push_stream(
        [dst, src, bytes](cudaStream_t s) {
          CSB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        },
        {}, GT, OpKind::Copy, -1, 0, Dispatch::Inline);
  } else if (flags & kStepBackward) {
    for (int k : produce_order_) {
      void* dst = g_[k];
      const void* src = src_[k];
      const uint64_t n = cfg_.sizes[k];
      {
        const uint64_t spin = spin_ns_[k];
        const int ctas = cfg_.backward_ctas;
        engine_.push_stream(
            [dst, src, n, gdt, spin, ctas](cudaStream_t s) { synth_backward(src, dst, n, gdt, spin, ctas, s); },
            {}, {gt_[k]}, OpKind::Compute, k, 0, Dispatch::Inline);
      }
    }
  }
  auto gslots = [&](const std::vector<int>& keys) {
    std::vector<TensorSlot> v;
    for (int k : keys) v.push_back(TensorSlot{G[k], gdt, cfg_.sizes[k], GT[k]});
    return v;
  };
  auto wslots = [&](const std::vector<int>& keys) {
    std::vector<TensorSlot> v;
    for (int k : keys) v.push_back(TensorSlot{w_[k], cfg_.wdt, cfg_.sizes[k], wt_[k]});
    return v;
  };
  const SgdConfig sgd{cfg_.lr, cfg_.rescale, cfg_.momentum};
  // push_sgd_update (trainer.cpp:74-80) as one op over a key list: reads the
  // gradients, mutates the weights, kernel (c) in one launch
  auto local_sgd = [&](const std::vector<int>& keys) {
    if (cfg_.momentum != 0.0 && mom_local_.empty()) {
      engine_.bind_device();
      const uint64_t es = cfg_.wdt == CS_F64 ? 8 : 4;
      for (int k = 0; k < K; ++k) {
        void* p = nullptr;
        CSB_CUDA(cudaMalloc(&p, round_up(cfg_.sizes[k] * es, kAlign)));
        CSB_CUDA(cudaMemset(p, 0, round_up(cfg_.sizes[k] * es, kAlign)));
        mom_local_.push_back(p);
      }
      CSB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
    std::vector<cs_update_entry> es;
    std::vector<Tag> r, m;
    for (int k : keys) {
      es.push_back(cs_update_entry{w_[k], G[k], mom_local_.empty() ? nullptr : mom_local_[k],
                                   cfg_.sizes[k]});
      r.push_back(GT[k]);
      m.push_back(wt_[k]);
    }
    const int wdt = cfg_.wdt;
    const double lr = cfg_.lr, rs = cfg_.rescale;
    const double mu = cfg_.momentum;
    DeviceTable* tab = &local_tab_;  // resident table, lane 0 only
    engine_.push_stream(
        [es, wdt, gdt, lr, rs, mu, tab](cudaStream_t s) {
          tab->sgd(es.data(), static_cast<int>(es.size()), wdt, gdt, lr, rs, mu, s);
        },
        r, m, OpKind::Compute, keys.front(), 0, Dispatch::Inline);
  };

  if (flags & kStepComm) {
    if (cfg_.mode == KvMode::Funnel || cfg_.mode == KvMode::ConCom) {
      int since = 0;
      for (const auto& keys : groups_) {
        kv_.push(keys, gslots(keys));
        if (cfg_.fused) {
          kv_.pull_update(keys, wslots(keys), sgd);
        } else {
          kv_.pull(keys, gslots(keys));
          local_sgd(keys);
        }
        if (cfg_.mode == KvMode::ConCom && ++since == cfg_.outstanding) {
          kv_.barrier();
          since = 0;
        }
      }
      if (cfg_.mode == KvMode::ConCom && since > 0) kv_.barrier();
    } else {
      std::vector<int> all;
      for (const auto& keys : groups_) all.insert(all.end(), keys.begin(), keys.end());
      kv_.push(all, gslots(all));
      if (cfg_.fused) {
        kv_.pull_update(all, wslots(all), sgd);
      } else {
        kv_.pull(all, gslots(all));
        local_sgd(all);
      }
    }
  } else if (flags & kStepLocalUpdate) {
    std::vector<int> all(K);
    for (int k = 0; k < K; ++k) all[k] = K - 1 - k;
    local_sgd(all);
  }

  if (flags & kStepChecksum) {
    void* w = w_arena_;
    const uint64_t n = w_arena_elems_;
    const int wdt = cfg_.wdt;
    const int slot = sum_next_;
    double* d = sum_dev_ + slot;
    double* h = sum_host_ + slot;
    engine_.push_stream(
        [w, n, wdt, d, h](cudaStream_t s) {
          ::csb::checksum(w, n, wdt, d, s);
          CSB_CUDA(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, s));
        },
        wt_, {sum_tag_[slot]}, OpKind::Copy, -1, 0, Dispatch::Inline);
    sum_last_ = slot;
    sum_next_ = slot ^ 1;
  }
}

double SynthModel::run(int steps, int flags) {
  engine_.wait_all();
  engine_.bind_device();
  const int L = engine_.num_lanes();
  cudaEvent_t start, end;
  CSB_CUDA(cudaEventCreate(&start));
  CSB_CUDA(cudaEventCreate(&end));
  std::vector<cudaEvent_t> joins(static_cast<size_t>(L));
  for (auto& e : joins) CSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaStream_t s0 = engine_.lane_stream(0);
  const auto h0 = std::chrono::steady_clock::now();
  CSB_CUDA(cudaEventRecord(start, s0));
  for (int l = 1; l < L; ++l) CSB_CUDA(cudaStreamWaitEvent(engine_.lane_stream(l), start, 0));
  for (int i = 0; i < steps; ++i) enqueue_step(flags);
  // wait for dispatch only (no device sync) so the join below sees all work
  while (engine_.ops_completed() < engine_.ops_pushed()) std::this_thread::yield();
  last_host_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  for (int l = 1; l < L; ++l) {
    CSB_CUDA(cudaEventRecord(joins[l], engine_.lane_stream(l)));
    CSB_CUDA(cudaStreamWaitEvent(s0, joins[l], 0));
  }
  CSB_CUDA(cudaEventRecord(end, s0));
  engine_.wait_all();
  CSB_CUDA(cudaEventSynchronize(end));
  float ms = 0.f;
  CSB_CUDA(cudaEventElapsedTime(&ms, start, end));
  cudaEventDestroy(start);
  cudaEventDestroy(end);
  for (auto& e : joins) cudaEventDestroy(e);
  return ms;
}

double SynthModel::run_e2e(int steps, int flags) {
  engine_.wait_all();
  const auto t0 = std::chrono::steady_clock::now();
  // every step uploads its inputs and reads its result back; the host reads
  // step i's result after queueing step i+1 (one step of lag, as a training
  // loop that logs the previous loss), so the next upload is not held back
  int prev = -1;
  for (int i = 0; i < steps; ++i) {
    enqueue_step(flags | kStepChecksum);
    if (prev >= 0) {
      engine_.wait_for(sum_tag_[prev]);
      volatile double v = sum_host_[prev];
      (void)v;
    }
    prev = sum_last_;
  }
  if (prev >= 0) {
    engine_.wait_for(sum_tag_[prev]);  // the last step's result is on the host
    volatile double v = sum_host_[prev];
    (void)v;
  }
  const auto t1 = std::chrono::steady_clock::now();
  engine_.wait_all();
  return std::chrono::duration<double, std::milli>(t1 - t0).count();
}

void SynthModel::read_weights(void* host, uint64_t bytes) {
  const uint64_t ws = dtype_size(cfg_.wdt);
  uint64_t need = 0;
  for (uint64_t n : cfg_.sizes) need += n * ws;
  if (bytes != need) throw UsageError("synth: read_weights buffer size differs from the weights' bytes");
  engine_.wait_all();
  engine_.bind_device();
  char* out = static_cast<char*>(host);
  for (size_t k = 0; k < cfg_.sizes.size(); ++k) {
    CSB_CUDA(cudaMemcpy(out, w_[k], cfg_.sizes[k] * ws, cudaMemcpyDeviceToHost));
    out += cfg_.sizes[k] * ws;
  }
}

double SynthModel::checksum() {
  enqueue_step(kStepChecksum);
  engine_.wait_for(sum_tag_[sum_last_]);
  return sum_host_[sum_last_];
}

}  // namespace csb
