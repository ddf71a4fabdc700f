// ref_driver.cpp -- C-ABI driver around the UNMODIFIED reference (collsim),
// compiled together with /root/reference/proj/core/src/*.cpp by
// oracle/Makefile into oracle/_ref/libcollsim_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/golden/make_golden.py to freeze
// golden vectors, by tests/ to pin oracle/oracle.c, and by bench.py's
// `--impl reference` / cpu_baseline leg to time the reference's own CPU path.
// It contains no reference source; it only calls the reference's public API
// (engine.hpp, collective.hpp, kvstore.hpp, model.hpp, runner.hpp).
//
// Loop shapes follow R/core/src/trainer.cpp:112-141 (train_epoch) and the
// kv_ranks fixture R/tests/test_kvstore.cpp:18-40.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "collsim/collective.hpp"
#include "collsim/engine.hpp"
#include "collsim/kvstore.hpp"
#include "collsim/model.hpp"
#include "collsim/runner.hpp"
#include "collsim/tensor.hpp"
#include "collsim/trace.hpp"

using namespace collsim;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (auto* ce = dynamic_cast<const Error*>(&e)) {
    switch (ce->kind()) {
      case Error::Kind::Config: return -1;
      case Error::Kind::Usage: return -2;
      case Error::Kind::Mismatch: return -3;
      case Error::Kind::DeadlockTimeout: return -4;
      case Error::Kind::Engine: return -5;
    }
  }
  return -9;
}

// One engine + store per rank thread over a shared transport
// (R/tests/test_kvstore.cpp:18-40).  Errors are recorded per rank.
template <typename Body>
int kv_ranks(int R, int engine_threads, KvConfig cfg, Transport& transport, TraceSink* sink,
             Body body) {
  std::vector<CommId> comms;
  if (cfg.mode == KvMode::ConCom) comms = create_communicators(transport, cfg.outstanding);
  std::vector<int> status(static_cast<size_t>(R), 0);
  std::vector<std::thread> threads;
  for (int r = 0; r < R; ++r) {
    threads.emplace_back([&, r] {
      Engine engine(engine_threads, r, sink);
      try {
        KvStore store(engine, transport, r, cfg, comms);
        body(r, engine, store);
        engine.wait_all();
      } catch (const std::exception& e) {
        status[static_cast<size_t>(r)] = fail(e);
        try {
          engine.wait_all();
        } catch (...) {
        }
      }
      engine.shutdown();
    });
  }
  for (auto& t : threads) t.join();
  for (int s : status)
    if (s != 0) return s;
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) { return mix_seed(seed, salt); }

void ref_random_uniform(double* out, int64_t n, uint64_t seed) {
  Tensor t = random_uniform(Shape{n}, seed);
  std::memcpy(out, t.data(), static_cast<size_t>(n) * sizeof(double));
}

// In-place Transport::allreduce_sum over R rank threads.  bufs: R*n doubles,
// rank-major; overwritten with the result each rank sees.
int ref_allreduce(int R, int64_t n, double* bufs) {
  try {
    Transport t(R, std::chrono::milliseconds(10000));
    std::vector<Tensor> ts;
    for (int r = 0; r < R; ++r) {
      Tensor x(Shape{n});
      std::memcpy(x.data(), bufs + r * n, static_cast<size_t>(n) * 8);
      ts.push_back(std::move(x));
    }
    std::vector<std::thread> th;
    for (int r = 0; r < R; ++r)
      th.emplace_back([&, r] { t.allreduce_sum(Transport::world(), r, ts[static_cast<size_t>(r)]); });
    for (auto& x : th) x.join();
    for (int r = 0; r < R; ++r)
      std::memcpy(bufs + r * n, ts[static_cast<size_t>(r)].data(), static_cast<size_t>(n) * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One full aggregation + SGD step through the reference KvStore, trainer
// loop shape for `mode` (trainer.cpp:112-141).  K keys of sizes[k]
// elements; rank r's gradient for key k is grads[(r*K + k)] (pointer array,
// R*K entries); weights start as w0[k] on rank 0 and zeros elsewhere
// (broadcast at init, kvstore.cpp:76-97).  Final weights of every rank are
// written to w_out[(r*K + k)].  iters steps are run with the same gradients.
int ref_train_steps(const char* mode_name, int R, int K, const int64_t* sizes,
                    const double* const* grads, const double* const* w0, double** w_out,
                    int iters, double lr, double rescale, int engine_threads, int outstanding,
                    const char* trace_path) {
  try {
    TraceSink sink;
    TraceSink* sp = (trace_path && trace_path[0]) ? &sink : nullptr;
    Transport transport(R, std::chrono::milliseconds(20000), sp);
    KvMode mode = parse_kv_mode(mode_name);
    KvConfig cfg{mode, outstanding, K};
    int rc = kv_ranks(R, engine_threads, cfg, transport, sp,
                      [&](int rank, Engine& engine, KvStore& store) {
                        std::vector<Tensor> w, g;
                        std::vector<Tag> wt, gt;
                        for (int k = 0; k < K; ++k) {
                          Tensor wk(Shape{sizes[k]});
                          if (rank == 0)
                            std::memcpy(wk.data(), w0[k], static_cast<size_t>(sizes[k]) * 8);
                          w.push_back(std::move(wk));
                          g.push_back(Tensor(Shape{sizes[k]}));
                          wt.push_back(engine.new_variable());
                          gt.push_back(engine.new_variable());
                        }
                        for (int k = 0; k < K; ++k) store.init(k, TensorSlot{w[k], wt[k]});
                        engine.wait_all();
                        auto sgd = [&](int k) {
                          Tensor* wp = &w[k];
                          Tensor* gp = &g[k];
                          engine.push([wp, gp, lr, rescale] { sgd_update(*wp, *gp, lr, rescale); },
                                      {gt[k]}, {wt[k]}, OpKind::Compute, k);
                        };
                        for (int it = 0; it < iters; ++it) {
                          // "backward": the gradient is (re)produced by an engine op
                          for (int k = K - 1; k >= 0; --k) {
                            Tensor* gp = &g[k];
                            const double* src = grads[rank * K + k];
                            int64_t n = sizes[k];
                            engine.push([gp, src, n] { std::memcpy(gp->data(), src, static_cast<size_t>(n) * 8); },
                                        {}, {gt[k]}, OpKind::Compute, k);
                          }
                          if (mode == KvMode::Funnel || mode == KvMode::ConCom) {
                            int since = 0;
                            for (int k = 0; k < K; ++k) {
                              store.push(k, TensorSlot{g[k], gt[k]});
                              store.pull(k, TensorSlot{g[k], gt[k]});
                              sgd(k);
                              if (mode == KvMode::ConCom && ++since == outstanding) {
                                store.barrier();
                                since = 0;
                              }
                            }
                            if (mode == KvMode::ConCom && since > 0) store.barrier();
                          } else {
                            for (int k = 0; k < K; ++k) store.push(k, TensorSlot{g[k], gt[k]});
                            for (int k = 0; k < K; ++k) {
                              store.pull(k, TensorSlot{g[k], gt[k]});
                              sgd(k);
                            }
                          }
                          engine.wait_all();
                        }
                        for (int k = 0; k < K; ++k)
                          std::memcpy(w_out[rank * K + k], w[k].data(),
                                      static_cast<size_t>(sizes[k]) * 8);
                      });
    if (sp) sink.write_jsonl(trace_path);
    return rc;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Appendix A scenario: run_scenario on the diamond model, trace to JSONL.
int ref_run_scenario(const char* mode, int workers, int engine_threads, int outstanding,
                     int epochs, int batch, int samples, uint64_t seed, const char* trace_path,
                     double* final_loss, double* accuracy) {
  try {
    RunConfig cfg;
    cfg.mode = parse_kv_mode(mode);
    cfg.workers = workers;
    cfg.engine_threads = engine_threads;
    cfg.outstanding = outstanding;
    cfg.epochs = epochs;
    cfg.global_batch = batch;
    cfg.samples = samples;
    cfg.seed = seed;
    cfg.trace_path = trace_path ? trace_path : "";
    Metrics m = run_scenario(cfg);
    if (final_loss) *final_loss = m.final_train_loss;
    if (accuracy) *accuracy = m.test_accuracy;
    if (!m.error.empty()) {
      g_err = m.error;
      return -3;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CPU bench arm (the reference's own path, timed): R rank threads x T engine
// threads, K keys of sizes[k] fp64 elements, gradients g = random_uniform(n_k,
// 1000 + rank*K + k) (test_kvstore.cpp:304 seeds).  One iteration is the
// trainer loop of `mode` (trainer.cpp:112-141): push(g) / pull(out) / sgd
// (w -= lr*rescale*out) -- the same work the GPU headline step times
// (push = pack, allreduce, pull + update).  flags:
//   1  compute only: sgd ops without the kvstore (exposed-comm denominator)
//   2  also a synthetic backward per iteration: one copy op per key
//      (src -> g) in descending key order, chained on one "backward" tag
// stats[0] = mean ms/iter (max over ranks), stats[1] = fp64 grad bytes/iter/rank.
int ref_bench(const char* mode_name, int R, int T, int outstanding, int K, const int64_t* sizes,
              int warmup, int iters, int flags, double lr, double rescale,
              double* stats) {
  const bool compute_only = (flags & 1) != 0, backward = (flags & 2) != 0;
  try {
    Transport transport(R, std::chrono::milliseconds(600000));
    KvMode mode = parse_kv_mode(mode_name);
    KvConfig cfg{mode, outstanding, K};
    std::vector<double> ms(static_cast<size_t>(R), 0.0);
    int64_t total = 0;
    for (int k = 0; k < K; ++k) total += sizes[k];
    int rc = kv_ranks(R, T, cfg, transport, nullptr, [&](int rank, Engine& engine, KvStore& store) {
      std::vector<Tensor> w, g, src, out;
      std::vector<Tag> wt, gt, ot;
      for (int k = 0; k < K; ++k) {
        w.push_back(random_uniform(Shape{sizes[k]}, mix_seed(7, static_cast<uint64_t>(k))));
        src.push_back(random_uniform(Shape{sizes[k]}, 1000 + static_cast<uint64_t>(rank * K + k)));
        g.push_back(src.back());
        out.push_back(Tensor(Shape{sizes[k]}));
        wt.push_back(engine.new_variable());
        gt.push_back(engine.new_variable());
        ot.push_back(engine.new_variable());
      }
      Tag bwd = engine.new_variable();
      if (!compute_only) {
        for (int k = 0; k < K; ++k) store.init(k, TensorSlot{w[k], wt[k]});
      }
      engine.wait_all();
      // sgd_update(w, aggregated gradient) as push_sgd_update (trainer.cpp:74-80)
      auto sgd = [&](int k, bool aggregated) {
        Tensor* wp = &w[k];
        Tensor* gp = aggregated ? &out[k] : &g[k];
        engine.push([wp, gp, lr, rescale] { sgd_update(*wp, *gp, lr, rescale); },
                    {aggregated ? ot[k] : gt[k]}, {wt[k]}, OpKind::Compute, k);
      };
      auto one_iter = [&] {
        if (backward) {
          for (int k = K - 1; k >= 0; --k) {
            Tensor* gp = &g[k];
            const Tensor* sp = &src[k];
            engine.push([gp, sp] { copy(*sp, *gp); }, {}, {gt[k], bwd}, OpKind::Compute, k);
          }
        }
        if (compute_only) {
          for (int k = 0; k < K; ++k) sgd(k, false);
        } else if (mode == KvMode::Funnel || mode == KvMode::ConCom) {
          int since = 0;
          for (int k = 0; k < K; ++k) {
            store.push(k, TensorSlot{g[k], gt[k]});
            store.pull(k, TensorSlot{out[k], ot[k]});
            sgd(k, true);
            if (mode == KvMode::ConCom && ++since == outstanding) {
              store.barrier();
              since = 0;
            }
          }
          if (mode == KvMode::ConCom && since > 0) store.barrier();
        } else {
          for (int k = 0; k < K; ++k) store.push(k, TensorSlot{g[k], gt[k]});
          for (int k = 0; k < K; ++k) {
            store.pull(k, TensorSlot{out[k], ot[k]});
            sgd(k, true);
          }
        }
        engine.wait_all();
      };
      for (int i = 0; i < warmup; ++i) one_iter();
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < iters; ++i) one_iter();
      auto t1 = std::chrono::steady_clock::now();
      ms[static_cast<size_t>(rank)] =
          std::chrono::duration<double, std::milli>(t1 - t0).count() / std::max(iters, 1);
    });
    double mx = 0.0;
    for (double v : ms) mx = std::max(mx, v);
    stats[0] = mx;
    stats[1] = static_cast<double>(total) * 8.0;
    return rc;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
