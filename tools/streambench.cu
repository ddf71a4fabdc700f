// streambench.cu -- design probe for the HBM-bound kernels on B200 (sm_100a).
//
// The fused one-rank kernel (a)+(c) moves g -> bucket and updates w, v:
// 3 streams read (g, w, v), 3 written (bucket, w, v), 24 B / element fp32.
// Two ways to keep enough bytes in flight:
//   vec  : every thread issues U x 16-B vector loads per stream, then stores
//          (register-limited occupancy; the round-1 design)
//   tma  : one thread per CTA streams tiles of every stream into shared
//          memory with cp.async.bulk (TMA, mbarrier complete_tx), S stages
//          deep; all threads update the tile in shared memory; the results
//          leave with cp.async.bulk stores (bulk_group), so the bytes in
//          flight no longer depend on registers.
// Also the pure copy (kernel (a)) in both styles, for the STREAM reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o streambench tools/streambench.cu
//   ./streambench [n_elems]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                 \
    }                                                                               \
  } while (0)

// ------------------------------------------------------------ vec style
template <int U, bool COPY_ONLY>
__global__ void __launch_bounds__(256) vec_kernel(const float* __restrict__ g, float* __restrict__ b,
                                                  float* __restrict__ w, float* __restrict__ v, uint64_t n4,
                                                  float step, float mu) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* b4 = reinterpret_cast<float4*>(b);
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* v4 = reinterpret_cast<float4*>(v);
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 gg[U], ww[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gg[u] = __ldcs(g4 + i + u * stride);
      if (!COPY_ONLY) {
        ww[u] = __ldcs(w4 + i + u * stride);
        vv[u] = __ldcs(v4 + i + u * stride);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      __stcs(b4 + i + u * stride, gg[u]);
      if (!COPY_ONLY) {
        float* gp = &gg[u].x;
        float* wp = &ww[u].x;
        float* vp = &vv[u].x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float nv = __fsub_rn(__fmul_rn(mu, vp[j]), __fmul_rn(step, gp[j]));
          vp[j] = nv;
          wp[j] = __fadd_rn(wp[j], nv);
        }
        __stcs(w4 + i + u * stride, ww[u]);
        __stcs(v4 + i + u * stride, vv[u]);
      }
    }
  }
  for (; i < n4; i += stride) {
    float4 gg = __ldcs(g4 + i);
    __stcs(b4 + i, gg);
    if (!COPY_ONLY) {
      float4 ww = __ldcs(w4 + i), vv = __ldcs(v4 + i);
      float* gp = &gg.x;
      float* wp = &ww.x;
      float* vp = &vv.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float nv = __fsub_rn(__fmul_rn(mu, vp[j]), __fmul_rn(step, gp[j]));
        vp[j] = nv;
        wp[j] = __fadd_rn(wp[j], nv);
      }
      __stcs(w4 + i, ww);
      __stcs(v4 + i, vv);
    }
  }
}

// Same arithmetic, but CTA c owns one contiguous chunk [n4*c/G, n4*(c+1)/G)
// (the round-1 table kernels' even split); LDCS: streaming loads, else
// default (L1-allocating) loads for w / v; STCS: streaming stores, else default.
template <int U, bool LDCS, bool STCS>
__global__ void __launch_bounds__(256) chunk_kernel(const float* __restrict__ g, float* __restrict__ b,
                                                    float* __restrict__ w, float* __restrict__ v, uint64_t n4,
                                                    float step, float mu) {
  const uint64_t lo = n4 * blockIdx.x / gridDim.x, hi = n4 * (blockIdx.x + 1) / gridDim.x;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* b4 = reinterpret_cast<float4*>(b);
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* v4 = reinterpret_cast<float4*>(v);
  const int T = blockDim.x;
  uint64_t i = lo + threadIdx.x;
  for (; i + (U - 1) * T < hi; i += U * T) {
    float4 gg[U], ww[U], vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      gg[u] = __ldcs(g4 + i + u * T);
      ww[u] = LDCS ? __ldcs(w4 + i + u * T) : w4[i + u * T];
      vv[u] = LDCS ? __ldcs(v4 + i + u * T) : v4[i + u * T];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float* gp = &gg[u].x;
      float* wp = &ww[u].x;
      float* vp = &vv[u].x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float nv = __fsub_rn(__fmul_rn(mu, vp[j]), __fmul_rn(step, gp[j]));
        vp[j] = nv;
        wp[j] = __fadd_rn(wp[j], nv);
      }
      if (STCS) {
        __stcs(b4 + i + u * T, gg[u]);
        __stcs(w4 + i + u * T, ww[u]);
        __stcs(v4 + i + u * T, vv[u]);
      } else {
        b4[i + u * T] = gg[u];
        w4[i + u * T] = ww[u];
        v4[i + u * T] = vv[u];
      }
    }
  }
  for (; i < hi; i += T) {
    float4 gg = __ldcs(g4 + i), ww = w4[i], vv = v4[i];
    float* gp = &gg.x;
    float* wp = &ww.x;
    float* vp = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float nv = __fsub_rn(__fmul_rn(mu, vp[j]), __fmul_rn(step, gp[j]));
      vp[j] = nv;
      wp[j] = __fadd_rn(wp[j], nv);
    }
    b4[i] = gg;
    w4[i] = ww;
    v4[i] = vv;
  }
}

// The library's walker shape: a thread owns a GROUP of 8 floats (2 x 16 B
// per stream), chunk j of 256 groups to CTA j mod G; TAB emulates the
// per-chunk table lookup (first[j], first[j+1], the entry) before the loads.
struct FakeEnt {
  const float* g;
  float* b;
  float* w;
  float* v;
  uint64_t n, gstart, gend;
};
template <bool TAB>
__global__ void __launch_bounds__(256) group_kernel(const FakeEnt* __restrict__ tab, const uint32_t* __restrict__ first,
                                                    uint64_t total, float step, float mu) {
  const uint64_t C = 256, nch = (total + C - 1) / C;
  for (uint64_t j = blockIdx.x; j < nch; j += gridDim.x) {
    const uint64_t q = j * C + threadIdx.x;
    if (q >= total) continue;
    FakeEnt en;
    if (TAB) {
      int lo = first[j], hi = first[j + 1];
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tab[mid].gstart <= q) lo = mid;
        else hi = mid - 1;
      }
      en = tab[lo];
    } else {
      en = tab[0];
    }
    const uint64_t i = (q - en.gstart) * 2;  // float4 index
    const float4* g4 = reinterpret_cast<const float4*>(en.g) + i;
    float4* b4 = reinterpret_cast<float4*>(en.b) + i;
    float4* w4 = reinterpret_cast<float4*>(en.w) + i;
    float4* v4 = reinterpret_cast<float4*>(en.v) + i;
    float4 gg[2], ww[2], vv[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      gg[u] = __ldcs(g4 + u);
      ww[u] = __ldcs(w4 + u);
      vv[u] = __ldcs(v4 + u);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float* gp = &gg[u].x;
      float* wp = &ww[u].x;
      float* vp = &vv[u].x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float nv = __fsub_rn(__fmul_rn(mu, vp[k]), __fmul_rn(step, gp[k]));
        vp[k] = nv;
        wp[k] = __fadd_rn(wp[k], nv);
      }
      __stcs(b4 + u, gg[u]);
      __stcs(w4 + u, ww[u]);
      __stcs(v4 + u, vv[u]);
    }
  }
}

// ------------------------------------------------------------ tma style
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TILE floats per stream per stage; S stages; 256 threads.  Tiles are
// assigned round-robin to CTAs (grid = SMs x ctas_per_sm, persistent).
template <int TILE, int S, bool COPY_ONLY>
__global__ void __launch_bounds__(256) tma_kernel(const float* __restrict__ g, float* __restrict__ b,
                                                  float* __restrict__ w, float* __restrict__ v, uint64_t n,
                                                  float step, float mu) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NS = COPY_ONLY ? 1 : 3;
  float* tiles = reinterpret_cast<float*>(smem);  // [S][NS][TILE]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + sizeof(float) * S * NS * TILE);
  const uint64_t ntiles = n / TILE;  // full tiles only (the probe uses n % TILE == 0)
  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint64_t mine = first < ntiles ? (ntiles - first + stride - 1) / stride : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t k) {  // k-th tile of this CTA into stage k % S
    const int s = static_cast<int>(k % S);
    const uint64_t t = first + k * stride;
    float* st = tiles + static_cast<size_t>(s) * NS * TILE;
    mbar_expect_tx(&full[s], NS * TILE * 4);
    bulk_load(st, g + t * TILE, TILE * 4, &full[s]);
    if (!COPY_ONLY) {
      bulk_load(st + TILE, w + t * TILE, TILE * 4, &full[s]);
      bulk_load(st + 2 * TILE, v + t * TILE, TILE * 4, &full[s]);
    }
  };
  if (threadIdx.x == 0)
    for (uint64_t k = 0; k < mine && k < S - 1; ++k) issue(k);
  for (uint64_t k = 0; k < mine; ++k) {
    const int s = static_cast<int>(k % S);
    const uint64_t t = first + k * stride;
    // refill: tile k+S-1 goes into the stage tile k-1 used; its stores
    // (the group before the newest) must have finished reading it
    if (threadIdx.x == 0 && k + S - 1 < mine) {
      bulk_wait_read<0>();
      issue(k + S - 1);
    }
    mbar_wait(&full[s], static_cast<uint32_t>((k / S) & 1));
    float* st = tiles + static_cast<size_t>(s) * NS * TILE;
    if (!COPY_ONLY) {
      float4* g4 = reinterpret_cast<float4*>(st);
      float4* w4 = reinterpret_cast<float4*>(st + TILE);
      float4* v4 = reinterpret_cast<float4*>(st + 2 * TILE);
      for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) {
        float4 gg = g4[i], ww = w4[i], vv = v4[i];
        float* gp = &gg.x;
        float* wp = &ww.x;
        float* vp = &vv.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float nv = __fsub_rn(__fmul_rn(mu, vp[j]), __fmul_rn(step, gp[j]));
          vp[j] = nv;
          wp[j] = __fadd_rn(wp[j], nv);
        }
        w4[i] = ww;
        v4[i] = vv;
      }
      fence_async_smem();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(b + t * TILE, st, TILE * 4);
      if (!COPY_ONLY) {
        bulk_store(w + t * TILE, st + TILE, TILE * 4);
        bulk_store(v + t * TILE, st + 2 * TILE, TILE * 4);
      }
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ------------------------------------------------------------ driver
struct Bufs {
  float *g, *b, *w, *v;
};

template <typename F>
float time_it(F f, int iters) {
  cudaEvent_t a, z;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&z));
  for (int i = 0; i < 3; ++i) f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) f();
  CK(cudaEventRecord(z));
  CK(cudaEventSynchronize(z));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, z));
  CK(cudaGetLastError());
  return ms / iters;
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (25557032ull / 16384) * 16384;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  Bufs B;
  CK(cudaMalloc(&B.g, n * 4));
  CK(cudaMalloc(&B.b, n * 4));
  CK(cudaMalloc(&B.w, n * 4));
  CK(cudaMalloc(&B.v, n * 4));
  CK(cudaMemset(B.g, 0, n * 4));
  CK(cudaMemset(B.w, 0, n * 4));
  CK(cudaMemset(B.v, 0, n * 4));
  const int iters = 20;
  const double fused_bytes = 24.0 * n, copy_bytes = 8.0 * n;
  auto report = [&](const char* name, double bytes, float ms) {
    std::printf("{\"kernel\": \"%s\", \"us\": %.2f, \"GBps\": %.1f}\n", name, ms * 1e3, bytes / (ms * 1e6));
  };
  const uint64_t n4 = n / 4;
  // torch-like reference copy
  report("cudaMemcpy_d2d", copy_bytes, time_it([&] { CK(cudaMemcpyAsync(B.b, B.g, n * 4, cudaMemcpyDeviceToDevice)); }, iters));
  for (int cps : {2, 3, 4, 6, 8}) {
    const int grid = sms * cps;
    char nm[64];
    std::snprintf(nm, sizeof nm, "vec_fused_U2_cps%d", cps);
    report(nm, fused_bytes, time_it([&] { vec_kernel<2, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
    std::snprintf(nm, sizeof nm, "vec_fused_U1_cps%d", cps);
    report(nm, fused_bytes, time_it([&] { vec_kernel<1, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
    std::snprintf(nm, sizeof nm, "vec_copy_U4_cps%d", cps);
    report(nm, copy_bytes, time_it([&] { vec_kernel<4, true><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 0, 0); }, iters));
  }
  for (int rep = 0; rep < 2; ++rep)
    for (int cps : {2, 3, 4}) {
      const int grid = sms * cps;
      char nm[64];
      std::snprintf(nm, sizeof nm, "chunk_U2_default_cps%d", cps);
      report(nm, fused_bytes, time_it([&] { chunk_kernel<2, false, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
      std::snprintf(nm, sizeof nm, "chunk_U2_cs_cps%d", cps);
      report(nm, fused_bytes, time_it([&] { chunk_kernel<2, true, true><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
      std::snprintf(nm, sizeof nm, "chunk_U1_cs_cps%d", cps);
      report(nm, fused_bytes, time_it([&] { chunk_kernel<1, true, true><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
      std::snprintf(nm, sizeof nm, "gridstride_U2_cs_cps%d", cps);
      report(nm, fused_bytes, time_it([&] { vec_kernel<2, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
      std::snprintf(nm, sizeof nm, "gridstride_U1_cs_cps%d", cps);
      report(nm, fused_bytes, time_it([&] { vec_kernel<1, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
    }
  {
    // one entry covering everything (161-key tables behave like this: big keys)
    const uint64_t groups = n / 8;
    FakeEnt h{B.g, B.b, B.w, B.v, n, 0, groups};
    FakeEnt* dt;
    uint32_t* df;
    CK(cudaMalloc(&dt, sizeof(FakeEnt)));
    CK(cudaMemcpy(dt, &h, sizeof(FakeEnt), cudaMemcpyHostToDevice));
    const uint64_t nch = (groups + 255) / 256;
    std::vector<uint32_t> f(nch + 1, 0);
    CK(cudaMalloc(&df, f.size() * 4));
    CK(cudaMemcpy(df, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 2; ++rep)
      for (int cps : {2, 3, 4}) {
        const int grid = sms * cps;
        char nm[64];
        std::snprintf(nm, sizeof nm, "group_notab_cps%d", cps);
        report(nm, fused_bytes, time_it([&] { group_kernel<false><<<grid, 256>>>(dt, df, groups, 1e-3f, 0.9f); }, iters));
        std::snprintf(nm, sizeof nm, "group_tab_cps%d", cps);
        report(nm, fused_bytes, time_it([&] { group_kernel<true><<<grid, 256>>>(dt, df, groups, 1e-3f, 0.9f); }, iters));
        std::snprintf(nm, sizeof nm, "gridstride_U1_cs_cps%d", cps);
        report(nm, fused_bytes, time_it([&] { vec_kernel<1, false><<<grid, 256>>>(B.g, B.b, B.w, B.v, n4, 1e-3f, 0.9f); }, iters));
      }
  }
  if (argc > 2) return 0;
  auto tma_run = [&](auto kern, int tile, int stages, int ns, int cps, bool copy, const char* tag) {
    const size_t smem = sizeof(float) * stages * ns * tile + 8 * stages;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int grid = sms * cps;
    char nm[96];
    std::snprintf(nm, sizeof nm, "tma_%s_tile%d_S%d_cps%d", tag, tile, stages, cps);
    report(nm, copy ? copy_bytes : fused_bytes,
           time_it([&] { kern<<<grid, 256, smem>>>(B.g, B.b, B.w, B.v, n, 1e-3f, 0.9f); }, iters));
  };
  tma_run(tma_kernel<2048, 3, false>, 2048, 3, 3, 1, false, "fused");
  tma_run(tma_kernel<2048, 4, false>, 2048, 4, 3, 1, false, "fused");
  tma_run(tma_kernel<2048, 3, false>, 2048, 3, 3, 2, false, "fused");
  tma_run(tma_kernel<4096, 3, false>, 4096, 3, 3, 1, false, "fused");
  tma_run(tma_kernel<4096, 4, false>, 4096, 4, 3, 1, false, "fused");
  tma_run(tma_kernel<1024, 4, false>, 1024, 4, 3, 2, false, "fused");
  tma_run(tma_kernel<1024, 6, false>, 1024, 6, 3, 2, false, "fused");
  tma_run(tma_kernel<4096, 4, true>, 4096, 4, 1, 1, true, "copy");
  tma_run(tma_kernel<8192, 4, true>, 8192, 4, 1, 1, true, "copy");
  tma_run(tma_kernel<4096, 6, true>, 4096, 6, 1, 2, true, "copy");
  return 0;
}
