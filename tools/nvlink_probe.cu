// NVLink access-pattern probe: one process drives N GPUs (peer access
// enabled), every GPU runs the same pattern at once, device time is the max
// over GPUs.  Used to pick the shape of the peer-memory allreduce phases.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/nvlink_probe tools/nvlink_probe.cu
//   /tmp/nvlink_probe 4 100      # 4 GPUs, 100 MiB bucket per GPU
//
// Patterns (S = bucket bytes, shard = S/N):
//   pull    : GPU g copies shard g of every peer's bucket into local scratch
//   push    : GPU g writes shard p of its bucket into peer p's scratch
//   pullred : GPU g sums shard g over all N buckets (rank order), local store
//   bulk    : pull through TMA bulk copies (cp.async.bulk global->shared
//             from the peer, shared->global local)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int kMax = 8;
struct Bufs {
  float4* b[kMax];  // every GPU's bucket (peer-mapped)
  float4* s[kMax];  // every GPU's scratch (peer-mapped)
  int n, g;
  uint64_t shard;  // float4 per shard
};

template <int U>
__global__ void pull_k(Bufs p) {
  const uint64_t G = gridDim.x, c = blockIdx.x, T = p.shard;
  const uint64_t a = T * c / G, e = T * (c + 1) / G;
  for (int k = 1; k < p.n; ++k) {
    const int src = (p.g + k) % p.n;
    const float4* in = p.b[src] + (uint64_t)p.g * T;
    float4* out = p.s[p.g] + (uint64_t)src * T;
    uint64_t i = a + threadIdx.x;
    for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = in[i + u * blockDim.x];
#pragma unroll
      for (int u = 0; u < U; ++u) out[i + u * blockDim.x] = v[u];
    }
    for (; i < e; i += blockDim.x) out[i] = in[i];
  }
}

template <int U>
__global__ void push_k(Bufs p) {
  const uint64_t G = gridDim.x, c = blockIdx.x, T = p.shard;
  const uint64_t a = T * c / G, e = T * (c + 1) / G;
  for (int k = 1; k < p.n; ++k) {
    const int dst = (p.g + k) % p.n;
    const float4* in = p.b[p.g] + (uint64_t)dst * T;
    float4* out = p.s[dst] + (uint64_t)p.g * T;
    uint64_t i = a + threadIdx.x;
    for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = in[i + u * blockDim.x];
#pragma unroll
      for (int u = 0; u < U; ++u) out[i + u * blockDim.x] = v[u];
    }
    for (; i < e; i += blockDim.x) out[i] = in[i];
  }
}

template <int U>
__global__ void pullred_k(Bufs p) {
  const uint64_t G = gridDim.x, c = blockIdx.x, T = p.shard;
  const uint64_t a = T * c / G, e = T * (c + 1) / G;
  const uint64_t base = (uint64_t)p.g * T;
  for (uint64_t i = a + threadIdx.x; i < e; i += U * blockDim.x) {
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = make_float4(0, 0, 0, 0);
    for (int r = 0; r < p.n; ++r) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * blockDim.x < e) v[u] = p.b[r][base + i + u * blockDim.x];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x = __fadd_rn(acc[u].x, v[u].x);
        acc[u].y = __fadd_rn(acc[u].y, v[u].y);
        acc[u].z = __fadd_rn(acc[u].z, v[u].z);
        acc[u].w = __fadd_rn(acc[u].w, v[u].w);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < e) p.s[p.g][base + i + u * blockDim.x] = acc[u];
  }
}

// TMA bulk pull: one elected thread keeps ST CH-byte chunks in flight
// peer->smem (mbarrier per stage) and drains each with a bulk store to local
// global memory.
template <int CH, int ST>
__global__ void bulk_k(Bufs p) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[ST];
  const uint64_t G = gridDim.x, c = blockIdx.x;
  const uint64_t Tb = p.shard * 16;  // shard bytes
  const uint64_t a = (Tb * c / G) & ~uint64_t(15), e = (Tb * (c + 1) / G) & ~uint64_t(15);
  if (threadIdx.x != 0 || e <= a) return;
  for (int s = 0; s < ST; ++s) {
    uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint64_t per = (e - a + CH - 1) / CH;  // chunks per peer
  const uint64_t C = per * (p.n - 1);
  auto chunk = [&](uint64_t j, const char*& in, char*& out, uint32_t& bytes) {
    const int src = (p.g + 1 + static_cast<int>(j / per)) % p.n;
    const uint64_t o = a + (j % per) * CH;
    bytes = static_cast<uint32_t>(e - o < CH ? e - o : CH);
    in = reinterpret_cast<const char*>(p.b[src]) + (uint64_t)p.g * Tb + o;
    out = reinterpret_cast<char*>(p.s[p.g]) + (uint64_t)src * Tb + o;
  };
  auto load = [&](uint64_t j) {
    const char* in;
    char* out;
    uint32_t bytes;
    chunk(j, in, out, bytes);
    const int s = static_cast<int>(j % ST);
    uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(sm + s * CH));
    uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa),
                 "l"(in), "r"(bytes), "r"(ba)
                 : "memory");
  };
  for (uint64_t j = 0; j < C && j < ST; ++j) load(j);
  for (uint64_t j = 0; j < C; ++j) {
    const int s = static_cast<int>(j % ST);
    uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(&bar[s]));
    const uint32_t par = static_cast<uint32_t>((j / ST) & 1);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0, 1, 0, q; }"
                   : "=r"(done)
                   : "r"(ba), "r"(par)
                   : "memory");
    }
    const char* in;
    char* out;
    uint32_t bytes;
    chunk(j, in, out, bytes);
    uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(sm + s * CH));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out), "r"(sa), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (j >= 1 && j - 1 + ST < C) {  // refill the previous chunk's slot once its store has read smem
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      load(j - 1 + ST);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using KFn = void (*)(Bufs);

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 4;
  const double mib = argc > 2 ? atof(argv[2]) : 100;
  const uint64_t bytes = static_cast<uint64_t>(mib * (1 << 20)) / (16 * n) * (16 * n);
  std::vector<Bufs> P(n);
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < n; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
  }
  float4* b[kMax];
  float4* s[kMax];
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMalloc(&s[g], bytes));
    CK(cudaMemset(b[g], 0, bytes));
  }
  for (int g = 0; g < n; ++g) {
    for (int h = 0; h < n; ++h) {
      P[g].b[h] = b[h];
      P[g].s[h] = s[h];
    }
    P[g].n = n;
    P[g].g = g;
    P[g].shard = bytes / 16 / n;
  }
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  auto run = [&](const char* name, KFn fn, int grid, int block, int smem, double link_bytes) {
    for (int g = 0; g < n; ++g) {
      CK(cudaSetDevice(g));
      if (smem) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    const int iters = 20;
    for (int rep = 0; rep < 2; ++rep) {
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaStreamSynchronize(st[g]));
      }
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        for (int i = 0; i < (rep ? iters : 3); ++i) fn<<<grid, block, smem, st[g]>>>(P[g]);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0;
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      if (rep) {
        const double us = 1000.0 * worst / iters;
        printf("{\"pattern\": \"%s\", \"grid\": %d, \"block\": %d, \"us\": %.2f, \"link_GBps_per_dir\": %.1f}\n",
               name, grid, block, us, link_bytes / (us * 1e3));
      }
    }
  };
  const double inbound = static_cast<double>(bytes) * (n - 1) / n;  // per GPU per direction
  for (int grid : {148, 296}) {
    for (int block : {256, 512}) {
      run("pull_u1", pull_k<1>, grid, block, 0, inbound);
      run("pull_u4", pull_k<4>, grid, block, 0, inbound);
      run("push_u1", push_k<1>, grid, block, 0, inbound);
      run("push_u4", push_k<4>, grid, block, 0, inbound);
      run("pullred_u1", pullred_k<1>, grid, block, 0, inbound);
      run("pullred_u2", pullred_k<2>, grid, block, 0, inbound);
    }
  }
  if (!(argc > 3 && atoi(argv[3]) == 1)) {
    for (int grid : {148, 296, 592}) {
      run("bulk_16k_s4", bulk_k<16384, 4>, grid, 32, 4 * 16384, inbound);
      run("bulk_8k_s8", bulk_k<8192, 8>, grid, 32, 8 * 8192, inbound);
    }
  }
  // Copy engines: the same all-to-all exchange through cudaMemcpyPeerAsync
  // (no SM involved).  pull = the destination GPU's stream issues the copy,
  // push = the source GPU's; "1s" = one stream per GPU (copies serialise),
  // "ps" = one stream per peer (copies run concurrently on several CEs);
  // "oneway" = GPU 0 pulls from GPU 1 only (the 770 GB/s reference figure).
  std::vector<std::vector<cudaStream_t>> ps(n, std::vector<cudaStream_t>(kMax));
  std::vector<std::vector<cudaEvent_t>> pe(n, std::vector<cudaEvent_t>(kMax));
  for (int g = 0; g < n; ++g) {
    CK(cudaSetDevice(g));
    for (int k = 0; k < kMax; ++k) {
      CK(cudaStreamCreateWithFlags(&ps[g][k], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&pe[g][k], cudaEventDisableTiming));
    }
  }
  const uint64_t Tb = bytes / n;
  auto run_ce = [&](const char* name, bool push, bool par, bool oneway) {
    const int iters = 20;
    for (int rep = 0; rep < 2; ++rep) {
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        for (int k = 1; k < n; ++k) CK(cudaStreamWaitEvent(ps[g][k], e0[g], 0));
        for (int i = 0; i < (rep ? iters : 3); ++i) {
          for (int k = 1; k < n; ++k) {
            if (oneway && (g != 0 || k != 1)) continue;
            cudaStream_t cs = par ? ps[g][k] : st[g];
            const int p = (g + k) % n;
            if (!push) CK(cudaMemcpyPeerAsync(reinterpret_cast<char*>(s[g]) + p * Tb, g,
                                              reinterpret_cast<char*>(b[p]) + g * Tb, p, Tb, cs));
            else CK(cudaMemcpyPeerAsync(reinterpret_cast<char*>(s[p]) + g * Tb, p,
                                        reinterpret_cast<char*>(b[g]) + p * Tb, g, Tb, cs));
          }
        }
        if (par)
          for (int k = 1; k < n; ++k) {
            CK(cudaEventRecord(pe[g][k], ps[g][k]));
            CK(cudaStreamWaitEvent(st[g], pe[g][k], 0));
          }
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0;
      for (int g = 0; g < n; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      if (rep) {
        const double us = 1000.0 * worst / iters;
        const double lb = oneway ? static_cast<double>(Tb) : inbound;
        printf("{\"pattern\": \"%s\", \"us\": %.2f, \"link_GBps_per_dir\": %.1f}\n", name, us, lb / (us * 1e3));
      }
    }
  };
  run_ce("ce_pull_oneway", false, false, true);
  run_ce("ce_pull_1s", false, false, false);
  run_ce("ce_pull_ps", false, true, false);
  run_ce("ce_push_1s", true, false, false);
  run_ce("ce_push_ps", true, true, false);
  return 0;
}
