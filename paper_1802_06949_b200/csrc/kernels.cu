// kernels.cu -- the memory-bound sm_100a kernels of the aggregation path.
//
//   (a) cs_pack        : table-driven copy/cast  (tensor.cpp:61-64 `copy`, used at
//                        kvstore.cpp:109 to stage g -> comm_buf, and at
//                        kvstore.cpp:160/170 to copy comm_buf -> out)
//   (b) cs_sum_buffers : multi-buffer rank-order sum, multi-output
//                        (collective.cpp:228-236: acc = b0; acc += b1 ...; copy to all)
//   (c) cs_sgd_update  : fused unpack + rescale + SGD / momentum update
//                        (model.cpp:17-27, trainer.cpp:74-80)
//   cs_synth_backward  : synthetic per-key backward producer (bench only)
//   cs_checksum        : deterministic fp64 checksum (e2e result read-back)
//
// Design (B200, HBM-bound, no tensor cores):
//   * 256-thread CTAs; every thread moves 8 elements per step as 16-byte
//     vectors (ld/st .v4 / .v2.f64), 2 steps unrolled with all loads issued
//     before any store -> 4096-element chunks, >= 64 B in flight per thread.
//   * A launch covers a whole table of keys (one bucket): the per-entry
//     chunk prefix sums, pointers and sizes travel in a __grid_constant__
//     kernel-parameter block (<= 15 KB, constant bank), so no host->device
//     copy precedes a launch; a CTA finds its entry by binary search.
//   * Grid = min(chunks, 148 SMs x 8 resident CTAs), grid-stride over chunks.
//   * Arithmetic uses explicit round-to-nearest intrinsics (__dmul_rn,
//     __fsub_rn, ...) so nothing is contracted into an FMA: fp64 results are
//     bit-identical to the reference, fp32 to the oracle's fp32 restatement.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace csb {
namespace {

constexpr int kThreads = 256;
constexpr int kVec = 8;     // elements per thread per step
constexpr int kUnroll = 2;  // steps in flight per thread
constexpr int kChunk = kThreads * kVec * kUnroll;  // 4096 elements

// ------------------------------------------------------------ vector IO

template <int DT>
struct Elem;
template <>
struct Elem<CS_F64> {
  using T = double;
};
template <>
struct Elem<CS_F32> {
  using T = float;
};
template <>
struct Elem<CS_BF16> {
  using T = __nv_bfloat16;
};

template <int A, int B>
struct AccOf {
  using T = float;
};
template <int B>
struct AccOf<CS_F64, B> {
  using T = double;
};
template <int A>
struct AccOf<A, CS_F64> {
  using T = double;
};
template <>
struct AccOf<CS_F64, CS_F64> {
  using T = double;
};

__device__ __forceinline__ float to_f(double x) { return __double2float_rn(x); }
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ double to_d(double x) { return x; }
__device__ __forceinline__ double to_d(float x) { return static_cast<double>(x); }
__device__ __forceinline__ double to_d(__nv_bfloat16 x) {
  return static_cast<double>(__bfloat162float(x));
}

template <typename Acc, typename T>
__device__ __forceinline__ Acc to_acc(T x);
template <>
__device__ __forceinline__ float to_acc<float, double>(double x) { return to_f(x); }
template <>
__device__ __forceinline__ float to_acc<float, float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_acc<float, __nv_bfloat16>(__nv_bfloat16 x) { return to_f(x); }
template <>
__device__ __forceinline__ double to_acc<double, double>(double x) { return x; }
template <>
__device__ __forceinline__ double to_acc<double, float>(float x) { return to_d(x); }
template <>
__device__ __forceinline__ double to_acc<double, __nv_bfloat16>(__nv_bfloat16 x) {
  return to_d(x);
}

template <typename T>
__device__ __forceinline__ T from_acc(float x);
template <typename T>
__device__ __forceinline__ T from_acc(double x);
template <>
__device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <>
__device__ __forceinline__ double from_acc<double>(float x) { return static_cast<double>(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ float from_acc<float>(double x) { return __double2float_rn(x); }
template <>
__device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(double x) {
  return __double2bfloat16(x);
}

// 8 contiguous elements <-> registers, as 16-byte vector accesses.
template <int DT, typename Acc>
__device__ __forceinline__ void load8(const void* base, uint64_t i, Acc (&v)[kVec]) {
  if constexpr (DT == CS_F64) {
    const double2* p = reinterpret_cast<const double2*>(static_cast<const double*>(base) + i);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 d = __ldcs(p + q);
      v[2 * q] = to_acc<Acc>(d.x);
      v[2 * q + 1] = to_acc<Acc>(d.y);
    }
  } else if constexpr (DT == CS_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + i);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float4 f = __ldcs(p + q);
      v[4 * q] = to_acc<Acc>(f.x);
      v[4 * q + 1] = to_acc<Acc>(f.y);
      v[4 * q + 2] = to_acc<Acc>(f.z);
      v[4 * q + 3] = to_acc<Acc>(f.w);
    }
  } else {
    const uint4* p =
        reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + i);
    uint4 u = __ldcs(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[q]);
      v[2 * q] = to_acc<Acc>(__low2bfloat16(h));
      v[2 * q + 1] = to_acc<Acc>(__high2bfloat16(h));
    }
  }
}

// Same, through the default (L2-allocating) path for data that is read and
// then rewritten in the same kernel (weights, momentum).
template <int DT, typename Acc>
__device__ __forceinline__ void load8_rw(const void* base, uint64_t i, Acc (&v)[kVec]) {
  if constexpr (DT == CS_F64) {
    const double2* p = reinterpret_cast<const double2*>(static_cast<const double*>(base) + i);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double2 d = p[q];
      v[2 * q] = to_acc<Acc>(d.x);
      v[2 * q + 1] = to_acc<Acc>(d.y);
    }
  } else if constexpr (DT == CS_F32) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + i);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float4 f = p[q];
      v[4 * q] = to_acc<Acc>(f.x);
      v[4 * q + 1] = to_acc<Acc>(f.y);
      v[4 * q + 2] = to_acc<Acc>(f.z);
      v[4 * q + 3] = to_acc<Acc>(f.w);
    }
  } else {
    const uint4* p =
        reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + i);
    uint4 u = *p;
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[q]);
      v[2 * q] = to_acc<Acc>(__low2bfloat16(h));
      v[2 * q + 1] = to_acc<Acc>(__high2bfloat16(h));
    }
  }
}

template <int DT, typename Acc>
__device__ __forceinline__ void store8(void* base, uint64_t i, const Acc (&v)[kVec]) {
  if constexpr (DT == CS_F64) {
    double2* p = reinterpret_cast<double2*>(static_cast<double*>(base) + i);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      p[q] = make_double2(from_acc<double>(v[2 * q]), from_acc<double>(v[2 * q + 1]));
  } else if constexpr (DT == CS_F32) {
    float4* p = reinterpret_cast<float4*>(static_cast<float*>(base) + i);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      p[q] = make_float4(from_acc<float>(v[4 * q]), from_acc<float>(v[4 * q + 1]),
                         from_acc<float>(v[4 * q + 2]), from_acc<float>(v[4 * q + 3]));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 h = __halves2bfloat162(from_acc<__nv_bfloat16>(v[2 * q]),
                                            from_acc<__nv_bfloat16>(v[2 * q + 1]));
      w[q] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + i) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int DT, typename Acc>
__device__ __forceinline__ Acc load1(const void* base, uint64_t i) {
  using T = typename Elem<DT>::T;
  return to_acc<Acc>(static_cast<const T*>(base)[i]);
}
template <int DT, typename Acc>
__device__ __forceinline__ void store1(void* base, uint64_t i, Acc x) {
  using T = typename Elem<DT>::T;
  static_cast<T*>(base)[i] = from_acc<T>(x);
}

// Round-to-nearest arithmetic that is never contracted into an FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// ------------------------------------------------------- table lookup

template <int CAP>
__device__ __forceinline__ int find_entry(const uint32_t* chunk_start, int n_entries, uint32_t c) {
  // largest e with chunk_start[e] <= c  (chunk_start[0] = 0, strictly
  // increasing over non-empty entries; empty entries are never produced)
  int lo = 0, hi = n_entries - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (chunk_start[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// ------------------------------------------------------------ (a) pack

template <int CAP>
struct PackParams {
  int n_entries;
  uint32_t total_chunks;
  uint32_t chunk_start[CAP];
  const void* src[CAP];
  void* dst[CAP];
  uint64_t n[CAP];
  uint8_t vec_ok[CAP];
};

template <int SDT, int DDT, int CAP>
__global__ void __launch_bounds__(kThreads) pack_kernel(const __grid_constant__ PackParams<CAP> p) {
  using Acc = typename AccOf<SDT, DDT>::T;
  for (uint32_t c = blockIdx.x; c < p.total_chunks; c += gridDim.x) {
    const int e = find_entry<CAP>(p.chunk_start, p.n_entries, c);
    const uint64_t base = static_cast<uint64_t>(c - p.chunk_start[e]) * kChunk;
    const uint64_t n = p.n[e];
    const uint64_t end = min(n, base + kChunk);
    const void* src = p.src[e];
    void* dst = p.dst[e];
    if (p.vec_ok[e]) {
      Acc v[kUnroll][kVec];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * kVec;
        if (i + kVec <= end) load8<SDT, Acc>(src, i, v[u]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * kVec;
        if (i + kVec <= end) {
          store8<DDT, Acc>(dst, i, v[u]);
        } else {
          for (uint64_t j = i; j < end; ++j) store1<DDT, Acc>(dst, j, load1<SDT, Acc>(src, j));
        }
      }
    } else {
      for (uint64_t j = base + threadIdx.x; j < end; j += kThreads)
        store1<DDT, Acc>(dst, j, load1<SDT, Acc>(src, j));
    }
  }
}

// ------------------------------------------------------------- (b) sum

struct SumParams {
  const void* in[CS_MAX_RANKS];
  void* out[CS_MAX_RANKS];
  int m;
  int nout;
  uint64_t n;
  uint32_t total_chunks;
  int vec_ok;
};

template <int DT, int M>
__global__ void __launch_bounds__(kThreads) sum_kernel(const __grid_constant__ SumParams p) {
  using Acc = typename AccOf<DT, DT>::T;  // f64 -> f64, f32 -> f32, bf16 -> f32
  const int m = (M > 0) ? M : p.m;
  for (uint32_t c = blockIdx.x; c < p.total_chunks; c += gridDim.x) {
    const uint64_t base = static_cast<uint64_t>(c) * kChunk;
    const uint64_t end = min(p.n, base + kChunk);
    if (p.vec_ok) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * kVec;
        if (i + kVec <= end) {
          Acc acc[kVec];
          load8_rw<DT, Acc>(p.in[0], i, acc);
          // fixed rank order: ((b0 + b1) + b2) + ...  (collective.cpp:229-233)
#pragma unroll 4
          for (int r = 1; r < m; ++r) {
            Acc x[kVec];
            load8_rw<DT, Acc>(p.in[r], i, x);
#pragma unroll
            for (int q = 0; q < kVec; ++q) acc[q] = add_rn(acc[q], x[q]);
          }
          for (int o = 0; o < p.nout; ++o) store8<DT, Acc>(p.out[o], i, acc);
        } else if (i < end) {
          for (uint64_t j = i; j < end; ++j) {
            Acc a = load1<DT, Acc>(p.in[0], j);
            for (int r = 1; r < m; ++r) a = add_rn(a, load1<DT, Acc>(p.in[r], j));
            for (int o = 0; o < p.nout; ++o) store1<DT, Acc>(p.out[o], j, a);
          }
        }
      }
    } else {
      for (uint64_t j = base + threadIdx.x; j < end; j += kThreads) {
        Acc a = load1<DT, Acc>(p.in[0], j);
        for (int r = 1; r < m; ++r) a = add_rn(a, load1<DT, Acc>(p.in[r], j));
        for (int o = 0; o < p.nout; ++o) store1<DT, Acc>(p.out[o], j, a);
      }
    }
  }
}

// ----------------------------------------------------------- (c) update

template <int CAP>
struct SgdParams {
  int n_entries;
  uint32_t total_chunks;
  double step;  // lr * rescale, computed in fp64 exactly as model.cpp:21
  double mu;
  uint32_t chunk_start[CAP];
  void* w[CAP];
  const void* g[CAP];
  void* mom[CAP];
  uint64_t n[CAP];
  uint8_t vec_ok[CAP];
};

template <int WDT, int GDT, bool MOM, int CAP>
__global__ void __launch_bounds__(kThreads) sgd_kernel(const __grid_constant__ SgdParams<CAP> p) {
  using Acc = typename AccOf<WDT, WDT>::T;  // f64 weights -> f64 math, else f32
  constexpr int MDT = (WDT == CS_F64) ? CS_F64 : CS_F32;
  const Acc step = static_cast<Acc>(p.step);
  const Acc mu = static_cast<Acc>(p.mu);
  for (uint32_t c = blockIdx.x; c < p.total_chunks; c += gridDim.x) {
    const int e = find_entry<CAP>(p.chunk_start, p.n_entries, c);
    const uint64_t base = static_cast<uint64_t>(c - p.chunk_start[e]) * kChunk;
    const uint64_t end = min(p.n[e], base + kChunk);
    void* w = p.w[e];
    const void* g = p.g[e];
    void* mom = p.mom[e];
    if (p.vec_ok[e]) {
      Acc gv[kUnroll][kVec], wv[kUnroll][kVec], mv[kUnroll][kVec];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * kVec;
        if (i + kVec <= end) {
          load8<GDT, Acc>(g, i, gv[u]);
          load8_rw<WDT, Acc>(w, i, wv[u]);
          if constexpr (MOM) load8_rw<MDT, Acc>(mom, i, mv[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t i = base + (static_cast<uint64_t>(u) * kThreads + threadIdx.x) * kVec;
        if (i + kVec <= end) {
#pragma unroll
          for (int q = 0; q < kVec; ++q) {
            if constexpr (MOM) {
              const Acc v = sub_rn(mul_rn(mu, mv[u][q]), mul_rn(step, gv[u][q]));
              mv[u][q] = v;
              wv[u][q] = add_rn(wv[u][q], v);
            } else {
              wv[u][q] = sub_rn(wv[u][q], mul_rn(step, gv[u][q]));
            }
          }
          store8<WDT, Acc>(w, i, wv[u]);
          if constexpr (MOM) store8<MDT, Acc>(mom, i, mv[u]);
        } else {
          for (uint64_t j = i; j < end; ++j) {
            Acc gg = load1<GDT, Acc>(g, j), ww = load1<WDT, Acc>(w, j);
            if constexpr (MOM) {
              const Acc v = sub_rn(mul_rn(mu, load1<MDT, Acc>(mom, j)), mul_rn(step, gg));
              store1<MDT, Acc>(mom, j, v);
              ww = add_rn(ww, v);
            } else {
              ww = sub_rn(ww, mul_rn(step, gg));
            }
            store1<WDT, Acc>(w, j, ww);
          }
        }
      }
    } else {
      for (uint64_t j = base + threadIdx.x; j < end; j += kThreads) {
        Acc gg = load1<GDT, Acc>(g, j), ww = load1<WDT, Acc>(w, j);
        if constexpr (MOM) {
          const Acc v = sub_rn(mul_rn(mu, load1<MDT, Acc>(mom, j)), mul_rn(step, gg));
          store1<MDT, Acc>(mom, j, v);
          ww = add_rn(ww, v);
        } else {
          ww = sub_rn(ww, mul_rn(step, gg));
        }
        store1<WDT, Acc>(w, j, ww);
      }
    }
  }
}

// ------------------------------------------------- synthetic backward

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int DT>
__global__ void __launch_bounds__(kThreads) synth_backward_kernel(const void* src, void* dst,
                                                                  uint64_t n, uint64_t spin_ns) {
  using Acc = typename AccOf<DT, DT>::T;
  const uint64_t t0 = globaltimer();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; j < n; j += stride)
    store1<DT, Acc>(dst, j, load1<DT, Acc>(src, j));
  if (spin_ns > 0 && threadIdx.x == 0) {
    while (globaltimer() - t0 < spin_ns) __nanosleep(500);
  }
}

// ------------------------------------------------------------ checksum

constexpr int kSumBlocks = 592;  // 148 SMs x 4

template <int DT>
__global__ void __launch_bounds__(kThreads) checksum_kernel(const void* x, uint64_t n, double* partial,
                                                            unsigned int* counter, double* out) {
  __shared__ double red[kThreads];
  double acc = 0.0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; j < n; j += stride)
    acc += load1<DT, double>(x, j);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = red[0];
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += const_cast<volatile double*>(partial)[b];
    *out = s;
    *counter = 0;  // re-arm for the next launch on this stream
  }
}

// ------------------------------------------------------------ host side

int sm_count_for_current_device() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (static_cast<int>(cache.size()) <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int sms = 0;
    CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = sms;
  }
  return cache[dev];
}

inline int grid_for(uint32_t chunks) {
  const int cap = sm_count_for_current_device() * (2048 / kThreads);
  return static_cast<int>(std::max<uint32_t>(1, std::min<uint32_t>(chunks, cap)));
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw_cuda(e, what, __FILE__, __LINE__);
}

template <int CAP>
void launch_pack_cap(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s);

template <int SDT, int DDT, int CAP>
void launch_pack_typed(const PackParams<CAP>& p, cudaStream_t s) {
  pack_kernel<SDT, DDT, CAP><<<grid_for(p.total_chunks), kThreads, 0, s>>>(p);
  check_launch("pack_kernel");
}

template <int CAP>
void launch_pack_cap(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s) {
  PackParams<CAP> p;
  p.n_entries = 0;
  uint32_t chunks = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].src || !es[i].dst) throw UsageError("cs_pack: null pointer in entry");
    const int k = p.n_entries++;
    p.chunk_start[k] = chunks;
    p.src[k] = es[i].src;
    p.dst[k] = es[i].dst;
    p.n[k] = es[i].n;
    p.vec_ok[k] = aligned16(es[i].src) && aligned16(es[i].dst);
    const uint64_t c = (es[i].n + kChunk - 1) / kChunk;
    if (chunks + c > 0xFFFFFFF0ull) throw UsageError("cs_pack: table too large");
    chunks += static_cast<uint32_t>(c);
  }
  p.total_chunks = chunks;
  if (p.n_entries == 0) return;
#define CSB_PACK_CASE(S, D) \
  if (sdt == S && ddt == D) return launch_pack_typed<S, D, CAP>(p, s);
  CSB_PACK_CASE(CS_F64, CS_F64)
  CSB_PACK_CASE(CS_F64, CS_F32)
  CSB_PACK_CASE(CS_F64, CS_BF16)
  CSB_PACK_CASE(CS_F32, CS_F64)
  CSB_PACK_CASE(CS_F32, CS_F32)
  CSB_PACK_CASE(CS_F32, CS_BF16)
  CSB_PACK_CASE(CS_BF16, CS_F64)
  CSB_PACK_CASE(CS_BF16, CS_F32)
  CSB_PACK_CASE(CS_BF16, CS_BF16)
#undef CSB_PACK_CASE
  throw UsageError("cs_pack: unsupported dtype pair");
}

template <int WDT, int GDT, bool MOM, int CAP>
void launch_sgd_typed(const SgdParams<CAP>& p, cudaStream_t s) {
  sgd_kernel<WDT, GDT, MOM, CAP><<<grid_for(p.total_chunks), kThreads, 0, s>>>(p);
  check_launch("sgd_kernel");
}

template <int CAP>
void launch_sgd_cap(const cs_update_entry* es, int n, int wdt, int gdt, double lr, double rescale,
                    double momentum, cudaStream_t s) {
  SgdParams<CAP> p;
  p.n_entries = 0;
  p.step = lr * rescale;  // model.cpp:21, fp64 on the host
  p.mu = momentum;
  const bool mom = momentum != 0.0;
  uint32_t chunks = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].w || !es[i].g) throw UsageError("cs_sgd_update: null pointer in entry");
    if (mom && !es[i].mom) throw UsageError("cs_sgd_update: momentum > 0 needs a momentum buffer");
    const int k = p.n_entries++;
    p.chunk_start[k] = chunks;
    p.w[k] = es[i].w;
    p.g[k] = es[i].g;
    p.mom[k] = es[i].mom;
    p.n[k] = es[i].n;
    p.vec_ok[k] = aligned16(es[i].w) && aligned16(es[i].g) && (!mom || aligned16(es[i].mom));
    chunks += static_cast<uint32_t>((es[i].n + kChunk - 1) / kChunk);
  }
  p.total_chunks = chunks;
  if (p.n_entries == 0) return;
#define CSB_SGD_CASE(W, G)                                                  \
  if (wdt == W && gdt == G) {                                               \
    if (mom) return launch_sgd_typed<W, G, true, CAP>(p, s);                \
    return launch_sgd_typed<W, G, false, CAP>(p, s);                        \
  }
  CSB_SGD_CASE(CS_F64, CS_F64)
  CSB_SGD_CASE(CS_F32, CS_F32)
  CSB_SGD_CASE(CS_F32, CS_BF16)
  CSB_SGD_CASE(CS_BF16, CS_BF16)
  CSB_SGD_CASE(CS_BF16, CS_F32)
#undef CSB_SGD_CASE
  throw UsageError(std::string("cs_sgd_update: unsupported dtype pair w=") + dtype_name(wdt) +
                   " g=" + dtype_name(gdt));
}

// Parameter-block capacities: small tables keep the launch's parameter
// upload short; big buckets (ResNet-152: up to a few hundred keys) use 512.
constexpr int kCaps[] = {4, 32, 512};

}  // namespace

// ---------------------------------------------------------------- API

void pack(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s) {
  if (n < 0) throw UsageError("cs_pack: negative entry count");
  for (int off = 0; off < n; off += 512) {
    const int m = std::min(512, n - off);
    if (m <= kCaps[0]) launch_pack_cap<4>(es + off, m, sdt, ddt, s);
    else if (m <= kCaps[1]) launch_pack_cap<32>(es + off, m, sdt, ddt, s);
    else launch_pack_cap<512>(es + off, m, sdt, ddt, s);
  }
}

void sgd_update(const cs_update_entry* es, int n, int wdt, int gdt, double lr, double rescale,
                double momentum, cudaStream_t s) {
  if (n < 0) throw UsageError("cs_sgd_update: negative entry count");
  for (int off = 0; off < n; off += 512) {
    const int m = std::min(512, n - off);
    if (m <= kCaps[0]) launch_sgd_cap<4>(es + off, m, wdt, gdt, lr, rescale, momentum, s);
    else if (m <= kCaps[1]) launch_sgd_cap<32>(es + off, m, wdt, gdt, lr, rescale, momentum, s);
    else launch_sgd_cap<512>(es + off, m, wdt, gdt, lr, rescale, momentum, s);
  }
}

void sum_buffers(const void* const* in, int m, void* const* out, int nout, uint64_t n, int dt,
                 cudaStream_t s) {
  if (m < 1 || m > CS_MAX_RANKS || nout < 0 || nout > CS_MAX_RANKS)
    throw UsageError("cs_sum_buffers: 1 <= m <= 16 and 0 <= nout <= 16 required");
  if (n == 0 || nout == 0) return;
  SumParams p{};
  bool vec = true;
  for (int r = 0; r < m; ++r) {
    if (!in[r]) throw UsageError("cs_sum_buffers: null input");
    p.in[r] = in[r];
    vec = vec && aligned16(in[r]);
  }
  for (int o = 0; o < nout; ++o) {
    if (!out[o]) throw UsageError("cs_sum_buffers: null output");
    p.out[o] = out[o];
    vec = vec && aligned16(out[o]);
  }
  p.m = m;
  p.nout = nout;
  p.n = n;
  p.total_chunks = static_cast<uint32_t>((n + kChunk - 1) / kChunk);
  p.vec_ok = vec ? 1 : 0;
  const int grid = grid_for(p.total_chunks);
#define CSB_SUM_M(DT)                                                                   \
  switch (m) {                                                                          \
    case 1: sum_kernel<DT, 1><<<grid, kThreads, 0, s>>>(p); break;                      \
    case 2: sum_kernel<DT, 2><<<grid, kThreads, 0, s>>>(p); break;                      \
    case 4: sum_kernel<DT, 4><<<grid, kThreads, 0, s>>>(p); break;                      \
    case 8: sum_kernel<DT, 8><<<grid, kThreads, 0, s>>>(p); break;                      \
    default: sum_kernel<DT, 0><<<grid, kThreads, 0, s>>>(p); break;                     \
  }
  switch (dt) {
    case CS_F64: CSB_SUM_M(CS_F64); break;
    case CS_F32: CSB_SUM_M(CS_F32); break;
    case CS_BF16: CSB_SUM_M(CS_BF16); break;
    default: throw UsageError("cs_sum_buffers: unknown dtype");
  }
#undef CSB_SUM_M
  check_launch("sum_kernel");
}

void synth_backward(const void* src, void* dst, uint64_t n, int dt, uint64_t spin_ns, int ctas,
                    cudaStream_t s) {
  const int grid = ctas > 0 ? ctas : sm_count_for_current_device();
  switch (dt) {
    case CS_F64: synth_backward_kernel<CS_F64><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    case CS_F32: synth_backward_kernel<CS_F32><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    case CS_BF16: synth_backward_kernel<CS_BF16><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    default: throw UsageError("cs_synth_backward: unknown dtype");
  }
  check_launch("synth_backward_kernel");
}

namespace {
struct ChecksumScratch {
  double* partial = nullptr;
  unsigned int* counter = nullptr;
};
}  // namespace

void checksum(const void* x, uint64_t n, int dt, double* out, cudaStream_t s) {
  static std::mutex mu;
  static std::vector<ChecksumScratch> per_dev;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  ChecksumScratch sc;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(dev + 1);
    if (!per_dev[dev].partial) {
      CSB_CUDA(cudaMalloc(&per_dev[dev].partial, kSumBlocks * sizeof(double)));
      CSB_CUDA(cudaMalloc(&per_dev[dev].counter, sizeof(unsigned int)));
      CSB_CUDA(cudaMemset(per_dev[dev].counter, 0, sizeof(unsigned int)));
    }
    sc = per_dev[dev];
  }
  switch (dt) {
    case CS_F64: checksum_kernel<CS_F64><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    case CS_F32: checksum_kernel<CS_F32><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    case CS_BF16: checksum_kernel<CS_BF16><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    default: throw UsageError("cs_checksum: unknown dtype");
  }
  check_launch("checksum_kernel");
}

}  // namespace csb
