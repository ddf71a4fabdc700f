// kernels.cu -- the memory-bound sm_100a kernels of the aggregation path.
//
//   (a) cs_pack        : table-driven copy/cast  (tensor.cpp:61-64 `copy`, used at
//                        kvstore.cpp:109 to stage g -> comm_buf, and at
//                        kvstore.cpp:160/170 to copy comm_buf -> out)
//   (b) cs_sum_buffers : multi-buffer rank-order sum, multi-output
//                        (collective.cpp:228-236: acc = b0; acc += b1 ...; copy to all)
//   (c) cs_sgd_update  : fused unpack + rescale + SGD / momentum update
//                        (model.cpp:17-27, trainer.cpp:74-80)
//   pack_sgd_tab_kernel: (a)+(c) fused for one rank (the allreduce between
//                        them is the identity): DepCha's whole step in one
//                        launch; registered gradients skip the staging store
//   p2p_allreduce_kernel / p2p_zero_kernel
//                      : (b)+(c) fused over CUDA-IPC peer memory or an NVSwitch
//                        multicast VA, one cooperative launch per bucket,
//                        rank-order sums, pair barriers per CTA; the ZeRO-1
//                        form updates a sharded master and all-gathers weights;
//                        gradients staged in-kernel or read in place from every
//                        rank's registered region (direct); optional per-CTA
//                        phase stamps (CSB_P2P_TRACE)
//   cs_synth_backward  : synthetic per-key backward producer (bench only)
//   cs_checksum        : deterministic fp64 checksum (e2e result read-back)
//
// Sections: vector IO | table lookup | (a) pack | (b) sum | (c) update |
// device-resident tables | fused NVLink allreduce | ZeRO-1 | synthetic
// backward | checksum | host side (launch accounting, launchers) | API |
// DeviceTable.
//
// Design of the streaming kernels (B200, HBM-bound, no tensor cores):
//   * 256-thread CTAs, one wave (148 SMs x resident CTAs); work in chunks of
//     256 x U 8-element groups dealt round-robin to the CTAs (for_chunks),
//     the last partial round split over every CTA; inside a chunk each lane
//     moves 16-byte slots lane-contiguously, every load of the chunk issued
//     before its first store.
//   * A launch covers a whole table of keys (one bucket): the entries live
//     in a device-resident table (DeviceTable, re-uploaded only when an entry
//     changes) with each chunk's first entry precomputed, or -- for the
//     one-off C-ABI launches -- in a __grid_constant__ parameter block.
//   * Streaming data moves with evict-first global loads / stores (LDG/STG
//     .EF.128 in SASS); the one-rank kernel is launched with programmatic
//     dependent launch.
//   * Arithmetic uses explicit round-to-nearest intrinsics (__dmul_rn,
//     __fsub_rn, ...) so nothing is contracted into an FMA: fp64 results are
//     bit-identical to the reference, fp32 to the oracle's fp32 restatement.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "hostprof.hpp"
#include "kernels.hpp"

namespace csb {
namespace {

constexpr int kThreads = 256;
constexpr int kVec = 8;     // elements per thread per step

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

// ------------------------------------------------------- work split

// Work is counted in GROUPS of kVec = 8 consecutive elements (one or more
// 16-byte vectors).  A launch covers the concatenation of its table's
// entries, T groups in total, dealt out in CHUNKS of kThreads x U groups:
// chunk j goes to CTA j mod G (a grid-stride over chunks; G = SMs x resident
// CTAs, one wave).  At any moment the G CTAs therefore stream G neighbouring
// chunks, so the whole GPU walks every array front to back and the DRAM rows
// it opens are shared by many CTAs.  Round 1 gave each CTA one contiguous
// range instead (T*c/G .. T*(c+1)/G); tools/streambench.cu measured that
// 10-25 % slower on B200 (the fused 24 B/element pattern: 4.7-5.5 TB/s
// contiguous vs 6.1-6.3 TB/s interleaved), the G concurrent streams per
// array each opening their own DRAM rows.
//
// A thread resolves its group's table entry per chunk: the host precomputes
// first[j], the entry holding chunk j's first group, so a chunk inside one
// key (the common case) needs no search and a chunk spanning small keys a
// binary search over just those keys.

__device__ __forceinline__ int find_entry(const uint64_t* group_start, int n_entries, uint64_t g) {
  // largest e with group_start[e] <= g (group_start[0] = 0; entries non-empty)
  int lo = 0, hi = n_entries - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (group_start[mid] <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// One table entry as a walker sees it: a/b/c/d per kernel (see DeviceTable::Entry).
struct Ent {
  const void* a;
  const void* b;
  void* c;
  void* d;
  uint64_t n, gstart;
  bool vec;
};

// Entries of a device-resident table (DeviceTable): first[j] = entry of
// chunk j's first group, first[nchunks] = the last entry.
struct TabView {
  const DeviceTable::Entry* __restrict__ tab;
  const uint32_t* __restrict__ first;
  const uint8_t* __restrict__ vecf;
  __device__ __forceinline__ Ent resolve(uint64_t j, uint64_t q) const {
    int lo = static_cast<int>(first[j]), hi = static_cast<int>(first[j + 1]);
    while (lo < hi) {  // largest e in [lo, hi] with gstart <= q
      const int mid = (lo + hi + 1) >> 1;
      if (tab[mid].gstart <= q) lo = mid;
      else hi = mid - 1;
    }
    const DeviceTable::Entry& en = tab[lo];
    return Ent{en.a, en.b, en.c, en.d, en.n, en.gstart, vecf[lo] != 0};
  }
};

// 16-byte vector IO for data touched once per launch: streaming
// (evict-first) loads and stores, explicitly global (LDG/STG, no generic
// address resolution).
template <int DT, typename Acc>
__device__ __forceinline__ void load8s(const void* base, uint64_t i, Acc (&v)[kVec]) {
  load8<DT, Acc>(base, i, v);  // __ldcs: ld.global.cs
}

template <int DT, typename Acc>
__device__ __forceinline__ void store8s(void* base, uint64_t i, const Acc (&v)[kVec]) {
  if constexpr (DT == CS_F64) {
    double2* p = reinterpret_cast<double2*>(static_cast<double*>(base) + i);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      __stcs(p + q, make_double2(from_acc<double>(v[2 * q]), from_acc<double>(v[2 * q + 1])));
  } else if constexpr (DT == CS_F32) {
    float4* p = reinterpret_cast<float4*>(static_cast<float*>(base) + i);
#pragma unroll
    for (int q = 0; q < 2; ++q)
      __stcs(p + q, make_float4(from_acc<float>(v[4 * q]), from_acc<float>(v[4 * q + 1]),
                                from_acc<float>(v[4 * q + 2]), from_acc<float>(v[4 * q + 3])));
  } else {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      __nv_bfloat162 h = __halves2bfloat162(from_acc<__nv_bfloat16>(v[2 * q]),
                                            from_acc<__nv_bfloat16>(v[2 * q + 1]));
      w[q] = *reinterpret_cast<uint32_t*>(&h);
    }
    __stcs(reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + i), make_uint4(w[0], w[1], w[2], w[3]));
  }
}

// E-element slots (one 16-byte vector of the widest dtype a kernel touches):
// streaming (evict-first), explicitly global loads / stores.
template <int DT>
constexpr int elem_bytes() {
  return DT == CS_F64 ? 8 : (DT == CS_F32 ? 4 : 2);
}

template <int DT, int E, typename Acc>
__device__ __forceinline__ void loadE(const void* base, uint64_t i, Acc (&v)[E]) {
  if constexpr (DT == CS_F64) {
    static_assert(E == 2 || E == 1, "f64 slots hold 1-2 elements");
    const double* p = static_cast<const double*>(base) + i;
    if constexpr (E == 2) {
      const double2 d = __ldcs(reinterpret_cast<const double2*>(p));
      v[0] = to_acc<Acc>(d.x);
      v[1] = to_acc<Acc>(d.y);
    } else {
      v[0] = to_acc<Acc>(__ldcs(p));
    }
  } else if constexpr (DT == CS_F32) {
    const float* p = static_cast<const float*>(base) + i;
    if constexpr (E == 4) {
      const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
      v[0] = to_acc<Acc>(f.x);
      v[1] = to_acc<Acc>(f.y);
      v[2] = to_acc<Acc>(f.z);
      v[3] = to_acc<Acc>(f.w);
    } else {
      static_assert(E == 2, "f32 slots hold 2 or 4 elements");
      const float2 f = __ldcs(reinterpret_cast<const float2*>(p));
      v[0] = to_acc<Acc>(f.x);
      v[1] = to_acc<Acc>(f.y);
    }
  } else {
    const __nv_bfloat16* p = static_cast<const __nv_bfloat16*>(base) + i;
    uint32_t w[E / 2];
    if constexpr (E == 8) {
      const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
      w[0] = u.x; w[1] = u.y; w[2] = u.z; w[3] = u.w;
    } else if constexpr (E == 4) {
      const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
      w[0] = u.x; w[1] = u.y;
    } else {
      static_assert(E == 2, "bf16 slots hold 2, 4 or 8 elements");
      w[0] = __ldcs(reinterpret_cast<const unsigned int*>(p));
    }
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[q]);
      v[2 * q] = to_acc<Acc>(__low2bfloat16(h));
      v[2 * q + 1] = to_acc<Acc>(__high2bfloat16(h));
    }
  }
}

template <int DT, int E, typename Acc>
__device__ __forceinline__ void storeE(void* base, uint64_t i, const Acc (&v)[E]) {
  if constexpr (DT == CS_F64) {
    double* p = static_cast<double*>(base) + i;
    if constexpr (E == 2) __stcs(reinterpret_cast<double2*>(p), make_double2(from_acc<double>(v[0]), from_acc<double>(v[1])));
    else __stcs(p, from_acc<double>(v[0]));
  } else if constexpr (DT == CS_F32) {
    float* p = static_cast<float*>(base) + i;
    if constexpr (E == 4)
      __stcs(reinterpret_cast<float4*>(p), make_float4(from_acc<float>(v[0]), from_acc<float>(v[1]),
                                                       from_acc<float>(v[2]), from_acc<float>(v[3])));
    else __stcs(reinterpret_cast<float2*>(p), make_float2(from_acc<float>(v[0]), from_acc<float>(v[1])));
  } else {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + i;
    uint32_t w[E / 2];
#pragma unroll
    for (int q = 0; q < E / 2; ++q) {
      __nv_bfloat162 h = __halves2bfloat162(from_acc<__nv_bfloat16>(v[2 * q]), from_acc<__nv_bfloat16>(v[2 * q + 1]));
      w[q] = *reinterpret_cast<uint32_t*>(&h);
    }
    if constexpr (E == 8) __stcs(reinterpret_cast<uint4*>(p), make_uint4(w[0], w[1], w[2], w[3]));
    else if constexpr (E == 4) __stcs(reinterpret_cast<uint2*>(p), make_uint2(w[0], w[1]));
    else __stcs(reinterpret_cast<unsigned int*>(p), w[0]);
  }
}

// Slot geometry of a walk: a chunk of kThreads x U groups is cut into slots
// of E elements; thread t takes slots t, t + kThreads, ..., so every vector
// instruction of the CTA covers one contiguous span (a group of 8 per thread
// -- two 16-B vectors 32 B apart per lane -- measured 8 % slower:
// tools/streambench.cu group_* vs gridstride_U1).
template <int... DTS>
constexpr int slot_elems() {
  int m = 0;
  ((m = elem_bytes<DTS>() > m ? elem_bytes<DTS>() : m), ...);
  return 16 / m;
}

// Chunk schedule of the streaming walkers: the full rounds deal whole chunks
// round-robin (chunk j to CTA j mod G, a grid-stride over chunks); the last,
// partial round's `rem` chunks are each split over P = G / rem CTAs, so the
// kernel does not end with one round in which most SMs have nothing to do
// (ResNet-50 at one rank: 12,480 chunks over 444 CTAs left 48 CTAs alone in
// a 29th round, ~3 % of the launch).  f(j, qa, qb): groups [qa, qb) of chunk j.
template <typename F>
__device__ __forceinline__ void for_chunks(uint64_t total, uint64_t C, F&& f) {
  const uint64_t G = gridDim.x, c = blockIdx.x;
  const uint64_t nch = (total + C - 1) / C;
  const uint64_t full = nch / G * G;
  for (uint64_t j = c; j < full; j += G) f(j, j * C, min(total, j * C + C));
  const uint64_t rem = nch - full;
  if (rem == 0) return;
  const uint64_t P = G / rem;  // >= 1 (rem < G)
  if (c >= rem * P) return;
  const uint64_t j = full + c % rem, part = c / rem;
  const uint64_t a = j * C, L = min(total, a + C) - a;
  f(j, a + L * part / P, a + L * (part + 1) / P);
}

__device__ __forceinline__ void cta_range(uint64_t T, uint64_t& g0, uint64_t& g1) {
  g0 = T * blockIdx.x / gridDim.x;
  g1 = T * (blockIdx.x + 1) / gridDim.x;
}

// ------------------------------------------------------------ (a) pack

template <int CAP>
struct PackParams {
  int n_entries;
  uint64_t total_groups;
  uint64_t group_start[CAP];
  const void* src[CAP];
  void* dst[CAP];
  uint64_t n[CAP];
  uint8_t vec_ok[CAP];
};

// groups [lo, hi) of one entry, all threads of the CTA
template <int SDT, int DDT, int NT = kThreads>
__device__ __forceinline__ void pack_segment(const void* src, void* dst, uint64_t n, bool vec,
                                             uint64_t lo, uint64_t hi) {
  constexpr int kThreads = NT;  // block size of the caller (the peer kernels use 512)
  using Acc = typename AccOf<SDT, DDT>::T;
  constexpr int U = 4;
  uint64_t q = lo + threadIdx.x;
  if (vec) {
    const uint64_t hi_full = min(hi, n / kVec);  // groups with all 8 elements present
    for (; q + (U - 1) * kThreads < hi_full; q += U * kThreads) {
      Acc v[U][kVec];
#pragma unroll
      for (int u = 0; u < U; ++u) load8<SDT, Acc>(src, (q + u * kThreads) * kVec, v[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) store8<DDT, Acc>(dst, (q + u * kThreads) * kVec, v[u]);
    }
    for (; q < hi_full; q += kThreads) {
      Acc v[kVec];
      load8<SDT, Acc>(src, q * kVec, v);
      store8<DDT, Acc>(dst, q * kVec, v);
    }
  }
  for (; q < hi; q += kThreads) {
    const uint64_t end = min(n, (q + 1) * kVec);
    for (uint64_t j = q * kVec; j < end; ++j) store1<DDT, Acc>(dst, j, load1<SDT, Acc>(src, j));
  }
}

// Walkers: U groups per thread per chunk, every load of the chunk issued
// before its first store.  `full` groups (8 elements present, 16-B aligned
// pointers) move as 16-B vectors, the rest element by element.
template <int SDT, int DDT, int U, typename View>
__device__ __forceinline__ void pack_walk(const View& t, uint64_t total) {
  using Acc = typename AccOf<SDT, DDT>::T;
  constexpr int E = slot_elems<SDT, DDT>();
  constexpr int SPG = kVec / E;  // slots per group
  constexpr int K = U * SPG;     // slots per thread per chunk
  constexpr uint64_t C = static_cast<uint64_t>(kThreads) * U;
  for_chunks(total, C, [&](uint64_t j, uint64_t qa, uint64_t qb) {
    Ent en[K];
    uint64_t el[K];
    bool act[K], full[K];
    Acc v[K][E];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t sl = static_cast<uint64_t>(k) * kThreads + threadIdx.x;
      const uint64_t q = qa + sl / SPG;
      act[k] = q < qb;
      full[k] = false;
      if (act[k]) {
        en[k] = t.resolve(j, q);
        el[k] = (q - en[k].gstart) * kVec + (sl % SPG) * E;
        act[k] = el[k] < en[k].n;
        full[k] = act[k] && en[k].vec && el[k] + E <= en[k].n;
        if (full[k]) loadE<SDT, E, Acc>(en[k].a, el[k], v[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!act[k]) continue;
      if (full[k]) {
        storeE<DDT, E, Acc>(en[k].c, el[k], v[k]);
      } else {
        const uint64_t end = min(en[k].n, el[k] + E);
        for (uint64_t i = el[k]; i < end; ++i) store1<DDT, Acc>(en[k].c, i, load1<SDT, Acc>(en[k].a, i));
      }
    }
  });
}

template <int CAP>
struct PackView {
  const PackParams<CAP>* p;
  __device__ __forceinline__ Ent resolve(uint64_t, uint64_t q) const {
    const int e = find_entry(p->group_start, p->n_entries, q);
    return Ent{p->src[e], nullptr, p->dst[e], nullptr, p->n[e], p->group_start[e], p->vec_ok[e] != 0};
  }
};

constexpr int kPackU = 2;  // groups per thread per chunk: 2 x 32 B in flight per thread (fp32)
constexpr int kSgdU = 1;   // 3 streams x 32 B in flight per thread already

template <int SDT, int DDT, int CAP>
__global__ void __launch_bounds__(kThreads) pack_kernel(const __grid_constant__ PackParams<CAP> p) {
  pack_walk<SDT, DDT, kPackU>(PackView<CAP>{&p}, p.total_groups);
}

// ------------------------------------------------------------- (b) sum

struct SumParams {
  const void* in[CS_MAX_RANKS];
  void* out[CS_MAX_RANKS];
  int m;
  int nout;
  uint64_t n;
  uint64_t total_groups;
  int vec_ok;
};

// fixed rank order: ((b0 + b1) + b2) + ...  (collective.cpp:229-233); all M
// inputs of a group are loaded before the first add, so a thread keeps M
// 16-byte loads in flight (local or NVLink peer addresses alike).
template <int DT, int M>
__global__ void __launch_bounds__(kThreads) sum_kernel(const __grid_constant__ SumParams p) {
  using Acc = typename AccOf<DT, DT>::T;  // f64 -> f64, f32 -> f32, bf16 -> f32
  const int m = (M > 0) ? M : p.m;
  const uint64_t full_groups = p.vec_ok ? p.n / kVec : 0;
  // chunks of kThreads groups, chunk j to CTA j mod G (see "work split")
  for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; q < p.total_groups;
       q += static_cast<uint64_t>(gridDim.x) * kThreads) {
    if (q < full_groups) {
      const uint64_t i = q * kVec;
      Acc acc[kVec];
      if constexpr (M > 0) {
        Acc x[M][kVec];
#pragma unroll
        for (int r = 0; r < M; ++r) load8_rw<DT, Acc>(p.in[r], i, x[r]);
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = x[0][j];
#pragma unroll
        for (int r = 1; r < M; ++r)
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[r][j]);
      } else {
        load8_rw<DT, Acc>(p.in[0], i, acc);
        for (int r = 1; r < m; ++r) {
          Acc x[kVec];
          load8_rw<DT, Acc>(p.in[r], i, x);
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[j]);
        }
      }
      for (int o = 0; o < p.nout; ++o) store8<DT, Acc>(p.out[o], i, acc);
    } else {
      const uint64_t end = min(p.n, (q + 1) * kVec);
      for (uint64_t j = q * kVec; j < end; ++j) {
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
  uint64_t total_groups;
  double step;  // lr * rescale, computed in fp64 exactly as model.cpp:21
  double mu;
  uint64_t group_start[CAP];
  void* w[CAP];
  const void* g[CAP];
  void* mom[CAP];
  uint64_t n[CAP];
  uint8_t vec_ok[CAP];
};

template <bool MOM, typename Acc>
__device__ __forceinline__ void sgd_elem(Acc& w, Acc g, Acc& m, Acc step, Acc mu) {
  if constexpr (MOM) {
    const Acc v = sub_rn(mul_rn(mu, m), mul_rn(step, g));  // v = mu*v - step*g
    m = v;
    w = add_rn(w, v);                                      // w = w + v
  } else {
    w = sub_rn(w, mul_rn(step, g));                        // w -= step*g (model.cpp:25)
  }
}

template <int WDT, int GDT, bool MOM, int NT = kThreads>
__device__ __forceinline__ void sgd_segment(void* w, const void* g, void* mom, uint64_t n, bool vec,
                                            uint64_t lo, uint64_t hi, double step_d, double mu_d) {
  constexpr int kThreads = NT;  // block size of the caller (the peer kernel uses 512)
  using Acc = typename AccOf<WDT, WDT>::T;  // f64 weights -> f64 math, else f32
  constexpr int MDT = (WDT == CS_F64) ? CS_F64 : CS_F32;
  constexpr int U = 2;
  const Acc step = static_cast<Acc>(step_d);
  const Acc mu = static_cast<Acc>(mu_d);
  uint64_t q = lo + threadIdx.x;
  if (vec) {
    const uint64_t hi_full = min(hi, n / kVec);
    for (; q + (U - 1) * kThreads < hi_full; q += U * kThreads) {
      Acc gv[U][kVec], wv[U][kVec], mv[U][kVec];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = (q + u * kThreads) * kVec;
        load8<GDT, Acc>(g, i, gv[u]);
        load8_rw<WDT, Acc>(w, i, wv[u]);
        if constexpr (MOM) load8_rw<MDT, Acc>(mom, i, mv[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = (q + u * kThreads) * kVec;
#pragma unroll
        for (int j = 0; j < kVec; ++j) sgd_elem<MOM>(wv[u][j], gv[u][j], mv[u][j], step, mu);
        store8<WDT, Acc>(w, i, wv[u]);
        if constexpr (MOM) store8<MDT, Acc>(mom, i, mv[u]);
      }
    }
    for (; q < hi_full; q += kThreads) {
      const uint64_t i = q * kVec;
      Acc gv[kVec], wv[kVec], mv[kVec];
      load8<GDT, Acc>(g, i, gv);
      load8_rw<WDT, Acc>(w, i, wv);
      if constexpr (MOM) load8_rw<MDT, Acc>(mom, i, mv);
#pragma unroll
      for (int j = 0; j < kVec; ++j) sgd_elem<MOM>(wv[j], gv[j], mv[j], step, mu);
      store8<WDT, Acc>(w, i, wv);
      if constexpr (MOM) store8<MDT, Acc>(mom, i, mv);
    }
  }
  for (; q < hi; q += kThreads) {
    const uint64_t end = min(n, (q + 1) * kVec);
    for (uint64_t j = q * kVec; j < end; ++j) {
      Acc ww = load1<WDT, Acc>(w, j), mm = Acc(0);
      if constexpr (MOM) mm = load1<MDT, Acc>(mom, j);
      sgd_elem<MOM>(ww, load1<GDT, Acc>(g, j), mm, step, mu);
      if constexpr (MOM) store1<MDT, Acc>(mom, j, mm);
      store1<WDT, Acc>(w, j, ww);
    }
  }
}

// Kernel (c) walker: a = g (comm dtype), b = momentum, c = weights.
template <int WDT, int GDT, bool MOM, int U, typename View>
__device__ __forceinline__ void sgd_walk(const View& t, uint64_t total, double step_d, double mu_d) {
  using Acc = typename AccOf<WDT, WDT>::T;  // f64 weights -> f64 math, else f32
  constexpr int MDT = (WDT == CS_F64) ? CS_F64 : CS_F32;
  constexpr int E = slot_elems<WDT, GDT, MDT>();
  constexpr int SPG = kVec / E;
  constexpr int K = U * SPG;
  constexpr uint64_t C = static_cast<uint64_t>(kThreads) * U;
  const Acc step = static_cast<Acc>(step_d);
  const Acc mu = static_cast<Acc>(mu_d);
  for_chunks(total, C, [&](uint64_t j, uint64_t qa, uint64_t qb) {
    Ent en[K];
    uint64_t el[K];
    bool act[K], full[K];
    Acc gv[K][E], wv[K][E], mv[K][E];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t sl = static_cast<uint64_t>(k) * kThreads + threadIdx.x;
      const uint64_t q = qa + sl / SPG;
      act[k] = q < qb;
      full[k] = false;
      if (act[k]) {
        en[k] = t.resolve(j, q);
        el[k] = (q - en[k].gstart) * kVec + (sl % SPG) * E;
        act[k] = el[k] < en[k].n;
        full[k] = act[k] && en[k].vec && el[k] + E <= en[k].n;
        if (full[k]) {
          loadE<GDT, E, Acc>(en[k].a, el[k], gv[k]);
          loadE<WDT, E, Acc>(en[k].c, el[k], wv[k]);
          if constexpr (MOM) loadE<MDT, E, Acc>(en[k].b, el[k], mv[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!act[k]) continue;
      void* mom = const_cast<void*>(en[k].b);
      if (full[k]) {
#pragma unroll
        for (int x = 0; x < E; ++x) sgd_elem<MOM>(wv[k][x], gv[k][x], mv[k][x], step, mu);
        storeE<WDT, E, Acc>(en[k].c, el[k], wv[k]);
        if constexpr (MOM) storeE<MDT, E, Acc>(mom, el[k], mv[k]);
      } else {
        const uint64_t end = min(en[k].n, el[k] + E);
        for (uint64_t i = el[k]; i < end; ++i) {
          Acc ww = load1<WDT, Acc>(en[k].c, i), mm = Acc(0);
          if constexpr (MOM) mm = load1<MDT, Acc>(mom, i);
          sgd_elem<MOM>(ww, load1<GDT, Acc>(en[k].a, i), mm, step, mu);
          if constexpr (MOM) store1<MDT, Acc>(mom, i, mm);
          store1<WDT, Acc>(en[k].c, i, ww);
        }
      }
    }
  });
}

template <int CAP>
struct SgdView {
  const SgdParams<CAP>* p;
  __device__ __forceinline__ Ent resolve(uint64_t, uint64_t q) const {
    const int e = find_entry(p->group_start, p->n_entries, q);
    return Ent{p->g[e], p->mom[e], p->w[e], nullptr, p->n[e], p->group_start[e], p->vec_ok[e] != 0};
  }
};

template <int WDT, int GDT, bool MOM, int CAP>
__global__ void __launch_bounds__(kThreads) sgd_kernel(const __grid_constant__ SgdParams<CAP> p) {
  sgd_walk<WDT, GDT, MOM, kSgdU>(SgdView<CAP>{&p}, p.total_groups, p.step, p.mu);
}

// ------------------------------------ device-resident tables (buckets)

using DevEntry = DeviceTable::Entry;

// The same walkers over a resident table: each chunk's first entry was
// precomputed on the host (DeviceTable::sync), entries are read through L1.
template <int SDT, int DDT>
__global__ void __launch_bounds__(kThreads)
    pack_tab_kernel(const DevEntry* __restrict__ tab, const uint32_t* __restrict__ first,
                    const uint8_t* __restrict__ vec, uint64_t total) {
  pack_walk<SDT, DDT, kPackU>(TabView{tab, first, vec}, total);
}

template <int WDT, int GDT, bool MOM>
__global__ void __launch_bounds__(kThreads)
    sgd_tab_kernel(const DevEntry* __restrict__ tab, const uint32_t* __restrict__ first,
                   const uint8_t* __restrict__ vec, uint64_t total, double step, double mu) {
  sgd_walk<WDT, GDT, MOM, kSgdU>(TabView{tab, first, vec}, total, step, mu);
}

// (a)+(c) fused for one rank (the allreduce between them is the identity):
// stage the gradient into its comm-bucket slot and update the weights from
// the staged value in the same pass -- kernel (a)'s cast (comm_rounded) and
// kernel (c)'s arithmetic on the same registers, so the result is bit for
// bit the unfused pack -> identity -> update chain.  Entry: a = g, b = mom,
// c = w, d = bucket slot (d == a: an in-place bucket view, no store).
template <int CDT, typename Acc>
__device__ __forceinline__ Acc comm_cast(Acc x) {
  if constexpr (CDT == CS_BF16) return static_cast<Acc>(__bfloat162float(__float2bfloat16_rn(static_cast<float>(x))));
  else if constexpr (CDT == CS_F32) return static_cast<Acc>(static_cast<float>(x));
  else return x;
}

template <int GDT, int CDT, int WDT, bool MOM, int U>
__device__ __forceinline__ void pack_sgd_walk(const TabView& t, uint64_t total, double step_d, double mu_d) {
  using Acc = typename AccOf<WDT, WDT>::T;
  constexpr int MDT = (WDT == CS_F64) ? CS_F64 : CS_F32;
  constexpr int E = slot_elems<GDT, CDT, WDT, MDT>();
  constexpr int SPG = kVec / E;
  constexpr int K = U * SPG;
  constexpr uint64_t C = static_cast<uint64_t>(kThreads) * U;
  const Acc step = static_cast<Acc>(step_d);
  const Acc mu = static_cast<Acc>(mu_d);
  for_chunks(total, C, [&](uint64_t j, uint64_t qa, uint64_t qb) {
    Ent en[K];
    uint64_t el[K];
    bool act[K], full[K];
    Acc gv[K][E], wv[K][E], mv[K][E];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t sl = static_cast<uint64_t>(k) * kThreads + threadIdx.x;
      const uint64_t q = qa + sl / SPG;
      act[k] = q < qb;
      full[k] = false;
      if (act[k]) {
        en[k] = t.resolve(j, q);
        el[k] = (q - en[k].gstart) * kVec + (sl % SPG) * E;
        act[k] = el[k] < en[k].n;
        full[k] = act[k] && en[k].vec && el[k] + E <= en[k].n;
        if (full[k]) {
          loadE<GDT, E, Acc>(en[k].a, el[k], gv[k]);
          loadE<WDT, E, Acc>(en[k].c, el[k], wv[k]);
          if constexpr (MOM) loadE<MDT, E, Acc>(en[k].b, el[k], mv[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!act[k]) continue;
      void* mom = const_cast<void*>(en[k].b);
      const bool stage = en[k].d != en[k].a;
      if (full[k]) {
#pragma unroll
        for (int x = 0; x < E; ++x) gv[k][x] = comm_cast<CDT>(gv[k][x]);
        if (stage) storeE<CDT, E, Acc>(en[k].d, el[k], gv[k]);
#pragma unroll
        for (int x = 0; x < E; ++x) sgd_elem<MOM>(wv[k][x], gv[k][x], mv[k][x], step, mu);
        storeE<WDT, E, Acc>(en[k].c, el[k], wv[k]);
        if constexpr (MOM) storeE<MDT, E, Acc>(mom, el[k], mv[k]);
      } else {
        const uint64_t end = min(en[k].n, el[k] + E);
        for (uint64_t i = el[k]; i < end; ++i) {
          const Acc gg = comm_cast<CDT>(load1<GDT, Acc>(en[k].a, i));
          if (stage) store1<CDT, Acc>(en[k].d, i, gg);
          Acc ww = load1<WDT, Acc>(en[k].c, i), mm = Acc(0);
          if constexpr (MOM) mm = load1<MDT, Acc>(mom, i);
          sgd_elem<MOM>(ww, gg, mm, step, mu);
          if constexpr (MOM) store1<MDT, Acc>(mom, i, mm);
          store1<WDT, Acc>(en[k].c, i, ww);
        }
      }
    }
  });
}

// Launched with programmatic dependent launch (CSB_PDL, default on): the
// next step's grid may be scheduled while this one drains, and waits in
// griddepcontrol.wait until this grid has completed and flushed -- the launch
// latency between two steps overlaps the previous step's tail.  Without the
// launch attribute both instructions are no-ops.
template <int GDT, int CDT, int WDT, bool MOM, int U>
__global__ void __launch_bounds__(kThreads)
    pack_sgd_tab_kernel(const DevEntry* __restrict__ tab, const uint32_t* __restrict__ first,
                        const uint8_t* __restrict__ vec, uint64_t total, double step, double mu) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  pack_sgd_walk<GDT, CDT, WDT, MOM, U>(TabView{tab, first, vec}, total, step, mu);
}

// ------------------------- fused NVLink allreduce (+ SGD) over peer memory
//
// One kernel per bucket per rank, all ranks launched with the same grid G
// (cooperative launch, so every CTA is resident).  With T groups in the
// bucket and N ranks, rank r owns shard r = groups [T*r/N, T*(r+1)/N); CTA
// c owns chunk c of every shard (an even split over G).
//   phase 1  CTA c of rank r reads chunk c of shard r from all N buckets
//            (NVLink peer loads), adds them in rank order -- exactly the
//            reference's ((b0 + b1) + b2) + ... (collective.cpp:229-233),
//            so every rank ends with bit-identical sums -- and stores the
//            sum into all N buckets (peer stores).
//   phase 2  after CTA c of every rank has finished phase 1 (pairwise
//            flags), CTA c runs the fused SGD / momentum update over chunk
//            c of every shard, reading the reduced gradient from its LOCAL
//            bucket (kernel (c), no separate launch, no copy-back).
// Synchronisation is per CTA pair: CTA c on rank r only waits for CTA c on
// the other ranks (st.release.sys / ld.acquire.sys on epoch-stamped flags
// in each rank's flag region), so there is no grid-wide barrier.  The
// matching ledger guarantees every rank launches the same op sequence.

constexpr int kP2PMaxCtas = 1184;
// 512-thread CTAs, one per SM: the NVLink phases run on the first 256 threads
// (more outstanding peer requests measured slower), the local HBM update phase
// on all 512.
constexpr int kP2PThreads = 512;
constexpr int kP2PLinkThreads = 256;
// Threads issuing the peer loads of a reduce phase.  With 2 ranks each
// thread has only one remote 16-B load in flight, so the whole CTA takes
// part (tools/nvlink_probe.cu at 2 GPUs: 266 GB/s with 256 threads/SM,
// 532 with 1024); from 3 ranks on, 256 threads keep enough in flight.
template <int M>
constexpr int reduce_threads() {
  return M == 2 ? kP2PThreads : kP2PLinkThreads;
}

struct P2PParams {
  void* bufs[CS_MAX_RANKS];
  uint32_t* flags[CS_MAX_RANKS];
  void* mc;  // NVLS: multicast VA of the bucket (bufs unused in phase 1)
  void* wm[CS_MAX_RANKS];    // ZeRO-1: every rank's master-weight shard (shard-local layout)
  void* mom_b;               // ZeRO-1: this rank's momentum shard (shard-local layout)
  const DevEntry* tab;
  uint32_t* abort_word;      // host-mapped: [0] abort code, [1..3] rank / phase / CTA of a timeout
  uint64_t timeout_ns;
  uint64_t groups;
  double step, mu;
  int nranks, rank, n_entries, shard_only;
  int sys_fence;  // explicit fence.sc.sys before the release store of a pair barrier (CSB_P2P_FENCE)
  int pack;       // stage the gradients (entry d) into this rank's bucket (entry a) before barrier 0
  uint32_t epoch;
  uint64_t piece;  // groups per piece of the interleaved CTA map (0: one contiguous range per CTA)
  uint64_t kmin;   // at least this many pieces per CTA when each would still hold >= 256 groups
  // direct: phase 1 reads every rank's gradients in place -- rank r's copy of
  // entry e is gbase[r] + (e.d - gbase[rank]) (registered regions, identical
  // layout on every rank) -- instead of staged bucket copies; nothing is packed
  int direct;
  void* gbase[CS_MAX_RANKS];
  // CSB_P2P_TRACE: per-CTA %globaltimer stamps of the launch's phases
  // (kP2PStamps per CTA: start, past barrier 0, own shard done, past
  // barrier 1, end), host-mapped; null = off
  uint64_t* stamps;
};

constexpr int kP2PStamps = 5;
__device__ __forceinline__ void p2p_stamp(const P2PParams& p, int i) {
  if (p.stamps && threadIdx.x == 0) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.stamps[static_cast<size_t>(blockIdx.x) * kP2PStamps + i] = t;
  }
}

// CTA c's share of shard s: the shard is cut into G x K equal pieces
// (K ~ L / (G x piece)), piece i to CTA i mod G -- interleaved like the
// streaming kernels' chunks ("work split": the GPU walks each array front to
// back), balanced to a group.  The map depends only on (T, N, G, piece),
// identical on every rank, so CTA c handles the same pieces everywhere --
// what the per-CTA pair barriers pair.  piece = 0: one contiguous range per
// CTA.  Default 4096 groups (128 KiB of fp32 per piece): ResNet-50 ZeRO-1
// step at 2 GPUs 0.263 ms vs 0.397 contiguous, at 4 GPUs 0.340 vs 0.343;
// small pieces (512) measured slower at 4 GPUs (0.427 ms).
// pieces per CTA of shard s (host twin: p2p_pieces_per_cta)
__device__ __forceinline__ uint64_t shard_k(const P2PParams& p, int s, uint64_t G) {
  const uint64_t T = p.groups;
  const uint64_t L = T * (s + 1) / p.nranks - T * s / p.nranks;
  uint64_t K = p.piece ? max(static_cast<uint64_t>(1), L / (G * p.piece)) : 1;
  if (p.piece && K < p.kmin && L / (G * p.kmin) >= 256) K = p.kmin;
  return K;
}

template <typename F>
__device__ __forceinline__ void for_pieces(const P2PParams& p, int s, F&& f) {
  const uint64_t T = p.groups, G = gridDim.x, c = blockIdx.x;
  const uint64_t s0 = T * s / p.nranks, L = T * (s + 1) / p.nranks - s0;
  const uint64_t K = shard_k(p, s, G);
  const uint64_t P = G * K;
  for (uint64_t k = 0; k < K; ++k) {
    const uint64_t i = c + k * G;
    f(s0, s0 + L * i / P, s0 + L * (i + 1) / P);
  }
}

__device__ __forceinline__ void flag_store(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t flag_load(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t abort_load(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// phase: 0 = arrival (my bucket is packed), 1 = my shard sums are stored,
// 2 = (shard_only) my update finished reading the owners' buckets.
// Returns false when the launch was aborted: the host set the abort word
// (engine watchdog, Transport::abort, a failed peer), or this CTA waited
// longer than timeout_ns for a peer and recorded kAbortDeviceTimeout.  The
// caller then returns at once -- the GPU stays usable (no __trap), and the
// host reports DeadlockTimeout.  The abort word lives in host memory, so it
// is read only after the first ~20 us of waiting, then every ~20 us.
__device__ __forceinline__ bool pair_barrier(const P2PParams& p, int phase) {
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = 0;
  __syncthreads();
  const int t = threadIdx.x;
  if (t < p.nranks) {
    // the release store publishes what this CTA wrote before the __syncthreads
    // (barrier + release, as CUTLASS's arrive); CSB_P2P_FENCE=1 adds a
    // fence.sc.sys in front (measured ~10 % slower on 25 MiB buckets)
    if (p.sys_fence) __threadfence_system();
    const size_t slot = (static_cast<size_t>(phase) * CS_MAX_RANKS + p.rank) * kP2PMaxCtas + blockIdx.x;
    flag_store(p.flags[t] + slot, p.epoch);
    const uint32_t* mine =
        p.flags[p.rank] + (static_cast<size_t>(phase) * CS_MAX_RANKS + t) * kP2PMaxCtas + blockIdx.x;
    uint64_t t0 = 0, next_poll = 0;
    while (static_cast<int32_t>(flag_load(mine) - p.epoch) < 0) {
      const uint64_t now = now_ns();
      if (t0 == 0) {
        t0 = now;
        next_poll = now + 20000;
      } else if (now >= next_poll) {
        next_poll = now + 20000;
        if (p.abort_word && abort_load(p.abort_word) != 0) {
          s_abort = 1;
          break;
        }
        if (now - t0 > p.timeout_ns) {
          if (p.abort_word) {
            // where: rank, phase, CTA and the peer that never arrived
            p.abort_word[1] = static_cast<uint32_t>(p.rank);
            p.abort_word[2] = static_cast<uint32_t>(phase) | (static_cast<uint32_t>(t) << 8);
            p.abort_word[3] = blockIdx.x;
            __threadfence_system();
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.abort_word), "r"(2u) : "memory");
          }
          s_abort = 1;
          break;
        }
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  return s_abort == 0;
}

// Phase 1 of the direct form: bucket groups [a, b), every rank's values read
// in place from its registered gradients, summed in rank order exactly as the
// staged form sums bucket copies; sink(q, acc) consumes group q's sum.
// Groups between keys (bucket padding) are skipped; the partial last group of
// a key reads its n % 8 elements and sums zeros beyond them, as the
// zero-padded bucket slot would.  A thread walks its groups in increasing
// order, so its entry only moves forward (one search per range).
template <int CDT, int M, typename Sink>
__device__ __forceinline__ void direct_reduce_range(const P2PParams& p, uint64_t a, uint64_t b, Sink&& sink) {
  using Acc = typename AccOf<CDT, CDT>::T;
  using T = typename Elem<CDT>::T;
  constexpr int NT = reduce_threads<M>();
  const int m = (M > 0) ? M : p.nranks;
  if (threadIdx.x >= NT || a >= b || p.n_entries == 0) return;
  int lo = 0, hi = p.n_entries;  // first entry with gend > a
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.tab[mid].gend <= a) lo = mid + 1;
    else hi = mid;
  }
  int e = lo;
  if (e >= p.n_entries) return;  // the range is trailing bucket padding
  const char* mine = static_cast<const char*>(p.gbase[p.rank]);
  for (uint64_t q = a + threadIdx.x; q < b; q += NT) {
    if (p.tab[e].gend <= q) {  // a stride of NT groups can skip many small keys: search, do not scan
      int l = e + 1, h = p.n_entries;
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (p.tab[mid].gend <= q) l = mid + 1;
        else h = mid;
      }
      e = l;
    }
    if (e >= p.n_entries) return;
    const uint64_t gstart = p.tab[e].gstart, n = p.tab[e].n;
    if (q < gstart) continue;  // padding between keys
    const uint64_t off = static_cast<uint64_t>(static_cast<const char*>(p.tab[e].d) - mine);
    const uint64_t el = (q - gstart) * kVec;
    Acc acc[kVec];
    if (el + kVec <= n) {
      if constexpr (M > 0) {
        Acc x[M][kVec];
#pragma unroll
        for (int r = 0; r < M; ++r) load8_rw<CDT, Acc>(static_cast<const char*>(p.gbase[r]) + off, el, x[r]);
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = x[0][j];
#pragma unroll
        for (int r = 1; r < M; ++r)
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[r][j]);
      } else {
        load8_rw<CDT, Acc>(static_cast<const char*>(p.gbase[0]) + off, el, acc);
        for (int r = 1; r < m; ++r) {
          Acc x[kVec];
          load8_rw<CDT, Acc>(static_cast<const char*>(p.gbase[r]) + off, el, x);
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[j]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        acc[j] = Acc(0);
        if (el + j < n) {
          acc[j] = to_acc<Acc>(reinterpret_cast<const T*>(static_cast<const char*>(p.gbase[0]) + off)[el + j]);
          for (int r = 1; r < m; ++r)
            acc[j] = add_rn(acc[j], to_acc<Acc>(reinterpret_cast<const T*>(static_cast<const char*>(p.gbase[r]) +
                                                                              off)[el + j]));
        }
      }
    }
    sink(q, acc);
  }
}

template <int CDT, int M>
__device__ __forceinline__ void p2p_reduce_chunk(const P2PParams& p, uint64_t a, uint64_t b) {
  using Acc = typename AccOf<CDT, CDT>::T;
  const int m = (M > 0) ? M : p.nranks;
  constexpr int NT = reduce_threads<M>();
  if (threadIdx.x >= NT) return;
  if (p.direct) {
    direct_reduce_range<CDT, M>(p, a, b, [&](uint64_t q, const Acc (&acc)[kVec]) {
      if (p.shard_only) store8<CDT, Acc>(p.bufs[p.rank], q * kVec, acc);
      else
        for (int r = 0; r < m; ++r) store8<CDT, Acc>(p.bufs[r], q * kVec, acc);
    });
    return;
  }
  for (uint64_t q = a + threadIdx.x; q < b; q += NT) {
    const uint64_t i = q * kVec;
    Acc acc[kVec];
    if constexpr (M > 0) {
      Acc x[M][kVec];
#pragma unroll
      for (int r = 0; r < M; ++r) load8_rw<CDT, Acc>(p.bufs[r], i, x[r]);
#pragma unroll
      for (int j = 0; j < kVec; ++j) acc[j] = x[0][j];
#pragma unroll
      for (int r = 1; r < M; ++r)
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[r][j]);
      if (p.shard_only) {
        store8<CDT, Acc>(p.bufs[p.rank], i, acc);
      } else {
#pragma unroll
        for (int r = 0; r < M; ++r) store8<CDT, Acc>(p.bufs[r], i, acc);
      }
    } else {
      load8_rw<CDT, Acc>(p.bufs[0], i, acc);
      for (int r = 1; r < m; ++r) {
        Acc x[kVec];
        load8_rw<CDT, Acc>(p.bufs[r], i, x);
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = add_rn(acc[j], x[j]);
      }
      if (p.shard_only) store8<CDT, Acc>(p.bufs[p.rank], i, acc);
      else
        for (int r = 0; r < m; ++r) store8<CDT, Acc>(p.bufs[r], i, acc);
    }
  }
}

// NVLS phase 1: the NVSwitch sums every rank's copy (multimem.ld_reduce on the
// multicast VA) and multimem.st writes the sum into every rank's copy.  The
// switch's reduction order is not the reference's rank order, so this path is
// within tolerance, not bit-exact (the IPC path above is bit-exact).
template <int CDT>
__device__ __forceinline__ void nvls_reduce_chunk(const P2PParams& p, uint64_t a, uint64_t b) {
  // 16-byte vectors; the multicast ops have long latency, so every thread
  // keeps U reductions in flight and all 512 threads take part (no peer
  // load queues to protect here)
  constexpr uint64_t kVPG = (CDT == CS_F32) ? 2 : 1;  // vectors per group
  constexpr int U = 4;
  const uint64_t va = a * kVPG, vb = b * kVPG;
  auto ld = [&](uint64_t v, uint32_t (&r)[4]) {
    if constexpr (CDT == CS_F32) {
      const float* ptr = static_cast<const float*>(p.mc) + v * 4;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(ptr) : "memory");
    } else {
      const __nv_bfloat16* ptr = static_cast<const __nv_bfloat16*>(p.mc) + v * 8;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(ptr) : "memory");
    }
  };
  auto st = [&](uint64_t v, const uint32_t (&r)[4]) {
    if constexpr (CDT == CS_F32) {
      float* ptr = static_cast<float*>(p.mc) + v * 4;
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
                   ::"l"(ptr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
    } else {
      __nv_bfloat16* ptr = static_cast<__nv_bfloat16*>(p.mc) + v * 8;
      asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};"
                   ::"l"(ptr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
    }
  };
  uint64_t v = va + threadIdx.x;
  for (; v + (U - 1) * kP2PThreads < vb; v += U * kP2PThreads) {
    uint32_t r[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) ld(v + u * kP2PThreads, r[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) st(v + u * kP2PThreads, r[u]);
  }
  for (; v < vb; v += kP2PThreads) {
    uint32_t r[4];
    ld(v, r);
    st(v, r);
  }
  // the sums were written through the multicast VA and are read back through
  // the unicast one after the pair barrier: virtually aliased accesses need a
  // proxy fence on both sides (the consumer side is after barrier 1)
  asm volatile("fence.proxy.alias;" ::: "memory");
}

// Kernel (a) folded into the peer kernels' phase 0.  CTA c stages column c
// of this rank's bucket -- chunk c of every shard, exactly the groups the
// peers' CTA c read from this bucket after the pair barrier -- from the
// gradients (entry d) into the bucket slots (entry a), on all 512 threads.
// The pair barrier that follows is the one the separate pack kernel's
// completion used to satisfy, so no launch, stream hop or extra barrier is
// added, and CTAs that finish staging early start reducing while others
// still stage.
template <int CDT>
__device__ __forceinline__ void p2p_pack_range(const P2PParams& p, uint64_t a, uint64_t b) {
  if (a >= b || p.n_entries == 0) return;
  int lo = 0, hi = p.n_entries;  // first entry with gend > a
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.tab[mid].gend <= a) lo = mid + 1;
    else hi = mid;
  }
  for (int e = lo; e < p.n_entries; ++e) {
    const DevEntry en = p.tab[e];
    if (en.gstart >= b) break;
    if (!en.d || en.d == en.a) continue;  // a bucket view: already in place
    const uint64_t s0 = max(a, en.gstart), s1 = min(b, en.gend);
    const bool vec = ((reinterpret_cast<uintptr_t>(en.a) | reinterpret_cast<uintptr_t>(en.d)) & 15u) == 0;
    pack_segment<CDT, CDT, kP2PThreads>(en.d, const_cast<void*>(en.a), en.n, vec, s0 - en.gstart,
                                        s1 - en.gstart);
  }
}

template <int CDT>
__device__ __forceinline__ void p2p_pack_column(const P2PParams& p) {
  for (int k = 0; k < p.nranks; ++k)  // own shard first
    for_pieces(p, (p.rank + k) % p.nranks, [&](uint64_t, uint64_t a, uint64_t b) { p2p_pack_range<CDT>(p, a, b); });
}

// SGD over bucket groups [a, b) of shard `owner` through the entries
// (bucket-group coordinates).  shard_only: the reduced gradient of another
// owner's shard is read from that owner's bucket over NVLink.
template <int WDT, int CDT, bool MOM>
__device__ __forceinline__ void p2p_update_range(const P2PParams& p, int owner, uint64_t a, uint64_t b) {
  if (a >= b || p.n_entries == 0) return;
  int lo = 0, hi = p.n_entries;  // first entry with gend > a
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.tab[mid].gend <= a) lo = mid + 1;
    else hi = mid;
  }
  for (int e = lo; e < p.n_entries; ++e) {
    const DevEntry en = p.tab[e];
    if (en.gstart >= b) break;
    const uint64_t s0 = max(a, en.gstart), s1 = min(b, en.gend);
    const bool vec = ((reinterpret_cast<uintptr_t>(en.a) | reinterpret_cast<uintptr_t>(en.b) |
                       reinterpret_cast<uintptr_t>(en.c)) & 15u) == 0;
    const void* g = en.a;
    if (p.shard_only && owner != p.rank)
      g = static_cast<const char*>(p.bufs[owner]) +
          (static_cast<const char*>(en.a) - static_cast<const char*>(p.bufs[p.rank]));
    sgd_segment<WDT, CDT, MOM, kP2PThreads>(en.c, g, const_cast<void*>(en.b), en.n, vec, s0 - en.gstart,
                                            s1 - en.gstart, p.step, p.mu);
  }
}

template <int CDT, int WDT, bool UPDATE, bool MOM, int M, bool NVLS = false>
__global__ void __launch_bounds__(kP2PThreads, 2) p2p_allreduce_kernel(const __grid_constant__ P2PParams p) {
  p2p_stamp(p, 0);
  if constexpr (UPDATE && !NVLS) {
    if (p.pack && !p.direct) p2p_pack_column<CDT>(p);
  }
  if (!pair_barrier(p, 0)) return;
  p2p_stamp(p, 1);
  for_pieces(p, p.rank, [&](uint64_t, uint64_t a, uint64_t b) {
    if constexpr (NVLS) nvls_reduce_chunk<CDT>(p, a, b);
    else p2p_reduce_chunk<CDT, M>(p, a, b);
  });
  auto update_shard = [&](int s) {
    for_pieces(p, s, [&](uint64_t, uint64_t a, uint64_t b) { p2p_update_range<WDT, CDT, MOM>(p, s, a, b); });
  };
  if constexpr (UPDATE && !NVLS) {
    // this CTA just wrote its chunk of the own shard: update it before
    // waiting for the peers (absorbs their skew)
    __syncthreads();
    update_shard(p.rank);
  }
  __syncthreads();
  p2p_stamp(p, 2);
  if (!pair_barrier(p, 1)) return;
  p2p_stamp(p, 3);
  if constexpr (NVLS) asm volatile("fence.proxy.alias;" ::: "memory");
  if constexpr (UPDATE) {
    // the other shards, staggered so the ranks start on different owners
    for (int k = NVLS ? 0 : 1; k < p.nranks; ++k) update_shard((p.rank + k) % p.nranks);
    // shard_only: owners may repack their buckets only after every reader is done
    if (p.shard_only) pair_barrier(p, 2);
  }
  __syncthreads();
  p2p_stamp(p, 4);
}

// ------------------------------------------------ ZeRO-1
//
// Reduce-scatter + sharded update + all-gather of the WEIGHTS in one
// cooperative launch.  Rank r keeps the master weights and the momentum of
// its shard only (shard-local layout, 1/N of the optimizer state):
//   phase 1  CTA c sums chunk c of shard r over the N buckets (peer loads,
//            rank order -- bit-identical sums) and, with the sum still in
//            registers, applies the SGD / momentum update to the master
//            shard (the same arithmetic as kernel (c) on the same values);
//   phase 2  after the pair barrier, CTA c copies chunk c of every owner's
//            updated master shard into this rank's weight tensors (peer
//            loads, staggered owners), through the key table.
// No trailing barrier: an owner rewrites its master only in the next launch,
// after that launch's arrival barrier, which every reader reaches only once
// this launch has finished on its GPU.

template <int CDT, typename Acc>
__device__ __forceinline__ Acc comm_rounded(Acc x) {  // the value the bucket would hold
  if constexpr (CDT == CS_BF16) return __bfloat162float(__float2bfloat16_rn(x));
  else return x;
}

template <int CDT, int WDT, bool MOM, int M>
__device__ __forceinline__ void zero_reduce_update(const P2PParams& p, uint64_t s0, uint64_t a, uint64_t b) {
  using CAcc = typename AccOf<CDT, CDT>::T;
  using WAcc = typename AccOf<WDT, WDT>::T;
  constexpr int MDT = (WDT == CS_F64) ? CS_F64 : CS_F32;
  const WAcc step = static_cast<WAcc>(p.step), mu = static_cast<WAcc>(p.mu);
  const int m = (M > 0) ? M : p.nranks;
  constexpr int NT = reduce_threads<M>();
  if (threadIdx.x >= NT) return;
  void* wm = p.wm[p.rank];
  // kernel (c) on the master shard, the sum still in registers
  auto update = [&](uint64_t q, const CAcc (&acc)[kVec]) {
    const uint64_t j = (q - s0) * kVec;  // shard-local element
    WAcc w[kVec], mv[kVec] = {};
    load8_rw<WDT, WAcc>(wm, j, w);
    if constexpr (MOM) load8_rw<MDT, WAcc>(p.mom_b, j, mv);
#pragma unroll
    for (int v = 0; v < kVec; ++v)
      sgd_elem<MOM>(w[v], static_cast<WAcc>(comm_rounded<CDT>(acc[v])), mv[v], step, mu);
    store8<WDT, WAcc>(wm, j, w);
    if constexpr (MOM) store8<MDT, WAcc>(p.mom_b, j, mv);
  };
  if (p.direct) {
    direct_reduce_range<CDT, M>(p, a, b, update);
    return;
  }
  for (uint64_t q = a + threadIdx.x; q < b; q += NT) {
    const uint64_t i = q * kVec;  // bucket element
    CAcc acc[kVec];
    if constexpr (M > 0) {
      CAcc x[M][kVec];
#pragma unroll
      for (int r = 0; r < M; ++r) load8_rw<CDT, CAcc>(p.bufs[r], i, x[r]);
#pragma unroll
      for (int v = 0; v < kVec; ++v) acc[v] = x[0][v];
#pragma unroll
      for (int r = 1; r < M; ++r)
#pragma unroll
        for (int v = 0; v < kVec; ++v) acc[v] = add_rn(acc[v], x[r][v]);
    } else {
      load8_rw<CDT, CAcc>(p.bufs[0], i, acc);
      for (int r = 1; r < m; ++r) {
        CAcc x[kVec];
        load8_rw<CDT, CAcc>(p.bufs[r], i, x);
#pragma unroll
        for (int v = 0; v < kVec; ++v) acc[v] = add_rn(acc[v], x[v]);
      }
    }
    update(q, acc);
  }
}

// owner s's updated master weights, bucket groups [a, b) of its shard (which
// starts at group s0), into this rank's weight tensors (table: c = weights)
template <int WDT>
__device__ __forceinline__ void zero_gather(const P2PParams& p, int s, uint64_t s0, uint64_t a, uint64_t b) {
  if (a >= b || p.n_entries == 0) return;
  constexpr uint64_t kElem = (WDT == CS_F64) ? 8 : 4;
  int lo = 0, hi = p.n_entries;  // first entry with gend > a
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.tab[mid].gend <= a) lo = mid + 1;
    else hi = mid;
  }
  const uintptr_t shard_base = reinterpret_cast<uintptr_t>(p.wm[s]);
  for (int e = lo; e < p.n_entries; ++e) {
    const DevEntry en = p.tab[e];
    if (en.gstart >= b) break;
    const uint64_t g0 = max(a, en.gstart), g1 = min(b, en.gend);
    // the key's element 0 sits at shard-local element (gstart - s0) * 8 (may
    // precede the shard when the key straddles it; only [g0, g1) is touched)
    const uintptr_t src = shard_base + (en.gstart * kVec - s0 * kVec) * kElem;
    const bool vec = ((src | reinterpret_cast<uintptr_t>(en.c)) & 15u) == 0;
    pack_segment<WDT, WDT, kP2PThreads>(reinterpret_cast<const void*>(src), en.c, en.n, vec, g0 - en.gstart,
                                        g1 - en.gstart);
  }
}

template <int CDT, int WDT, bool MOM, int M>
__global__ void __launch_bounds__(kP2PThreads, 2) p2p_zero_kernel(const __grid_constant__ P2PParams p) {
  p2p_stamp(p, 0);
  if (p.pack && !p.direct) p2p_pack_column<CDT>(p);
  if (!pair_barrier(p, 0)) return;
  p2p_stamp(p, 1);
  for_pieces(p, p.rank, [&](uint64_t s0, uint64_t a, uint64_t b) { zero_reduce_update<CDT, WDT, MOM, M>(p, s0, a, b); });
  __syncthreads();
  // own shard: no need to wait for the peers
  for_pieces(p, p.rank, [&](uint64_t s0, uint64_t a, uint64_t b) { zero_gather<WDT>(p, p.rank, s0, a, b); });
  __syncthreads();
  p2p_stamp(p, 2);
  if (!pair_barrier(p, 1)) return;
  p2p_stamp(p, 3);
  for (int k = 1; k < p.nranks; ++k) {
    const int s = (p.rank + k) % p.nranks;
    for_pieces(p, s, [&](uint64_t s0, uint64_t a, uint64_t b) { zero_gather<WDT>(p, s, s0, a, b); });
  }
  __syncthreads();
  p2p_stamp(p, 4);
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

// Launch counter (always on) and per-launch event timing (profiling on).
std::atomic<uint64_t> g_launches{0};
std::atomic<bool> g_prof_on{false};
struct ProfRec {
  int kind;
  int dev;
  cudaEvent_t a, b;
  double bytes;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_pending;
std::vector<std::pair<int, cudaEvent_t>> g_prof_free;
KernelStats g_prof_stats[kKernKinds];
uint64_t g_launch_kind[kKernKinds];

cudaEvent_t prof_event(int dev) {
  {
    std::lock_guard<std::mutex> lock(g_prof_mu);
    for (size_t i = 0; i < g_prof_free.size(); ++i) {
      if (g_prof_free[i].first == dev) {
        cudaEvent_t e = g_prof_free[i].second;
        g_prof_free.erase(g_prof_free.begin() + static_cast<long>(i));
        return e;
      }
    }
  }
  cudaEvent_t e;
  CSB_CUDA(cudaEventCreate(&e));
  return e;
}

// Brackets one launch: counts it, and when profiling is on records a pair
// of timing events on the launch stream (the kernel's own stream).
struct LaunchScope {
  int kind;
  double bytes;
  cudaStream_t s;
  int dev = -1;
  cudaEvent_t a = nullptr, b = nullptr;
  hostprof::Scope prof{hostprof::kLaunch};
  LaunchScope(int k, double by, cudaStream_t st) : kind(k), bytes(by), s(st) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (g_prof_on.load(std::memory_order_relaxed)) {
      CSB_CUDA(cudaGetDevice(&dev));
      a = prof_event(dev);
      b = prof_event(dev);
      CSB_CUDA(cudaEventRecord(a, s));
    }
  }
  void done() {
    if (!a) return;
    CSB_CUDA(cudaEventRecord(b, s));
    std::lock_guard<std::mutex> lock(g_prof_mu);
    g_prof_pending.push_back(ProfRec{kind, dev, a, b, bytes});
    g_launch_kind[kind]++;
  }
};

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

// One full wave: SMs x resident CTAs of this kernel (occupancy queried once
// per instantiation), fewer when there is less than a group per thread.
// CTAs per SM the streaming kernels may take.  Leaving part of every SM's
// register file free lets a concurrently launched collective (NCCL's CTAs,
// the cooperative peer kernel) start beside them instead of queueing behind
// a full-occupancy wave; 3 x 256 threads per SM is also the measured optimum
// of the standalone kernels (fewer CTAs contending for the L1tex queue).
// CSB_STREAM_CTAS_PER_SM overrides (default 3).
int stream_ctas_per_sm() {
  static const int v = [] {
    const char* e = std::getenv("CSB_STREAM_CTAS_PER_SM");
    const int x = e ? std::atoi(e) : 3;
    return std::max(1, std::min(8, x));
  }();
  return v;
}

template <typename Kernel>
int wave_grid(Kernel kernel, uint64_t groups, int u = 1) {
  // resident CTAs per SM, per kernel (instantiations share Kernel's type)
  static std::mutex mu;
  static std::map<const void*, int> occs;
  int occ;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = occs.find(reinterpret_cast<const void*>(kernel));
    if (it == occs.end()) {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess) b = 1;
      it = occs.emplace(reinterpret_cast<const void*>(kernel), std::max(1, std::min(b, stream_ctas_per_sm()))).first;
    }
    occ = it->second;
  }
  const uint64_t full = static_cast<uint64_t>(sm_count_for_current_device()) * occ;
  const uint64_t chunk = static_cast<uint64_t>(kThreads) * static_cast<uint64_t>(u);
  const uint64_t need = (groups + chunk - 1) / chunk;  // chunks: no CTA without one
  return static_cast<int>(std::max<uint64_t>(1, std::min(full, need)));
}

inline uint64_t groups_of(uint64_t n) { return (n + kVec - 1) / kVec; }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw_cuda(e, what, __FILE__, __LINE__);
}

template <int CAP>
void launch_pack_cap(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s);

template <int SDT, int DDT, int CAP>
void launch_pack_typed(const PackParams<CAP>& p, cudaStream_t s) {
  double elems = 0;
  for (int i = 0; i < p.n_entries; ++i) elems += static_cast<double>(p.n[i]);
  LaunchScope ls(kKernPack, elems * (sizeof(typename Elem<SDT>::T) + sizeof(typename Elem<DDT>::T)), s);
  pack_kernel<SDT, DDT, CAP><<<wave_grid(pack_kernel<SDT, DDT, CAP>, p.total_groups, kPackU), kThreads, 0, s>>>(p);
  check_launch("pack_kernel");
  ls.done();
}

template <int CAP>
void launch_pack_cap(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s) {
  PackParams<CAP> p;
  p.n_entries = 0;
  uint64_t groups = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].src || !es[i].dst) throw UsageError("cs_pack: null pointer in entry");
    const int k = p.n_entries++;
    p.group_start[k] = groups;
    p.src[k] = es[i].src;
    p.dst[k] = es[i].dst;
    p.n[k] = es[i].n;
    p.vec_ok[k] = aligned16(es[i].src) && aligned16(es[i].dst);
    groups += groups_of(es[i].n);
  }
  p.total_groups = groups;
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
  double elems = 0;
  for (int i = 0; i < p.n_entries; ++i) elems += static_cast<double>(p.n[i]);
  const double mom_bytes = MOM ? 2.0 * (WDT == CS_F64 ? 8 : 4) : 0.0;
  LaunchScope ls(kKernSgd,
                 elems * (2.0 * sizeof(typename Elem<WDT>::T) + sizeof(typename Elem<GDT>::T) + mom_bytes), s);
  sgd_kernel<WDT, GDT, MOM, CAP><<<wave_grid(sgd_kernel<WDT, GDT, MOM, CAP>, p.total_groups, kSgdU), kThreads, 0, s>>>(p);
  check_launch("sgd_kernel");
  ls.done();
}

template <int CAP>
void launch_sgd_cap(const cs_update_entry* es, int n, int wdt, int gdt, double lr, double rescale,
                    double momentum, cudaStream_t s) {
  SgdParams<CAP> p;
  p.n_entries = 0;
  p.step = lr * rescale;  // model.cpp:21, fp64 on the host
  p.mu = momentum;
  const bool mom = momentum != 0.0;
  uint64_t groups = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].w || !es[i].g) throw UsageError("cs_sgd_update: null pointer in entry");
    if (mom && !es[i].mom) throw UsageError("cs_sgd_update: momentum > 0 needs a momentum buffer");
    const int k = p.n_entries++;
    p.group_start[k] = groups;
    p.w[k] = es[i].w;
    p.g[k] = es[i].g;
    p.mom[k] = es[i].mom;
    p.n[k] = es[i].n;
    p.vec_ok[k] = aligned16(es[i].w) && aligned16(es[i].g) && (!mom || aligned16(es[i].mom));
    groups += groups_of(es[i].n);
  }
  p.total_groups = groups;
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
  p.total_groups = groups_of(n);
  p.vec_ok = vec ? 1 : 0;
  LaunchScope ls(kKernSum, static_cast<double>(n) * dtype_size(dt) * (m + nout), s);
#define CSB_SUM_LAUNCH(DT, M) \
  sum_kernel<DT, M><<<wave_grid(sum_kernel<DT, M>, p.total_groups), kThreads, 0, s>>>(p)
#define CSB_SUM_M(DT)                          \
  switch (m) {                                 \
    case 1: CSB_SUM_LAUNCH(DT, 1); break;      \
    case 2: CSB_SUM_LAUNCH(DT, 2); break;      \
    case 3: CSB_SUM_LAUNCH(DT, 3); break;      \
    case 4: CSB_SUM_LAUNCH(DT, 4); break;      \
    case 8: CSB_SUM_LAUNCH(DT, 8); break;      \
    default: CSB_SUM_LAUNCH(DT, 0); break;     \
  }
  switch (dt) {
    case CS_F64: CSB_SUM_M(CS_F64); break;
    case CS_F32: CSB_SUM_M(CS_F32); break;
    case CS_BF16: CSB_SUM_M(CS_BF16); break;
    default: throw UsageError("cs_sum_buffers: unknown dtype");
  }
#undef CSB_SUM_M
#undef CSB_SUM_LAUNCH
  check_launch("sum_kernel");
  ls.done();
}

void synth_backward(const void* src, void* dst, uint64_t n, int dt, uint64_t spin_ns, int ctas,
                    cudaStream_t s) {
  const int grid = ctas > 0 ? ctas : sm_count_for_current_device();
  LaunchScope ls(kKernSynth, static_cast<double>(n) * 2 * (n ? dtype_size(dt) : 0), s);
  switch (dt) {
    case CS_F64: synth_backward_kernel<CS_F64><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    case CS_F32: synth_backward_kernel<CS_F32><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    case CS_BF16: synth_backward_kernel<CS_BF16><<<grid, kThreads, 0, s>>>(src, dst, n, spin_ns); break;
    default: throw UsageError("cs_synth_backward: unknown dtype");
  }
  check_launch("synth_backward_kernel");
  ls.done();
}

namespace {
struct ChecksumScratch {
  double* partial = nullptr;
  unsigned int* counter = nullptr;
};
}  // namespace

void checksum(const void* x, uint64_t n, int dt, double* out, cudaStream_t s) {
  // scratch per (device, stream): checksums on different streams of one
  // device (rank threads sharing a GPU) must not share the last-block counter
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, ChecksumScratch> scratch;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  ChecksumScratch sc;
  {
    std::lock_guard<std::mutex> lock(mu);
    ChecksumScratch& e = scratch[{dev, s}];
    if (!e.partial) {
      CSB_CUDA(cudaMalloc(&e.partial, kSumBlocks * sizeof(double)));
      CSB_CUDA(cudaMalloc(&e.counter, sizeof(unsigned int)));
      CSB_CUDA(cudaMemset(e.counter, 0, sizeof(unsigned int)));
    }
    sc = e;
  }
  LaunchScope ls(kKernChecksum, static_cast<double>(n) * dtype_size(dt), s);
  switch (dt) {
    case CS_F64: checksum_kernel<CS_F64><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    case CS_F32: checksum_kernel<CS_F32><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    case CS_BF16: checksum_kernel<CS_BF16><<<kSumBlocks, kThreads, 0, s>>>(x, n, sc.partial, sc.counter, out); break;
    default: throw UsageError("cs_checksum: unknown dtype");
  }
  check_launch("checksum_kernel");
  ls.done();
}

// ------------------------------------------------------- DeviceTable

DeviceTable::~DeviceTable() {
  if (dev_) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev_device_);
    cudaFree(dev_);
    cudaSetDevice(prev);
  }
}

// Computes every chunk's first entry (chunk = kThreads x U groups, see
// "work split"; first_[nchunks] = the last entry) and makes the device copy
// current (uploading only when the bytes differ).  chunk_groups = 0: entries
// only (the peer kernels' tables).
void DeviceTable::sync(uint64_t chunk_groups, cudaStream_t s) {
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  // steady state (same keys every step): nothing to recompute or upload
  if (dev_ && dev == dev_device_ && chunk_groups == chunk_ && host_.size() == last_host_.size() &&
      vec_ == last_vec_ &&
      std::memcmp(host_.data(), last_host_.data(), host_.size() * sizeof(Entry)) == 0)
    return;
  last_host_ = host_;
  last_vec_ = vec_;
  chunk_ = chunk_groups;
  first_.clear();
  if (chunk_groups > 0 && groups_ > 0) {
    const uint64_t nch = (groups_ + chunk_groups - 1) / chunk_groups;
    first_.assign(static_cast<size_t>(nch) + 1, 0);
    size_t e = 0;
    for (uint64_t j = 0; j <= nch; ++j) {
      const uint64_t g0 = std::min(j * chunk_groups, groups_ - 1);
      while (e + 1 < host_.size() && host_[e].gend <= g0) ++e;
      first_[static_cast<size_t>(j)] = static_cast<uint32_t>(e);
    }
  }
  const size_t eb = host_.size() * sizeof(Entry), fb = first_.size() * 4, vb = vec_.size();
  std::vector<unsigned char> img(eb + fb + vb);
  std::memcpy(img.data(), host_.data(), eb);
  std::memcpy(img.data() + eb, first_.data(), fb);
  std::memcpy(img.data() + eb + fb, vec_.data(), vb);
  if (dev_ && dev == dev_device_ && img == shadow_) return;
  void* fresh = nullptr;
  CSB_CUDA(cudaMallocAsync(&fresh, img.size(), s));
  // pageable source: staged before the call returns, ordered on `s`
  CSB_CUDA(cudaMemcpyAsync(fresh, img.data(), img.size(), cudaMemcpyHostToDevice, s));
  if (dev_) {
    if (dev == dev_device_) CSB_CUDA(cudaFreeAsync(dev_, s));
    else throw UsageError("DeviceTable: used from a different device");
  }
  dev_ = fresh;
  dev_device_ = dev;
  shadow_.swap(img);
  ++uploads_;
}

void DeviceTable::pack(const cs_copy_entry* es, int n, int sdt, int ddt, cudaStream_t s) {
  host_.clear();
  vec_.clear();
  groups_ = 0;
  double elems = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].src || !es[i].dst) throw UsageError("cs_pack: null pointer in entry");
    const uint64_t g = groups_of(es[i].n);
    host_.push_back(Entry{es[i].src, nullptr, es[i].dst, es[i].n, groups_, groups_ + g});
    vec_.push_back(aligned16(es[i].src) && aligned16(es[i].dst));
    groups_ += g;
    elems += static_cast<double>(es[i].n);
  }
  if (host_.empty()) return;
  LaunchScope ls(kKernPack, elems * static_cast<double>(dtype_size(sdt) + dtype_size(ddt)), s);
#define CSB_PACK_TAB(S, D)                                                              \
  if (sdt == S && ddt == D) {                                                           \
    grid_ = wave_grid(pack_tab_kernel<S, D>, groups_, kPackU);                          \
    sync(static_cast<uint64_t>(kThreads) * kPackU, s);                                  \
    const char* base = static_cast<const char*>(dev_);                                  \
    pack_tab_kernel<S, D><<<grid_, kThreads, 0, s>>>(                                   \
        reinterpret_cast<const Entry*>(base),                                           \
        reinterpret_cast<const uint32_t*>(base + host_.size() * sizeof(Entry)),         \
        reinterpret_cast<const uint8_t*>(base + host_.size() * sizeof(Entry) + first_.size() * 4), \
        groups_);                                                                       \
    check_launch("pack_tab_kernel");                                                    \
    ls.done();                                                                          \
    return;                                                                             \
  }
  CSB_PACK_TAB(CS_F64, CS_F64)
  CSB_PACK_TAB(CS_F32, CS_F32)
  CSB_PACK_TAB(CS_F32, CS_BF16)
  CSB_PACK_TAB(CS_BF16, CS_F32)
  CSB_PACK_TAB(CS_BF16, CS_BF16)
  CSB_PACK_TAB(CS_F32, CS_F64)
  CSB_PACK_TAB(CS_F64, CS_F32)
  CSB_PACK_TAB(CS_BF16, CS_F64)
  CSB_PACK_TAB(CS_F64, CS_BF16)
#undef CSB_PACK_TAB
  throw UsageError("cs_pack: unsupported dtype pair");
}

void DeviceTable::sgd(const cs_update_entry* es, int n, int wdt, int gdt, double lr, double rescale,
                      double momentum, cudaStream_t s) {
  host_.clear();
  vec_.clear();
  groups_ = 0;
  const bool mom = momentum != 0.0;
  double elems = 0;
  for (int i = 0; i < n; ++i) {
    if (es[i].n == 0) continue;
    if (!es[i].w || !es[i].g) throw UsageError("cs_sgd_update: null pointer in entry");
    if (mom && !es[i].mom) throw UsageError("cs_sgd_update: momentum > 0 needs a momentum buffer");
    const uint64_t g = groups_of(es[i].n);
    host_.push_back(Entry{es[i].g, es[i].mom, es[i].w, es[i].n, groups_, groups_ + g});
    vec_.push_back(aligned16(es[i].w) && aligned16(es[i].g) && (!mom || aligned16(es[i].mom)));
    groups_ += g;
    elems += static_cast<double>(es[i].n);
  }
  if (host_.empty()) return;
  const double step = lr * rescale;  // model.cpp:21, fp64 on the host
  const double mom_bytes = mom ? 2.0 * (wdt == CS_F64 ? 8 : 4) : 0.0;
  LaunchScope ls(kKernSgd, elems * (2.0 * dtype_size(wdt) + dtype_size(gdt) + mom_bytes), s);
#define CSB_SGD_TAB(W, G, M)                                                            \
  if (wdt == W && gdt == G && mom == M) {                                               \
    grid_ = wave_grid(sgd_tab_kernel<W, G, M>, groups_, kSgdU);                         \
    sync(static_cast<uint64_t>(kThreads) * kSgdU, s);                                   \
    const char* base = static_cast<const char*>(dev_);                                  \
    sgd_tab_kernel<W, G, M><<<grid_, kThreads, 0, s>>>(                                 \
        reinterpret_cast<const Entry*>(base),                                           \
        reinterpret_cast<const uint32_t*>(base + host_.size() * sizeof(Entry)),         \
        reinterpret_cast<const uint8_t*>(base + host_.size() * sizeof(Entry) + first_.size() * 4), \
        groups_, step, momentum);                                                       \
    check_launch("sgd_tab_kernel");                                                     \
    ls.done();                                                                          \
    return;                                                                             \
  }
  CSB_SGD_TAB(CS_F64, CS_F64, false)
  CSB_SGD_TAB(CS_F64, CS_F64, true)
  CSB_SGD_TAB(CS_F32, CS_F32, false)
  CSB_SGD_TAB(CS_F32, CS_F32, true)
  CSB_SGD_TAB(CS_F32, CS_BF16, false)
  CSB_SGD_TAB(CS_F32, CS_BF16, true)
  CSB_SGD_TAB(CS_BF16, CS_BF16, false)
  CSB_SGD_TAB(CS_BF16, CS_BF16, true)
  CSB_SGD_TAB(CS_BF16, CS_F32, false)
  CSB_SGD_TAB(CS_BF16, CS_F32, true)
#undef CSB_SGD_TAB
  throw UsageError(std::string("cs_sgd_update: unsupported dtype pair w=") + dtype_name(wdt) +
                   " g=" + dtype_name(gdt));
}

bool DeviceTable::pack_sgd_supported(int gdt, int cdt, int wdt) {
  return (gdt == CS_F32 && cdt == CS_F32 && wdt == CS_F32) || (gdt == CS_BF16 && cdt == CS_BF16 && wdt == CS_F32) ||
         (gdt == CS_F32 && cdt == CS_BF16 && wdt == CS_F32) || (gdt == CS_BF16 && cdt == CS_F32 && wdt == CS_F32) ||
         (gdt == CS_F64 && cdt == CS_F64 && wdt == CS_F64);
}

// kernel launch with the programmatic-stream-serialization attribute (PDL)
// unless CSB_PDL=0
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, cudaStream_t s, Args... args) {
  static const bool pdl = [] {
    const char* e = std::getenv("CSB_PDL");
    return !(e && std::string(e) == "0");
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  CSB_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

void DeviceTable::pack_sgd(const std::vector<PackUpdate>& es, int gdt, int cdt, int wdt, double lr, double rescale,
                           double momentum, cudaStream_t s) {
  if (!pack_sgd_supported(gdt, cdt, wdt)) throw UsageError("pack_sgd: unsupported dtype combination");
  host_.clear();
  vec_.clear();
  groups_ = 0;
  const bool mom = momentum != 0.0;
  double bytes = 0;
  for (const PackUpdate& e : es) {
    if (e.n == 0) continue;
    if (!e.g || !e.bucket || !e.w) throw UsageError("pack_sgd: null pointer in entry");
    if (mom && !e.mom) throw UsageError("pack_sgd: momentum > 0 needs a momentum buffer");
    const uint64_t g = groups_of(e.n);
    Entry en{e.g, e.mom, e.w, e.n, groups_, groups_ + g};
    en.d = e.bucket;
    host_.push_back(en);
    vec_.push_back(aligned16(e.g) && aligned16(e.bucket) && aligned16(e.w) && (!mom || aligned16(e.mom)));
    groups_ += g;
    bytes += static_cast<double>(e.n) *
             (dtype_size(gdt) + (e.bucket != e.g ? dtype_size(cdt) : 0) + 2.0 * dtype_size(wdt) +
              (mom ? 2.0 * (wdt == CS_F64 ? 8 : 4) : 0.0));
  }
  if (host_.empty()) return;
  const double step = lr * rescale;  // model.cpp:21, fp64 on the host
  LaunchScope ls(kKernPackSgd, bytes, s);
  // groups per thread per chunk (CSB_SGD_U = 1 or 2)
  static const int u = [] {
    const char* e = std::getenv("CSB_SGD_U");
    return (e && std::atoi(e) == 2) ? 2 : 1;
  }();
#define CSB_PACK_SGD_U(G, C, W, M, U)                                                         \
  if (gdt == G && cdt == C && wdt == W && mom == M && u == U) {                               \
    grid_ = wave_grid(pack_sgd_tab_kernel<G, C, W, M, U>, groups_, U);                        \
    sync(static_cast<uint64_t>(kThreads) * U, s);                                             \
    const char* base = static_cast<const char*>(dev_);                                        \
    launch_pdl(pack_sgd_tab_kernel<G, C, W, M, U>, grid_, s, reinterpret_cast<const Entry*>(base),  \
               reinterpret_cast<const uint32_t*>(base + host_.size() * sizeof(Entry)),         \
               reinterpret_cast<const uint8_t*>(base + host_.size() * sizeof(Entry) + first_.size() * 4), \
               groups_, step, momentum);                                                       \
    check_launch("pack_sgd_tab_kernel");                                                      \
    ls.done();                                                                                \
    return;                                                                                   \
  }
#define CSB_PACK_SGD(G, C, W, M) CSB_PACK_SGD_U(G, C, W, M, 1) CSB_PACK_SGD_U(G, C, W, M, 2)
  CSB_PACK_SGD(CS_F32, CS_F32, CS_F32, false)
  CSB_PACK_SGD(CS_F32, CS_F32, CS_F32, true)
  CSB_PACK_SGD(CS_BF16, CS_BF16, CS_F32, false)
  CSB_PACK_SGD(CS_BF16, CS_BF16, CS_F32, true)
  CSB_PACK_SGD(CS_F32, CS_BF16, CS_F32, false)
  CSB_PACK_SGD(CS_F32, CS_BF16, CS_F32, true)
  CSB_PACK_SGD(CS_BF16, CS_F32, CS_F32, false)
  CSB_PACK_SGD(CS_BF16, CS_F32, CS_F32, true)
  CSB_PACK_SGD(CS_F64, CS_F64, CS_F64, false)
  CSB_PACK_SGD(CS_F64, CS_F64, CS_F64, true)
#undef CSB_PACK_SGD
#undef CSB_PACK_SGD_U
}

const DeviceTable::Entry* DeviceTable::resident(const std::vector<Entry>& es, cudaStream_t s) {
  host_ = es;
  vec_.assign(es.size(), 0);
  groups_ = 0;
  grid_ = 0;
  first_.clear();
  if (es.empty()) return nullptr;
  sync(0, s);
  return static_cast<const Entry*>(dev_);
}

size_t p2p_flag_bytes() { return sizeof(uint32_t) * 3 * CS_MAX_RANKS * kP2PMaxCtas; }

uint64_t p2p_shard_elems(uint64_t count, int nranks) {
  return (count / kVec + nranks - 1) / nranks * kVec;
}

// The grid is a pure function of (groups, nranks): identical on every rank,
// as the per-CTA pairing requires; one 512-thread CTA per SM so the
// cooperative launch fits beside the other lanes' kernels.  Colocated ranks
// (every rank's grid on one device, local peer transport) share the SMs:
// each grid gets at most 1/nranks of the device's resident 512-thread CTAs,
// so all nranks grids are resident at once and the pair barriers can meet.
int p2p_grid(uint64_t groups, int nranks, bool colocated, int concurrent) {
  static const uint64_t cap = [] {
    const char* e = std::getenv("CSB_P2P_CTAS");  // identical on every rank (same environment)
    return static_cast<uint64_t>(e ? std::max(1, std::atoi(e)) : 148);
  }();
  uint64_t limit = std::min<uint64_t>(cap, kP2PMaxCtas);
  if (colocated || concurrent > 1) {
    const uint64_t resident = static_cast<uint64_t>(sm_count_for_current_device()) * 2;  // __launch_bounds__(512, 2)
    const uint64_t share = static_cast<uint64_t>(colocated ? nranks : 1) * static_cast<uint64_t>(std::max(1, concurrent));
    limit = std::min<uint64_t>(limit, std::max<uint64_t>(1, resident / share));
  }
  const uint64_t per_rank = groups / static_cast<uint64_t>(nranks);
  const uint64_t want = std::max<uint64_t>(1, per_rank / (2 * kP2PLinkThreads));
  return static_cast<int>(std::min<uint64_t>(want, limit));
}

uint64_t p2p_timeout_ns() {
  static const uint64_t v = [] {
    const char* e = std::getenv("CSB_P2P_TIMEOUT_MS");
    const long long ms = e ? std::atoll(e) : 30000;
    return static_cast<uint64_t>(std::max<long long>(1, ms)) * 1000000ull;
  }();
  return v;
}

void p2p_allreduce(const P2PArgs& a, cudaStream_t s) {
  if (a.nranks < 2 || a.nranks > CS_MAX_RANKS) throw UsageError("p2p_allreduce: 2 <= nranks <= 16");
  if (a.count % kVec) throw UsageError("p2p_allreduce: bucket count must be a multiple of 8");
  P2PParams p{};
  for (int r = 0; r < a.nranks; ++r) {
    p.bufs[r] = a.bufs[r];
    p.flags[r] = a.flags[r];
    if (!a.mc && !aligned16(a.bufs[r])) throw UsageError("p2p_allreduce: bucket not 16-byte aligned");
  }
  p.mc = a.mc;
  if (a.mc && !aligned16(a.mc)) throw UsageError("p2p_allreduce: multicast bucket not 16-byte aligned");
  p.tab = a.tab;
  p.n_entries = a.n_entries;
  p.groups = a.count / kVec;
  p.step = a.lr * a.rescale;  // model.cpp:21
  p.mu = a.momentum;
  p.nranks = a.nranks;
  p.rank = a.rank;
  p.epoch = a.epoch;
  p.shard_only = (a.shard_only && a.update && !a.mc) ? 1 : 0;
  p.pack = (a.pack && a.update && a.tab && a.n_entries > 0 && !a.mc) ? 1 : 0;
  const bool zero = a.zero && a.update && !a.mc;
  if (a.zero && !zero) throw UsageError("p2p_allreduce: ZeRO-1 needs the fused update over peer memory");
  for (int r = 0; zero && r < a.nranks; ++r) {
    p.wm[r] = a.wm[r];
    if (!aligned16(a.wm[r])) throw UsageError("p2p_allreduce: master shard not 16-byte aligned");
  }
  p.mom_b = a.mom_b;
  p.direct = (a.direct && a.tab && a.n_entries > 0 && !a.mc) ? 1 : 0;
  if (a.direct && !p.direct) throw UsageError("p2p_allreduce: direct gradient reads need the key table over peer memory");
  for (int r = 0; p.direct && r < a.nranks; ++r) {
    p.gbase[r] = a.gbase[r];
    if (!aligned16(a.gbase[r])) throw UsageError("p2p_allreduce: gradient region not 16-byte aligned");
  }
  p.abort_word = a.abort_word;
  p.stamps = a.stamps;

  static const uint64_t piece = [] {
    const char* e = std::getenv("CSB_P2P_PIECE");  // identical on every rank (same environment)
    return static_cast<uint64_t>(e ? std::max(0, std::atoi(e)) : 4096);
  }();
  p.piece = piece;
  static const uint64_t kmin = [] {
    const char* e = std::getenv("CSB_P2P_KMIN");  // identical on every rank (same environment)
    return static_cast<uint64_t>(e ? std::max(1, std::atoi(e)) : 1);
  }();
  p.kmin = kmin;
  p.timeout_ns = a.timeout_ns ? a.timeout_ns : p2p_timeout_ns();
  const int grid = p2p_grid(p.groups, a.nranks, a.colocated, a.concurrent);
  const bool upd = a.update && a.tab && a.n_entries > 0;
  const bool mom = a.momentum != 0.0;
  const double elems = static_cast<double>(a.count);
  const double bytes = elems * dtype_size(a.cdt) * 2.0 / a.nranks * a.nranks +
                       (upd ? elems * (dtype_size(a.cdt) + 2.0 * dtype_size(a.wdt) + (mom ? 8.0 : 0.0)) : 0.0);
  LaunchScope ls(kKernSum, bytes, s);
  void* args[] = {&p};
  const void* fn = nullptr;
#define CSB_P2P_PICK(C, W, U, MO)                                                                  \
  if (a.cdt == C && (!U || a.wdt == W) && upd == U && (!U || mom == MO)) {                         \
    switch (a.nranks) {                                                                            \
      case 2: fn = reinterpret_cast<const void*>(p2p_allreduce_kernel<C, W, U, MO, 2>); break;     \
      case 4: fn = reinterpret_cast<const void*>(p2p_allreduce_kernel<C, W, U, MO, 4>); break;     \
      case 8: fn = reinterpret_cast<const void*>(p2p_allreduce_kernel<C, W, U, MO, 8>); break;     \
      default: fn = reinterpret_cast<const void*>(p2p_allreduce_kernel<C, W, U, MO, 0>); break;    \
    }                                                                                              \
  }
  CSB_P2P_PICK(CS_F32, CS_F32, false, false)
  CSB_P2P_PICK(CS_BF16, CS_F32, false, false)
  CSB_P2P_PICK(CS_F64, CS_F64, false, false)
  CSB_P2P_PICK(CS_F32, CS_F32, true, false)
  CSB_P2P_PICK(CS_F32, CS_F32, true, true)
  CSB_P2P_PICK(CS_BF16, CS_F32, true, false)
  CSB_P2P_PICK(CS_BF16, CS_F32, true, true)
  CSB_P2P_PICK(CS_F64, CS_F64, true, false)
  CSB_P2P_PICK(CS_F64, CS_F64, true, true)
#undef CSB_P2P_PICK
  if (a.mc) {  // in-switch reduction through the multicast VA
    fn = nullptr;
#define CSB_NVLS_PICK(C, W, U, MO)                                                                       \
  if (a.cdt == C && (!U || a.wdt == W) && upd == U && (!U || mom == MO))                                 \
    fn = reinterpret_cast<const void*>(p2p_allreduce_kernel<C, W, U, MO, 0, true>);
    CSB_NVLS_PICK(CS_F32, CS_F32, false, false)
    CSB_NVLS_PICK(CS_BF16, CS_F32, false, false)
    CSB_NVLS_PICK(CS_F32, CS_F32, true, false)
    CSB_NVLS_PICK(CS_F32, CS_F32, true, true)
    CSB_NVLS_PICK(CS_BF16, CS_F32, true, false)
    CSB_NVLS_PICK(CS_BF16, CS_F32, true, true)
#undef CSB_NVLS_PICK
  }
  if (zero) {
    fn = nullptr;
#define CSB_ZERO_PICK(C, W, MO)                                                                  \
  if (a.cdt == C && a.wdt == W && mom == MO) {                                                   \
    switch (a.nranks) {                                                                          \
      case 2: fn = reinterpret_cast<const void*>(p2p_zero_kernel<C, W, MO, 2>); break;           \
      case 4: fn = reinterpret_cast<const void*>(p2p_zero_kernel<C, W, MO, 4>); break;           \
      case 8: fn = reinterpret_cast<const void*>(p2p_zero_kernel<C, W, MO, 8>); break;           \
      default: fn = reinterpret_cast<const void*>(p2p_zero_kernel<C, W, MO, 0>); break;          \
    }                                                                                            \
  }
    CSB_ZERO_PICK(CS_F32, CS_F32, false)
    CSB_ZERO_PICK(CS_F32, CS_F32, true)
    CSB_ZERO_PICK(CS_BF16, CS_F32, false)
    CSB_ZERO_PICK(CS_BF16, CS_F32, true)
    CSB_ZERO_PICK(CS_F64, CS_F64, false)
    CSB_ZERO_PICK(CS_F64, CS_F64, true)
#undef CSB_ZERO_PICK
  }
  if (!fn) throw UsageError("p2p_allreduce: unsupported dtype combination");
  // cooperative launch: the driver guarantees every CTA is resident (the
  // pair barriers need it); CSB_P2P_COOP=0 measured no faster
  static const bool coop = [] {
    const char* e = std::getenv("CSB_P2P_COOP");
    return !(e && std::string(e) == "0");
  }();
  static const int fence = [] {
    const char* e = std::getenv("CSB_P2P_FENCE");
    return (e && std::string(e) == "1") ? 1 : 0;
  }();
  p.sys_fence = fence;
  // colocated grids share one device: a cooperative launch would claim the
  // whole device per grid, so those launch plainly (p2p_grid keeps them co-resident)
  if (coop && !a.colocated && a.concurrent <= 1)
    CSB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kP2PThreads), args, 0, s));
  else CSB_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(kP2PThreads), args, 0, s));
  ls.done();
}

uint64_t launch_count() { return g_launches.load(); }

void profile_enable(bool on) { g_prof_on.store(on); }

KernelStats profile_collect(int kind) {
  if (kind < 0 || kind >= kKernKinds) throw UsageError("profile: unknown kernel kind");
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lock(g_prof_mu);
    recs.swap(g_prof_pending);
  }
  int prev = 0;
  CSB_CUDA(cudaGetDevice(&prev));
  for (const ProfRec& r : recs) {
    CSB_CUDA(cudaSetDevice(r.dev));
    CSB_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    std::lock_guard<std::mutex> lock(g_prof_mu);
    g_prof_stats[r.kind].launches++;
    g_prof_stats[r.kind].total_ms += ms;
    g_prof_stats[r.kind].bytes += r.bytes;
    g_prof_free.push_back({r.dev, r.a});
    g_prof_free.push_back({r.dev, r.b});
  }
  CSB_CUDA(cudaSetDevice(prev));
  std::lock_guard<std::mutex> lock(g_prof_mu);
  return g_prof_stats[kind];
}

void profile_reset() {
  profile_collect(0);
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& s : g_prof_stats) s = KernelStats{};
}

}  // namespace csb
