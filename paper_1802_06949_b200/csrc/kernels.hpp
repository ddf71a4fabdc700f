// kernels.hpp -- host launchers of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "collsim_b200.h"

namespace csb {

void pack(const cs_copy_entry* entries, int n, int src_dt, int dst_dt, cudaStream_t s);
void sum_buffers(const void* const* in, int m, void* const* out, int nout, uint64_t n, int dt,
                 cudaStream_t s);
void sgd_update(const cs_update_entry* entries, int n, int w_dt, int g_dt, double lr,
                double rescale, double momentum, cudaStream_t s);
void synth_backward(const void* src, void* dst, uint64_t n, int dt, uint64_t spin_ns, int ctas,
                    cudaStream_t s);
void checksum(const void* x, uint64_t n, int dt, double* out, cudaStream_t s);

}  // namespace csb
