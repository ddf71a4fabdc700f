// common.hpp -- error taxonomy, CUDA/NCCL checks and dtype helpers shared by
// the host runtime (engine / transport / kvstore) and the kernels.
//
// Error kinds and their stable names follow the reference
// (R/core/include/collsim/error.hpp:10-62); CUDA and NCCL failures are two
// additional kinds that only exist on the device path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "collsim_b200.h"

namespace csb {

class Error : public std::runtime_error {
 public:
  enum class Kind { Config, Usage, Mismatch, DeadlockTimeout, Engine, Cuda, Nccl, Internal };
  Error(Kind kind, const std::string& msg) : std::runtime_error(msg), kind_(kind) {}
  Kind kind() const { return kind_; }
  const char* kind_name() const { return name_of(kind_); }
  static const char* name_of(Kind k) {
    switch (k) {
      case Kind::Config: return "ConfigError";
      case Kind::Usage: return "UsageError";
      case Kind::Mismatch: return "MismatchError";
      case Kind::DeadlockTimeout: return "DeadlockTimeout";
      case Kind::Engine: return "EngineError";
      case Kind::Cuda: return "CudaError";
      case Kind::Nccl: return "NcclError";
      case Kind::Internal: return "InternalError";
    }
    return "Error";
  }
  int status() const {
    switch (kind_) {
      case Kind::Config: return CS_ERR_CONFIG;
      case Kind::Usage: return CS_ERR_USAGE;
      case Kind::Mismatch: return CS_ERR_MISMATCH;
      case Kind::DeadlockTimeout: return CS_ERR_DEADLOCK;
      case Kind::Engine: return CS_ERR_ENGINE;
      case Kind::Cuda: return CS_ERR_CUDA;
      case Kind::Nccl: return CS_ERR_NCCL;
      case Kind::Internal: return CS_ERR_INTERNAL;
    }
    return CS_ERR_INTERNAL;
  }

 private:
  Kind kind_;
};

struct ConfigError : Error {
  explicit ConfigError(const std::string& m) : Error(Kind::Config, m) {}
};
struct UsageError : Error {
  explicit UsageError(const std::string& m) : Error(Kind::Usage, m) {}
};
struct MismatchError : Error {
  explicit MismatchError(const std::string& m) : Error(Kind::Mismatch, m) {}
};
struct DeadlockTimeout : Error {
  explicit DeadlockTimeout(const std::string& m) : Error(Kind::DeadlockTimeout, m) {}
};
struct EngineError : Error {
  explicit EngineError(const std::string& m) : Error(Kind::Engine, m) {}
};
struct CudaError : Error {
  explicit CudaError(const std::string& m) : Error(Kind::Cuda, m) {}
};
struct NcclError : Error {
  explicit NcclError(const std::string& m) : Error(Kind::Nccl, m) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                  std::to_string(line) + ")");
}

#define CSB_CUDA(call)                                                   \
  do {                                                                   \
    cudaError_t csb_e_ = (call);                                         \
    if (csb_e_ != cudaSuccess) ::csb::throw_cuda(csb_e_, #call, __FILE__, __LINE__); \
  } while (0)

inline size_t dtype_size(int dt) {
  switch (dt) {
    case CS_F64: return 8;
    case CS_F32: return 4;
    case CS_BF16: return 2;
  }
  throw UsageError("unknown dtype " + std::to_string(dt));
}

inline const char* dtype_name(int dt) {
  switch (dt) {
    case CS_F64: return "f64";
    case CS_F32: return "f32";
    case CS_BF16: return "bf16";
  }
  return "?";
}

}  // namespace csb
