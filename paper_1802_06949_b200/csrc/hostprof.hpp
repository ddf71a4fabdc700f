// hostprof.hpp -- opt-in host-side section timers (CSB_HOST_PROFILE=1).
// Used to find where dispatch time goes; off by default (one relaxed load).
#pragma once

#include <atomic>
#include <chrono>
#include <cstdint>
#include <string>

namespace csb {
namespace hostprof {

enum Section {
  kKvPush = 0,
  kKvPull,
  kEnqueue,
  kDispatchWait,
  kDispatchBody,
  kDispatchRecord,
  kComplete,
  kLedger,
  kLaunch,
  kSections
};

bool enabled();
void add(Section s, uint64_t ns);
std::string report_json();
void reset();

struct Scope {
  Section s;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit Scope(Section sec) : s(sec), on(enabled()) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  ~Scope() {
    if (on)
      add(s, static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                       std::chrono::steady_clock::now() - t0)
                                       .count()));
  }
};

}  // namespace hostprof
}  // namespace csb
