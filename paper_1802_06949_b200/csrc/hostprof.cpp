// hostprof.cpp -- see hostprof.hpp.
#include "hostprof.hpp"

#include <cstdlib>
#include <sstream>

namespace csb {
namespace hostprof {

namespace {
const char* kNames[kSections] = {"kv_push", "kv_pull", "engine_enqueue", "dispatch_wait", "dispatch_body",
                                 "dispatch_record", "complete", "ledger", "launch"};
std::atomic<uint64_t> g_ns[kSections];
std::atomic<uint64_t> g_n[kSections];
const bool g_on = [] {
  const char* e = std::getenv("CSB_HOST_PROFILE");
  return e && e[0] == '1';
}();
}  // namespace

bool enabled() { return g_on; }

void add(Section s, uint64_t ns) {
  g_ns[s].fetch_add(ns, std::memory_order_relaxed);
  g_n[s].fetch_add(1, std::memory_order_relaxed);
}

std::string report_json() {
  std::ostringstream os;
  os << "{";
  for (int i = 0; i < kSections; ++i) {
    if (i) os << ",";
    os << "\"" << kNames[i] << "\":{\"calls\":" << g_n[i].load() << ",\"us\":" << g_ns[i].load() / 1000.0
       << "}";
  }
  os << "}";
  return os.str();
}

void reset() {
  for (int i = 0; i < kSections; ++i) {
    g_ns[i] = 0;
    g_n[i] = 0;
  }
}

}  // namespace hostprof
}  // namespace csb
