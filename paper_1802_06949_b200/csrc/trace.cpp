// trace.cpp -- TraceSink (reference: R/core/src/trace.cpp:11-47).
#include "trace.hpp"

#include <fstream>
#include <stdexcept>

namespace csb {

TraceSink::TraceSink() : start_(std::chrono::steady_clock::now()) {}

void TraceSink::emit(TraceEvent ev) {
  std::lock_guard<std::mutex> lock(mu_);
  // stamped under the lock: per-sink emission order == t_us order
  ev.t_us = std::chrono::duration_cast<std::chrono::microseconds>(
                std::chrono::steady_clock::now() - start_)
                .count();
  events_.push_back(std::move(ev));
}

std::vector<TraceEvent> TraceSink::snapshot() const {
  std::lock_guard<std::mutex> lock(mu_);
  return events_;
}

size_t TraceSink::count() const {
  std::lock_guard<std::mutex> lock(mu_);
  return events_.size();
}

// Keys in lexicographic order, compact separators: byte-identical to
// nlohmann::json::dump() of the reference's object (std::map-ordered).
std::string trace_event_json(const TraceEvent& ev) {
  std::string s = "{";
  bool first = true;
  auto field = [&](const char* k, const std::string& v, bool quote) {
    if (!first) s += ",";
    first = false;
    s += "\"";
    s += k;
    s += "\":";
    if (quote) s += "\"";
    s += v;
    if (quote) s += "\"";
  };
  if (ev.bucket >= 0) field("bucket", std::to_string(ev.bucket), false);
  if (ev.comm >= 0) field("comm", std::to_string(ev.comm), false);
  field("event", ev.event, true);
  if (ev.key >= 0) field("key", std::to_string(ev.key), false);
  if (!ev.kind.empty()) field("kind", ev.kind, true);
  if (ev.op >= 0) field("op", std::to_string(ev.op), false);
  field("rank", std::to_string(ev.rank), false);
  if (ev.seq >= 0) field("seq", std::to_string(ev.seq), false);
  field("t_us", std::to_string(ev.t_us), false);
  s += "}";
  return s;
}

void TraceSink::write_jsonl(const std::string& path) const {
  std::vector<TraceEvent> events = snapshot();
  std::ofstream out(path);
  if (!out) throw std::runtime_error("trace: cannot open " + path);
  for (const TraceEvent& ev : events) out << trace_event_json(ev) << '\n';
}

}  // namespace csb
