// watch.cpp -- see watch.hpp.
#include "watch.hpp"

#include <map>
#include <mutex>

namespace csb::watch {

namespace {
struct Entry {
  Poll poll;
  Abort abort;
};
std::mutex& mu() {
  static std::mutex m;
  return m;
}
std::map<int, Entry>& reg() {
  static std::map<int, Entry> r;
  return r;
}
int next_id = 1;
}  // namespace

int add(Poll p, Abort a) {
  std::lock_guard<std::mutex> lock(mu());
  const int id = next_id++;
  reg()[id] = Entry{std::move(p), std::move(a)};
  return id;
}

void remove(int id) {
  std::lock_guard<std::mutex> lock(mu());
  reg().erase(id);
}

// Callbacks run under the registry lock, so a transport cannot be destroyed
// (remove() takes the same lock) while one of its callbacks runs.
std::string poll() {
  std::lock_guard<std::mutex> lock(mu());
  for (auto& [id, e] : reg()) {
    std::string m = e.poll ? e.poll() : std::string();
    if (!m.empty()) return m;
  }
  return {};
}

void abort_all(const std::string& why) {
  std::lock_guard<std::mutex> lock(mu());
  for (auto& [id, e] : reg())
    if (e.abort) e.abort(why);
}

}  // namespace csb::watch
