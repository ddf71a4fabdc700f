// watch.hpp -- process-wide failure detection for device-side collectives.
//
// The reference's Transport turns a hang into DeadlockTimeout with a report
// and latches the failure (R/core/src/collective.cpp:92-105, 249-264).  On
// the GPU a hang is a kernel that never finishes (an NCCL kernel whose peer
// died, a peer-memory kernel whose pair barrier never completes), and it is
// the Engine's device waits (Engine::sync_event / sync_lanes) that notice.
// Transports register two callbacks here:
//   poll   -- a non-empty string reports an asynchronous failure
//             (ncclCommGetAsyncError, a peer kernel's device timeout);
//   abort  -- release every device wait: set the peer kernels' abort word,
//             ncclCommAbort, latch the ledger.
// The Engine polls while it waits on device work and, on an asynchronous
// failure or its own watchdog, aborts every registered transport before it
// throws -- the kernels return instead of trapping, so the GPU stays usable.
#pragma once

#include <functional>
#include <string>

namespace csb::watch {

using Poll = std::function<std::string()>;
using Abort = std::function<void(const std::string&)>;

int add(Poll poll, Abort abort);
void remove(int id);
// First failure any registered transport reports ("" when healthy).
std::string poll();
// Aborts every registered transport (idempotent per transport).
void abort_all(const std::string& why);

}  // namespace csb::watch
