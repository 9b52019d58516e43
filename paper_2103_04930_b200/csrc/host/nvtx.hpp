// NVTX ranges over the server's cycle phases (receive, queue + forward, reply)
// and the dispatcher's forward, so an nsys / ncu --nvtx timeline of avec-server
// shows where a cycle's time goes next to the kernels. Header-only NVTX 3: a
// no-op until a tool injects itself (one pointer check per range).
#pragma once

#include <nvtx3/nvToolsExt.h>

namespace avec::trace {

class Range {
 public:
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

}  // namespace avec::trace
