// Pipelined (Ghysels-Vanroose) Jacobi-PCG streaming team solver (stream.cuh),
// compiled in its own translation unit.  LRB_PIPE_DEFER=1 at team creation
// selects the variant that reads each reduction one phase late (flat teams).
#include <cstdlib>

#include "launch.h"
#include "stream.cuh"

namespace lrb {

const void* pipecg_stream_kernel(bool inl) {
  const char* e = std::getenv("LRB_PIPE_DEFER");
  const bool defer = e && e[0] == '1';
  if (defer)
    return inl ? (const void*)team_pipecg_stream_kernel<true, true>
               : (const void*)team_pipecg_stream_kernel<false, true>;
  return inl ? (const void*)team_pipecg_stream_kernel<true, false>
             : (const void*)team_pipecg_stream_kernel<false, false>;
}

}  // namespace lrb
