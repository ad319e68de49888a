// Pipelined (Ghysels-Vanroose) Jacobi-PCG streaming team solver (stream.cuh),
// own-row vectors loaded per row (teams with several tiles per CTA); compiled in its own translation unit.  LRB_PIPE_DEFER=1 at team
// creation selects the variant that reads each reduction one phase late.
#include <cstdlib>

#include "launch.h"
#include "stream.cuh"

namespace lrb {

const void* pipecg_stream_kernel(bool inl) {
  const char* e = std::getenv("LRB_PIPE_DEFER");
  const bool defer = e && e[0] == '1';
  if (defer)
    return inl ? (const void*)team_pipecg_stream_kernel<true, true, false>
               : (const void*)team_pipecg_stream_kernel<false, true, false>;
  return inl ? (const void*)team_pipecg_stream_kernel<true, false, false>
             : (const void*)team_pipecg_stream_kernel<false, false, false>;
}

}  // namespace lrb
