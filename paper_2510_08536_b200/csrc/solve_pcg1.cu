// Single-reduction Jacobi-PCG streaming team solver (stream.cuh), compiled in
// its own translation unit.
#include "launch.h"
#include "stream.cuh"

namespace lrb {

const void* pcg1_stream_kernel(bool inl) {
  return inl ? (const void*)team_pcg1_stream_kernel<true> : (const void*)team_pcg1_stream_kernel<false>;
}

}  // namespace lrb
