// BiCGStab team solvers (classic: kernels.cuh, streaming: stream.cuh),
// compiled in their own translation unit.
#include "launch.h"
#include "stream.cuh"

namespace lrb {

const void* bicgstab_classic_kernel(bool inl) {
  return inl ? (const void*)team_bicgstab_kernel<true> : (const void*)team_bicgstab_kernel<false>;
}

const void* bicgstab_stream_kernel(bool inl) {
  return inl ? (const void*)team_bicgstab_stream_kernel<true> : (const void*)team_bicgstab_stream_kernel<false>;
}

}  // namespace lrb
