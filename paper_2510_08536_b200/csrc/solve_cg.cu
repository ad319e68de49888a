// CG / Jacobi-PCG team solvers (classic: kernels.cuh, streaming: stream.cuh),
// compiled in their own translation unit.
#include "launch.h"
#include "stream.cuh"

namespace lrb {

const void* cg_classic_kernel(bool jac, bool inl) {
  if (jac) return inl ? (const void*)team_cg_kernel<true, true> : (const void*)team_cg_kernel<true, false>;
  return inl ? (const void*)team_cg_kernel<false, true> : (const void*)team_cg_kernel<false, false>;
}

const void* cg_stream_kernel(bool jac, bool inl) {
  if (jac)
    return inl ? (const void*)team_cg_stream_kernel<true, true> : (const void*)team_cg_stream_kernel<true, false>;
  return inl ? (const void*)team_cg_stream_kernel<false, true> : (const void*)team_cg_stream_kernel<false, false>;
}

}  // namespace lrb
