// Kernel entry points of the separately compiled CUDA translation units
// (scatter.cu, solve_cg.cu, solve_bicgstab.cu, solve_pcg1.cu, solve_pipecg*.cu), for the host
// side in device.cu.  Internal; not part of the public interface.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lrb_internal.h"

namespace lrb {

// Scatter of rows [r0, r1) of part P on stream st (scatter.cu).
cudaError_t scatter_launch(const PartDev& P, int64_t r0, int64_t r1, cudaStream_t st);
// Fused GPU-side perturb_coefficients + scatter from a device copy of the base buffer.
cudaError_t perturb_launch(const PartDev& P, const double* base, double scale, cudaStream_t st);
// dinv from the diagonal values (after lrb_part_write_values).
cudaError_t dinv_refresh_launch(const PartDev& P, cudaStream_t st);

// Host stubs of the persistent team solvers (kernel function pointers for
// cudaLaunch[Cooperative]Kernel / occupancy queries).
const void* cg_classic_kernel(bool jac, bool inl);       // solve_cg.cu
const void* cg_stream_kernel(bool jac, bool inl);        // solve_cg.cu
const void* bicgstab_classic_kernel(bool inl);           // solve_bicgstab.cu
const void* bicgstab_stream_kernel(bool inl);            // solve_bicgstab.cu
const void* pcg1_stream_kernel(bool inl);                // solve_pcg1.cu
const void* pipecg_stream_kernel(bool inl);              // solve_pipecg.cu (own-row vectors loaded)
const void* pipecg_t_stream_kernel(bool inl);            // solve_pipecg_t.cu (own-row vectors staged)

}  // namespace lrb
