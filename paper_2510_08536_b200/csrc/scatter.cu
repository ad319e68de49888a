// Update path kernel: gather-permute of the receive buffer into the fused
// SELL values (apply_scatter, update.py:105-112).
//
//   val[e] = recv[src[e]]      for every SELL slot e of rows [r0, r1)
//   dinv[i] = 1 / val[diag]    (Jacobi; correctly rounded like numpy)
//
// Pure copies, so the result is bit-exact with the reference.  20 algorithmic
// bytes per entry (4 B src + 8 B recv + 8 B val), HBM-bound.
//
// Thread per row, a warp per SELL slice: the src loads (128 B) and val stores
// (256 B) of a slot are coalesced across the warp; the recv gathers follow the
// pack order [diag | upper | lower | ifaces] (update.py:40-45), so each warp's
// gathers touch a handful of monotone streams that L2 reuses.
//
// One launch per source segment (its rows are one contiguous range,
// repart.py:253-270) on the segment's stream right after its H2D copy, or one
// launch over the part (apply_scatter).  Measured at C3 (200^3, 8M rows, one
// launch): 0.19 ms = 5.87 TB/s algorithmic (0.90 of the measured copy peak);
// persistent grid-stride variants (32/40/64 registers, streaming cache hints,
// two rows per thread) were all slower, 4.6-5.0 TB/s
// (profiles/r2_experiments.md).
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "lrb_internal.h"

namespace lrb {

#ifndef LRB_SCATTER_CHUNK   // slots per pass: 8 covers a 7-point stencil row in one pass
#define LRB_SCATTER_CHUNK 8
#endif
constexpr int kScChunk = LRB_SCATTER_CHUNK;
#ifndef LRB_SCATTER_TPB
#define LRB_SCATTER_TPB 128   // 128 vs 256 vs 512 threads: 0.187 vs 0.189 vs 0.193 ms at C3
#endif
constexpr int kScTPB = LRB_SCATTER_TPB;

__device__ __forceinline__ void scatter_row(const PartDev& P, int64_t i) {
  const RowRef rr = row_ref(P, i);
  const int dk = __ldg(P.dpos + i);
  for (int k0 = 0; k0 < rr.w; k0 += kScChunk) {
    int b[kScChunk];
    double v[kScChunk];
#pragma unroll
    for (int u = 0; u < kScChunk; ++u)
      b[u] = (k0 + u < rr.w) ? __ldg(P.src + rr.base + int64_t(k0 + u) * kSlice) : -1;
#pragma unroll
    for (int u = 0; u < kScChunk; ++u) v[u] = b[u] >= 0 ? __ldg(P.recv + b[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kScChunk; ++u) {
      if (b[u] < 0) continue;
      P.val[rr.base + int64_t(k0 + u) * kSlice] = v[u];
      if (k0 + u == dk) P.dinv[i] = 1.0 / v[u];
    }
  }
}

__global__ void __launch_bounds__(kScTPB) scatter_rows_kernel(PartDev P, int64_t r0, int64_t r1) {
  const int64_t i = (r0 & ~int64_t(31)) + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < r0 || i >= r1) return;
  scatter_row(P, i);
}

// GPU-side producer of the reference's pseudo-timestep (perturb_coefficients,
// assembly.py:225-243: diag scaled by (1 + step/100), everything else the
// pristine base) fused with the scatter: val[e] = base[src[e]], times `scale`
// on the row's diagonal slot (correctly rounded, like numpy's m.diag * f),
// dinv refreshed.  No host coefficients move (the paper's
// "refactoring approach").  20 B per entry, like the scatter.
__global__ void __launch_bounds__(kScTPB) perturb_rows_kernel(PartDev P, const double* __restrict__ base,
                                                               double scale) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const RowRef rr = row_ref(P, i);
  const int dk = __ldg(P.dpos + i);
  for (int k0 = 0; k0 < rr.w; k0 += kScChunk) {
    int b[kScChunk];
    double v[kScChunk];
#pragma unroll
    for (int u = 0; u < kScChunk; ++u)
      b[u] = (k0 + u < rr.w) ? __ldg(P.src + rr.base + int64_t(k0 + u) * kSlice) : -1;
#pragma unroll
    for (int u = 0; u < kScChunk; ++u) v[u] = b[u] >= 0 ? __ldg(base + b[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < kScChunk; ++u) {
      if (b[u] < 0) continue;
      double x = v[u];
      if (k0 + u == dk) {
        x = __dmul_rn(x, scale);
        P.dinv[i] = 1.0 / x;
      }
      P.val[rr.base + int64_t(k0 + u) * kSlice] = x;
    }
  }
}

cudaError_t perturb_launch(const PartDev& P, const double* base, double scale, cudaStream_t st) {
  if (P.n <= 0) return cudaSuccess;
  perturb_rows_kernel<<<unsigned((P.n + kScTPB - 1) / kScTPB), kScTPB, 0, st>>>(P, base, scale);
  return cudaGetLastError();
}

// Jacobi refresh after values were written directly (lrb_part_write_values):
// dinv[i] = 1 / val[diagonal slot of row i].
__global__ void __launch_bounds__(kScTPB) dinv_refresh_kernel(PartDev P) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const int dk = __ldg(P.dpos + i);
  if (dk < 0) return;
  const RowRef rr = row_ref(P, i);
  P.dinv[i] = 1.0 / P.val[rr.base + int64_t(dk) * kSlice];
}

cudaError_t dinv_refresh_launch(const PartDev& P, cudaStream_t st) {
  if (P.n <= 0) return cudaSuccess;
  dinv_refresh_kernel<<<unsigned((P.n + kScTPB - 1) / kScTPB), kScTPB, 0, st>>>(P);
  return cudaGetLastError();
}

// Launch the scatter of rows [r0, r1) of part P on stream st.
cudaError_t scatter_launch(const PartDev& P, int64_t r0, int64_t r1, cudaStream_t st) {
  if (r1 <= r0) return cudaSuccess;
  const int64_t first = r0 & ~int64_t(31);
  const int64_t blocks = (r1 - first + kScTPB - 1) / kScTPB;
  scatter_rows_kernel<<<unsigned(blocks), kScTPB, 0, st>>>(P, r0, r1);
  return cudaGetLastError();
}

}  // namespace lrb
