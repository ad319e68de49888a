// sm_100a kernels of the hot path: segment scatter (update), distributed SpMV
// and the persistent team Krylov solvers (CG / Jacobi-PCG / BiCGStab).
//
// Rounding contract (parity with the reference, solver.py:80-147):
//  * every product and sum is a separately rounded __dmul_rn / __dadd_rn /
//    __dsub_rn (no FMA contraction), in the reference's elementwise order;
//  * a row's SpMV accumulates its local entries in stored order, then its
//    non-local entries, starting from 0.0 — bit-identical to np.add.at;
//  * dot products: per-tile fixed-order tree, tiles summed in fixed order per
//    part, parts summed in ascending GPU rank ((p0 + p1) + p2)... exactly the
//    reference's allreduce order (transport.py:450-458).  Only the in-part
//    summation order differs from OpenBLAS ddot (tolerance parity).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ldurepart_b200.h"
#include "lrb_internal.h"

namespace lrb {

__device__ __forceinline__ double vload(const double* p) { return *(const volatile double*)p; }
__device__ __forceinline__ unsigned vload(const unsigned* p) { return *(const volatile unsigned*)p; }

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// SELL-32 row access
// ---------------------------------------------------------------------------
struct RowRef {
  int64_t base;
  int w;
};
__device__ __forceinline__ RowRef row_ref(const PartDev& P, int64_t i) {
  const int64_t s = i >> 5;
  const int64_t b = __ldg(P.slice_ptr + s);
  const int64_t e = __ldg(P.slice_ptr + s + 1);
  return RowRef{b + (i & 31), int((e - b) >> 5)};
}

// Halo push (PartDev::hm): the owner of row i stores v, its new value of
// mirrored vector vid, into the halo mirror of every part that reads row i
// (peer memory for parts on other GPUs).  Interior rows return after two
// compares.  Ordering: the team barrier's system-scope fence (team_sync)
// publishes the pushes together with the phase's other writes.
__device__ __forceinline__ void hpush(const PartDev& P, const PartDev* __restrict__ parts, int vid,
                                      int64_t i, double v) {
  if (i >= P.sq_lo && i < P.sq_hi) return;
  for (int k = 0; k < P.n_snd; ++k) {
    const int64_t* s = P.snd + 4 * k;
    const int64_t lo = __ldg(s), hi = __ldg(s + 1);
    if (i >= lo && i < hi) {
      const PartDev& Q = parts[__ldg(s + 2)];
      Q.hm[int64_t(vid) * Q.n_halo + __ldg(s + 3) + (i - lo)] = v;
    }
  }
}

// y_i = sum_k a_ik * f(col_k), reference order, no FMA.  f(Q, j) returns the
// vector value at row j of part Q (local part or halo owner).
//
// Entries are processed in chunks of kChunk: all column loads of a chunk are
// issued, then all value loads and vector gathers, then the products are
// accumulated in entry order.  The slice width is warp-uniform, so the chunk
// loop never diverges; padding (col -1) only predicates lanes off.  This keeps
// ~3*kChunk independent loads in flight per thread instead of a dependent
// col -> x -> add chain per entry.
#ifndef LRB_CHUNK
#define LRB_CHUNK 4
#endif
constexpr int kChunk = LRB_CHUNK;

// Minimum resident blocks per SM requested from ptxas for the persistent
// solvers (register cap 65536 / (256 * LRB_MINB)).  Measured on B200 at C3
// (tools/variants.sh): occupancy beats spill-free code — MINB 6 / chunk 4
// (40 regs, 75% occupancy) runs the PCG solve 2x faster than MINB 2 (111 regs).
#ifndef LRB_MINB
#define LRB_MINB 6
#endif
#ifndef LRB_SPLITB
#define LRB_SPLITB 0
#endif
// Tiles of a phase: grid-strided (default: the whole grid sweeps the rows as
// one wavefront, so a row's +-plane neighbours are fetched into L2 by another
// block at about the same time) or contiguous per block (measured 11% slower
// at C3).  Partials are per tile either way: results do not depend on the
// choice or on the grid size.
#ifndef LRB_CONTIG
#define LRB_CONTIG 0
#endif

template <class F>
__device__ __forceinline__ double row_spmv(const PartDev& P, const PartDev* __restrict__ parts,
                                           int64_t i, F&& f) {
  const RowRef rr = row_ref(P, i);
  const int n = int(P.n);
  const int pid = __ldg(P.slice_pat + (i >> 5));   // warp-uniform
  const int32_t* poff = P.pat_off + pid * kPatW;
  double acc = 0.0;
  for (int k0 = 0; k0 < rr.w; k0 += kChunk) {
    int c[kChunk];
    double a[kChunk], xv[kChunk];
    if (pid >= 0) {
      const unsigned msk = __ldg(P.rmask + i);
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        c[u] = (k0 + u < rr.w && ((msk >> (k0 + u)) & 1u)) ? int(i) + __ldg(poff + k0 + u) : -1;
    } else {
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        c[u] = (k0 + u < rr.w) ? __ldg(P.col + rr.base + int64_t(k0 + u) * kSlice) : -1;
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      a[u] = 0.0;
      xv[u] = 0.0;
      if (c[u] >= 0) {
        a[u] = __ldg(P.val + rr.base + int64_t(k0 + u) * kSlice);
        if (c[u] < n) {
          xv[u] = f(P, int64_t(c[u]));
        } else {
          const int h = c[u] - n;
          xv[u] = f(parts[__ldg(P.hpart + h)], int64_t(__ldg(P.hidx + h)));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
      if (c[u] >= 0) acc = __dadd_rn(acc, __dmul_rn(a[u], xv[u]));
  }
  return acc;
}

// Same, with the local-column operand from floc(c) (staged in shared memory
// for pattern tiles) and halo columns from fhalo(owner part, row).
template <class FL, class FH>
__device__ __forceinline__ double row_spmv2(const PartDev& P, const PartDev* __restrict__ parts,
                                            int64_t i, FL&& floc, FH&& fhalo) {
  const RowRef rr = row_ref(P, i);
  const int n = int(P.n);
  const int pid = __ldg(P.slice_pat + (i >> 5));   // warp-uniform
  const int32_t* poff = P.pat_off + pid * kPatW;
  double acc = 0.0;
  for (int k0 = 0; k0 < rr.w; k0 += kChunk) {
    int c[kChunk];
    double a[kChunk], xv[kChunk];
    if (pid >= 0) {
      const unsigned msk = __ldg(P.rmask + i);
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        c[u] = (k0 + u < rr.w && ((msk >> (k0 + u)) & 1u)) ? int(i) + __ldg(poff + k0 + u) : -1;
    } else {
#pragma unroll
      for (int u = 0; u < kChunk; ++u)
        c[u] = (k0 + u < rr.w) ? __ldg(P.col + rr.base + int64_t(k0 + u) * kSlice) : -1;
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u) {
      a[u] = 0.0;
      xv[u] = 0.0;
      if (c[u] >= 0) {
        a[u] = __ldg(P.val + rr.base + int64_t(k0 + u) * kSlice);
        if (c[u] < n) {
          xv[u] = floc(int64_t(c[u]));
        } else {
          const int h = c[u] - n;
          xv[u] = fhalo(parts[__ldg(P.hpart + h)], int64_t(__ldg(P.hidx + h)));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kChunk; ++u)
      if (c[u] >= 0) acc = __dadd_rn(acc, __dmul_rn(a[u], xv[u]));
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Distributed SpMV y = A x for the API spmv(): x in part.s, y in part.t
// (halo read straight from the owner's x, any device of the team).
// ---------------------------------------------------------------------------
// (a template so that only the TU launching it instantiates it)
template <int = 0>
__global__ void __launch_bounds__(256) spmv_kernel(const PartDev* __restrict__ parts, int p) {
  const PartDev& P = parts[p];
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  const double y = row_spmv(P, parts, i, [](const PartDev& Q, int64_t j) { return Q.s[j]; });
  P.t[i] = y;
}

// ---------------------------------------------------------------------------
// Team barrier with fused deterministic reduction.
// ---------------------------------------------------------------------------
// Canonical reduction tree (both solver families, every phase).  The leaves
// are tile partials tau_t (t = part-local tile; a tile's value is the
// canonical tile tree of its rows, below).  Tiles form units of K
// consecutive tiles (K = the phase's pack factor, 1 for SpMV phases); lane
// v < kLanes sums, from 0.0 and in ascending t, the tau_t of the units
// u = v (mod kLanes).  The lane values are reduced in groups of 32
// (butterfly xor 16..1, lanes >= kLanes hold 0.0), group sums in group order.
//
// kLanes = 148, the B200's SM count: with one streaming CTA per SM, CTA c
// processes exactly the units of lane c (its stage k is unit c + k * 148),
// so it computes its lane value itself, in stage order (T.lane_vals; the
// reducer warp, stream.cuh), and the barrier's last CTA only combines 148
// values per part.  Everywhere else (classic kernels, other grids, several
// parts per device) the last CTA computes the lanes from the tile partials —
// the same tree, so all configurations stay bit-identical.  (The previous
// tree had 512 strided lanes over 32-byte partial records: 500 KB through
// ONE SM per barrier, 10.4 us of the 10.8 us barrier at 200^3.)
#ifndef LRB_LANES
#define LRB_LANES 148
#endif
constexpr int kLanes = LRB_LANES;
constexpr int kLaneGroups = (kLanes + 31) / 32;
constexpr int kVecTileBytes = kTile * 8;   // one vector's rows of a tile
constexpr int kMaxPack = 4;                // tiles per stage in elementwise phases
// CG's x update: LRB_LAZY_X = 1 moves it out of phase B into the next SpMV
// phase (stream.cuh); the streaming phase B then stages 3 (PCG) / 2 (CG)
// tile vectors instead of 5 / 4 — the tree's units follow (pack_factor).
// Off by default: -8 B/row per iteration, but phase A pays nearly what B
// saves and the check phases get a window more (C3 -0.5%, C1/C2 +5%;
// profiles/r1_experiments.md).
#ifndef LRB_LAZY_X
#define LRB_LAZY_X 0
#endif
template <bool JAC>
constexpr int kCgBVecs = LRB_LAZY_X ? (JAC ? 3 : 2) : (JAC ? 5 : 4);

// Packing factor of an elementwise phase with ntv vectors (the streaming
// kernels' stage geometry; the classic kernels use it for the tree's units).
__device__ __forceinline__ int pack_factor(const TeamDev& T, int ntv) {
  const int k = T.stage_bytes / (kHdrBytes + ntv * kVecTileBytes);
  return k < 1 ? 1 : (k > kMaxPack ? kMaxPack : k);
}

// Does CTA c compute lane c itself in this phase?  Single local part
// (T.lane_fast, set by the host for streaming single-part teams), and every
// CTA's units belong to one lane: grid == kLanes, or at most one unit per CTA.
__device__ __forceinline__ bool lanes_by_cta(const TeamDev& T, int64_t ntiles, int K) {
  const int64_t units = (ntiles + K - 1) / K;
  return T.lane_fast && (int(gridDim.x) == kLanes || units <= int64_t(gridDim.x));
}

// Team barriers passed by this CTA in the current launch (every solver kernel
// zeroes it first).  Barrier b completes when the launch's arrival counter
// (SolveOut::flat_count, zeroed before the launch) reaches (b + 1) * grid, so
// no counter is reset in flight.  Its parity selects the lane-value buffer: a CTA
// can write barrier b+1's lane value only after every CTA arrived at b+1, i.e.
// after every CTA finished reading barrier b's lane values.
static __shared__ unsigned s_flat_bar;
__device__ __forceinline__ double* lane_slots(const TeamDev& T, unsigned bar) {
  return T.lane_vals + size_t(bar & 1u) * kLanes * kMaxRed;
}

// Lane v's value from the tile partials (the slow path): its tiles in
// ascending order, loads batched so the chain costs ceil(tiles / 16) trips.
template <int NR>
__device__ __forceinline__ void lane_from_partials(const TeamDev& T, const PartDev& P, int K, int v,
                                                   double (&acc)[NR]) {
  const double* __restrict__ base = T.partials + P.tile0;
  const int64_t stride = T.n_tiles, ntiles = P.ntiles;
  int64_t u = v;   // current unit, kk its tile
  int kk = 0;
  for (;;) {
    constexpr int kB = 16;
    double x[kB][NR];
    int nb = 0;
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const int64_t t = u * K + kk;
      const bool in = t < ntiles;
#pragma unroll
      for (int j = 0; j < NR; ++j) x[b][j] = in ? __ldcg(base + j * stride + t) : 0.0;
      nb += in ? 1 : 0;
      if (++kk == K) {
        kk = 0;
        u += kLanes;
      }
    }
#pragma unroll
    for (int b = 0; b < kB; ++b)
      if (b < nb)
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j] = __dadd_rn(acc[j], x[b][j]);
    if (nb < kB) break;
  }
}

// Part value (last CTA of the barrier, all threads): lanes, then the group tree.
template <int NR>
__device__ __forceinline__ void part_value(const TeamDev& T, int p, int K, double (*gs)[kMaxRed],
                                           double* out, unsigned bar) {
  const PartDev& P = T.parts[p];
  double acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.0;
  const int v = threadIdx.x;
  if (v < kLanes) {
    if (lanes_by_cta(T, P.ntiles, K)) {
      // lanes >= grid have no units (lanes_by_cta) and were not written
      const double* lv = lane_slots(T, bar) + (size_t(p - T.part_begin) * kLanes + v) * kMaxRed;
      if (v < int(gridDim.x))
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j] = __ldcg(lv + j);
    } else {
      lane_from_partials<NR>(T, P, K, v, acc);
    }
  }
  const int warp = threadIdx.x >> 5;
  if (warp < kLaneGroups) {
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] = __dadd_rn(acc[j], __shfl_xor_sync(0xffffffffu, acc[j], o));
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int j = 0; j < NR; ++j) gs[warp][j] = acc[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double s = gs[0][j];
      for (int g = 1; g < kLaneGroups; ++g) s = __dadd_rn(s, gs[g][j]);
      out[j] = s;
    }
  }
  __syncthreads();
}

// All local parts' values in one pass (several parts per device, e.g. C2 /
// C5 on one GPU): warp tasks (part q, lane group g) over the CTA's warps, the
// canonical lane values and group butterflies exactly as part_value, group
// sums parked in `scratch` (shared memory the caller owns and does not need
// across the barrier), then thread q sums part q's groups in group order.
// Two block barriers in total instead of two per part.  Out of line: it runs
// only in the barrier's last CTA and must not perturb the register
// allocation of the phase bodies.  scratch: [nloc * NR] part values followed
// by [nloc * kLaneGroups * NR] group sums.
template <int NR>
__device__ __noinline__ void parts_values(const TeamDev& T, int K, double* scratch) {
  const int nloc = T.part_end - T.part_begin;
  double* grp = scratch + nloc * NR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = int(blockDim.x >> 5);
  for (int task = warp; task < nloc * kLaneGroups; task += nw) {
    const int q = task / kLaneGroups, g = task - q * kLaneGroups;
    const int p = T.part_begin + q;
    const PartDev& P = T.parts[p];
    double acc[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) acc[j] = 0.0;
    const int v = g * 32 + lane;
    if (v < kLanes) {
      if (lanes_by_cta(T, P.ntiles, K)) {
        const double* lv = T.lane_vals + (size_t(q) * kLanes + v) * kMaxRed;
        if (v < int(gridDim.x))
#pragma unroll
          for (int j = 0; j < NR; ++j) acc[j] = __ldcg(lv + j);
      } else {
        lane_from_partials<NR>(T, P, K, v, acc);
      }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] = __dadd_rn(acc[j], __shfl_xor_sync(0xffffffffu, acc[j], o));
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < NR; ++j) grp[(q * kLaneGroups + g) * NR + j] = acc[j];
  }
  __syncthreads();
  if (int(threadIdx.x) < nloc) {
    const int q = threadIdx.x;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double s = grp[(q * kLaneGroups) * NR + j];
      for (int g = 1; g < kLaneGroups; ++g) s = __dadd_rn(s, grp[(q * kLaneGroups + g) * NR + j]);
      scratch[q * NR + j] = s;
    }
  }
  // the scratch is the bulk-copy ring of the streaming kernels: order these
  // generic writes before the next phase's async-proxy copies into it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
}

__device__ __forceinline__ int64_t tile_first(const TeamDev& T) {
  return LRB_CONTIG ? int64_t(blockIdx.x) * T.n_tiles / gridDim.x : int64_t(blockIdx.x);
}
__device__ __forceinline__ int64_t tile_end(const TeamDev& T) {
  return LRB_CONTIG ? (int64_t(blockIdx.x) + 1) * T.n_tiles / gridDim.x : T.n_tiles;
}
__device__ __forceinline__ int64_t tile_step() { return LRB_CONTIG ? 1 : int64_t(gridDim.x); }
__device__ __forceinline__ int64_t tile_of(const TeamDev& T, int t) {
  return tile_first(T) + int64_t(t) * tile_step();
}

static __device__ void team_fail(const TeamDev& T, int code) {
  atomicCAS((int*)&T.out->status, 0, code);
}

// All blocks of this device arrive; the last one reduces the tile partials of
// every local part in fixed order, exchanges part values with the peer devices
// (NVLink peer stores + release/acquire flags), sums all parts in ascending
// GPU rank and releases everybody.  Returns the team-reduced values in red[].
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu64(unsigned long long* p) {
  unsigned long long old;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(p) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu64(unsigned long long* p) {
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void st_release_gpu64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

#ifndef LRB_FLAT_BAR   // 0: single-part lane_fast teams take the last-CTA barrier too
#define LRB_FLAT_BAR 1
#endif
#ifndef LRB_FLAT_POLL_NS
#define LRB_FLAT_POLL_NS 32
#endif
// Flat barrier (one device, one part, CTA c = reduction lane c): every CTA
// publishes its lane value, arrives with a release add on a launch-monotonic
// counter and waits for the count of this barrier; then EVERY CTA sums the
// lane values itself in the canonical order (part_value's tree), so nobody
// waits for a last CTA to reduce, publish and release.  Bit-identical to the
// last-CTA barrier.  Critical path: the last arrival's add, one poll, one
// batch of lane loads.
template <int NR>
__device__ __forceinline__ void flat_sync(const TeamDev& T, double* red, double (*gs)[kMaxRed], double* pv,
                                          unsigned& s_last) {
  const unsigned b = s_flat_bar;   // every thread, before thread 0 advances it
  if (threadIdx.x == 0) {
    unsigned long long* cnt = &T.out->flat_count;
    const unsigned long long target = (unsigned long long)(b + 1) * gridDim.x;
    if (T.prof) {   // diagnostics: the last arrival stamps the phase end
      s_last = atom_add_acq_rel_gpu64(cnt) + 1 == target;
      if (s_last && *T.prof_n < T.prof_cap) T.prof[(*T.prof_n)++] = global_ns();
    } else {
      red_add_release_gpu64(cnt);
    }
    const long long t0 = global_ns();
    while (ld_acquire_gpu64(cnt) < target) {
      if (LRB_FLAT_POLL_NS) __nanosleep(LRB_FLAT_POLL_NS);
      if (global_ns() - t0 > T.timeout_ns) {
        team_fail(T, LRB_ETIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
  double acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.0;
  const int v = threadIdx.x;
  if (v < int(gridDim.x)) {   // lanes >= grid have no units (lanes_by_cta)
    const double* lv = lane_slots(T, b) + size_t(v) * kMaxRed;
#pragma unroll
    for (int j = 0; j < NR; ++j) acc[j] = __ldcg(lv + j);
  }
  const int warp = threadIdx.x >> 5;
  if (warp < kLaneGroups) {
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] = __dadd_rn(acc[j], __shfl_xor_sync(0xffffffffu, acc[j], o));
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int j = 0; j < NR; ++j) gs[warp][j] = acc[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double s = gs[0][j];
      for (int g = 1; g < kLaneGroups; ++g) s = __dadd_rn(s, gs[g][j]);
      pv[j] = s;
    }
    s_flat_bar = b + 1;
    if (T.prof && s_last && *T.prof_n < T.prof_cap) T.prof[(*T.prof_n)++] = global_ns();
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NR; ++j) red[j] = pv[j];
}

// All blocks of this device arrive; the last one reduces the tile partials of
// every local part in fixed order, exchanges part values with the peer devices
// (NVLink peer stores + release/acquire flags), sums all parts in ascending
// GPU rank and releases everybody.  Returns the team-reduced values in red[].
// Single-device teams keep the part values in shared memory (no global round
// trip); arrival and release are acq_rel / release atomics (cumulative over
// the CTA's writes through the preceding __syncthreads).
constexpr int kSmemParts = 16;
template <int NR>
__device__ void team_sync(const TeamDev& T, double* red, int K, double* scratch = nullptr) {
  __shared__ unsigned s_last;
  __shared__ double gs[kLaneGroups][kMaxRed];
  __shared__ double pv[kMaxRed];
  __shared__ double pvals[kSmemParts][kMaxRed];
  __syncthreads();
  if (LRB_FLAT_BAR && T.n_dev == 1 && T.n_parts == 1 && lanes_by_cta(T, T.n_tiles, K)) {
    flat_sync<NR>(T, red, gs, pv, s_last);
    return;
  }
  const unsigned bar = s_flat_bar;   // every thread, before thread 0 advances it
  if (threadIdx.x == 0) {
    if (T.n_dev > 1) __threadfence_system();
    const unsigned long long t = atom_add_acq_rel_gpu64(&T.out->flat_count);
    s_last = (t + 1 == (unsigned long long)(bar + 1) * gridDim.x);
  }
  __syncthreads();
  if (s_last) {
    if (threadIdx.x == 0 && T.prof && *T.prof_n < T.prof_cap) T.prof[(*T.prof_n)++] = global_ns();
    const bool local = T.n_dev == 1 && T.n_parts <= kSmemParts;
    // Part values are double-buffered by epoch parity: a fast peer may already
    // publish epoch e+1 into our buffer while we still read epoch e (it only
    // needs our flag for e, which we raise before summing).  It cannot reach
    // e+2 before our flag for e+1, i.e. before we finished reading e.
    const unsigned long long e_next = (T.n_dev > 1) ? *(volatile unsigned long long*)T.epoch + 1 : 0;
    const int64_t pbuf = int64_t(e_next & 1) * T.n_parts * kMaxRed;
    // several local parts: all their values in one pass (parts_values)
    const bool batched = scratch != nullptr && T.part_end - T.part_begin > 1;
    if (batched) parts_values<NR>(T, K, scratch);
    for (int p = T.part_begin; p < T.part_end; ++p) {
      if (batched) {
        if (threadIdx.x == 0)
#pragma unroll
          for (int j = 0; j < NR; ++j) pv[j] = scratch[(p - T.part_begin) * NR + j];
      } else {
        part_value<NR>(T, p, K, gs, pv, bar);
      }
#ifdef LRB_STAMP3
      if (threadIdx.x == 0 && T.prof && *T.prof_n < T.prof_cap) T.prof[(*T.prof_n)++] = global_ns();
#endif
      if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          if (local) {
            pvals[p][j] = pv[j];
          } else {
            T.part_red[pbuf + p * kMaxRed + j] = pv[j];
            for (int d = 0; d < T.n_dev; ++d)
              if (d != T.dev_rank) T.peer_part_red[d][pbuf + p * kMaxRed + j] = pv[j];
          }
        }
      }
    }
    if (threadIdx.x == 0) {
      if (T.n_dev > 1) {
        __threadfence_system();
        const unsigned long long e = e_next;
        *T.epoch = e;
        for (int d = 0; d < T.n_dev; ++d)
          if (d != T.dev_rank) st_release_sys(T.peer_flags[d] + T.dev_rank, e);
        const long long t0 = global_ns();
        for (int d = 0; d < T.n_dev; ++d) {
          if (d == T.dev_rank) continue;
          while (ld_acquire_sys(T.flags + d) < e) {
            __nanosleep(64);
            if (global_ns() - t0 > T.timeout_ns) {
              team_fail(T, LRB_ETIMEOUT);
              break;
            }
          }
        }
        __threadfence_system();
      }
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        double s = local ? pvals[0][j] : vload(T.part_red + pbuf + j);
        for (int p = 1; p < T.n_parts; ++p)
          s = __dadd_rn(s, local ? pvals[p][j] : vload(T.part_red + pbuf + p * kMaxRed + j));
        T.red[j] = s;
        pv[j] = s;
      }
      if (T.prof && *T.prof_n < T.prof_cap) T.prof[(*T.prof_n)++] = global_ns();
      s_flat_bar = bar + 1;
      st_release_gpu64(&T.out->flat_gen, bar + 1);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NR; ++j) red[j] = pv[j];
    return;
  }
  if (threadIdx.x == 0) {
    const long long t0 = global_ns();
    s_flat_bar = bar + 1;
    while (ld_acquire_gpu64(&T.out->flat_gen) < bar + 1) {
      __nanosleep(32);
      if (global_ns() - t0 > T.timeout_ns) {
        team_fail(T, LRB_ETIMEOUT);
        break;
      }
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) pv[j] = vload(T.red + j);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NR; ++j) red[j] = pv[j];
}

// Tile partials.  Canonical tree (shared by the classic and the streaming
// solvers, stream.cuh): a tile's kTile rows form kGroups groups of 32
// consecutive rows; each group's row values are butterfly-reduced (xor 16, 8,
// 4, 2, 1) and the tile partial is the sum of the group sums in group order.
// Warps never wait for each other inside a phase: group sums are parked in
// shared memory and summed per tile after the block's last tile.  Row order,
// trees and orders are fixed, so the per-tile partials are deterministic and
// independent of the grid size and of the kernel family.
constexpr int kWarps = kTPB / 32;
constexpr int kGroups = kTile / 32;

__host__ __device__ constexpr size_t phase_smem_bytes(int64_t tiles_per_block) {
  return size_t(tiles_per_block) * kGroups * kMaxRed * sizeof(double);
}

template <int NR>
__device__ __forceinline__ void group_reduce(double (&acc)[NR]) {
#pragma unroll
  for (int j = 0; j < NR; ++j)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[j] = __dadd_rn(acc[j], __shfl_xor_sync(0xffffffffu, acc[j], o));
}

template <int NR, class Body>
__device__ __forceinline__ void tile_rows(const PartDev& P, int64_t tile, double (&acc)[kRPT][NR],
                                          Body&& body) {
  const int64_t row0 = (tile - P.tile0) * kTile;
#pragma unroll
  for (int m = 0; m < kRPT; ++m) {
    const int64_t i = row0 + m * kTPB + threadIdx.x;
    if (i < P.n) body(P, i, acc[m]);
  }
}

// Elementwise phases: every row's loads of the tile are issued first
// (load(P, i) -> L), then the updates (apply(P, i, L, acc)) — the stores of
// one row cannot hold back the loads of the next (no aliasing proof needed).
template <int NR, class Load, class Apply>
struct SplitBody {
  Load load;
  Apply apply;
};

template <int NR, class Load, class Apply>
__device__ __forceinline__ void tile_rows(const PartDev& P, int64_t tile, double (&acc)[kRPT][NR],
                                          SplitBody<NR, Load, Apply>& body) {
  const int64_t row0 = (tile - P.tile0) * kTile;
  decltype(body.load(P, int64_t(0))) v[kRPT];
#pragma unroll
  for (int m = 0; m < kRPT; ++m) {
    const int64_t i = row0 + m * kTPB + threadIdx.x;
    if (i < P.n) v[m] = body.load(P, i);
  }
#pragma unroll
  for (int m = 0; m < kRPT; ++m) {
    const int64_t i = row0 + m * kTPB + threadIdx.x;
    if (i < P.n) body.apply(P, i, v[m], acc[m]);
  }
}

template <int NR, class Load, class Apply>
__device__ __forceinline__ SplitBody<NR, Load, Apply> split_body(Load&& l, Apply&& a) {
  return SplitBody<NR, Load, Apply>{l, a};
}

// Tile loop of one phase, then the team barrier with the fused reduction.
// INL: local part descriptors come from the kernel parameter (T.lp).
// ntv: the streaming kernel's tile vectors for this (elementwise) phase, 0
// for SpMV phases — it fixes the reduction tree's units (pack_factor).
template <int NR, bool INL, class Body>
__device__ __forceinline__ void team_phase(const TeamDev& T, double* red, int ntv, Body&& body) {
  extern __shared__ double wsm[];   // [tiles of this block][kGroups][kMaxRed]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tl = 0;
  for (int64_t tile = tile_first(T); tile < tile_end(T); tile += tile_step(), ++tl) {
    const int p = __ldg(T.tile_part + tile);
    double acc[kRPT][NR];
#pragma unroll
    for (int m = 0; m < kRPT; ++m)
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[m][j] = 0.0;
    if constexpr (INL) {
      tile_rows<NR>(T.lp[p - T.part_begin], tile, acc, body);
    } else {
      const PartDev P = T.parts[p];  // by value: no aliasing with the vector stores
      tile_rows<NR>(P, tile, acc, body);
    }
#pragma unroll
    for (int m = 0; m < kRPT; ++m) {
      group_reduce<NR>(acc[m]);
      if (lane == 0)
#pragma unroll
        for (int j = 0; j < NR; ++j) wsm[(tl * kGroups + m * kWarps + warp) * kMaxRed + j] = acc[m][j];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < tl * NR; idx += kTPB) {
    const int t = idx / NR, j = idx - t * NR;
    double s = wsm[(t * kGroups) * kMaxRed + j];
#pragma unroll
    for (int g = 1; g < kGroups; ++g) s = __dadd_rn(s, wsm[(t * kGroups + g) * kMaxRed + j]);
    T.partials[j * T.n_tiles + tile_of(T, t)] = s;
  }
  team_sync<NR>(T, red, ntv ? pack_factor(T, ntv) : 1);
}

// SpMV phase: body(P, i, acc, floc) with floc(c) = vecf(P, c) for local columns.
template <int NR, bool INL, class VecF, class Body>
__device__ __forceinline__ void team_phase_spmv(const TeamDev& T, double* red, VecF&& vecf,
                                                Body&& body) {
  team_phase<NR, INL>(T, red, 0, [&](const PartDev& P, int64_t i, double (&acc)[NR]) {
    body(P, i, acc, [&](int64_t c) { return vecf(P, c); });
  });
}

__device__ __forceinline__ bool team_failed(const TeamDev& T) {
  return *(const volatile int*)&T.out->status != 0;
}

// ---------------------------------------------------------------------------
// CG / Jacobi-PCG (solver.py:100-147).
//
// Per iteration two fused phases (+ the true-residual phase every 10th
// iteration or when the recurrence residual meets tol):
//  A: p_new = z + beta*p_old computed on the fly for every row and neighbour
//     (z = r for CG; for PCG z = dinv*r was stored by phase B, so a neighbour
//     costs two loads), q = A p_new, store p_new and q, partial p.q
//  B: x += step*p, r -= step*q, partial r.r (PCG: z = dinv*r stored, r.z)
//  C: y = A x, partial |b - y|^2
// p is double-buffered so phase A can read neighbours' p_old while writing p_new.
// ---------------------------------------------------------------------------
template <bool JAC, bool INL>
__global__ void __launch_bounds__(kTPB, LRB_MINB) team_cg_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  if (threadIdx.x == 0) s_flat_bar = 0;   // ordered by team_sync's entry barrier
  double red[2];
  // phase 0: x = 0, r = b, partial b.b (and r.z)
  team_phase<2, INL>(T, red, JAC ? 2 : 1, [&](const PartDev& P, int64_t i, double (&acc)[2]) {
    const double b = P.b[i];
    P.x[i] = 0.0;
    P.r[i] = b;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(b, b));
    if (JAC) {
      const double z = __dmul_rn(P.dinv[i], b);
      P.s[i] = z;  // z = dinv * r lives in s for Jacobi-PCG
      acc[1] = __dadd_rn(acc[1], __dmul_rn(b, z));
    }
  });
  const double bb = red[0];
  SolveOut* out = T.out;
  const bool lead = (blockIdx.x == 0 && threadIdx.x == 0);
  if (bb == 0.0 || team_failed(T)) {
    if (lead && bb == 0.0) {
      out->iterations = 0;
      out->converged = 1;
      out->residual = 0.0;
      out->bnorm = 0.0;
    }
    return;
  }
  const double bnorm = sqrt(bb);
  double rho = JAC ? red[1] : bb;
  double beta = 0.0, res = 1.0;
  int pa = 0;  // p_old lives in p0 when pa == 0
  bool first = true, converged = false;
  int it = 0;
  for (it = 1; it <= T.max_iter; ++it) {
    // ---- phase A: p_new, q = A p_new, p.q
    auto pnew = [&](const PartDev& Q, int64_t j) -> double {
      const double z = JAC ? Q.s[j] : Q.r[j];
      if (first) return z;
      const double po = pa ? Q.p1[j] : Q.p0[j];
      return __dadd_rn(z, __dmul_rn(beta, po));
    };
    team_phase_spmv<1, INL>(T, red, pnew,
                            [&](const PartDev& P, int64_t i, double (&acc)[1], auto&& floc) {
      const double pi = floc(i);
      const double qi = row_spmv2(P, parts, i, floc, pnew);
      (pa ? P.p0 : P.p1)[i] = pi;
      P.q[i] = qi;
      acc[0] = __dadd_rn(acc[0], __dmul_rn(pi, qi));
    });
    if (team_failed(T)) break;
    const double pq = red[0];
    if (pq <= 0.0) {
      if (lead) team_fail(T, LRB_ENOTPD);
      break;
    }
    const double step = rho / pq;
    pa ^= 1;  // p_new is now p_old for the elementwise phase and the next iteration
    // ---- phase B: x += step p, r -= step q, r.r (, r.z)
    struct BIn {
      double p, x, r, q, d;
    };
    auto phase_b = split_body<2>(
        [&](const PartDev& P, int64_t i) -> BIn {
          return BIn{(pa ? P.p1 : P.p0)[i], P.x[i], P.r[i], P.q[i], JAC ? P.dinv[i] : 0.0};
        },
        [&](const PartDev& P, int64_t i, const BIn& v, double (&acc)[2]) {
          const double x = __dadd_rn(v.x, __dmul_rn(step, v.p));
          const double r = __dsub_rn(v.r, __dmul_rn(step, v.q));
          P.x[i] = x;
          P.r[i] = r;
          acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
          if (JAC) {
            const double z = __dmul_rn(v.d, r);
            P.s[i] = z;
            acc[1] = __dadd_rn(acc[1], __dmul_rn(r, z));
          }
        });
#if LRB_SPLITB
    team_phase<2, INL>(T, red, kCgBVecs<JAC>, phase_b);
#else
    team_phase<2, INL>(T, red, kCgBVecs<JAC>, [&](const PartDev& P, int64_t i, double (&acc)[2]) {
      phase_b.apply(P, i, phase_b.load(P, i), acc);
    });
#endif
    if (team_failed(T)) break;
    const double rr_new = red[0];
    const double rho_new = JAC ? red[1] : rr_new;
    const double rec = sqrt(rr_new) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      // ---- phase C: true residual |b - A x|
      auto xval = [](const PartDev& Q, int64_t j) -> double { return Q.x[j]; };
      team_phase_spmv<1, INL>(T, red, xval,
                              [&](const PartDev& P, int64_t i, double (&acc)[1], auto&& floc) {
        const double ax = row_spmv2(P, parts, i, floc, xval);
        const double d = __dsub_rn(P.b[i], ax);
        acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
      });
      if (team_failed(T)) break;
      res = sqrt(red[0]) / bnorm;
      if (res <= T.tol) {
        converged = true;
        break;
      }
    } else {
      res = rec;
    }
    beta = rho_new / rho;
    rho = rho_new;
    first = false;
  }
  if (lead) {
    out->iterations = it > T.max_iter ? T.max_iter : it;
    out->converged = converged ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

// ---------------------------------------------------------------------------
// BiCGStab (oracle/krylov.py:bicgstab).  Three fused phases:
//  1: p_new = r + beta*(p_old - omega*v_old) on the fly, v = A p_new, rhat.v
//  2: s = r - alpha*v on the fly, t = A s, t.s, t.t
//  3: x = (x + alpha p) + omega s, r = s - omega t, r.r, rhat.r
// p and v are double-buffered.
// ---------------------------------------------------------------------------
template <bool INL>
__global__ void __launch_bounds__(kTPB, LRB_MINB) team_bicgstab_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  if (threadIdx.x == 0) s_flat_bar = 0;   // ordered by team_sync's entry barrier
  double red[2];
  team_phase<1, INL>(T, red, 1, [&](const PartDev& P, int64_t i, double (&acc)[1]) {
    const double b = P.b[i];
    P.x[i] = 0.0;
    P.r[i] = b;
    P.rhat[i] = b;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(b, b));
  });
  const double bb = red[0];
  SolveOut* out = T.out;
  const bool lead = (blockIdx.x == 0 && threadIdx.x == 0);
  if (bb == 0.0 || team_failed(T)) {
    if (lead && bb == 0.0) {
      out->iterations = 0;
      out->converged = 1;
      out->residual = 0.0;
      out->bnorm = 0.0;
    }
    return;
  }
  const double bnorm = sqrt(bb);
  double rho = bb, rho_prev = 1.0, alpha = 1.0, omega = 1.0, beta = 0.0, res = 1.0;
  int pa = 0;  // p_old/v_old in p0/v0 when pa == 0
  bool converged = false, breakdown = false;
  int it = 0;
  for (it = 1; it <= T.max_iter; ++it) {
    const bool first = (it == 1);
    if (!first) beta = __dmul_rn(rho / rho_prev, alpha / omega);
    // ---- phase 1
    team_phase<1, INL>(T, red, 0, [&](const PartDev& P, int64_t i, double (&acc)[1]) {
      auto pnew = [&](const PartDev& Q, int64_t j) -> double {
        const double r = Q.r[j];
        if (first) return r;
        const double po = pa ? Q.p1[j] : Q.p0[j];
        const double vo = pa ? Q.v1[j] : Q.v0[j];
        return __dadd_rn(r, __dmul_rn(beta, __dsub_rn(po, __dmul_rn(omega, vo))));
      };
      const double pi = pnew(P, i);
      const double vi = row_spmv(P, parts, i, pnew);
      (pa ? P.p0 : P.p1)[i] = pi;
      (pa ? P.v0 : P.v1)[i] = vi;
      acc[0] = __dadd_rn(acc[0], __dmul_rn(P.rhat[i], vi));
    });
    if (team_failed(T)) break;
    pa ^= 1;
    const double rv = red[0];
    if (rv == 0.0) {
      breakdown = true;
      break;
    }
    alpha = rho / rv;
    // ---- phase 2
    team_phase<2, INL>(T, red, 0, [&](const PartDev& P, int64_t i, double (&acc)[2]) {
      auto sval = [&](const PartDev& Q, int64_t j) -> double {
        const double v = pa ? Q.v1[j] : Q.v0[j];
        return __dsub_rn(Q.r[j], __dmul_rn(alpha, v));
      };
      const double si = sval(P, i);
      const double ti = row_spmv(P, parts, i, sval);
      P.s[i] = si;
      P.t[i] = ti;
      acc[0] = __dadd_rn(acc[0], __dmul_rn(ti, si));
      acc[1] = __dadd_rn(acc[1], __dmul_rn(ti, ti));
    });
    if (team_failed(T)) break;
    omega = red[1] != 0.0 ? red[0] / red[1] : 0.0;
    // ---- phase 3 (6: the streaming kernel's tile vectors, incl. u = p - omega v)
    team_phase<2, INL>(T, red, 6, [&](const PartDev& P, int64_t i, double (&acc)[2]) {
      const double p = (pa ? P.p1 : P.p0)[i];
      const double s = P.s[i];
      const double x = __dadd_rn(__dadd_rn(P.x[i], __dmul_rn(alpha, p)), __dmul_rn(omega, s));
      const double r = __dsub_rn(s, __dmul_rn(omega, P.t[i]));
      P.x[i] = x;
      P.r[i] = r;
      acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
      acc[1] = __dadd_rn(acc[1], __dmul_rn(P.rhat[i], r));
    });
    if (team_failed(T)) break;
    const double rr = red[0];
    rho_prev = rho;
    rho = red[1];
    const double rec = sqrt(rr) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      team_phase<1, INL>(T, red, 0, [&](const PartDev& P, int64_t i, double (&acc)[1]) {
        const double ax =
            row_spmv(P, parts, i, [](const PartDev& Q, int64_t j) { return Q.x[j]; });
        const double d = __dsub_rn(P.b[i], ax);
        acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
      });
      if (team_failed(T)) break;
      res = sqrt(red[0]) / bnorm;
      if (res <= T.tol) {
        converged = true;
        break;
      }
    } else {
      res = rec;
    }
    if (omega == 0.0 || rho == 0.0) {
      breakdown = true;
      break;
    }
  }
  if (lead) {
    out->iterations = it > T.max_iter ? T.max_iter : it;
    out->converged = converged ? 1 : 0;
    out->breakdown = breakdown ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

}  // namespace lrb
