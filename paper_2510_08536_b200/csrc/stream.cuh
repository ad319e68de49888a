// Streaming (warp-specialized) persistent Krylov solvers for sm_100a.
//
// Same algorithms, rounding contract, tile decomposition and reduction order as
// the classic team kernels in kernels.cuh (so both produce bit-identical
// iterates), but the HBM traffic is moved by the bulk-copy engine instead of
// per-thread gathers:
//
//   * one CTA per SM: 16 consumer warps (one thread per tile row; warp g is
//     group g of the canonical tile tree, kernels.cuh) + 1 producer warp;
//   * the producer walks this CTA's tiles of the current phase and, per tile,
//     issues cp.async.bulk copies global -> shared into a ring of n_stages
//     stages, each completing on the stage's "full" mbarrier (expect_tx):
//       SpMV phases : the tile's SELL values (one contiguous run), its row
//                     masks, and the <= kMaxWin operand windows of each vector
//                     the phase reads (tile_win, plan.cpp), + tile vectors;
//       elementwise : the tile's slice of every vector the phase reads;
//   * consumers wait on "full", compute from shared memory, store results with
//     coalesced st.global, and release the stage on its "empty" mbarrier;
//   * phases end in the same deterministic team barrier/reduction (team_sync).
//
// A tile whose pattern is not stageable (no windows: irregular slices, or too
// large for a stage) is computed by the consumers with direct global loads,
// exactly like the classic kernel.  Non-local (halo) columns are always read
// directly from the owning part (peer memory for other devices).
#pragma once

#include "kernels.cuh"

namespace lrb {

constexpr int kConsumers = kTile;               // one consumer thread per tile row (16 warps)
constexpr int kStreamThreads = kConsumers + 64;  // + two producer warps (see produce_phase)
constexpr int kMaskBytes = kTile * 2;          // uint16 row masks of a tile
constexpr int kVecTileBytes = kTile * 8;       // one vector's rows of a tile
constexpr int kStreamMaxStages = 4;
constexpr int kMaxPack = 4;                     // tiles per stage in elementwise phases
#ifndef LRB_SPMV_ISSUERS
#define LRB_SPMV_ISSUERS 2
#endif
constexpr int kSpmvIssuers = LRB_SPMV_ISSUERS;  // producer warps alternating SpMV stages
constexpr int kSlotRing = 2 * kStreamMaxStages; // group-sum slots (see consume_phase)
constexpr int kConsumerBar = 1;                // named barrier of the consumer warps


__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Spin on an mbarrier phase.  A ring that never completes is a bug, not a
// slow peer: after timeout_ns the kernel traps (a clean launch error instead
// of a hung device).
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity, long long timeout_ns) {
  if (mbar_try_wait(b, parity)) return;
  const long long t0 = global_ns();
  for (unsigned k = 1;; ++k) {
    if (mbar_try_wait(b, parity)) return;
    if ((k & 1023u) == 0 && global_ns() - t0 > timeout_ns) __trap();
  }
}
// 1D bulk copy global -> shared (TMA engine), completes tx bytes on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync %0, %1;" ::"n"(kConsumerBar), "n"(kConsumers) : "memory");
}

// Ring position shared by producer and consumers (both walk the same tiles).
struct Ring {
  int stage = 0;
  unsigned phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++stage == n) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

struct StreamSmem {
  char* stages;        // n_stages * stage_bytes
  uint64_t* full;      // [n_stages]
  uint64_t* empty;     // [n_stages]
  double* wpart;       // [2][kGroups][kMaxRed]
  int32_t* stile;      // [n_stages] first tile of each stage (-1: end of phase)
  int32_t* scnt;       // [n_stages] tiles packed in the stage (elementwise phases: up to kMaxPack)
  int32_t* ssub;       // [n_stages] byte stride between the packed tiles
  double* wsum;        // [kSlotRing][kMaxPack][kGroups][2] group sums awaiting their tile sum
  int32_t* wtile;      // [kSlotRing] first tile of the stage in the slot
  int32_t* wcnt;       // [kSlotRing] tiles of the stage in the slot
  int32_t* ring;       // [2] ring position after the phase (stage, phase)
  unsigned long long* cnt;   // [kCnt] wait-cycle counters (diagnostics, T.prof_cta)
};
// Diagnostic counters per CTA: [phase kind (0 init, 1 A, 2 B, 3 C)][what]
// what: 0 consumer warp 0 waiting for data, 1 end-of-phase consumer barrier,
// 2 producer waiting for a free stage, 3 team barrier (thread 0, arrival ->
// release), 4 warp 0 row bodies, 5 warp 0 group reduce + park, 6 warp 0 tile
// sums, 7 producer issuing (stage free -> copies issued).
#ifndef LRB_PROF
#define LRB_PROF 0   // build with -DLRB_PROF=1 for the wait/issue counters
#endif
constexpr bool kProf = LRB_PROF != 0;
constexpr int kCntPer = 8;
constexpr int kCnt = 4 * kCntPer;

__device__ __forceinline__ const PartDev& part_of(const TeamDev& T, int p, bool inl) {
  return inl ? T.lp[p - T.part_begin] : T.parts[p];
}

// What one phase stages: window vectors (SpMV phases) and whole-tile vectors.
struct Spec {
  int nwv;                 // window vectors (0: elementwise phase)
  int ntv;                 // tile vectors
  const double* wv[2];
  const double* tv[5];
};

__device__ __forceinline__ int stage_tail_offset(const StageHdr& H, int nwv) {
  return nwv ? kRecBytes + H.vbytes + nwv * H.wtot * 8 : kHdrBytes;
}

// ---------------------------------------------------------------------------
// Producer: warp 8, lane 0.  Tile headers are precomputed at team creation
// (T.tile_hdr, one StageHdr per device tile); the producer reads the next
// tile's addressing fields one tile ahead (their latency hides behind the
// current tile's copies) and bulk-copies the header itself into the stage.
// ---------------------------------------------------------------------------
struct HdrAddr {   // the fields the producer needs, 48 bytes
  int64_t row0, e0;
  int64_t wa[kMaxWin];
  int32_t rows, part;
};
__device__ __forceinline__ void load_hdr_addr(const StageHdr* h, HdrAddr& a, int32_t (&wl)[kMaxWin],
                                              int32_t (&woff)[kMaxWin], int32_t& nw, int32_t& wtot,
                                              int32_t& tma, int32_t& vbytes) {
  a.row0 = __ldg(&h->row0);
  a.e0 = __ldg(&h->e0);
#pragma unroll
  for (int w = 0; w < kMaxWin; ++w) {
    a.wa[w] = __ldg(&h->wa[w]);
    wl[w] = __ldg(&h->wl[w]);
    woff[w] = __ldg(&h->woff[w]);
  }
  a.rows = __ldg(&h->rows);
  a.part = __ldg(&h->part);
  nw = __ldg(&h->nw);
  wtot = __ldg(&h->wtot);
  tma = __ldg(&h->tma);
  vbytes = __ldg(&h->vbytes);
}

// Tiles are handed out dynamically: the producer grabs the next tile of the
// phase from the device's phase counter (atomicAdd, issued one tile ahead so
// its latency hides behind the current tile's copies), so CTAs finish a
// phase together whatever their bandwidth share.  Partials are per tile, so
// results do not depend on which CTA computed a tile.  After the last tile the
// producer publishes a sentinel (stile = -1) through the ring.
template <bool INL, class SpecF>
__device__ __forceinline__ void produce_phase(const TeamDev& T, const StreamSmem& S, Ring& ring,
                                              int kind, unsigned*, SpecF&& spec_of) {
  if ((threadIdx.x & 31) != 0) return;
  // kSpmvIssuers producer warps take alternate stages of the ring (stage
  // sequence k -> warp k % kSpmvIssuers), each issuing all copies of its
  // tiles: the per-copy issue cost no longer adds up on one thread.  Tiles
  // are static (tile of stage k = cta + k * grid) so every issuer knows
  // where the sentinel stage K* (first k with tile(k) >= n_tiles) falls.
  // The ring position is re-synchronised from the consumers after the phase.
  const int pw = (int(threadIdx.x) - kConsumers) >> 5;
  if (pw >= kSpmvIssuers) return;
  const uint64_t pol_stream = policy_evict_first();   // values / masks: read once per phase
  const uint64_t pol_vec = policy_evict_normal();     // vectors: re-read by neighbour tiles
  const StageHdr* hdrs = reinterpret_cast<const StageHdr*>(T.tile_hdr);
  const int64_t n_tiles = T.n_tiles;
  HdrAddr cur{}, nxt{};
  int32_t cwl[kMaxWin], cwoff[kMaxWin], cnw = 0, cwtot = 0, ctma = 0, cvb = 0;
  int32_t nwl[kMaxWin], nwoff[kMaxWin], nnw = 0, nwtot = 0, ntma = 0, nvb = 0;
  const int64_t step = int64_t(gridDim.x) * kSpmvIssuers;
  int64_t tile = int64_t(blockIdx.x) + int64_t(pw) * gridDim.x;
  for (int q = 0; q < pw; ++q) ring.next(T.n_stages);   // this issuer's first stage
  if (tile < n_tiles) load_hdr_addr(hdrs + tile, cur, cwl, cwoff, cnw, cwtot, ctma, cvb);
  while (true) {
    if (tile >= n_tiles && tile - gridDim.x >= n_tiles) break;   // K* is another issuer's
    const int64_t tn = tile + step;
    if (tn < n_tiles) load_hdr_addr(hdrs + tn, nxt, nwl, nwoff, nnw, nwtot, ntma, nvb);
    char* st = S.stages + size_t(ring.stage) * T.stage_bytes;
    uint64_t* full = S.full + ring.stage;
    {
      const long long c0 = (kProf && T.prof_cta) ? clock64() : 0;
      mbar_wait(S.empty + ring.stage, ring.phase ^ 1u, T.timeout_ns);
      if (kProf && T.prof_cta) S.cnt[kind * kCntPer + 2] += clock64() - c0;
    }
    if (tile >= n_tiles) {   // sentinel stage K*: the consumers leave the phase
      S.stile[ring.stage] = -1;
      mbar_arrive(full);
      break;
    }
    const long long ci = (kProf && T.prof_cta) ? clock64() : 0;
    S.stile[ring.stage] = int32_t(tile);
    S.scnt[ring.stage] = 1;
    S.ssub[ring.stage] = 0;
    const PartDev& P = part_of(T, cur.part, INL);
    const Spec sp = spec_of(P);
    const int rows = cur.rows;
    const int64_t row0 = cur.row0;
    const unsigned vec_bytes = unsigned((rows * 8 + 15) & ~15);
    if (sp.nwv) {
      const bool tma = ctma != 0;
      // record (header | slot tables | masks) in one copy, then the values
      const unsigned bytes = tma ? kRecBytes + unsigned(cvb) + unsigned(sp.nwv * cwtot * 8) +
                                       unsigned(sp.ntv) * vec_bytes
                                 : kHdrBytes;
      mbar_expect_tx(full, bytes);
      const TileRec* recs = reinterpret_cast<const TileRec*>(T.tile_rec);
      bulk_g2s(st, recs + tile, tma ? kRecBytes : kHdrBytes, full, pol_vec);
      if (tma) {
        char* d = st + kRecBytes;
        bulk_g2s(d, P.val + cur.e0, unsigned(cvb), full, pol_stream);
        d += cvb;
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int w = 0; w < kMaxWin; ++w)
            if (v < sp.nwv && w < cnw)
              bulk_g2s(d + (size_t(v) * cwtot + cwoff[w]) * 8, sp.wv[v] + cur.wa[w],
                       unsigned(cwl[w] * 8), full, pol_vec);
        d += size_t(sp.nwv) * cwtot * 8;
#pragma unroll
        for (int v = 0; v < 5; ++v)
          if (v < sp.ntv) bulk_g2s(d + size_t(v) * kVecTileBytes, sp.tv[v] + row0, vec_bytes, full, pol_vec);
      }
    } else {
      mbar_expect_tx(full, kHdrBytes + unsigned(sp.ntv) * vec_bytes);
      bulk_g2s(st, hdrs + tile, kHdrBytes, full, pol_vec);
      char* d = st + kHdrBytes;
#pragma unroll
      for (int v = 0; v < 5; ++v)
        if (v < sp.ntv) bulk_g2s(d + size_t(v) * kVecTileBytes, sp.tv[v] + row0, vec_bytes, full, pol_vec);
    }
    if (kProf && T.prof_cta) S.cnt[kind * kCntPer + 7] += clock64() - ci;
    for (int q = 0; q < kSpmvIssuers; ++q) ring.next(T.n_stages);
    const bool last = tile + gridDim.x >= n_tiles;   // stage k+1 (sentinel or not) belongs to the next issuer
    tile = tn;
    cur = nxt;
    if (last && kSpmvIssuers > 1) {
      // stages after this one: the sentinel falls at the first k with
      // tile(k) >= n_tiles; if that is not ours, stop here
      if (tile >= n_tiles && (tile - step + gridDim.x) >= n_tiles) {
        // our next tile is past the end and the sentinel stage belongs to the
        // issuer right after us: nothing more to issue
        break;
      }
    }
#pragma unroll
    for (int w = 0; w < kMaxWin; ++w) {
      cwl[w] = nwl[w];
      cwoff[w] = nwoff[w];
    }
    cnw = nnw;
    cwtot = nwtot;
    ctma = ntma;
    cvb = nvb;
  }
}

// Elementwise phases: a tile needs only kHdrBytes + ntv * kVecTileBytes, so
// the producer grabs K consecutive tiles per atomic and packs them into one
// stage (K = stage_bytes / tile bytes, at most kMaxPack): K times the bytes in
// flight of one tile per stage, with the same ring.
template <bool INL, class SpecF>
__device__ __forceinline__ void produce_elementwise(const TeamDev& T, const StreamSmem& S, Ring& ring,
                                                    int kind, unsigned* ctr, SpecF&& spec_of) {
  if ((threadIdx.x & 31) != 0 || threadIdx.x >= kConsumers + 32) return;   // producer warp 0
  const uint64_t pol_vec = policy_evict_normal();
  const StageHdr* hdrs = reinterpret_cast<const StageHdr*>(T.tile_hdr);
  const int64_t n_tiles = T.n_tiles;
  const bool one_part = T.part_end - T.part_begin == 1;
  const int ntv = spec_of(part_of(T, T.part_begin, INL)).ntv;
  const int sub = kHdrBytes + ntv * kVecTileBytes;
  int K = T.stage_bytes / sub;
  K = K < 1 ? 1 : (K > kMaxPack ? kMaxPack : K);
  int64_t c0 = atomicAdd(ctr, unsigned(K));
  int64_t c1 = c0 < n_tiles ? int64_t(atomicAdd(ctr, unsigned(K))) : n_tiles;
  while (true) {
    const int64_t c2 = c1 < n_tiles ? int64_t(atomicAdd(ctr, unsigned(K))) : n_tiles;
    char* st = S.stages + size_t(ring.stage) * T.stage_bytes;
    uint64_t* full = S.full + ring.stage;
    {
      const long long t0 = (kProf && T.prof_cta) ? clock64() : 0;
      mbar_wait(S.empty + ring.stage, ring.phase ^ 1u, T.timeout_ns);
      if (kProf && T.prof_cta) S.cnt[kind * kCntPer + 2] += clock64() - t0;
    }
    if (c0 >= n_tiles) {
      S.stile[ring.stage] = -1;
      mbar_arrive(full);
      ring.next(T.n_stages);
      break;
    }
    const long long ci = (kProf && T.prof_cta) ? clock64() : 0;
    const int cnt = int(n_tiles - c0 < K ? n_tiles - c0 : K);
    S.stile[ring.stage] = int32_t(c0);
    S.scnt[ring.stage] = cnt;
    S.ssub[ring.stage] = sub;
    int part[kMaxPack], rows[kMaxPack];
    int64_t row0[kMaxPack];
    unsigned bytes = 0;
#pragma unroll
    for (int j = 0; j < kMaxPack; ++j) {
      if (j < cnt) {
        const int64_t tile = c0 + j;
        part[j] = one_part ? T.part_begin : __ldg(T.tile_part + tile);
        const PartDev& P = part_of(T, part[j], INL);
        row0[j] = (tile - P.tile0) * kTile;
        rows[j] = int(P.n - row0[j] < kTile ? P.n - row0[j] : int64_t(kTile));
        bytes += kHdrBytes;
      }
    }
    if (part[0] == part[cnt - 1])
      bytes += unsigned(ntv) * unsigned(((row0[cnt - 1] + rows[cnt - 1] - row0[0]) * 8 + 15) & ~int64_t(15));
    else
      for (int j = 0; j < cnt; ++j) bytes += unsigned(ntv) * unsigned((rows[j] * 8 + 15) & ~15);
    mbar_expect_tx(full, bytes);
    // stage layout: [cnt headers][vector 0: cnt tiles][vector 1: cnt tiles]...
    // consecutive tiles of one part are contiguous rows: one copy per vector
    bulk_g2s(st, hdrs + c0, unsigned(cnt) * kHdrBytes, full, pol_vec);
    char* vbase = st + size_t(cnt) * kHdrBytes;
    const size_t vstride = size_t(cnt) * kVecTileBytes;
    if (part[0] == part[cnt - 1]) {
      const PartDev& P = part_of(T, part[0], INL);
      const Spec sp = spec_of(P);
      const unsigned vb = unsigned(((row0[cnt - 1] + rows[cnt - 1] - row0[0]) * 8 + 15) & ~int64_t(15));
#pragma unroll
      for (int v = 0; v < 5; ++v)
        if (v < sp.ntv) bulk_g2s(vbase + v * vstride, sp.tv[v] + row0[0], vb, full, pol_vec);
    } else {
#pragma unroll
      for (int j = 0; j < kMaxPack; ++j) {
        if (j < cnt) {
          const PartDev& P = part_of(T, part[j], INL);
          const Spec sp = spec_of(P);
          const unsigned vb = unsigned((rows[j] * 8 + 15) & ~15);
#pragma unroll
          for (int v = 0; v < 5; ++v)
            if (v < sp.ntv)
              bulk_g2s(vbase + v * vstride + size_t(j) * kVecTileBytes, sp.tv[v] + row0[j], vb, full, pol_vec);
        }
      }
    }
    if (kProf && T.prof_cta) S.cnt[kind * kCntPer + 7] += clock64() - ci;
    ring.next(T.n_stages);
    c0 = c1;
    c1 = c2;
  }
}

// Position of local column c in the staged windows (or -1).
struct WinMap {
  int64_t wa0, wa1, wa2;
  int wl0, wl1, wl2, wo1, wo2;
  __device__ __forceinline__ int pos(int64_t c) const {
    unsigned d = unsigned(c - wa0);
    if (d < unsigned(wl0)) return int(d);
    d = unsigned(c - wa1);
    if (d < unsigned(wl1)) return wo1 + int(d);
    d = unsigned(c - wa2);
    if (d < unsigned(wl2)) return wo2 + int(d);
    return -1;
  }
};
__device__ __forceinline__ WinMap win_map(const StageHdr& H) {
  WinMap M;
  M.wa0 = H.wa[0];
  M.wa1 = H.wa[1];
  M.wa2 = H.wa[2];
  M.wl0 = H.nw > 0 ? H.wl[0] : 0;
  M.wl1 = H.nw > 1 ? H.wl[1] : 0;
  M.wl2 = H.nw > 2 ? H.wl[2] : 0;
  M.wo1 = H.woff[1];
  M.wo2 = H.woff[2];
  return M;
}

// Staged SpMV of the consumer thread's row (lr = tid).  Per warp slice, lane k
// owns pattern slot k: its column offset and the shared-memory index delta of
// the window holding that offset's columns (computed once per slice instead
// of a window search per entry), broadcast with shuffles.  Every local column
// of a staged tile lies in a window by construction (plan.cpp
// build_tile_windows).  Entries accumulate in stored order with the reference
// rounding.  xs(q): staged operand at smem index q; fh(owner part, row): halo
// column.  Returns A_row . x.
// Operand of a staged window position: NV = 1: w0[q]; NV = 2: the on-the-fly
// p_new = w0[q] + beta * w1[q] (z and p_old windows, reference rounding).
template <int NV>
__device__ __forceinline__ double staged_operand(const double* __restrict__ w0,
                                                 const double* __restrict__ w1, double beta, int q) {
  if constexpr (NV == 1) {
    return w0[q];
  } else {
    return __dadd_rn(w0[q], __dmul_rn(beta, w1[q]));
  }
}

// Fixed-width row product: WM pattern slots, all operand loads issued
// before the accumulation chain (slots k >= w and holes are masked to 0).
template <int NV, int WM>
__device__ __forceinline__ double row_fixed(int w, int ii, int eb, unsigned msk,
                                            const int2* __restrict__ slot,
                                            const double* __restrict__ sval,
                                            const double* __restrict__ w0,
                                            const double* __restrict__ w1, double beta) {
  double a[WM], x[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    const bool on = k < w && ((msk >> k) & 1u);
    const int2 se = slot[k];
    a[k] = on ? sval[eb + k * kSlice] : 0.0;
    x[k] = on ? staged_operand<NV>(w0, w1, beta, ii + se.y) : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < WM; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], x[k]));
  return acc;
}

// Slot table of the warp's slice in the staged StageTab.
__device__ __forceinline__ const int2* slice_slots(const char* st, const StageHdr& H, int sl) {
  return reinterpret_cast<const int2*>(st + kHdrBytes) + H.spat[sl] * 16;
}

template <int NV, bool HALO, class FH>
__device__ __forceinline__ double row_spmv_staged(const int n, const int32_t* __restrict__ hpart,
                                                  const int32_t* __restrict__ hidx,
                                                  const PartDev* __restrict__ parts, const StageHdr& H,
                                                  const int2* __restrict__ slot,
                                                  const double* __restrict__ sval,
                                                  const uint16_t* __restrict__ smask,
                                                  const double* __restrict__ w0,
                                                  const double* __restrict__ w1, double beta, int lr,
                                                  FH&& fh) {
  const int lane = threadIdx.x & 31;
  const int rows = H.rows;
  const int lr0 = lr & ~31;                    // warp-uniform
  const int sl = lr0 >> 5;
  const int s0 = H.sp[sl];
  const int w = lr0 < rows ? (H.sp[sl + 1] - s0) >> 5 : 0;
  const int eb = s0 + lane;
  const int ii = int(H.row0) + lr;
  const unsigned msk = lr < rows ? unsigned(smask[lr]) : 0u;
  if constexpr (!HALO) {
    if (w == 7) return row_fixed<NV, 7>(w, ii, eb, msk, slot, sval, w0, w1, beta);
    if (w <= 8) return row_fixed<NV, 8>(w, ii, eb, msk, slot, sval, w0, w1, beta);
    return row_fixed<NV, kPatW>(w, ii, eb, msk, slot, sval, w0, w1, beta);
  } else {
    // holes (mask bit clear) have value 0.0 in the SELL layout and get operand
    // 0.0 here, so acc + 0 * 0 leaves acc unchanged (acc is never -0.0)
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
      const int2 se = slot[k];
      const bool on = (msk >> k) & 1u;
      const double a = sval[eb + k * kSlice];
      const int c = ii + se.x;
      double xv;
      if (on && c >= n) {
        xv = fh(parts[__ldg(hpart + (c - n))], int64_t(__ldg(hidx + (c - n))));
      } else {
        xv = staged_operand<NV>(w0, w1, beta, on ? ii + se.y : 0);
        xv = on ? xv : 0.0;
      }
      acc = __dadd_rn(acc, __dmul_rn(a, xv));
    }
    return acc;
  }
}

// Vectors of one packed elementwise tile: vector v at base + v * stride.
struct VecView {
  const char* base;
  size_t stride;
  __device__ __forceinline__ const double* operator[](int v) const {
    return reinterpret_cast<const double*>(base + v * stride);
  }
};

// Tile sum of the stage in slot ss: group g's sum of sub-tile j was parked at
// wsum[ss % kSlotRing][j][g] by warp g; warp (ss*kMaxPack + j) % kGroups adds
// the 16 group sums in group order (the canonical tile tree, kernels.cuh).
template <int NR>
__device__ __forceinline__ void sum_stage_slot(const TeamDev& T, const StreamSmem& S, int ss) {
  const int sl = ss % kSlotRing;
  const int cnt = S.wcnt[sl];
  const int64_t t0 = S.wtile[sl];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = 0; j < cnt; ++j) {
    if (warp == ((ss * kMaxPack + j) & (kGroups - 1)) && lane < NR) {
      const double* w = S.wsum + (size_t(sl * kMaxPack + j) * kGroups) * 2;
      double sum = w[lane];
#pragma unroll
      for (int g = 1; g < kGroups; ++g) sum = __dadd_rn(sum, w[g * 2 + lane]);
      T.partials[(t0 + j) * kMaxRed + lane] = sum;
    }
  }
}

// L2 prefetch of a future tile (the bulk copies of whoever processes it then
// hit L2): its SELL values and row masks (SpMV phases) and its own rows of
// every vector the phase reads.  Issued by the consumers, spread one line
// per thread, PD = kPrefetchRounds * grid tiles ahead of the tile being
// computed (dynamic scheduling hands tiles out in increasing order, so every
// tile is prefetched once, about that many tiles before it is copied).
// Off by default: measured on B200 at C3 it slows the solve 11.1 -> 15.5 ms
// (the consumers stall on the prefetch addresses and the extra L2 requests
// compete with the bulk copies).  -DLRB_PREFETCH_ROUNDS=2 to experiment.
#ifndef LRB_PREFETCH_ROUNDS
#define LRB_PREFETCH_ROUNDS 0
#endif
constexpr int kPrefetchRounds = LRB_PREFETCH_ROUNDS;

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

struct PrefetchTarget {
  int64_t row0, e0;
  int32_t rows, part, vbytes, ok;
};

__device__ __forceinline__ PrefetchTarget prefetch_target(const TeamDev& T, int64_t tile) {
  PrefetchTarget f{0, 0, 0, 0, 0, 0};
  if (kPrefetchRounds > 0 && tile < T.n_tiles) {
    const StageHdr* h = reinterpret_cast<const StageHdr*>(T.tile_hdr) + tile;
    f.row0 = __ldg(&h->row0);
    f.e0 = __ldg(&h->e0);
    f.rows = __ldg(&h->rows);
    f.part = __ldg(&h->part);
    f.vbytes = __ldg(&h->vbytes);
    f.ok = 1;
  }
  return f;
}

template <bool INL, class SpecF>
__device__ __forceinline__ void prefetch_tile(const TeamDev& T, const PrefetchTarget& f, SpecF&& spec_of) {
  if (!f.ok) return;
  const PartDev& Q = part_of(T, f.part, INL);
  const Spec sp = spec_of(Q);
  const int t = threadIdx.x;
  const int vl = (f.rows * 8 + 127) >> 7;   // 128-byte lines of one vector's rows
  int line = t;
  if (sp.nwv) {
    const char* vb = reinterpret_cast<const char*>(Q.val + f.e0);
    for (int off = t * 128; off < f.vbytes; off += kConsumers * 128) prefetch_l2(vb + off);
    line -= (f.vbytes + 127) >> 7;
    const int ml = (f.rows * 2 + 127) >> 7;
    if (line >= 0 && line < ml) prefetch_l2(reinterpret_cast<const char*>(Q.rmask + f.row0) + line * 128);
    line -= ml;
  }
  if (line < 0) line += kConsumers;   // threads past the values take the vectors
  const int nv = sp.nwv + sp.ntv;
  if (line >= 0 && line < nv * vl) {
    const int v = line / vl;
    const double* vec = v < sp.nwv ? sp.wv[v] : sp.tv[v - sp.nwv];
    prefetch_l2(reinterpret_cast<const char*>(vec + f.row0) + (line - v * vl) * 128);
  }
}

// Consumer side of one phase: thread tid computes row tid of each tile
// (body(P, H, st, acc)); warp g's butterfly sum is group g of the canonical
// tile tree and is parked in the stage's group-sum slot.  No per-tile block
// barrier: a warp that starts stage ss knows (through the ring: the producer
// refilled that stage only after every warp released stage ss - n_stages)
// that all group sums of stage ss - n_stages are written, and sums them then;
// the last n_stages stages are summed after one barrier at the end.  Slots
// are reused after kSlotRing = 2 * max stages, beyond the fastest warp's lead.
template <int NR, bool INL, class SpecF, class Body>
__device__ __forceinline__ void consume_phase(const TeamDev& T, const StreamSmem& S, Ring& ring,
                                              int kind, SpecF&& spec_of, Body&& body) {
  static_assert(NR <= 2, "group-sum slots hold two reductions");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ns = T.n_stages;
  int ss = 0;
  for (;; ++ss) {
    const char* st0 = S.stages + size_t(ring.stage) * T.stage_bytes;
    const long long c0 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
    mbar_wait(S.full + ring.stage, ring.phase, T.timeout_ns);
    if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 0] += clock64() - c0;
    {
      const long long c2 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      if (ss >= ns) sum_stage_slot<NR>(T, S, ss - ns);
      if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 6] += clock64() - c2;
    }
    const int64_t tile0 = S.stile[ring.stage];
    if (tile0 < 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(S.empty + ring.stage);
      ring.next(ns);
      break;
    }
    const int cnt = S.scnt[ring.stage];
    const int sub = S.ssub[ring.stage];
    const int sl = ss % kSlotRing;
    if (threadIdx.x == 0) {
      S.wtile[sl] = int32_t(tile0);
      S.wcnt[sl] = cnt;
    }
    const int64_t pd = int64_t(kPrefetchRounds) * gridDim.x;
    for (int j = 0; j < cnt; ++j) {
      const PrefetchTarget pf = prefetch_target(T, tile0 + j + pd);
      // SpMV stages hold one tile at st0; packed elementwise stages hold cnt
      // headers, then each vector's cnt tiles (produce_elementwise)
      const char* st = sub ? st0 + size_t(j) * kHdrBytes : st0;
      const VecView V{sub ? st0 + size_t(cnt) * kHdrBytes + size_t(j) * kVecTileBytes : nullptr,
                      size_t(cnt) * kVecTileBytes};
      const StageHdr& H = *reinterpret_cast<const StageHdr*>(st);
      const PartDev& P = part_of(T, H.part, INL);
      double acc[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) acc[q] = 0.0;
      const long long c3 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      body(P, H, st, V, acc);
      prefetch_tile<INL>(T, pf, spec_of);
      const long long c4 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      group_reduce<NR>(acc);
      if (lane == 0) {
        double* w = S.wsum + (size_t(sl * kMaxPack + j) * kGroups + warp) * 2;
#pragma unroll
        for (int q = 0; q < NR; ++q) w[q] = acc[q];
      }
      if (kProf && T.prof_cta && threadIdx.x == 0) {
        const long long c5 = clock64();
        S.cnt[kind * kCntPer + 4] += c4 - c3;
        S.cnt[kind * kCntPer + 5] += c5 - c4;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(S.empty + ring.stage);   // group sums written before the release
    ring.next(ns);
  }
  const long long c1 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
  consumer_bar();
  if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 1] += clock64() - c1;
  for (int s2 = (ss - ns + 1 > 0 ? ss - ns + 1 : 0); s2 < ss; ++s2) sum_stage_slot<NR>(T, S, s2);
}

// The consumer thread's row of a tile: lr = tid, i = row0 + lr.
#define LRB_FOR_ROW(H, i, lr)                                   \
  if (const int lr = int(threadIdx.x); lr < (H).rows)           \
    if (const int64_t i = (H).row0 + lr; true)

__device__ __forceinline__ StreamSmem stream_smem(const TeamDev& T) {
  extern __shared__ __align__(128) char dsm[];
  StreamSmem S;
  S.stages = dsm;
  char* tail = dsm + size_t(T.n_stages) * T.stage_bytes;
  S.full = reinterpret_cast<uint64_t*>(tail);
  S.empty = S.full + kStreamMaxStages;
  S.wpart = reinterpret_cast<double*>(S.empty + kStreamMaxStages);
  S.cnt = reinterpret_cast<unsigned long long*>(S.wpart + 2 * kGroups * kMaxRed);
  S.stile = reinterpret_cast<int32_t*>(S.cnt + kCnt);
  S.scnt = S.stile + kStreamMaxStages;
  S.ssub = S.scnt + kStreamMaxStages;
  S.wtile = S.ssub + kStreamMaxStages;
  S.wcnt = S.wtile + kSlotRing;
  S.ring = S.wcnt + kSlotRing;
  S.wsum = reinterpret_cast<double*>(S.ring + 2);   // 8-byte aligned
  return S;
}
__host__ __device__ constexpr size_t stream_smem_bytes(int stage_bytes, int n_stages) {
  return size_t(stage_bytes) * n_stages + 2 * kStreamMaxStages * 8 + 2 * kGroups * kMaxRed * 8 +
         kCnt * 8 + 3 * kStreamMaxStages * 4 + 2 * kSlotRing * 4 + 8 +
         size_t(kSlotRing) * kMaxPack * kGroups * 2 * 8;
}

__device__ __forceinline__ void stream_init(const TeamDev& T, const StreamSmem& S) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < T.n_stages; ++s) {
      mbar_init(S.full + s, 1);
      mbar_init(S.empty + s, kGroups);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < kCnt) S.cnt[threadIdx.x] = 0;
  __syncthreads();
}

// Phase wrapper: producer warp streams, consumers compute, then the team
// barrier with the fused reduction (all threads).
template <int NR, bool INL, bool ELEM, class SpecF, class Body>
__device__ __forceinline__ void stream_phase(const TeamDev& T, const StreamSmem& S, Ring& ring,
                                             double* red, int kind, int& seq, SpecF&& spec_of,
                                             Body&& body) {
  unsigned* ctr = T.tile_ctr + (seq & 1);   // phase seq grabs tiles here; reset at its barrier
  if (threadIdx.x >= kConsumers) {
    fence_proxy_async_global();   // peers' generic writes of the last phase -> our bulk reads
    if constexpr (ELEM)
      produce_elementwise<INL>(T, S, ring, kind, ctr, spec_of);
    else
      produce_phase<INL>(T, S, ring, kind, ctr, spec_of);
  } else {
    consume_phase<NR, INL>(T, S, ring, kind, spec_of, body);
  }
  if (threadIdx.x == 0) {   // the consumers' ring position is the truth for every thread
    S.ring[0] = ring.stage;
    S.ring[1] = int(ring.phase);
  }
  fence_proxy_async_global();
  const long long c0 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
  team_sync<NR, kRedLanes / kConsumers>(T, red, ctr);
  if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 3] += clock64() - c0;
  ring.stage = S.ring[0];
  ring.phase = unsigned(S.ring[1]);
  ++seq;
}

// Diagnostics: this CTA's counters to T.prof_cta[blockIdx.x * kCnt ...].
__device__ __forceinline__ void stream_flush_counters(const TeamDev& T, const StreamSmem& S) {
  __syncthreads();
  if (kProf && T.prof_cta && threadIdx.x < kCnt) T.prof_cta[blockIdx.x * kCnt + threadIdx.x] = (long long)S.cnt[threadIdx.x];
}

// ---------------------------------------------------------------------------
// CG / Jacobi-PCG, streaming.  Phases and arithmetic are those of
// team_cg_kernel (kernels.cuh): A = {p_new, q = A p_new, p.q},
// B = {x, r update, r.r (r.z)}, C = {|b - A x|^2}.
// ---------------------------------------------------------------------------
template <bool JAC, bool INL>
__global__ void __launch_bounds__(kStreamThreads, 1)
    team_cg_stream_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  const StreamSmem S = stream_smem(T);
  stream_init(T, S);
  Ring ring;
  int seq = 0;   // phase sequence number (tile counter parity)
  double red[2];
  // ---- phase 0: x = 0, r = b, (z = dinv*b), b.b (, b.z)
  stream_phase<2, INL, true>(
      T, S, ring, red, 0, seq,
      [&](const PartDev& P) {
        return Spec{0, JAC ? 2 : 1, {nullptr, nullptr}, {P.b, JAC ? P.dinv : nullptr}};
      },
      [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, double (&acc)[2]) {
        const double* vb = V[0];
        const double* vd = V[1];
        LRB_FOR_ROW(H, i, lr) {
          const double b = vb[lr];
          P.x[i] = 0.0;
          P.r[i] = b;
          acc[0] = __dadd_rn(acc[0], __dmul_rn(b, b));
          if (JAC) {
            const double z = __dmul_rn(vd[lr], b);
            P.s[i] = z;
            acc[1] = __dadd_rn(acc[1], __dmul_rn(b, z));
          }
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
  int pa = 0;
  bool first = true, converged = false;
  int it = 0;
  for (it = 1; it <= T.max_iter; ++it) {
    // ---- phase A: p_new = z + beta p_old (staged windows), q = A p_new, p.q
    auto pnew_g = [&](const PartDev& Q, int64_t j) -> double {
      const double z = JAC ? Q.s[j] : Q.r[j];
      if (first) return z;
      const double po = pa ? Q.p1[j] : Q.p0[j];
      return __dadd_rn(z, __dmul_rn(beta, po));
    };
    stream_phase<1, INL, false>(
        T, S, ring, red, 1, seq,
        [&](const PartDev& P) {
          const double* z = JAC ? P.s : P.r;
          const double* po = pa ? P.p1 : P.p0;
          return first ? Spec{1, 0, {z, nullptr}, {}} : Spec{2, 0, {z, po}, {}};
        },
        [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, double (&acc)[1]) {
          double* pout = pa ? P.p0 : P.p1;
          if (H.tma) {
            const double* sval = reinterpret_cast<const double*>(st + kRecBytes);
            const uint16_t* smask = reinterpret_cast<const uint16_t*>(st + kHdrBytes + kTabBytes);
            const double* zw = reinterpret_cast<const double*>(st + kRecBytes + H.vbytes);
            const double* pw = zw + H.wtot;   // p_old windows (not staged in the first iteration)
            const int lr = int(threadIdx.x);
            const int sl = lr >> 5;
            const int2* slot = slice_slots(st, H, sl);
            const int n = int(P.n);
            double qi;
            if (first) {
              qi = P.n_halo ? row_spmv_staged<1, true>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, zw, pw,
                                                      beta, lr, pnew_g)
                            : row_spmv_staged<1, false>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, zw,
                                                       pw, beta, lr, pnew_g);
            } else {
              qi = P.n_halo ? row_spmv_staged<2, true>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, zw, pw,
                                                      beta, lr, pnew_g)
                            : row_spmv_staged<2, false>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, zw,
                                                       pw, beta, lr, pnew_g);
            }
            if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              const int qd = int(i) + slot[H.sdiag[H.spat[sl]]].y;   // the diagonal's operand
              const double pi = first ? zw[qd] : staged_operand<2>(zw, pw, beta, qd);
              pout[i] = pi;
              P.q[i] = qi;
              acc[0] = __dadd_rn(acc[0], __dmul_rn(pi, qi));
            }
          } else {
            LRB_FOR_ROW(H, i, lr) {
              const double pi = pnew_g(P, i);
              const double qi = row_spmv(P, parts, i, pnew_g);
              pout[i] = pi;
              P.q[i] = qi;
              acc[0] = __dadd_rn(acc[0], __dmul_rn(pi, qi));
            }
          }
        });
    if (team_failed(T)) break;
    const double pq = red[0];
    if (pq <= 0.0) {
      if (lead) team_fail(T, LRB_ENOTPD);
      break;
    }
    const double step = rho / pq;
    pa ^= 1;
    // ---- phase B: x += step p, r -= step q, r.r (, r.z)
    stream_phase<2, INL, true>(
        T, S, ring, red, 2, seq,
        [&](const PartDev& P) {
          return Spec{0, JAC ? 5 : 4, {nullptr, nullptr},
                      {pa ? P.p1 : P.p0, P.x, P.r, P.q, JAC ? P.dinv : nullptr}};
        },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, double (&acc)[2]) {
          const double* vp = V[0];
          const double* vx = V[1];
          const double* vr = V[2];
          const double* vq = V[3];
          const double* vd = V[4];
          LRB_FOR_ROW(H, i, lr) {
            const double x = __dadd_rn(vx[lr], __dmul_rn(step, vp[lr]));
            const double r = __dsub_rn(vr[lr], __dmul_rn(step, vq[lr]));
            P.x[i] = x;
            P.r[i] = r;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
            if (JAC) {
              const double z = __dmul_rn(vd[lr], r);
              P.s[i] = z;
              acc[1] = __dadd_rn(acc[1], __dmul_rn(r, z));
            }
          }
        });
    if (team_failed(T)) break;
    const double rr_new = red[0];
    const double rho_new = JAC ? red[1] : rr_new;
    const double rec = sqrt(rr_new) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      // ---- phase C: true residual |b - A x|
      auto xg = [](const PartDev& Q, int64_t j) -> double { return Q.x[j]; };
      stream_phase<1, INL, false>(
          T, S, ring, red, 3, seq, [&](const PartDev& P) { return Spec{1, 1, {P.x, nullptr}, {P.b}}; },
          [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, double (&acc)[1]) {
            if (H.tma) {
              const double* sval = reinterpret_cast<const double*>(st + kRecBytes);
              const uint16_t* smask = reinterpret_cast<const uint16_t*>(st + kHdrBytes + kTabBytes);
              const double* xw = reinterpret_cast<const double*>(st + kRecBytes + H.vbytes);
              const double* vb = reinterpret_cast<const double*>(st + stage_tail_offset(H, 1));
              const int lr = int(threadIdx.x);
              const int2* slot = slice_slots(st, H, lr >> 5);
              const int n = int(P.n);
              const double ax =
                  P.n_halo ? row_spmv_staged<1, true>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, xw, xw,
                                                     0.0, lr, xg)
                           : row_spmv_staged<1, false>(n, P.hpart, P.hidx, parts, H, slot, sval, smask, xw,
                                                      xw, 0.0, lr, xg);
              if (lr < H.rows) {
                const double d = __dsub_rn(vb[lr], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            } else {
              LRB_FOR_ROW(H, i, lr) {
                const double ax = row_spmv(P, parts, i, xg);
                const double d = __dsub_rn(P.b[i], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            }
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
  stream_flush_counters(T, S);
  if (lead) {
    out->iterations = it > T.max_iter ? T.max_iter : it;
    out->converged = converged ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

}  // namespace lrb
