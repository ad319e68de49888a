// Streaming (warp-specialized) persistent Krylov solvers for sm_100a.
//
// Same algorithms, rounding contract, tile decomposition and reduction order
// as the classic team kernels in kernels.cuh (both produce bit-identical
// iterates), but the HBM traffic is moved by the bulk-copy (TMA) engine into
// a shared-memory ring instead of by per-thread gathers.
//
// CTA = one per SM:
//   * kIssuers producer warps; stage k of a phase is issued by warp
//     k % kIssuers (lane 0), which waits for the slot's "empty" mbarrier and
//     issues every bulk copy of the stage against its "full" mbarrier
//     (expect_tx).  cp.async.bulk serializes per issuing thread at ~0.1-0.35
//     us per copy (tools/tma_probe.cu), so alternate stages go to different
//     warps (measured at C3: one issuer 11.2 ms/step, two 9.2 ms);
//   * two consumer teams of 8 warps; team k % 2 consumes stage k.  Team
//     thread t computes rows t and t + kTPB of the tile — the classic
//     kernels' row mapping, so warp w of a team produces groups w and w + 8
//     of the canonical tile tree (kernels.cuh);
//   * phases end in the deterministic team barrier/reduction (team_sync).
//
// Stage contents:
//   SpMV phases (A: q = A p_new, C: |b - A x|): one tile = the tile record
//     (header | slot tables | row masks, one copy), its SELL values (one
//     copy), the <= kMaxWin operand windows of each vector the phase reads
//     (tile_win, plan.cpp) and whole-tile vectors;
//   elementwise phases (init, B): K consecutive tiles (the packing factor
//     K = stage_bytes / tile bytes): their headers, then each vector's K
//     tiles (one copy per vector).
// Tiles are assigned statically (stage k of CTA c holds tile c + k * grid,
// elementwise: chunk c + k * grid), so producers and consumers both know a
// phase's stage count and no sentinel stages are needed.
//
// A tile whose pattern is not stageable (irregular slices, or too large for a
// stage) is computed by the consumers with direct global loads, exactly like
// the classic kernel.  Non-local (halo) columns are always read directly from
// the owning part (peer memory for other devices).
#pragma once

#include "kernels.cuh"

namespace lrb {

#ifndef LRB_TEAMS
#define LRB_TEAMS 2
#endif
constexpr int kTeams = LRB_TEAMS;                 // 16 consumer warps in one or two teams
constexpr int kConsumers = 16 * 32;
constexpr int kTeamThreads = kConsumers / kTeams;
constexpr int kTeamWarps = kTeamThreads / 32;
constexpr int kSRPT = kTile / kTeamThreads;       // rows per team thread and tile
static_assert((kTeams == 1 || kTeams == 2) && kSRPT * kTeamThreads == kTile,
              "a team thread computes rows t + m * kTeamThreads (m < kSRPT); warp w of a team "
              "produces groups w + m * kTeamWarps of the canonical tile tree");
#ifndef LRB_ISSUERS
#define LRB_ISSUERS 2
#endif
constexpr int kIssuers = LRB_ISSUERS;             // producer warps (alternate stages)
// Two teams: issuer p fills exactly the stages team p consumes (G % kTeams ==
// p).  One team: the issuers alternate; the issuer of stage G waits for the
// slot's use G - ns, and its own previous stage (G - 2) needed G - 2 - ns
// consumed, so G - 2 ns was consumed before (one team consumes in order): the
// parity wait is never a stale phase.
static_assert(kIssuers == 1 || kIssuers == 2, "one or two issuer warps");
// One CTA per SM; 19 warps put 5 on some SM sub-partitions, so a thread
// gets at most 96 registers (16384 per sub-partition).
#define LRB_STREAM_BOUNDS __launch_bounds__(kStreamThreads, 1)
// + one reducer warp: sums each stage's tile partials in stage order (the
// CTA's reduction lane, kernels.cuh) off the consumers' path
constexpr int kReducer = kConsumers + 32 * kIssuers;
constexpr int kStreamThreads = kReducer + 32;
#ifndef LRB_MAX_STAGES
#define LRB_MAX_STAGES (kTile <= 256 ? 6 : 4)
#endif
constexpr int kStreamMaxStages = LRB_MAX_STAGES;
constexpr int kSlotRing = 8;                      // group-sum slots (a power of two)
static_assert((kSlotRing & (kSlotRing - 1)) == 0, "group-sum ring is a power of two");
constexpr int kSlotNR = 4;                        // reductions a group-sum slot holds

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
// try_wait with a suspend-time hint: a waiting warp is parked by the
// hardware until the phase completes (or the hint expires) instead of
// spinning through issue slots the working warps need.
#ifndef LRB_WAIT_HINT_NS
#define LRB_WAIT_HINT_NS 1000000
#endif
template <bool HINT = true>
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, unsigned parity) {
  uint32_t ok;
  if constexpr (HINT && LRB_WAIT_HINT_NS > 0) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "n"(LRB_WAIT_HINT_NS)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
  return ok != 0;
}
// Spin on an mbarrier phase.  A ring that never completes is a bug, not a
// slow peer: after timeout_ns the kernel traps (a clean launch error instead
// of a hung device).
// BACKOFF_NS > 0: sleep between polls (warps whose wake-up latency is not on
// the critical path, so their polling does not take issue slots from the
// consumers on the same SM sub-partition).
template <bool HINT = true, int BACKOFF_NS = 0>
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity, long long timeout_ns) {
  if (mbar_try_wait<HINT>(b, parity)) return;
  const long long t0 = global_ns();
  for (unsigned k = 1;; ++k) {
    if constexpr (BACKOFF_NS > 0) __nanosleep(BACKOFF_NS);
    if (mbar_try_wait<HINT>(b, parity)) return;
    if ((k & 15u) == 0 && global_ns() - t0 > timeout_ns) __trap();
  }
}
// Measured at C3 (profiles/r2_experiments.md): 64 ns for the issuers' slot
// waits and the reducer's parked waits takes phase A 137.3 -> 135.3 us.
#ifndef LRB_ISSUER_BACKOFF_NS
#define LRB_ISSUER_BACKOFF_NS 64
#endif
#ifndef LRB_REDUCER_BACKOFF_NS
#define LRB_REDUCER_BACKOFF_NS 64
#endif
// 1D bulk copy global -> shared (TMA engine), completes tx bytes on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a global range by the bulk-copy engine (no shared memory,
// no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
#ifndef LRB_DIAG_NOPLANE
#define LRB_DIAG_NOPLANE 0
#endif
#ifndef LRB_ISSUER_PREFETCH
#define LRB_ISSUER_PREFETCH 1
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
#ifndef LRB_NO_PROXY_FENCE   // diagnostics only (timing; unsafe ordering)
#define LRB_NO_PROXY_FENCE 0
#endif
__device__ __forceinline__ void fence_proxy_async_global() {
  if (!LRB_NO_PROXY_FENCE) asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Diagnostic counters per CTA (build with -DLRB_PROF=1; lrb_team_profile_counters):
// [phase kind (0 init, 1 A, 2 B, 3 C)][what]: 0 consumer thread 0 waiting for
// data, 1 end-of-phase consumer barrier, 2 issuer 0 waiting for a free stage,
// 3 team barrier (thread 0, arrival -> release), 4 thread 0 row bodies,
// 5 thread 0 group reduce + park, 6 thread 0 waiting for its group-sum slot,
// 7 issuer 0 issuing.
#ifndef LRB_PROF
#define LRB_PROF 0
#endif
constexpr bool kProf = LRB_PROF != 0;
constexpr int kCntPer = 8;
// + a timeline of the last phase A per CTA (globaltimer ns): entry, issuer
// past the proxy fence, issuer before / after its first stage's copies,
// consumers' first data, consumers done, reducer done, barrier exit
constexpr int kStamps = 8;
constexpr int kCnt = 4 * kCntPer + kStamps;

struct StreamSmem {
  char* stages;        // n_stages * stage_bytes
  uint64_t* full;      // [kStreamMaxStages][kTeams]
  uint64_t* empty;     // [kStreamMaxStages][kTeams]
  uint64_t* reduced;   // [kSlotRing] group-sum slot summed by the reducer (count 1)
  uint64_t* parked;    // [kSlotRing] group sums of the slot's stage parked (count kTeamWarps)
  double* wsum;        // [kSlotRing][kMaxPack][kGroups][kSlotNR] group sums awaiting their tile sum
  unsigned long long* cnt;   // [kCnt]
};

__device__ __forceinline__ StreamSmem stream_smem(const TeamDev& T) {
  extern __shared__ __align__(128) char dsm[];
  StreamSmem S;
  S.stages = dsm;
  char* tail = dsm + size_t(T.n_stages) * T.stage_bytes;
  S.full = reinterpret_cast<uint64_t*>(tail);
  S.empty = S.full + kStreamMaxStages * kTeams;
  S.reduced = S.empty + kStreamMaxStages * kTeams;
  S.parked = S.reduced + kSlotRing;
  S.wsum = reinterpret_cast<double*>(S.parked + kSlotRing);
  S.cnt = reinterpret_cast<unsigned long long*>(S.wsum + size_t(kSlotRing) * kMaxPack * kGroups * kSlotNR);
  return S;
}
__host__ __device__ constexpr size_t stream_smem_bytes(int stage_bytes, int n_stages) {
  return size_t(stage_bytes) * n_stages + 2 * kStreamMaxStages * kTeams * 8 + 2 * kSlotRing * 8 +
         size_t(kSlotRing) * kMaxPack * kGroups * kSlotNR * 8 + kCnt * 8;
}

__device__ __forceinline__ const PartDev& part_of(const TeamDev& T, int p, bool inl) {
  return inl ? T.lp[p - T.part_begin] : T.parts[p];
}

// What one phase stages: window vectors (SpMV phases) and whole-tile vectors.
struct Spec {
  int nwv;                 // window vectors (0: elementwise phase)
  int ntv;                 // tile vectors
  const double* wv[4];
  const double* tv[6];
  int npv;                 // SpMV phases: tile vectors the consumers load themselves,
  const double* pv[6];     //   pulled toward L2 when the tile's copies are issued
};


// Static stage sequence of a phase for this CTA: stage k holds unit
// cta + k * grid (a tile in SpMV phases, a chunk of K tiles in elementwise
// phases); the CTA's stage count.
__device__ __forceinline__ int stage_count(int64_t units) {
  return int64_t(blockIdx.x) < units ? int((units - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
}
// Ring position of the CTA's global stage number G (G = gseq + phase-local
// stage; identical in every thread).  Stage G lives in slot G % n_stages and
// belongs to consumer team (and issuer) G % kTeams.  Every (slot, team) pair
// has its own full/empty mbarriers: a pair recurs every L = lcm(n_stages,
// kTeams) stages, always for the same team, so each barrier is waited on in
// phase order by one team (consumers) or after its previous phase was seen
// (issuers) — a parity wait can never be satisfied by a stale phase, which a
// slot shared by two teams would allow.
struct RingPos {
  int slot;
  int team;
  int bar;           // slot * kTeams + team
  unsigned parity;   // parity of this use of the pair's barriers
};
// The ring's divisors as multiply-high magics (a runtime modulo costs ~20
// instructions and ring positions are taken once per stage per warp):
// q = umulhi(G, ceil(2^32 / d)) is exact for G * d < 2^32; stage numbers
// stay far below that (the host bounds max_iter), and larger G falls back.
struct Ring {
  int ns, L;
  unsigned mns, mL;
};
__device__ __forceinline__ Ring make_ring(int n_stages) {
  Ring R;
  R.ns = n_stages;
  R.L = (n_stages % kTeams) ? n_stages * kTeams : n_stages;
  R.mns = 0xFFFFFFFFu / unsigned(R.ns) + 1u;
  R.mL = 0xFFFFFFFFu / unsigned(R.L) + 1u;
  return R;
}
__device__ __forceinline__ RingPos ring_pos(int G, const Ring& R) {
  int qs, qL;
  if (G < (1 << 26)) {
    qs = int(__umulhi(unsigned(G), R.mns));
    qL = int(__umulhi(unsigned(G), R.mL));
  } else {
    qs = G / R.ns;
    qL = G / R.L;
  }
  const int slot = G - qs * R.ns, team = G & (kTeams - 1);
  return RingPos{slot, team, slot * kTeams + team, unsigned(qL & 1)};
}
// Group-sum slot of stage G: slot G % kSlotRing and the parity of this use of
// the slot's parked / reduced barriers.  Consumers refill a slot only after
// the reducer freed its previous use, and the reducer waits on `parked` (not
// on the ring's empty barriers), so neither side can see a stale phase.
struct WPos {
  int slot;
  unsigned parity;
};
__device__ __forceinline__ WPos wsum_pos(int G) {
  return WPos{G % kSlotRing, unsigned((G / kSlotRing) & 1)};
}
// First phase-local stage k of this CTA with (gseq + k) % m == r.
__device__ __forceinline__ int first_stage(int gseq, int r, int m) {
  return ((r - gseq) % m + m) % m;
}
// Issuer side: before filling stage G, wait until the previous stage in the
// same slot (G - n_stages, possibly of an earlier phase) was released.
__device__ __forceinline__ void wait_slot_free(const StreamSmem& S, int G, const Ring& R, long long timeout_ns) {
  const int Gp = G - R.ns;
  if (Gp < 0) return;
  const RingPos pp = ring_pos(Gp, R);
  mbar_wait<true, LRB_ISSUER_BACKOFF_NS>(S.empty + pp.bar, pp.parity, timeout_ns);
}

// ---------------------------------------------------------------------------
// Producers
// ---------------------------------------------------------------------------
struct HdrAddr {   // the header fields a producer needs
  int64_t row0, e0;
  int64_t wa[kMaxWin];
  int32_t wl[kMaxWin], woff[kMaxWin];
  int32_t rows, part, nw, wtot, tma, vbytes;
};
__device__ __forceinline__ void load_hdr_addr(const StageHdr* h, HdrAddr& a) {
  a.row0 = __ldg(&h->row0);
  a.e0 = __ldg(&h->e0);
#pragma unroll
  for (int w = 0; w < kMaxWin; ++w) {
    a.wa[w] = __ldg(&h->wa[w]);
    a.wl[w] = __ldg(&h->wl[w]);
    a.woff[w] = __ldg(&h->woff[w]);
  }
  a.rows = __ldg(&h->rows);
  a.part = __ldg(&h->part);
  a.nw = __ldg(&h->nw);
  a.wtot = __ldg(&h->wtot);
  a.tma = __ldg(&h->tma);
  a.vbytes = __ldg(&h->vbytes);
}

#ifndef LRB_PF_DIST
#define LRB_PF_DIST 1
#endif
struct PfAddr {
  int64_t e0;
  int32_t vbytes, part, tma;
};
__device__ __forceinline__ void load_pf_addr(const StageHdr* h, PfAddr& a) {
  a.e0 = __ldg(&h->e0);
  a.vbytes = __ldg(&h->vbytes);
  a.part = __ldg(&h->part);
  a.tma = __ldg(&h->tma);
}

// Header of each issuer's first stage of the coming SpMV phase, loaded by
// the issuer before the preceding barrier (prefetch_next_spmv) so the phase's
// first copies are issued without a global-memory round trip.  Tag: the
// global stage index it belongs to (-1: none).  Only the issuer lane touches
// its entry.
static __shared__ HdrAddr s_hdr[kIssuers];
static __shared__ int s_hdr_g[kIssuers];

// SpMV phases: issuer pw issues stages k = pw, pw + kIssuers, ... (tile
// cta + k * grid), reading each tile's header one of its stages ahead.
template <bool INL, class SpecF>
__device__ __forceinline__ void produce_spmv(const TeamDev& T, const StreamSmem& S, int gseq, int kind,
                                             SpecF&& spec_of) {
  const int pw = (int(threadIdx.x) - kConsumers) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  const uint64_t pol_stream = policy_evict_first();   // values: read once per phase
  const uint64_t pol_vec = policy_evict_normal();     // vectors: re-read by neighbour tiles
  const StageHdr* hdrs = reinterpret_cast<const StageHdr*>(T.tile_hdr);
  const TileRec* recs = reinterpret_cast<const TileRec*>(T.tile_rec);
  const int64_t G = gridDim.x;
  const int count = stage_count(T.n_tiles);
  const Ring R = make_ring(T.n_stages);
  HdrAddr cur{}, nxt{};
  const int k0 = first_stage(gseq, pw, kIssuers);
  if (k0 < count) {
    if (s_hdr_g[pw] == gseq + k0)
      cur = s_hdr[pw];
    else
      load_hdr_addr(hdrs + blockIdx.x + k0 * G, cur);
  }
  // Deep L2 prefetch of the values LRB_PF_DIST of this issuer's tiles ahead
  // (the TMA ring holds ~1 stage in flight per SM; L2 prefetches need no
  // shared memory).  pf = the header fields of the tile prefetched next.
  constexpr int kPf = LRB_PF_DIST;
  PfAddr pf{};
  if (kPf > 1) {
#pragma unroll
    for (int j = 1; j < kPf; ++j) {
      const int kj = k0 + j * kIssuers;
      if (kj < count) {
        PfAddr a;
        load_pf_addr(hdrs + blockIdx.x + int64_t(kj) * G, a);
        if (a.tma) bulk_prefetch_l2(part_of(T, a.part, INL).val + a.e0, unsigned(a.vbytes));
      }
    }
    if (k0 + kPf * kIssuers < count) load_pf_addr(hdrs + blockIdx.x + int64_t(k0 + kPf * kIssuers) * G, pf);
  }
  for (int k = k0; k < count; k += kIssuers) {
    const int64_t tile = blockIdx.x + k * G;
    const RingPos rp = ring_pos(gseq + k, R);
    char* st = S.stages + size_t(rp.slot) * T.stage_bytes;
    uint64_t* full = S.full + rp.bar;
    const bool tl = kProf && T.prof_cta && kind == 1 && k == k0 && pw == 0;   // timeline stamps
    if (tl) S.cnt[4 * kCntPer + 2] = (unsigned long long)global_ns();
    {
      const long long c0 = (kProf && T.prof_cta && pw == 0) ? clock64() : 0;
      wait_slot_free(S, gseq + k, R, T.timeout_ns);
      if (kProf && T.prof_cta && pw == 0) S.cnt[kind * kCntPer + 2] += clock64() - c0;
    }
    const long long ci = (kProf && T.prof_cta && pw == 0) ? clock64() : 0;
    const PartDev& P = part_of(T, cur.part, INL);
    const Spec sp = spec_of(P);
    const unsigned vec_bytes = unsigned((cur.rows * 8 + 15) & ~15);
    if (!cur.tma) {
      mbar_expect_tx(full, kHdrBytes);
      bulk_g2s(st, hdrs + tile, kHdrBytes, full, pol_vec);
    } else {
      // record (header | slot tables | masks), values, windows, tile vectors
#if LRB_DIAG_NOPLANE   // diagnostics (timing only, wrong results): no +-plane windows
      const bool skip_pl = cur.nw == 3;
      mbar_expect_tx(full, kRecBytes + unsigned(cur.vbytes) +
                               unsigned(sp.nwv * (skip_pl ? cur.wl[1] : cur.wtot) * 8) +
                               unsigned(sp.ntv) * vec_bytes);
#else
      constexpr bool skip_pl = false;
      mbar_expect_tx(full, kRecBytes + unsigned(cur.vbytes) + unsigned(sp.nwv * cur.wtot * 8) +
                               unsigned(sp.ntv) * vec_bytes);
#endif
      bulk_g2s(st, recs + tile, kRecBytes, full, pol_vec);
      char* d = st + kRecBytes;
      bulk_g2s(d, P.val + cur.e0, unsigned(cur.vbytes), full, pol_stream);
      d += cur.vbytes;
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int w = 0; w < kMaxWin; ++w)
          if (v < sp.nwv && w < cur.nw && !(skip_pl && w != 1))
            bulk_g2s(d + (size_t(v) * cur.wtot + cur.woff[w]) * 8, sp.wv[v] + cur.wa[w],
                     unsigned(cur.wl[w] * 8), full, pol_vec);
      d += size_t(sp.nwv) * cur.wtot * 8;
#pragma unroll
      for (int v = 0; v < 6; ++v)
        if (v < sp.ntv) bulk_g2s(d + size_t(v) * kVecTileBytes, sp.tv[v] + cur.row0, vec_bytes, full, pol_vec);
#pragma unroll
      for (int v = 0; v < 6; ++v)
        if (v < sp.npv) bulk_prefetch_l2(sp.pv[v] + cur.row0, vec_bytes);
    }
    if (kProf && T.prof_cta && pw == 0) S.cnt[kind * kCntPer + 7] += clock64() - ci;
    if (tl) S.cnt[4 * kCntPer + 3] = (unsigned long long)global_ns();
    // this issuer's next tile: its header, and its values and operand windows
    // toward L2 while this issuer waits for its next slot (the copies then
    // hit L2).  After the issue, so a phase's first copies never wait on it.
    if (k + kIssuers < count) load_hdr_addr(hdrs + tile + kIssuers * G, nxt);
    if (kPf > 1 && k + kPf * kIssuers < count) {
      if (pf.tma) bulk_prefetch_l2(part_of(T, pf.part, INL).val + pf.e0, unsigned(pf.vbytes));
      if (k + (kPf + 1) * kIssuers < count) load_pf_addr(hdrs + tile + int64_t(kPf + 1) * kIssuers * G, pf);
    }
    if (LRB_ISSUER_PREFETCH && k + kIssuers < count && nxt.tma) {
      const PartDev& Pn = part_of(T, nxt.part, INL);
      const Spec spn = spec_of(Pn);
      bulk_prefetch_l2(Pn.val + nxt.e0, unsigned(nxt.vbytes));
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int w = 0; w < kMaxWin; ++w)
          if (v < spn.nwv && w < nxt.nw) bulk_prefetch_l2(spn.wv[v] + nxt.wa[w], unsigned(nxt.wl[w] * 8));
#pragma unroll
      for (int v = 0; v < 6; ++v)
        if (v < spn.npv) bulk_prefetch_l2(spn.pv[v] + nxt.row0, unsigned((nxt.rows * 8 + 15) & ~15));
    }
    cur = nxt;
  }
}

// Cross-phase L2 prefetch (issuers, before the elementwise phase's barrier):
// the next phase is an SpMV phase over the same tiles (CG: A or the check C;
// BiCGStab: phase 1 or the check), and a tile's record and values do not
// depend on the barrier's results, so the CTA's first LRB_XPF tiles of it are
// pulled toward L2 while the barrier completes; the phase's first bulk copies
// then hit L2 instead of paying the DRAM latency at the phase start.
#ifndef LRB_XPF
#define LRB_XPF 3
#endif
template <bool INL>
__device__ __forceinline__ void prefetch_next_spmv(const TeamDev& T, int gnext) {
  if (LRB_XPF <= 0 || !T.tile_hdr) return;
  const int pw = (int(threadIdx.x) - kConsumers) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  const StageHdr* hdrs = reinterpret_cast<const StageHdr*>(T.tile_hdr);
  const TileRec* recs = reinterpret_cast<const TileRec*>(T.tile_rec);
  const int64_t G = gridDim.x;
  {   // this issuer's first header of the next phase (produce_spmv's cur)
    const int k0 = first_stage(gnext, pw, kIssuers);
    if (k0 < stage_count(T.n_tiles)) {
      load_hdr_addr(hdrs + blockIdx.x + int64_t(k0) * G, s_hdr[pw]);
      s_hdr_g[pw] = gnext + k0;
    }
  }
  for (int k = pw; k < LRB_XPF; k += kIssuers) {
    const int64_t tile = blockIdx.x + int64_t(k) * G;
    if (tile >= T.n_tiles) break;
    PfAddr a;
    load_pf_addr(hdrs + tile, a);
    if (!a.tma) continue;
    bulk_prefetch_l2(recs + tile, kRecBytes);
    bulk_prefetch_l2(part_of(T, a.part, INL).val + a.e0, unsigned(a.vbytes));
  }
}

// Elementwise phases: stage k holds chunk q = cta + k * grid = tiles
// [q * K, q * K + K) ∩ [0, n_tiles): the headers, then each vector's tiles
// (one copy per vector when the tiles belong to one part).
template <bool INL, class SpecF>
__device__ __forceinline__ void produce_elementwise(const TeamDev& T, const StreamSmem& S, int gseq,
                                                    int kind, SpecF&& spec_of) {
  const int pw = (int(threadIdx.x) - kConsumers) >> 5;
  if ((threadIdx.x & 31) != 0) return;
  const uint64_t pol_vec = policy_evict_normal();
  const StageHdr* hdrs = reinterpret_cast<const StageHdr*>(T.tile_hdr);
  const int64_t n_tiles = T.n_tiles;
  const bool one_part = T.part_end - T.part_begin == 1;
  const int ntv = spec_of(part_of(T, T.part_begin, INL)).ntv;
  const int K = pack_factor(T, ntv);
  const int count = stage_count((n_tiles + K - 1) / K);
  const Ring R = make_ring(T.n_stages);
  for (int k = first_stage(gseq, pw, kIssuers); k < count; k += kIssuers) {
    const int64_t c0 = (int64_t(blockIdx.x) + int64_t(k) * gridDim.x) * K;
    const RingPos rp = ring_pos(gseq + k, R);
    char* st = S.stages + size_t(rp.slot) * T.stage_bytes;
    uint64_t* full = S.full + rp.bar;
    {
      const long long t0 = (kProf && T.prof_cta && pw == 0) ? clock64() : 0;
      wait_slot_free(S, gseq + k, R, T.timeout_ns);
      if (kProf && T.prof_cta && pw == 0) S.cnt[kind * kCntPer + 2] += clock64() - t0;
    }
    const long long ci = (kProf && T.prof_cta && pw == 0) ? clock64() : 0;
    const int cnt = int(n_tiles - c0 < K ? n_tiles - c0 : K);
    int part[kMaxPack], rows[kMaxPack];
    int64_t row0[kMaxPack];
    unsigned bytes = unsigned(cnt) * kHdrBytes;
#pragma unroll
    for (int j = 0; j < kMaxPack; ++j) {
      part[j] = T.part_begin;
      rows[j] = 0;
      row0[j] = 0;
      if (j < cnt) {
        const int64_t tile = c0 + j;
        part[j] = one_part ? T.part_begin : __ldg(T.tile_part + tile);
        const PartDev& P = part_of(T, part[j], INL);
        row0[j] = (tile - P.tile0) * kTile;
        rows[j] = int(P.n - row0[j] < kTile ? P.n - row0[j] : int64_t(kTile));
      }
    }
    const bool merged = part[0] == part[cnt - 1];
    const unsigned span = unsigned(((row0[cnt - 1] + rows[cnt - 1] - row0[0]) * 8 + 15) & ~int64_t(15));
    if (merged)
      bytes += unsigned(ntv) * span;
    else
      for (int j = 0; j < cnt; ++j) bytes += unsigned(ntv) * unsigned((rows[j] * 8 + 15) & ~15);
    mbar_expect_tx(full, bytes);
    bulk_g2s(st, hdrs + c0, unsigned(cnt) * kHdrBytes, full, pol_vec);
    char* vbase = st + size_t(cnt) * kHdrBytes;
    const size_t vstride = size_t(cnt) * kVecTileBytes;
    if (merged) {
      const Spec sp = spec_of(part_of(T, part[0], INL));
#pragma unroll
      for (int v = 0; v < 6; ++v)
        if (v < sp.ntv) bulk_g2s(vbase + v * vstride, sp.tv[v] + row0[0], span, full, pol_vec);
    } else {
#pragma unroll
      for (int j = 0; j < kMaxPack; ++j) {
        if (j < cnt) {
          const Spec sp = spec_of(part_of(T, part[j], INL));
          const unsigned vb = unsigned((rows[j] * 8 + 15) & ~15);
#pragma unroll
          for (int v = 0; v < 6; ++v)
            if (v < sp.ntv)
              bulk_g2s(vbase + v * vstride + size_t(j) * kVecTileBytes, sp.tv[v] + row0[j], vb, full, pol_vec);
        }
      }
    }
    if (kProf && T.prof_cta && pw == 0) S.cnt[kind * kCntPer + 7] += clock64() - ci;
  }
}

// ---------------------------------------------------------------------------
// Consumers: staged row products
// ---------------------------------------------------------------------------
// Staged operands.  Every SpMV phase reads its operand at staged window
// position q through one of these (reference rounding, no FMA):
//   Win1   x = w0[q]
//   PnewCG p_new = z + beta * p_old            (w0 = z, w1 = p_old; BiCGStab: r + beta * u)
//   SBiCG  s = r - alpha * v                   (w0 = r, w1 = v)
struct Win1 {
  const double* __restrict__ w0;
  __device__ __forceinline__ double operator()(int q) const { return w0[q]; }
};
struct PnewCG {
  const double* __restrict__ w0;
  const double* __restrict__ w1;
  double beta;
  __device__ __forceinline__ double operator()(int q) const { return __dadd_rn(w0[q], __dmul_rn(beta, w1[q])); }
};
struct SBiCG {
  const double* __restrict__ w0;
  const double* __restrict__ w1;
  double alpha;
  __device__ __forceinline__ double operator()(int q) const { return __dsub_rn(w0[q], __dmul_rn(alpha, w1[q])); }
};

// Single-reduction PCG operand: u_new = dinv * (r - alpha * (w + beta * s_old))
// (w0 = r, w1 = dinv, w2 = w, w3 = s_old; first iteration: s = w).
struct UCG1 {
  const double* __restrict__ w0;
  const double* __restrict__ w1;
  const double* __restrict__ w2;
  const double* __restrict__ w3;
  double alpha, beta;
  bool first;
  __device__ __forceinline__ double s(int q) const {
    return first ? w2[q] : __dadd_rn(w2[q], __dmul_rn(beta, w3[q]));
  }
  __device__ __forceinline__ double operator()(int q) const {
    return __dmul_rn(w1[q], __dsub_rn(w0[q], __dmul_rn(alpha, s(q))));
  }
};

// Slot table of a slice in the staged StageTab (SoA): for slot k the column
// offset off[k] (col - row) and the shared-memory delta del[k] such that row
// i's operand sits at staged index i + del[k].
struct Slots {
  const int32_t* off;
  const int32_t* del;
};
__device__ __forceinline__ Slots slice_slots(const char* st, const StageHdr& H, int sl) {
  const int32_t* tab = reinterpret_cast<const int32_t*>(st + kHdrBytes);
  const int p = H.spat[sl];
  return Slots{tab + p * kPatW, tab + (kHdrPats + p) * kPatW};
}
// Slot of the diagonal (offset 0) of a slice's pattern; staged index of row
// i's own operand.
__device__ __forceinline__ int diag_slot(const StageHdr& H, int sl) { return H.sdiag[H.spat[sl]]; }
__device__ __forceinline__ int diag_pos(const StageHdr& H, const Slots& slot, int sl, int64_t i) {
  return int(i) + slot.del[diag_slot(H, sl)];
}

#ifndef LRB_FASTPATH
#define LRB_FASTPATH 0
#endif
#ifndef LRB_ABENCH      // diagnostics: run phase A LRB_ABENCH times, nothing else
#define LRB_ABENCH 0
#endif
#ifndef LRB_NOCOMPUTE   // diagnostics: SpMV consumers skip the row bodies
#define LRB_NOCOMPUTE 0
#endif
// Fixed-width row product: WM pattern slots, all operand loads issued
// before the accumulation chain.  MASK: slots k >= w and holes get a zero
// operand (a hole's value is a finite 0.0 in the SELL layout, so acc + a * 0
// leaves acc unchanged — acc is never -0.0); !MASK: the whole warp's rows
// are fully occupied (w == WM), no selects.  xd = the operand of slot dk
// (the diagonal's, for the phase's own-row update) from the same registers.
template <int WM, bool MASK, class XS>
__device__ __forceinline__ double row_fixed(int w, int ii, int eb, unsigned msk, const int32_t* __restrict__ del,
                                            int dk, const double* __restrict__ sval, const XS& xs, double& xd) {
  constexpr int kQ = (WM + 3) / 4;
  int d[4 * kQ];
#pragma unroll
  for (int q = 0; q < kQ; ++q) {
    const int4 v = reinterpret_cast<const int4*>(del)[q];
    d[4 * q] = v.x;
    d[4 * q + 1] = v.y;
    d[4 * q + 2] = v.z;
    d[4 * q + 3] = v.w;
  }
  double a[WM], x[WM];
#pragma unroll
  for (int k = 0; k < WM; ++k) {
    if constexpr (MASK) {
      const bool on = k < w && ((msk >> k) & 1u);
      a[k] = k < w ? sval[eb + k * kSlice] : 0.0;
      x[k] = on ? xs(ii + d[k]) : 0.0;
    } else {
      a[k] = sval[eb + k * kSlice];
      x[k] = xs(ii + d[k]);
    }
  }
  xd = x[0];
#pragma unroll
  for (int k = 1; k < WM; ++k)
    if (k == dk) xd = x[k];
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < WM; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], x[k]));
  return acc;
}

// The halo mirror of part P seen as a part whose mirrored vectors have one
// element per halo slot (operand lambdas index it with the slot).
__device__ __forceinline__ PartDev mirror_of(const PartDev& P) {
  PartDev M;
  const int64_t h = P.n_halo;
  M.x = P.hm + kMx * h;
  M.r = P.hm + kMr * h;
  M.p0 = P.hm + kMp0 * h;
  M.p1 = P.hm + kMp1 * h;
  M.s = P.hm + kMs * h;
  M.v0 = P.hm + kMv0 * h;
  M.v1 = P.hm + kMv1 * h;
  return M;
}

// Staged SpMV of tile row lr (its 32-row slice is warp-uniform; every lane
// of the warp calls it); xs(q) is the staged operand, fh(owner part, row) a
// halo column's operand; xd receives the row's diagonal operand.
template <bool HALO, class XS, class FH>
__device__ __forceinline__ double row_spmv_staged(const int n, const int32_t* __restrict__ hpart,
                                                  const int32_t* __restrict__ hidx, const PartDev* mp,
                                                  const PartDev* __restrict__ parts, const StageHdr& H,
                                                  const Slots& slot, const double* __restrict__ sval,
                                                  const uint16_t* __restrict__ smask, int lr, const XS& xs,
                                                  FH&& fh, double& xd) {
  const int lane = threadIdx.x & 31;
  const int rows = H.rows;
  const int lr0 = lr & ~31;
  const int sl = lr0 >> 5;
  const int s0 = H.sp[sl];
  const int w = lr0 < rows ? (H.sp[sl + 1] - s0) >> 5 : 0;
  const int eb = s0 + lane;
  const int ii = int(H.row0) + lr;
  const unsigned msk = lr < rows ? unsigned(smask[lr]) : 0u;
  const int dk = diag_slot(H, sl);
  if constexpr (!HALO) {
    if (w == 7) {
      if (LRB_FASTPATH && __all_sync(0xffffffffu, msk == 0x7Fu))
        return row_fixed<7, false>(w, ii, eb, msk, slot.del, dk, sval, xs, xd);
      return row_fixed<7, true>(w, ii, eb, msk, slot.del, dk, sval, xs, xd);
    }
    if (w <= 8) return row_fixed<8, true>(w, ii, eb, msk, slot.del, dk, sval, xs, xd);
    return row_fixed<kPatW, true>(w, ii, eb, msk, slot.del, dk, sval, xs, xd);
  } else {
    double acc = 0.0;
    for (int k = 0; k < w; ++k) {
      const bool on = (msk >> k) & 1u;
      const double a = sval[eb + k * kSlice];
      const int c = ii + slot.off[k];
      double xv;
      if (on && c >= n) {
        // halo operand: from this part's mirror (pushed by the owner) or
        // straight from the owning part (peer memory)
        xv = mp ? fh(mirror_of(*mp), int64_t(c - n))
                : fh(parts[__ldg(hpart + (c - n))], int64_t(__ldg(hidx + (c - n))));
      } else {
        xv = xs(on ? ii + slot.del[k] : 0);
        xv = on ? xv : 0.0;
      }
      acc = __dadd_rn(acc, __dmul_rn(a, xv));
    }
    xd = dk >= 0 ? xs(ii + slot.del[dk]) : 0.0;
    return acc;
  }
}

// Staged pointers of an SpMV tile: values, masks, window vector v, tail vector.
struct StagedTile {
  const double* sval;
  const uint16_t* smask;
  const double* win;     // window vector 0; vector v at win + v * wtot
  int wtot;
  int nwv;
  const char* st;
  int vbytes;
  __device__ __forceinline__ const double* w(int v) const { return win + size_t(v) * wtot; }
  __device__ __forceinline__ const double* tail(int v) const {
    return reinterpret_cast<const double*>(st + kRecBytes + vbytes + size_t(nwv) * wtot * 8) + size_t(v) * kTile;
  }
};
__device__ __forceinline__ StagedTile staged_tile(const char* st, const StageHdr& H, int nwv) {
  StagedTile t;
  t.sval = reinterpret_cast<const double*>(st + kRecBytes);
  t.smask = reinterpret_cast<const uint16_t*>(st + kHdrBytes + kTabBytes);
  t.win = reinterpret_cast<const double*>(st + kRecBytes + H.vbytes);
  t.wtot = H.wtot;
  t.nwv = nwv;
  t.st = st;
  t.vbytes = H.vbytes;
  return t;
}
// Dispatch on whether the part has halo columns.  MIRROR: the kernel keeps
// the halo mirrors current (hpush on every write of a mirrored vector), so
// halo operands come from the part's own mirror when the team has them on.
template <bool MIRROR = false, class XS, class FH>
__device__ __forceinline__ double staged_row(const PartDev& P, const PartDev* __restrict__ parts,
                                             const StageHdr& H, const StagedTile& t, const Slots& slot, int lr,
                                             const XS& xs, FH&& fh, double& xd) {
  const int n = int(P.n);
  const PartDev* mp = (MIRROR && P.mir) ? &P : nullptr;
  // only tiles holding rows with halo columns take the per-entry halo test;
  // every other tile of a multi-part / multi-GPU part keeps the fixed-width path
  return (P.n_halo && H.halo)
             ? row_spmv_staged<true>(n, P.hpart, P.hidx, mp, parts, H, slot, t.sval, t.smask, lr, xs, fh, xd)
             : row_spmv_staged<false>(n, P.hpart, P.hidx, mp, parts, H, slot, t.sval, t.smask, lr, xs, fh, xd);
}
template <bool MIRROR = false, class XS, class FH>
__device__ __forceinline__ double staged_row(const PartDev& P, const PartDev* __restrict__ parts,
                                             const StageHdr& H, const StagedTile& t, const Slots& slot, int lr,
                                             const XS& xs, FH&& fh) {
  double xd;
  return staged_row<MIRROR>(P, parts, H, t, slot, lr, xs, fh, xd);
}

// Vectors of one packed elementwise tile: vector v at base + v * stride.
struct VecView {
  const char* base;
  size_t stride;
  __device__ __forceinline__ const double* operator[](int v) const {
    return reinterpret_cast<const double*>(base + v * stride);
  }
};

// ---------------------------------------------------------------------------
// Consumers: phase loop and deferred tile sums
// ---------------------------------------------------------------------------
// Team tm consumes stages k = tm, tm + 2, ...; per tile each thread computes
// rows t and t + kTPB (body(P, H, st, V, lr, acc)), butterfly-reduces each into
// its group (warp w of the team: groups w and w + 8) and parks the group sums
// in the stage's group-sum slot, then releases the stage.  No per-tile
// barrier and no tile sums here: the reducer warp sums the parked groups.
template <int NR, bool INL, bool ELEM, class Body>
__device__ __forceinline__ void consume_phase(const TeamDev& T, const StreamSmem& S, int gseq, int kind,
                                              int ntv, Body&& body) {
  static_assert(NR <= kSlotNR, "group-sum slots hold kSlotNR reductions");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = warp / kTeamWarps;             // team
  const int wt = warp - tm * kTeamWarps;        // warp within the team
  const int tt = int(threadIdx.x) - tm * kTeamThreads;
  const Ring R = make_ring(T.n_stages);
  const int64_t G = gridDim.x;
  const int K = ELEM ? pack_factor(T, ntv) : 1;
  const int64_t n_tiles = T.n_tiles;
  const int count = stage_count(ELEM ? (n_tiles + K - 1) / K : n_tiles);
  for (int k = first_stage(gseq, tm, kTeams); k < count; k += kTeams) {
    const int Gk = gseq + k;
    const RingPos rp = ring_pos(Gk, R);
    const char* st0 = S.stages + size_t(rp.slot) * T.stage_bytes;
    {
      const long long c0 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      mbar_wait(S.full + rp.bar, rp.parity, T.timeout_ns);
      if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 0] += clock64() - c0;
      if (kProf && T.prof_cta && threadIdx.x == 0 && !ELEM && kind == 1 && k == first_stage(gseq, tm, kTeams))
        S.cnt[4 * kCntPer + 4] = (unsigned long long)global_ns();
    }
    const WPos wp = wsum_pos(Gk);
    if (Gk >= kSlotRing) {   // the slot's previous stage must be summed
      const long long c2 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      mbar_wait(S.reduced + wp.slot, wp.parity ^ 1u, T.timeout_ns);
      if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 6] += clock64() - c2;
    }
    const int64_t t0 = (int64_t(blockIdx.x) + int64_t(k) * G) * K;
    const int cnt = int(n_tiles - t0 < K ? n_tiles - t0 : K);
    for (int j = 0; j < cnt; ++j) {
      // SpMV stages hold one tile at st0; packed elementwise stages hold cnt
      // headers, then each vector's cnt tiles (produce_elementwise)
      const char* st = ELEM ? st0 + size_t(j) * kHdrBytes : st0;
      const VecView V{ELEM ? st0 + size_t(cnt) * kHdrBytes + size_t(j) * kVecTileBytes : nullptr,
                      size_t(cnt) * kVecTileBytes};
      const StageHdr& H = *reinterpret_cast<const StageHdr*>(st);
      const PartDev& P = part_of(T, H.part, INL);
      double acc[kSRPT][NR];
      const long long c3 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
#pragma unroll
      for (int m = 0; m < kSRPT; ++m) {
#pragma unroll
        for (int q = 0; q < NR; ++q) acc[m][q] = 0.0;
        if (!(LRB_NOCOMPUTE && !ELEM)) body(P, H, st, V, tt + m * kTeamThreads, acc[m]);
      }
      const long long c4 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
      double* ws = S.wsum + size_t(wp.slot * kMaxPack + j) * kGroups * kSlotNR;
#pragma unroll
      for (int m = 0; m < kSRPT; ++m) {
        group_reduce<NR>(acc[m]);
        if (lane == 0)
#pragma unroll
          for (int q = 0; q < NR; ++q) ws[(m * kTeamWarps + wt) * kSlotNR + q] = acc[m][q];
      }
      if (kProf && T.prof_cta && threadIdx.x == 0) {
        const long long c5 = clock64();
        S.cnt[kind * kCntPer + 4] += c4 - c3;
        S.cnt[kind * kCntPer + 5] += c5 - c4;
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(S.parked + wp.slot);   // group sums written before both arrivals
      mbar_arrive(S.empty + rp.bar);
    }
  }
}

#ifndef LRB_REDUCER_HINT   // reducer waits without the suspend hint (prompt wake-up)
#define LRB_REDUCER_HINT 0
#endif
// Reducer warp: for every stage of the phase, in stage order, wait until its
// group sums are parked (8 warps arrive on the slot's `parked` barrier), add
// each tile's 16 group sums in group
// order (the canonical tile tree) and free the group-sum slot.  Lane q < NR
// owns reduction q and keeps the CTA's lane value: with T.lane_fast this CTA
// IS reduction lane blockIdx.x (kernels.cuh), and its tiles arrive in
// ascending order, so the running sum is that lane's value; otherwise the
// tile partials go to T.partials for the last CTA.
template <int NR, bool ELEM>
__device__ __forceinline__ void reduce_phase(const TeamDev& T, const StreamSmem& S, int gseq, int ntv) {
  const int lane = threadIdx.x & 31;
  const int K = ELEM ? pack_factor(T, ntv) : 1;
  const int64_t n_tiles = T.n_tiles;
  const int count = stage_count(ELEM ? (n_tiles + K - 1) / K : n_tiles);
  const bool fast = lanes_by_cta(T, n_tiles, K);   // single part: its tiles are the device's
  double lacc = 0.0;
  for (int k = 0; k < count; ++k) {
    const int Gk = gseq + k;
    const WPos wp = wsum_pos(Gk);
    mbar_wait<LRB_REDUCER_HINT, LRB_REDUCER_BACKOFF_NS>(S.parked + wp.slot, wp.parity, T.timeout_ns);
    const int64_t t0 = (int64_t(blockIdx.x) + int64_t(k) * gridDim.x) * K;
    const int cnt = int(n_tiles - t0 < K ? n_tiles - t0 : K);
    if (lane < NR) {
      for (int j = 0; j < cnt; ++j) {
        const double* w = S.wsum + (size_t(wp.slot * kMaxPack + j) * kGroups) * kSlotNR;
        double sum = w[lane];
#pragma unroll
        for (int g = 1; g < kGroups; ++g) sum = __dadd_rn(sum, w[g * kSlotNR + lane]);
        if (!fast) T.partials[lane * n_tiles + t0 + j] = sum;
        lacc = __dadd_rn(lacc, sum);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(S.reduced + wp.slot);
  }
  if (fast && lane < NR) lane_slots(T, s_flat_bar)[size_t(blockIdx.x) * kMaxRed + lane] = lacc;
}

__device__ __forceinline__ void stream_init(const TeamDev& T, const StreamSmem& S) {
  if (threadIdx.x == 0) {
    for (int b = 0; b < T.n_stages * kTeams; ++b) {
      mbar_init(S.full + b, 1);
      mbar_init(S.empty + b, kTeamWarps);
    }
    for (int b = 0; b < kSlotRing; ++b) {
      mbar_init(S.reduced + b, 1);
      mbar_init(S.parked + b, kTeamWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < kCnt) S.cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_flat_bar = 0;
  if (threadIdx.x < kIssuers) s_hdr_g[threadIdx.x] = -1;
  __syncthreads();
}

// Phase wrapper: issuers stream, consumer teams compute, then the team
// barrier with the fused reduction (all threads); gseq advances by the
// phase's stage count (identical in every thread).
template <int NR, bool INL, bool ELEM, bool PF_NEXT = false, class SpecF, class Body>
__device__ __forceinline__ void stream_phase(const TeamDev& T, const StreamSmem& S, int& gseq, double* red,
                                             int kind, SpecF&& spec_of, Body&& body) {
  const int ntv = ELEM ? spec_of(part_of(T, T.part_begin, INL)).ntv : 0;
  const bool stamp = kProf && T.prof_cta && !ELEM && kind == 1;   // timeline of phase A
  unsigned long long* const ts = S.cnt + 4 * kCntPer;
  if (stamp && threadIdx.x == 0) ts[0] = (unsigned long long)global_ns();
  if (threadIdx.x >= kReducer) {
    reduce_phase<NR, ELEM>(T, S, gseq, ntv);
    if (stamp && threadIdx.x == kReducer) ts[6] = (unsigned long long)global_ns();
  } else if (threadIdx.x >= kConsumers) {
    fence_proxy_async_global();   // peers' generic writes of the last phase -> our bulk reads
    if (stamp && threadIdx.x == kConsumers) ts[1] = (unsigned long long)global_ns();
    if constexpr (ELEM)
      produce_elementwise<INL>(T, S, gseq, kind, spec_of);
    else
      produce_spmv<INL>(T, S, gseq, kind, spec_of);
    if constexpr (PF_NEXT) {
      const int K = ELEM ? pack_factor(T, ntv) : 1;
      prefetch_next_spmv<INL>(T, gseq + stage_count(ELEM ? (T.n_tiles + K - 1) / K : T.n_tiles));
    }
  } else {
    consume_phase<NR, INL, ELEM>(T, S, gseq, kind, ntv, body);
    if (stamp && threadIdx.x == 0) ts[5] = (unsigned long long)global_ns();
  }
  fence_proxy_async_global();
  const long long c0 = (kProf && T.prof_cta && threadIdx.x == 0) ? clock64() : 0;
  const int K = ELEM ? pack_factor(T, ntv) : 1;
  // the ring is idle here (every stage of the phase was consumed): its shared
  // memory is the scratch of the multi-part barrier reduction
  team_sync<NR>(T, red, K, reinterpret_cast<double*>(S.stages));
  if (stamp && threadIdx.x == 0) ts[7] = (unsigned long long)global_ns();
  if (kProf && T.prof_cta && threadIdx.x == 0) S.cnt[kind * kCntPer + 3] += clock64() - c0;
  gseq += stage_count(ELEM ? (T.n_tiles + K - 1) / K : T.n_tiles);
}

// Diagnostics: this CTA's counters to T.prof_cta[blockIdx.x * kCnt ...].
__device__ __forceinline__ void stream_flush_counters(const TeamDev& T, const StreamSmem& S) {
  __syncthreads();
  if (kProf && T.prof_cta && threadIdx.x < kCnt)
    T.prof_cta[blockIdx.x * kCnt + threadIdx.x] = (long long)S.cnt[threadIdx.x];
}

// ---------------------------------------------------------------------------
// CG / Jacobi-PCG, streaming.  Phases and arithmetic are those of
// team_cg_kernel (kernels.cuh): A = {p_new, q = A p_new, p.q},
// B = {x, r update, r.r (r.z)}, C = {|b - A x|^2}.
// ---------------------------------------------------------------------------
template <bool JAC, bool INL>
__global__ void LRB_STREAM_BOUNDS
    team_cg_stream_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  const StreamSmem S = stream_smem(T);
  stream_init(T, S);
  int gseq = 0;
  double red[2];
  // ---- phase 0: x = 0, r = b, (z = dinv*b), b.b (, b.z)
  stream_phase<2, INL, true, true>(
      T, S, gseq, red, 0,
      [&](const PartDev& P) {
        return Spec{0, JAC ? 2 : 1, {nullptr, nullptr}, {P.b, JAC ? P.dinv : nullptr}};
      },
      [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[2]) {
        if (lr >= H.rows) return;
        const int64_t i = H.row0 + lr;
        const double b = V[0][lr];
        P.x[i] = 0.0;
        P.r[i] = b;
        hpush(P, parts, kMx, i, 0.0);
        if (!JAC) hpush(P, parts, kMr, i, b);
        acc[0] = __dadd_rn(acc[0], __dmul_rn(b, b));
        if (JAC) {
          const double z = __dmul_rn(V[1][lr], b);
          P.s[i] = z;
          hpush(P, parts, kMs, i, z);
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
  int pa = 0;
  bool first = true, converged = false;
  // lazy x (LRB_LAZY_X): phase B leaves x += step * p pending; the next
  // phase A applies it to its own rows (it stages p_old anyway), phase C
  // forms x + step * p on the fly, a last elementwise pass applies it at exit.
  // Same operations, same rounding as updating x in B: 8 B/row less traffic.
  bool pend = false;
  double step_x = 0.0;
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
        T, S, gseq, red, 1,
        [&](const PartDev& P) {
          const double* z = JAC ? P.s : P.r;
          const double* po = pa ? P.p1 : P.p0;
          return first ? Spec{1, 0, {z, nullptr}, {}}
                       : (pend ? Spec{2, 1, {z, po}, {P.x}} : Spec{2, 0, {z, po}, {}});
        },
        [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[1]) {
          double* pout = pa ? P.p0 : P.p1;
          if (H.tma) {
            const StagedTile t = staged_tile(st, H, first ? 1 : 2);
            const int sl = lr >> 5;
            const Slots slot = slice_slots(st, H, sl);
            const PnewCG pn{t.w(0), t.w(1), beta};
            const Win1 z1{t.w(0)};
            double pi;   // p_new of the row itself: the diagonal slot's operand
            const double qi = first ? staged_row<true>(P, parts, H, t, slot, lr, z1, pnew_g, pi)
                                    : staged_row<true>(P, parts, H, t, slot, lr, pn, pnew_g, pi);
            if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              pout[i] = pi;
              hpush(P, parts, pa ? kMp0 : kMp1, i, pi);
              P.q[i] = qi;
              acc[0] = __dadd_rn(acc[0], __dmul_rn(pi, qi));
              if (pend) {   // the pending x update: p_old of the row itself
                const double po = t.w(1)[diag_pos(H, slot, sl, i)];
                const double xn = __dadd_rn(t.tail(0)[lr], __dmul_rn(step_x, po));
                P.x[i] = xn;
                hpush(P, parts, kMx, i, xn);
              }
            }
          } else if (lr < H.rows) {
            const int64_t i = H.row0 + lr;
            const double pi = pnew_g(P, i);
            const double qi = row_spmv(P, parts, i, pnew_g);
            pout[i] = pi;
            hpush(P, parts, pa ? kMp0 : kMp1, i, pi);
            P.q[i] = qi;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(pi, qi));
            if (pend) {
              const double xn = __dadd_rn(P.x[i], __dmul_rn(step_x, (pa ? P.p1 : P.p0)[i]));
              P.x[i] = xn;
              hpush(P, parts, kMx, i, xn);
            }
          }
        });
    pend = false;
    if (team_failed(T)) break;
#if LRB_ABENCH
    // diagnostics build: phase A alone, back to back (timing only)
    first = false;
    beta = 0.5;
    pa ^= 1;
    if (it >= LRB_ABENCH) break;
    continue;
#endif
    const double pq = red[0];
    if (pq <= 0.0) {
      if (lead) team_fail(T, LRB_ENOTPD);
      break;
    }
    const double step = rho / pq;
    pa ^= 1;
#if LRB_LAZY_X
    // ---- phase B: r -= step q, r.r (, z = dinv r, r.z); x += step p pending
    stream_phase<2, INL, true, true>(
        T, S, gseq, red, 2,
        [&](const PartDev& P) {
          return Spec{0, kCgBVecs<JAC>, {nullptr, nullptr}, {P.r, P.q, JAC ? P.dinv : nullptr}};
        },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[2]) {
          if (lr >= H.rows) return;
          const int64_t i = H.row0 + lr;
          const double r = __dsub_rn(V[0][lr], __dmul_rn(step, V[1][lr]));
          P.r[i] = r;
          if (!JAC) hpush(P, parts, kMr, i, r);
          acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
          if (JAC) {
            const double z = __dmul_rn(V[2][lr], r);
            P.s[i] = z;
            hpush(P, parts, kMs, i, z);
            acc[1] = __dadd_rn(acc[1], __dmul_rn(r, z));
          }
        });
    pend = true;
    step_x = step;
#else
    // ---- phase B: x += step p, r -= step q, r.r (, r.z)
    stream_phase<2, INL, true, true>(
        T, S, gseq, red, 2,
        [&](const PartDev& P) {
          return Spec{0, kCgBVecs<JAC>, {nullptr, nullptr},
                      {pa ? P.p1 : P.p0, P.x, P.r, P.q, JAC ? P.dinv : nullptr}};
        },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[2]) {
          if (lr >= H.rows) return;
          const int64_t i = H.row0 + lr;
          const double x = __dadd_rn(V[1][lr], __dmul_rn(step, V[0][lr]));
          const double r = __dsub_rn(V[2][lr], __dmul_rn(step, V[3][lr]));
          P.x[i] = x;
          P.r[i] = r;
          hpush(P, parts, kMx, i, x);
          if (!JAC) hpush(P, parts, kMr, i, r);
          acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
          if (JAC) {
            const double z = __dmul_rn(V[4][lr], r);
            P.s[i] = z;
            hpush(P, parts, kMs, i, z);
            acc[1] = __dadd_rn(acc[1], __dmul_rn(r, z));
          }
        });
#endif
    if (team_failed(T)) break;
    const double rr_new = red[0];
    const double rho_new = JAC ? red[1] : rr_new;
    const double rec = sqrt(rr_new) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      // ---- phase C: true residual |b - A x| (x with its pending update formed
      //      on the fly: x is read by neighbours here, so it is not written)
      auto xg = [&](const PartDev& Q, int64_t j) -> double {
        return pend ? __dadd_rn(Q.x[j], __dmul_rn(step_x, (pa ? Q.p1 : Q.p0)[j])) : Q.x[j];
      };
      stream_phase<1, INL, false>(
          T, S, gseq, red, 3,
          [&](const PartDev& P) {
            return pend ? Spec{2, 1, {P.x, pa ? P.p1 : P.p0}, {P.b}} : Spec{1, 1, {P.x, nullptr}, {P.b}};
          },
          [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr,
              double (&acc)[1]) {
            if (H.tma) {
              const StagedTile t = staged_tile(st, H, pend ? 2 : 1);
              const Slots slot = slice_slots(st, H, lr >> 5);
              const double ax = pend ? staged_row<true>(P, parts, H, t, slot, lr, PnewCG{t.w(0), t.w(1), step_x}, xg)
                                     : staged_row<true>(P, parts, H, t, slot, lr, Win1{t.w(0)}, xg);
              if (lr < H.rows) {
                const double d = __dsub_rn(t.tail(0)[lr], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            } else if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              const double ax = row_spmv(P, parts, i, xg);
              const double d = __dsub_rn(P.b[i], ax);
              acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
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
  if (pend && !team_failed(T)) {
    // ---- the last pending x update (x is the solver's output)
    stream_phase<1, INL, true>(
        T, S, gseq, red, 2,
        [&](const PartDev& P) { return Spec{0, 2, {nullptr, nullptr}, {P.x, pa ? P.p1 : P.p0}}; },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&)[1]) {
          if (lr >= H.rows) return;
          P.x[H.row0 + lr] = __dadd_rn(V[0][lr], __dmul_rn(step_x, V[1][lr]));
        });
  }
  stream_flush_counters(T, S);
  if (lead) {
    out->iterations = it > T.max_iter ? T.max_iter : it;
    out->converged = converged ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

// ---------------------------------------------------------------------------
// BiCGStab, streaming (momentum; phases and arithmetic of team_bicgstab_kernel,
// kernels.cuh).  1: p_new = r + beta (p_old - omega v_old) on the fly (three
// staged windows), v = A p_new, rhat.v;  2: s = r - alpha v on the fly, t =
// A s, t.s, t.t;  3: x = (x + alpha p) + omega s, r = s - omega t, r.r,
// rhat.r;  check: |b - A x|^2.  p and v are double-buffered.
// ---------------------------------------------------------------------------
template <bool INL>
__global__ void LRB_STREAM_BOUNDS
    team_bicgstab_stream_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  const StreamSmem S = stream_smem(T);
  stream_init(T, S);
  int gseq = 0;
  double red[2];
  stream_phase<1, INL, true, true>(
      T, S, gseq, red, 0, [&](const PartDev& P) { return Spec{0, 1, {nullptr, nullptr}, {P.b}}; },
      [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[1]) {
        if (lr >= H.rows) return;
        const int64_t i = H.row0 + lr;
        const double b = V[0][lr];
        P.x[i] = 0.0;
        P.r[i] = b;
        P.rhat[i] = b;
        hpush(P, parts, kMx, i, 0.0);
        hpush(P, parts, kMr, i, b);
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
  int pa = 0;   // p_old/v_old in p0/v0 when pa == 0
  bool converged = false, breakdown = false;
  int it = 0;
  for (it = 1; it <= T.max_iter; ++it) {
    const bool first = (it == 1);
    if (!first) beta = __dmul_rn(rho / rho_prev, alpha / omega);
    // ---- phase 1: p_new, v = A p_new, rhat.v
    // u = p_old - omega v_old was stored over p_old by the previous phase 3
    // (same rounding as forming it here), so p_new needs two windows, not three
    auto pnew_g = [&](const PartDev& Q, int64_t j) -> double {
      const double r = Q.r[j];
      if (first) return r;
      const double u = pa ? Q.p1[j] : Q.p0[j];
      return __dadd_rn(r, __dmul_rn(beta, u));
    };
    stream_phase<1, INL, false>(
        T, S, gseq, red, 1,
        [&](const PartDev& P) {
          return first ? Spec{1, 1, {P.r, nullptr}, {P.rhat}}
                       : Spec{2, 1, {P.r, pa ? P.p1 : P.p0}, {P.rhat}};
        },
        [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[1]) {
          double* pout = pa ? P.p0 : P.p1;
          double* vout = pa ? P.v0 : P.v1;
          if (H.tma) {
            const StagedTile t = staged_tile(st, H, first ? 1 : 2);
            const int sl = lr >> 5;
            const Slots slot = slice_slots(st, H, sl);
            const Win1 r1{t.w(0)};
            const PnewCG pn{t.w(0), t.w(1), beta};   // r + beta u
            double pi;
            const double vi = first ? staged_row<true>(P, parts, H, t, slot, lr, r1, pnew_g, pi)
                                    : staged_row<true>(P, parts, H, t, slot, lr, pn, pnew_g, pi);
            if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              pout[i] = pi;
              vout[i] = vi;
              hpush(P, parts, pa ? kMp0 : kMp1, i, pi);
              hpush(P, parts, pa ? kMv0 : kMv1, i, vi);
              acc[0] = __dadd_rn(acc[0], __dmul_rn(t.tail(0)[lr], vi));
            }
          } else if (lr < H.rows) {
            const int64_t i = H.row0 + lr;
            const double pi = pnew_g(P, i);
            const double vi = row_spmv(P, parts, i, pnew_g);
            pout[i] = pi;
            vout[i] = vi;
            hpush(P, parts, pa ? kMp0 : kMp1, i, pi);
            hpush(P, parts, pa ? kMv0 : kMv1, i, vi);
            acc[0] = __dadd_rn(acc[0], __dmul_rn(P.rhat[i], vi));
          }
        });
    if (team_failed(T)) break;
    pa ^= 1;
    const double rv = red[0];
    if (rv == 0.0) {
      breakdown = true;
      break;
    }
    alpha = rho / rv;
    // ---- phase 2: s = r - alpha v, t = A s, t.s, t.t
    auto sval_g = [&](const PartDev& Q, int64_t j) -> double {
      const double v = pa ? Q.v1[j] : Q.v0[j];
      return __dsub_rn(Q.r[j], __dmul_rn(alpha, v));
    };
    stream_phase<2, INL, false>(
        T, S, gseq, red, 1, [&](const PartDev& P) { return Spec{2, 0, {P.r, pa ? P.v1 : P.v0}, {}}; },
        [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[2]) {
          if (H.tma) {
            const StagedTile t = staged_tile(st, H, 2);
            const int sl = lr >> 5;
            const Slots slot = slice_slots(st, H, sl);
            const SBiCG sv{t.w(0), t.w(1), alpha};
            double si;
            const double ti = staged_row<true>(P, parts, H, t, slot, lr, sv, sval_g, si);
            if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              P.s[i] = si;
              P.t[i] = ti;
              acc[0] = __dadd_rn(acc[0], __dmul_rn(ti, si));
              acc[1] = __dadd_rn(acc[1], __dmul_rn(ti, ti));
            }
          } else if (lr < H.rows) {
            const int64_t i = H.row0 + lr;
            const double si = sval_g(P, i);
            const double ti = row_spmv(P, parts, i, sval_g);
            P.s[i] = si;
            P.t[i] = ti;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(ti, si));
            acc[1] = __dadd_rn(acc[1], __dmul_rn(ti, ti));
          }
        });
    if (team_failed(T)) break;
    omega = red[1] != 0.0 ? red[0] / red[1] : 0.0;
    // ---- phase 3: x = (x + alpha p) + omega s, r = s - omega t, r.r, rhat.r;
    //      u = p - omega v over p (the next phase 1's operand)
    stream_phase<2, INL, true, true>(
        T, S, gseq, red, 2,
        [&](const PartDev& P) {
          return Spec{0, 6, {nullptr, nullptr},
                      {pa ? P.p1 : P.p0, P.s, P.x, P.t, P.rhat, pa ? P.v1 : P.v0}};
        },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[2]) {
          if (lr >= H.rows) return;
          const int64_t i = H.row0 + lr;
          const double s = V[1][lr];
          const double x = __dadd_rn(__dadd_rn(V[2][lr], __dmul_rn(alpha, V[0][lr])), __dmul_rn(omega, s));
          const double r = __dsub_rn(s, __dmul_rn(omega, V[3][lr]));
          const double u = __dsub_rn(V[0][lr], __dmul_rn(omega, V[5][lr]));
          (pa ? P.p1 : P.p0)[i] = u;
          P.x[i] = x;
          P.r[i] = r;
          hpush(P, parts, pa ? kMp1 : kMp0, i, u);
          hpush(P, parts, kMx, i, x);
          hpush(P, parts, kMr, i, r);
          acc[0] = __dadd_rn(acc[0], __dmul_rn(r, r));
          acc[1] = __dadd_rn(acc[1], __dmul_rn(V[4][lr], r));
        });
    if (team_failed(T)) break;
    const double rr = red[0];
    rho_prev = rho;
    rho = red[1];
    const double rec = sqrt(rr) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      auto xg = [](const PartDev& Q, int64_t j) -> double { return Q.x[j]; };
      stream_phase<1, INL, false>(
          T, S, gseq, red, 3, [&](const PartDev& P) { return Spec{1, 1, {P.x, nullptr}, {P.b}}; },
          [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr,
              double (&acc)[1]) {
            if (H.tma) {
              const StagedTile t = staged_tile(st, H, 1);
              const Slots slot = slice_slots(st, H, lr >> 5);
              const double ax = staged_row<true>(P, parts, H, t, slot, lr, Win1{t.w(0)}, xg);
              if (lr < H.rows) {
                const double d = __dsub_rn(t.tail(0)[lr], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            } else if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              const double ax = row_spmv(P, parts, i, xg);
              const double d = __dsub_rn(P.b[i], ax);
              acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
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
    if (omega == 0.0 || rho == 0.0) {
      breakdown = true;
      break;
    }
  }
  stream_flush_counters(T, S);
  if (lead) {
    out->iterations = it > T.max_iter ? T.max_iter : it;
    out->converged = converged ? 1 : 0;
    out->breakdown = breakdown ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

// ---------------------------------------------------------------------------
// Single-reduction Jacobi-PCG (Chronopoulos-Gear, method
// "pcg1"): ONE fused SpMV phase and one team barrier per iteration instead of
// two.  With u = M r (M = diag^-1), w = A u, s = A p kept as recurrences:
//   beta = gamma / gamma_prev, eta = delta - beta * gamma / alpha_prev,
//   alpha = gamma / eta;  p = u + beta p, s = w + beta s,
//   x += alpha p, r -= alpha s, u = M r, w = A u,
//   gamma = r.u, delta = w.u, rho = r.r   (one fused reduction)
// The neighbours' u_new = dinv (r - alpha (w + beta s_old)) is computed on the
// fly from four staged windows (r, dinv, w, s_old); r, w, s are double-
// buffered.  Mathematically CG's iterates; rounding differs from the
// two-phase kernel (parity by tolerance).
// Buffers: x, p = p0; r in {r, rhat}; w in {v0, v1}; s in {s, t}.
// ---------------------------------------------------------------------------
template <bool INL>
__global__ void LRB_STREAM_BOUNDS
    team_pcg1_stream_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  const StreamSmem S = stream_smem(T);
  stream_init(T, S);
  int gseq = 0;
  double red[4];
  auto rbuf = [](const PartDev& Q, int b) -> double* { return b ? Q.rhat : Q.r; };
  auto wbuf = [](const PartDev& Q, int b) -> double* { return b ? Q.v1 : Q.v0; };
  auto sbuf = [](const PartDev& Q, int b) -> double* { return b ? Q.t : Q.s; };
  // ---- phase 0: x = 0, r = b, b.b
  stream_phase<1, INL, true>(
      T, S, gseq, red, 0, [&](const PartDev& P) { return Spec{0, 1, {nullptr}, {P.b}}; },
      [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[1]) {
        if (lr >= H.rows) return;
        const int64_t i = H.row0 + lr;
        const double b = V[0][lr];
        P.x[i] = 0.0;
        P.r[i] = b;
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
  // ---- phase 0b: u0 = M r0, w0 = A u0, gamma = r.u, delta = w.u
  auto u0_g = [](const PartDev& Q, int64_t j) -> double { return __dmul_rn(Q.dinv[j], Q.r[j]); };
  stream_phase<2, INL, false>(
      T, S, gseq, red, 1, [&](const PartDev& P) { return Spec{2, 0, {P.r, P.dinv}, {}}; },
      [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[2]) {
        double wi, ui;
        if (H.tma) {
          const StagedTile t = staged_tile(st, H, 2);
          const int sl = lr >> 5;
          const Slots slot = slice_slots(st, H, sl);
          const double* rw = t.w(0);
          const double* dw = t.w(1);
          auto u = [&](int q) { return __dmul_rn(dw[q], rw[q]); };
          wi = staged_row(P, parts, H, t, slot, lr, u, u0_g, ui);
          if (lr >= H.rows) return;
        } else {
          if (lr >= H.rows) return;
          const int64_t i = H.row0 + lr;
          wi = row_spmv(P, parts, i, u0_g);
          ui = u0_g(P, i);
        }
        const int64_t i = H.row0 + lr;
        P.v0[i] = wi;
        acc[0] = __dadd_rn(acc[0], __dmul_rn(P.r[i], ui));
        acc[1] = __dadd_rn(acc[1], __dmul_rn(wi, ui));
      });
  if (team_failed(T)) return;
  double gamma = red[0], delta = red[1], gamma_prev = 1.0, alpha_prev = 1.0, res = 1.0;
  int par = 0;   // current r, w, s buffers; the phase writes the other ones
  bool converged = false;
  int it = 0;
  for (it = 1; it <= T.max_iter; ++it) {
    const bool first = (it == 1);
    const double beta = first ? 0.0 : gamma / gamma_prev;
    const double eta = first ? delta : __dsub_rn(delta, __dmul_rn(beta, gamma / alpha_prev));
    if (eta <= 0.0) {
      if (lead) team_fail(T, LRB_ENOTPD);
      break;
    }
    const double alpha = gamma / eta;
    // ---- fused phase: p, s, x, r updates, u_new, w_new = A u_new, three dots
    auto s_g = [&](const PartDev& Q, int64_t j) -> double {
      const double w = wbuf(Q, par)[j];
      return first ? w : __dadd_rn(w, __dmul_rn(beta, sbuf(Q, par)[j]));
    };
    auto u_g = [&](const PartDev& Q, int64_t j) -> double {
      return __dmul_rn(Q.dinv[j], __dsub_rn(rbuf(Q, par)[j], __dmul_rn(alpha, s_g(Q, j))));
    };
    stream_phase<3, INL, false>(
        T, S, gseq, red, 1,
        [&](const PartDev& P) {
          return Spec{first ? 3 : 4, 2, {rbuf(P, par), P.dinv, wbuf(P, par), sbuf(P, par)}, {P.p0, P.x}};
        },
        [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[3]) {
          double wn, r_i, s_i, d_i, po, xo;
          if (H.tma) {
            const StagedTile t = staged_tile(st, H, first ? 3 : 4);
            const int sl = lr >> 5;
            const Slots slot = slice_slots(st, H, sl);
            const UCG1 u{t.w(0), t.w(1), t.w(2), t.w(3), alpha, beta, first};
            wn = staged_row(P, parts, H, t, slot, lr, u, u_g);
            if (lr >= H.rows) return;
            const int qd = diag_pos(H, slot, sl, H.row0 + lr);
            r_i = t.w(0)[qd];
            d_i = t.w(1)[qd];
            s_i = u.s(qd);
            po = t.tail(0)[lr];
            xo = t.tail(1)[lr];
          } else {
            if (lr >= H.rows) return;
            const int64_t i = H.row0 + lr;
            wn = row_spmv(P, parts, i, u_g);
            r_i = rbuf(P, par)[i];
            d_i = P.dinv[i];
            s_i = s_g(P, i);
            po = P.p0[i];
            xo = P.x[i];
          }
          const int64_t i = H.row0 + lr;
          const double u_old = __dmul_rn(d_i, r_i);
          const double p_i = first ? u_old : __dadd_rn(u_old, __dmul_rn(beta, po));
          const double r_new = __dsub_rn(r_i, __dmul_rn(alpha, s_i));
          const double u_new = __dmul_rn(d_i, r_new);
          P.p0[i] = p_i;
          P.x[i] = __dadd_rn(xo, __dmul_rn(alpha, p_i));
          rbuf(P, par ^ 1)[i] = r_new;
          sbuf(P, par ^ 1)[i] = s_i;
          wbuf(P, par ^ 1)[i] = wn;
          acc[0] = __dadd_rn(acc[0], __dmul_rn(r_new, u_new));
          acc[1] = __dadd_rn(acc[1], __dmul_rn(wn, u_new));
          acc[2] = __dadd_rn(acc[2], __dmul_rn(r_new, r_new));
        });
    if (team_failed(T)) break;
    par ^= 1;
    gamma_prev = gamma;
    alpha_prev = alpha;
    gamma = red[0];
    delta = red[1];
    const double rec = sqrt(red[2]) / bnorm;
    if (lead && T.hist && it <= T.hist_cap) T.hist[it - 1] = rec;
    if (rec <= T.tol || it % 10 == 0) {
      auto xg = [](const PartDev& Q, int64_t j) -> double { return Q.x[j]; };
      stream_phase<1, INL, false>(
          T, S, gseq, red, 3, [&](const PartDev& P) { return Spec{1, 1, {P.x}, {P.b}}; },
          [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr,
              double (&acc)[1]) {
            if (H.tma) {
              const StagedTile t = staged_tile(st, H, 1);
              const Slots slot = slice_slots(st, H, lr >> 5);
              const double ax = staged_row(P, parts, H, t, slot, lr, Win1{t.w(0)}, xg);
              if (lr < H.rows) {
                const double d = __dsub_rn(t.tail(0)[lr], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            } else if (lr < H.rows) {
              const int64_t i = H.row0 + lr;
              const double ax = row_spmv(P, parts, i, xg);
              const double d = __dsub_rn(P.b[i], ax);
              acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
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

namespace lrb {

// ---------------------------------------------------------------------------
// Pipelined Jacobi-PCG (Ghysels-Vanroose, method "pipecg").
// The iteration's SpMV n = A (M w) does not depend on the scalars of the
// reduction issued at the end of the previous phase, so on a flat team (one
// device, one part: every CTA its own reduction lane, kernels.cuh flat_sync)
// the barrier between phases only waits for the arrivals (neighbour data
// complete) and the reduction itself is read one phase late: the reducer warp
// combines the previous barrier's lane values (the canonical tree) while the
// consumers run the SpMV of their first stage, and the consumers pick the
// scalars up before the first elementwise update.  Other teams reduce at the
// barrier (same tree, same bits).
//   beta = gamma / gamma_prev, eta = delta - beta * gamma / alpha_prev,
//   alpha = gamma / eta;  n = A (M w);  z = n + beta z;  s = w + beta s;
//   p = M r + beta p;  x += alpha p;  r -= alpha s;  w -= alpha z;
//   (gamma, delta, rho) = (r.Mr, w.Mr, r.r)
// oracle/krylov.py pipecg restates it.  The scalars of state k are known only
// during phase k+1, so the stopping decision for iteration k is taken after
// phase k+1: x is double-buffered (x_k in buffer k & 1) and that decision's
// true-residual check reads x_k; w is double-buffered (the SpMV reads its
// window while the phase writes the new w).  Buffers: x in {x, p1}, w in
// {v0, v1}, z = t, s, p = p0, r.
// ---------------------------------------------------------------------------
static __shared__ unsigned s_pgen;            // deferred reductions published (reducer warp)
// by generation parity: a slow thread may still read generation g's values
// after the phase barrier while the reducer of the next phase writes g + 1
static __shared__ double s_pscal[2][8];       // their values [0, 3), alpha, beta, breakdown
static __shared__ double s_pread[kMaxRed];    // flat_read_last

// Canonical tree of barrier b's lane values (flat_sync's, bit for bit), by
// one warp; lane 0 writes out[0..NR).
template <int NR>
__device__ __forceinline__ void lanes_tree_warp(const TeamDev& T, unsigned b, double* out) {
  const int lane = threadIdx.x & 31;
  const double* lv = lane_slots(T, b);
  double x[kLaneGroups][NR];
#pragma unroll
  for (int g = 0; g < kLaneGroups; ++g) {
    const int v = g * 32 + lane;
#pragma unroll
    for (int j = 0; j < NR; ++j) x[g][j] = v < int(gridDim.x) ? __ldcg(lv + size_t(v) * kMaxRed + j) : 0.0;
  }
  double s[NR];
#pragma unroll
  for (int g = 0; g < kLaneGroups; ++g)
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      double a = x[g][j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
      s[j] = g == 0 ? a : __dadd_rn(s[j], a);
    }
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NR; ++j) out[j] = s[j];
}

// Arrival-only flat barrier: lane values stay in their parity slot for a
// later lanes_tree_warp; the count is launch-monotonic like flat_sync's.
__device__ __forceinline__ void flat_arrive(const TeamDev& T) {
  __syncthreads();
  const unsigned b = s_flat_bar;
  if (threadIdx.x == 0) {
    unsigned long long* cnt = &T.out->flat_count;
    const unsigned long long target = (unsigned long long)(b + 1) * gridDim.x;
    red_add_release_gpu64(cnt);
    const long long t0 = global_ns();
    while (ld_acquire_gpu64(cnt) < target) {
      if (LRB_FLAT_POLL_NS) __nanosleep(LRB_FLAT_POLL_NS);
      if (global_ns() - t0 > T.timeout_ns) {
        team_fail(T, LRB_ETIMEOUT);
        break;
      }
    }
    s_flat_bar = b + 1;
  }
  __syncthreads();
}

// The last barrier's pending lane values, read now by every thread.
template <int NR>
__device__ __forceinline__ void flat_read_last(const TeamDev& T, double* red) {
  __syncthreads();   // every thread has read the previous s_pscal values
  if (threadIdx.x < 32) lanes_tree_warp<NR>(T, s_flat_bar - 1, s_pread);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NR; ++j) red[j] = s_pread[j];
  __syncthreads();
}

// SpMV phase with the pipelined barrier: din = the reducer publishes the
// previous barrier's reduction and coef()'s scalars from it (generation
// `want`) before its own stages;
// dout = arrival-only barrier (flat teams), else the reducing team_sync.
template <int NR, bool INL, class SpecF, class CoefF, class PreF, class Body>
__device__ __forceinline__ void stream_phase_pipe(const TeamDev& T, const StreamSmem& S, int& gseq, double* red,
                                                  int kind, bool din, bool dout, unsigned want, SpecF&& spec_of,
                                                  CoefF&& coef, PreF&& pre, Body&& body) {
  if (threadIdx.x >= kReducer) {
    if (din) {
      double* ps = s_pscal[want & 1];
      lanes_tree_warp<NR>(T, s_flat_bar - 1, ps);
      if ((threadIdx.x & 31) == 0) {
        coef(ps);   // ps[NR..]: the phase's own scalars
        asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(&s_pgen)), "r"(want) : "memory");
      }
      __syncwarp();
    }
    reduce_phase<NR, false>(T, S, gseq, 0);
  } else if (threadIdx.x >= kConsumers) {
    fence_proxy_async_global();
    produce_spmv<INL>(T, S, gseq, kind, spec_of);
  } else {
    if (din) {   // the reducer publishes before its own stages, while the first copies fly
      unsigned g;
      do {   // acquire: orders the scalar reads in pre()
        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(g) : "r"(smem_u32(&s_pgen)) : "memory");
      } while (g < want);
      pre(s_pscal[want & 1]);
    }
    consume_phase<NR, INL, false>(T, S, gseq, kind, 0, body);
  }
  fence_proxy_async_global();
  if (dout)
    flat_arrive(T);
  else
    team_sync<NR>(T, red, 1, reinterpret_cast<double*>(S.stages));
  gseq += stage_count(T.n_tiles);
}

template <bool INL, bool DEFER, bool TAILS>
__global__ void LRB_STREAM_BOUNDS
    team_pipecg_stream_kernel(const __grid_constant__ TeamDev T) {
  const PartDev* __restrict__ parts = T.parts;
  const StreamSmem S = stream_smem(T);
  stream_init(T, S);
  if (threadIdx.x == 0) s_pgen = 0;
  int gseq = 0;
  double red[4];
  auto xbuf = [](const PartDev& Q, int b) -> double* { return b ? Q.p1 : Q.x; };
  auto wbuf = [](const PartDev& Q, int b) -> double* { return b ? Q.v1 : Q.v0; };
  // ---- phase 0: x = 0, r = b, b.b
  stream_phase<1, INL, true>(
      T, S, gseq, red, 0, [&](const PartDev& P) { return Spec{0, 1, {nullptr}, {P.b}}; },
      [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&acc)[1]) {
        if (lr >= H.rows) return;
        const int64_t i = H.row0 + lr;
        const double b = V[0][lr];
        P.x[i] = 0.0;
        P.r[i] = b;
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
  // ---- phase 0b: w0 = A (M r0) into v0, gamma = r.Mr, delta = w.Mr
  auto u0_g = [](const PartDev& Q, int64_t j) -> double { return __dmul_rn(Q.dinv[j], Q.r[j]); };
  stream_phase<2, INL, false>(
      T, S, gseq, red, 1, [&](const PartDev& P) { return Spec{2, 0, {P.r, P.dinv}, {}}; },
      [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[2]) {
        double wi, ui;
        if (H.tma) {
          const StagedTile t = staged_tile(st, H, 2);
          const int sl = lr >> 5;
          const Slots slot = slice_slots(st, H, sl);
          const double* rw = t.w(0);
          const double* dw = t.w(1);
          auto u = [&](int q) { return __dmul_rn(dw[q], rw[q]); };
          wi = staged_row(P, parts, H, t, slot, lr, u, u0_g, ui);
          if (lr >= H.rows) return;
        } else {
          if (lr >= H.rows) return;
          const int64_t i = H.row0 + lr;
          wi = row_spmv(P, parts, i, u0_g);
          ui = u0_g(P, i);
        }
        const int64_t i = H.row0 + lr;
        P.v0[i] = wi;
        acc[0] = __dadd_rn(acc[0], __dmul_rn(P.r[i], ui));
        acc[1] = __dadd_rn(acc[1], __dmul_rn(wi, ui));
      });
  if (team_failed(T)) return;
  const bool flat =
      DEFER && LRB_FLAT_BAR && T.n_dev == 1 && T.n_parts == 1 && lanes_by_cta(T, T.n_tiles, 1);
  // scalars of the newest state whose reduction was read
  double gamma = red[0], delta = red[1], gamma_prev = 1.0, alpha_prev = 1.0, res = 1.0;
  bool pend = false;        // the newest state's reduction still sits in the lane slots
  bool converged = false, stop = false;
  int last = 0;             // newest iteration whose stopping decision was taken
  unsigned pgen = 0;
  // alpha, beta of a phase from the scalars (g, d) of the state before it
  // (the reducer warp and, after the phase, every thread: same bits)
  auto coef = [&](bool first, double g, double d, double& alpha, double& beta) -> bool {
    beta = first ? 0.0 : g / gamma_prev;
    const double eta = first ? d : __dsub_rn(d, __dmul_rn(beta, g / alpha_prev));
    alpha = g / eta;
    return !(eta > 0.0);
  };
  for (int k = 1;; ++k) {
    const bool run = k <= T.max_iter;
    const bool first = (k == 1);
    const bool din = pend && run;
    double alpha = 0.0, beta = 0.0;
    bool bad = false;
    int jd[2];          // iterations whose stopping decision is due after this step
    double rrd[2];
    int nd = 0;
    if (run) {
      if (!din) {
        bad = coef(first, gamma, delta, alpha, beta);
        if (bad) {   // iteration k-1 was decided (not converged): breakdown now
          if (lead) team_fail(T, LRB_ENOTPD);
          break;
        }
      }
      const int ob = (k - 1) & 1, nb = k & 1;   // x / w buffers: read ob, write nb
      auto m_g = [ob](const PartDev& Q, int64_t j) -> double {
        return __dmul_rn(Q.dinv[j], (ob ? Q.v1 : Q.v0)[j]);
      };
      const unsigned want = pgen + 1;
      stream_phase_pipe<3, INL>(
          T, S, gseq, red, 1, din, flat, want,
          [&](const PartDev& P) {
            if (TAILS) return Spec{2, 5, {wbuf(P, ob), P.dinv}, {P.t, P.s, P.p0, xbuf(P, ob), P.r}};
            return Spec{2, 0, {wbuf(P, ob), P.dinv}, {}, 5, {P.t, P.s, P.p0, xbuf(P, ob), P.r}};
          },
          [&](double* pab) {   // reducer warp, lane 0: this phase's alpha, beta, breakdown
            double a, b;
            const bool bk = coef(first, pab[0], pab[1], a, b);
            pab[3] = a;
            pab[4] = b;
            pab[5] = bk ? 1.0 : 0.0;
          },
          [&](const double* pab) {   // consumers: the phase's scalars from the reducer
            alpha = pab[3];
            beta = pab[4];
            bad = pab[5] != 0.0;
          },
          [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[3]) {
            double n_i, w_i, d_i, z_o, s_o, p_o, x_o, r_i;
            if (H.tma) {
              const StagedTile t = staged_tile(st, H, 2);
              const int sl = lr >> 5;
              const Slots slot = slice_slots(st, H, sl);
              const double* ww = t.w(0);
              const double* dw = t.w(1);
              auto m = [&](int q) { return __dmul_rn(dw[q], ww[q]); };
              n_i = staged_row(P, parts, H, t, slot, lr, m, m_g);
              if (lr >= H.rows || bad) return;
              const int qd = diag_pos(H, slot, sl, H.row0 + lr);
              w_i = ww[qd];
              d_i = dw[qd];
              if (TAILS) {
                z_o = t.tail(0)[lr];
                s_o = t.tail(1)[lr];
                p_o = t.tail(2)[lr];
                x_o = t.tail(3)[lr];
                r_i = t.tail(4)[lr];
              } else {   // own-row vectors straight from global memory (smaller stages, deeper ring)
                const int64_t i = H.row0 + lr;
                z_o = __ldcs(P.t + i);
                s_o = __ldcs(P.s + i);
                p_o = __ldcs(P.p0 + i);
                x_o = __ldcs(xbuf(P, ob) + i);
                r_i = __ldcs(P.r + i);
              }
            } else {
              if (lr >= H.rows || bad) return;
              const int64_t i = H.row0 + lr;
              n_i = row_spmv(P, parts, i, m_g);
              w_i = wbuf(P, ob)[i];
              d_i = P.dinv[i];
              z_o = P.t[i];
              s_o = P.s[i];
              p_o = P.p0[i];
              x_o = xbuf(P, ob)[i];
              r_i = P.r[i];
            }
            const int64_t i = H.row0 + lr;
            const double u_i = __dmul_rn(d_i, r_i);
            const double z = first ? n_i : __dadd_rn(n_i, __dmul_rn(beta, z_o));
            const double s = first ? w_i : __dadd_rn(w_i, __dmul_rn(beta, s_o));
            const double p = first ? u_i : __dadd_rn(u_i, __dmul_rn(beta, p_o));
            const double r = __dsub_rn(r_i, __dmul_rn(alpha, s));
            const double w = __dsub_rn(w_i, __dmul_rn(alpha, z));
            const double un = __dmul_rn(d_i, r);
            P.t[i] = z;
            P.s[i] = s;
            P.p0[i] = p;
            xbuf(P, nb)[i] = __dadd_rn(x_o, __dmul_rn(alpha, p));
            P.r[i] = r;
            wbuf(P, nb)[i] = w;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(r, un));
            acc[1] = __dadd_rn(acc[1], __dmul_rn(w, un));
            acc[2] = __dadd_rn(acc[2], __dmul_rn(r, r));
          });
      if (team_failed(T)) break;
      if (din) {   // state k-1's reduction, read by the reducer during phase k
        pgen = want;
        const double* ps = s_pscal[want & 1];
        const double g = ps[0];
        bad = coef(first, g, ps[1], alpha, beta);
        jd[nd] = k - 1;
        rrd[nd++] = ps[2];
        gamma_prev = g;
      } else {
        gamma_prev = gamma;
      }
      alpha_prev = alpha;
      pend = flat;
      if (!flat) {   // state k's reduction came with the barrier
        gamma = red[0];
        delta = red[1];
        jd[nd] = k;
        rrd[nd++] = red[2];
      }
    } else {   // max_iter reached: the last state's decision may still be pending
      if (!pend) break;
      flat_read_last<3>(T, red);
      pend = false;
      jd[nd] = k - 1;
      rrd[nd++] = red[2];
    }
    // stopping decisions (solver.py:136-142), oldest first: recurrence
    // residual, true residual of x_j (buffer j & 1) at tol or every 10th
    for (int q = 0; q < nd && !stop; ++q) {
      const int j = jd[q];
      const double rec = sqrt(rrd[q]) / bnorm;
      if (lead && T.hist && j <= T.hist_cap) T.hist[j - 1] = rec;
      last = j;
      if (rec <= T.tol || j % 10 == 0) {
        if (pend) {   // the check's barrier reuses the lane slots: take state k's first
          flat_read_last<3>(T, red);
          pend = false;
          gamma = red[0];
          delta = red[1];
          jd[nd] = k;
          rrd[nd++] = red[2];
        }
        const int xb = j & 1;
        auto xg = [xb](const PartDev& Q, int64_t c) -> double { return (xb ? Q.p1 : Q.x)[c]; };
        stream_phase<1, INL, false>(
            T, S, gseq, red, 3, [&](const PartDev& P) { return Spec{1, 1, {xbuf(P, xb)}, {P.b}}; },
            [&](const PartDev& P, const StageHdr& H, const char* st, const VecView&, int lr, double (&acc)[1]) {
              if (H.tma) {
                const StagedTile t = staged_tile(st, H, 1);
                const Slots slot = slice_slots(st, H, lr >> 5);
                const double ax = staged_row(P, parts, H, t, slot, lr, Win1{t.w(0)}, xg);
                if (lr < H.rows) {
                  const double d = __dsub_rn(t.tail(0)[lr], ax);
                  acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
                }
              } else if (lr < H.rows) {
                const int64_t i = H.row0 + lr;
                const double ax = row_spmv(P, parts, i, xg);
                const double d = __dsub_rn(P.b[i], ax);
                acc[0] = __dadd_rn(acc[0], __dmul_rn(d, d));
              }
            });
        if (team_failed(T)) {
          stop = true;
          break;
        }
        res = sqrt(red[0]) / bnorm;
        if (res <= T.tol) {
          converged = true;
          stop = true;
        }
      } else {
        res = rec;
      }
      if (!stop && din && q == 0 && bad) {   // phase k broke down; iteration k-1 did not converge
        if (lead) team_fail(T, LRB_ENOTPD);
        stop = true;
      }
    }
    if (stop || !run) break;
  }
  if (!team_failed(T) && (last & 1)) {   // the result x_last sits in the second buffer
    stream_phase<1, INL, true>(
        T, S, gseq, red, 0, [&](const PartDev& P) { return Spec{0, 1, {nullptr}, {P.p1}}; },
        [&](const PartDev& P, const StageHdr& H, const char*, const VecView& V, int lr, double (&)[1]) {
          if (lr < H.rows) P.x[H.row0 + lr] = V[0][lr];
        });
  }
  stream_flush_counters(T, S);
  if (lead) {
    out->iterations = last;
    out->converged = converged ? 1 : 0;
    out->residual = res;
    out->bnorm = bnorm;
  }
}

}  // namespace lrb
