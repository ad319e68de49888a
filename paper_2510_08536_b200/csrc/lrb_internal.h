// Internal structures shared by the host builder, the CUDA kernels and the C-ABI.
// Not part of the public interface (see include/ldurepart_b200.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace lrb {

// ---------------------------------------------------------------------------
// Device layout of one fused owner part ("GPU part k", repart.py:307-318).
//
// The fused matrix is stored once, in SELL-32: rows are grouped in slices of
// 32 consecutive rows (one warp), each slice padded to its longest row and
// laid out column-major (entry k of the slice's 32 rows are 32 consecutive
// words).  A row's entries are its local entries in ascending column order
// followed by its non-local entries in ascending halo order — exactly the
// reference's row-major `local` then `non_local` order (solver.py:92-97), so a
// per-row sequential product sum reproduces solver.spmv bit for bit.
//   col[e] <  n         : part-local column
//   col[e] >= n         : halo slot (col - n), resolved via hpart/hidx
//   col[e] == -1        : padding (always at the end of a row)
//   src[e]              : receive-buffer position scattered into val[e]
// ---------------------------------------------------------------------------
constexpr int kSlice = 32;

// Pattern dictionary: a full slice whose rows' column offsets (col - row) fit
// in at most kPatW distinct values is laid out on the sorted union of those
// offsets; its columns are not streamed from HBM but rebuilt as
// row + pat_off[pid][slot] for the slots set in the row's rmask.  On the
// cavity stencil nearly every slice qualifies, which removes 4 of the 12
// matrix bytes per entry and the dependent col -> x load chain.
constexpr int kPatW = 16;      // widest row a pattern may describe
constexpr int kMaxPat = 1024;  // dictionary size

// Shared-memory staging of the SpMV operand for pattern tiles: a tile's rows
// read the vector only at row + {pattern offsets}; those indices form at most
// kMaxWin contiguous windows (on the 7-point stencil: -plane, [-d0, d0], +plane
// around the tile).  The block stages the windows with coalesced loads once
// (computing p_new = z + beta*p_old once per element) and the rows read shared
// memory instead of 14 dependent gathers each.  tile_win[t] = {n_win, total,
// start0, len0, start1, len1, start2, len2} (starts relative to the tile's
// first row, clipped to [0, n)); n_win = 0: no staging for that tile.
constexpr int kMaxWin = 3;
constexpr int kWinStride = 2 + 2 * kMaxWin;
constexpr int kMaxStage = 4096;   // doubles of staged operand per block

struct PartDev {
  int64_t n;          // owned rows
  int64_t n_halo;
  int64_t n_buf;      // receive-buffer length (= nnz, bijection)
  int64_t n_slices;
  const int64_t* slice_ptr;   // [n_slices+1] entry offsets
  const int32_t* slice_pat;   // [n_slices] pattern id or -1
  const int32_t* pat_off;     // [n_pat * kPatW]
  const uint16_t* rmask;      // [n] occupied pattern slots of each row
  const int32_t* tile_win;    // [ntiles_part * kWinStride] staging windows
  const int32_t* col;         // [E]
  const int32_t* src;         // [E] scatter inverse (buffer position or -1)
  const int16_t* dpos;         // [n] slot k of the diagonal in the row, -1 if none
  const int32_t* hpart;       // [n_halo] team part that owns halo slot
  const int32_t* hidx;        // [n_halo] row of that part
  double* val;                // [E]
  double* recv;               // [n_buf]
  // Krylov vectors, [n] each
  double *x, *r, *p0, *p1, *q, *b, *dinv;
  double *rhat, *v0, *v1, *s, *t;
  // tiling inside the team kernel
  int64_t tile0;      // first tile of this part in its device's tile space
  int64_t ntiles;
  // Halo mirror (arena-resident, [kMirVecs][n_halo]): the owners of this
  // part's halo rows push their new values of the mirrored Krylov vectors
  // here while they compute them (peer stores over NVLink for other GPUs), so
  // the next SpMV reads its halo operands from local memory instead of
  // issuing remote loads on its critical path (solver.py:86-90: the halo is
  // filled before the multiply).
  double* hm;
  // Team-level fields (set at team creation in the team's part table):
  const int64_t* snd;   // [n_snd][4] push runs of THIS part's rows: {row_lo, row_hi, reader part,
                        //   reader halo slot of row_lo}; slots are consecutive along a run
  int32_t n_snd;
  int32_t mir;          // 1: the streaming solvers read halo operands from hm (mirrors on)
  int64_t sq_lo, sq_hi; // rows in [sq_lo, sq_hi) are in no run (interior: nothing to push)
};

// Mirrored vectors (halo mirror slot ids).
enum MirVec { kMx = 0, kMr = 1, kMp0 = 2, kMp1 = 3, kMs = 4, kMv0 = 5, kMv1 = 6, kMirVecs = 7 };
constexpr int kMaxSndRuns = 32;   // more push runs for a part: mirrors off for the team

// Work decomposition of the persistent kernels: a tile is kTPB*kRPT rows of
// one part.  The per-tile partial dot products are reduced in fixed order,
// so results do not depend on grid size or scheduling.
#ifndef LRB_TPB
#define LRB_TPB 256
#endif
constexpr int kTPB = LRB_TPB;   // threads per classic block = rows per streaming team pass
#ifndef LRB_RPT
#define LRB_RPT 2
#endif
constexpr int kRPT = LRB_RPT;
constexpr int kTile = kTPB * kRPT;
constexpr int kMaxRed = 4;   // reductions fused into one barrier

// Per-tile header of the streaming solvers (stream.cuh), precomputed at team
// creation and bulk-copied into the shared-memory stage with the tile's data.
constexpr int kHdrBytes = 256;
constexpr int kHdrPats = 4;    // distinct slice patterns a staged tile may hold
struct StageHdrFields {
  int64_t row0;          // first row of the tile (part-local)
  int64_t e0;            // first SELL entry of the tile
  int64_t wa[kMaxWin];   // aligned start of each operand window (part-local row)
  int32_t rows;
  int32_t part;          // team part index
  int32_t tile;          // device tile index
  int32_t tma;           // 1: values + windows staged; 0: direct global loads
  int32_t nw;            // windows
  int32_t wtot;          // staged elements per window vector (even)
  int32_t wl[kMaxWin];   // aligned window lengths (even)
  int32_t woff[kMaxWin]; // window offsets inside a vector's staged run
  int32_t vbytes;        // staged value bytes
  int32_t npat;          // distinct patterns of the tile (slot tables in StageTab)
  int32_t halo;          // 1: some row of the tile has non-local (halo) columns
  int32_t sp[kTile / kSlice + 1];   // slice entry offsets relative to e0
  int32_t pat[kTile / kSlice];      // slice pattern ids (dictionary)
  int8_t spat[kTile / kSlice];      // slice -> slot table of the tile's StageTab
  int8_t sdiag[kHdrPats];           // slot of the diagonal (offset 0) per table
};
static_assert(sizeof(StageHdrFields) <= kHdrBytes, "stage header fields exceed kHdrBytes");
struct alignas(16) StageHdr : StageHdrFields {
  char reserved_[kHdrBytes - sizeof(StageHdrFields)];
};
static_assert(sizeof(StageHdr) == kHdrBytes, "stage header must be exactly kHdrBytes");

// Slot tables of a staged tile: for each distinct pattern and slot k, the
// column offset (col - row) and the shared-memory delta e such that a row i's
// operand for that slot sits at staged index i + e (window arithmetic done
// once on the host instead of per warp and row on the device).
// Structure of arrays: a slice's deltas are 16-byte aligned, so a warp reads
// four slots per vector load.
constexpr int kTabBytes = kHdrPats * kPatW * 8;
struct alignas(16) StageTab {
  int32_t off[kHdrPats][kPatW];
  int32_t del[kHdrPats][kPatW];
};

// What a staged SpMV tile carries besides values and windows, as ONE
// contiguous record so the producer moves it with one bulk copy: the header,
// the slot tables and the tile's row masks (a copy of rmask).
constexpr int kRecMaskBytes = kTile * 2;
constexpr int kRecBytes = kHdrBytes + kTabBytes + kRecMaskBytes;
struct alignas(16) TileRec {
  StageHdr h;
  StageTab t;
  uint16_t mask[kTile];
};
static_assert(sizeof(TileRec) == kRecBytes, "tile record layout");
enum Method { kCG = 0, kPCG = 1, kBiCGStab = 2 };

struct SolveOut {
  int32_t iterations;
  int32_t converged;
  int32_t status;      // 0 ok, LRB_ENOTPD, LRB_ETIMEOUT
  int32_t breakdown;
  double residual;
  double bnorm;
  // arrivals at the flat team barrier (kernels.cuh: team_sync); zeroed with
  // the rest of the record before every launch
  unsigned long long flat_count;
  // barriers released by the last CTA (kernels.cuh: team_sync), same lifetime
  unsigned long long flat_gen;
};

// Descriptors of up to kInlineParts local parts ride in the kernel parameter
// space (__grid_constant__): their fields are warp-uniform constant-bank
// operands, rematerialised instead of pinned in registers.
constexpr int kInlineParts = 8;

// Per-device team state, passed by value as the kernel parameter.
struct TeamDev {
  int32_t n_parts;          // team-wide
  int32_t dev_rank;         // this device's rank in the team
  int32_t n_dev;
  int32_t part_begin;       // parts [part_begin, part_end) live on this device
  int32_t part_end;
  int32_t pad_;
  int64_t n_tiles;          // tiles of this device
  PartDev* parts;           // [n_parts] (remote parts carry peer pointers)
  const int32_t* tile_part; // [n_tiles]
  double* partials;         // [kMaxRed][n_tiles] (one reduction's tiles contiguous)
  double* part_red;         // [2][n_parts][kMaxRed] all parts' values, by epoch parity
  double* red;              // [kMaxRed] team-reduced values (this device)
  unsigned long long* epoch;    // barrier epoch (this device)
  unsigned long long* flags;    // [n_dev] arrival epochs written by peers
  // peers' arrays (index = device rank), valid when n_dev > 1
  unsigned long long** peer_flags;
  double** peer_part_red;
  SolveOut* out;
  double* hist;             // [hist_cap] recurrence residual per iteration (nullable)
  int32_t hist_cap;
  int32_t max_iter;
  const void* tile_hdr;     // streaming solvers: StageHdr per device tile
  const void* tile_rec;     // streaming solvers: TileRec per device tile (header | tables | masks)
  long long* prof;          // phase-release timestamps (nullable, diagnostics)
  long long* prof_cta;      // per-CTA wait-cycle counters (nullable, streaming solvers)
  int32_t* prof_n;
  int32_t prof_cap;
  int32_t lane_fast;        // CTA c computes reduction lane c itself (kernels.cuh: canonical tree)
  int32_t stage_bytes;      // streaming solvers: bytes of one shared-memory stage (classic: the
  int32_t n_stages;         //   streaming geometry, for the tree's units) and ring depth (stream.cuh)
  double* lane_vals;        // [2][kLanes][kMaxRed] lane values by flat-barrier parity (lane_fast)
  double tol;
  long long timeout_ns;
  PartDev lp[kInlineParts];  // local parts [part_begin, part_end) when they fit
};

// ---------------------------------------------------------------------------
// Host plan produced by the create path (plan.cpp).
// ---------------------------------------------------------------------------
struct Plan {
  int64_t total = 0, lo = 0, hi = 0, n = 0, n_buf = 0;
  std::vector<int64_t> loc_ptr, nl_ptr;     // [n+1]
  std::vector<int32_t> loc_col, loc_src;    // part-local col, buffer pos
  std::vector<int32_t> nl_col, nl_src;      // halo slot, buffer pos
  std::vector<int64_t> halo_cols;           // ascending global
  std::vector<int32_t> hpart, hidx;         // halo owner part / row in it
  std::vector<int64_t> seg_off;             // receive offsets [n_src+1]
  std::vector<int64_t> seg_rows;            // segment row ranges (part-local) [n_src+1]
  // SELL
  int64_t n_slices = 0;
  std::vector<int64_t> slice_ptr;
  std::vector<int32_t> sell_col, sell_src;
  std::vector<int16_t> dpos;
  std::vector<int32_t> slice_pat;           // [n_slices]
  std::vector<int32_t> pat_off;             // [n_pat * kPatW]
  std::vector<uint16_t> rmask;              // [n] occupied slots of a pattern row
  std::vector<int32_t> loc_sell, nl_sell;   // SELL slot of every CSR entry
  std::vector<int32_t> tile_win;            // [ntiles * kWinStride]
  int64_t max_stage = 0;
  int64_t n_pat() const { return int64_t(pat_off.size()) / kPatW; }
  int64_t sell_entries() const { return slice_ptr.empty() ? 0 : slice_ptr.back(); }
};

void set_error(const std::string& msg);

}  // namespace lrb
