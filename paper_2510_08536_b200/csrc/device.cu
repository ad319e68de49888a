// Device part / team management and the C-ABI entry points of the hot path.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a (see build.py).

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ldurepart_b200.h"
#include "launch.h"
#include "stream.cuh"
#include "lrb_internal.h"

struct lrb_plan;

namespace lrb {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
static std::atomic<uint64_t> g_launches{0};
const Plan& plan_of(const lrb_plan* p);

#define LRB_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" +   \
                std::to_string(__LINE__) + ")");                                           \
      return LRB_ECUDA;                                                                    \
    }                                                                                      \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static int64_t align256(int64_t v) { return (v + 255) & ~int64_t(255); }

// Arena layout of one part (all sections 256-byte aligned).
struct Layout {
  int64_t slice_ptr, slice_pat, pat_off, rmask, tile_win, col, src, dpos, hpart, hidx, hm, val,
      recv, vec, total;
  static constexpr int kVecs = 12;
};

static Layout layout_of(const Plan& P) {
  Layout L{};
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    int64_t at = o;
    o = align256(o + std::max<int64_t>(bytes, 1));
    return at;
  };
  const int64_t E = P.sell_entries();
  const int64_t h = int64_t(P.halo_cols.size());
  L.slice_ptr = take(8 * (P.n_slices + 1));
  L.slice_pat = take(4 * P.n_slices);
  L.pat_off = take(4 * int64_t(P.pat_off.size()));
  L.rmask = take(2 * P.n);
  L.tile_win = take(4 * int64_t(P.tile_win.size()));
  L.col = take(4 * E);
  L.src = take(4 * E);
  L.dpos = take(2 * P.n);
  L.hpart = take(4 * h);
  L.hidx = take(4 * h);
  L.hm = take(8 * kMirVecs * h);
  L.val = take(8 * E);
  L.recv = take(8 * P.n_buf);
  L.vec = o;
  o += Layout::kVecs * align256(8 * std::max<int64_t>(P.n, 1));
  L.total = o;
  return L;
}

int64_t part_device_bytes(const Plan& P) { return layout_of(P).total; }

}  // namespace lrb

using namespace lrb;

struct lrb_part {
  int device = 0;
  PartDev d{};                      // device pointers (host copy)
  std::vector<int64_t> seg_off, seg_rows, slice_ptr;
  std::vector<int32_t> tile_win;           // host copies (stage headers of the streaming solvers)
  std::vector<int32_t> slice_pat_host, pat_off_host;
  std::vector<uint16_t> rmask_host;
  std::vector<int32_t> loc_sell, nl_sell;  // SELL slot of each CSR entry (value mirror)
  std::vector<char> tile_halo;             // per tile: some row has halo (non-local) columns
  int64_t nnz_l = 0, nnz_n = 0;
  cudaStream_t main = nullptr;
  std::vector<cudaStream_t> seg_stream;
  std::vector<cudaEvent_t> seg_h2d, seg_done;
  std::vector<char> seg_pending;
  cudaEvent_t main_done = nullptr, mark_a = nullptr, mark_b = nullptr;
  int marks = 0;
  double* stage = nullptr;          // pinned, n_buf doubles (caller-owned)
  int64_t stage_len = 0;
  cudaEvent_t stage_free = nullptr; // last H2D from the whole-buffer stage
  cudaEvent_t staged_done = nullptr; // after the last whole-buffer (staged / fill) scatter on main
  // [0] pinned pieces copied zero-copy, [1] pageable pieces staged,
  // [2] H2D bytes, [3] scatter launches
  std::atomic<int64_t> stats[4] = {0, 0, 0, 0};
  std::mutex mu;
  double* base = nullptr;           // device copy of the base receive buffer (lrb_part_capture_base)
};

namespace lrb {

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

static int launch_scatter(lrb_part* P, int64_t r0, int64_t r1, cudaStream_t st) {
  if (r1 <= r0) return LRB_OK;
  LRB_CUDA(scatter_launch(P->d, r0, r1, st));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  P->stats[3] += 1;
  return LRB_OK;
}

}  // namespace lrb

extern "C" {

const char* lrb_last_error(void) { return lrb::g_err.c_str(); }
const char* lrb_version(void) { return "ldurepart_b200 0.1.0 (sm_100a)"; }
uint64_t lrb_launch_count(void) { return lrb::g_launches.load(); }

int lrb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int lrb_part_create(const lrb_plan* plan, int32_t device, void* dev_arena, int64_t dev_bytes,
                    double* host_stage, int64_t host_stage_len, lrb_part** out) {
  if (!plan || !dev_arena || !out) {
    set_error("lrb_part_create: null argument");
    return LRB_EVALUE;
  }
  const Plan& P = plan_of(plan);
  const Layout L = layout_of(P);
  if (dev_bytes < L.total) {
    set_error("lrb_part_create: device arena too small");
    return LRB_EVALUE;
  }
  if ((reinterpret_cast<uintptr_t>(dev_arena) & 255) != 0) {
    set_error("lrb_part_create: device arena must be 256-byte aligned");
    return LRB_EVALUE;
  }
  DeviceGuard g(device);
  auto part = std::make_unique<lrb_part>();
  part->device = device;
  char* base = static_cast<char*>(dev_arena);
  PartDev& D = part->d;
  D.n = P.n;
  D.n_halo = int64_t(P.halo_cols.size());
  D.n_buf = P.n_buf;
  D.n_slices = P.n_slices;
  D.slice_ptr = reinterpret_cast<const int64_t*>(base + L.slice_ptr);
  D.slice_pat = reinterpret_cast<const int32_t*>(base + L.slice_pat);
  D.pat_off = reinterpret_cast<const int32_t*>(base + L.pat_off);
  D.rmask = reinterpret_cast<const uint16_t*>(base + L.rmask);
  D.tile_win = reinterpret_cast<const int32_t*>(base + L.tile_win);
  D.col = reinterpret_cast<const int32_t*>(base + L.col);
  D.src = reinterpret_cast<const int32_t*>(base + L.src);
  D.dpos = reinterpret_cast<const int16_t*>(base + L.dpos);
  D.hpart = reinterpret_cast<const int32_t*>(base + L.hpart);
  D.hidx = reinterpret_cast<const int32_t*>(base + L.hidx);
  D.hm = D.n_halo ? reinterpret_cast<double*>(base + L.hm) : nullptr;
  D.val = reinterpret_cast<double*>(base + L.val);
  D.recv = reinterpret_cast<double*>(base + L.recv);
  double* vecs[Layout::kVecs];
  const int64_t vstride = align256(8 * std::max<int64_t>(P.n, 1));
  for (int i = 0; i < Layout::kVecs; ++i) vecs[i] = reinterpret_cast<double*>(base + L.vec + i * vstride);
  D.x = vecs[0];
  D.r = vecs[1];
  D.p0 = vecs[2];
  D.p1 = vecs[3];
  D.q = vecs[4];
  D.b = vecs[5];
  D.dinv = vecs[6];
  D.rhat = vecs[7];
  D.v0 = vecs[8];
  D.v1 = vecs[9];
  D.s = vecs[10];
  D.t = vecs[11];

  LRB_CUDA(cudaStreamCreateWithFlags(&part->main, cudaStreamNonBlocking));
  const int n_seg = int(P.seg_off.size()) - 1;
  part->seg_stream.resize(n_seg);
  part->seg_h2d.resize(n_seg);
  part->seg_done.resize(n_seg);
  part->seg_pending.assign(n_seg, 0);
  for (int s = 0; s < n_seg; ++s) {
    LRB_CUDA(cudaStreamCreateWithFlags(&part->seg_stream[s], cudaStreamNonBlocking));
    LRB_CUDA(cudaEventCreateWithFlags(&part->seg_h2d[s], cudaEventDisableTiming));
    LRB_CUDA(cudaEventCreateWithFlags(&part->seg_done[s], cudaEventDisableTiming));
  }
  LRB_CUDA(cudaEventCreateWithFlags(&part->main_done, cudaEventDisableTiming));
  LRB_CUDA(cudaEventCreateWithFlags(&part->stage_free, cudaEventDisableTiming));
  LRB_CUDA(cudaEventCreateWithFlags(&part->staged_done, cudaEventDisableTiming));
  LRB_CUDA(cudaEventRecord(part->staged_done, part->main));
  LRB_CUDA(cudaEventCreate(&part->mark_a));
  LRB_CUDA(cudaEventCreate(&part->mark_b));
  part->seg_off = P.seg_off;
  part->seg_rows = P.seg_rows;
  part->loc_sell = P.loc_sell;
  part->nl_sell = P.nl_sell;
  part->slice_ptr = P.slice_ptr;
  part->tile_win = P.tile_win;
  part->slice_pat_host = P.slice_pat;
  part->pat_off_host = P.pat_off;
  part->rmask_host = P.rmask;
  part->tile_halo.assign(size_t((P.n + kTile - 1) / kTile), 0);
  for (int64_t r = 0; r < P.n; ++r)
    if (P.nl_ptr[r + 1] > P.nl_ptr[r]) part->tile_halo[r / kTile] = 1;
  part->nnz_l = int64_t(P.loc_col.size());
  part->nnz_n = int64_t(P.nl_col.size());
  part->stage = host_stage;
  part->stage_len = host_stage_len;

  // upload the create-once index arrays; values and vectors start at zero
  cudaStream_t st = part->main;
  const int64_t E = P.sell_entries();
  LRB_CUDA(cudaMemsetAsync(dev_arena, 0, L.total, st));
  LRB_CUDA(cudaMemcpyAsync(base + L.slice_ptr, P.slice_ptr.data(), 8 * (P.n_slices + 1),
                           cudaMemcpyHostToDevice, st));
  if (P.n_slices)
    LRB_CUDA(cudaMemcpyAsync(base + L.slice_pat, P.slice_pat.data(), 4 * P.n_slices,
                             cudaMemcpyHostToDevice, st));
  LRB_CUDA(cudaMemcpyAsync(base + L.pat_off, P.pat_off.data(), 4 * P.pat_off.size(),
                           cudaMemcpyHostToDevice, st));
  if (P.n)
    LRB_CUDA(cudaMemcpyAsync(base + L.rmask, P.rmask.data(), 2 * P.n, cudaMemcpyHostToDevice, st));
  if (!P.tile_win.empty())
    LRB_CUDA(cudaMemcpyAsync(base + L.tile_win, P.tile_win.data(), 4 * P.tile_win.size(),
                             cudaMemcpyHostToDevice, st));
  if (E) {
    LRB_CUDA(cudaMemcpyAsync(base + L.col, P.sell_col.data(), 4 * E, cudaMemcpyHostToDevice, st));
    LRB_CUDA(cudaMemcpyAsync(base + L.src, P.sell_src.data(), 4 * E, cudaMemcpyHostToDevice, st));
  }
  if (P.n) LRB_CUDA(cudaMemcpyAsync(base + L.dpos, P.dpos.data(), 2 * P.n, cudaMemcpyHostToDevice, st));
  if (D.n_halo) {
    LRB_CUDA(cudaMemcpyAsync(base + L.hpart, P.hpart.data(), 4 * D.n_halo, cudaMemcpyHostToDevice, st));
    LRB_CUDA(cudaMemcpyAsync(base + L.hidx, P.hidx.data(), 4 * D.n_halo, cudaMemcpyHostToDevice, st));
  }
  LRB_CUDA(cudaStreamSynchronize(st));
  LRB_CUDA(cudaEventRecord(part->main_done, st));
  *out = part.release();
  return LRB_OK;
}

void lrb_part_destroy(lrb_part* part) {
  if (!part) return;
  {
    DeviceGuard g(part->device);
    cudaStreamSynchronize(part->main);
    for (auto s : part->seg_stream) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    for (auto e : part->seg_h2d) cudaEventDestroy(e);
    for (auto e : part->seg_done) cudaEventDestroy(e);
    cudaEventDestroy(part->main_done);
    cudaEventDestroy(part->stage_free);
    cudaEventDestroy(part->staged_done);
    cudaEventDestroy(part->mark_a);
    cudaEventDestroy(part->mark_b);
    cudaStreamDestroy(part->main);
  }
  delete part;
}

int lrb_part_pointers(const lrb_part* part, void** ptrs) {
  if (!part || !ptrs) {
    set_error("lrb_part_pointers: null argument");
    return LRB_EVALUE;
  }
  const PartDev& D = part->d;
  void* v[16] = {D.recv, D.val, D.x, D.r, D.p0, D.p1, D.q, D.b, D.dinv, D.rhat, D.v0, D.v1, D.s, D.t,
                 (void*)D.col, (void*)D.src};
  std::memcpy(ptrs, v, sizeof(v));
  return LRB_OK;
}

static int check_pieces(lrb_part* part, int64_t expect, int32_t n_pieces, const int64_t* piece_len,
                        const char* who, int seg) {
  int64_t tot = 0;
  for (int i = 0; i < n_pieces; ++i) tot += piece_len[i];
  if (tot != expect) {
    set_error(std::string("update pattern violation: ") + who + " " + std::to_string(seg) +
              " delivered " + std::to_string(tot) + " coefficients, pattern expects " +
              std::to_string(expect));
    return LRB_EVALUE;
  }
  return LRB_OK;
}

// H2D of one source segment into the receive buffer (pinned pieces straight,
// pageable ones through the part's pinned stage in overlapped chunks), on
// the segment's stream; returns once the host pieces may be reused.  No
// ordering against the solve: the solve never reads the receive buffer.
static int upload_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                          const int64_t* piece_len, const char* who) {
  if (!part || seg < 0 || seg >= int(part->seg_stream.size())) {
    set_error(std::string(who) + ": bad segment");
    return LRB_EVALUE;
  }
  const int64_t off = part->seg_off[seg], len = part->seg_off[seg + 1] - off;
  int rc = check_pieces(part, len, n_pieces, piece_len, "segment", seg);
  if (rc) return rc;
  DeviceGuard g(part->device);
  cudaStream_t st = part->seg_stream[seg];
  // a whole-buffer scatter on the solve stream (staged update) may still read
  // the receive buffer
  LRB_CUDA(cudaStreamWaitEvent(st, part->staged_done, 0));
  // Per piece: pinned (or registered) host memory goes straight to the
  // device, runs of pieces adjacent in host memory as one copy (a producer
  // writing in pack order into one pinned block); pageable
  // pieces go through the part's pinned stage, host-copying chunk c while the
  // copy engine moves chunk c-1.
  std::vector<char> pinned(size_t(std::max(n_pieces, 0)), 0);
  int n_pinned = 0;
  for (int i = 0; i < n_pieces; ++i) {
    pinned[i] = piece_len[i] == 0 || is_pinned(pieces[i]);
    n_pinned += pinned[i] && piece_len[i] ? 1 : 0;
  }
  double* dst = part->d.recv + off;
  part->stats[0] += n_pinned;
  part->stats[1] += n_pieces - n_pinned;
  part->stats[2] += 8 * len;
  bool staged = false;
  constexpr int64_t kChunkDoubles = int64_t(1) << 19;   // 4 MB
  int64_t o = 0;
  for (int i = 0; i < n_pieces;) {
    if (pinned[i]) {
      const double* src = pieces[i];
      int64_t run = piece_len[i];
      int j = i + 1;
      while (j < n_pieces && pinned[j] && (piece_len[j] == 0 || pieces[j] == src + run)) run += piece_len[j++];
      if (run) LRB_CUDA(cudaMemcpyAsync(dst + o, src, 8 * run, cudaMemcpyHostToDevice, st));
      o += run;
      i = j;
      continue;
    }
    if (!staged) {
      if (!part->stage || part->stage_len < part->seg_off.back()) {
        set_error(std::string(who) + ": pageable input needs a pinned stage");
        return LRB_EVALUE;
      }
      // the previous copy out of this stage slice must have landed
      LRB_CUDA(cudaEventSynchronize(part->seg_h2d[seg]));
      LRB_CUDA(cudaEventSynchronize(part->stage_free));
      staged = true;
    }
    for (int64_t a = 0; a < piece_len[i];) {
      const int64_t take = std::min(piece_len[i] - a, kChunkDoubles);
      std::memcpy(part->stage + off + o, pieces[i] + a, 8 * take);
      LRB_CUDA(cudaMemcpyAsync(dst + o, part->stage + off + o, 8 * take, cudaMemcpyHostToDevice, st));
      a += take;
      o += take;
    }
    ++i;
  }
  LRB_CUDA(cudaEventRecord(part->seg_h2d[seg], st));
  return LRB_OK;
}

// Scatter of one segment on its stream, after the last solve on the part.
static int scatter_segment(lrb_part* part, int32_t seg) {
  DeviceGuard g(part->device);
  cudaStream_t st = part->seg_stream[seg];
  // the scatter rewrites values the last solve may still read
  LRB_CUDA(cudaStreamWaitEvent(st, part->main_done, 0));
  if (!part->seg_rows.empty()) {
    int rc = launch_scatter(part, part->seg_rows[seg], part->seg_rows[seg + 1], st);
    if (rc) return rc;
  }
  std::lock_guard<std::mutex> lk(part->mu);
  LRB_CUDA(cudaEventRecord(part->seg_done[seg], st));
  part->seg_pending[seg] = 1;
  return LRB_OK;
}

int lrb_update_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                       const int64_t* piece_len) {
  int rc = upload_segment(part, seg, n_pieces, pieces, piece_len, "lrb_update_segment");
  if (rc) return rc;
  rc = scatter_segment(part, seg);
  if (rc) return rc;
  // host pieces are reusable once the copy has landed
  DeviceGuard g(part->device);
  LRB_CUDA(cudaEventSynchronize(part->seg_h2d[seg]));
  return LRB_OK;
}

int lrb_update_segments(lrb_part* part, int32_t n_seg, const int32_t* segs, const int32_t* seg_pieces,
                        const double* const* pieces, const int64_t* piece_len) {
  if (!part || n_seg < 0 || (n_seg && (!segs || !seg_pieces))) {
    set_error("lrb_update_segments: bad arguments");
    return LRB_EVALUE;
  }
  int64_t total = 0;
  for (int i = 0; i < n_seg; ++i) {
    if (segs[i] < 0 || segs[i] >= int(part->seg_stream.size())) {
      set_error("lrb_update_segments: bad segment");
      return LRB_EVALUE;
    }
    total += seg_pieces[i];
  }
  for (int64_t i = 0; i < total; ++i)
    if (piece_len[i] && !is_pinned(pieces[i])) {
      set_error("lrb_update_segments: pageable piece (use one lrb_update_segment per source)");
      return LRB_EVALUE;
    }
  // Copies: runs that are contiguous both in host memory and in the receive
  // buffer (consecutive segments whose sources were produced in pack order
  // into one pinned block) merge across pieces and segments; each run goes
  // on the stream of the segment it starts in, and every segment's scatter
  // follows all the runs that fill it.
  DeviceGuard g(part->device);
  int64_t at = 0;
  std::vector<int64_t> seg_at(n_seg + 1, 0);
  for (int i = 0; i < n_seg; ++i) {
    const int64_t off = part->seg_off[segs[i]], len = part->seg_off[segs[i] + 1] - off;
    int rc = check_pieces(part, len, seg_pieces[i], piece_len + at, "segment", segs[i]);
    if (rc) return rc;
    at += seg_pieces[i];
    seg_at[i + 1] = at;
  }
  struct Piece { double* dst; const double* src; int64_t n; int seg; };
  std::vector<Piece> ps;
  for (int i = 0; i < n_seg; ++i) {
    int64_t o = part->seg_off[segs[i]];
    for (int64_t k = seg_at[i]; k < seg_at[i + 1]; ++k) {
      if (piece_len[k]) ps.push_back({part->d.recv + o, pieces[k], piece_len[k], i});
      o += piece_len[k];
    }
    part->stats[0] += seg_pieces[i];
    part->stats[2] += 8 * (part->seg_off[segs[i] + 1] - part->seg_off[segs[i]]);
  }
  for (int i = 0; i < n_seg; ++i) LRB_CUDA(cudaStreamWaitEvent(part->seg_stream[segs[i]], part->staged_done, 0));
  // waits[i]: the other segments whose streams carry a run that fills part of segment i
  std::vector<std::vector<int>> waits(n_seg);
  for (size_t k = 0; k < ps.size();) {
    size_t e = k + 1;
    int64_t run = ps[k].n;
    while (e < ps.size() && ps[e].src == ps[k].src + run && ps[e].dst == ps[k].dst + run) run += ps[e++].n;
    const int home = ps[k].seg;
    LRB_CUDA(cudaMemcpyAsync(ps[k].dst, ps[k].src, 8 * run, cudaMemcpyHostToDevice,
                             part->seg_stream[segs[home]]));
    for (size_t q = k; q < e; ++q) {
      auto& w = waits[ps[q].seg];
      if (ps[q].seg != home && (w.empty() || w.back() != home)) w.push_back(home);
    }
    k = e;
  }
  // each stream's copies are all issued: mark them, then the scatters wait
  for (int i = 0; i < n_seg; ++i)
    LRB_CUDA(cudaEventRecord(part->seg_h2d[segs[i]], part->seg_stream[segs[i]]));
  for (int i = 0; i < n_seg; ++i)
    for (int h : waits[i]) LRB_CUDA(cudaStreamWaitEvent(part->seg_stream[segs[i]], part->seg_h2d[segs[h]], 0));
  for (int i = 0; i < n_seg; ++i) {
    int rc = scatter_segment(part, segs[i]);
    if (rc) return rc;
  }
  for (int i = 0; i < n_seg; ++i) LRB_CUDA(cudaEventSynchronize(part->seg_h2d[segs[i]]));
  return LRB_OK;
}

int lrb_host_register(void* ptr, int64_t bytes) {
  if (!ptr || bytes <= 0) {
    set_error("lrb_host_register: bad range");
    return LRB_EVALUE;
  }
  LRB_CUDA(cudaHostRegister(ptr, size_t(bytes), cudaHostRegisterDefault));
  return LRB_OK;
}

int lrb_host_unregister(void* ptr) {
  if (!ptr) return LRB_OK;
  LRB_CUDA(cudaHostUnregister(ptr));
  return LRB_OK;
}

int lrb_upload_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                       const int64_t* piece_len) {
  int rc = upload_segment(part, seg, n_pieces, pieces, piece_len, "lrb_upload_segment");
  if (rc) return rc;
  DeviceGuard g(part->device);
  LRB_CUDA(cudaEventSynchronize(part->seg_h2d[seg]));
  return LRB_OK;
}

int lrb_scatter_segment(lrb_part* part, int32_t seg) {
  if (!part || seg < 0 || seg >= int(part->seg_stream.size())) {
    set_error("lrb_scatter_segment: bad segment");
    return LRB_EVALUE;
  }
  return scatter_segment(part, seg);
}

int lrb_part_join(lrb_part* part) {
  if (!part) {
    set_error("lrb_part_join: null part");
    return LRB_EVALUE;
  }
  DeviceGuard g(part->device);
  bool any = false;
  std::lock_guard<std::mutex> lk(part->mu);
  for (size_t s = 0; s < part->seg_pending.size(); ++s) {
    if (!part->seg_pending[s]) continue;
    LRB_CUDA(cudaStreamWaitEvent(part->main, part->seg_done[s], 0));
    part->seg_pending[s] = 0;
    any = true;
  }
  if (any && part->seg_rows.empty()) {
    int rc = launch_scatter(part, 0, part->d.n, part->main);
    if (rc) return rc;
    LRB_CUDA(cudaEventRecord(part->staged_done, part->main));
    LRB_CUDA(cudaEventRecord(part->main_done, part->main));
  }
  return LRB_OK;
}

int lrb_update_staged(lrb_part* part, int32_t n_pieces, const double* const* pieces,
                      const int64_t* piece_len) {
  if (!part) {
    set_error("lrb_update_staged: null part");
    return LRB_EVALUE;
  }
  const int64_t total = part->seg_off.back();
  int rc = check_pieces(part, total, n_pieces, piece_len, "owner", 0);
  if (rc) return rc;
  if (!part->stage || part->stage_len < total) {
    set_error("lrb_update_staged: no pinned stage");
    return LRB_EVALUE;
  }
  rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  LRB_CUDA(cudaEventSynchronize(part->stage_free));
  for (size_t s = 0; s < part->seg_h2d.size(); ++s) LRB_CUDA(cudaEventSynchronize(part->seg_h2d[s]));
  int64_t o = 0;
  for (int i = 0; i < n_pieces; ++i) {
    if (piece_len[i] && pieces[i] != part->stage + o)
      std::memcpy(part->stage + o, pieces[i], 8 * piece_len[i]);
    o += piece_len[i];
  }
  if (total)
    LRB_CUDA(cudaMemcpyAsync(part->d.recv, part->stage, 8 * total, cudaMemcpyHostToDevice, part->main));
  LRB_CUDA(cudaEventRecord(part->stage_free, part->main));
  rc = launch_scatter(part, 0, part->d.n, part->main);
  if (rc) return rc;
  LRB_CUDA(cudaEventRecord(part->staged_done, part->main));
  LRB_CUDA(cudaEventRecord(part->main_done, part->main));
  LRB_CUDA(cudaEventSynchronize(part->stage_free));
  return LRB_OK;
}

int lrb_stage_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                      const int64_t* piece_len) {
  if (!part || seg < 0 || seg >= int(part->seg_stream.size())) {
    set_error("lrb_stage_segment: bad segment");
    return LRB_EVALUE;
  }
  const int64_t off = part->seg_off[seg], len = part->seg_off[seg + 1] - off;
  int rc = check_pieces(part, len, n_pieces, piece_len, "segment", seg);
  if (rc) return rc;
  if (!part->stage || part->stage_len < part->seg_off.back()) {
    set_error("lrb_stage_segment: no pinned stage");
    return LRB_EVALUE;
  }
  DeviceGuard g(part->device);
  LRB_CUDA(cudaEventSynchronize(part->stage_free));
  LRB_CUDA(cudaEventSynchronize(part->seg_h2d[seg]));
  int64_t o = 0;
  for (int i = 0; i < n_pieces; ++i) {
    if (piece_len[i]) std::memcpy(part->stage + off + o, pieces[i], 8 * piece_len[i]);
    o += piece_len[i];
  }
  return LRB_OK;
}

int lrb_apply_scatter(lrb_part* part) {
  if (!part) {
    set_error("lrb_apply_scatter: null part");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  rc = launch_scatter(part, 0, part->d.n, part->main);
  if (rc) return rc;
  LRB_CUDA(cudaEventRecord(part->staged_done, part->main));
  LRB_CUDA(cudaEventRecord(part->main_done, part->main));
  return LRB_OK;
}

int lrb_apply_scatter_timed(int32_t n_parts, lrb_part* const* parts, float* device_ms) {
  if (n_parts < 1 || !parts || !device_ms) {
    set_error("lrb_apply_scatter_timed: bad arguments");
    return LRB_EVALUE;
  }
  for (int i = 0; i < n_parts; ++i) {
    if (!parts[i] || parts[i]->device != parts[0]->device) {
      set_error("lrb_apply_scatter_timed: parts must share one CUDA device");
      return LRB_EVALUE;
    }
    int rc = lrb_part_join(parts[i]);
    if (rc) return rc;
  }
  lrb_part* P0 = parts[0];
  DeviceGuard g(P0->device);
  // the start event is recorded right before the first launch and every
  // part's stream starts behind it; the end event after all scatters
  LRB_CUDA(cudaEventRecord(P0->mark_a, P0->main));
  for (int i = 1; i < n_parts; ++i) LRB_CUDA(cudaStreamWaitEvent(parts[i]->main, P0->mark_a, 0));
  for (int i = 0; i < n_parts; ++i) {
    int rc = launch_scatter(parts[i], 0, parts[i]->d.n, parts[i]->main);
    if (rc) return rc;
    LRB_CUDA(cudaEventRecord(parts[i]->staged_done, parts[i]->main));
    LRB_CUDA(cudaEventRecord(parts[i]->main_done, parts[i]->main));
  }
  for (int i = 1; i < n_parts; ++i) LRB_CUDA(cudaStreamWaitEvent(P0->main, parts[i]->main_done, 0));
  LRB_CUDA(cudaEventRecord(P0->mark_b, P0->main));
  LRB_CUDA(cudaEventSynchronize(P0->mark_b));
  LRB_CUDA(cudaEventElapsedTime(device_ms, P0->mark_a, P0->mark_b));
  P0->marks = 0;
  return LRB_OK;
}

int lrb_part_fill(lrb_part* part, int64_t offset, const double* values, int64_t n) {
  if (!part || offset < 0 || n < 0 || offset + n > part->d.n_buf) {
    set_error("device buffer fill out of bounds");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  if (n) LRB_CUDA(cudaMemcpyAsync(part->d.recv + offset, values, 8 * n, cudaMemcpyHostToDevice, part->main));
  LRB_CUDA(cudaStreamSynchronize(part->main));
  return LRB_OK;
}

int lrb_part_read_buffer(lrb_part* part, double* out) {
  if (!part || !out) {
    set_error("lrb_part_read_buffer: null argument");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  if (part->d.n_buf)
    LRB_CUDA(cudaMemcpyAsync(out, part->d.recv, 8 * part->d.n_buf, cudaMemcpyDeviceToHost, part->main));
  LRB_CUDA(cudaStreamSynchronize(part->main));
  return LRB_OK;
}

int lrb_part_read_values(lrb_part* part, double* local_vals, double* nonlocal_vals) {
  if (!part) {
    set_error("lrb_part_read_values: null part");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  const int64_t E = part->slice_ptr.back();
  std::vector<double> sell(E);
  if (E) LRB_CUDA(cudaMemcpyAsync(sell.data(), part->d.val, 8 * E, cudaMemcpyDeviceToHost, part->main));
  LRB_CUDA(cudaStreamSynchronize(part->main));
  if (local_vals)
    for (size_t j = 0; j < part->loc_sell.size(); ++j) local_vals[j] = sell[part->loc_sell[j]];
  if (nonlocal_vals)
    for (size_t j = 0; j < part->nl_sell.size(); ++j) nonlocal_vals[j] = sell[part->nl_sell[j]];
  return LRB_OK;
}

int lrb_part_write_values(lrb_part* part, const double* local_vals, const double* nonlocal_vals) {
  if (!part) {
    set_error("lrb_part_write_values: null part");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  const int64_t E = part->slice_ptr.back();
  std::vector<double> sell(E);
  if (E) LRB_CUDA(cudaMemcpyAsync(sell.data(), part->d.val, 8 * E, cudaMemcpyDeviceToHost, part->main));
  LRB_CUDA(cudaStreamSynchronize(part->main));
  if (local_vals)
    for (size_t j = 0; j < part->loc_sell.size(); ++j) sell[part->loc_sell[j]] = local_vals[j];
  if (nonlocal_vals)
    for (size_t j = 0; j < part->nl_sell.size(); ++j) sell[part->nl_sell[j]] = nonlocal_vals[j];
  if (E) LRB_CUDA(cudaMemcpyAsync(part->d.val, sell.data(), 8 * E, cudaMemcpyHostToDevice, part->main));
  LRB_CUDA(dinv_refresh_launch(part->d, part->main));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  LRB_CUDA(cudaStreamSynchronize(part->main));
  LRB_CUDA(cudaEventRecord(part->main_done, part->main));
  return LRB_OK;
}

int lrb_part_capture_base(lrb_part* part, void* dev_buf, int64_t bytes) {
  if (!part || !dev_buf || bytes < 8 * part->d.n_buf) {
    set_error("lrb_part_capture_base: need a device buffer of 8 * n_buf bytes");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  part->base = static_cast<double*>(dev_buf);
  if (part->d.n_buf)
    LRB_CUDA(cudaMemcpyAsync(part->base, part->d.recv, 8 * part->d.n_buf, cudaMemcpyDeviceToDevice,
                             part->main));
  LRB_CUDA(cudaStreamSynchronize(part->main));
  return LRB_OK;
}

int lrb_update_perturb(lrb_part* part, double diag_scale) {
  if (!part || !part->base) {
    set_error("lrb_update_perturb: no captured base coefficients (lrb_part_capture_base)");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  LRB_CUDA(perturb_launch(part->d, part->base, diag_scale, part->main));
  // a later segment scatter (host update) must land after these values
  LRB_CUDA(cudaEventRecord(part->main_done, part->main));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  part->stats[3] += 1;
  return LRB_OK;
}

int lrb_part_sync(lrb_part* part) {
  if (!part) {
    set_error("lrb_part_sync: null part");
    return LRB_EVALUE;
  }
  int rc = lrb_part_join(part);
  if (rc) return rc;
  DeviceGuard g(part->device);
  LRB_CUDA(cudaStreamSynchronize(part->main));
  for (auto s : part->seg_stream) LRB_CUDA(cudaStreamSynchronize(s));
  return LRB_OK;
}

int lrb_part_stats(const lrb_part* part, int64_t* out) {
  if (!part || !out) {
    set_error("lrb_part_stats: null argument");
    return LRB_EVALUE;
  }
  for (int i = 0; i < 4; ++i) out[i] = part->stats[i].load();
  return LRB_OK;
}

int lrb_part_mark(lrb_part* part) {
  if (!part) {
    set_error("lrb_part_mark: null part");
    return LRB_EVALUE;
  }
  DeviceGuard g(part->device);
  std::swap(part->mark_a, part->mark_b);
  LRB_CUDA(cudaEventRecord(part->mark_b, part->main));
  part->marks++;
  return LRB_OK;
}

int lrb_part_elapsed_ms(lrb_part* part, float* ms) {
  if (!part || !ms || part->marks < 2) {
    set_error("lrb_part_elapsed_ms: need two marks");
    return LRB_EVALUE;
  }
  DeviceGuard g(part->device);
  LRB_CUDA(cudaEventSynchronize(part->mark_b));
  LRB_CUDA(cudaEventElapsedTime(ms, part->mark_a, part->mark_b));
  return LRB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Team
// ---------------------------------------------------------------------------
namespace lrb {

constexpr int kMethods = 5;
// the streaming kernels' static shared memory (team_sync scratch, ~3.2 KB)
// shares the opt-in per-block limit with the dynamic ring
constexpr int64_t kStaticSmemMargin = 4096;

// Largest shared-memory need of any SpMV phase of a method for a staged tile
// with `base` bytes of record + values and `wb` bytes per window vector.
// PIPECG stages its five own-row vectors only on teams whose devices have at
// most one tile per CTA and phase (latency-bound; stream.cuh TAILS)
static bool pipe_staged_tails(int64_t n_tiles) { return n_tiles <= kLanes; }

static int64_t method_need(int method, int64_t base, int64_t wb, bool staged_tails) {
  const int64_t tv = kVecTileBytes;
  switch (method) {
    case LRB_METHOD_BICGSTAB:   // phase 1: r, u = p_old - omega v_old windows + rhat tile
      return base + std::max({2 * wb + tv, 2 * wb, wb + tv});
    case LRB_METHOD_PCG1:       // fused phase: r, dinv, w, s_old windows + p, x tiles
      return base + std::max({4 * wb + 2 * tv, 2 * wb, wb + tv});
    case LRB_METHOD_PIPECG:     // pipelined phase: w, dinv windows (+ z, s, p, x, r tiles)
      return base + std::max({2 * wb + (staged_tails ? 5 : 0) * tv, 2 * wb, wb + tv});
    default:                    // CG / PCG: z, p_old windows (+ x tile); check: x (+ p) windows + b tile
      return base + (LRB_LAZY_X ? 2 * wb + tv : std::max(2 * wb, wb + tv));
  }
}

struct TeamDevice {
  int device = 0;       // CUDA device
  int rank = 0;         // device rank in the team
  std::vector<int> parts;
  int64_t n_tiles = 0;
  bool inl = false;               // local part descriptors in the kernel parameter
  bool cooperative = true;        // whole device to one team kernel
  size_t ws_bytes = 0;
  const void* fn[kMethods] = {};
  int grid[kMethods] = {};          // per method (CG, PCG, BiCGStab, PCG1, PIPECG)
  size_t smem[kMethods] = {};
  int block[kMethods] = {kTPB, kTPB, kTPB, kTPB, kTPB};
  int stage_bytes[kMethods] = {};   // streaming ring per method (BiCGStab / PCG1 / PIPECG stage more)
  int n_stages[kMethods] = {};
  bool streaming[kMethods] = {};    // streaming (bulk-copy) kernel for this method
  cudaStream_t stream = nullptr;  // main stream of the first local part
  void* ws = nullptr;             // device workspace (cudaMalloc, create time)
  TeamDev host{};                 // kernel argument
  PartDev* parts_dev = nullptr;
  SolveOut* out_dev = nullptr;
  double* hist_dev = nullptr;
  int hist_cap = 0;
  long long* prof_dev = nullptr;  // phase timestamps (lrb_team_profile), [0] holds the count
  int prof_cap = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;   // stream-ordered entry points
  bool mirrors = false;           // halo mirrors on (streaming CG/PCG/BiCGStab push, read locally)
  int64_t push_runs = 0;          // halo push runs of the local parts
};

}  // namespace lrb

struct lrb_team {
  std::vector<lrb_part*> parts;     // local parts by team part index (nullptr: remote)
  std::vector<lrb::TeamDevice> devs;
  std::vector<int> dev_of_part;
  std::vector<void*> ipc_opened;    // peer allocations opened via CUDA IPC
  int ipc_dev = -1;
  // set when a cross-device barrier timed out: the devices' barrier epochs and
  // flags no longer agree, so a later solve could pair stale part values
  bool poisoned = false;
  std::mutex mu;
};

namespace lrb {

static const void* solve_kernel(int method, bool inl);
static const void* stream_kernel(int method, bool inl);
static int stream_grid(const void* kernel, int device, int64_t n_tiles, int n_share, size_t smem);
static int stream_stage_bytes(const TeamDevice& D, lrb_part* const* by_index, int* n_stages);
static int64_t tile_geometry(const lrb_part* P, int64_t lt, int part_index, int64_t dev_tile, StageHdr& h);
static void build_stage_headers(const TeamDevice& D, lrb_part* const* by_index, int stage_bytes,
                                std::vector<StageHdr>& out, std::vector<StageTab>& tabs);
static int solver_choice();
static int max_grid(const void* kernel, int device, int64_t n_tiles, int n_share,
                    int64_t stage_doubles, size_t* smem);

// Halo push plan of a team (SURVEY §8 e: the halo exchange).  For every part
// p, the runs of its rows that other parts read as halo operands, from the
// readers' hpart/hidx tables (device, peer or IPC memory; read once at team
// creation): {row_lo, row_hi, reader part, reader's halo slot of row_lo},
// rows and slots consecutive along a run.  Mirrors are on for the team iff
// every part has at most kMaxSndRuns runs (slab partitions: <= 2 per
// neighbour); the decision depends only on team-wide data, so every process
// of a multi-process team takes the same one.  LRB_HALO=direct turns them
// off (remote loads inside the SpMV, the round-1 data path).
struct HaloPush {
  bool on = false;
  std::vector<std::vector<int64_t>> runs;            // [part] 4 per run
  std::vector<std::pair<int64_t, int64_t>> quiet;    // [part] largest row range with no run
};

static int plan_halo_push(const std::vector<PartDev>& table, HaloPush& hp) {
  const int np = int(table.size());
  hp.runs.assign(np, {});
  hp.quiet.assign(np, {0, 0});
  const char* env = getenv("LRB_HALO");
  hp.on = !(env && std::strcmp(env, "direct") == 0);
  for (int q = 0; q < np && hp.on; ++q) {
    const PartDev& Q = table[q];
    if (!Q.n_halo) continue;
    if (!Q.hm) {
      hp.on = false;
      break;
    }
    std::vector<int32_t> hpart(Q.n_halo), hidx(Q.n_halo);
    LRB_CUDA(cudaMemcpy(hpart.data(), Q.hpart, sizeof(int32_t) * Q.n_halo, cudaMemcpyDefault));
    LRB_CUDA(cudaMemcpy(hidx.data(), Q.hidx, sizeof(int32_t) * Q.n_halo, cudaMemcpyDefault));
    for (int64_t h = 0; h < Q.n_halo;) {
      const int p = hpart[h];
      int64_t e = h + 1;
      while (e < Q.n_halo && hpart[e] == p && int64_t(hidx[e]) == hidx[h] + (e - h)) ++e;
      if (p < 0 || p >= np || p == q) {
        set_error("lrb_team_create: halo slot owned by an invalid part");
        return LRB_EVALUE;
      }
      auto& R = hp.runs[p];
      R.insert(R.end(), {int64_t(hidx[h]), int64_t(hidx[h]) + (e - h), int64_t(q), h});
      if (int64_t(R.size()) / 4 > kMaxSndRuns) hp.on = false;
      h = e;
    }
  }
  if (!hp.on) {
    for (auto& R : hp.runs) R.clear();
    return LRB_OK;
  }
  for (int p = 0; p < np; ++p) {   // largest gap between the runs: the no-push interval
    std::vector<std::pair<int64_t, int64_t>> iv;
    for (size_t k = 0; k < hp.runs[p].size(); k += 4) iv.emplace_back(hp.runs[p][k], hp.runs[p][k + 1]);
    std::sort(iv.begin(), iv.end());
    int64_t cur = 0, best_lo = 0, best_hi = 0;
    for (auto& r : iv) {
      if (r.first - cur > best_hi - best_lo) best_lo = cur, best_hi = r.first;
      cur = std::max(cur, r.second);
    }
    if (table[p].n - cur > best_hi - best_lo) best_lo = cur, best_hi = table[p].n;
    hp.quiet[p] = {best_lo, best_hi};
  }
  return LRB_OK;
}

// Workspace, tile map, launch geometry of one device of a team.  table holds
// every team part's descriptor; local parts get their tile ranges here.
static int setup_device(TeamDevice& D, std::vector<PartDev>& table, lrb_part* const* by_index,
                        int n_parts, int n_dev, int n_share, const HaloPush& hp) {
  int64_t t = 0;
  int64_t n_runs = 0;
  for (int p : D.parts) {
    lrb_part* P = by_index[p];
    P->d.tile0 = t;
    P->d.ntiles = (P->d.n + kTile - 1) / kTile;
    t += P->d.ntiles;
    table[p] = P->d;
    table[p].mir = hp.on && table[p].n_halo > 0;
    n_runs += hp.on ? int64_t(hp.runs[p].size()) / 4 : 0;
  }
  D.n_tiles = t;
  DeviceGuard g(D.device);
  D.stream = by_index[D.parts.front()]->main;
  const int64_t n_tiles = std::max<int64_t>(D.n_tiles, 1);
  size_t bytes = 0;
  auto take = [&](size_t b) {
    size_t at = bytes;
    bytes = (bytes + b + 255) & ~size_t(255);
    return at;
  };
  const size_t o_parts = take(sizeof(PartDev) * n_parts);
  const size_t o_tp = take(sizeof(int32_t) * n_tiles);
  const size_t o_partials = take(sizeof(double) * kMaxRed * n_tiles);
  const size_t o_lanes = take(sizeof(double) * kMaxRed * kLanes * 2);   // lane_fast: one part
  const size_t o_pred = take(sizeof(double) * kMaxRed * n_parts * 2);  // epoch parity
  const size_t o_red = take(sizeof(double) * kMaxRed);
  const size_t o_epoch = take(sizeof(unsigned long long));
  const size_t o_flags = take(sizeof(unsigned long long) * n_dev);
  const size_t o_peer_flags = take(sizeof(void*) * n_dev);
  const size_t o_peer_red = take(sizeof(void*) * n_dev);
  const size_t o_out = take(sizeof(SolveOut));
  const size_t o_snd = take(sizeof(int64_t) * 4 * std::max<int64_t>(n_runs, 1));
  // streaming solvers: stage size from the largest stageable tile, and the
  // per-tile stage headers
  const bool want_stream = solver_choice() != 1;
  int n_stages = 0;
  // computed for the classic kernels too: the stage geometry fixes the
  // reduction tree's units (pack_factor), so both families stay bit-identical
  const int stage_bytes = stream_stage_bytes(D, by_index, &n_stages);
  // the ring needs a stage per issuer and per consumer team in flight
  const bool use_stream = want_stream && n_stages >= std::max(kTeams, kIssuers);
  const size_t o_hdr = use_stream ? take(sizeof(StageHdr) * n_tiles) : 0;
  const size_t o_rec = use_stream ? take(sizeof(TileRec) * n_tiles) : 0;
  LRB_CUDA(cudaMalloc(&D.ws, bytes));
  LRB_CUDA(cudaMemset(D.ws, 0, bytes));
  D.ws_bytes = bytes;
  char* w = static_cast<char*>(D.ws);
  D.parts_dev = reinterpret_cast<PartDev*>(w + o_parts);
  D.out_dev = reinterpret_cast<SolveOut*>(w + o_out);
  TeamDev& H = D.host;
  H.n_parts = n_parts;
  H.dev_rank = D.rank;
  H.n_dev = n_dev;
  H.part_begin = D.parts.front();
  H.part_end = D.parts.back() + 1;
  H.n_tiles = D.n_tiles;
  H.parts = D.parts_dev;
  H.tile_part = reinterpret_cast<int32_t*>(w + o_tp);
  H.partials = reinterpret_cast<double*>(w + o_partials);
  H.lane_vals = reinterpret_cast<double*>(w + o_lanes);
  H.lane_fast = 0;
  H.part_red = reinterpret_cast<double*>(w + o_pred);
  H.red = reinterpret_cast<double*>(w + o_red);
  H.epoch = reinterpret_cast<unsigned long long*>(w + o_epoch);
  H.flags = reinterpret_cast<unsigned long long*>(w + o_flags);
  H.peer_flags = reinterpret_cast<unsigned long long**>(w + o_peer_flags);
  H.peer_part_red = reinterpret_cast<double**>(w + o_peer_red);
  H.out = D.out_dev;
  // halo push runs of the local parts
  {
    int64_t* snd = reinterpret_cast<int64_t*>(w + o_snd);
    int64_t at = 0;
    for (size_t q = 0; q < D.parts.size(); ++q) {
      const int p = D.parts[q];
      PartDev& E = table[p];
      const int64_t nr = hp.on ? int64_t(hp.runs[p].size()) / 4 : 0;
      E.snd = nr ? snd + 4 * at : nullptr;
      E.n_snd = int32_t(nr);
      E.sq_lo = hp.on ? hp.quiet[p].first : 0;
      E.sq_hi = hp.on ? hp.quiet[p].second : E.n;
      if (nr)
        LRB_CUDA(cudaMemcpy(snd + 4 * at, hp.runs[p].data(), sizeof(int64_t) * 4 * nr, cudaMemcpyHostToDevice));
      at += nr;
    }
    D.mirrors = hp.on;
    D.push_runs = at;
  }
  {
    const char* env = getenv("LRB_BARRIER_TIMEOUT_S");
    const double s = env ? atof(env) : 20.0;
    H.timeout_ns = (long long)((s > 0 ? s : 20.0) * 1e9);
  }
  std::vector<int32_t> tp(n_tiles, 0);
  for (int p : D.parts)
    for (int64_t q = 0; q < by_index[p]->d.ntiles; ++q) tp[by_index[p]->d.tile0 + q] = p;
  LRB_CUDA(cudaMemcpy((void*)H.tile_part, tp.data(), sizeof(int32_t) * n_tiles, cudaMemcpyHostToDevice));
  LRB_CUDA(cudaEventCreate(&D.t0));
  LRB_CUDA(cudaEventCreate(&D.t1));
  LRB_CUDA(cudaEventCreateWithFlags(&D.ev_in, cudaEventDisableTiming));
  LRB_CUDA(cudaEventCreateWithFlags(&D.ev_out, cudaEventDisableTiming));
  D.inl = int(D.parts.size()) <= kInlineParts;
  if (D.inl)
    for (size_t q = 0; q < D.parts.size(); ++q) H.lp[q] = table[D.parts[q]];
  D.cooperative = (n_share == 1);
  const int64_t stage = 0;   // classic kernels: no staged operand
  H.stage_bytes = stage_bytes;
  H.n_stages = n_stages;
  H.tile_hdr = nullptr;
  H.tile_rec = nullptr;
  if (use_stream) {
    std::vector<StageHdr> hdr;
    std::vector<StageTab> tab;
    build_stage_headers(D, by_index, stage_bytes, hdr, tab);
    std::vector<TileRec> rec(hdr.size());
    for (size_t t = 0; t < hdr.size(); ++t) {
      rec[t].h = hdr[t];
      rec[t].t = tab[t];
      std::memset(rec[t].mask, 0, sizeof(rec[t].mask));
    }
    for (int p : D.parts) {
      const lrb_part* P = by_index[p];
      for (int64_t lt = 0; lt < P->d.ntiles; ++lt) {
        TileRec& r = rec[P->d.tile0 + lt];
        const int64_t row0 = lt * kTile, rows = std::min<int64_t>(kTile, P->d.n - row0);
        if (int64_t(P->rmask_host.size()) >= row0 + rows)
          std::memcpy(r.mask, P->rmask_host.data() + row0, sizeof(uint16_t) * rows);
      }
    }
    H.tile_hdr = w + o_hdr;
    H.tile_rec = w + o_rec;
    LRB_CUDA(cudaMemcpy(w + o_hdr, hdr.data(), sizeof(StageHdr) * hdr.size(), cudaMemcpyHostToDevice));
    LRB_CUDA(cudaMemcpy(w + o_rec, rec.data(), sizeof(TileRec) * rec.size(), cudaMemcpyHostToDevice));
  }
  // BiCGStab and PCG1 stage more windows than CG: their own, larger rings over
  // the same stageable tiles (no streaming kernel if two stages do not fit)
  int m_bytes[kMethods] = {}, m_stages[kMethods] = {};
  if (n_stages >= std::max(kTeams, kIssuers)) {
    int dev_smem = 0;
    cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, D.device);
    const int64_t budget = int64_t(dev_smem) - int64_t(stream_smem_bytes(0, 0)) - kStaticSmemMargin;
    for (int m = LRB_METHOD_BICGSTAB; m < kMethods; ++m) {
      int64_t best = 3 * (kHdrBytes + 5 * int64_t(kVecTileBytes));
      StageHdr h;
      for (int p : D.parts) {
        const lrb_part* P = by_index[p];
        for (int64_t lt = 0; lt < P->d.ntiles; ++lt) {
          const int64_t need = tile_geometry(P, lt, p, 0, h);
          if (need <= 0 || need > stage_bytes) continue;   // not staged (direct loads)
          best = std::max(best, method_need(m, kRecBytes + h.vbytes, int64_t(h.wtot) * 8,
                                            pipe_staged_tails(D.n_tiles)));
        }
      }
      best = (best + 127) & ~int64_t(127);
      const int64_t n = std::min<int64_t>(kStreamMaxStages, budget / best);
      if (n >= std::max(kTeams, kIssuers)) {
        m_bytes[m] = int(best);
        m_stages[m] = int(n);
      }
    }
    m_bytes[LRB_METHOD_CG] = m_bytes[LRB_METHOD_PCG] = stage_bytes;
    m_stages[LRB_METHOD_CG] = m_stages[LRB_METHOD_PCG] = n_stages;
  }
  for (int m = 0; m < kMethods; ++m) {
    const void* sfn = (use_stream && m_stages[m])
                          ? (m == LRB_METHOD_PIPECG && pipe_staged_tails(D.n_tiles) ? pipecg_t_stream_kernel(D.inl)
                                                                                   : stream_kernel(m, D.inl))
                          : nullptr;
    if (sfn) {
      D.fn[m] = sfn;
      D.block[m] = kStreamThreads;
      D.streaming[m] = true;
      D.stage_bytes[m] = m_bytes[m];
      D.n_stages[m] = m_stages[m];
      D.smem[m] = stream_smem_bytes(D.stage_bytes[m], D.n_stages[m]);
      D.grid[m] = stream_grid(sfn, D.device, D.n_tiles, n_share, D.smem[m]);
    } else {
      D.stage_bytes[m] = m_bytes[m];   // the reduction tree's units (classic kernels)
      D.fn[m] = solve_kernel(m, D.inl);
      if (!D.fn[m]) continue;   // PCG1 / PIPECG exist only as streaming kernels
      D.grid[m] = max_grid(D.fn[m], D.device, D.n_tiles, n_share, stage, &D.smem[m]);
    }
    if (D.grid[m] <= 0) {
      set_error("lrb_team_create: cannot size the persistent grid of method " + std::to_string(m) +
                " (" + (D.streaming[m] ? "streaming" : "classic") + ", dynamic smem " +
                std::to_string(D.smem[m]) + " B, status " + std::to_string(D.grid[m]) + ": " +
                cudaGetErrorString(cudaGetLastError()) + ")");
      return LRB_ERUNTIME;
    }
  }
  return LRB_OK;
}

// Every device's copy of the part table, the flag and part-value peer tables.
static int publish_tables(TeamDevice& D, const std::vector<PartDev>& table,
                          const std::vector<void*>& pf, const std::vector<void*>& pr) {
  DeviceGuard g(D.device);
  const int n_dev = int(pf.size());
  LRB_CUDA(cudaMemcpy(D.parts_dev, table.data(), sizeof(PartDev) * table.size(), cudaMemcpyHostToDevice));
  LRB_CUDA(cudaMemcpy(D.host.peer_flags, pf.data(), sizeof(void*) * n_dev, cudaMemcpyHostToDevice));
  LRB_CUDA(cudaMemcpy(D.host.peer_part_red, pr.data(), sizeof(void*) * n_dev, cudaMemcpyHostToDevice));
  return LRB_OK;
}

}  // namespace lrb

namespace lrb {

static int team_hist_capacity(TeamDevice& D, int cap) {
  if (cap <= D.hist_cap) return LRB_OK;
  DeviceGuard g(D.device);
  if (D.hist_dev) cudaFree(D.hist_dev);
  D.hist_dev = nullptr;
  LRB_CUDA(cudaMalloc(&D.hist_dev, sizeof(double) * cap));
  D.hist_cap = cap;
  return LRB_OK;
}

static const void* solve_kernel(int method, bool inl) {
  switch (method) {
    case LRB_METHOD_CG:
      return cg_classic_kernel(false, inl);
    case LRB_METHOD_PCG:
      return cg_classic_kernel(true, inl);
    case LRB_METHOD_BICGSTAB:
      return bicgstab_classic_kernel(inl);
    default:
      return nullptr;
  }
}

// Largest co-resident grid (one wave) for a persistent team kernel; the
// dynamic shared memory holds the warp partials of the block's tiles.
static int max_grid(const void* kernel, int device, int64_t n_tiles, int n_share,
                    int64_t stage_doubles, size_t* smem) {
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  const int64_t tiles = std::max<int64_t>(n_tiles, 1);
  const size_t stage = size_t(stage_doubles) * sizeof(double);
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) !=
      cudaSuccess)
    return -1;
  // start from the register-limited occupancy, shrink until the shared memory
  // of the resulting tiles-per-block fits as well
  for (int per_sm = 32; per_sm >= 1; --per_sm) {
    const int64_t cap = int64_t(sms) * per_sm / std::max(n_share, 1);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(cap, tiles)));
    const size_t need = phase_smem_bytes((tiles + grid - 1) / grid) + stage;
    if (need > 200 * 1024) continue;
    int fit = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kernel, kTPB, need) != cudaSuccess)
      return -1;
    if (int64_t(fit) * sms / std::max(n_share, 1) >= grid) {   // one co-resident wave
      *smem = std::max(*smem, need);
      return grid;
    }
  }
  return -2;
}

// LRB_SOLVER=classic selects the per-thread-gather kernels (kernels.cuh);
// default: the streaming kernels (stream.cuh) where a method has one.
static int solver_choice() {
  const char* e = getenv("LRB_SOLVER");
  if (e && std::strcmp(e, "classic") == 0) return 1;
  return 0;
}

static const void* stream_kernel(int method, bool inl) {
  switch (method) {
    case LRB_METHOD_CG:
      return cg_stream_kernel(false, inl);
    case LRB_METHOD_PCG:
      return cg_stream_kernel(true, inl);
    case LRB_METHOD_BICGSTAB:
      return bicgstab_stream_kernel(inl);
    case LRB_METHOD_PCG1:
      return pcg1_stream_kernel(inl);
    case LRB_METHOD_PIPECG:
      return pipecg_stream_kernel(inl);
    default:
      return nullptr;
  }
}

// Geometry of one tile as the streaming producer stages it (StageHdr without
// the staging decision); need = the largest stage any phase asks for.
static int64_t tile_geometry(const lrb_part* P, int64_t lt, int part_index, int64_t dev_tile,
                             StageHdr& h) {
  std::memset(&h, 0, sizeof(h));
  const int64_t n = P->d.n;
  const int64_t row0 = lt * kTile, rows = std::min<int64_t>(kTile, n - row0);
  const int64_t s0 = row0 / kSlice, s1 = (row0 + rows + kSlice - 1) / kSlice;
  h.row0 = row0;
  h.rows = int32_t(rows);
  h.part = part_index;
  h.tile = int32_t(dev_tile);
  h.e0 = P->slice_ptr[s0];
  h.vbytes = int32_t(8 * (P->slice_ptr[s1] - P->slice_ptr[s0]));
  h.halo = (lt < int64_t(P->tile_halo.size()) && P->tile_halo[lt]) ? 1 : 0;
  for (int64_t s = s0; s <= s1; ++s) h.sp[s - s0] = int32_t(P->slice_ptr[s] - P->slice_ptr[s0]);
  const bool have_win = int64_t(P->tile_win.size()) >= (lt + 1) * kWinStride;
  const int32_t* tw = have_win ? &P->tile_win[lt * kWinStride] : nullptr;
  h.nw = tw ? tw[0] : 0;
  int64_t wtot = 0;
  for (int w = 0; w < h.nw; ++w) {
    const int64_t a = row0 + tw[2 + 2 * w], l = tw[3 + 2 * w];
    const int64_t a2 = a & ~int64_t(1), b2 = (a + l + 1) & ~int64_t(1);
    h.wa[w] = a2;
    h.wl[w] = int32_t(b2 - a2);
    h.woff[w] = int32_t(wtot);
    wtot += b2 - a2;
  }
  h.wtot = int32_t(wtot);
  if (h.nw <= 0) return 0;
  const int64_t base = kRecBytes + h.vbytes;
  // CG / PCG: z, p_old windows (+ the x tile when its update is pending,
  // LRB_LAZY_X); the check phase: x (+ p) windows + the b tile
  return LRB_LAZY_X ? base + 2 * wtot * 8 + kVecTileBytes
                    : std::max(base + 2 * wtot * 8, base + wtot * 8 + kVecTileBytes);
}

// Largest stage any phase needs for a stageable tile of this device's parts,
// and how many stages fit in shared memory (at least two, else no streaming).
static int stream_stage_bytes(const TeamDevice& D, lrb_part* const* by_index, int* n_stages) {
  int dev_smem = 0;
  cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, D.device);
  const int64_t budget = int64_t(dev_smem) - int64_t(stream_smem_bytes(0, 0)) - kStaticSmemMargin;
  const int64_t cap = budget / 2;   // at least double-buffered
  int64_t best = kHdrBytes + 5 * kVecTileBytes;   // elementwise phases
  StageHdr h;
  for (int p : D.parts) {
    const lrb_part* P = by_index[p];
    const int64_t ntiles = (P->d.n + kTile - 1) / kTile;
    for (int64_t lt = 0; lt < ntiles; ++lt) {
      const int64_t need = tile_geometry(P, lt, p, 0, h);
      if (need > 0 && need <= cap) best = std::max(best, need);
    }
  }
  best = (best + 127) & ~int64_t(127);
  int64_t n = std::min<int64_t>(kStreamMaxStages, budget / best);
  // grow the stage to pack 3 elementwise tiles when that keeps the ring depth
  const int64_t packed = (3 * (kHdrBytes + 5 * int64_t(kVecTileBytes)) + 127) & ~int64_t(127);
  if (packed > best && std::min<int64_t>(kStreamMaxStages, budget / packed) >= n) best = packed;
  int64_t stages = std::min<int64_t>(kStreamMaxStages, budget / best);
  if (const char* e = getenv("LRB_STREAM_STAGES")) {   // experiments: cap the ring depth
    const int64_t cap_n = atoi(e);
    if (cap_n >= 2) stages = std::min(stages, cap_n);
  }
  *n_stages = int(stages);
  return int(best);
}

// One StageHdr + StageTab per device tile; tiles without windows, larger
// than a stage, or with more than kHdrPats distinct slice patterns are marked
// for the consumers' direct-load path (tma = 0).
static void build_stage_headers(const TeamDevice& D, lrb_part* const* by_index, int stage_bytes,
                                std::vector<StageHdr>& out, std::vector<StageTab>& tabs) {
  out.assign(size_t(std::max<int64_t>(D.n_tiles, 1)), StageHdr{});
  tabs.assign(out.size(), StageTab{});
  for (int p : D.parts) {
    const lrb_part* P = by_index[p];
    const int64_t n = P->d.n;
    for (int64_t lt = 0; lt < P->d.ntiles; ++lt) {
      StageHdr& h = out[P->d.tile0 + lt];
      StageTab& tb = tabs[P->d.tile0 + lt];
      const int64_t need = tile_geometry(P, lt, p, P->d.tile0 + lt, h);
      h.tma = (need > 0 && need <= stage_bytes) ? 1 : 0;
      const int64_t s0 = h.row0 / kSlice, nsl = (h.rows + kSlice - 1) / kSlice;
      std::vector<int32_t> local;   // distinct pattern ids, first-seen order
      for (int64_t s = 0; s < nsl; ++s) {
        const int32_t pid = P->slice_pat_host[s0 + s];
        h.pat[s] = pid;
        auto it = std::find(local.begin(), local.end(), pid);
        if (it == local.end()) {
          local.push_back(pid);
          it = local.end() - 1;
        }
        h.spat[s] = int8_t(std::min<int64_t>(it - local.begin(), kHdrPats - 1));
      }
      if (int(local.size()) > kHdrPats) h.tma = 0;
      h.npat = int32_t(std::min<size_t>(local.size(), kHdrPats));
      if (!h.tma) continue;
      for (int j = 0; j < h.npat; ++j) {
        h.sdiag[j] = -1;
        if (local[j] < 0) {
          h.tma = 0;
          break;
        }
        for (int k = 0; k < kPatW; ++k) {
          const int32_t off = P->pat_off_host[size_t(local[j]) * kPatW + k];
          // the window holding this offset's local columns (one per tile)
          const int64_t c = std::min<int64_t>(std::max<int64_t>(h.row0 + off, 0), n - 1);
          int32_t e = 0;
          for (int w = 0; w < h.nw; ++w)
            if (c >= h.wa[w] && c < h.wa[w] + h.wl[w]) e = int32_t(h.woff[w] - h.wa[w] + off);
          tb.off[j][k] = off;
          tb.del[j][k] = e;
          if (off == 0 && h.sdiag[j] < 0) h.sdiag[j] = int8_t(k);
        }
      }
    }
  }
}

static int stream_grid(const void* kernel, int device, int64_t n_tiles, int n_share, size_t smem) {
  int sms = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess)
    return -1;
  // The attribute is per kernel FUNCTION, shared by every team: set it to the
  // most any launch may ask for (opt-in limit minus the kernel's static
  // shared memory), never to this team's need — a later team with smaller
  // stages must not shrink it under an earlier team's launches.
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) return -1;
  const int cap_smem = optin - int(fa.sharedSizeBytes);
  if (int64_t(smem) > cap_smem) return -3;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, cap_smem) != cudaSuccess)
    return -1;
  int fit = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kernel, kStreamThreads, smem) != cudaSuccess ||
      fit < 1)
    return -2;
  const int64_t cap = int64_t(sms) * fit / std::max(n_share, 1);
  return int(std::max<int64_t>(1, std::min<int64_t>(cap, std::max<int64_t>(n_tiles, 1))));
}

}  // namespace lrb

extern "C" {

// dev_rank_of_part (nullable): explicit device rank per part; parts sharing a
// CUDA device but given different ranks run as separate kernels (used by the
// tests to exercise the cross-device protocol on one GPU).
int lrb_team_create_ex(int32_t n_parts, lrb_part* const* parts, const int32_t* dev_rank_of_part,
                       lrb_team** out) {
  if (n_parts < 1 || !parts || !out) {
    set_error("lrb_team_create: bad arguments");
    return LRB_EVALUE;
  }
  auto team = std::make_unique<lrb_team>();
  team->parts.assign(parts, parts + n_parts);
  // device ranks: by explicit map, else by CUDA device in order of appearance
  std::vector<int> rank_of(n_parts);
  std::map<int, int> seen;
  for (int p = 0; p < n_parts; ++p) {
    int key = dev_rank_of_part ? dev_rank_of_part[p] : parts[p]->device;
    auto it = seen.find(key);
    if (it == seen.end()) it = seen.emplace(key, int(seen.size())).first;
    rank_of[p] = it->second;
  }
  const int n_dev = int(seen.size());
  team->devs.resize(n_dev);
  team->dev_of_part = rank_of;
  for (int p = 0; p < n_parts; ++p) {
    auto& D = team->devs[rank_of[p]];
    if (!D.parts.empty() && parts[D.parts.back()]->device != parts[p]->device) {
      set_error("lrb_team_create: parts of one device rank must share a CUDA device");
      return LRB_EVALUE;
    }
    if (!D.parts.empty() && D.parts.back() != p - 1) {
      set_error("lrb_team_create: parts of one device must be consecutive GPU ranks");
      return LRB_EVALUE;
    }
    D.parts.push_back(p);
    D.device = parts[p]->device;
    D.rank = rank_of[p];
  }
  // physical sharing (several device ranks on one CUDA device)
  std::map<int, int> share;
  for (auto& D : team->devs) share[D.device]++;
  // peer access between distinct devices
  for (auto& A : team->devs)
    for (auto& B : team->devs)
      if (A.device != B.device) {
        DeviceGuard g(A.device);
        int can = 0;
        LRB_CUDA(cudaDeviceCanAccessPeer(&can, A.device, B.device));
        if (!can) {
          set_error("lrb_team_create: no peer access between devices");
          return LRB_EVALUE;
        }
        cudaError_t e = cudaDeviceEnablePeerAccess(B.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          set_error(std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
          return LRB_ECUDA;
        }
        cudaGetLastError();
      }
  // per-device workspace, then the shared part / peer tables
  std::vector<PartDev> table(n_parts);
  for (int p = 0; p < n_parts; ++p) table[p] = parts[p]->d;
  HaloPush hp;
  int rc0 = plan_halo_push(table, hp);
  if (rc0) return rc0;
  for (auto& D : team->devs) {
    int rc = setup_device(D, table, parts, n_parts, n_dev, share[D.device], hp);
    if (rc) return rc;
  }
  std::vector<void*> pf(n_dev), pr(n_dev);
  for (auto& D : team->devs) {
    pf[D.rank] = D.host.flags;
    pr[D.rank] = D.host.part_red;
  }
  for (auto& D : team->devs) {
    int rc = publish_tables(D, table, pf, pr);
    if (rc) return rc;
  }
  *out = team.release();
  return LRB_OK;
}

}  // extern "C"

// ---- multi-process teams (CUDA IPC) ---------------------------------------
namespace {

struct PartBlob {   // fixed layout inside LRB_BLOB_BYTES
  char magic[8];
  cudaIpcMemHandle_t arena;
  int64_t arena_off;      // offset of the arena start inside the IPC allocation
  PartDev d;              // pointers rewritten as offsets from the arena start
};
struct TeamBlob {
  char magic[8];
  cudaIpcMemHandle_t ws;
  int64_t flags_off, part_red_off;
};
static_assert(sizeof(PartBlob) <= LRB_BLOB_BYTES, "blob too small");
static_assert(sizeof(TeamBlob) <= LRB_BLOB_BYTES, "blob too small");

template <class T>
T* rebase(T* p, const char* from, char* to) {
  return p ? reinterpret_cast<T*>(to + (reinterpret_cast<const char*>(p) - from)) : nullptr;
}

// base of the cudaMalloc allocation containing p (driver API, loaded lazily so
// the library still loads on machines without a driver)
int alloc_base(const void* p, char** base) {
  typedef int (*fn_t)(unsigned long long*, size_t*, unsigned long long);
  static fn_t fn = nullptr;
  if (!fn) {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (h) fn = reinterpret_cast<fn_t>(dlsym(h, "cuMemGetAddressRange_v2"));
    if (!fn) {
      set_error("cuMemGetAddressRange_v2 unavailable");
      return LRB_ECUDA;
    }
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) {
    set_error("cuMemGetAddressRange failed");
    return LRB_ECUDA;
  }
  *base = reinterpret_cast<char*>(b);
  return LRB_OK;
}

}  // namespace

extern "C" {

int lrb_part_export(const lrb_part* part, void* blob) {
  if (!part || !blob) {
    set_error("lrb_part_export: null argument");
    return LRB_EVALUE;
  }
  DeviceGuard g(part->device);
  std::memset(blob, 0, LRB_BLOB_BYTES);
  PartBlob b{};
  std::memcpy(b.magic, "LRBPART", 8);
  char* arena = const_cast<char*>(reinterpret_cast<const char*>(part->d.slice_ptr));
  char* base = nullptr;
  int rc = alloc_base(arena, &base);
  if (rc) return rc;
  LRB_CUDA(cudaIpcGetMemHandle(&b.arena, base));
  b.arena_off = arena - base;
  b.d = part->d;
  // pointers -> offsets from the arena start (rebased by the importer)
  char* zero = nullptr;
  PartDev& d = b.d;
  d.slice_ptr = rebase(d.slice_ptr, arena, zero);
  d.slice_pat = rebase(d.slice_pat, arena, zero);
  d.pat_off = rebase(d.pat_off, arena, zero);
  d.rmask = rebase(d.rmask, arena, zero);
  d.col = rebase(d.col, arena, zero);
  d.src = rebase(d.src, arena, zero);
  d.dpos = rebase(d.dpos, arena, zero);
  d.hpart = rebase(d.hpart, arena, zero);
  d.hidx = rebase(d.hidx, arena, zero);
  d.hm = rebase(d.hm, arena, zero);
  d.val = rebase(d.val, arena, zero);
  d.recv = rebase(d.recv, arena, zero);
  for (double** v : {&d.x, &d.r, &d.p0, &d.p1, &d.q, &d.b, &d.dinv, &d.rhat, &d.v0, &d.v1, &d.s, &d.t})
    *v = rebase(*v, arena, zero);
  std::memcpy(blob, &b, sizeof(b));
  return LRB_OK;
}

int lrb_team_create_ipc(int32_t n_parts, int32_t part_begin, int32_t n_local,
                        lrb_part* const* local_parts, const void* part_blobs, int32_t dev_rank,
                        int32_t n_dev, lrb_team** out, void* team_blob) {
  if (n_parts < 1 || n_local < 1 || part_begin < 0 || part_begin + n_local > n_parts ||
      !local_parts || !part_blobs || !out || !team_blob || dev_rank < 0 || dev_rank >= n_dev) {
    set_error("lrb_team_create_ipc: bad arguments");
    return LRB_EVALUE;
  }
  const int device = local_parts[0]->device;
  for (int i = 0; i < n_local; ++i)
    if (local_parts[i]->device != device) {
      set_error("lrb_team_create_ipc: local parts must share one CUDA device");
      return LRB_EVALUE;
    }
  DeviceGuard g(device);
  auto team = std::make_unique<lrb_team>();
  team->ipc_dev = device;
  team->parts.assign(n_parts, nullptr);
  for (int i = 0; i < n_local; ++i) team->parts[part_begin + i] = local_parts[i];
  std::vector<PartDev> table(n_parts);
  const char* blobs = static_cast<const char*>(part_blobs);
  for (int p = 0; p < n_parts; ++p) {
    if (p >= part_begin && p < part_begin + n_local) continue;
    PartBlob b;
    std::memcpy(&b, blobs + size_t(p) * LRB_BLOB_BYTES, sizeof(b));
    if (std::memcmp(b.magic, "LRBPART", 8) != 0) {
      set_error("lrb_team_create_ipc: bad part blob");
      return LRB_EVALUE;
    }
    void* base = nullptr;
    LRB_CUDA(cudaIpcOpenMemHandle(&base, b.arena, cudaIpcMemLazyEnablePeerAccess));
    team->ipc_opened.push_back(base);
    char* arena = static_cast<char*>(base) + b.arena_off;
    PartDev d = b.d;
    const char* zero = nullptr;
    d.slice_ptr = rebase(d.slice_ptr, zero, arena);
    d.slice_pat = rebase(d.slice_pat, zero, arena);
    d.pat_off = rebase(d.pat_off, zero, arena);
    d.rmask = rebase(d.rmask, zero, arena);
    d.col = rebase(d.col, zero, arena);
    d.src = rebase(d.src, zero, arena);
    d.dpos = rebase(d.dpos, zero, arena);
    d.hpart = rebase(d.hpart, zero, arena);
    d.hidx = rebase(d.hidx, zero, arena);
    d.hm = rebase(d.hm, zero, arena);
    d.val = rebase(d.val, zero, arena);
    d.recv = rebase(d.recv, zero, arena);
    for (double** v : {&d.x, &d.r, &d.p0, &d.p1, &d.q, &d.b, &d.dinv, &d.rhat, &d.v0, &d.v1, &d.s, &d.t})
      *v = rebase(*v, zero, arena);
    table[p] = d;
  }
  team->devs.resize(1);
  TeamDevice& D = team->devs[0];
  D.device = device;
  D.rank = dev_rank;
  for (int i = 0; i < n_local; ++i) D.parts.push_back(part_begin + i);
  team->dev_of_part.assign(n_parts, -1);
  for (int i = 0; i < n_local; ++i) table[part_begin + i] = local_parts[i]->d;
  HaloPush hp;
  int rc = plan_halo_push(table, hp);
  if (rc) return rc;
  for (int p = 0; p < n_parts; ++p) table[p].mir = hp.on && table[p].n_halo > 0;
  rc = setup_device(D, table, team->parts.data(), n_parts, n_dev, 1, hp);
  if (rc) return rc;
  // local table now; peer tables after connect
  LRB_CUDA(cudaMemcpy(D.parts_dev, table.data(), sizeof(PartDev) * n_parts, cudaMemcpyHostToDevice));
  std::memset(team_blob, 0, LRB_BLOB_BYTES);
  TeamBlob tb{};
  std::memcpy(tb.magic, "LRBTEAM", 8);
  LRB_CUDA(cudaIpcGetMemHandle(&tb.ws, D.ws));
  tb.flags_off = reinterpret_cast<char*>(D.host.flags) - static_cast<char*>(D.ws);
  tb.part_red_off = reinterpret_cast<char*>(D.host.part_red) - static_cast<char*>(D.ws);
  std::memcpy(team_blob, &tb, sizeof(tb));
  *out = team.release();
  return LRB_OK;
}

int lrb_team_connect_ipc(lrb_team* team, const void* team_blobs) {
  if (!team || !team_blobs || team->devs.size() != 1) {
    set_error("lrb_team_connect_ipc: bad arguments");
    return LRB_EVALUE;
  }
  TeamDevice& D = team->devs[0];
  DeviceGuard g(D.device);
  const int n_dev = D.host.n_dev;
  std::vector<void*> pf(n_dev), pr(n_dev);
  const char* blobs = static_cast<const char*>(team_blobs);
  for (int r = 0; r < n_dev; ++r) {
    if (r == D.rank) {
      pf[r] = D.host.flags;
      pr[r] = D.host.part_red;
      continue;
    }
    TeamBlob tb;
    std::memcpy(&tb, blobs + size_t(r) * LRB_BLOB_BYTES, sizeof(tb));
    if (std::memcmp(tb.magic, "LRBTEAM", 8) != 0) {
      set_error("lrb_team_connect_ipc: bad team blob");
      return LRB_EVALUE;
    }
    void* base = nullptr;
    LRB_CUDA(cudaIpcOpenMemHandle(&base, tb.ws, cudaIpcMemLazyEnablePeerAccess));
    team->ipc_opened.push_back(base);
    pf[r] = static_cast<char*>(base) + tb.flags_off;
    pr[r] = static_cast<char*>(base) + tb.part_red_off;
  }
  std::vector<PartDev> table(D.host.n_parts);
  LRB_CUDA(cudaMemcpy(table.data(), D.parts_dev, sizeof(PartDev) * table.size(), cudaMemcpyDeviceToHost));
  return publish_tables(D, table, pf, pr);
}

int lrb_team_read_vector(lrb_team* team, int32_t part, int32_t vec, int64_t n, double* out) {
  if (!team || !out || vec < 2 || vec > 13 || part < 0) {
    set_error("lrb_team_read_vector: bad arguments");
    return LRB_EVALUE;
  }
  TeamDevice& D = team->devs[0];
  if (part >= D.host.n_parts) {
    set_error("lrb_team_read_vector: bad part");
    return LRB_EVALUE;
  }
  DeviceGuard g(D.device);
  PartDev P;
  LRB_CUDA(cudaMemcpy(&P, D.parts_dev + part, sizeof(PartDev), cudaMemcpyDeviceToHost));
  double* v[12] = {P.x, P.r, P.p0, P.p1, P.q, P.b, P.dinv, P.rhat, P.v0, P.v1, P.s, P.t};
  if (n > P.n) n = P.n;
  LRB_CUDA(cudaMemcpy(out, v[vec - 2], 8 * n, cudaMemcpyDefault));
  return LRB_OK;
}

int lrb_team_debug(lrb_team* team, int64_t* out) {
  if (!team || !out) {
    set_error("lrb_team_debug: null argument");
    return LRB_EVALUE;
  }
  TeamDevice& D = team->devs[0];
  DeviceGuard g(D.device);
  unsigned long long e = 0;
  std::vector<unsigned long long> f(D.host.n_dev);
  LRB_CUDA(cudaMemcpy(&e, D.host.epoch, sizeof(e), cudaMemcpyDeviceToHost));
  LRB_CUDA(cudaMemcpy(f.data(), D.host.flags, 8 * f.size(), cudaMemcpyDeviceToHost));
  out[0] = int64_t(e);
  for (size_t i = 0; i < f.size(); ++i) out[1 + i] = int64_t(f[i]);
  return LRB_OK;
}

int lrb_team_kernel_info(lrb_team* team, int32_t method, int64_t* out) {
  if (!team || !out || method < LRB_METHOD_CG || method >= kMethods) {
    set_error("lrb_team_kernel_info: bad arguments");
    return LRB_EVALUE;
  }
  const TeamDevice& D = team->devs[0];
  out[0] = D.streaming[method] ? 1 : 0;
  out[1] = D.grid[method];
  out[2] = D.block[method];
  out[3] = D.streaming[method] ? D.n_stages[method] : 0;
  out[4] = D.streaming[method] ? D.stage_bytes[method] : 0;
  out[5] = int64_t(D.smem[method]);
  out[6] = D.mirrors ? 1 : 0;
  out[7] = D.push_runs;
  return LRB_OK;
}

int lrb_team_profile(lrb_team* team, int32_t cap) {
  if (!team || cap < 0) {
    set_error("lrb_team_profile: bad arguments");
    return LRB_EVALUE;
  }
  std::lock_guard<std::mutex> lk(team->mu);
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    if (D.prof_dev) cudaFree(D.prof_dev);
    D.prof_dev = nullptr;
    D.prof_cap = 0;
    D.host.prof = nullptr;
    D.host.prof_n = nullptr;
    D.host.prof_cap = 0;
    D.host.prof_cta = nullptr;
    if (cap > 0) {
      const size_t extra = size_t(*std::max_element(D.grid, D.grid + 3)) * kCnt;
      const size_t words = size_t(cap) + 1 + extra;
      LRB_CUDA(cudaMalloc(&D.prof_dev, sizeof(long long) * words));
      LRB_CUDA(cudaMemset(D.prof_dev, 0, sizeof(long long) * words));
      D.prof_cap = cap;
      D.host.prof = D.prof_dev + 1;
      D.host.prof_cta = D.prof_dev + 1 + cap;
      D.host.prof_n = reinterpret_cast<int32_t*>(D.prof_dev);
      D.host.prof_cap = cap;
    }
  }
  return LRB_OK;
}

int lrb_team_profile_read(lrb_team* team, int64_t* out, int32_t cap) {
  if (!team || !out || cap < 0) {
    set_error("lrb_team_profile_read: bad arguments");
    return LRB_EVALUE;
  }
  const TeamDevice& D = team->devs[0];
  if (!D.prof_dev) return 0;
  DeviceGuard g(D.device);
  std::vector<long long> buf(size_t(D.prof_cap) + 1);
  LRB_CUDA(cudaMemcpy(buf.data(), D.prof_dev, sizeof(long long) * buf.size(), cudaMemcpyDeviceToHost));
  const int n = std::min<int>(int(*reinterpret_cast<int32_t*>(buf.data())), std::min(cap, D.prof_cap));
  for (int i = 0; i < n; ++i) out[i] = int64_t(buf[1 + i]);
  return n;
}

int lrb_team_profile_counters(lrb_team* team, int32_t method, int64_t* out, int32_t cap) {
  if (!team || !out || method < LRB_METHOD_CG || method >= kMethods) {
    set_error("lrb_team_profile_counters: bad arguments");
    return LRB_EVALUE;
  }
  const TeamDevice& D = team->devs[0];
  if (!D.prof_dev || !D.streaming[method]) return 0;
  DeviceGuard g(D.device);
  const int n = std::min(cap, D.grid[method] * kCnt);
  std::vector<long long> buf(size_t(std::max(n, 0)));
  if (n > 0)
    LRB_CUDA(cudaMemcpy(buf.data(), D.host.prof_cta, sizeof(long long) * n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i) out[i] = int64_t(buf[i]);
  return n;
}

int lrb_team_create(int32_t n_parts, lrb_part* const* parts, lrb_team** out) {
  return lrb_team_create_ex(n_parts, parts, nullptr, out);
}

void lrb_team_destroy(lrb_team* team) {
  if (!team) return;
  // The parts (and their streams) may already be gone: Python finalizes the
  // objects of a reference cycle in arbitrary order.  cudaFree synchronizes.
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    if (D.ws) cudaFree(D.ws);
    if (D.hist_dev) cudaFree(D.hist_dev);
    if (D.prof_dev) cudaFree(D.prof_dev);
    if (D.t0) cudaEventDestroy(D.t0);
    if (D.t1) cudaEventDestroy(D.t1);
    if (D.ev_in) cudaEventDestroy(D.ev_in);
    if (D.ev_out) cudaEventDestroy(D.ev_out);
  }
  if (team->ipc_dev >= 0) {
    DeviceGuard g(team->ipc_dev);
    for (void* p : team->ipc_opened) cudaIpcCloseMemHandle(p);
  }
  delete team;
}

// Every part's main stream: pending scatters joined; other local parts' main
// streams made to wait for the device stream's previous work and vice versa.
static int team_prologue(lrb_team* team, lrb::TeamDevice& D) {
  for (int p : D.parts) {
    int rc = lrb_part_join(team->parts[p]);
    if (rc) return rc;
  }
  DeviceGuard g(D.device);
  for (int p : D.parts) {
    lrb_part* P = team->parts[p];
    if (P->main == D.stream) continue;
    LRB_CUDA(cudaEventRecord(P->main_done, P->main));
    LRB_CUDA(cudaStreamWaitEvent(D.stream, P->main_done, 0));
  }
  return LRB_OK;
}

static int team_epilogue(lrb_team* team, lrb::TeamDevice& D) {
  DeviceGuard g(D.device);
  LRB_CUDA(cudaEventRecord(team->parts[D.parts.front()]->main_done, D.stream));
  for (int p : D.parts) {
    lrb_part* P = team->parts[p];
    if (P->main != D.stream) LRB_CUDA(cudaStreamWaitEvent(P->main, team->parts[D.parts.front()]->main_done, 0));
    LRB_CUDA(cudaEventRecord(P->main_done, D.stream));
  }
  return LRB_OK;
}

int lrb_team_spmv(lrb_team* team, const double* const* x_host, double* const* y_host) {
  if (!team || !x_host || !y_host) {
    set_error("lrb_team_spmv: null argument");
    return LRB_EVALUE;
  }
  if (team->ipc_dev >= 0 && team->devs[0].host.n_dev > 1) {
    set_error("lrb_team_spmv: not available on multi-process teams (use lrb_team_solve)");
    return LRB_EVALUE;
  }
  std::lock_guard<std::mutex> lk(team->mu);
  for (auto& D : team->devs) {
    int rc = team_prologue(team, D);
    if (rc) return rc;
    DeviceGuard g(D.device);
    for (int p : D.parts) {
      lrb_part* P = team->parts[p];
      if (P->d.n)
        LRB_CUDA(cudaMemcpyAsync(P->d.s, x_host[p], 8 * P->d.n, cudaMemcpyHostToDevice, D.stream));
    }
  }
  // all x must be resident before any device reads halo values
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    LRB_CUDA(cudaStreamSynchronize(D.stream));
  }
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    for (int p : D.parts) {
      lrb_part* P = team->parts[p];
      if (!P->d.n) continue;
      spmv_kernel<><<<unsigned((P->d.n + 255) / 256), 256, 0, D.stream>>>(D.parts_dev, p);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      LRB_CUDA(cudaGetLastError());
      LRB_CUDA(cudaMemcpyAsync(y_host[p], P->d.t, 8 * P->d.n, cudaMemcpyDeviceToHost, D.stream));
    }
  }
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    LRB_CUDA(cudaStreamSynchronize(D.stream));
    int rc = team_epilogue(team, D);
    if (rc) return rc;
  }
  return LRB_OK;
}

int lrb_team_solve(lrb_team* team, int32_t method, const double* const* b_host,
                   double* const* x_host, double tol, int32_t max_iter, lrb_report* rep,
                   double* hist, int32_t hist_cap) {
  if (!team || !rep) {
    set_error("lrb_team_solve: null argument");
    return LRB_EVALUE;
  }
  if (!(tol > 0)) {
    set_error("tol must be positive");
    return LRB_EVALUE;
  }
  if (method < LRB_METHOD_CG || method >= kMethods) {
    set_error("lrb_team_solve: unknown method");
    return LRB_EVALUE;
  }
  for (auto& D : team->devs)
    if (!D.fn[method]) {
      set_error("lrb_team_solve: pcg1 / pipecg need the streaming solver "
                "(unset LRB_SOLVER=classic; stages must fit shared memory)");
      return LRB_EVALUE;
    }
  std::lock_guard<std::mutex> lk(team->mu);
  if (team->poisoned) {
    set_error("team poisoned: a cross-device barrier timed out in an earlier solve; "
              "destroy and recreate the team");
    return LRB_ETIMEOUT;
  }
  const bool multi = team->devs.size() > 1;
  for (auto& D : team->devs) {
    int rc = team_prologue(team, D);
    if (rc) return rc;
    if (hist && hist_cap > 0) {
      rc = team_hist_capacity(D, hist_cap);
      if (rc) return rc;
    }
    DeviceGuard g(D.device);
    if (b_host)
      for (int p : D.parts) {
        lrb_part* P = team->parts[p];
        if (P->d.n)
          LRB_CUDA(cudaMemcpyAsync(P->d.b, b_host[p], 8 * P->d.n, cudaMemcpyHostToDevice, D.stream));
      }
    LRB_CUDA(cudaMemsetAsync(D.out_dev, 0, sizeof(SolveOut), D.stream));
    if (D.prof_dev) LRB_CUDA(cudaMemsetAsync(D.prof_dev, 0, sizeof(long long), D.stream));
    TeamDev& H = D.host;
    H.tol = tol;
    H.max_iter = max_iter;
    H.stage_bytes = D.stage_bytes[method];
    H.n_stages = D.n_stages[method];
    // one streaming CTA per SM = one reduction lane per CTA (kernels.cuh)
    H.lane_fast = (D.streaming[method] && D.grid[method] <= kLanes && D.parts.size() == 1) ? 1 : 0;
    H.hist = (hist && hist_cap > 0) ? D.hist_dev : nullptr;
    H.hist_cap = hist_cap;
  }
  if (multi) {
    // a device must not start reading peers' b/x before their copies land
    for (auto& D : team->devs) {
      DeviceGuard g(D.device);
      LRB_CUDA(cudaStreamSynchronize(D.stream));
    }
  }
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    void* args[] = {&D.host};
    const void* fn = D.fn[method];
    const int grid = D.grid[method];
    const size_t smem = D.smem[method];
    LRB_CUDA(cudaEventRecord(D.t0, D.stream));
    if (!D.cooperative) {
      // several device ranks share this GPU (test mode): each grid is sized
      // to a share of one wave (max_grid), so they are co-resident
      LRB_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(D.block[method]), args, smem, D.stream));
    } else {
      LRB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(D.block[method]), args, smem, D.stream));
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LRB_CUDA(cudaEventRecord(D.t1, D.stream));
    if (x_host)
      for (int p : D.parts) {
        lrb_part* P = team->parts[p];
        if (P->d.n && x_host[p])
          LRB_CUDA(cudaMemcpyAsync(x_host[p], P->d.x, 8 * P->d.n, cudaMemcpyDeviceToHost, D.stream));
      }
  }
  SolveOut so{};
  float ms = 0.f;
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    LRB_CUDA(cudaStreamSynchronize(D.stream));
    SolveOut o{};
    LRB_CUDA(cudaMemcpy(&o, D.out_dev, sizeof(SolveOut), cudaMemcpyDeviceToHost));
    float m = 0.f;
    LRB_CUDA(cudaEventElapsedTime(&m, D.t0, D.t1));
    ms = std::max(ms, m);
    if (D.rank == 0) so = o;
    if (o.status && !so.status) so.status = o.status;
    int rc = team_epilogue(team, D);
    if (rc) return rc;
  }
  if (hist && hist_cap > 0) {
    auto& D0 = team->devs[0];
    DeviceGuard g(D0.device);
    int n = std::min<int>(hist_cap, std::max(so.iterations, 0));
    if (n) LRB_CUDA(cudaMemcpy(hist, D0.hist_dev, sizeof(double) * n, cudaMemcpyDeviceToHost));
  }
  rep->iterations = so.iterations;
  rep->converged = so.converged;
  rep->breakdown = so.breakdown;
  rep->status = so.status;
  rep->residual = so.residual;
  rep->bnorm = so.bnorm;
  rep->device_ms = ms;
  if (so.status == LRB_ENOTPD) {
    set_error("cg: matrix is not positive definite");
    return LRB_ENOTPD;
  }
  if (so.status == LRB_ETIMEOUT) {
    team->poisoned = true;
    set_error("team barrier timed out (a device of the team did not arrive)");
    return LRB_ETIMEOUT;
  }
  return LRB_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Stream-ordered entry points (GPU-resident caller)
// ---------------------------------------------------------------------------
namespace lrb {

__global__ void report_kernel(const SolveOut* __restrict__ o, lrb_report* __restrict__ r) {
  r->iterations = o->iterations;
  r->converged = o->converged;
  r->breakdown = o->breakdown;
  r->status = o->status;
  r->residual = o->residual;
  r->bnorm = o->bnorm;
  r->device_ms = -1.0;
}

static bool is_device_or_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

// The caller's stream of device rank r (NULL array: none).
static cudaStream_t caller_stream(const lrb_stream_t* streams, int r) {
  return streams ? reinterpret_cast<cudaStream_t>(streams[r]) : nullptr;
}

// Device streams wait for the callers' streams (and, for multi-device teams,
// for every device's inputs: a device must not read peers' halo operands
// before their copies land — the async form of lrb_team_solve's host sync).
static int order_after_callers(lrb_team* team, const lrb_stream_t* streams) {
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    if (streams) {
      LRB_CUDA(cudaEventRecord(D.ev_in, caller_stream(streams, D.rank)));
      LRB_CUDA(cudaStreamWaitEvent(D.stream, D.ev_in, 0));
    }
  }
  return LRB_OK;
}

static int join_devices(lrb_team* team) {
  if (team->devs.size() < 2) return LRB_OK;
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    LRB_CUDA(cudaEventRecord(D.ev_in, D.stream));
  }
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    for (auto& E : team->devs)
      if (&E != &D) LRB_CUDA(cudaStreamWaitEvent(D.stream, E.ev_in, 0));
  }
  return LRB_OK;
}

static int callers_wait(lrb_team* team, const lrb_stream_t* streams) {
  for (auto& D : team->devs) {
    int rc = team_epilogue(team, D);
    if (rc) return rc;
    if (!streams) continue;
    DeviceGuard g(D.device);
    LRB_CUDA(cudaEventRecord(D.ev_out, D.stream));
    LRB_CUDA(cudaStreamWaitEvent(caller_stream(streams, D.rank), D.ev_out, 0));
  }
  return LRB_OK;
}

}  // namespace lrb

extern "C" {

int lrb_update_segment_async(lrb_part* part, int32_t seg, int32_t n_pieces,
                             const double* const* pieces, const int64_t* piece_len,
                             lrb_stream_t stream) {
  if (!part || seg < 0 || seg >= int(part->seg_stream.size())) {
    set_error("lrb_update_segment_async: bad segment");
    return LRB_EVALUE;
  }
  const int64_t off = part->seg_off[seg], len = part->seg_off[seg + 1] - off;
  int rc = check_pieces(part, len, n_pieces, piece_len, "segment", seg);
  if (rc) return rc;
  for (int i = 0; i < n_pieces; ++i)
    if (piece_len[i] && !is_device_or_pinned(pieces[i])) {
      set_error("lrb_update_segment_async: piece " + std::to_string(i) +
                " is pageable host memory (stream-ordered copies need pinned or device memory)");
      return LRB_EVALUE;
    }
  DeviceGuard g(part->device);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  LRB_CUDA(cudaStreamWaitEvent(st, part->main_done, 0));
  LRB_CUDA(cudaStreamWaitEvent(st, part->staged_done, 0));
  double* dst = part->d.recv + off;
  int64_t o = 0;
  for (int i = 0; i < n_pieces; ++i) {
    if (piece_len[i])
      LRB_CUDA(cudaMemcpyAsync(dst + o, pieces[i], 8 * piece_len[i], cudaMemcpyDefault, st));
    o += piece_len[i];
  }
  part->stats[0] += n_pieces;
  part->stats[2] += 8 * len;
  if (!part->seg_rows.empty()) {
    rc = launch_scatter(part, part->seg_rows[seg], part->seg_rows[seg + 1], st);
    if (rc) return rc;
  }
  std::lock_guard<std::mutex> lk(part->mu);
  LRB_CUDA(cudaEventRecord(part->seg_done[seg], st));
  part->seg_pending[seg] = 1;
  return LRB_OK;
}

int lrb_team_solve_async(lrb_team* team, int32_t method, const double* const* b_dev,
                         double* const* x_dev, double tol, int32_t max_iter,
                         const lrb_stream_t* streams, lrb_report* rep_out) {
  if (!team) {
    set_error("lrb_team_solve_async: null team");
    return LRB_EVALUE;
  }
  if (!(tol > 0)) {
    set_error("tol must be positive");
    return LRB_EVALUE;
  }
  if (method < LRB_METHOD_CG || method >= kMethods) {
    set_error("lrb_team_solve_async: unknown method");
    return LRB_EVALUE;
  }
  if (team->ipc_dev >= 0) {
    set_error("lrb_team_solve_async: single-process teams only (use lrb_team_solve)");
    return LRB_EVALUE;
  }
  for (auto& D : team->devs)
    if (!D.fn[method]) {
      set_error("lrb_team_solve_async: pcg1 / pipecg need the streaming solver");
      return LRB_EVALUE;
    }
  std::lock_guard<std::mutex> lk(team->mu);
  if (team->poisoned) {
    set_error("team poisoned: a cross-device barrier timed out in an earlier solve; "
              "destroy and recreate the team");
    return LRB_ETIMEOUT;
  }
  int rc = order_after_callers(team, streams);
  if (rc) return rc;
  for (auto& D : team->devs) {
    rc = team_prologue(team, D);
    if (rc) return rc;
    DeviceGuard g(D.device);
    if (b_dev)
      for (int p : D.parts) {
        lrb_part* P = team->parts[p];
        if (P->d.n && b_dev[p] && b_dev[p] != P->d.b)
          LRB_CUDA(cudaMemcpyAsync(P->d.b, b_dev[p], 8 * P->d.n, cudaMemcpyDeviceToDevice, D.stream));
      }
    LRB_CUDA(cudaMemsetAsync(D.out_dev, 0, sizeof(SolveOut), D.stream));
  }
  rc = join_devices(team);
  if (rc) return rc;
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    TeamDev H = D.host;   // by-value kernel argument: the stored one stays as is
    H.tol = tol;
    H.max_iter = max_iter;
    H.stage_bytes = D.stage_bytes[method];
    H.n_stages = D.n_stages[method];
    H.lane_fast = (D.streaming[method] && D.grid[method] <= kLanes && D.parts.size() == 1) ? 1 : 0;
    H.hist = nullptr;
    H.hist_cap = 0;
    H.prof = nullptr;   // diagnostics belong to the synchronous entry point
    H.prof_cta = nullptr;
    H.prof_cap = 0;
    void* args[] = {&H};
    if (!D.cooperative)
      LRB_CUDA(cudaLaunchKernel(D.fn[method], dim3(D.grid[method]), dim3(D.block[method]), args,
                                D.smem[method], D.stream));
    else
      LRB_CUDA(cudaLaunchCooperativeKernel(D.fn[method], dim3(D.grid[method]), dim3(D.block[method]),
                                           args, D.smem[method], D.stream));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (x_dev)
      for (int p : D.parts) {
        lrb_part* P = team->parts[p];
        if (P->d.n && x_dev[p] && x_dev[p] != P->d.x)
          LRB_CUDA(cudaMemcpyAsync(x_dev[p], P->d.x, 8 * P->d.n, cudaMemcpyDeviceToDevice, D.stream));
      }
    if (rep_out && D.rank == 0) {
      report_kernel<<<1, 1, 0, D.stream>>>(D.out_dev, rep_out);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      LRB_CUDA(cudaGetLastError());
    }
  }
  return callers_wait(team, streams);
}

int lrb_team_spmv_async(lrb_team* team, const double* const* x_dev, double* const* y_dev,
                        const lrb_stream_t* streams) {
  if (!team || !x_dev || !y_dev) {
    set_error("lrb_team_spmv_async: null argument");
    return LRB_EVALUE;
  }
  if (team->ipc_dev >= 0) {
    set_error("lrb_team_spmv_async: single-process teams only");
    return LRB_EVALUE;
  }
  std::lock_guard<std::mutex> lk(team->mu);
  int rc = order_after_callers(team, streams);
  if (rc) return rc;
  for (auto& D : team->devs) {
    rc = team_prologue(team, D);
    if (rc) return rc;
    DeviceGuard g(D.device);
    for (int p : D.parts) {
      lrb_part* P = team->parts[p];
      if (P->d.n)
        LRB_CUDA(cudaMemcpyAsync(P->d.s, x_dev[p], 8 * P->d.n, cudaMemcpyDeviceToDevice, D.stream));
    }
  }
  rc = join_devices(team);
  if (rc) return rc;
  for (auto& D : team->devs) {
    DeviceGuard g(D.device);
    for (int p : D.parts) {
      lrb_part* P = team->parts[p];
      if (!P->d.n) continue;
      spmv_kernel<><<<unsigned((P->d.n + 255) / 256), 256, 0, D.stream>>>(D.parts_dev, p);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      LRB_CUDA(cudaGetLastError());
      LRB_CUDA(cudaMemcpyAsync(y_dev[p], P->d.t, 8 * P->d.n, cudaMemcpyDeviceToDevice, D.stream));
    }
  }
  // a later call rewrites s: no device may still be reading a peer's s
  rc = join_devices(team);
  if (rc) return rc;
  return callers_wait(team, streams);
}

}  // extern "C"
