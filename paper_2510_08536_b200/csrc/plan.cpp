// Create path: fused owner plan (host, multi-threaded, O(nnz), no global sort).
//
// Reference algorithm (repart.py:143-318): extract every source's global
// pattern (ldu_to_coo lexsort), ship it to the owner, localize couplings whose
// column lies in I_GPU(k), lexsort + dedupe the fused local / non-local
// patterns, then binary-search every packed-buffer entry's (row, col) key to
// get the scatter map.  Here the same outputs come from a counting sort by
// row of the buffer provenance (buffer position -> (row, col), pack layout
// update.py:40-45) followed by a per-row sort by column: rows are short
// (7 entries on the cavity), so the whole build is linear and parallel.
// Row-major order with ascending columns is exactly the reference's lexsort
// order, and the inverse of the bucket assignment is the scatter map.

#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <iterator>
#include <limits>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ldurepart_b200.h"
#include "lrb_internal.h"

namespace lrb {

namespace {

void parallel_for(int64_t n, int n_threads, const std::function<void(int64_t, int64_t)>& fn) {
  if (n <= 0) return;
  int64_t nt = std::max<int64_t>(1, std::min<int64_t>(n_threads, (n + 65535) / 65536));
  if (nt == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt);
  for (int64_t t = 0; t < nt; ++t) {
    int64_t b = n * t / nt, e = n * (t + 1) / nt;
    th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& t : th) t.join();
}

int resolve_threads(int32_t n) {
  if (n > 0) return n;
  unsigned h = std::thread::hardware_concurrency();
  return h ? int(h) : 1;
}

// Provenance of a buffer entry: its global (row, col).  Gen must provide
//   for_range(b0, b1, fn(b, row, col))   over buffer positions [b0, b1).
struct LduGen {
  int32_t n_src;
  const int64_t *src_rows, *face_off, *lower, *upper, *ifc_off, *ifc_row, *ifc_col;
  std::vector<int64_t> seg_off;  // buffer offsets per source

  LduGen(int32_t ns, const int64_t* sr, const int64_t* fo, const int64_t* lo_,
         const int64_t* up_, const int64_t* io, const int64_t* ir, const int64_t* ic)
      : n_src(ns), src_rows(sr), face_off(fo), lower(lo_), upper(up_), ifc_off(io),
        ifc_row(ir), ifc_col(ic), seg_off(ns + 1, 0) {
    for (int s = 0; s < ns; ++s) {
      int64_t n = src_rows[s + 1] - src_rows[s];
      int64_t F = face_off[s + 1] - face_off[s];
      int64_t I = ifc_off[s + 1] - ifc_off[s];
      seg_off[s + 1] = seg_off[s] + n + 2 * F + I;
    }
  }

  template <class Fn>
  void for_range(int64_t b0, int64_t b1, Fn&& fn) const {
    // locate the first source
    int s = int(std::upper_bound(seg_off.begin(), seg_off.end(), b0) - seg_off.begin()) - 1;
    for (; s < n_src && seg_off[s] < b1; ++s) {
      const int64_t base = seg_off[s], rlo = src_rows[s];
      const int64_t n = src_rows[s + 1] - rlo;
      const int64_t F = face_off[s + 1] - face_off[s];
      const int64_t* lw = lower + face_off[s];
      const int64_t* up = upper + face_off[s];
      const int64_t* irow = ifc_row + ifc_off[s];
      const int64_t* icol = ifc_col + ifc_off[s];
      const int64_t I = ifc_off[s + 1] - ifc_off[s];
      int64_t j0 = std::max<int64_t>(b0 - base, 0);
      int64_t j1 = std::min<int64_t>(b1 - base, n + 2 * F + I);
      // sections: diag [0,n), upper [n, n+F), lower [n+F, n+2F), iface [n+2F, ...)
      for (int64_t j = std::max<int64_t>(j0, 0); j < std::min<int64_t>(j1, n); ++j)
        fn(base + j, rlo + j, rlo + j);
      for (int64_t j = std::max<int64_t>(j0, n); j < std::min<int64_t>(j1, n + F); ++j) {
        int64_t f = j - n;
        fn(base + j, rlo + lw[f], rlo + up[f]);
      }
      for (int64_t j = std::max<int64_t>(j0, n + F); j < std::min<int64_t>(j1, n + 2 * F); ++j) {
        int64_t f = j - n - F;
        fn(base + j, rlo + up[f], rlo + lw[f]);
      }
      for (int64_t j = std::max<int64_t>(j0, n + 2 * F); j < j1; ++j) {
        int64_t e = j - n - 2 * F;
        fn(base + j, rlo + irow[e], icol[e]);
      }
    }
  }
};

struct CooGen {
  const int64_t *row, *col;
  template <class Fn>
  void for_range(int64_t b0, int64_t b1, Fn&& fn) const {
    for (int64_t b = b0; b < b1; ++b) fn(b, row[b], col[b]);
  }
};

struct BuildError {
  std::atomic<int> code{0};
  std::string msg;
  std::atomic<int64_t> first_row{std::numeric_limits<int64_t>::max()};
  std::atomic_flag lock = ATOMIC_FLAG_INIT;
  void set(int c, const std::string& m, int64_t row = -1) {
    // keep the earliest row for deterministic messages
    int64_t key = row < 0 ? std::numeric_limits<int64_t>::max() - 1 : row;
    while (lock.test_and_set()) {
    }
    if (code.load() == 0 || key < first_row.load()) {
      code = c;
      msg = m;
      first_row = key;
    }
    lock.clear();
  }
};

// Staging windows per tile (lrb_internal.h): the union over the tile's
// pattern slices of [row0 + off, row0 + off + rows) for every local offset,
// clipped to [0, n), merged into at most kMaxWin sorted intervals.
void build_tile_windows(Plan& P) {
  const int64_t n = P.n;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  P.tile_win.assign(ntiles * kWinStride, 0);
  P.max_stage = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const int64_t row0 = t * kTile, rows = std::min<int64_t>(kTile, n - row0);
    std::vector<int32_t> offs;
    bool ok = true;
    for (int64_t s = row0 / kSlice; s < (row0 + rows + kSlice - 1) / kSlice && ok; ++s) {
      const int pid = P.slice_pat[s];
      if (pid < 0) {
        ok = false;
        break;
      }
      const int64_t w = (P.slice_ptr[s + 1] - P.slice_ptr[s]) / kSlice;
      for (int64_t k = 0; k < w; ++k) offs.push_back(P.pat_off[pid * kPatW + k]);
    }
    if (!ok) continue;
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    std::vector<std::pair<int64_t, int64_t>> iv;  // [a, b) relative to row0
    for (int32_t o : offs) {
      int64_t a = std::max<int64_t>(row0 + o, 0), b = std::min<int64_t>(row0 + o + rows, n);
      if (a >= b) continue;  // halo column (col >= n) or outside the part
      a -= row0;
      b -= row0;
      if (!iv.empty() && a <= iv.back().second)
        iv.back().second = std::max(iv.back().second, b);
      else
        iv.emplace_back(a, b);
    }
    int64_t total = 0;
    for (auto& x : iv) total += x.second - x.first;
    if (iv.empty() || int64_t(iv.size()) > kMaxWin || total > kMaxStage) continue;
    int32_t* tw = &P.tile_win[t * kWinStride];
    tw[0] = int32_t(iv.size());
    tw[1] = int32_t(total);
    for (size_t w = 0; w < iv.size(); ++w) {
      tw[2 + 2 * w] = int32_t(iv[w].first);
      tw[3 + 2 * w] = int32_t(iv[w].second - iv[w].first);
    }
    P.max_stage = std::max(P.max_stage, total);
  }
}

template <class Gen>
int build(Plan& P, int64_t total, int64_t lo, int64_t hi, int64_t n_buf,
          const std::vector<int64_t>& seg_off, const Gen& gen, int32_t n_gpu,
          const int64_t* gpu_offsets, int n_threads, bool ldu_segments) {
  if (lo < 0 || hi <= lo || hi > total) {
    set_error("invalid owner row range");
    return LRB_EVALUE;
  }
  P.total = total;
  P.lo = lo;
  P.hi = hi;
  P.n = hi - lo;
  P.n_buf = n_buf;
  P.seg_off = seg_off;
  if (P.n >= (int64_t(1) << 31) - 1 || n_buf >= (int64_t(1) << 31) - 1) {
    set_error("part too large for 32-bit device indices");
    return LRB_EVALUE;
  }
  const int64_t n = P.n;
  std::vector<int64_t> cnt_l(n + 1, 0), cnt_n(n + 1, 0);
  BuildError err;

  // 1) count entries per row (atomic buckets)
  parallel_for(n_buf, n_threads, [&](int64_t b0, int64_t b1) {
    gen.for_range(b0, b1, [&](int64_t b, int64_t row, int64_t col) {
      int64_t r = row - lo;
      if (r < 0 || r >= n || col < 0 || col >= total) {
        err.set(LRB_EVALUE, "buffer entry " + std::to_string(b) + " at (" +
                                std::to_string(row) + ", " + std::to_string(col) +
                                ") is out of range for owner rows [" + std::to_string(lo) +
                                ", " + std::to_string(hi) + ")");
        return;
      }
      if (col >= lo && col < hi)
        __atomic_fetch_add(&cnt_l[r + 1], 1, __ATOMIC_RELAXED);
      else
        __atomic_fetch_add(&cnt_n[r + 1], 1, __ATOMIC_RELAXED);
    });
  });
  if (err.code) {
    set_error(err.msg);
    return err.code;
  }
  for (int64_t i = 0; i < n; ++i) {
    cnt_l[i + 1] += cnt_l[i];
    cnt_n[i + 1] += cnt_n[i];
  }
  const int64_t nnz_l = cnt_l[n], nnz_n = cnt_n[n];
  P.loc_ptr = cnt_l;
  P.nl_ptr = cnt_n;

  // 2) fill buckets (order inside a row fixed by the sort below)
  std::vector<int64_t> cur_l(cnt_l.begin(), cnt_l.end() - 1), cur_n(cnt_n.begin(), cnt_n.end() - 1);
  P.loc_col.assign(nnz_l, 0);
  P.loc_src.assign(nnz_l, 0);
  std::vector<int64_t> nl_gcol(nnz_n);
  P.nl_src.assign(nnz_n, 0);
  parallel_for(n_buf, n_threads, [&](int64_t b0, int64_t b1) {
    gen.for_range(b0, b1, [&](int64_t b, int64_t row, int64_t col) {
      int64_t r = row - lo;
      if (col >= lo && col < hi) {
        int64_t p = __atomic_fetch_add(&cur_l[r], 1, __ATOMIC_RELAXED);
        P.loc_col[p] = int32_t(col - lo);
        P.loc_src[p] = int32_t(b);
      } else {
        int64_t p = __atomic_fetch_add(&cur_n[r], 1, __ATOMIC_RELAXED);
        nl_gcol[p] = col;
        P.nl_src[p] = int32_t(b);
      }
    });
  });

  // 3) per-row sort by column; duplicates = overlapping ownership (repart.py:222-230)
  parallel_for(n, n_threads, [&](int64_t r0, int64_t r1) {
    for (int64_t r = r0; r < r1; ++r) {
      for (int64_t i = P.loc_ptr[r] + 1; i < P.loc_ptr[r + 1]; ++i) {
        int32_t c = P.loc_col[i], s = P.loc_src[i];
        int64_t j = i - 1;
        while (j >= P.loc_ptr[r] && (P.loc_col[j] > c || (P.loc_col[j] == c && P.loc_src[j] > s))) {
          P.loc_col[j + 1] = P.loc_col[j];
          P.loc_src[j + 1] = P.loc_src[j];
          --j;
        }
        P.loc_col[j + 1] = c;
        P.loc_src[j + 1] = s;
      }
      for (int64_t i = P.loc_ptr[r] + 1; i < P.loc_ptr[r + 1]; ++i)
        if (P.loc_col[i] == P.loc_col[i - 1]) {
          err.set(LRB_EVALUE,
                  "overlapping ownership: duplicate local entry (" + std::to_string(r + lo) +
                      ", " + std::to_string(int64_t(P.loc_col[i]) + lo) + ")",
                  r);
          break;
        }
      for (int64_t i = P.nl_ptr[r] + 1; i < P.nl_ptr[r + 1]; ++i) {
        int64_t c = nl_gcol[i];
        int32_t s = P.nl_src[i];
        int64_t j = i - 1;
        while (j >= P.nl_ptr[r] && (nl_gcol[j] > c || (nl_gcol[j] == c && P.nl_src[j] > s))) {
          nl_gcol[j + 1] = nl_gcol[j];
          P.nl_src[j + 1] = P.nl_src[j];
          --j;
        }
        nl_gcol[j + 1] = c;
        P.nl_src[j + 1] = s;
      }
      for (int64_t i = P.nl_ptr[r] + 1; i < P.nl_ptr[r + 1]; ++i)
        if (nl_gcol[i] == nl_gcol[i - 1]) {
          err.set(LRB_EVALUE,
                  "overlapping ownership: duplicate non-local entry (" + std::to_string(r + lo) +
                      ", " + std::to_string(nl_gcol[i]) + ")",
                  r);
          break;
        }
    }
  });
  if (err.code) {
    set_error(err.msg);
    return err.code;
  }

  // 4) halo: ascending unique non-local columns (repart.py:312-316)
  P.halo_cols = nl_gcol;
  std::sort(P.halo_cols.begin(), P.halo_cols.end());
  P.halo_cols.erase(std::unique(P.halo_cols.begin(), P.halo_cols.end()), P.halo_cols.end());
  P.nl_col.assign(nnz_n, 0);
  parallel_for(nnz_n, n_threads, [&](int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i)
      P.nl_col[i] = int32_t(std::lower_bound(P.halo_cols.begin(), P.halo_cols.end(), nl_gcol[i]) -
                            P.halo_cols.begin());
  });
  const int64_t h = int64_t(P.halo_cols.size());
  P.hpart.assign(h, -1);
  P.hidx.assign(h, -1);
  if (n_gpu > 0 && gpu_offsets) {
    for (int64_t s = 0; s < h; ++s) {
      int64_t c = P.halo_cols[s];
      int g = int(std::upper_bound(gpu_offsets, gpu_offsets + n_gpu + 1, c) - gpu_offsets) - 1;
      if (g < 0 || g >= n_gpu) {
        set_error("halo column owned by no rank");
        return LRB_EVALUE;
      }
      P.hpart[s] = g;
      P.hidx[s] = int32_t(c - gpu_offsets[g]);
    }
  }

  // 5) per-segment row ranges, used to scatter a segment as soon as its copy lands.
  //    Valid when each segment's entries own a contiguous row range exclusively
  //    (always true for LDU sources: every entry of source r has its row in
  //    I_CPU(r), repart.py:253-270).
  const int n_seg = int(seg_off.size()) - 1;
  P.seg_rows.clear();
  if (ldu_segments) {
    // filled by the caller (source row ranges)
  } else if (n_seg >= 1) {
    std::vector<int64_t> rows(n_seg + 1, -1);
    bool ok = true;
    int seg_prev = 0;
    rows[0] = 0;
    for (int64_t r = 0; r < n && ok; ++r) {
      int seg_r = -1;
      auto seg_of = [&](int32_t b) {
        return int(std::upper_bound(seg_off.begin(), seg_off.end(), int64_t(b)) - seg_off.begin()) - 1;
      };
      for (int64_t i = P.loc_ptr[r]; i < P.loc_ptr[r + 1] && ok; ++i) {
        int sg = seg_of(P.loc_src[i]);
        if (seg_r < 0) seg_r = sg;
        ok = ok && sg == seg_r;
      }
      for (int64_t i = P.nl_ptr[r]; i < P.nl_ptr[r + 1] && ok; ++i) {
        int sg = seg_of(P.nl_src[i]);
        if (seg_r < 0) seg_r = sg;
        ok = ok && sg == seg_r;
      }
      if (seg_r < 0) seg_r = seg_prev;  // empty row
      if (seg_r < seg_prev) ok = false;
      while (ok && seg_prev < seg_r) rows[++seg_prev] = r;
    }
    while (ok && seg_prev < n_seg) rows[++seg_prev] = n;
    if (ok) P.seg_rows = rows;
  }

  // 6) SELL-32 layout with a pattern dictionary (lrb_internal.h).  A row's
  //    entries are (col - row) offsets in ascending order — local columns,
  //    then halo columns encoded n + slot, which are always larger — so
  //    laying a slice out on the sorted union of its rows' offsets keeps
  //    every row in the reference's entry order; rows lacking an offset get a
  //    hole (src -1, masked off).
  P.n_slices = (n + kSlice - 1) / kSlice;
  const int64_t ns = P.n_slices;
  std::vector<std::vector<int32_t>> uni(ns);
  std::vector<int32_t> maxlen(ns, 0);
  auto row_off = [&](int64_t r, std::vector<int32_t>& out) {
    out.clear();
    for (int64_t i = P.loc_ptr[r]; i < P.loc_ptr[r + 1]; ++i) out.push_back(int32_t(P.loc_col[i] - r));
    for (int64_t i = P.nl_ptr[r]; i < P.nl_ptr[r + 1]; ++i)
      out.push_back(int32_t(n + P.nl_col[i] - r));
  };
  parallel_for(ns, n_threads, [&](int64_t s0, int64_t s1) {
    std::vector<int32_t> ro, merged;
    for (int64_t s = s0; s < s1; ++s) {
      std::vector<int32_t>& u = uni[s];
      u.clear();
      bool ok = (s + 1) * kSlice <= n;  // only full slices
      for (int64_t r = s * kSlice; r < std::min<int64_t>(n, (s + 1) * kSlice); ++r) {
        row_off(r, ro);
        maxlen[s] = std::max<int32_t>(maxlen[s], int32_t(ro.size()));
        if (!ok) continue;
        merged.clear();
        std::set_union(u.begin(), u.end(), ro.begin(), ro.end(), std::back_inserter(merged));
        u.swap(merged);
        if (int64_t(u.size()) > kPatW) ok = false;
      }
      if (!ok) u.clear();
    }
  });
  P.slice_ptr.assign(ns + 1, 0);
  P.slice_pat.assign(ns, -1);
  P.pat_off.clear();
  {
    std::map<std::vector<int32_t>, int32_t> ids;
    for (int64_t s = 0; s < ns; ++s) {
      int64_t w = maxlen[s];
      if (!uni[s].empty()) {
        auto it = ids.find(uni[s]);
        if (it == ids.end() && int64_t(ids.size()) < kMaxPat) {
          it = ids.emplace(uni[s], int32_t(ids.size())).first;
          P.pat_off.resize(P.pat_off.size() + kPatW, 0);
          std::copy(uni[s].begin(), uni[s].end(), P.pat_off.end() - kPatW);
        }
        if (it != ids.end()) {
          P.slice_pat[s] = it->second;
          w = int64_t(uni[s].size());
        }
      }
      P.slice_ptr[s + 1] = P.slice_ptr[s] + w * kSlice;
    }
    if (P.pat_off.empty()) P.pat_off.assign(kPatW, 0);  // keep one (unused) row
  }
  const int64_t E = P.slice_ptr[ns];
  if (E >= (int64_t(1) << 31) - 1) {
    set_error("part too large for 32-bit device indices");
    return LRB_EVALUE;
  }
  P.sell_col.assign(E, -1);
  P.sell_src.assign(E, -1);
  P.dpos.assign(n, -1);
  P.rmask.assign(n, 0);
  P.loc_sell.assign(nnz_l, 0);
  P.nl_sell.assign(nnz_n, 0);
  std::atomic<bool> dpos_overflow{false};
  parallel_for(n, n_threads, [&](int64_t r0, int64_t r1) {
    std::vector<int32_t> ro;
    for (int64_t r = r0; r < r1; ++r) {
      const int64_t s = r / kSlice;
      const int64_t base = P.slice_ptr[s] + (r % kSlice);
      const int pid = P.slice_pat[s];
      const std::vector<int32_t>& u = uni[s];
      row_off(r, ro);
      uint32_t mask = 0;
      for (int64_t k = 0; k < int64_t(ro.size()); ++k) {
        int64_t slot = k;
        if (pid >= 0) slot = std::lower_bound(u.begin(), u.end(), ro[k]) - u.begin();
        const int64_t e = base + slot * kSlice;
        const int64_t nloc = P.loc_ptr[r + 1] - P.loc_ptr[r];
        if (k < nloc) {
          const int64_t j = P.loc_ptr[r] + k;
          P.sell_col[e] = P.loc_col[j];
          P.sell_src[e] = P.loc_src[j];
          P.loc_sell[j] = int32_t(e);
          if (P.loc_col[j] == r) {
            if (slot > 32767) dpos_overflow = true;
            else P.dpos[r] = int16_t(slot);
          }
        } else {
          const int64_t j = P.nl_ptr[r] + (k - nloc);
          P.sell_col[e] = int32_t(n + P.nl_col[j]);
          P.sell_src[e] = P.nl_src[j];
          P.nl_sell[j] = int32_t(e);
        }
        mask |= 1u << (slot & 31);
      }
      if (pid >= 0) P.rmask[r] = uint16_t(mask);
    }
  });
  if (dpos_overflow) {   // Jacobi reads the diagonal through an int16 slot index
    set_error("row too long: diagonal beyond SELL slot 32767");
    return LRB_EVALUE;
  }
  build_tile_windows(P);
  return LRB_OK;
}

}  // namespace

int64_t part_device_bytes(const Plan& P);

}  // namespace lrb

using lrb::Plan;

struct lrb_plan {
  Plan p;
};

extern "C" int lrb_plan_build_ldu(int64_t total_cells, int64_t row_lo, int64_t row_hi,
                                  int32_t n_src, const int64_t* src_rows,
                                  const int64_t* face_off, const int64_t* lower,
                                  const int64_t* upper, const int64_t* ifc_off,
                                  const int64_t* ifc_row, const int64_t* ifc_col, int32_t n_gpu,
                                  const int64_t* gpu_offsets, int32_t n_threads, lrb_plan** out) {
  try {
    if (n_src < 1 || !src_rows || !face_off || !ifc_off || !out) {
      lrb::set_error("lrb_plan_build_ldu: bad arguments");
      return LRB_EVALUE;
    }
    if (src_rows[0] != row_lo || src_rows[n_src] != row_hi) {
      lrb::set_error("received patterns must tile I_GPU in ascending source order");
      return LRB_EVALUE;
    }
    for (int s = 0; s < n_src; ++s) {
      if (src_rows[s + 1] <= src_rows[s]) {
        lrb::set_error("empty part: every rank must own at least one cell");
        return LRB_EVALUE;
      }
    }
    lrb::LduGen gen(n_src, src_rows, face_off, lower, upper, ifc_off, ifc_row, ifc_col);
    auto* plan = new lrb_plan();
    int rc = lrb::build(plan->p, total_cells, row_lo, row_hi, gen.seg_off.back(), gen.seg_off, gen,
                        n_gpu, gpu_offsets, lrb::resolve_threads(n_threads), true);
    if (rc != LRB_OK) {
      delete plan;
      return rc;
    }
    plan->p.seg_rows.assign(n_src + 1, 0);
    for (int s = 0; s <= n_src; ++s) plan->p.seg_rows[s] = src_rows[s] - row_lo;
    *out = plan;
    return LRB_OK;
  } catch (const std::exception& e) {
    lrb::set_error(std::string("plan build failed: ") + e.what());
    return LRB_ERUNTIME;
  }
}

extern "C" int lrb_plan_build_coo(int64_t total_cells, int64_t row_lo, int64_t row_hi,
                                  int64_t n_buf, const int64_t* buf_row, const int64_t* buf_col,
                                  int32_t n_seg, const int64_t* seg_off, int32_t n_gpu,
                                  const int64_t* gpu_offsets, lrb_plan** out) {
  try {
    if (!out || n_buf < 0 || (n_buf > 0 && (!buf_row || !buf_col))) {
      lrb::set_error("lrb_plan_build_coo: bad arguments");
      return LRB_EVALUE;
    }
    std::vector<int64_t> segs;
    if (n_seg >= 1 && seg_off)
      segs.assign(seg_off, seg_off + n_seg + 1);
    else
      segs = {0, n_buf};
    lrb::CooGen gen{buf_row, buf_col};
    auto* plan = new lrb_plan();
    int rc = lrb::build(plan->p, total_cells, row_lo, row_hi, n_buf, segs, gen, n_gpu, gpu_offsets,
                        lrb::resolve_threads(0), false);
    if (rc != LRB_OK) {
      delete plan;
      return rc;
    }
    *out = plan;
    return LRB_OK;
  } catch (const std::exception& e) {
    lrb::set_error(std::string("plan build failed: ") + e.what());
    return LRB_ERUNTIME;
  }
}

extern "C" int lrb_plan_info(const lrb_plan* plan, int64_t* info) {
  if (!plan || !info) {
    lrb::set_error("lrb_plan_info: null argument");
    return LRB_EVALUE;
  }
  const Plan& P = plan->p;
  int64_t maxlen = 0;
  for (int64_t s = 0; s < P.n_slices; ++s)
    maxlen = std::max<int64_t>(maxlen, (P.slice_ptr[s + 1] - P.slice_ptr[s]) / lrb::kSlice);
  info[0] = P.n;
  info[1] = int64_t(P.loc_col.size());
  info[2] = int64_t(P.nl_col.size());
  info[3] = int64_t(P.halo_cols.size());
  info[4] = P.n_buf;
  info[5] = P.n_slices;
  info[6] = P.sell_entries();
  info[7] = maxlen;
  info[8] = int64_t(P.seg_off.size()) - 1;
  info[9] = lrb::part_device_bytes(P);
  int64_t uniform = 0, uniform_entries = 0;
  for (int64_t s = 0; s < P.n_slices; ++s)
    if (P.slice_pat[s] >= 0) {
      ++uniform;
      uniform_entries += P.slice_ptr[s + 1] - P.slice_ptr[s];
    }
  info[10] = uniform;
  info[11] = P.n_pat();
  info[12] = uniform_entries;
  return LRB_OK;
}

extern "C" int lrb_plan_export_csr(const lrb_plan* plan, int64_t* loc_ptr, int64_t* loc_col,
                                   int64_t* nl_ptr, int64_t* nl_col, int64_t* halo_cols) {
  if (!plan) {
    lrb::set_error("lrb_plan_export_csr: null plan");
    return LRB_EVALUE;
  }
  const Plan& P = plan->p;
  if (loc_ptr) std::copy(P.loc_ptr.begin(), P.loc_ptr.end(), loc_ptr);
  if (nl_ptr) std::copy(P.nl_ptr.begin(), P.nl_ptr.end(), nl_ptr);
  if (loc_col) std::copy(P.loc_col.begin(), P.loc_col.end(), loc_col);
  if (nl_col) std::copy(P.nl_col.begin(), P.nl_col.end(), nl_col);
  if (halo_cols) std::copy(P.halo_cols.begin(), P.halo_cols.end(), halo_cols);
  return LRB_OK;
}

extern "C" int lrb_plan_export_scatter(const lrb_plan* plan, uint8_t* to_local, int64_t* index) {
  if (!plan || !to_local || !index) {
    lrb::set_error("lrb_plan_export_scatter: null argument");
    return LRB_EVALUE;
  }
  const Plan& P = plan->p;
  for (int64_t j = 0; j < int64_t(P.loc_src.size()); ++j) {
    to_local[P.loc_src[j]] = 1;
    index[P.loc_src[j]] = j;
  }
  for (int64_t j = 0; j < int64_t(P.nl_src.size()); ++j) {
    to_local[P.nl_src[j]] = 0;
    index[P.nl_src[j]] = j;
  }
  return LRB_OK;
}

extern "C" int lrb_plan_export_halo(const lrb_plan* plan, int32_t* hpart, int32_t* hidx) {
  if (!plan) {
    lrb::set_error("lrb_plan_export_halo: null plan");
    return LRB_EVALUE;
  }
  if (hpart) std::copy(plan->p.hpart.begin(), plan->p.hpart.end(), hpart);
  if (hidx) std::copy(plan->p.hidx.begin(), plan->p.hidx.end(), hidx);
  return LRB_OK;
}

extern "C" int lrb_plan_export_sell(const lrb_plan* plan, int64_t* slice_ptr, int32_t* col,
                                    int32_t* src, int16_t* dpos) {
  if (!plan) {
    lrb::set_error("lrb_plan_export_sell: null plan");
    return LRB_EVALUE;
  }
  const Plan& P = plan->p;
  if (slice_ptr) std::copy(P.slice_ptr.begin(), P.slice_ptr.end(), slice_ptr);
  if (col) std::copy(P.sell_col.begin(), P.sell_col.end(), col);
  if (src) std::copy(P.sell_src.begin(), P.sell_src.end(), src);
  if (dpos) std::copy(P.dpos.begin(), P.dpos.end(), dpos);
  return LRB_OK;
}

extern "C" void lrb_plan_destroy(lrb_plan* plan) { delete plan; }

// Expose the Plan of an opaque handle to the device code.
namespace lrb {
const Plan& plan_of(const lrb_plan* p) { return p->p; }
}  // namespace lrb
