"""Device parts and teams: thin owners of native handles + PyTorch buffers.

PyTorch allocates the memory (one device arena per part, one pinned host
stage); everything else — layout, uploads, H2D copies, kernels — happens in
libldurepart_b200.so behind the C ABI.
"""

import ctypes as C
import threading
import weakref

import numpy as np

from . import _native as N


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("ldurepart_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def device_count() -> int:
    return _torch().cuda.device_count()


class Plan:
    """Host create-path artifact (lrb_plan): fused patterns + scatter inverse."""

    def __init__(self, handle):
        self.h = handle
        info = np.zeros(13, dtype=np.int64)
        N.check(N.lrb_plan_info(self.h, N.ptr(info)))
        (self.n, self.nnz_local, self.nnz_nonlocal, self.n_halo, self.n_buf, self.n_slices,
         self.sell_entries, self.max_row_len, self.n_seg, self.device_bytes,
         self.uniform_slices, self.n_patterns, self.uniform_entries) = (int(v) for v in info)
        self._csr = None

    @classmethod
    def from_ldu(cls, total, lo, hi, src_rows, face_off, lower, upper, ifc_off, ifc_row, ifc_col,
                 gpu_offsets, n_threads=0):
        h = C.c_void_p()
        arrs = [N.i64(a) for a in (src_rows, face_off, lower, upper, ifc_off, ifc_row, ifc_col,
                                   gpu_offsets)]
        src_rows, face_off, lower, upper, ifc_off, ifc_row, ifc_col, gpu_offsets = arrs
        N.check(N.lrb_plan_build_ldu(total, lo, hi, len(src_rows) - 1, N.ptr(src_rows),
                                     N.ptr(face_off), N.ptr(lower), N.ptr(upper), N.ptr(ifc_off),
                                     N.ptr(ifc_row), N.ptr(ifc_col), len(gpu_offsets) - 1,
                                     N.ptr(gpu_offsets), n_threads, C.byref(h)))
        return cls(h)

    @classmethod
    def from_coo(cls, total, lo, hi, buf_row, buf_col, seg_off=None, gpu_offsets=None):
        h = C.c_void_p()
        buf_row, buf_col = N.i64(buf_row), N.i64(buf_col)
        seg = None if seg_off is None else N.i64(seg_off)
        go = None if gpu_offsets is None else N.i64(gpu_offsets)
        N.check(N.lrb_plan_build_coo(total, lo, hi, len(buf_row), N.ptr(buf_row), N.ptr(buf_col),
                                     0 if seg is None else len(seg) - 1, N.ptr(seg),
                                     0 if go is None else len(go) - 1, N.ptr(go), C.byref(h)))
        return cls(h)

    def csr(self):
        """(loc_ptr, loc_col, nl_ptr, nl_col, halo_cols) int64, frozen."""
        if self._csr is None:
            out = (np.empty(self.n + 1, np.int64), np.empty(self.nnz_local, np.int64),
                   np.empty(self.n + 1, np.int64), np.empty(self.nnz_nonlocal, np.int64),
                   np.empty(self.n_halo, np.int64))
            N.check(N.lrb_plan_export_csr(self.h, *(N.ptr(a) for a in out)))
            for a in out:
                a.setflags(write=False)
            self._csr = out
        return self._csr

    def scatter(self):
        to_local = np.empty(self.n_buf, np.uint8)
        index = np.empty(self.n_buf, np.int64)
        N.check(N.lrb_plan_export_scatter(self.h, N.ptr(to_local), N.ptr(index)))
        return to_local.view(bool), index

    def sell(self):
        """Device layout as built on the host: (slice_ptr, col, src, dpos)."""
        sp = np.empty(self.n_slices + 1, np.int64)
        col = np.empty(self.sell_entries, np.int32)
        src = np.empty(self.sell_entries, np.int32)
        dpos = np.empty(self.n, np.int16)
        N.check(N.lrb_plan_export_sell(self.h, N.ptr(sp), N.ptr(col), N.ptr(src), N.ptr(dpos)))
        return sp, col, src, dpos

    def halo_owners(self):
        hp = np.empty(self.n_halo, np.int32)
        hi = np.empty(self.n_halo, np.int32)
        N.check(N.lrb_plan_export_halo(self.h, N.ptr(hp), N.ptr(hi)))
        return hp, hi

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            N.lrb_plan_destroy(h)


class _HostPins:
    """Page-lock producer arrays in place when they come back.

    The reference's perturb_coefficients returns the SAME off-diagonal and
    interface arrays every timestep (only the diagonal is new), so a pageable
    drop-in caller hands the update mostly the same host buffers step after
    step.  An owning array of >= 4 MB seen in a second update is registered
    (lrb_host_register) and its bytes then go straight to the device instead
    of through the part's pinned stage; the registration is dropped when the
    array is garbage collected (weakref.finalize runs before its memory is
    freed), so no stale range is ever used.  Fresh arrays (the diagonal) are
    never registered: registering costs more than one staged copy."""

    MIN_BYTES = 4 << 20

    def __init__(self):
        import os
        self._lock = threading.Lock()
        self._seen = {}      # id(owner) -> sightings (owner alive: finalize removes it)
        # LRB_PIN_REUSED=0: never page-lock caller arrays (always stage them)
        self.enabled = os.environ.get("LRB_PIN_REUSED", "1") != "0"

    @staticmethod
    def _owner(a):
        o = a
        while isinstance(o.base, np.ndarray):
            o = o.base
        return o if o.base is None and o.flags.owndata else None

    def note(self, arrays):
        if not self.enabled:
            return
        for a in arrays:
            if a.nbytes < self.MIN_BYTES:
                continue
            o = self._owner(a)
            if o is None or o.nbytes < self.MIN_BYTES:
                continue
            key = id(o)
            with self._lock:
                n = self._seen.get(key, 0)
                if n < 0 or n >= 2:
                    continue
                self._seen[key] = n + 1
                if n == 0:
                    weakref.finalize(o, self._forget, key, 0)
                    continue
                ptr = o.ctypes.data
                if N.lrb_host_register(ptr, o.nbytes) != N.LRB_OK:
                    self._seen[key] = -1      # not registrable (e.g. already pinned): stop trying
                    continue
                weakref.finalize(o, self._forget, key, ptr)

    def _forget(self, key, ptr):
        with self._lock:
            self._seen.pop(key, None)
        if ptr:
            N.lrb_host_unregister(ptr)


_host_pins = _HostPins()


class DevicePart:
    """One fused owner part on one GPU (lrb_part) with its PyTorch-owned memory."""

    def __init__(self, plan: Plan, device: int):
        torch = _torch()
        self.plan = plan
        self.device = int(device)
        self.n = plan.n
        self.n_buf = plan.n_buf
        self.arena = torch.empty(plan.device_bytes + 256, dtype=torch.uint8,
                                 device=f"cuda:{self.device}")
        base = self.arena.data_ptr()
        aligned = (base + 255) & ~255
        self.stage = torch.empty(max(plan.n_buf, 1), dtype=torch.float64, pin_memory=True)
        self.stage_np = self.stage.numpy()
        h = C.c_void_p()
        N.check(N.lrb_part_create(plan.h, self.device, aligned, plan.device_bytes,
                                  self.stage.data_ptr(), plan.n_buf, C.byref(h)))
        self.h = h
        self._values_cache = None
        self._version = 0
        self._lock = threading.Lock()
        # update epochs per segment (drop-in update(), direct mode): the last
        # epoch whose upload / scatter has been enqueued; repartition's
        # initial transfer is epoch 0
        self.seg_h2d_epoch = [0] * plan.n_seg
        self.seg_scat_epoch = [0] * plan.n_seg
        self.epoch_cv = threading.Condition()

    # ---- update path -----------------------------------------------------
    @staticmethod
    def _pieces(pieces):
        arrs = [np.ascontiguousarray(p, dtype=np.float64) for p in pieces]
        ptrs = N.ptr_array([a.ctypes.data for a in arrs])
        lens = np.array([len(a) for a in arrs], dtype=np.int64)
        return arrs, ptrs, lens

    def update_segment(self, seg, pieces):
        arrs, ptrs, lens = self._pieces(pieces)
        _host_pins.note(arrs)
        N.check(N.lrb_update_segment(self.h, seg, len(arrs), ptrs, N.ptr(lens)))
        self._touch()

    def update_segments(self, segs, pieces_per_seg):
        """Direct updates of several segments from this thread
        (lrb_update_segments); False if a piece is pageable (nothing moved)."""
        arrs = [np.ascontiguousarray(p, dtype=np.float64) for ps in pieces_per_seg for p in ps]
        ptrs = N.ptr_array([a.ctypes.data for a in arrs])
        lens = np.array([len(a) for a in arrs], dtype=np.int64)
        sg = np.asarray(segs, dtype=np.int32)
        npc = np.array([len(ps) for ps in pieces_per_seg], dtype=np.int32)
        rc = N.lrb_update_segments(self.h, len(sg), N.ptr(sg), N.ptr(npc), ptrs, N.ptr(lens))
        if rc == N.LRB_EVALUE and "pageable" in N.last_error():
            return False
        N.check(rc)
        self._touch()
        return True

    def upload_segment(self, seg, pieces):
        """H2D of one source segment only (lrb_upload_segment)."""
        arrs, ptrs, lens = self._pieces(pieces)
        _host_pins.note(arrs)
        N.check(N.lrb_upload_segment(self.h, seg, len(arrs), ptrs, N.ptr(lens)))

    def scatter_segment(self, seg):
        """The owner's scatter of one uploaded segment (lrb_scatter_segment)."""
        N.check(N.lrb_scatter_segment(self.h, seg))
        self._touch()

    def update_segment_async(self, seg, pieces, stream=0):
        """Stream-ordered direct update (lrb_update_segment_async): pieces are
        pinned host or CUDA torch tensors (float64, contiguous); no host sync.
        ``stream`` is a raw cudaStream_t (e.g. ``torch.cuda.current_stream().cuda_stream``)."""
        ptrs = N.ptr_array([t.data_ptr() for t in pieces])
        lens = np.array([t.numel() for t in pieces], dtype=np.int64)
        N.check(N.lrb_update_segment_async(self.h, seg, len(pieces), ptrs, N.ptr(lens), int(stream)))
        self._touch()

    def stage_segment(self, seg, pieces):
        arrs, ptrs, lens = self._pieces(pieces)
        N.check(N.lrb_stage_segment(self.h, seg, len(arrs), ptrs, N.ptr(lens)))

    def update_staged_from_stage(self):
        ptrs = N.ptr_array([self.stage.data_ptr()])
        lens = np.array([self.n_buf], dtype=np.int64)
        N.check(N.lrb_update_staged(self.h, 1, ptrs, N.ptr(lens)))
        self._touch()

    def apply_scatter(self):
        N.check(N.lrb_apply_scatter(self.h))
        self._touch()

    def apply_scatter_timed(self, others=()):
        """apply_scatter of this part (and ``others`` on the same GPU) with the
        scatter kernels' device time in ms (synchronous)."""
        parts = [self, *others]
        ms = C.c_float()
        N.check(N.lrb_apply_scatter_timed(len(parts), N.ptr_array([p.h.value for p in parts]),
                                          C.byref(ms)))
        for p in parts:
            p._touch()
        return float(ms.value)

    def fill(self, offset, values):
        values = np.ascontiguousarray(values, dtype=np.float64)
        N.check(N.lrb_part_fill(self.h, int(offset), N.ptr(values), len(values)))

    def read_buffer(self):
        out = np.empty(self.n_buf, np.float64)
        N.check(N.lrb_part_read_buffer(self.h, N.ptr(out)))
        return out

    def _touch(self):
        with self._lock:
            self._version += 1
            self._values_cache = None

    def read_values(self):
        """(local vals, non-local vals) in the reference's row-major order."""
        with self._lock:
            if self._values_cache is None:
                lv = np.empty(self.plan.nnz_local, np.float64)
                nv = np.empty(self.plan.nnz_nonlocal, np.float64)
                N.check(N.lrb_part_read_values(self.h, N.ptr(lv), N.ptr(nv)))
                self._values_cache = (lv, nv)
            lv, nv = self._values_cache
        return {"local": lv.copy(), "non_local": nv.copy()}

    def capture_base(self):
        """Keep a device copy of the receive buffer as it is now (the base
        coefficients) for update_perturb (lrb_part_capture_base)."""
        torch = _torch()
        self.base = torch.empty(max(self.n_buf, 1), dtype=torch.float64, device=f"cuda:{self.device}")
        N.check(N.lrb_part_capture_base(self.h, self.base.data_ptr(), 8 * self.base.numel()))

    def update_perturb(self, diag_scale):
        """Device-side perturb_coefficients + scatter (lrb_update_perturb)."""
        N.check(N.lrb_update_perturb(self.h, float(diag_scale)))
        self._touch()

    def write_values(self, which, values):
        """Write one block ("local" / "non_local") in the reference's row-major
        order into the device part (lrb_part_write_values); dinv follows."""
        values = np.ascontiguousarray(values, dtype=np.float64)
        want = self.plan.nnz_local if which == "local" else self.plan.nnz_nonlocal
        if len(values) != want:
            raise ValueError(f"{which} values: expected {want}, got {len(values)}")
        lp, np_ = (N.ptr(values), None) if which == "local" else (None, N.ptr(values))
        N.check(N.lrb_part_write_values(self.h, lp, np_))
        with self._lock:
            self._version += 1
            self._values_cache = None

    def join(self):
        N.check(N.lrb_part_join(self.h))

    def sync(self):
        N.check(N.lrb_part_sync(self.h))

    def stats(self):
        out = np.zeros(4, np.int64)
        N.check(N.lrb_part_stats(self.h, N.ptr(out)))
        return dict(zip(("pinned_pieces", "pageable_pieces", "h2d_bytes", "scatters"),
                        (int(v) for v in out)))

    def mark(self):
        N.check(N.lrb_part_mark(self.h))

    def elapsed_ms(self):
        ms = C.c_float()
        N.check(N.lrb_part_elapsed_ms(self.h, C.byref(ms)))
        return float(ms.value)

    def export(self) -> bytes:
        """Opaque blob (CUDA IPC handle + layout) for peers in other processes."""
        buf = (C.c_char * N.BLOB_BYTES)()
        N.check(N.lrb_part_export(self.h, buf))
        return bytes(buf)

    def pointers(self):
        arr = (C.c_void_p * 16)()
        N.check(N.lrb_part_pointers(self.h, arr))
        names = ("recv", "val", "x", "r", "p0", "p1", "q", "b", "dinv", "rhat", "v0", "v1", "s",
                 "t", "col", "src")
        return dict(zip(names, (int(p or 0) for p in arr)))

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            N.lrb_part_destroy(h)


class Team:
    """The owner parts of C_a; parts on one device share one persistent kernel."""

    def __init__(self, parts, dev_ranks=None):
        self.parts = list(parts)
        arr = N.ptr_array([p.h.value for p in self.parts])
        h = C.c_void_p()
        if dev_ranks is None:
            N.check(N.lrb_team_create(len(self.parts), arr, C.byref(h)))
        else:
            dr = np.ascontiguousarray(dev_ranks, dtype=np.int32)
            N.check(N.lrb_team_create_ex(len(self.parts), arr, N.ptr(dr), C.byref(h)))
        self.h = h
        self._lock = threading.Lock()

    @classmethod
    def across_processes(cls, local_parts, part_begin, n_parts, dev_rank, n_dev, allgather):
        """Team spanning processes (one per GPU).  ``allgather(bytes) -> [bytes]``
        exchanges blobs in device-rank order (e.g. torch.distributed over gloo);
        halo values and partial dots then move by NVLink peer memory only."""
        self = cls.__new__(cls)
        self.parts = [None] * n_parts
        for i, p in enumerate(local_parts):
            self.parts[part_begin + i] = p
        self._local = list(local_parts)
        self._part_begin = part_begin
        mine = b"".join(p.export() for p in local_parts)
        every = allgather(mine)
        blobs = b"".join(every)
        if len(blobs) != n_parts * N.BLOB_BYTES:
            raise ValueError("team blobs do not cover every part exactly once")
        arr = N.ptr_array([p.h.value for p in local_parts])
        h = C.c_void_p()
        team_blob = (C.c_char * N.BLOB_BYTES)()
        N.check(N.lrb_team_create_ipc(n_parts, part_begin, len(local_parts), arr, blobs, dev_rank,
                                      n_dev, C.byref(h), team_blob))
        self.h = h
        self._lock = threading.Lock()
        tblobs = b"".join(allgather(bytes(team_blob)))
        N.check(N.lrb_team_connect_ipc(self.h, tblobs))
        return self

    VECS = {"x": 2, "r": 3, "p0": 4, "p1": 5, "q": 6, "b": 7, "dinv": 8, "rhat": 9, "v0": 10,
            "v1": 11, "s": 12, "t": 13}

    def read_vector(self, part, name, n):
        """Read a vector of any team part through the team's pointer table
        (peer memory for remote parts) — diagnostics and tests."""
        out = np.empty(n, np.float64)
        N.check(N.lrb_team_read_vector(self.h, part, self.VECS[name], n, N.ptr(out)))
        return out

    def kernel_info(self, method):
        """Solve-kernel geometry on device rank 0 (lrb_team_kernel_info)."""
        out = np.zeros(8, np.int64)
        N.check(N.lrb_team_kernel_info(self.h, N.METHODS[method], N.ptr(out)))
        keys = ("streaming", "grid", "block", "stages", "stage_bytes", "smem", "halo_mirrors",
                "push_runs")
        return dict(zip(keys, (int(v) for v in out)))

    def profile(self, cap):
        """Record phase-release timestamps in later solves (cap entries; 0: off)."""
        N.check(N.lrb_team_profile(self.h, int(cap)))
        self._prof_cap = int(cap)

    def phase_times_ns(self):
        """Timestamps (ns) of the last solve's barrier releases on device rank 0."""
        cap = getattr(self, "_prof_cap", 0)
        out = np.zeros(max(cap, 1), np.int64)
        n = N.lrb_team_profile_read(self.h, N.ptr(out), cap)
        if n < 0:
            N.check(n)
        return out[:n]

    def wait_counters(self, method):
        """Per-CTA SM-cycle counters of the last streaming solve, shape
        (grid, 4 phase kinds, 8) — see stream.cuh kCnt."""
        grid = self.kernel_info(method)["grid"]
        out = np.zeros(grid * 40, np.int64)
        n = N.lrb_team_profile_counters(self.h, N.METHODS[method], N.ptr(out), len(out))
        if n < 0:
            N.check(n)
        per = out[:n].reshape(-1, 40)
        self.last_timeline_ns = per[:, 32:40]   # last phase A: see stream.cuh kStamps
        return per[:, :32].reshape(-1, 4, 8)

    def debug(self, n_dev):
        out = np.zeros(1 + n_dev, np.int64)
        N.check(N.lrb_team_debug(self.h, N.ptr(out)))
        return out

    def spmv(self, xs):
        xs = [np.ascontiguousarray(x, dtype=np.float64) for x in xs]
        ys = [np.empty(p.n, np.float64) for p in self.parts]
        N.check(N.lrb_team_spmv(self.h, N.ptr_array([x.ctypes.data for x in xs]),
                                N.ptr_array([y.ctypes.data for y in ys])))
        return ys

    def solve(self, method, bs, tol, max_iter, want_x=True, hist_cap=0):
        """Run one Krylov solve; bs None = right-hand sides already on device."""
        rep = N.Report()
        bptr = None
        if bs is not None:   # entries for remote parts (multi-process teams) are None
            bs = [None if b is None else np.ascontiguousarray(b, dtype=np.float64) for b in bs]
            bptr = N.ptr_array([0 if b is None else b.ctypes.data for b in bs])
        # solutions land in pinned host memory (torch's caching host allocator
        # recycles the blocks); the ndarray keeps its tensor alive
        torch = _torch()
        xs = [None if p is None else
              torch.empty(max(p.n, 1), dtype=torch.float64, pin_memory=True).numpy()[:p.n]
              for p in self.parts] if want_x else None
        xptr = N.ptr_array([0 if x is None else x.ctypes.data for x in xs]) if want_x else None
        hist = np.zeros(max(hist_cap, 0), np.float64)
        rc = N.lrb_team_solve(self.h, N.METHODS[method], bptr, xptr, float(tol), int(max_iter),
                              C.byref(rep), N.ptr(hist) if hist_cap > 0 else None, int(hist_cap))
        N.check(rc)
        return xs, rep, hist[:max(min(rep.iterations, hist_cap), 0)]

    @staticmethod
    def _streams(streams):
        return None if streams is None else (C.c_void_p * len(streams))(*[int(s) or None for s in streams])

    def solve_async(self, method, b_dev, x_dev, tol, max_iter, streams=None, report=None):
        """Stream-ordered solve on device tensors (lrb_team_solve_async):
        ``b_dev``/``x_dev`` one CUDA float64 tensor per part (or None lists),
        ``streams`` one raw cudaStream_t per device rank, ``report`` a pinned
        or CUDA uint8 tensor of >= 40 bytes receiving an lrb_report."""
        bp = None if b_dev is None else N.ptr_array([0 if b is None else b.data_ptr() for b in b_dev])
        xp = None if x_dev is None else N.ptr_array([0 if x is None else x.data_ptr() for x in x_dev])
        N.check(N.lrb_team_solve_async(self.h, N.METHODS[method], bp, xp, float(tol), int(max_iter),
                                       self._streams(streams),
                                       None if report is None else report.data_ptr()))

    @staticmethod
    def report_from(buf):
        """Decode an lrb_report written by solve_async (host copy of ``buf``)."""
        raw = bytes(buf.cpu().numpy().tobytes()[:C.sizeof(N.Report)])
        return N.Report.from_buffer_copy(raw)

    def spmv_async(self, x_dev, y_dev, streams=None):
        """Stream-ordered distributed SpMV on device tensors (lrb_team_spmv_async)."""
        N.check(N.lrb_team_spmv_async(self.h, N.ptr_array([x.data_ptr() for x in x_dev]),
                                      N.ptr_array([y.data_ptr() for y in y_dev]),
                                      self._streams(streams)))

    def __del__(self):
        h, self.h = getattr(self, "h", None), None
        if h:
            N.lrb_team_destroy(h)
