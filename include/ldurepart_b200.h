/*
 * ldurepart_b200 — C ABI of the B200-native repartition / update / solve path.
 *
 * Drop-in boundary for the reference package `ldurepart`
 * (/root/reference/pkg/src/ldurepart/).  Every entry point names the reference
 * interface it replaces (file:line).  Plain pointers and sizes only: device
 * pointers are `void*`/typed pointers into memory owned by the caller (PyTorch
 * in this repo), host pointers are ordinary (pinned or pageable) memory.
 *
 * Status codes: 0 = ok; LRB_EVALUE maps to Python ValueError, LRB_ERUNTIME to
 * RuntimeError, LRB_ECUDA to a CUDA failure, LRB_ENOTPD to
 * ValueError("cg: matrix is not positive definite") (solver.py:129-130),
 * LRB_ETIMEOUT to a cross-device barrier timeout.  The thread-local message of
 * the last failure is returned by lrb_last_error().
 *
 * There is no CPU fallback: every compute entry point launches sm_100a code.
 */
#ifndef LDUREPART_B200_H
#define LDUREPART_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRB_OK 0
#define LRB_EVALUE (-1)
#define LRB_ERUNTIME (-2)
#define LRB_ECUDA (-3)
#define LRB_ENOTPD (-4)
#define LRB_ETIMEOUT (-5)

#define LRB_METHOD_CG 0        /* solver.py:100-147 (unpreconditioned CG) */
#define LRB_METHOD_PCG 1       /* Jacobi-PCG */
#define LRB_METHOD_BICGSTAB 2  /* BiCGStab */
#define LRB_METHOD_PCG1 3      /* single-reduction (Chronopoulos-Gear) Jacobi-PCG, SURVEY.md §8 f1:
                                  one team barrier per iteration; CG's iterates up to rounding */
#define LRB_METHOD_PIPECG 4    /* pipelined (Ghysels-Vanroose) Jacobi-PCG: the
                                  iteration's reduction completes behind the next SpMV (flat
                                  teams read it one phase late); CG's iterates up to rounding */

const char* lrb_last_error(void);
const char* lrb_version(void);
int lrb_device_count(void);
/* Number of kernels this library has launched since load (bench gpu_launches). */
uint64_t lrb_launch_count(void);

/* ------------------------------------------------------------------------
 * Create path (host, integer; bit-exact with the reference).
 * ------------------------------------------------------------------------ */
typedef struct lrb_plan lrb_plan;

/* Fused owner plan from the LDU addressing of its alpha sources.
 * Replaces, for one owner k, extract_sparsity (repart.py:143-174),
 * fuse_patterns (repart.py:197-236), pack_order_pairs (repart.py:253-270),
 * build_scatter_map (repart.py:273-304) and _build_matrix (repart.py:307-318).
 *   total_cells        pm.total_cells
 *   row_lo, row_hi     I_GPU(k) (core.py:198-202)
 *   n_src              alpha; src_rows[n_src+1] = global row offsets of the sources
 *   face_off[n_src+1], lower[], upper[]   concatenated source-local face addresses
 *   ifc_off[n_src+1], ifc_row[] (source-local), ifc_col[] (global)
 *                      interface entries in pack order (blocks by neighbour rank)
 *   n_gpu, gpu_offsets[n_gpu+1]  GPU row ranges, to resolve halo owners
 *   n_threads          host worker threads (<= 0: hardware concurrency)          */
int lrb_plan_build_ldu(int64_t total_cells, int64_t row_lo, int64_t row_hi, int32_t n_src,
                       const int64_t* src_rows, const int64_t* face_off,
                       const int64_t* lower, const int64_t* upper, const int64_t* ifc_off,
                       const int64_t* ifc_row, const int64_t* ifc_col, int32_t n_gpu,
                       const int64_t* gpu_offsets, int32_t n_threads, lrb_plan** out);

/* Same plan from explicit buffer provenance: buffer entry b carries global
 * (buf_row[b], buf_col[b]); seg_off[n_seg+1] splits the buffer by source.
 * Serves the low-level fuse_patterns / build_scatter_map API (repart.py:197-304). */
int lrb_plan_build_coo(int64_t total_cells, int64_t row_lo, int64_t row_hi, int64_t n_buf,
                       const int64_t* buf_row, const int64_t* buf_col, int32_t n_seg,
                       const int64_t* seg_off, int32_t n_gpu, const int64_t* gpu_offsets,
                       lrb_plan** out);

/* info[0..12] = n_rows, nnz_local, nnz_nonlocal, n_halo, n_buf, n_slices,
 *               sell_entries, max_row_len, n_seg, part_device_bytes,
 *               uniform (pattern) slices, n_patterns, entries in uniform slices */
int lrb_plan_info(const lrb_plan* plan, int64_t* info);
/* Reference DistributedCooMatrix patterns in CSR form (core.py:247-288):
 * loc_ptr/nl_ptr [n+1]; loc_col part-local; nl_col = index into halo_cols. */
int lrb_plan_export_csr(const lrb_plan* plan, int64_t* loc_ptr, int64_t* loc_col,
                        int64_t* nl_ptr, int64_t* nl_col, int64_t* halo_cols);
/* Reference ScatterMap (repart.py:82-106): to_local[b], index[b] per buffer entry. */
int lrb_plan_export_scatter(const lrb_plan* plan, uint8_t* to_local, int64_t* index);
/* Halo owners: hpart[s] (GPU rank) and hidx[s] (row in that part) per halo slot. */
int lrb_plan_export_halo(const lrb_plan* plan, int32_t* hpart, int32_t* hidx);
/* The device layout (SELL-32) as built on the host: slice_ptr[n_slices+1],
 * col/src[sell_entries] (col >= n: halo slot col-n; -1: padding), dpos[n]. */
int lrb_plan_export_sell(const lrb_plan* plan, int64_t* slice_ptr, int32_t* col, int32_t* src,
                         int16_t* dpos);
void lrb_plan_destroy(lrb_plan* plan);

/* ------------------------------------------------------------------------
 * Device part (one fused owner part on one GPU).
 * ------------------------------------------------------------------------ */
typedef struct lrb_part lrb_part;

/* Lay the part out in a caller-owned device arena of plan_info()[9] bytes
 * (256-byte aligned) and upload the SELL matrix, scatter inverse and halo
 * tables.  host_stage (pinned, n_buf doubles, nullable) serves pageable and
 * staged updates.  Replaces ctx.alloc_device (repart.py:347). */
int lrb_part_create(const lrb_plan* plan, int32_t device, void* dev_arena, int64_t dev_bytes,
                    double* host_stage, int64_t host_stage_len, lrb_part** out);
void lrb_part_destroy(lrb_part* part);
/* Device pointers of the receive buffer and vectors (for tests / bench). */
int lrb_part_pointers(const lrb_part* part, void** ptrs /* [16] */);

/* Direct update of one source segment (update.py:72-83, transport.py:115-123):
 * n_pieces host arrays are copied back to back into segment `seg` of the
 * owner's receive buffer (diag | upper | lower | interface blocks: no host
 * pack), pinned pieces straight to the device, pageable pieces via the pinned
 * stage; then that segment's scatter kernel runs on the segment's stream.
 * Returns once the host pieces may be reused (H2D complete). */
int lrb_update_segment(lrb_part* part, int32_t seg, int32_t n_pieces,
                       const double* const* pieces, const int64_t* piece_len);
/* The direct update split at its two owners (update.py:72-83 + 105-112): a
 * source rank uploads its segment into the receive buffer (returns when its
 * pieces may be reused; never waits for the owner — the solve does not read
 * the receive buffer), and the owner, once its previous solve is done,
 * scatters every uploaded segment on that segment's stream.  The drop-in's
 * update() orders the two by update epochs, so a source's upload of the next
 * system overlaps the owner's solves of another (C4: pressure coefficients
 * during the momentum solves). */
/* Page-lock an existing host range in place (cudaHostRegister) / release it:
 * the drop-in registers a producer's coefficient arrays that come back in a
 * second update (the reference's perturb_coefficients returns the same
 * off-diagonal arrays every timestep), so their bytes go straight to the
 * device instead of through the stage; unregistered when the array dies. */
int lrb_host_register(void* ptr, int64_t bytes);
int lrb_host_unregister(void* ptr);
int lrb_upload_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                       const int64_t* piece_len);
/* Several sources' direct updates of one part from ONE host thread: segment
 * segs[i] gets the next seg_pieces[i] pieces (all pinned; a pageable piece
 * is rejected with LRB_EVALUE before anything moves); every H2D + scatter is
 * enqueued on its segment's stream before the single wait.  For hosts that
 * drive many sources per GPU (C5: 16 sources per part). */
int lrb_update_segments(lrb_part* part, int32_t n_seg, const int32_t* segs, const int32_t* seg_pieces,
                        const double* const* pieces, const int64_t* piece_len);
int lrb_scatter_segment(lrb_part* part, int32_t seg);
/* Staged update (update.py:85-102): the owner copies all sources' pieces
 * into the pinned stage, then one H2D of the whole buffer and the scatter. */
int lrb_update_staged(lrb_part* part, int32_t n_pieces, const double* const* pieces,
                      const int64_t* piece_len);
/* Staged update, source side: copy one source's pieces into the owner's
 * pinned host stage at segment `seg` (the owner-side host gather,
 * update.py:85-100); the owner then calls lrb_update_staged with the stage. */
int lrb_stage_segment(lrb_part* part, int32_t seg, int32_t n_pieces, const double* const* pieces,
                      const int64_t* piece_len);
/* apply_scatter (update.py:105-112) of the whole device-resident buffer. */
int lrb_apply_scatter(lrb_part* part);
/* The same for n_parts parts of one device, synchronously, returning the
 * device time from just before the first scatter launch to the end of the
 * last (CUDA events around the launches, no host gap inside; bench `value`). */
int lrb_apply_scatter_timed(int32_t n_parts, lrb_part* const* parts, float* device_ms);
/* Write host values into the receive buffer (DeviceBuffer.fill, transport.py:115-123). */
int lrb_part_fill(lrb_part* part, int64_t offset, const double* values, int64_t n);
/* Read back the receive buffer (DeviceBuffer.values, transport.py:125-127). */
int lrb_part_read_buffer(lrb_part* part, double* out);
/* Read the fused values in the reference's row-major local / non-local order
 * (DistributedCooMatrix.local.vals / non_local.vals). */
int lrb_part_read_values(lrb_part* part, double* local_vals, double* nonlocal_vals);
/* Write values in the reference's row-major local / non-local order into the
 * part (either pointer nullable: that block is kept), then refresh the Jacobi
 * diagonal.  Backs the drop-in's writable DistributedCooMatrix .vals (the
 * reference keeps CooMatrix values writable by design, tests/test_core.py:121). */
int lrb_part_write_values(lrb_part* part, const double* local_vals, const double* nonlocal_vals);
/* GPU-side producer (the paper's "refactoring approach",
 * PAPER.md:23-27).  lrb_part_capture_base copies the receive buffer as it is
 * now (the pristine base coefficients, e.g. right after repartition) into a
 * caller-owned device buffer of 8 * n_buf bytes; lrb_update_perturb then
 * produces a timestep's values on the device — the base with every diagonal
 * scaled by diag_scale, which is perturb_coefficients (assembly.py:225-243)
 * for diag_scale = 1 + step/100 — fused with the scatter, ordered on the
 * part's solve stream.  Values equal the host path bit for bit; no
 * coefficients cross PCIe.  The receive buffer keeps the last transferred
 * values. */
int lrb_part_capture_base(lrb_part* part, void* dev_buf, int64_t bytes);
int lrb_update_perturb(lrb_part* part, double diag_scale);
/* Make the part's solve stream wait for all pending segment scatters. */
int lrb_part_join(lrb_part* part);
int lrb_part_sync(lrb_part* part);
/* out[4] = pieces copied zero-copy from pinned memory, pageable pieces staged,
 * H2D bytes, scatter launches (since create). */
int lrb_part_stats(const lrb_part* part, int64_t* out);
/* Device time (ms) between the last two lrb_part_mark() calls on the solve stream. */
int lrb_part_mark(lrb_part* part);
int lrb_part_elapsed_ms(lrb_part* part, float* ms);

/* ------------------------------------------------------------------------
 * Team: the owner parts of the active communicator C_a (transport.py:461-472).
 * Parts are in GPU-rank order.  Parts on the same device run in one
 * persistent kernel; parts on different devices of this process exchange halo
 * values and partial dot products through NVLink peer memory.
 * ------------------------------------------------------------------------ */
typedef struct lrb_team lrb_team;

int lrb_team_create(int32_t n_parts, lrb_part* const* parts, lrb_team** out);
/* As lrb_team_create with an explicit device rank per part: parts on one CUDA
 * device but with different ranks run as separate kernels that synchronise
 * through the cross-device (peer-memory flag) protocol — exercised by the
 * tests on a single GPU. */
int lrb_team_create_ex(int32_t n_parts, lrb_part* const* parts, const int32_t* dev_rank_of_part,
                       lrb_team** out);
void lrb_team_destroy(lrb_team* team);

/* Teams spanning processes (one process per GPU, e.g. torchrun): the caller
 * exchanges opaque blobs (e.g. torch.distributed all_gather) — no NCCL on
 * the data path; halo values and partial dot products move by NVLink peer
 * loads/stores from inside the solve kernels.
 *  1. every process: lrb_part_export(part, blob) for its part(s);
 *  2. all-gather the part blobs in GPU-rank order;
 *  3. lrb_team_create_ipc(...) opens the peers' arenas and returns this
 *     device's team-workspace blob;
 *  4. all-gather the team blobs; lrb_team_connect_ipc(team, blobs). */
#define LRB_BLOB_BYTES 512
int lrb_part_export(const lrb_part* part, void* blob);
int lrb_team_create_ipc(int32_t n_parts, int32_t part_begin, int32_t n_local,
                        lrb_part* const* local_parts, const void* part_blobs /* n_parts x 512 */,
                        int32_t dev_rank, int32_t n_dev, lrb_team** out, void* team_blob);
int lrb_team_connect_ipc(lrb_team* team, const void* team_blobs /* n_dev x 512 */);
/* Diagnostics: copy n doubles of vector `vec` (index as in lrb_part_pointers,
 * 2 = x ... 13 = t) of team part `part` — local or a peer's, through the
 * team's own pointer table — into host memory; and this device's barrier
 * state: out[0] = epoch, out[1..n_dev] = arrival flags written by peers. */
int lrb_team_read_vector(lrb_team* team, int32_t part, int32_t vec, int64_t n, double* out);
int lrb_team_debug(lrb_team* team, int64_t* out);
/* Launch geometry of the solve kernel of `method` on device rank 0:
 * out[0] = 1 streaming (bulk-copy, stream.cuh) / 0 classic (kernels.cuh),
 * out[1] = grid, out[2] = block, out[3] = ring stages, out[4] = stage bytes,
 * out[5] = dynamic shared memory bytes, out[6] = 1 if halo mirrors are on
 * (owners push boundary rows into the readers' mirrors; the streaming CG /
 * PCG / BiCGStab kernels read halo operands locally; LRB_HALO=direct at team
 * creation turns them off), out[7] = halo push runs of device rank 0's parts.  LRB_SOLVER=classic at team creation
 * selects the classic kernels. */
int lrb_team_kernel_info(lrb_team* team, int32_t method, int64_t* out /* [8] */);
/* Phase profiling (diagnostics): with cap > 0 every later solve records the
 * globaltimer (ns) at each team-barrier release, up to cap entries (cap = 0
 * turns it off).  lrb_team_profile_read copies the last solve's timestamps of
 * device rank 0 and returns their count (negative: error).  Phase order:
 * init, then per iteration A (SpMV + p.q), B (update + r.r), [C (true
 * residual)]. */
int lrb_team_profile(lrb_team* team, int32_t cap);
int lrb_team_profile_read(lrb_team* team, int64_t* out, int32_t cap);
/* Streaming solvers with profiling on: per-CTA SM-cycle counters of the last
 * solve of `method`, 32 per CTA = [phase kind: init, A, B, C][consumer data
 * wait, end-of-phase barrier, producer stage wait, team barrier, row bodies,
 * group reduce, tile sums, producer issue] (stream.cuh kCnt); returns the
 * number of values copied (0: not streaming / profiling off). */
int lrb_team_profile_counters(lrb_team* team, int32_t method, int64_t* out, int32_t cap);

/* Distributed SpMV y = A x (solver.py:80-97): x_host/y_host per part. */
int lrb_team_spmv(lrb_team* team, const double* const* x_host, double* const* y_host);

typedef struct lrb_report {
  int32_t iterations;
  int32_t converged;
  int32_t breakdown;
  int32_t status;
  double residual;
  double bnorm;
  double device_ms;   /* solve-kernel device time */
} lrb_report;

/* Krylov solve (cg_solve, solver.py:100-147; PCG/BiCGStab per SURVEY App. A).
 * b_host/x_host per part (nullable: b already on device / leave x on device).
 * hist (nullable) receives the recurrence residual per iteration.
 * LRB_ETIMEOUT: a cross-device barrier waited longer than
 * LRB_BARRIER_TIMEOUT_S (default 20 s) for a peer; the team is then poisoned
 * (its devices' barrier epochs disagree) and every later solve on it fails
 * with LRB_ETIMEOUT until it is destroyed and recreated. */
int lrb_team_solve(lrb_team* team, int32_t method, const double* const* b_host,
                   double* const* x_host, double tol, int32_t max_iter, lrb_report* rep,
                   double* hist, int32_t hist_cap);

/* ------------------------------------------------------------------------
 * Stream-ordered entry points for a GPU-resident caller (the OGL lduMatrix
 * solver plugin role; SURVEY.md §8(b) lrb_update_h2d /
 * lrb_krylov).  Nothing here synchronises the host: the work is enqueued
 * after everything already on the caller's stream, and the caller's stream
 * is made to wait for it.  lrb_stream_t is cudaStream_t (NULL = the legacy
 * default stream).
 * ------------------------------------------------------------------------ */
typedef struct CUstream_st* lrb_stream_t;

/* Direct update of one source segment (update.py:72-83 + apply_scatter,
 * update.py:105-112) ordered on `stream`: the pieces (pinned host or device
 * memory — pageable host memory is rejected with LRB_EVALUE, it cannot be
 * copied stream-ordered) are copied into segment `seg` of the receive
 * buffer, then that segment's scatter runs on the same stream.  The pieces
 * must stay valid until the stream reaches the copy.  The next solve on the
 * part waits for it. */
int lrb_update_segment_async(lrb_part* part, int32_t seg, int32_t n_pieces,
                             const double* const* pieces, const int64_t* piece_len,
                             lrb_stream_t stream);

/* Krylov solve (cg_solve, solver.py:100-147) ordered on streams[dev_rank]
 * (streams nullable; a NULL array means each device's team stream with no
 * caller ordering).  b_dev / x_dev: one DEVICE pointer per team part on the
 * part's GPU (nullable array: b already in the part / x left in the part).
 * rep_out (nullable): pinned host or device memory; the report is written
 * stream-ordered after the solve (device_ms = -1: no host timing).  Status
 * codes of the solve itself (not positive definite, barrier timeout) land in
 * rep_out->status.  Single-process teams only. */
int lrb_team_solve_async(lrb_team* team, int32_t method, const double* const* b_dev,
                         double* const* x_dev, double tol, int32_t max_iter,
                         const lrb_stream_t* streams, lrb_report* rep_out);

/* Distributed SpMV y = A x (solver.py:80-97) on device pointers, ordered on
 * streams[dev_rank] like lrb_team_solve_async.  Single-process teams only. */
int lrb_team_spmv_async(lrb_team* team, const double* const* x_dev, double* const* y_dev,
                        const lrb_stream_t* streams);

#ifdef __cplusplus
}
#endif
#endif /* LDUREPART_B200_H */
