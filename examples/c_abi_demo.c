/*
 * c_abi_demo.c — the drop-in boundary driven from C, no Python: what a
 * compiled host (e.g. the OGL lduMatrix solver plugin of the paper,
 * PAPER.md:202) would do with include/ldurepart_b200.h.
 *
 * A unit 3D Laplacian on an N^3 grid, assembled by 2 "CPU ranks" as slabs
 * along z in LDU form (assembly.py:120-222 numbering: x fastest, faces
 * sorted by (lower, upper), interface blocks toward the neighbour slab),
 * repartitioned onto ONE GPU part (alpha 2): create the plan from the LDU
 * addressing, lay the part out in a caller-owned device arena, then per
 * timestep upload each source's coefficient pieces (diag scaled by
 * 1 + step/100, off-diagonals -1) from pinned memory and run Jacobi-PCG to
 * 1e-6 on b = ones — synchronously, and once more stream-ordered with device
 * b / x (lrb_update_segment_async + lrb_team_solve_async).
 *
 *   build: see tests/test_c_abi_demo.py (gcc ... -lldurepart_b200 -lcudart)
 *   run:   ./c_abi_demo N  -> one JSON line per timestep
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ldurepart_b200.h"

#define CHECK(x)                                                             \
  do {                                                                       \
    int rc_ = (x);                                                           \
    if (rc_ != 0) {                                                          \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, lrb_last_error());     \
      return 1;                                                              \
    }                                                                        \
  } while (0)
#define CUDA(x)                                                              \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));               \
      return 1;                                                              \
    }                                                                        \
  } while (0)

typedef struct {
  int64_t lo, n, nz, n_faces, n_ifc;
  int64_t *lower, *upper;       /* source-local face addressing */
  int64_t *ifc_row, *ifc_col;   /* interface entries: source-local row, global column */
  double* vals;                 /* pinned: [diag | upper | lower | iface] (pack order) */
} Source;

static void build_source(Source* s, int64_t N, int64_t z0, int64_t z1, int rank, int n_ranks) {
  const int64_t P = N * N;
  s->lo = z0 * P;
  s->nz = z1 - z0;
  s->n = s->nz * P;
  s->n_faces = 0;
  s->lower = malloc(sizeof(int64_t) * 3 * s->n);
  s->upper = malloc(sizeof(int64_t) * 3 * s->n);
  for (int64_t i = 0; i < s->n; ++i) {   /* faces sorted by (l, u): u = l+1, l+N, l+P */
    const int64_t x = i % N, y = (i / N) % N, z = i / P;
    if (x < N - 1) s->lower[s->n_faces] = i, s->upper[s->n_faces++] = i + 1;
    if (y < N - 1) s->lower[s->n_faces] = i, s->upper[s->n_faces++] = i + N;
    if (z < s->nz - 1) s->lower[s->n_faces] = i, s->upper[s->n_faces++] = i + P;
  }
  /* interface blocks by ascending neighbour rank, each in (row, col) order */
  s->n_ifc = 0;
  s->ifc_row = malloc(sizeof(int64_t) * 2 * P);
  s->ifc_col = malloc(sizeof(int64_t) * 2 * P);
  if (rank > 0)   /* first plane -> previous slab's last plane */
    for (int64_t c = 0; c < P; ++c) s->ifc_row[s->n_ifc] = c, s->ifc_col[s->n_ifc++] = s->lo + c - P;
  if (rank < n_ranks - 1)   /* last plane -> next slab's first plane */
    for (int64_t c = 0; c < P; ++c)
      s->ifc_row[s->n_ifc] = (s->nz - 1) * P + c, s->ifc_col[s->n_ifc++] = s->lo + s->n + c;
}

static int64_t pack_len(const Source* s) { return s->n + 2 * s->n_faces + s->n_ifc; }

static void produce(Source* s, int step) {   /* perturb_coefficients (assembly.py:225-243) */
  const double f = 1.0 + step / 100.0;
  double* v = s->vals;
  for (int64_t i = 0; i < s->n; ++i) v[i] = 6.0 * f;   /* 6 faces per cell */
  for (int64_t i = s->n; i < pack_len(s); ++i) v[i] = -1.0;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 32;
  const int n_src = 2;
  const int64_t total = N * N * N;
  Source src[2];
  build_source(&src[0], N, 0, N / 2, 0, 2);
  build_source(&src[1], N, N / 2, N, 1, 2);

  /* ---- create: concatenated addressing of the owner's sources ---- */
  int64_t src_rows[3] = {0, src[1].lo, total}, face_off[3], ifc_off[3];
  face_off[0] = ifc_off[0] = 0;
  for (int k = 0; k < 2; ++k) {
    face_off[k + 1] = face_off[k] + src[k].n_faces;
    ifc_off[k + 1] = ifc_off[k] + src[k].n_ifc;
  }
  int64_t* lower = malloc(sizeof(int64_t) * face_off[2]);
  int64_t* upper = malloc(sizeof(int64_t) * face_off[2]);
  int64_t* irow = malloc(sizeof(int64_t) * (ifc_off[2] + 1));
  int64_t* icol = malloc(sizeof(int64_t) * (ifc_off[2] + 1));
  for (int k = 0; k < 2; ++k) {
    memcpy(lower + face_off[k], src[k].lower, sizeof(int64_t) * src[k].n_faces);
    memcpy(upper + face_off[k], src[k].upper, sizeof(int64_t) * src[k].n_faces);
    memcpy(irow + ifc_off[k], src[k].ifc_row, sizeof(int64_t) * src[k].n_ifc);
    memcpy(icol + ifc_off[k], src[k].ifc_col, sizeof(int64_t) * src[k].n_ifc);
  }
  int64_t gpu_offsets[2] = {0, total};
  lrb_plan* plan = NULL;
  CHECK(lrb_plan_build_ldu(total, 0, total, n_src, src_rows, face_off, lower, upper, ifc_off, irow,
                           icol, 1, gpu_offsets, 0, &plan));
  int64_t info[13];
  CHECK(lrb_plan_info(plan, info));
  const int64_t n = info[0], n_buf = info[4], bytes = info[9];

  /* caller-owned memory: device arena, pinned stage, pinned coefficients */
  void* arena = NULL;
  double* stage = NULL;
  CUDA(cudaMalloc(&arena, (size_t)bytes));
  CUDA(cudaMallocHost((void**)&stage, sizeof(double) * n_buf));
  for (int k = 0; k < 2; ++k) CUDA(cudaMallocHost((void**)&src[k].vals, sizeof(double) * pack_len(&src[k])));
  lrb_part* part = NULL;
  CHECK(lrb_part_create(plan, 0, arena, bytes, stage, n_buf, &part));
  lrb_team* team = NULL;
  CHECK(lrb_team_create(1, &part, &team));

  double *b = NULL, *x = NULL;
  CUDA(cudaMallocHost((void**)&b, sizeof(double) * n));
  CUDA(cudaMallocHost((void**)&x, sizeof(double) * n));
  for (int64_t i = 0; i < n; ++i) b[i] = 1.0;

  /* ---- timesteps: update every source's segment, then Jacobi-PCG ---- */
  for (int step = 2; step <= 4; ++step) {
    for (int k = 0; k < 2; ++k) {
      produce(&src[k], step);
      const double* pieces[1] = {src[k].vals};   /* one pack-order piece per source */
      const int64_t lens[1] = {pack_len(&src[k])};
      CHECK(lrb_update_segment(part, k, 1, pieces, lens));
    }
    CHECK(lrb_part_join(part));
    const double* bs[1] = {b};
    double* xs[1] = {x};
    lrb_report rep;
    CHECK(lrb_team_solve(team, LRB_METHOD_PCG, bs, xs, 1e-6, 2000, &rep, NULL, 0));
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) sum += x[i];
    printf("{\"mode\": \"sync\", \"step\": %d, \"iterations\": %d, \"converged\": %d, "
           "\"residual\": %.17g, \"x_sum\": %.17g, \"x0\": %.17g}\n",
           step, rep.iterations, rep.converged, rep.residual, sum, x[0]);
  }

  /* ---- the same last step stream-ordered, b and x in device memory ---- */
  cudaStream_t st;
  CUDA(cudaStreamCreate(&st));
  double *b_dev = NULL, *x_dev = NULL;
  lrb_report* rep_h = NULL;
  CUDA(cudaMalloc((void**)&b_dev, sizeof(double) * n));
  CUDA(cudaMalloc((void**)&x_dev, sizeof(double) * n));
  CUDA(cudaMallocHost((void**)&rep_h, sizeof(lrb_report)));
  CUDA(cudaMemcpyAsync(b_dev, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  for (int k = 0; k < 2; ++k) {
    const double* pieces[1] = {src[k].vals};
    const int64_t lens[1] = {pack_len(&src[k])};
    CHECK(lrb_update_segment_async(part, k, 1, pieces, lens, st));
  }
  const double* bd[1] = {b_dev};
  double* xd[1] = {x_dev};
  CHECK(lrb_team_solve_async(team, LRB_METHOD_PCG, bd, xd, 1e-6, 2000, &st, rep_h));
  CUDA(cudaMemcpyAsync(x, x_dev, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  CUDA(cudaStreamSynchronize(st));
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) sum += x[i];
  printf("{\"mode\": \"async\", \"step\": 4, \"iterations\": %d, \"converged\": %d, "
         "\"residual\": %.17g, \"x_sum\": %.17g, \"x0\": %.17g}\n",
         rep_h->iterations, rep_h->converged, rep_h->residual, sum, x[0]);

  lrb_team_destroy(team);
  lrb_part_destroy(part);
  lrb_plan_destroy(plan);
  cudaFree(arena);
  cudaFree(b_dev);
  cudaFree(x_dev);
  return 0;
}
