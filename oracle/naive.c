/*
 * C restatement of the reference brute-force executor naive_apply
 * (/root/reference/pkg/src/sparsestencil/core.py:151-182) — TEST
 * INFRASTRUCTURE ONLY (parity checker and bench.py CPU-baseline arm).
 *
 * Same semantics as the numpy original: taps in row-major kernel order
 * (rho outer, delta inner; 3D extension: rho_z, rho_y, delta), fp64
 * accumulator starting at 0, acc = acc + (w * x) with the multiply and the add
 * rounded separately (build with -ffp-contract=off), Jacobi double buffer, the
 * halo is read but never written.  Bit-identical to numpy per element.
 * Rows are split across POSIX threads (the numpy original is single-threaded).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int d, r, ntaps;
  const double* w;
  const int64_t* off; /* tap offsets in elements */
  int64_t nz, ny, nx, h, nyd, nxd;
  const double* in;
  double* out;
  int64_t row_begin, row_end; /* over nz*ny interior rows */
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  for (int64_t row = j->row_begin; row < j->row_end; ++row) {
    int64_t z = row / j->ny, y = row % j->ny;
    int64_t base = (j->d == 3 ? (z + j->h) * j->nyd * j->nxd : 0) + (y + j->h) * j->nxd + j->h;
    const double* src = j->in + base;
    double* dst = j->out + base;
    for (int64_t x = 0; x < j->nx; ++x) {
      double acc = 0.0;
      for (int t = 0; t < j->ntaps; ++t) {
        double prod = j->w[t] * src[x + j->off[t]];
        acc = acc + prod;
      }
      dst[x] = acc;
    }
  }
  return NULL;
}

static void tap_offsets(int d, int r, int64_t nyd, int64_t nxd, int64_t* off) {
  int t = 0;
  if (d == 1) {
    for (int dx = -r; dx <= r; ++dx) off[t++] = dx;
  } else if (d == 2) {
    for (int ry = -r; ry <= r; ++ry)
      for (int dx = -r; dx <= r; ++dx) off[t++] = (int64_t)ry * nxd + dx;
  } else {
    for (int rz = -r; rz <= r; ++rz)
      for (int ry = -r; ry <= r; ++ry)
        for (int dx = -r; dx <= r; ++dx) off[t++] = ((int64_t)rz * nyd + ry) * nxd + dx;
  }
}

/* Jacobi steps on two caller-owned dense buffers (both holding the halo):
 * step s reads bufs[s % 2] and writes bufs[(s + 1) % 2]; no copies, no
 * allocation of grid-sized memory (the bench's CPU-baseline arm).  Returns the
 * index (0 = a, 1 = b) of the buffer holding the result, or -1. */
int oracle_naive_steps(int d, int r, const double* coeffs, int64_t nz, int64_t ny, int64_t nx, int halo, double* a,
                       double* b, int steps, int threads) {
  if (steps < 1 || halo < r || d < 1 || d > 3) return -1;
  if (threads < 1) threads = 1;
  int span = 2 * r + 1;
  int ntaps = d == 1 ? span : (d == 2 ? span * span : span * span * span);
  int64_t h = halo, nxd = nx + 2 * h, nyd = ny + 2 * h;
  if (d != 3) nz = 1;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * ntaps);
  tap_offsets(d, r, nyd, nxd, off);
  double* bufs[2] = {a, b};
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
  int64_t rows = nz * ny;
  int cur = 0;
  for (int s = 0; s < steps; ++s) {
    for (int k = 0; k < threads; ++k) {
      job_t* j = &jobs[k];
      j->d = d; j->r = r; j->ntaps = ntaps; j->w = coeffs; j->off = off;
      j->nz = nz; j->ny = ny; j->nx = nx; j->h = h; j->nyd = nyd; j->nxd = nxd;
      j->in = bufs[cur]; j->out = bufs[1 - cur];
      j->row_begin = rows * k / threads;
      j->row_end = rows * (k + 1) / threads;
      if (threads > 1) pthread_create(&tid[k], NULL, worker, j);
      else worker(j);
    }
    if (threads > 1)
      for (int k = 0; k < threads; ++k) pthread_join(tid[k], NULL);
    cur = 1 - cur;
  }
  free(jobs);
  free(tid);
  free(off);
  return cur;
}

/* in/out: dense halo-padded arrays (2D: (ny+2h)(nx+2h), 1D uses ny = 1;
 * 3D: (nz+2h)(ny+2h)(nx+2h)).  out receives the result after `steps` steps;
 * scratch is a second buffer of the same size.  Returns 0 or -1. */
int oracle_naive_f64(int d, int r, const double* coeffs, int64_t nz, int64_t ny, int64_t nx, int halo,
                     const double* in, double* out, double* scratch, int steps, int threads) {
  if (steps < 1 || halo < r || d < 1 || d > 3) return -1;
  if (threads < 1) threads = 1;
  int span = 2 * r + 1;
  int ntaps = d == 1 ? span : (d == 2 ? span * span : span * span * span);
  int64_t h = halo, nxd = nx + 2 * h, nyd = ny + 2 * h, nzd = d == 3 ? nz + 2 * h : 1;
  if (d != 3) nz = 1;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * ntaps);
  int t = 0;
  if (d == 1) {
    for (int dx = -r; dx <= r; ++dx) off[t++] = dx;
  } else if (d == 2) {
    for (int ry = -r; ry <= r; ++ry)
      for (int dx = -r; dx <= r; ++dx) off[t++] = (int64_t)ry * nxd + dx;
  } else {
    for (int rz = -r; rz <= r; ++rz)
      for (int ry = -r; ry <= r; ++ry)
        for (int dx = -r; dx <= r; ++dx) off[t++] = ((int64_t)rz * nyd + ry) * nxd + dx;
  }
  size_t total = (size_t)(nzd * nyd * nxd);
  memcpy(out, in, total * sizeof(double));
  memcpy(scratch, in, total * sizeof(double));
  double* bufs[2] = {out, scratch};
  int cur = steps % 2 == 0 ? 0 : 1; /* the last step writes `out` */
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * threads);
  int64_t rows = nz * ny;
  for (int s = 0; s < steps; ++s) {
    for (int k = 0; k < threads; ++k) {
      job_t* j = &jobs[k];
      j->d = d; j->r = r; j->ntaps = ntaps; j->w = coeffs; j->off = off;
      j->nz = nz; j->ny = ny; j->nx = nx; j->h = h; j->nyd = nyd; j->nxd = nxd;
      j->in = bufs[cur]; j->out = bufs[1 - cur];
      j->row_begin = rows * k / threads;
      j->row_end = rows * (k + 1) / threads;
      if (threads > 1) pthread_create(&tid[k], NULL, worker, j);
      else worker(j);
    }
    if (threads > 1)
      for (int k = 0; k < threads; ++k) pthread_join(tid[k], NULL);
    cur = 1 - cur;
  }
  free(jobs);
  free(tid);
  free(off);
  return 0;
}
