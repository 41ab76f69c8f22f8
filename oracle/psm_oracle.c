/*
 * psm_oracle.c -- C restatement of the reference line smoother.
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY.  Nothing in paper_1208_1975_b200
 * links or calls this; tests/ use it as a checker and bench.py times it as
 * the CPU baseline ("port": the reference is pure Python and has no native
 * code to build).
 *
 * Follows /root/reference/pkg/src/patchsmooth:
 *   fill_physical_ghosts   grid.py:311-330  (ghost = -interior, x, y, z)
 *   block_residual         stencil.py:93-112 (acc = c*u; acc += face*nbr in
 *                          order -x,+x,-y,+y,-z,+z; r = f - acc)
 *   _jacobi_step           smoother.py:138-153 (v = u + omega*Ainv r)
 *   residual_norm          smoother.py:96-109 (sum of r^2; here a plain
 *                          ordered sum, not fsum)
 * with the exact line-block inverse applied by a Thomas solve along x
 * (the closure-free block of stencil.py:115-138 is tridiag(f-x, c, f+x)).
 * Lines are distributed over OpenMP threads.  Also: serial line GS
 * (oracle_line_gs) and the residual sum of squares, for the full-size
 * parity checks of tests/test_configs_gpu.py.
 */
#include <math.h>
#include <stdlib.h>
#include <omp.h>

#define IDX(i, j, k) ((size_t)(i) + px * ((size_t)(j) + py * (size_t)(k)))

void oracle_fill_ghosts(double* u, int nx, int ny, int nz, int nthreads) {
  const size_t px = nx + 2, py = ny + 2, pz = nz + 2;
#pragma omp parallel for num_threads(nthreads) collapse(2)
  for (size_t k = 0; k < pz; ++k)
    for (size_t j = 0; j < py; ++j) {
      u[IDX(0, j, k)] = -u[IDX(1, j, k)];
      u[IDX(px - 1, j, k)] = -u[IDX(px - 2, j, k)];
    }
#pragma omp parallel for num_threads(nthreads) collapse(2)
  for (size_t k = 0; k < pz; ++k)
    for (size_t i = 0; i < px; ++i) {
      u[IDX(i, 0, k)] = -u[IDX(i, 1, k)];
      u[IDX(i, py - 1, k)] = -u[IDX(i, py - 2, k)];
    }
#pragma omp parallel for num_threads(nthreads) collapse(2)
  for (size_t j = 0; j < py; ++j)
    for (size_t i = 0; i < px; ++i) {
      u[IDX(i, j, 0)] = -u[IDX(i, j, 1)];
      u[IDX(i, j, pz - 1)] = -u[IDX(i, j, pz - 2)];
    }
}

static inline double resid(const double* u, size_t c, size_t px, size_t pxy, double f, double cc,
                           const double* fc) {
  double acc = cc * u[c];
  acc += fc[0] * u[c - 1];
  acc += fc[1] * u[c + 1];
  acc += fc[2] * u[c - px];
  acc += fc[3] * u[c + px];
  acc += fc[4] * u[c - pxy];
  acc += fc[5] * u[c + pxy];
  return f - acc;
}

/* One line-Jacobi sweep of a single patch: v interior <- u + omega*Ainv r.
 * Returns sum of r^2 (the residual norm^2 of u).  u must have fresh ghosts. */
double oracle_line_jacobi(const double* u, const double* f, double* v, int nx, int ny, int nz, double cc,
                          const double* fc, double omega, int solve, int nthreads) {
  const size_t px = nx + 2, py = ny + 2, pxy = px * py;
  double* cp = (double*)malloc(sizeof(double) * nx);
  double* im = (double*)malloc(sizeof(double) * nx);
  double prev = 0.0;
  for (int i = 0; i < nx; ++i) {
    double m = cc - fc[0] * prev;
    im[i] = 1.0 / m;
    cp[i] = fc[1] / m;
    prev = cp[i];
  }
  double total = 0.0;
  const long lines = (long)ny * nz;
#pragma omp parallel num_threads(nthreads) reduction(+ : total)
  {
    double* y = (double*)malloc(sizeof(double) * nx);
#pragma omp for schedule(static)
    for (long l = 0; l < lines; ++l) {
      const int j = (int)(l % ny), k = (int)(l / ny);
      const size_t base = IDX(1, j + 1, k + 1);
      const double* fr = f + (size_t)l * nx;
      double ss = 0.0, pr = 0.0;
      for (int i = 0; i < nx; ++i) {
        const double r = resid(u, base + i, px, pxy, fr[i], cc, fc);
        ss += r * r;
        pr = (r - fc[0] * pr) * im[i];
        y[i] = pr;
      }
      total += ss;
      if (solve) {
        for (int i = nx - 2; i >= 0; --i) y[i] -= cp[i] * y[i + 1];
        for (int i = 0; i < nx; ++i) v[base + i] = u[base + i] + omega * y[i];
      }
    }
    free(y);
  }
  free(cp);
  free(im);
  return total;
}

/* One serial (lexicographic) line Gauss-Seidel sweep of a single patch, in
 * place: smoother.py:156-169 under the serial strategy (runtime.py:164-168),
 * lines (j,k) in x-fastest block order (grid.py:300-307), each line's
 * residual read from the current u (block_residual, stencil.py:93-112) and
 * u_line <- u_line + omega * Ainv r (block_update, smoother.py:90-93).  The
 * ghosts are read as stored (lagged to step end, as in the reference).  The
 * line inverse is the same Thomas solve as oracle_line_jacobi.  One thread
 * per patch: callers run different patches on different threads. */
void oracle_line_gs(double* u, const double* f, int nx, int ny, int nz, double cc, const double* fc,
                    double omega) {
  const size_t px = nx + 2, py = ny + 2, pxy = px * py;
  double* cp = (double*)malloc(sizeof(double) * nx);
  double* im = (double*)malloc(sizeof(double) * nx);
  double* y = (double*)malloc(sizeof(double) * nx);
  double prev = 0.0;
  for (int i = 0; i < nx; ++i) {
    double m = cc - fc[0] * prev;
    im[i] = 1.0 / m;
    cp[i] = fc[1] / m;
    prev = cp[i];
  }
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j) {
      const size_t base = IDX(1, j + 1, k + 1);
      const double* fr = f + ((size_t)k * ny + j) * nx;
      double pr = 0.0;
      for (int i = 0; i < nx; ++i) {
        const double r = resid(u, base + i, px, pxy, fr[i], cc, fc);
        pr = (r - fc[0] * pr) * im[i];
        y[i] = pr;
      }
      for (int i = nx - 2; i >= 0; --i) y[i] -= cp[i] * y[i + 1];
      for (int i = 0; i < nx; ++i) u[base + i] = u[base + i] + omega * y[i];
    }
  free(cp);
  free(im);
  free(y);
}

/* Sum of r^2 over one patch interior (residual_norm, smoother.py:96-109, as a
 * plain ordered sum per line, lines summed in order). */
double oracle_residual_sumsq(const double* u, const double* f, int nx, int ny, int nz, double cc,
                             const double* fc) {
  const size_t px = nx + 2, py = ny + 2, pxy = px * py;
  double total = 0.0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j) {
      const size_t base = IDX(1, j + 1, k + 1);
      const double* fr = f + ((size_t)k * ny + j) * nx;
      double ss = 0.0;
      for (int i = 0; i < nx; ++i) {
        const double r = resid(u, base + i, px, pxy, fr[i], cc, fc);
        ss += r * r;
      }
      total += ss;
    }
  return total;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
