// C ABI of libpsmooth: factor tables, plans, and the stream-ordered entry
// points declared in include/psmooth.h.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "psm_internal.cuh"

namespace psm {
cudaError_t launch_line_tiles(int mode, const PatchDev* patches, int npatch, const unsigned char* active,
                              const StencilDev& st, double omega, double* partials, double* rbuf, long long tile_base,
                              long long ntiles, int threads, size_t smem, cudaStream_t stream);
cudaError_t launch_line_generic(int solve, const PatchDev* patches, int npatch, const unsigned char* active,
                                const StencilDev& st, double omega, double* partials, long long tile_base,
                                long long ntiles, cudaStream_t stream);
cudaError_t launch_line_apply(const LineFac* L, const double* r, double* x, long long count, cudaStream_t stream);
cudaError_t line_tile_kernel_setup(size_t smem);
bool line_nx_specialised(int nx);
int zmarch_rows(int nx);
cudaError_t launch_line_zmarch(int nx, int unit, const PatchDev* patches, const unsigned char* active,
                               const StencilDev& st, double omega, double* partials, const void* units, int nunits,
                               int grid, const LineFac& L, cudaStream_t stream, double* rglob = nullptr,
                               int peer = 0);
int line_nx_occupancy(int nx);
bool line_zgen_supported(int nx);
cudaError_t launch_line_zgen(const int* nxs, int nnx, int unit, const PatchDev* patches, const unsigned char* active,
                             const StencilDev& st, double omega, double* partials, const void* units, int nunits,
                             int grid, const LineFac& L, cudaStream_t stream);
cudaError_t launch_line_nx(int nx, int unit, const PatchDev& P, int act, const StencilDev& st, double omega,
                           double* partials, long long t0, long long t1, int grid, const LineFac& L,
                           cudaStream_t stream);
cudaError_t launch_physical_ghosts(const PatchDev* patches, int npatch, const unsigned char* active,
                                   long long max_face, int skip_x, int use_covered, cudaStream_t stream);
cudaError_t launch_interface_copies(const PatchDev* patches, const unsigned char* active, const CopyDev* copies,
                                    int ncopy, long long total, cudaStream_t stream);
cudaError_t launch_plane_sums(const PatchDev* patches, int npatch, const double* partials, double* plane_sums,
                              int nplanes, cudaStream_t stream);
cudaError_t launch_tree_sum(const double* in, long long n, double* out, cudaStream_t stream);
cudaError_t launch_history_reduce(const PatchDev* patches, int npatch, const double* partials, long long tstride,
                                  int nplanes, int nslots, double* out, cudaStream_t stream);
cudaError_t launch_halo_unpack(double* dst_plane, const double* src_plane, int px, int py, cudaStream_t stream);
cudaError_t launch_halo_signal(int* flag_a, int* flag_b, int value, cudaStream_t s);
cudaError_t launch_halo_wait(const int* flags, int n, int value, cudaStream_t s);
cudaError_t launch_line_gs(int mode, const PatchDev* patches, int npatch, const unsigned char* active,
                           const StencilDev& st, double omega, int* flags, long long nunits,
                           const int* unit_patch, const int* unit_plane, int threads, size_t smem, int grid,
                           cudaStream_t stream);
cudaError_t line_gs_kernel_setup(size_t smem);
int gs_chunks_for(int max_nx);
size_t gs_smem_per_warp(int nc);
int gs_occupancy(int nc, int threads, size_t smem);
cudaError_t launch_line_gs_generic(const PatchDev* patches, int npatch, const unsigned char* active,
                                   const StencilDev& st, double omega, int wave, long long nlines,
                                   cudaStream_t stream);
}  // namespace psm

using namespace psm;

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) return fail(PSM_ECUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// plane path (psm_plane.cu), C++ linkage
int psm_plane_build(const psm_stencil* st, int nx, int ny, psm_factors* F);  // psm_plane.cu
int psm_plane_apply(const psm_factors* F, const double* r, double* x, long long count, cudaStream_t stream);
int psm_plane_plan_setup(psm_plan* plan);  // psm_plane.cu
int psm_plane_plan_free(psm_plan* plan);
int psm_plane_jacobi(psm_plan* P, const unsigned char* d_active, double omega, double* partials, cudaStream_t s);
int psm_plane_gs(psm_plan* P, const unsigned char* d_active, double omega, cudaStream_t s);
// box path (psm_box.cu)
int psm_box_build(const psm_stencil* st, int ex, int ey, int ez, psm_factors* F);
namespace psm {
cudaError_t launch_box_sweep(const PatchDev* patches, const unsigned char* active, const StencilDev& st,
                             double omega, const int4* blocks, int nblocks, int inplace, int mx, int my, int mz,
                             int bx, int by, int bz, cudaStream_t s, const int4* gsdep = nullptr,
                             int* flags = nullptr, int* ticket = nullptr, const void* tmaps = nullptr);
cudaError_t box_build_tmaps(const PatchDev* hp, int npatch, void** out);
cudaError_t launch_box_apply(const BoxFac* F, const double* r, double* x, long long count, cudaStream_t s);
}
extern int psm_plane_band_mode;  // psm_plane.cu
// pipelined line GS (psm_line_gs_pipe.cu)
bool gs_pipe_supported(int nx);
int psm_gs_pipe_prepare(psm_plan* P, int* n_tickets);
void psm_gs_pipe_free(psm_plan* P);
bool psm_gs_pipe_multi_ok(const psm_plan* P);
int psm_gs_pipe_multi(psm_plan* P, const unsigned char* da, double omega, int chaotic, int steps, double* hist,
                      long long hist_stride, int* flags, int* tickets, cudaStream_t s);
int psm_gs_pipe_sweep(psm_plan* P, const unsigned char* da, double omega, int chaotic, int* flags, int* tickets,
                      cudaStream_t s);

int psm_set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}

extern "C" {

const char* psm_last_error(void) { return g_err.c_str(); }
int psm_version(void) { return 10000; }

// ---------------------------------------------------------------------------
// factors
// ---------------------------------------------------------------------------
// Tridiagonal tools in long double (80-bit on x86) so the tables are
// correctly rounded to fp64 in practice.
static void thomas_ld(int n, long double c, long double lo, long double up, const long double* rhs, long double* x) {
  std::vector<long double> cp(n), d(n);
  long double prevc = 0, prevd = 0;
  for (int i = 0; i < n; ++i) {
    long double m = c - lo * prevc;
    cp[i] = up / m;
    d[i] = (rhs[i] - lo * prevd) / m;
    prevc = cp[i];
    prevd = d[i];
  }
  x[n - 1] = d[n - 1];
  for (int i = n - 2; i >= 0; --i) x[i] = d[i] - cp[i] * x[i + 1];
}

static int build_line(const psm_stencil* st, int nx, psm_factors* F) {
  const long double c = st->center, lo = st->faces[0], up = st->faces[1];
  if (fabsl(lo) + fabsl(up) > c)
    return fail(PSM_ESINGULAR,
                "line block operator is not diagonally dominant (|%g|+|%g| > %g); the device Thomas solve "
                "requires dominance",
                (double)lo, (double)up, (double)c);
  LineFac& L = F->h_line;
  memset(&L, 0, sizeof L);
  std::vector<double> cpN(nx), invmN(nx);
  long double prev = 0;
  const long double scale = c + fabsl(lo) + fabsl(up);
  for (int i = 0; i < nx; ++i) {
    long double m = c - lo * prev;
    if (fabsl(m) < 1e-14L * scale) return fail(PSM_ESINGULAR, "pivot %g at %d below 1e-14*|A|", (double)m, i);
    invmN[i] = (double)(1.0L / m);
    cpN[i] = (double)(up / m);
    prev = up / m;
  }
  prev = 0;
  for (int i = 0; i < kSeg; ++i) {
    long double m = c - lo * prev;
    L.invm[i] = (double)(1.0L / m);
    L.cp[i] = (double)(up / m);
    prev = up / m;
  }
  L.lo = (double)lo;
  L.up = (double)up;
  L.nx = nx;
  L.nseg = (nx + kSeg - 1) / kSeg;
  L.tail = nx - kSeg * (L.nseg - 1);
  long double e[kSeg], z[kSeg];
  long double g[kSeg], h[kSeg], gT[kSeg];
  for (int i = 0; i < kSeg; ++i) e[i] = 0;
  e[0] = 1;
  thomas_ld(kSeg, c, lo, up, e, g);
  e[0] = 0;
  e[kSeg - 1] = 1;
  thomas_ld(kSeg, c, lo, up, e, h);
  for (int i = 0; i < kSeg; ++i) { e[i] = 0; gT[i] = 0; }
  e[0] = 1;
  thomas_ld(L.tail, c, lo, up, e, z);
  for (int i = 0; i < L.tail; ++i) gT[i] = z[i];
  for (int i = 0; i < kSeg; ++i) {
    L.g[i] = (double)g[i];
    L.h[i] = (double)h[i];
    L.gT[i] = (double)gT[i];
  }
  L.up_h31 = (double)(up * h[kSeg - 1]);
  L.lo_g0 = (double)(lo * g[0]);
  L.lo_gT0 = (double)(lo * gT[0]);
  L.d_full = (double)(1.0L / (1.0L - up * lo * h[kSeg - 1] * g[0]));
  L.d_tail = (double)(1.0L / (1.0L - up * lo * h[kSeg - 1] * gT[0]));
  {
    long double e16[16], g16[16], h16[16];
    for (int i = 0; i < 16; ++i) e16[i] = 0;
    e16[0] = 1;
    thomas_ld(16, c, lo, up, e16, g16);
    e16[0] = 0;
    e16[15] = 1;
    thomas_ld(16, c, lo, up, e16, h16);
    for (int i = 0; i < 16; ++i) {
      L.g16[i] = (double)g16[i];
      L.h16[i] = (double)h16[i];
    }
    L.up_h16 = (double)(up * h16[15]);
    L.lo_g16 = (double)(lo * g16[0]);
    L.d16 = (double)(1.0L / (1.0L - up * lo * h16[15] * g16[0]));
  }
  // couplings dropped by the 2x2 interface systems
  const long double dropped = fabsl(lo * g[kSeg - 1]) + fabsl(up * h[0]);
  L.partitioned = (L.nseg == 1) || (dropped < 1e-18L);
  const size_t bytes = sizeof(LineFac) + 2 * (size_t)nx * sizeof(double);
  if (cudaMalloc(&F->dev, bytes) != cudaSuccess) return fail(PSM_ENOMEM, "cudaMalloc(%zu) for line factors", bytes);
  double* tab = (double*)((char*)F->dev + sizeof(LineFac));
  L.cpN = tab;
  L.invmN = tab + nx;
  F->d_line = (LineFac*)F->dev;
  CUDA_TRY(cudaMemcpy(F->dev, &L, sizeof L, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(tab, cpN.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(tab + nx, invmN.data(), nx * sizeof(double), cudaMemcpyHostToDevice));
  return PSM_OK;
}


int psm_factors_create(int kind, const psm_stencil* st, int nx, int ny, psm_factors** out) {
  if (!st || !out) return fail(PSM_EINVAL, "null argument");
  *out = nullptr;
  if (!(st->center > 0) || !isfinite(st->center)) return fail(PSM_EINVAL, "center must be positive and finite");
  for (int i = 0; i < 6; ++i)
    if (!isfinite(st->faces[i])) return fail(PSM_EINVAL, "face coefficients must be finite");
  if (nx < 1 || ny < 1) return fail(PSM_EINVAL, "block extent must be positive, got (%d,%d)", nx, ny);
  psm_factors* F = new psm_factors();
  memset(F, 0, sizeof *F);
  F->kind = kind;
  F->nx = nx;
  F->ny = ny;
  F->center = st->center;
  memcpy(F->faces, st->faces, sizeof F->faces);
  int rc;
  if (kind == PSM_BLOCK_LINE) {
    rc = build_line(st, nx, F);
  } else if (kind == PSM_BLOCK_PLANE) {
    rc = psm_plane_build(st, nx, ny, F);
  } else {
    rc = fail(PSM_EINVAL, "unknown block kind %d", kind);
  }
  if (rc != PSM_OK) {
    if (F->dev) cudaFree(F->dev);
    delete F;
    return rc;
  }
  *out = F;
  return PSM_OK;
}

int psm_factors_create_box(const psm_stencil* st, int ex, int ey, int ez, psm_factors** out) {
  if (!st || !out) return fail(PSM_EINVAL, "null argument");
  *out = nullptr;
  if (!(st->center > 0) || !isfinite(st->center)) return fail(PSM_EINVAL, "center must be positive and finite");
  for (int i = 0; i < 6; ++i)
    if (!isfinite(st->faces[i])) return fail(PSM_EINVAL, "face coefficients must be finite");
  if (ex < 1 || ey < 1 || ez < 1) return fail(PSM_EINVAL, "block extent must be positive, got (%d,%d,%d)", ex, ey, ez);
  psm_factors* F = new psm_factors();
  memset(F, 0, sizeof *F);
  F->kind = PSM_BLOCK_BOX;
  F->nx = ex;
  F->ny = ey;
  F->nz = ez;
  F->center = st->center;
  memcpy(F->faces, st->faces, sizeof F->faces);
  const int rc = psm_box_build(st, ex, ey, ez, F);
  if (rc != PSM_OK) {
    if (F->dev) cudaFree(F->dev);
    delete F;
    return rc;
  }
  *out = F;
  return PSM_OK;
}

int psm_factors_destroy(psm_factors* F) {
  if (!F) return PSM_OK;
  if (F->dev) cudaFree(F->dev);
  delete F;
  return PSM_OK;
}


int psm_factors_apply(const psm_factors* F, const double* r, double* x, long long count, void* stream) {
  if (!F || !r || !x || count < 0) return fail(PSM_EINVAL, "bad arguments to psm_factors_apply");
  if (F->kind == PSM_BLOCK_LINE) {
    CUDA_TRY(launch_line_apply(F->d_line, r, x, count, (cudaStream_t)stream));
    return PSM_OK;
  }
  if (F->kind == PSM_BLOCK_BOX) {
    CUDA_TRY(launch_box_apply(F->d_box, r, x, count, (cudaStream_t)stream));
    return PSM_OK;
  }
  return psm_plane_apply(F, r, x, count, (cudaStream_t)stream);
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------

int psm_plan_create(const psm_patch_desc* patches, int npatch, const psm_copy_desc* copies, int ncopy,
                    const psm_stencil* st, int kind, psm_factors* const* fac, psm_plan** out) {
  if (!out) return fail(PSM_EINVAL, "null out");
  *out = nullptr;
  if (!patches || npatch < 1) return fail(PSM_EINVAL, "a plan needs at least one patch");
  if (ncopy < 0 || (ncopy > 0 && !copies)) return fail(PSM_EINVAL, "bad interface copy list");
  if (!st) return fail(PSM_EINVAL, "null stencil");
  if (kind != 0 && kind != PSM_BLOCK_LINE && kind != PSM_BLOCK_PLANE && kind != PSM_BLOCK_BOX)
    return fail(PSM_EINVAL, "bad kind %d", kind);
  psm_plan* P = new psm_plan();
  P->npatch = npatch;
  P->ncopy = ncopy;
  P->kind = kind;
  P->st = StencilDev{st->center, st->faces[0], st->faces[1], st->faces[2], st->faces[3], st->faces[4], st->faces[5]};
  P->hp.resize(npatch);
  P->fac.assign(npatch, nullptr);
  int max_nx = 0;
  for (int p = 0; p < npatch; ++p) {
    const psm_patch_desc& d = patches[p];
    if (d.nx < 1 || d.ny < 1 || d.nz < 1) { delete P; return fail(PSM_EINVAL, "patch %d has bad dims", p); }
    if (!d.buf[0] || !d.buf[1] || !d.f) { delete P; return fail(PSM_EINVAL, "patch %d has null buffers", p); }
    max_nx = std::max(max_nx, d.nx);
    if (kind != 0) {
      psm_factors* F = fac ? fac[p] : nullptr;
      if (!F || F->kind != kind) { delete P; return fail(PSM_EINVAL, "patch %d lacks matching factors", p); }
      if ((kind != PSM_BLOCK_BOX && F->nx != d.nx) || (kind == PSM_BLOCK_PLANE && F->ny != d.ny) ||
          (kind == PSM_BLOCK_BOX && (F->nx > d.nx || F->ny > d.ny || F->nz > d.nz))) {
        delete P;
        return fail(PSM_EINVAL, "patch %d factors are for another block shape", p);
      }
      if (F->center != st->center || memcmp(F->faces, st->faces, sizeof F->faces) != 0) {
        delete P;
        return fail(PSM_EINVAL, "patch %d factors were built for another stencil", p);
      }
      P->fac[p] = F;
      if (kind == PSM_BLOCK_LINE && !F->h_line.partitioned) P->tiled = 0;
    }
  }
  if (max_nx > 2048) P->tiled = 0;
  P->threads = 256;
  long long tile0 = 0, cell0 = 0;
  int plane0 = 0;
  long long g0 = 0;
  size_t smem = 0;
  std::vector<long long> gpre(npatch);
  for (int p = 0; p < npatch; ++p) {
    const psm_patch_desc& d = patches[p];
    PatchDev& h = P->hp[p];
    h.buf[0] = d.buf[0];
    h.buf[1] = d.buf[1];
    h.f = d.f;
    h.nx = d.nx;
    h.ny = d.ny;
    h.nz = d.nz;
    h.R = P->tiled ? std::max(1, kMaxTileCells / d.nx) : 1;
    h.tpp = (d.ny + h.R - 1) / h.R;
    h.tiles = h.tpp * d.nz;
    h.tile0 = tile0;
    h.plane0 = plane0;
    h.lf = (kind == PSM_BLOCK_LINE) ? P->fac[p]->d_line : nullptr;
    h.pf = (kind == PSM_BLOCK_PLANE) ? P->fac[p]->d_plane : nullptr;
    h.bf = (kind == PSM_BLOCK_BOX) ? P->fac[p]->d_box : nullptr;
    h.cell0 = cell0;
    cell0 += (long long)d.nx * d.ny * d.nz;
    tile0 += h.tiles;
    plane0 += d.nz;
    gpre[p] = g0;
    const long long px = d.nx + 2, py = d.ny + 2, pz = d.nz + 2;
    g0 += 2 * (py * pz + px * pz + px * py);
    P->ghost_max_face = std::max(P->ghost_max_face, std::max(py * pz, std::max(px * pz, px * py)));
    const int nseg = (d.nx + kSeg - 1) / kSeg;
    smem = std::max(smem, (size_t)(h.R * row_stride(d.nx) + 2 * h.R * nseg) * sizeof(double));
  }
  P->ntiles = tile0;
  P->nplanes = plane0;
  P->ghost_total = g0;
  P->smem = smem;
  std::vector<CopyDev> hc(ncopy);
  long long e0 = 0;
  for (int i = 0; i < ncopy; ++i) {
    const psm_copy_desc& c = copies[i];
    if (c.src < 0 || c.src >= npatch || c.dst < 0 || c.dst >= npatch || c.src == c.dst) {
      delete P;
      return fail(PSM_EINVAL, "copy %d references bad patches", i);
    }
    const int sd[3] = {patches[c.src].nx, patches[c.src].ny, patches[c.src].nz};
    const int dd[3] = {patches[c.dst].nx, patches[c.dst].ny, patches[c.dst].nz};
    for (int a = 0; a < 3; ++a) {
      if (c.extent[a] < 1 || c.src_lo[a] < 0 || c.src_lo[a] + c.extent[a] > sd[a] || c.dst_lo[a] < -1 ||
          c.dst_lo[a] + c.extent[a] > dd[a] + 1) {
        delete P;
        return fail(PSM_EINVAL, "copy %d leaves its patches", i);
      }
    }
    CopyDev& h = hc[i];
    h.src = c.src;
    h.dst = c.dst;
    for (int a = 0; a < 3; ++a) {
      h.src_lo[a] = c.src_lo[a];
      h.dst_lo[a] = c.dst_lo[a];
      h.ext[a] = c.extent[a];
    }
    h.elem0 = e0;
    e0 += (long long)c.extent[0] * c.extent[1] * c.extent[2];
    P->copy_max = std::max(P->copy_max, (long long)c.extent[0] * c.extent[1] * c.extent[2]);
  }
  P->copy_total = e0;
  // faces one copy covers entirely: the physical fill skips their interior
  for (int i = 0; i < ncopy; ++i) {
    const psm_copy_desc& c = copies[i];
    const int dd[3] = {patches[c.dst].nx, patches[c.dst].ny, patches[c.dst].nz};
    for (int a = 0; a < 3; ++a) {
      if (c.extent[a] != 1 || (c.dst_lo[a] != -1 && c.dst_lo[a] != dd[a])) continue;
      const int b1 = (a + 1) % 3, b2 = (a + 2) % 3;
      if (c.dst_lo[b1] == 0 && c.extent[b1] == dd[b1] && c.dst_lo[b2] == 0 && c.extent[b2] == dd[b2])
        P->hp[c.dst].covered |= 1 << (2 * a + (c.dst_lo[a] == -1 ? 0 : 1));
    }
  }
  cudaError_t err = cudaMalloc(&P->d_patches, npatch * sizeof(PatchDev));
  if (err == cudaSuccess) err = cudaMemcpy(P->d_patches, P->hp.data(), npatch * sizeof(PatchDev), cudaMemcpyHostToDevice);
  if (err == cudaSuccess) err = cudaMalloc(&P->d_gprefix, npatch * sizeof(long long));
  if (err == cudaSuccess) err = cudaMemcpy(P->d_gprefix, gpre.data(), npatch * sizeof(long long), cudaMemcpyHostToDevice);
  if (err == cudaSuccess && ncopy > 0) {
    err = cudaMalloc(&P->d_copies, ncopy * sizeof(CopyDev));
    if (err == cudaSuccess) err = cudaMemcpy(P->d_copies, hc.data(), ncopy * sizeof(CopyDev), cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess) err = cudaMalloc(&P->d_scratch, std::max<long long>(1, P->ntiles) * sizeof(double));
  if (err == cudaSuccess && kind == PSM_BLOCK_LINE && P->tiled) err = line_tile_kernel_setup(P->smem);
  if (err != cudaSuccess) {
    psm_plan_destroy(P);
    return fail(PSM_ECUDA, "plan setup: %s", cudaGetErrorString(err));
  }
  if (kind == PSM_BLOCK_BOX) {  // block list, wavefront-major (bi + bj + bk), then patch, then lexicographic
    // with each block's GS dependencies: its flag index (patch-major
    // lexicographic numbering) and those of its -x, -y, -z neighbour blocks
    std::vector<std::vector<int>> waves, wdeps;
    int fbase = 0;
    for (int p = 0; p < npatch; ++p) {
      const psm_factors* F = P->fac[p];
      const PatchDev& h = P->hp[p];
      const int cx = (h.nx + F->nx - 1) / F->nx, cy = (h.ny + F->ny - 1) / F->ny, cz = (h.nz + F->nz - 1) / F->nz;
      for (int bk = 0; bk < cz; ++bk)
        for (int bj = 0; bj < cy; ++bj)
          for (int bi = 0; bi < cx; ++bi) {
            const int w = bi + bj + bk;
            if ((int)waves.size() <= w) {
              waves.resize(w + 1);
              wdeps.resize(w + 1);
            }
            waves[w].insert(waves[w].end(), {p, bi * F->nx, bj * F->ny, bk * F->nz});
            const int id = fbase + bi + cx * (bj + cy * bk);
            wdeps[w].insert(wdeps[w].end(), {id, bi > 0 ? id - 1 : -1, bj > 0 ? id - cx : -1, bk > 0 ? id - cx * cy : -1});
          }
      fbase += cx * cy * cz;
    }
    std::vector<int> all, deps;
    P->box_wave_off.assign(1, 0);
    for (size_t w = 0; w < waves.size(); ++w) {
      all.insert(all.end(), waves[w].begin(), waves[w].end());
      deps.insert(deps.end(), wdeps[w].begin(), wdeps[w].end());
      P->box_wave_off.push_back((int)(all.size() / 4));
    }
    P->nboxes = (int)(all.size() / 4);
    // Jacobi regions: (8/b) blocks per axis (all patches share block dims up
    // to truncation: use the first patch's; truncated patches just clip)
    const psm_factors* F0 = P->fac[0];
    bool same = true;
    for (int p = 1; p < npatch; ++p) same = same && P->fac[p]->nx == F0->nx && P->fac[p]->ny == F0->ny &&
                                               P->fac[p]->nz == F0->nz;
    P->box_dims[0] = same ? F0->nx : 0;
    P->box_dims[1] = same ? F0->ny : 0;
    P->box_dims[2] = same ? F0->nz : 0;
    P->reg_m[0] = same ? std::max(1, 8 / F0->nx) : 1;
    P->reg_m[1] = same ? std::max(1, 8 / F0->ny) : 1;
    P->reg_m[2] = same ? std::max(1, 8 / F0->nz) : 1;
    std::vector<int> regs;
    for (int p = 0; p < npatch; ++p) {
      const psm_factors* F = P->fac[p];
      const PatchDev& h = P->hp[p];
      const int Rx = F->nx * P->reg_m[0], Ry = F->ny * P->reg_m[1], Rz = F->nz * P->reg_m[2];
      for (int z = 0; z < h.nz; z += Rz)
        for (int y = 0; y < h.ny; y += Ry)
          for (int x = 0; x < h.nx; x += Rx) regs.insert(regs.end(), {p, x, y, z});
    }
    P->nregions = (int)(regs.size() / 4);
    cudaError_t e = cudaMalloc(&P->d_boxes, std::max<size_t>(16, all.size() * sizeof(int)));
    if (e == cudaSuccess) e = cudaMemcpy(P->d_boxes, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_box_deps, std::max<size_t>(16, deps.size() * sizeof(int)));
    if (e == cudaSuccess) e = cudaMemcpy(P->d_box_deps, deps.data(), deps.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_box_flags, (size_t)(P->nboxes + 1) * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_box_regions, std::max<size_t>(16, regs.size() * sizeof(int)));
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_box_regions, regs.data(), regs.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = box_build_tmaps(P->hp.data(), npatch, &P->d_box_tmaps);
    if (e != cudaSuccess) {
      psm_plan_destroy(P);
      return fail(PSM_ECUDA, "box block list: %s", cudaGetErrorString(e));
    }
  }
  if (kind == PSM_BLOCK_PLANE) {
    int rc = psm_plane_plan_setup(P);
    if (rc != PSM_OK) {
      psm_plan_destroy(P);
      return rc;
    }
  }
  *out = P;
  return PSM_OK;
}

int psm_plan_destroy(psm_plan* P) {
  if (!P) return PSM_OK;
  cudaFree(P->d_patches);
  cudaFree(P->d_copies);
  cudaFree(P->d_gprefix);
  cudaFree(P->d_partials);
  cudaFree(P->d_plane_sums);
  cudaFree(P->d_sums);
  cudaFree(P->d_scratch);
  cudaFree(P->d_flags);
  cudaFree(P->d_unit_patch);
  cudaFree(P->d_unit_plane);
  cudaFree(P->d_gsflags);
  cudaFree(P->d_msflags);
  cudaFree(P->d_boxes);
  cudaFree(P->d_box_regions);
  cudaFree(P->d_box_deps);
  cudaFree(P->d_box_flags);
  cudaFree(P->d_box_tmaps);
  psm_gs_pipe_free(P);
  for (auto& kv : P->unit_cache) cudaFree(kv.second.first);
  for (auto& kv : P->active_cache) cudaFree(kv.second);
  if (P->kind == PSM_BLOCK_PLANE) psm_plane_plan_free(P);
  for (auto& kv : P->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  if (P->cap_stream) cudaStreamDestroy(P->cap_stream);
  for (int i = 0; i < psm_plan::kSide; ++i) {
    if (P->side[i]) cudaStreamDestroy(P->side[i]);
    if (P->side_join[i]) cudaEventDestroy(P->side_join[i]);
  }
  if (P->side_fork) cudaEventDestroy(P->side_fork);
  delete P;
  return PSM_OK;
}

int psm_plan_reserve_history(psm_plan* P, int slots) {
  if (!P || slots < 0) return fail(PSM_EINVAL, "bad arguments");
  if (slots <= P->cap_slots) return PSM_OK;
  int cap = std::max(slots, 2 * P->cap_slots);
  double *np = nullptr, *ns = nullptr, *nt = nullptr;
  const size_t tb = (size_t)std::max<long long>(1, P->ntiles) * sizeof(double);
  const size_t pb = (size_t)std::max(1, P->nplanes) * sizeof(double);
  if (cudaMalloc(&np, cap * tb) != cudaSuccess || cudaMalloc(&ns, cap * pb) != cudaSuccess ||
      cudaMalloc(&nt, cap * sizeof(double)) != cudaSuccess) {
    cudaFree(np);
    cudaFree(ns);
    cudaFree(nt);
    return fail(PSM_ENOMEM, "history workspace for %d slots", cap);
  }
  if (P->cap_slots > 0) {
    CUDA_TRY(cudaMemcpy(np, P->d_partials, P->cap_slots * tb, cudaMemcpyDeviceToDevice));
  }
  cudaFree(P->d_partials);
  cudaFree(P->d_plane_sums);
  cudaFree(P->d_sums);
  // captured graphs hold the old history pointers: drop them (re-captured)
  for (auto& kv : P->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  P->graphs.clear();
  P->d_partials = np;
  P->d_plane_sums = ns;
  P->d_sums = nt;
  P->cap_slots = cap;
  return PSM_OK;
}

static int get_active(psm_plan* P, const unsigned char* active, unsigned char** out) {
  if (!active) return fail(PSM_EINVAL, "null active vector");
  std::string key((const char*)active, P->npatch);
  for (char ch : key)
    if (ch != 0 && ch != 1) return fail(PSM_EINVAL, "active flags must be 0 or 1");
  auto it = P->active_cache.find(key);
  if (it != P->active_cache.end()) {
    *out = it->second;
    return PSM_OK;
  }
  unsigned char* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, P->npatch));
  CUDA_TRY(cudaMemcpy(d, active, P->npatch, cudaMemcpyHostToDevice));
  P->active_cache[key] = d;
  *out = d;
  return PSM_OK;
}

static double* slot_ptr(psm_plan* P, int slot, int* rc) {
  *rc = PSM_OK;
  if (slot < 0) return P->d_scratch;
  if (slot >= P->cap_slots) {
    *rc = fail(PSM_EINVAL, "history slot %d beyond reserved %d", slot, P->cap_slots);
    return nullptr;
  }
  return P->d_partials + (size_t)slot * std::max<long long>(1, P->ntiles);
}

int psm_refresh_ghosts(psm_plan* P, const unsigned char* active, int what, void* stream) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  if (what < 0 || what > 7) return fail(PSM_EINVAL, "bad ghost selection %d", what);
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  // after a sweep (SKIP_X) only what its epilogue left: nothing, the y/z
  // faces plus the x-face perimeters, or everything
  const int level = (what & PSM_GHOST_SKIP_X) ? P->phys_pending : 2;
  if (what & PSM_GHOST_PHYSICAL) {
    if (level > 0) {
      CUDA_TRY(launch_physical_ghosts(P->d_patches, P->npatch, da, P->ghost_max_face, level == 1 ? 1 : 0,
                                      (what & PSM_GHOST_INTERFACE) ? 1 : 0, s));
      P->launches += P->ghost_total > 0;
    }
    P->phys_pending = 0;
  }
  if (what & PSM_GHOST_INTERFACE) {
    CUDA_TRY(launch_interface_copies(P->d_patches, da, P->d_copies, P->ncopy, P->copy_max, s));
    P->launches += (P->ncopy > 0 && P->copy_total > 0);
  }
  return PSM_OK;
}

int psm_residual(psm_plan* P, const unsigned char* active, int slot, void* stream) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  double* part = slot_ptr(P, slot, &rc);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (P->tiled) {
    CUDA_TRY(launch_line_tiles(0, P->d_patches, P->npatch, da, P->st, 0.0, part, nullptr, 0, P->ntiles, P->threads, 0, s));
  } else {
    CUDA_TRY(launch_line_generic(0, P->d_patches, P->npatch, da, P->st, 0.0, part, 0, P->ntiles, s));
  }
  P->launches += 1;
  return PSM_OK;
}


// z-marching work units (patch, j0, k0, k1) for planes [ka, kb) of patches
// [p0, p1) -- patch-major, then plane chunk, then column, so concurrently
// running CTAs march neighbouring columns through the same planes.  Cached.
static int zmarch_units(psm_plan* P, int p0, int p1, int ka, int kb, void** d_units, int* nunits) {
  const std::string key = std::to_string(p0) + ":" + std::to_string(p1) + ":" + std::to_string(ka) + ":" +
                          std::to_string(kb);
  auto it = P->unit_cache.find(key);
  if (it != P->unit_cache.end()) {
    *d_units = it->second.first;
    *nunits = it->second.second;
    return PSM_OK;
  }
  long long cols = 0;
  for (int p = p0; p < p1; ++p) cols += P->hp[p].tpp;
  long long planes = 1;  // the deepest patch's plane range
  for (int p = p0; p < p1; ++p) planes = std::max<long long>(planes, (kb < 0 ? P->hp[p].nz : kb) - ka);
  // plane-chunk length: minimise the busiest persistent CTA's work,
  // ceil(units / SMs) * (chunk + ~2 planes of halo and pipeline fill)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int kc = (int)planes;
  double best = 1e300;
  for (long long nch = 1; nch <= std::min<long long>(planes, 256); ++nch) {
    const long long len = (planes + nch - 1) / nch;
    if (len < 4 && nch > 1) break;
    const double cost = (double)((cols * nch + sms - 1) / sms) * (double)(len + 2);
    if (cost < best - 1e-9) {
      best = cost;
      kc = (int)len;
    }
  }
  std::vector<int> u;
  for (int p = p0; p < p1; ++p) {
    const PatchDev& h = P->hp[p];
    const int a = ka, b = (kb < 0) ? h.nz : kb;
    for (int k0 = a; k0 < b; k0 += kc)
      for (int c = 0; c < h.tpp; ++c) {
        u.push_back(p);
        u.push_back(c * h.R);
        u.push_back(k0);
        u.push_back(std::min(b, k0 + kc));
      }
  }
  void* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, std::max<size_t>(16, u.size() * sizeof(int))));
  CUDA_TRY(cudaMemcpy(d, u.data(), u.size() * sizeof(int), cudaMemcpyHostToDevice));
  P->unit_cache[key] = {d, (int)(u.size() / 4)};
  *d_units = d;
  *nunits = (int)(u.size() / 4);
  return PSM_OK;
}

// 16-byte aligned buffers of every patch in [p, q) (the bulk copies' rule)
static bool group_aligned(const psm_plan* P, int p, int q) {
  for (int r = p; r < q; ++r) {
    const PatchDev& h = P->hp[r];
    if (((uintptr_t)h.buf[0] | (uintptr_t)h.buf[1] | (uintptr_t)h.f) & 15) return false;
  }
  return true;
}

// patch p can take the runtime-nx z-marching kernel
static bool zgen_ok(const psm_plan* P, int p) {
  const PatchDev& h = P->hp[p];
  return P->tiled && !line_nx_specialised(h.nx) && line_zgen_supported(h.nx) && group_aligned(P, p, p + 1);
}

// cells of planes [ka, kb) over the run of zgen-eligible patches from p (end -> *q)
static long long zgen_cells(const psm_plan* P, int p, int pb, int ka, int kb, int* q) {
  long long cells = 0;
  int r = p;
  for (; r < pb && zgen_ok(P, r); ++r)
    cells += (long long)P->hp[r].nx * P->hp[r].ny * ((kb < 0 ? P->hp[r].nz : kb) - ka);
  *q = r;
  return cells;
}

// Line-Jacobi sweep of planes [ka, kb) (kb < 0: all planes) of patches
// [pa, pb): consecutive patches sharing a specialised nx run the z-marching
// TMA kernel (one launch per group), the rest the generic tile kernel.
// groups below this many cells take the one-tile-per-CTA specialised line
// kernel instead of the z-marching pipeline
static long long zmarch_min_cells() {
  static const long long zmin = [] {
    const char* e = getenv("PSM_ZMARCH_MIN_CELLS");
    return e ? atoll(e) : (1LL << 21);
  }();
  return zmin;
}

// da: the device copy of the active flags, ha: the host one
static int sweep_planes(psm_plan* P, const unsigned char* da, const unsigned char* ha, double omega, double* part,
                        int pa, int pb, int ka, int kb, cudaStream_t s) {
  const bool unit = P->st.xm == -1.0 && P->st.xp == -1.0 && P->st.ym == -1.0 && P->st.yp == -1.0 &&
                    P->st.zm == -1.0 && P->st.zp == -1.0;
  int p = pa;
  while (p < pb) {
    const int nx = P->hp[p].nx;
    int q = p + 1;
    while (q < pb && P->hp[q].nx == nx) ++q;
    long long gcells = 0;  // cells of this group's plane range
    for (int r = p; r < q; ++r)
      gcells += (long long)P->hp[r].nx * P->hp[r].ny * ((kb < 0 ? P->hp[r].nz : kb) - ka);
    const long long zmin = zmarch_min_cells();
    bool peers = false;  // the fused halo lives in the z-marching kernel only
    for (int r = p; r < q; ++r) peers |= P->hp[r].iface != 0;
    if (P->tiled && line_nx_specialised(nx) && gcells < zmin && !peers) {
      // small groups: the one-tile-per-CTA specialised kernel (no TMA ring to
      // fill, no persistent pipeline to drain) is latency-cheaper
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      for (int r = p; r < q; ++r) {
        const PatchDev& h = P->hp[r];
        const int a = ka, b = (kb < 0) ? h.nz : kb;
        const long long t0 = h.tile0 + (long long)a * h.tpp, t1 = h.tile0 + (long long)b * h.tpp;
        CUDA_TRY(launch_line_nx(nx, unit ? 1 : 0, h, ha[r], P->st, omega, part, t0, t1, line_nx_occupancy(nx) * sms,
                                P->fac[r]->h_line, s));
        P->launches += 1;
      }
    } else if (P->tiled && line_nx_specialised(nx) && P->hp[p].R == zmarch_rows(nx)) {
      void* units;
      int nu;
      int rc = zmarch_units(P, p, q, ka, kb, &units, &nu);
      if (rc) return rc;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      CUDA_TRY(launch_line_zmarch(nx, unit ? 1 : 0, P->d_patches, da, P->st, omega, part, units, nu, sms,
                                   P->fac[p]->h_line, s, nullptr, peers ? 1 : 0));
      P->phys_pending = std::max(P->phys_pending, 1);  // y/z ghosts left to the refresh
      P->launches += 1;
    } else if (zgen_ok(P, p) && zgen_cells(P, p, pb, ka, kb, &q) >= zmin) {
      // other even nx: the z-marching pipeline with the line length per unit,
      // one launch over consecutive such patches whatever their nx
      void* units;
      int nu;
      int rc = zmarch_units(P, p, q, ka, kb, &units, &nu);
      if (rc) return rc;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      std::vector<int> nxs;
      for (int r = p; r < q; ++r) nxs.push_back(P->hp[r].nx);
      CUDA_TRY(launch_line_zgen(nxs.data(), (int)nxs.size(), unit ? 1 : 0, P->d_patches, da, P->st, omega, part,
                                units, nu, sms, P->fac[p]->h_line, s));
      P->phys_pending = std::max(P->phys_pending, 1);
      P->launches += 1;
    } else if (ka == 0 && kb < 0) {
      // whole-patch sweeps of consecutive patches the specialised kernels do
      // not cover (any nx) are one launch over their contiguous tile range
      while (q < pb && !(P->tiled && line_nx_specialised(P->hp[q].nx))) ++q;
      const long long t0 = P->hp[p].tile0, nt = P->hp[q - 1].tile0 + P->hp[q - 1].tiles - t0;
      if (P->tiled) {
        CUDA_TRY(launch_line_tiles(1, P->d_patches, P->npatch, da, P->st, omega, part, nullptr, t0, nt, P->threads,
                                   P->smem, s));
      } else {
        CUDA_TRY(launch_line_generic(1, P->d_patches, P->npatch, da, P->st, omega, part, t0, nt, s));
      }
      P->launches += 1;
    } else {
      for (int r = p; r < q; ++r) {
        const PatchDev& h = P->hp[r];
        const int a = ka, b = (kb < 0) ? h.nz : kb;
        const long long t0 = h.tile0 + (long long)a * h.tpp, nt = (long long)(b - a) * h.tpp;
        if (P->tiled) {
          CUDA_TRY(launch_line_tiles(1, P->d_patches, P->npatch, da, P->st, omega, part, nullptr, t0, nt, P->threads,
                                     P->smem, s));
        } else {
          CUDA_TRY(launch_line_generic(1, P->d_patches, P->npatch, da, P->st, omega, part, t0, nt, s));
        }
        P->launches += 1;
      }
    }
    p = q;
  }
  return PSM_OK;
}

// Residual r = f - A u of every cell into rbuf (cell-major, per patch at
// cell0) plus the history partials, for the plane path: the z-marching TMA
// kernel in residual-only mode where nx is specialised, else the tile kernel.
int psm_plane_residual(psm_plan* P, const unsigned char* da, double* partials, double* rbuf, cudaStream_t s) {
  const bool unit = P->st.xm == -1.0 && P->st.xp == -1.0 && P->st.ym == -1.0 && P->st.yp == -1.0 &&
                    P->st.zm == -1.0 && P->st.zp == -1.0;
  int p = 0;
  while (p < P->npatch) {
    const int nx = P->hp[p].nx;
    int q = p + 1;
    while (q < P->npatch && P->hp[q].nx == nx) ++q;
    if (P->tiled && line_nx_specialised(nx) && P->hp[p].R == zmarch_rows(nx)) {
      void* units;
      int nu;
      int rc = zmarch_units(P, p, q, 0, -1, &units, &nu);
      if (rc) return rc;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      LineFac dummy;
      memset(&dummy, 0, sizeof dummy);
      CUDA_TRY(launch_line_zmarch(nx, unit ? 1 : 0, P->d_patches, da, P->st, 0.0, partials, units, nu, sms, dummy, s,
                                  rbuf));
      P->launches += 1;
    } else {
      // consecutive patches without the z-marching kernel: one launch over
      // their contiguous tile range
      while (q < P->npatch &&
             !(P->tiled && line_nx_specialised(P->hp[q].nx) && P->hp[q].R == zmarch_rows(P->hp[q].nx)))
        ++q;
      const long long t0 = P->hp[p].tile0, nt = P->hp[q - 1].tile0 + P->hp[q - 1].tiles - t0;
      CUDA_TRY(launch_line_tiles(2, P->d_patches, P->npatch, da, P->st, 0.0, partials, rbuf, t0, nt, P->threads, 0,
                                 s));
      P->launches += 1;
    }
    p = q;
  }
  return PSM_OK;
}

int psm_jacobi_sweep(psm_plan* P, const unsigned char* active, double omega, int slot, void* stream) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  if (!(omega > 0.0 && omega <= 1.0)) return fail(PSM_EINVAL, "omega must lie in (0, 1], got %g", omega);
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  double* part = slot_ptr(P, slot, &rc);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (P->kind == PSM_BLOCK_LINE) return sweep_planes(P, da, active, omega, part, 0, P->npatch, 0, -1, s);
  if (P->kind != 0) P->phys_pending = std::max(P->phys_pending, 1);  // plane/box sweeps write x faces only
  if (P->kind == PSM_BLOCK_PLANE) return psm_plane_jacobi(P, da, omega, part, s);
  if (P->kind == PSM_BLOCK_BOX) {
    if (slot >= 0) {  // history entry of the current iterate (tile partials)
      if (P->tiled) {
        CUDA_TRY(launch_line_tiles(0, P->d_patches, P->npatch, da, P->st, 0.0, part, nullptr, 0, P->ntiles,
                                   P->threads, 0, s));
      } else {
        CUDA_TRY(launch_line_generic(0, P->d_patches, P->npatch, da, P->st, 0.0, part, 0, P->ntiles, s));
      }
      P->launches += 1;
    }
    CUDA_TRY(launch_box_sweep(P->d_patches, da, P->st, omega, P->d_box_regions, P->nregions, 0, P->reg_m[0],
                              P->reg_m[1], P->reg_m[2], P->box_dims[0], P->box_dims[1], P->box_dims[2], s, nullptr,
                              nullptr, nullptr, P->d_box_tmaps));
    P->launches += 1;
    return PSM_OK;
  }
  return fail(PSM_EINVAL, "plan was created without a block kind (ghost-only)");
}

int psm_jacobi_sweep_planes(psm_plan* P, const unsigned char* active, double omega, int slot, int patch, int k0,
                            int k1, void* stream) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  if (P->kind != PSM_BLOCK_LINE) return fail(PSM_EUNSUPPORTED, "plane-range sweeps are implemented for line plans");
  if (!(omega > 0.0 && omega <= 1.0)) return fail(PSM_EINVAL, "omega must lie in (0, 1], got %g", omega);
  if (patch < 0 || patch >= P->npatch) return fail(PSM_EINVAL, "bad patch %d", patch);
  const PatchDev& h = P->hp[patch];
  if (k0 < 0 || k1 > h.nz || k0 > k1) return fail(PSM_EINVAL, "bad plane range [%d,%d) for nz=%d", k0, k1, h.nz);
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  double* part = slot_ptr(P, slot, &rc);
  if (rc) return rc;
  if (k1 == k0) return PSM_OK;
  return sweep_planes(P, da, active, omega, part, patch, patch + 1, k0, k1, (cudaStream_t)stream);
}

int psm_halo_unpack(psm_plan* P, const unsigned char* active, int patch, int side, const double* plane_dev,
                    void* stream) {
  if (!P || !active || !plane_dev) return fail(PSM_EINVAL, "bad arguments");
  if (patch < 0 || patch >= P->npatch || (side != 0 && side != 1)) return fail(PSM_EINVAL, "bad patch/side");
  const PatchDev& h = P->hp[patch];
  const int a = active[patch];
  if (a != 0 && a != 1) return fail(PSM_EINVAL, "active flags must be 0 or 1");
  const long long px = h.nx + 2, py = h.ny + 2, pz = h.nz + 2;
  double* dst = h.buf[a] + (side ? (pz - 1) : 0) * px * py;
  CUDA_TRY(launch_halo_unpack(dst, plane_dev, (int)px, (int)py, (cudaStream_t)stream));
  P->launches += 1;
  return PSM_OK;
}

// Side streams of a plan: psm_side_fork makes n (<= kSide) side streams wait
// for everything queued on s so far; psm_side_join makes s wait for them.
// Both are legal inside a stream capture (parallel graph branches).
cudaError_t psm_side_fork(psm_plan* P, cudaStream_t s, int n) {
  if (!P->side_fork) {
    // create every stream and event first and publish side_fork last, so a
    // failure part way leaves nothing half-initialised for the next call
    cudaStream_t st[psm_plan::kSide] = {};
    cudaEvent_t ev[psm_plan::kSide] = {};
    cudaEvent_t fork = nullptr;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < psm_plan::kSide && e == cudaSuccess; ++i) {
      e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      for (int i = 0; i < psm_plan::kSide; ++i) {
        if (st[i]) cudaStreamDestroy(st[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
      }
      return e;
    }
    for (int i = 0; i < psm_plan::kSide; ++i) {
      P->side[i] = st[i];
      P->side_join[i] = ev[i];
    }
    P->side_fork = fork;
  }
  cudaError_t e = cudaEventRecord(P->side_fork, s);
  for (int i = 0; i < std::min(n, (int)psm_plan::kSide) && e == cudaSuccess; ++i)
    e = cudaStreamWaitEvent(P->side[i], P->side_fork, 0);
  return e;
}

cudaError_t psm_side_join(psm_plan* P, cudaStream_t s, int n) {
  cudaError_t e = cudaSuccess;
  for (int i = 0; i < std::min(n, (int)psm_plan::kSide) && e == cudaSuccess; ++i) {
    e = cudaEventRecord(P->side_join[i], P->side[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, P->side_join[i], 0);
  }
  return e;
}

// ---------------------------------------------------------------------------
// fused multi-GPU halo over peer memory (z-slabs)
// ---------------------------------------------------------------------------
typedef int (*MemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);

int psm_ipc_get_handle(const void* ptr, void* handle_out, long long* offset_out) {
  if (!ptr || !handle_out || !offset_out) return fail(PSM_EINVAL, "bad arguments");
  // the handle names the whole allocation (torch carves tensors out of
  // larger segments): report the pointer's offset from the allocation base
  static MemGetAddressRange_t range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (MemGetAddressRange_t)fn;
  }();
  if (!range) return fail(PSM_EUNSUPPORTED, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)ptr) != 0) return fail(PSM_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, (void*)base));
  memcpy(handle_out, &h, sizeof h);
  *offset_out = (long long)((unsigned long long)ptr - base);
  return PSM_OK;
}

static std::map<std::string, void*>& ipc_maps() {
  static std::map<std::string, void*> m;
  return m;
}

int psm_ipc_open_handle(const void* handle, long long offset, void** ptr_out) {
  if (!handle || !ptr_out || offset < 0) return fail(PSM_EINVAL, "bad arguments");
  std::string key((const char*)handle, sizeof(cudaIpcMemHandle_t));
  auto& m = ipc_maps();
  auto it = m.find(key);
  void* base = nullptr;
  if (it != m.end()) {
    base = it->second;
  } else {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    m[key] = base;
  }
  *ptr_out = (char*)base + offset;
  return PSM_OK;
}

int psm_device_pci_bus_id(char* out, int len) {
  if (!out || len < 16) return fail(PSM_EINVAL, "bad arguments");
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetPCIBusId(out, len, dev));
  return PSM_OK;
}

int psm_peer_access(const char* pci_bus_id, int* ok_out) {
  if (!pci_bus_id || !ok_out) return fail(PSM_EINVAL, "bad arguments");
  *ok_out = 0;
  int me = 0, peer = -1;
  CUDA_TRY(cudaGetDevice(&me));
  if (cudaDeviceGetByPCIBusId(&peer, pci_bus_id) != cudaSuccess) {
    cudaGetLastError();  // not visible here: no peer mapping possible
    return PSM_OK;
  }
  if (peer == me) {
    *ok_out = 1;
    return PSM_OK;
  }
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, me, peer));
  *ok_out = can ? 1 : 0;
  return PSM_OK;
}

int psm_ipc_close_all(void) {
  auto& m = ipc_maps();
  for (auto& kv : m) cudaIpcCloseMemHandle(kv.second);
  m.clear();
  return PSM_OK;
}

int psm_plan_set_peer_halo(psm_plan* P, int patch, int side, double* peer_buf0, double* peer_buf1, int peer_nz) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  if (patch < 0 || patch >= P->npatch || (side != 0 && side != 1)) return fail(PSM_EINVAL, "bad patch/side");
  if ((peer_buf0 == nullptr) != (peer_buf1 == nullptr)) return fail(PSM_EINVAL, "give both peer buffers or neither");
  PatchDev& h = P->hp[patch];
  if (peer_buf0) {
    if (P->kind != PSM_BLOCK_LINE || !P->tiled || !line_nx_specialised(h.nx) || h.R != zmarch_rows(h.nx))
      return fail(PSM_EUNSUPPORTED, "the fused halo needs the z-marching line-Jacobi kernel (nx=%d)", h.nx);
    if (side == 0 && peer_nz < 1) return fail(PSM_EINVAL, "the lower neighbour's nz must be positive");
  }
  if (side == 0) {
    h.peer_lo[0] = peer_buf0;
    h.peer_lo[1] = peer_buf1;
    h.peer_lo_nz = peer_buf0 ? peer_nz : 0;
  } else {
    h.peer_hi[0] = peer_buf0;
    h.peer_hi[1] = peer_buf1;
  }
  h.iface = (h.peer_lo[0] ? 1 : 0) | (h.peer_hi[0] ? 2 : 0);
  CUDA_TRY(cudaMemcpy(P->d_patches + patch, &h, sizeof h, cudaMemcpyHostToDevice));
  return PSM_OK;
}

int psm_halo_signal(int* flag_a, int* flag_b, int value, void* stream) {
  CUDA_TRY(launch_halo_signal(flag_a, flag_b, value, (cudaStream_t)stream));
  return PSM_OK;
}

int psm_halo_wait(const int* flags, int n, int value, void* stream) {
  if (!flags || n < 1 || n > 4096) return fail(PSM_EINVAL, "bad flag list");
  CUDA_TRY(launch_halo_wait(flags, n, value, (cudaStream_t)stream));
  return PSM_OK;
}

long long psm_plan_launches(const psm_plan* P) { return P ? P->launches : -1; }
// The launch sequence of smooth() (smoother.py:197-214) for `steps` steps:
// Jacobi: [refresh] then steps x (sweep into the inactive buffers with the
// history slot, all patches swap, refresh with the x faces skipped) [, final
// residual]; GS: [refresh, residual] then steps x (sweep, refresh [,
// residual]).  `act` is updated to the active flags after the steps.
// Line GS on one patch with physical faces: several steps per launch (the
// multi-sweep mode of the pipelined kernel, psm_line_gs_pipe.cu); 0 when the
// plan does not qualify (the caller then runs step by step)
static int gs_multi_steps(psm_plan* P, const unsigned char* active, double omega, int gs_mode, int steps,
                          int history, cudaStream_t s, int* done) {
  *done = 0;
  if (P->kind != PSM_BLOCK_LINE || steps < 2 || steps >= 0x7fff) return PSM_OK;
  const char* env = getenv("PSM_GS_MULTI");
  if (env && env[0] == '0') return PSM_OK;
  for (auto& h : P->hp)
    if (!gs_pipe_supported(h.nx) || (((uintptr_t)h.buf[0] | (uintptr_t)h.buf[1]) % 16) != 0) return PSM_OK;
  if (P->npatch != 1 || P->ncopy != 0) return PSM_OK;
  if (!P->gspipe) {
    int nt = 0;
    int rc = psm_gs_pipe_prepare(P, &nt);
    if (rc) return rc;
    P->gs_ntickets = nt;
    CUDA_TRY(cudaMalloc(&P->d_gsflags, (P->nplanes + nt) * sizeof(int)));
  }
  if (!psm_gs_pipe_multi_ok(P)) return PSM_OK;
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  // per-sweep progress words (steps * nplanes) and the tickets
  const long long nflags = (long long)steps * P->nplanes + P->gs_ntickets;
  if (nflags > P->ms_flag_cap) {
    if (P->d_msflags) cudaFree(P->d_msflags);
    P->d_msflags = nullptr;
    CUDA_TRY(cudaMalloc(&P->d_msflags, nflags * sizeof(int)));
    P->ms_flag_cap = nflags;
  }
  CUDA_TRY(cudaMemsetAsync(P->d_msflags, 0, nflags * sizeof(int), s));
  double* hist = nullptr;
  if (history) {
    hist = slot_ptr(P, 1, &rc);
    if (rc) return rc;
  }
  rc = psm_gs_pipe_multi(P, da, omega, gs_mode == PSM_GS_CHAOTIC, steps, hist, std::max<long long>(1, P->ntiles),
                         P->d_msflags, P->d_msflags + (long long)steps * P->nplanes, s);
  if (rc) return rc;
  P->phys_pending = 2;  // every physical ghost is left to the refresh
  *done = 1;
  return PSM_OK;
}

static int smooth_sequence(psm_plan* P, std::vector<unsigned char>& act, int scheme, double omega, int steps,
                           int gs_mode, int history, void* stream) {
  int rc;
  if (history) {
    rc = psm_refresh_ghosts(P, act.data(), PSM_GHOST_ALL, stream);
    if (rc) return rc;
  }
  if (scheme == 0) {
    for (int s = 0; s < steps; ++s) {
      rc = psm_jacobi_sweep(P, act.data(), omega, history ? s : -1, stream);
      if (rc) return rc;
      for (auto& a : act) a ^= 1;
      rc = psm_refresh_ghosts(P, act.data(), PSM_GHOST_ALL | PSM_GHOST_SKIP_X, stream);
      if (rc) return rc;
    }
    if (history) return psm_residual(P, act.data(), steps, stream);
    return PSM_OK;
  }
  if (history) {
    rc = psm_residual(P, act.data(), 0, stream);
    if (rc) return rc;
  }
  {
    int done = 0;
    rc = gs_multi_steps(P, act.data(), omega, gs_mode, steps, history, (cudaStream_t)stream, &done);
    if (rc) return rc;
    if (done) {
      rc = psm_refresh_ghosts(P, act.data(), PSM_GHOST_ALL | PSM_GHOST_SKIP_X, stream);
      if (rc) return rc;
      return history ? psm_residual(P, act.data(), steps, stream) : PSM_OK;
    }
  }
  for (int s = 0; s < steps; ++s) {
    rc = psm_gs_sweep(P, act.data(), omega, gs_mode, stream);
    if (rc) return rc;
    rc = psm_refresh_ghosts(P, act.data(), PSM_GHOST_ALL | PSM_GHOST_SKIP_X, stream);
    if (rc) return rc;
    if (history) {
      rc = psm_residual(P, act.data(), s + 1, stream);
      if (rc) return rc;
    }
  }
  return PSM_OK;
}

int psm_smooth_steps(psm_plan* P, unsigned char* active, int scheme, double omega, int steps, int gs_mode,
                     int history, void* stream) {
  if (!P || !active) return fail(PSM_EINVAL, "null argument");
  if (scheme != 0 && scheme != 1) return fail(PSM_EINVAL, "scheme must be 0 (Jacobi) or 1 (GS), got %d", scheme);
  if (steps < 1) return fail(PSM_EINVAL, "steps must be positive, got %d", steps);
  if (history && steps + 1 > P->cap_slots) return fail(PSM_EINVAL, "history needs %d reserved slots", steps + 1);
  std::vector<unsigned char> act(active, active + P->npatch);
  for (unsigned char a : act)
    if (a > 1) return fail(PSM_EINVAL, "active flags must be 0 or 1");
  char kb[96];
  // the key holds everything that changes the captured launch sequence:
  // the process-wide plane solver mode (psm_plane_solver) and the staged
  // plane-GS choice included, so changing either re-captures
  snprintf(kb, sizeof kb, "%d:%a:%d:%d:%d:%d:%d:", scheme, omega, steps, gs_mode, history, psm_plane_band_mode,
           getenv("PSM_PLANE_GS_STAGED") ? 1 : 0);
  auto& G = P->graphs[std::string(kb) + std::string((const char*)active, P->npatch)];
  if (G.exec == nullptr && G.seen == 0) {
    // first call with this key: eager, which also performs every lazy
    // allocation (active vectors, work units, factor tables, workspaces)
    G.seen = 1;
    const int rc = smooth_sequence(P, act, scheme, omega, steps, gs_mode, history, stream);
    if (rc) return rc;
  } else {
    if (G.exec == nullptr) {  // second call: capture once, replay from now on
      if (!P->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&P->cap_stream, cudaStreamNonBlocking));
      const long long before = P->launches;
      CUDA_TRY(cudaStreamBeginCapture(P->cap_stream, cudaStreamCaptureModeThreadLocal));
      const int rc = smooth_sequence(P, act, scheme, omega, steps, gs_mode, history, P->cap_stream);
      cudaGraph_t graph = nullptr;
      cudaError_t ce = cudaStreamEndCapture(P->cap_stream, &graph);
      if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (ce != cudaSuccess) return fail(PSM_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&G.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ce != cudaSuccess) {
        G.exec = nullptr;
        return fail(PSM_ECUDA, "graph instantiate: %s", cudaGetErrorString(ce));
      }
      G.kernels = P->launches - before;
      P->launches = before;
    }
    CUDA_TRY(cudaGraphLaunch(G.exec, (cudaStream_t)stream));
    P->launches += G.kernels;
  }
  // the active flags after the steps (Jacobi swaps every patch once per step)
  if (scheme == 0 && (steps & 1))
    for (int i = 0; i < P->npatch; ++i) active[i] ^= 1;
  return PSM_OK;
}


int psm_plane_solver(int mode) {
  const int prev = psm_plane_band_mode == 0 ? PSM_PLANE_DST : PSM_PLANE_AUTO;
  if (mode == PSM_PLANE_DST) psm_plane_band_mode = 0;
  else if (mode == PSM_PLANE_AUTO) psm_plane_band_mode = -1;
  return prev;
}


// Work units (patch, plane) in dependency order and the progress flags of
// the pipelined line GS kernel; built on first use.
static int psm_line_gs_prepare(psm_plan* P) {
  if (P->d_flags) return PSM_OK;
  int max_nx = 0;
  for (auto& h : P->hp) max_nx = std::max(max_nx, h.nx);
  const int nc = gs_chunks_for(max_nx);
  if (nc == 0) return fail(PSM_EUNSUPPORTED, "pipelined line GS needs nx <= 256");
  std::vector<int> up, uk;
  for (int p = 0; p < P->npatch; ++p)
    for (int k = 0; k < P->hp[p].nz; ++k) {
      up.push_back(p);
      uk.push_back(k);
    }
  P->nunits = (long long)up.size();
  CUDA_TRY(cudaMalloc(&P->d_flags, (P->nplanes + 1) * sizeof(int)));
  CUDA_TRY(cudaMalloc(&P->d_unit_patch, up.size() * sizeof(int)));
  CUDA_TRY(cudaMalloc(&P->d_unit_plane, uk.size() * sizeof(int)));
  CUDA_TRY(cudaMemcpy(P->d_unit_patch, up.data(), up.size() * sizeof(int), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(P->d_unit_plane, uk.data(), uk.size() * sizeof(int), cudaMemcpyHostToDevice));
  P->gs_threads = 128;
  P->gs_smem = 4 * gs_smem_per_warp(nc);
  int occ = gs_occupancy(nc, P->gs_threads, P->gs_smem);
  if (occ < 1) occ = 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (P->nunits + 3) / 4;
  long long grid = std::min<long long>((long long)occ * sms, std::max<long long>(1, want));
  P->gs_grid = (int)((grid << 4) | nc);
  return PSM_OK;
}

int psm_gs_sweep(psm_plan* P, const unsigned char* active, double omega, int mode, void* stream) {
  if (!P) return fail(PSM_EINVAL, "null plan");
  if (!(omega > 0.0 && omega <= 1.0)) return fail(PSM_EINVAL, "omega must lie in (0, 1], got %g", omega);
  if (mode != PSM_GS_WAVEFRONT && mode != PSM_GS_CHAOTIC) return fail(PSM_EINVAL, "bad GS mode %d", mode);
  unsigned char* da;
  int rc = get_active(P, active, &da);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  P->phys_pending = 2;  // GS sweeps leave every physical ghost to the refresh
  if (P->kind == PSM_BLOCK_PLANE) return psm_plane_gs(P, da, omega, s);
  if (P->kind == PSM_BLOCK_BOX) {  // lexicographic block order = wavefronts bi+bj+bk, in place
    // one persistent launch with per-block dependency flags when the blocks
    // have template dims (psm_box.cu), else one launch per wavefront
    const int bx = P->box_dims[0], by = P->box_dims[1], bz = P->box_dims[2];
    const bool tmpl = (bx == 2 && by == 2 && bz == 2) || (bx == 4 && by == 2 && bz == 2) ||
                      (bx == 4 && by == 4 && bz == 2) || (bx == 4 && by == 4 && bz == 4) ||
                      (bx == 8 && by == 4 && bz == 4) || (bx == 8 && by == 8 && bz == 4) ||
                      (bx == 8 && by == 8 && bz == 8);
    const char* env = getenv("PSM_BOX_GS_WAVES");
    if (tmpl && !(env && env[0] == '1')) {
      CUDA_TRY(cudaMemsetAsync(P->d_box_flags, 0, (size_t)(P->nboxes + 1) * sizeof(int), s));
      CUDA_TRY(launch_box_sweep(P->d_patches, da, P->st, omega, P->d_boxes, P->nboxes, 1, 1, 1, 1, bx, by, bz, s,
                                P->d_box_deps, P->d_box_flags, P->d_box_flags + P->nboxes, P->d_box_tmaps));
      P->launches += 1;
      return PSM_OK;
    }
    for (size_t w = 0; w + 1 < P->box_wave_off.size(); ++w) {
      const int b0 = P->box_wave_off[w], b1 = P->box_wave_off[w + 1];
      CUDA_TRY(launch_box_sweep(P->d_patches, da, P->st, omega, P->d_boxes + b0, b1 - b0, 1, 1, 1, 1,
                                P->box_dims[0], P->box_dims[1], P->box_dims[2], s));
      P->launches += 1;
    }
    return PSM_OK;
  }
  if (P->kind != PSM_BLOCK_LINE) return fail(PSM_EINVAL, "plan was created without a block kind (ghost-only)");
  bool pipe = true;
  for (auto& h : P->hp)  // TMA row copies need 16-byte aligned buffers
    pipe = pipe && gs_pipe_supported(h.nx) && (((uintptr_t)h.buf[0] | (uintptr_t)h.buf[1]) % 16 == 0);
  if (pipe) {
    if (!P->gspipe) {
      int nt = 0;
      rc = psm_gs_pipe_prepare(P, &nt);
      if (rc) return rc;
      P->gs_ntickets = nt;
      CUDA_TRY(cudaMalloc(&P->d_gsflags, (P->nplanes + nt) * sizeof(int)));
    }
    CUDA_TRY(cudaMemsetAsync(P->d_gsflags, 0, (P->nplanes + P->gs_ntickets) * sizeof(int), s));
    return psm_gs_pipe_sweep(P, da, omega, mode == PSM_GS_CHAOTIC, P->d_gsflags, P->d_gsflags + P->nplanes, s);
  }
  int max_nx = 0;
  for (auto& h : P->hp) max_nx = std::max(max_nx, h.nx);
  if (!P->tiled || gs_chunks_for(max_nx) == 0) {
    // generic path: one launch per wavefront d = j + k (all patches at once)
    int maxd = 0;
    long long nj = 0;
    for (auto& h : P->hp) {
      maxd = std::max(maxd, h.ny + h.nz - 1);
      nj += h.ny;
    }
    for (int d = 0; d < maxd; ++d)
      CUDA_TRY(launch_line_gs_generic(P->d_patches, P->npatch, da, P->st, omega, d, nj, s));
    P->launches += maxd;
    return PSM_OK;
  }
  rc = psm_line_gs_prepare(P);
  if (rc) return rc;
  CUDA_TRY(cudaMemsetAsync(P->d_flags, 0, (P->nplanes + 1) * sizeof(int), s));
  CUDA_TRY(launch_line_gs(mode, P->d_patches, P->npatch, da, P->st, omega, P->d_flags + 1, P->nunits,
                          P->d_unit_patch, P->d_unit_plane, P->gs_threads, P->gs_smem, P->gs_grid, s));
  P->launches += 1;
  return PSM_OK;
}

int psm_history_sumsq(psm_plan* P, int nslots, double* out_host, void* stream) {
  if (!P || nslots < 0 || (nslots > 0 && !out_host)) return fail(PSM_EINVAL, "bad arguments");
  if (nslots > P->cap_slots) return fail(PSM_EINVAL, "only %d history slots reserved", P->cap_slots);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t tstride = std::max<long long>(1, P->ntiles);
  if (nslots > 0) {  // one launch for every slot (same bits as plane sums + tree per slot)
    CUDA_TRY(launch_history_reduce(P->d_patches, P->npatch, P->d_partials, (long long)tstride, P->nplanes, nslots,
                                   P->d_sums, s));
    P->launches += 1;
  }
  if (nslots > 0) {
    CUDA_TRY(cudaMemcpyAsync(out_host, P->d_sums, nslots * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return PSM_OK;
}

int psm_history_planes(psm_plan* P, int slot, double* out_dev, void* stream) {
  if (!P || !out_dev) return fail(PSM_EINVAL, "bad arguments");
  if (slot < 0 || slot >= P->cap_slots) return fail(PSM_EINVAL, "bad slot %d", slot);
  const size_t tstride = std::max<long long>(1, P->ntiles);
  CUDA_TRY(launch_plane_sums(P->d_patches, P->npatch, P->d_partials + slot * tstride, out_dev, P->nplanes,
                             (cudaStream_t)stream));
  return PSM_OK;
}

int psm_tree_sum(const double* in_dev, long long n, double* out_dev, void* stream) {
  if (!in_dev || !out_dev || n < 0) return fail(PSM_EINVAL, "bad arguments");
  CUDA_TRY(launch_tree_sum(in_dev, n, out_dev, (cudaStream_t)stream));
  return PSM_OK;
}

}  // extern "C"
