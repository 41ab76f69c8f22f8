// Plane-block (xy-plane) kernels: exact plane inverse, Jacobi and GS sweeps.
//
// Replaces, for block_dims (>=nx, >=ny, 1):
//   InverseCache.get -> invert_dense of the (nx*ny)^2 plane operator
//       blocklinalg.py:132-151, stencil.py:115-138 (infeasible beyond ~48^2:
//       SURVEY F8), and its dense matvec blocklinalg.py:90-105
//   smoother._jacobi_step / _gs_step with plane blocks  smoother.py:138-169
//
// The closure-free plane operator c*I + a*(S_x (x) I) + (fy-, fy+ couplings
// in y) with symmetric x faces a = faces[0] = faces[1] is diagonalised along
// x by the orthonormal DST-I basis Q (Q = Q^T = Q^-1).  Per x-mode i the
// remaining operator is tridiagonal in y with diagonal c + 2a cos(pi i/(nx+1)).
// So Ainv r = Q * T_i^-1 * (Q r): a GEMM with Q along x, one Thomas solve
// along y per (plane, mode), and a GEMM back.  The two transforms are the
// hand-written DMMA tile kernels of psm_plane_dst.cu (parity-split DST-I,
// residual / relaxation fused into their prologue / epilogue); the modal
// Thomas solves are this file's kernels.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "psm_internal.cuh"

namespace psm {
void plane_band_tables(long double c, long double a, long double blo, long double bup, int nx, int ny, int* bw_out,
                       int* nj_out, std::vector<double>& H);
int band_k_for(int nx);
cudaError_t launch_plane_band_jacobi(int K, int BW, const PatchDev* patches, const unsigned char* active,
                                     double omega, const double* rbuf, double* zbuf, const int2* units,
                                     int nunits, const double* hinf_host, cudaStream_t s);
void dst_split_table(const std::vector<double>& Q, int nx, std::vector<double>& out);
size_t dst_table_doubles(int nx);
int dst_max_nx();
cudaError_t launch_dst_rows(int epi, const PatchDev* patches, int p0, int p1, long long c0, long long nrows, int nx,
                            const double* qf, const unsigned char* active, double omega, const double* in,
                            double* out, long long rows_per_patch, cudaStream_t s);
cudaError_t launch_plane_gs_chain(const PlaneFac* d_fac, int nx, int ny, int nj, const PatchDev* patches, int p0,
                                  int np, int maxnz, double czw, double* buf, cudaStream_t s);
enum { kDstEpiStore = 0, kDstEpiRelaxInPlace = 1, kDstEpiRelaxInto = 2 };
cudaError_t launch_line_tiles(int mode, const PatchDev* patches, int npatch, const unsigned char* active,
                              const StencilDev& st, double omega, double* partials, double* rbuf, long long tile_base,
                              long long ntiles, int threads, size_t smem, cudaStream_t stream);

// r = f - A u of every cell of plane `k` of every patch with nz > k (GS
// stage) into the compact stage buffer, rows of the same patch contiguous.
__global__ void plane_stage_residual_kernel(const PatchDev* __restrict__ patches, int npatch,
                                            const unsigned char* __restrict__ active, StencilDev st, int k,
                                            const long long* __restrict__ stage_off, double* __restrict__ rbuf,
                                            long long total) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = npatch - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (stage_off[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const PatchDev& P = patches[lo];
    if (k >= P.nz) continue;
    const long long e = g - stage_off[lo];
    const int nx = P.nx, ny = P.ny;
    if (e >= (long long)nx * ny) continue;
    const int j = (int)(e / nx), x = (int)(e - (long long)j * nx);
    const long long px = nx + 2, pxy = px * (ny + 2);
    const double* u = P.buf[active[lo]];
    const long long iu = (long long)(k + 1) * pxy + (long long)(j + 1) * px + x + 1;
    rbuf[g] = residual7(st, P.f[((long long)k * ny + j) * nx + x], u[iu], u[iu - 1], u[iu + 1], u[iu - px],
                        u[iu + px], u[iu - pxy], u[iu + pxy]);
  }
}

// Thomas along y for every (plane, mode) of a batch of planes that share one
// PlaneFac.  Layout: plane-major, then y, then mode (x-mode fastest), so
// threads of a warp take consecutive modes (coalesced).  In place.
__global__ void plane_modal_thomas_kernel(const PlaneFac* __restrict__ F, double* __restrict__ buf, long long nplanes) {
  constexpr int B = 16;  // rows per batch: the loads of a batch are issued together (latency once per B rows)
  const int nx = F->nx, ny = F->ny;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nplanes * nx) return;
  const long long pl = t / nx;
  const int i = (int)(t - pl * nx);
  double* b = buf + pl * (long long)nx * ny + i;
  const double* cp = F->cp + i;
  const double* invm = F->invm + i;
  const double lo = F->fy_lo;
  double prev = 0.0;
  int j = 0;
  for (; j + B <= ny; j += B) {
    double v[B], m[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      v[q] = b[(long long)(j + q) * nx];
      m[q] = __ldg(invm + (long long)(j + q) * nx);
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      prev = fma(-lo, prev, v[q]) * m[q];
      b[(long long)(j + q) * nx] = prev;
    }
  }
  for (; j < ny; ++j) {
    prev = fma(-lo, prev, b[(long long)j * nx]) * invm[(long long)j * nx];
    b[(long long)j * nx] = prev;
  }
  double next = prev;
  j = ny - 2;
  for (; j - B + 1 >= 0; j -= B) {
    double v[B], c[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      v[q] = b[(long long)(j - q) * nx];
      c[q] = __ldg(cp + (long long)(j - q) * nx);
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      next = fma(-c[q], next, v[q]);
      b[(long long)(j - q) * nx] = next;
    }
  }
  for (; j >= 0; --j) {
    next = fma(-cp[(long long)j * nx], next, b[(long long)j * nx]);
    b[(long long)j * nx] = next;
  }
}

// The same modal solves with two threads per line (symmetric y faces):
// the top thread eliminates rows 0..m-1 downwards, the bottom thread rows
// ny-1..m upwards with the same factors (for lo == up the elimination from
// the bottom is the mirror image), the pair meets in an exact 2x2 system for
// x(m-1), x(m) (values swapped by shuffle), and each back-substitutes
// outwards: half the dependent chain of the one-thread sweep, exact.
__global__ void plane_modal_thomas2_kernel(const PlaneFac* __restrict__ F, double* __restrict__ buf,
                                           long long nplanes) {
  constexpr int B = 16;
  const int nx = F->nx, ny = F->ny, m = ny / 2;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = t < 2 * nplanes * nx;  // whole warps stay for the shuffles
  const long long line = in ? t >> 1 : 0;
  const int bot = (int)(t & 1);
  const long long pl = line / nx;
  const int i = (int)(line - pl * nx);
  double* b = buf + pl * (long long)nx * ny + i;
  const double* cp = F->cp + i;
  const double* invm = F->invm + i;
  const double lo = F->fy_lo;  // == fy_up
  // this thread's rows: top j = jj, bottom j = ny-1-jj, jj = 0..len-1
  const int len = bot ? ny - m : m;
  const long long j0 = bot ? ny - 1 : 0, dj = bot ? -nx : nx;
  double prev = 0.0;
  int jj = 0;
  if (in) {
    for (; jj + B <= len; jj += B) {
      double v[B], mm[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        v[q] = b[j0 * nx + (jj + q) * dj];
        mm[q] = __ldg(invm + (long long)(jj + q) * nx);
      }
#pragma unroll
      for (int q = 0; q < B; ++q) {
        prev = fma(-lo, prev, v[q]) * mm[q];
        b[j0 * nx + (jj + q) * dj] = prev;
      }
    }
    for (; jj < len; ++jj) {
      prev = fma(-lo, prev, b[j0 * nx + jj * dj]) * invm[(long long)jj * nx];
      b[j0 * nx + jj * dj] = prev;
    }
  }
  // meet: top x(m-1) = yT - cT x(m), bottom x(m) = yB - cB x(m-1)
  const double c_own = in && len > 0 ? __ldg(cp + (long long)(len - 1) * nx) : 0.0;
  const double y_oth = __shfl_xor_sync(0xffffffffu, prev, 1);
  const double c_oth = __shfl_xor_sync(0xffffffffu, c_own, 1);
  const double yT = bot ? y_oth : prev, yB = bot ? prev : y_oth;
  const double cT = bot ? c_oth : c_own, cB = bot ? c_own : c_oth;
  const double xT = (yT - cT * yB) / (1.0 - cT * cB);
  double next = bot ? yB - cB * xT : xT;
  if (!in || len == 0) return;
  b[j0 * nx + (len - 1) * dj] = next;
  jj = len - 2;
  for (; jj - B + 1 >= 0; jj -= B) {
    double v[B], c[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      v[q] = b[j0 * nx + (jj - q) * dj];
      c[q] = __ldg(cp + (long long)(jj - q) * nx);
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      next = fma(-c[q], next, v[q]);
      b[j0 * nx + (jj - q) * dj] = next;
    }
  }
  for (; jj >= 0; --jj) {
    next = fma(-cp[(long long)jj * nx], next, b[j0 * nx + jj * dj]);
    b[j0 * nx + jj * dj] = next;
  }
}

static void launch_modal_thomas(const PlaneFac& h, const PlaneFac* d, double* buf, long long nplanes,
                                cudaStream_t s) {
  if (h.fy_lo == h.fy_up && h.ny >= 2 && !getenv("PSM_PLANE_THOMAS1")) {
    plane_modal_thomas2_kernel<<<(unsigned)((2 * nplanes * h.nx + 127) / 128), 128, 0, s>>>(d, buf, nplanes);
  } else {
    plane_modal_thomas_kernel<<<(unsigned)((nplanes * h.nx + 127) / 128), 128, 0, s>>>(d, buf, nplanes);
  }
}

// GS stage k epilogue fused with stage k+1's residual: u(k) += omega x in
// place, then r(k+1) = f - A u at the same (x, y), which reads u(k) only at
// this cell (its z-neighbour, just updated by this thread) and plane k+1's
// old values; r(k+1) overwrites x in the stage buffer (same element).
// grid (cell blocks of the largest plane, patch): no patch search per cell
__global__ void plane_stage_relax_residual_kernel(const PatchDev* __restrict__ patches, int npatch,
                                                  const unsigned char* __restrict__ active, StencilDev st,
                                                  double omega, int k, const long long* __restrict__ stage_off,
                                                  double* __restrict__ sbuf, long long total) {
  const int lo = blockIdx.y;
  const PatchDev& P = patches[lo];
  const int nx = P.nx, ny = P.ny;
  if (k >= P.nz) return;  // this patch has no stage k (nothing to relax, no plane k+1)
  const long long off = stage_off[lo];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)nx * ny;
       e += (long long)gridDim.x * blockDim.x) {
    const long long g = off + e;
    const int j = (int)(e / nx), x = (int)(e - (long long)j * nx);
    const long long px = nx + 2, pxy = px * (ny + 2);
    double* u = P.buf[active[lo]];
    const long long iu = (long long)(k + 1) * pxy + (long long)(j + 1) * px + x + 1;
    const double un = relax(u[iu], omega, sbuf[g]);
    u[iu] = un;
    if (k + 1 < P.nz) {
      const long long iv = iu + pxy;  // (x, j, k+1)
      const double zm = un;
      sbuf[g] = residual7(st, P.f[((long long)(k + 1) * ny + j) * nx + x], u[iv], u[iv - 1], u[iv + 1], u[iv - px],
                          u[iv + px], zm, u[iv + pxy]);
    }
  }
}

static unsigned blocks_for(long long n, int tpb) {
  long long b = (n + tpb - 1) / tpb;
  if (b > 148LL * 32) b = 148LL * 32;
  return (unsigned)std::max<long long>(1, b);
}

}  // namespace psm

using namespace psm;

// per-plan state of the plane path
struct PlaneRun {  // consecutive patches sharing one PlaneFac (same nx, ny)
  int p0, p1;
  const PlaneFac* d_fac;
  const PlaneFac* h_fac;
  const double* Q;
  const double* Qf;  // split DST table (psm_plane_dst.cu)
  int nx, ny;
  int bw = 0;              // banded factorised solve available (psm_plane_band.cu)
  int2* d_units = nullptr;  // (patch, plane) units of the run for the banded kernel
  int nunits = 0;
  std::vector<double> hinf;  // converged kernel H_nj (host copy, passed by value)
};
int psm_plane_band_mode = -1;  // -1: auto (banded where available), 0: DST only (tests/bench)

struct PlaneState {
  double* rbuf = nullptr;   // sum of cells: residual, then x
  double* rhat = nullptr;   // sum of cells: modal coefficients
  double* sbuf = nullptr;   // GS stage buffers (sum over patches of nx*ny), x2
  double* shat = nullptr;
  long long* d_stage_off = nullptr;
  long long stage_total = 0;
  long long stage_max = 0;  // cells of the largest patch plane

  std::vector<long long> stage_off;
  std::vector<PlaneRun> runs;
};


// error plumbing shared with psm_api.cu
int psm_set_error(int code, const char* msg);
extern "C" int psm_plane_residual(psm_plan* P, const unsigned char* da, double* partials, double* rbuf,
                                  cudaStream_t s);  // psm_api.cu
extern "C" cudaError_t psm_side_fork(psm_plan* P, cudaStream_t s, int n);  // psm_api.cu
extern "C" cudaError_t psm_side_join(psm_plan* P, cudaStream_t s, int n);

#define PCUDA(expr)                                                                      \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(_e));      \
  } while (0)

int psm_plane_build(const psm_stencil* st, int nx, int ny, psm_factors* F) {
  const long double c = st->center, a = st->faces[0], b = st->faces[1];
  const long double ylo = st->faces[2], yup = st->faces[3];
  if (a != b)
    return psm_set_error(PSM_EUNSUPPORTED,
                         "plane blocks need symmetric x faces (faces[0] == faces[1]) for the DST factorisation");
  if (2 * fabsl(a) + fabsl(ylo) + fabsl(yup) > c)
    return psm_set_error(PSM_ESINGULAR, "plane block operator is not diagonally dominant");
  const size_t nq = (size_t)nx * nx, nt = (size_t)nx * ny;
  std::vector<double> Q(nq), cp(nt), invm(nt);
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double sc = sqrtl(2.0L / (nx + 1));
  for (int p = 0; p < nx; ++p)
    for (int i = 0; i < nx; ++i) Q[(size_t)p * nx + i] = (double)(sc * sinl(pi * (p + 1) * (i + 1) / (nx + 1)));
  for (int i = 0; i < nx; ++i) {
    const long double d = c + 2.0L * a * cosl(pi * (i + 1) / (nx + 1));
    long double prev = 0;
    for (int j = 0; j < ny; ++j) {
      const long double m = d - ylo * prev;
      if (fabsl(m) < 1e-14L * c) return psm_set_error(PSM_ESINGULAR, "plane modal pivot below 1e-14*|A|");
      invm[(size_t)j * nx + i] = (double)(1.0L / m);
      cp[(size_t)j * nx + i] = (double)(yup / m);
      prev = yup / m;
    }
  }
  int bw = 0, nj = 0;
  std::vector<double> band;
  plane_band_tables(c, a, ylo, yup, nx, ny, &bw, &nj, band);
  std::vector<double> qf;
  if (nx <= dst_max_nx()) dst_split_table(Q, nx, qf);
  const size_t bytes = sizeof(PlaneFac) + (nq + 2 * nt + band.size() + qf.size()) * sizeof(double);
  if (cudaMalloc(&F->dev, bytes) != cudaSuccess) return psm_set_error(PSM_ENOMEM, "cudaMalloc for plane factors");
  double* tab = (double*)((char*)F->dev + sizeof(PlaneFac));
  PlaneFac& H = F->h_plane;
  memset(&H, 0, sizeof H);
  H.nx = nx;
  H.ny = ny;
  H.fy_lo = (double)ylo;
  H.fy_up = (double)yup;
  H.Q = tab;
  H.cp = tab + nq;
  H.invm = tab + nq + nt;
  H.bw = bw;
  H.nj = nj;
  H.H = band.empty() ? nullptr : tab + nq + 2 * nt;
  H.Qf = qf.empty() ? nullptr : tab + nq + 2 * nt + band.size();
  // first row from which both Thomas tables stay bitwise constant
  H.nconst = 0;
  for (int j = ny - 1; j > 0; --j) {
    bool same = true;
    for (int i = 0; i < nx && same; ++i)
      same = invm[(size_t)j * nx + i] == invm[(size_t)(j - 1) * nx + i] &&
             cp[(size_t)j * nx + i] == cp[(size_t)(j - 1) * nx + i];
    if (!same) {
      H.nconst = j;
      break;
    }
  }
  F->d_plane = (PlaneFac*)F->dev;
  PCUDA(cudaMemcpy(F->dev, &H, sizeof H, cudaMemcpyHostToDevice));
  PCUDA(cudaMemcpy(tab, Q.data(), nq * sizeof(double), cudaMemcpyHostToDevice));
  PCUDA(cudaMemcpy(tab + nq, cp.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  PCUDA(cudaMemcpy(tab + nq + nt, invm.data(), nt * sizeof(double), cudaMemcpyHostToDevice));
  if (!band.empty())
    PCUDA(cudaMemcpy(tab + nq + 2 * nt, band.data(), band.size() * sizeof(double), cudaMemcpyHostToDevice));
  if (!qf.empty())
    PCUDA(cudaMemcpy(tab + nq + 2 * nt + band.size(), qf.data(), qf.size() * sizeof(double),
                     cudaMemcpyHostToDevice));
  return PSM_OK;
}

// out = Q_x applied to `nvec` row-major vectors of length nx (the DMMA tile
// kernel of psm_plane_dst.cu, no fusion)
static int dst_rows(const PlaneFac& h, const double* in, double* out, long long nvec, cudaStream_t s) {
  if (!h.Qf)
    return psm_set_error(PSM_EUNSUPPORTED, "DST plane transforms support nx <= 512 (use the banded plane solver)");
  PCUDA(launch_dst_rows(kDstEpiStore, nullptr, 0, 0, 0, nvec, h.nx, h.Qf, nullptr, 0.0, in, out, 0, s));
  return PSM_OK;
}

int psm_plane_apply(const psm_factors* F, const double* r, double* x, long long count, cudaStream_t stream) {
  if (F->kind != PSM_BLOCK_PLANE) return psm_set_error(PSM_EINVAL, "not a plane factor object");
  const PlaneFac& H = F->h_plane;
  const long long n = (long long)H.nx * H.ny * count;
  if (n == 0) return PSM_OK;
  double* tmp = nullptr;
  PCUDA(cudaMallocAsync(&tmp, n * sizeof(double), stream));
  int rc = dst_rows(H, r, tmp, (long long)H.ny * count, stream);
  if (rc == PSM_OK) {
    launch_modal_thomas(H, F->d_plane, tmp, count, stream);
    rc = dst_rows(H, tmp, x, (long long)H.ny * count, stream);
  }
  cudaFreeAsync(tmp, stream);
  return rc;
}

int psm_plane_plan_setup(psm_plan* P) {
  PlaneState* S = new PlaneState();
  P->plane = S;
  long long cells = 0;
  for (auto& h : P->hp) cells += (long long)h.nx * h.ny * h.nz;
  PCUDA(cudaMalloc(&S->rbuf, cells * sizeof(double)));
  PCUDA(cudaMalloc(&S->rhat, cells * sizeof(double)));
  S->stage_off.resize(P->npatch);
  long long so = 0;
  for (int p = 0; p < P->npatch; ++p) {
    S->stage_off[p] = so;
    so += (long long)P->hp[p].nx * P->hp[p].ny;
  }
  S->stage_total = so;
  for (int p = 0; p < P->npatch; ++p)
    S->stage_max = std::max<long long>(S->stage_max, (long long)P->hp[p].nx * P->hp[p].ny);
  PCUDA(cudaMalloc(&S->sbuf, so * sizeof(double)));
  PCUDA(cudaMalloc(&S->shat, so * sizeof(double)));
  PCUDA(cudaMalloc(&S->d_stage_off, P->npatch * sizeof(long long)));
  PCUDA(cudaMemcpy(S->d_stage_off, S->stage_off.data(), P->npatch * sizeof(long long), cudaMemcpyHostToDevice));
  for (int p = 0; p < P->npatch;) {
    int q = p + 1;
    while (q < P->npatch && P->fac[q] == P->fac[p]) ++q;
    PlaneRun r;
    r.p0 = p;
    r.p1 = q;
    r.d_fac = P->fac[p]->d_plane;
    r.h_fac = &P->fac[p]->h_plane;
    r.Q = P->fac[p]->h_plane.Q;
    r.Qf = P->fac[p]->h_plane.Qf;
    r.nx = P->hp[p].nx;
    r.ny = P->hp[p].ny;
    r.bw = P->fac[p]->h_plane.bw;
    if (r.bw > 0) {
      const PlaneFac& hf = P->fac[p]->h_plane;
      r.hinf.resize(hf.bw + 1);
      PCUDA(cudaMemcpy(r.hinf.data(), hf.H + (size_t)hf.nj * (hf.bw + 1), (hf.bw + 1) * sizeof(double),
                       cudaMemcpyDeviceToHost));
      std::vector<int> uv;
      for (int q2 = p; q2 < q; ++q2)
        for (int k = 0; k < P->hp[q2].nz; ++k) {
          uv.push_back(q2);
          uv.push_back(k);
        }
      r.nunits = (int)(uv.size() / 2);
      PCUDA(cudaMalloc(&r.d_units, uv.size() * sizeof(int)));
      PCUDA(cudaMemcpy(r.d_units, uv.data(), uv.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    S->runs.push_back(r);
    p = q;
  }
  return PSM_OK;
}

int psm_plane_plan_free(psm_plan* P) {
  PlaneState* S = P->plane;
  if (!S) return PSM_OK;
  cudaFree(S->rbuf);
  cudaFree(S->rhat);
  cudaFree(S->sbuf);
  cudaFree(S->shat);
  cudaFree(S->d_stage_off);
  for (auto& r : S->runs) cudaFree(r.d_units);

  delete S;
  P->plane = nullptr;
  return PSM_OK;
}

// rows of each patch of a run when they are all equal (ny * nz), else 0
static long long run_rows_per_patch(const psm_plan* P, const PlaneRun& r) {
  for (int p = r.p0 + 1; p < r.p1; ++p)
    if (P->hp[p].nz != P->hp[r.p0].nz) return 0;
  return (long long)P->hp[r.p0].ny * P->hp[r.p0].nz;
}

// Jacobi: residual of every cell (tile kernel, mode 2 stores r and the
// history partials), then per run of patches sharing a factor either the
// banded factorised solve (writes v directly) or DST -> modal Thomas -> DST
// back -> relax into v.
int psm_plane_jacobi(psm_plan* P, const unsigned char* da, double omega, double* partials, cudaStream_t s) {
  PlaneState* S = P->plane;
  {
    const int rc = psm_plane_residual(P, da, partials, S->rbuf, s);
    if (rc) return rc;
  }
  // banded runs: several at once on side streams when there are several
  int nband = 0;
  for (const PlaneRun& r : S->runs) nband += (r.bw > 0 && psm_plane_band_mode != 0);
  const bool fan = nband > 1;
  if (fan) PCUDA(psm_side_fork(P, s, nband));  // runs are independent: several at once
  int bi = 0;
  for (const PlaneRun& r : S->runs) {
    const long long c0 = P->hp[r.p0].cell0;
    long long planes = 0, cells = 0;
    for (int p = r.p0; p < r.p1; ++p) {
      planes += P->hp[p].nz;
      cells += (long long)P->hp[p].nx * P->hp[p].ny * P->hp[p].nz;
    }
    if (r.bw > 0 && psm_plane_band_mode != 0) {
      cudaStream_t rs = fan ? P->side[bi++ % psm_plan::kSide] : s;
      PCUDA(launch_plane_band_jacobi(band_k_for(r.nx), r.bw, P->d_patches, da, omega, S->rbuf, S->rhat, r.d_units,
                                     r.nunits, r.hinf.data(), rs));
      P->launches += 1;
      continue;
    }
    // DST -> modal Thomas -> DST back with v = u + omega x (and v's x
    // ghosts) in the back transform's epilogue
    const long long nvec = planes * r.ny;
    (void)cells;
    const int rc = dst_rows(*r.h_fac, S->rbuf + c0, S->rhat + c0, nvec, s);
    if (rc) return rc;
    launch_modal_thomas(*r.h_fac, r.d_fac, S->rhat + c0, planes, s);
    PCUDA(cudaGetLastError());
    PCUDA(launch_dst_rows(kDstEpiRelaxInto, P->d_patches, r.p0, r.p1, c0, nvec, r.nx, r.Qf, da, omega, S->rhat + c0,
                          nullptr, run_rows_per_patch(P, r), s));
    P->launches += 3;
  }
  if (fan) PCUDA(psm_side_join(P, s, nband));
  return PSM_OK;
}

// Lexicographic plane GS: planes in k order, all patches of the level at
// each stage (patches couple only through step-end ghosts).
static int psm_plane_gs_staged(psm_plan* P, const unsigned char* da, double omega, cudaStream_t s);

// Plane GS with the stage recurrence in the transformed domain (see
// plane_gs_stage_kernel): residual of every plane from the pre-sweep iterate,
// one DST of all planes, maxnz stages of modal solves, one DST back, relax.
int psm_plane_gs(psm_plan* P, const unsigned char* da, double omega, cudaStream_t s) {
  PlaneState* S = P->plane;
  bool sym = !getenv("PSM_PLANE_GS_STAGED");
  for (const PlaneRun& r : S->runs) sym = sym && r.h_fac->fy_lo == r.h_fac->fy_up;
  if (!sym) return psm_plane_gs_staged(P, da, omega, s);
  for (const PlaneRun& r : S->runs)
    if (!r.Qf) return psm_set_error(PSM_EUNSUPPORTED, "plane GS supports nx <= 512");
  const double czw = P->st.zm * omega;
  // 1. the pre-sweep residual of every cell (z-marching line kernel, r only)
  {
    const int rc = psm_plane_residual(P, da, P->d_scratch, S->rbuf, s);
    if (rc) return rc;
  }
  for (const PlaneRun& r : S->runs) {
    const long long c0 = P->hp[r.p0].cell0;
    long long planes = 0;
    int maxnz = 0;
    for (int p = r.p0; p < r.p1; ++p) {
      planes += P->hp[p].nz;
      maxnz = std::max(maxnz, P->hp[p].nz);
    }
    // rhat = Q r_pre
    {
      const int rc = dst_rows(*r.h_fac, S->rbuf + c0, S->rhat + c0, planes * r.ny, s);
      if (rc) return rc;
    }
    // 2. every (patch, mode) chain over the stages k, one launch
    // (the chain kernel addresses planes by the patches' global cell0)
    PCUDA(launch_plane_gs_chain(r.d_fac, r.nx, r.ny, r.h_fac->nconst, P->d_patches, r.p0, r.p1 - r.p0, maxnz, czw,
                                S->rhat, s));
    // 3. x = Q xhat, relaxed into u in place
    PCUDA(launch_dst_rows(kDstEpiRelaxInPlace, P->d_patches, r.p0, r.p1, c0, planes * r.ny, r.nx, r.Qf, da, omega,
                          S->rhat + c0, nullptr, run_rows_per_patch(P, r), s));
    P->launches += 3;
  }
  return PSM_OK;
}

// Stage-by-stage form (any y faces): per stage DST, modal solves, DST back,
// relax in place fused with the next stage's residual.
static int psm_plane_gs_staged(psm_plan* P, const unsigned char* da, double omega, cudaStream_t s) {
  PlaneState* S = P->plane;
  int maxnz = 0;
  for (auto& h : P->hp) maxnz = std::max(maxnz, h.nz);
  plane_stage_residual_kernel<<<blocks_for(S->stage_total, 256), 256, 0, s>>>(P->d_patches, P->npatch, da, P->st, 0,
                                                                             S->d_stage_off, S->sbuf, S->stage_total);
  PCUDA(cudaGetLastError());
  P->launches += 1;
  for (int k = 0; k < maxnz; ++k) {
    for (const PlaneRun& r : S->runs) {
      // patches of the run that still have plane k (nz may differ)
      int p0 = r.p0;
      while (p0 < r.p1) {
        if (k >= P->hp[p0].nz) { ++p0; continue; }
        int p1 = p0 + 1;
        while (p1 < r.p1 && k < P->hp[p1].nz) ++p1;
        const long long o = S->stage_off[p0];
        const long long nplanes = p1 - p0;
        int rc = dst_rows(*r.h_fac, S->sbuf + o, S->shat + o, nplanes * r.ny, s);
        if (rc) return rc;
        launch_modal_thomas(*r.h_fac, r.d_fac, S->shat + o, nplanes, s);
        PCUDA(cudaGetLastError());
        rc = dst_rows(*r.h_fac, S->shat + o, S->sbuf + o, nplanes * r.ny, s);
        if (rc) return rc;
        P->launches += 3;
        p0 = p1;
      }
    }
    // relax stage k and form stage k+1's residual in one pass
    plane_stage_relax_residual_kernel<<<dim3(blocks_for(S->stage_max, 256), P->npatch), 256, 0, s>>>(
        P->d_patches, P->npatch, da, P->st, omega, k, S->d_stage_off, S->sbuf, S->stage_total);
    PCUDA(cudaGetLastError());
    P->launches += 1;
  }
  return PSM_OK;
}
