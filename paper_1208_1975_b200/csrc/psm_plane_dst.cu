// DST-I row transforms of the plane path on the fp64 tensor pipe.
//
// The exact plane-block inverse (blocklinalg.py:132-151 for block_dims
// (>=nx, >=ny, 1)) factors as Ainv = Q T^-1 Q with Q the orthonormal DST-I
// basis along x (psm_plane.cu).  Applying Q to every x-row of a level is a
// [rows x nx] x [nx x nx] product; this file computes it with hand-written
// mma.sync m8n8k4 f64 (DMMA) tiles, fused with what surrounds it:
//
//   prologue  the rows themselves (a buffer) or the residual r = f - A u of
//             the rows computed from the patch (block_residual,
//             stencil.py:93-112, the reference's rounding sequence)
//   epilogue  store the transformed rows, or relax in place u += omega x
//             (GS, smoother.py:156-169), or v = u + omega x plus v's x-face
//             ghosts (Jacobi, smoother.py:138-153)
//
// Half the multiply-adds of the dense product are skipped with the DST-I
// parity symmetry Q[n-1-p][i] = (-1)^i Q[p][i]:
//   y_{2m}   = sum_{p < n/2} Q[p][2m]   (x_p + x_{n-1-p})  (+ Q[mid][2m] x_mid, odd n)
//   y_{2m+1} = sum_{p < n/2} Q[p][2m+1] (x_p - x_{n-1-p})
// so each parity is an [rows x ceil(n/2)] x [ceil(n/2) x ceil(n/2)] product.
//
// Tile: 32 rows, 8 warps = 4 row groups (m8) x 2 parities.  A fragments are
// the pair sums / differences formed while loading from the shared-memory
// tile; B fragments come from the split table, stored in fragment order
// (one coalesced 256-byte load per DMMA), in shared memory when it fits.
// Outputs overwrite the tile in place (after a CTA barrier) in a
// de-interleaved layout (even outputs, then odd) and the epilogue writes
// rows back coalesced.
#include <math.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "psm_internal.cuh"

namespace psm {

constexpr int kDstRows = 32;
constexpr int kDstThreads = 256;
constexpr int kDstNG = 4;   // n-tiles accumulated at a time

// shared-memory geometry for row length nx
struct DstGeom {
  int ks, nt;   // k-steps of 4 and n-tiles of 8 per parity (padded)
  int odd_off;  // column of output 1 (odd outputs start here; == 8 mod 16)
  int ld;       // tile row stride in doubles (== 4 mod 16: conflict-free A loads)
  size_t qdoubles;
};

__host__ __device__ inline DstGeom dst_geom(int nx) {
  DstGeom g;
  const int h = (nx + 1) / 2;
  g.ks = (h + 3) / 4;
  g.nt = ((h + 7) / 8 + kDstNG - 1) / kDstNG * kDstNG;
  int off = (nx + 1) / 2;
  off += (8 - off % 16 + 16) % 16;
  g.odd_off = off;
  int ld = off + nx / 2;
  if (ld < nx) ld = nx;
  ld += (4 - ld % 16 + 16) % 16;
  g.ld = ld;
  g.qdoubles = (size_t)2 * g.ks * g.nt * 32;
  return g;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct DstRun {
  const PatchDev* patches;
  int p0, p1;        // the run's patches (same nx, ny)
  long long c0;      // cell0 of patch p0
  long long nrows;   // rows of the run (sum of ny*nz)
  int nx;
  const double* qf;  // split table, fragment order [parity][ks][nt][lane]
};

enum { kProRows = 0, kProResidual = 1 };
enum { kEpiStore = 0, kEpiRelaxInPlace = 1, kEpiRelaxInto = 2 };

template <int KSM, int PRO, int EPI, bool QSM>
__global__ void __launch_bounds__(kDstThreads) dst_tile_kernel(const DstRun R, const unsigned char* __restrict__ active,
                                                               const StencilDev st, double omega,
                                                               const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ __align__(16) double dsm[];
  const int nx = R.nx;
  const DstGeom G = dst_geom(nx);
  double* qs = dsm;
  double* tile = dsm + (QSM ? G.qdoubles : 0);
  __shared__ int row_patch[kDstRows], row_k[kDstRows], row_j[kDstRows];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = warp & 3, par = warp >> 2;
  if (QSM)
    for (size_t e = tid; e < G.qdoubles; e += kDstThreads) qs[e] = __ldg(R.qf + e);
  const long long ntiles = (R.nrows + kDstRows - 1) / kDstRows;
  const int half = nx >> 1, mid = (nx & 1) ? half : -1;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long g0 = t * kDstRows;
    if (tid < kDstRows) {
      const long long g = g0 + tid;
      int p = -1, k = 0, j = 0;
      if (g < R.nrows && (PRO == kProResidual || EPI != kEpiStore)) {
        const long long cell = R.c0 + g * nx;
        int lo = R.p0, hi = R.p1 - 1;
        while (lo < hi) {
          const int m = (lo + hi + 1) >> 1;
          if (R.patches[m].cell0 <= cell) lo = m; else hi = m - 1;
        }
        p = lo;
        const long long e = (cell - R.patches[p].cell0) / nx;
        const int ny = R.patches[p].ny;
        k = (int)(e / ny);
        j = (int)(e - (long long)k * ny);
      }
      row_patch[tid] = p;
      row_k[tid] = k;
      row_j[tid] = j;
    }
    __syncthreads();  // row map ready; the previous tile's epilogue is done with the tile
    // ---- prologue: the tile's rows -------------------------------------
    for (int r = warp; r < kDstRows; r += kDstThreads / 32) {
      double* trow = tile + r * G.ld;
      const long long g = g0 + r;
      if (g >= R.nrows) {
        for (int x = lane; x < nx; x += 32) trow[x] = 0.0;
        continue;
      }
      if (PRO == kProRows) {
        const double* src = in + g * nx;
        for (int x = lane; x < nx; x += 32) trow[x] = src[x];
      } else {
        const PatchDev& P = R.patches[row_patch[r]];
        const int k = row_k[r], j = row_j[r];
        const long long px = nx + 2, pxy = px * (P.ny + 2);
        const double* u = P.buf[active[row_patch[r]]] + (k + 1) * pxy + (j + 1) * px + 1;
        const double* f = P.f + ((long long)k * P.ny + j) * nx;
        for (int x = lane; x < nx; x += 32)
          trow[x] = residual7(st, f[x], u[x], u[x - 1], u[x + 1], u[x - px], u[x + px], u[x - pxy], u[x + pxy]);
      }
    }
    __syncthreads();
    // ---- split DST: this warp's 8 rows x one parity ----------------------
    // A fragments (pair sums / differences) for the whole K go to registers,
    // then a barrier: after it no warp reads the tile, so the outputs
    // overwrite it in place
    const double* arow = tile + (8 * mt + (lane >> 2)) * G.ld;
    const double sgn = par ? -1.0 : 1.0;
    double a[KSM];
#pragma unroll
    for (int s = 0; s < KSM; ++s) {
      const int p = 4 * s + (lane & 3);
      double v = 0.0;
      if (p < half) v = arow[p] + sgn * arow[nx - 1 - p];
      else if (p == mid && par == 0) v = arow[p];
      a[s] = v;
    }
    __syncthreads();
    {
      const double* qb = (QSM ? qs : R.qf) + (size_t)par * G.ks * G.nt * 32 + lane;
      // output (row, m = 8 nt + 2 (lane&3) + c) of parity par is x index
      // 2m + par, stored de-interleaved at column par * odd_off + m
      double* orow = tile + (8 * mt + (lane >> 2)) * G.ld + par * G.odd_off;
      const int cnt = par ? half : nx - half;  // outputs of this parity
      for (int n0 = 0; n0 < G.nt; n0 += kDstNG) {
        double acc[kDstNG][2];
#pragma unroll
        for (int q = 0; q < kDstNG; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
        for (int s = 0; s < KSM; ++s) {
          if (s < G.ks) {
#pragma unroll
            for (int q = 0; q < kDstNG; ++q) {
              const size_t o = ((size_t)s * G.nt + n0 + q) * 32;
              const double b = QSM ? qb[o] : __ldg(qb + o);
              dmma884(acc[q][0], acc[q][1], a[s], b);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < kDstNG; ++q) {
          const int m = 8 * (n0 + q) + 2 * (lane & 3);
          if (m < cnt) orow[m] = acc[q][0];
          if (m + 1 < cnt) orow[m + 1] = acc[q][1];
        }
      }
    }
    __syncthreads();
    // ---- epilogue: rows back, x order ------------------------------------
    for (int r = warp; r < kDstRows; r += kDstThreads / 32) {
      const long long g = g0 + r;
      if (g >= R.nrows) continue;
      const double* trow = tile + r * G.ld;
      if (EPI == kEpiStore) {
        double* dst = out + g * nx;
        for (int x = lane; x < nx; x += 32) dst[x] = trow[(x & 1) * G.odd_off + (x >> 1)];
      } else {
        const int p = row_patch[r];
        const PatchDev& P = R.patches[p];
        const int k = row_k[r], j = row_j[r];
        const long long px = nx + 2, pxy = px * (P.ny + 2);
        const long long base = (k + 1) * pxy + (j + 1) * px + 1;
        const int act = active[p];
        if (EPI == kEpiRelaxInPlace) {
          double* u = P.buf[act] + base;
          for (int x = lane; x < nx; x += 32) u[x] = relax(u[x], omega, trow[(x & 1) * G.odd_off + (x >> 1)]);
        } else {
          const double* u = P.buf[act] + base;
          double* v = P.buf[act ^ 1] + base;
          for (int x = lane; x < nx; x += 32) {
            const double nv = relax(u[x], omega, trow[(x & 1) * G.odd_off + (x >> 1)]);
            v[x] = nv;
            if (x == 0) v[-1] = -nv;
            if (x == nx - 1) v[nx] = -nv;
          }
        }
      }
    }
  }
}

// Plane GS modal recurrence (symmetric y faces), all stages in one launch.
// With rhat = Q r_pre (the transformed pre-sweep residual of every plane) the
// stage-k residual is r_pre(k) - zm omega x(k-1) at the same (x, y), so in the
// transformed domain every (patch, x-mode) line is an independent chain over
// k:  v = rhat(k) - zm omega xhat(k-1);  xhat(k) = T_mode^{-1} v  (Thomas along
// y).  Two threads per chain (top / bottom halves of y meeting in an exact
// 2x2 system, as plane_modal_thomas2_kernel); each thread re-reads only the
// xhat(k-1) values it wrote itself.  In place in `buf` (cell-major, cell0).
__global__ void __launch_bounds__(128) plane_gs_chain_kernel(const PlaneFac* __restrict__ F,
                                                             const PatchDev* __restrict__ patches, int p0,
                                                             long long nlines, int maxnz, double czw,
                                                             double* __restrict__ buf) {
  constexpr int B = 16;
  const int nx = F->nx, ny = F->ny, m = ny / 2;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = t < 2 * nlines;  // whole warps stay for the shuffles
  const long long line = in ? t >> 1 : 0;
  const int bot = (int)(t & 1);
  const int pl = (int)(line / nx);
  const int i = (int)(line - (long long)pl * nx);
  const PatchDev& P = patches[p0 + pl];
  const int nz = in ? P.nz : 0;
  const long long plane_cells = (long long)nx * ny;
  const double* cp = F->cp + i;
  const double* invm = F->invm + i;
  const double lo = F->fy_lo;
  const int len = bot ? ny - m : m;
  const long long j0 = bot ? ny - 1 : 0, dj = bot ? -nx : nx;
  const double c_own = len > 0 ? __ldg(cp + (long long)(len - 1) * nx) : 0.0;
  for (int k = 0; k < maxnz; ++k) {
    const bool act = k < nz;
    double* b = buf + P.cell0 + (long long)k * plane_cells + i;
    const double* bp = b - plane_cells;
    if (act && i == 0 && bot == 0 && k + 1 < nz && ((plane_cells * 8) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(b + plane_cells) & 15) == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b + plane_cells),
                   "r"((unsigned)(plane_cells * 8))
                   : "memory");
    double prev = 0.0;
    if (act) {
      int jj = 0;
      for (; jj + B <= len; jj += B) {
        double v[B], mm[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
          v[q] = b[j0 * nx + (jj + q) * dj];
          if (k > 0) v[q] = fma(-czw, bp[j0 * nx + (jj + q) * dj], v[q]);
          mm[q] = __ldg(invm + (long long)(jj + q) * nx);
        }
#pragma unroll
        for (int q = 0; q < B; ++q) {
          prev = fma(-lo, prev, v[q]) * mm[q];
          b[j0 * nx + (jj + q) * dj] = prev;
        }
      }
      for (; jj < len; ++jj) {
        double v = b[j0 * nx + jj * dj];
        if (k > 0) v = fma(-czw, bp[j0 * nx + jj * dj], v);
        prev = fma(-lo, prev, v) * invm[(long long)jj * nx];
        b[j0 * nx + jj * dj] = prev;
      }
    }
    const double y_oth = __shfl_xor_sync(0xffffffffu, prev, 1);
    const double c_oth = __shfl_xor_sync(0xffffffffu, c_own, 1);
    if (!act || len == 0) continue;
    const double yT = bot ? y_oth : prev, yB = bot ? prev : y_oth;
    const double cT = bot ? c_oth : c_own, cB = bot ? c_own : c_oth;
    const double xT = (yT - cT * yB) / (1.0 - cT * cB);
    double next = bot ? yB - cB * xT : xT;
    b[j0 * nx + (len - 1) * dj] = next;
    int jj = len - 2;
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
}

// ---------------------------------------------------------------- host side
int dst_max_nx() { return 512; }

// Fragment-ordered split table of the DST-I basis Q (row-major nx x nx):
// entry [par][ks][nt][lane] = Q[p][2 m + par], p = 4 ks + lane % 4,
// m = 8 nt + lane / 4; zero where p or the output index leaves its range
// (even outputs use p < ceil(nx/2), odd ones p < floor(nx/2)).
void dst_split_table(const std::vector<double>& Q, int nx, std::vector<double>& out) {
  const DstGeom G = dst_geom(nx);
  out.assign(G.qdoubles, 0.0);
  const int half = nx / 2, heven = (nx + 1) / 2;
  for (int par = 0; par < 2; ++par)
    for (int ks = 0; ks < G.ks; ++ks)
      for (int nt = 0; nt < G.nt; ++nt)
        for (int lane = 0; lane < 32; ++lane) {
          const int p = 4 * ks + (lane & 3), m = 8 * nt + (lane >> 2), i = 2 * m + par;
          const int plim = par ? half : heven;
          if (p < plim && i < nx)
            out[(((size_t)par * G.ks + ks) * G.nt + nt) * 32 + lane] = Q[(size_t)p * nx + i];
        }
}

size_t dst_table_doubles(int nx) { return dst_geom(nx).qdoubles; }

template <int KSM, int PRO, int EPI, bool QSM>
static cudaError_t dst_launch_t(const DstRun& R, const unsigned char* active, const StencilDev& st, double omega,
                                const double* in, double* out, cudaStream_t s) {
  const DstGeom G = dst_geom(R.nx);
  const size_t smem = ((QSM ? G.qdoubles : 0) + (size_t)kDstRows * G.ld) * sizeof(double);
  auto kern = dst_tile_kernel<KSM, PRO, EPI, QSM>;
  // the opt-in is per device and this size depends on nx: set it per launch
  // (host-side, no stream work)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDstThreads, smem);
  const long long ntiles = (R.nrows + kDstRows - 1) / kDstRows;
  const long long grid = std::max<long long>(1, std::min<long long>(ntiles, (long long)std::max(occ, 1) * sms));
  kern<<<(unsigned)grid, kDstThreads, smem, s>>>(R, active, st, omega, in, out);
  return cudaGetLastError();
}

template <int PRO, int EPI>
static cudaError_t dst_launch_k(const DstRun& R, const unsigned char* active, const StencilDev& st, double omega,
                                const double* in, double* out, cudaStream_t s) {
  const DstGeom G = dst_geom(R.nx);
  // the split table in shared memory when two CTAs per SM still fit
  const bool qsm = (G.qdoubles + (size_t)kDstRows * G.ld) * sizeof(double) <= 112 * 1024;
#define PSM_DST(K_)                                                                        \
  return qsm ? dst_launch_t<K_, PRO, EPI, true>(R, active, st, omega, in, out, s)           \
             : dst_launch_t<K_, PRO, EPI, false>(R, active, st, omega, in, out, s)
  if (G.ks <= 8) PSM_DST(8);
  if (G.ks <= 16) PSM_DST(16);
  if (G.ks <= 32) PSM_DST(32);
  PSM_DST(64);
#undef PSM_DST
}

// rows -> transformed rows (or fused residual / relax, see the enums)
cudaError_t launch_dst_rows(int pro, int epi, const PatchDev* patches, int p0, int p1, long long c0, long long nrows,
                            int nx, const double* qf, const unsigned char* active, const StencilDev& st,
                            double omega, const double* in, double* out, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  if (nx > dst_max_nx()) return cudaErrorInvalidValue;
  DstRun R{patches, p0, p1, c0, nrows, nx, qf};
  if (pro == kProRows && epi == kEpiStore) return dst_launch_k<kProRows, kEpiStore>(R, active, st, omega, in, out, s);
  if (pro == kProResidual && epi == kEpiStore)
    return dst_launch_k<kProResidual, kEpiStore>(R, active, st, omega, in, out, s);
  if (pro == kProRows && epi == kEpiRelaxInPlace)
    return dst_launch_k<kProRows, kEpiRelaxInPlace>(R, active, st, omega, in, out, s);
  if (pro == kProRows && epi == kEpiRelaxInto)
    return dst_launch_k<kProRows, kEpiRelaxInto>(R, active, st, omega, in, out, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_plane_gs_chain(const PlaneFac* d_fac, int nx, const PatchDev* patches, int p0, int np, int maxnz,
                                  double czw, double* buf, cudaStream_t s) {
  const long long nlines = (long long)np * nx;
  if (nlines == 0) return cudaSuccess;
  plane_gs_chain_kernel<<<(unsigned)((2 * nlines + 127) / 128), 128, 0, s>>>(d_fac, patches, p0, nlines, maxnz, czw,
                                                                             buf);
  return cudaGetLastError();
}

}  // namespace psm
