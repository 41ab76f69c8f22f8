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
#include <stdlib.h>

#include <atomic>
#include <vector>

#include "psm_async.cuh"
#include "psm_internal.cuh"

namespace psm {

constexpr int kDstRows = 32;
constexpr int kDstThreads = 256;
constexpr int kDstNG = 4;   // n-tile granularity of the split table (the kernel accumulates NG = 4 or 8 at a time)

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

enum { kProRows = 0 };
enum { kEpiStore = 0, kEpiRelaxInPlace = 1, kEpiRelaxInto = 2 };

// shared-memory layout of one launch
struct DstSmem {
  int ldu;          // u-row stride (EPI relax): [x = -1 .. nx], even
  int nstage;       // 1 or 2 (double-buffered input)
  size_t q, stage, ustage;  // doubles
  __host__ __device__ size_t total(bool relax) const {
    return q + nstage * (stage + (relax ? ustage : 0));
  }
};
// relax: stage the u rows too (EPI relax; else the epilogue reads u directly)
__host__ __device__ inline DstSmem dst_smem(int nx, bool qsm, bool relax, int nstage) {
  const DstGeom G = dst_geom(nx);
  DstSmem m;
  m.ldu = (nx + 2 + 1) / 2 * 2;
  m.nstage = nstage;
  m.q = qsm ? G.qdoubles : 0;
  m.stage = (size_t)kDstRows * G.ld;
  m.ustage = relax ? (size_t)kDstRows * m.ldu : 0;
  return m;
}

// Warp-specialised pipeline: warp 8 produces, warps 0-7 consume.  The
// producer maps each tile row to its patch, plane and row and streams the
// rows in with the TMA engine (one bulk copy per row into a padded shared
// row; with EPI relax also the row's u values, ghosts included) into a ring
// of NST stages, throttled by the consumers' "empty" arrivals; rows that are
// not 16-byte aligned (odd nx or odd workspace offset) it loads itself.  The
// consumers run split-DST MMA and epilogue per tile, synchronising among
// themselves only (named barrier 1), so loads for later tiles overlap them.
constexpr int kDstConsumers = 256;
constexpr int kDstAllThreads = kDstConsumers + 32;
constexpr int kDstStages = 3;

template <int KSM, int EPI, bool QSM, bool BULK, int NG>
__global__ void __launch_bounds__(kDstAllThreads, 1) dst_tile_kernel(const DstRun R, const unsigned char* __restrict__ active,
                                                                     double omega, const double* __restrict__ in,
                                                                     double* __restrict__ out, int nstage, int ustaged,
                                                                     long long rows_per_patch, int pingpong) {
  constexpr bool RELAX = EPI != kEpiStore;
  extern __shared__ __align__(16) double dsm[];
  const int nx = R.nx;
  const DstGeom G = dst_geom(nx);
  const DstSmem M = dst_smem(nx, QSM, RELAX && ustaged, nstage);
  double* qs = dsm;
  double* stage0 = dsm + M.q;
  __shared__ uint64_t full[kDstStages], empty[kDstStages];
  __shared__ int row_patch[kDstStages][kDstRows];
  __shared__ long long row_base[kDstStages][kDstRows];  // u index of (x = 0, j, k) in the row's patch buffer
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long ntiles = (R.nrows + kDstRows - 1) / kDstRows;
  const int half = nx >> 1, mid = (nx & 1) ? half : -1;
  auto stage = [&](int s) { return stage0 + (size_t)s * (M.stage + M.ustage); };
  auto ustage = [&](int s) { return stage0 + (size_t)s * (M.stage + M.ustage) + M.stage; };

  if (tid == 0) {
    for (int i = 0; i < kDstStages; ++i) {
      async::bar_init(&full[i], 1);
      async::bar_init(&empty[i], 1);
    }
    async::bar_fence_init();
  }
  if (QSM)
    for (size_t e = tid; e < G.qdoubles; e += kDstAllThreads) qs[e] = __ldg(R.qf + e);
  __syncthreads();

  if (warp == kDstConsumers / 32) {
    // ============================ producer ==================================
    int it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % nstage;
      if (it >= nstage) async::bar_wait(&empty[s], ((it / nstage) - 1) & 1);
      const long long g = t * kDstRows + lane;
      const bool valid = g < R.nrows;
      const int nvalid = (int)min((long long)kDstRows, R.nrows - t * kDstRows);
      int p = 0;
      long long ub = 0;
      if (RELAX && valid) {
        if (rows_per_patch > 0) {
          p = R.p0 + (int)(g / rows_per_patch);
        } else {
          const long long cell = R.c0 + g * nx;
          int lo = R.p0, hi = R.p1 - 1;
          while (lo < hi) {
            const int m = (lo + hi + 1) >> 1;
            if (R.patches[m].cell0 <= cell) lo = m; else hi = m - 1;
          }
          p = lo;
        }
        const PatchDev& P = R.patches[p];
        const long long e = (R.c0 + g * nx - P.cell0) / nx;
        const int k = (int)(e / P.ny), j = (int)(e - (long long)k * P.ny);
        ub = (long long)(k + 1) * (nx + 2) * (P.ny + 2) + (long long)(j + 1) * (nx + 2) + 1;
        row_patch[s][lane] = p;
        row_base[s][lane] = ub;
      }
      const bool us = RELAX && ustaged;
      if (BULK) {
        if (lane == 0)
          async::bar_expect(&full[s], (uint32_t)nvalid * ((uint32_t)nx * 8u + (us ? (uint32_t)(nx + 2) * 8u : 0u)));
        __syncwarp();
        if (valid) {
          async::bulk_g2s(stage(s) + lane * G.ld, in + g * nx, (uint32_t)nx * 8u, &full[s]);
          if (us) {
            const double* u = R.patches[p].buf[active[p]] + ub - 1;  // x = -1: even offset, 16-B aligned
            async::bulk_g2s(ustage(s) + lane * M.ldu, u, (uint32_t)(nx + 2) * 8u, &full[s]);
          }
        }
      } else {
        __syncwarp();
        for (int r = 0; r < nvalid; ++r) {
          const double* src = in + (t * kDstRows + r) * nx;
          for (int x = lane; x < nx; x += 32) stage(s)[r * G.ld + x] = src[x];
          if (us) {
            const int pr = row_patch[s][r];
            const double* u = R.patches[pr].buf[active[pr]] + row_base[s][r] - 1;
            for (int x = lane; x < nx + 2; x += 32) ustage(s)[r * M.ldu + x] = u[x];
          }
        }
        __syncwarp();
        if (lane == 0) async::bar_arrive(&full[s]);
      }
    }
    return;
  }

  // ============================== consumers ===================================
  // Two groups of four warps take alternate tiles (ping-pong), so one
  // group's A-load and epilogue phases overlap the other's MMA; warp w of a
  // group owns the 8-row m-tile w of its tile, both parities.
  // (PP: ping-pong, both parities per warp; large K keeps one group of eight
  // warps, one parity each, to bound the A-fragment registers; one stage
  // also means one group)
  constexpr bool PPK = KSM <= 16;
  const bool PP = PPK && pingpong && nstage >= 2;
  const int ngrp = PP ? 2 : 1;
  const int kGroupThreads = kDstConsumers / ngrp;
  const int grp = PP ? warp >> 2 : 0;
  const int mt = warp & 3;
  const int par_lo = PP ? 0 : warp >> 2;
  const int gtid = tid & (kGroupThreads - 1);
  const int bar_id = 1 + grp;
  int it = grp;
  for (long long t = blockIdx.x + (long long)grp * gridDim.x; t < ntiles; t += (long long)ngrp * gridDim.x,
                 it += ngrp) {
    const int s = it % nstage;
    async::bar_wait(&full[s], (it / nstage) & 1);
    double* st = stage(s);
    const int nvalid = (int)min((long long)kDstRows, R.nrows - t * kDstRows);
    // ---- split DST: this warp's 8 rows, both parities ---------------------
    // A fragments (pair sums and differences) for the whole K go to
    // registers; after the group barrier no warp of the group reads the rows,
    // so outputs overwrite them in place
    const int arow_i = 8 * mt + (lane >> 2);
    const double* arow = st + arow_i * G.ld;
    const bool arow_ok = arow_i < nvalid;
    constexpr int NPA = PPK ? 2 : 1;  // parities whose A fragments this warp holds
    double a[NPA][KSM];
#pragma unroll
    for (int q = 0; q < KSM; ++q) {
      const int p = 4 * q + (lane & 3);
      double e = 0.0, o = 0.0;
      if (arow_ok) {
        if (p < half) {
          const double l = arow[p], r = arow[nx - 1 - p];
          e = l + r;
          o = l - r;
        } else if (p == mid) {
          e = arow[p];
        }
      }
      if (PPK) {
        a[0][q] = e;
        a[NPA - 1][q] = o;
      } else {
        a[0][q] = par_lo ? o : e;
      }
    }
    async::named_sync(bar_id, kGroupThreads);
#pragma unroll
    for (int ai = 0; ai < NPA; ++ai) {  // compile-time index into a[]
      // PPK: a[0] even, a[1] odd; with one group (PP false) a warp runs only
      // its own parity par_lo, whose fragments a[par_lo] (PPK) or a[0] hold
      if (PPK && !PP && ai != par_lo) continue;
      const int par = PPK ? ai : par_lo;
      const double* qb = (QSM ? qs : R.qf) + (size_t)par * G.ks * G.nt * 32 + lane;
      // output (row, m = 8 nt + 2 (lane&3) + c) of parity par is x = 2 m + par
      double* orow = st + arow_i * G.ld + par;
      const int cnt = par ? half : nx - half;  // outputs of this parity
      for (int n0 = 0; n0 < G.nt; n0 += NG) {
        double acc[NG][2];
#pragma unroll
        for (int q = 0; q < NG; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KSM; ++ks) {
          if (ks < G.ks) {
#pragma unroll
            for (int q = 0; q < NG; ++q) {
              const size_t o = ((size_t)ks * G.nt + n0 + q) * 32;
              const double bb = QSM ? qb[o] : __ldg(qb + o);
              dmma884(acc[q][0], acc[q][1], a[ai][ks], bb);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const int m = 8 * (n0 + q) + 2 * (lane & 3);
          if (m < cnt) orow[2 * m] = acc[q][0];
          if (m + 1 < cnt) orow[2 * m + 2] = acc[q][1];
        }
      }
    }
    async::named_sync(bar_id, kGroupThreads);
    // ---- epilogue: coalesced row stores ---------------------------------
    for (int r = PP ? mt : warp; r < nvalid; r += PP ? 4 : 8) {
      const double* trow = st + r * G.ld;
      const long long g = t * kDstRows + r;
      if (EPI == kEpiStore) {
        double* dst = out + g * nx;
        for (int x = lane; x < nx; x += 32) dst[x] = trow[x];
      } else {
        const int p = row_patch[s][r];
        const PatchDev& P = R.patches[p];
        const int act = active[p];
        const double* uo = ustaged ? ustage(s) + r * M.ldu + 1 : P.buf[act] + row_base[s][r];  // x = 0
        if (EPI == kEpiRelaxInPlace) {
          double* u = P.buf[act] + row_base[s][r];
          for (int x = lane; x < nx; x += 32) u[x] = relax(uo[x], omega, trow[x]);
        } else {
          double* v = P.buf[act ^ 1] + row_base[s][r];
          for (int x = lane; x < nx; x += 32) {
            const double nv = relax(uo[x], omega, trow[x]);
            v[x] = nv;
            if (x == 0) v[-1] = -nv;
            if (x == nx - 1) v[nx] = -nv;
          }
        }
      }
    }
    async::named_sync(bar_id, kGroupThreads);  // the group is done with stage s
    if (gtid == 0) async::bar_arrive(&empty[s]);
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

// The same chains, each thread keeping its half-line's xhat(k-1) on chip
// across the stages (a private shared-memory column: conflict-free [jj][tid]
// layout) while plane k+1's transformed residuals stream into shared memory
// (cp.async, double-buffered) during plane k's solve; the Thomas factors
// come from shared memory too (rows jj < nj, then the converged row nj: the
// tables are bitwise constant from there on, checked on the host).  Global
// traffic is one read and one write of every value.  One CTA = 64 modes of
// one patch, two threads per mode.
template <int MPC>  // modes per CTA (two threads each)
__global__ void __launch_bounds__(2 * MPC) plane_gs_chain_smem_kernel(const PlaneFac* __restrict__ F,
                                                                     const PatchDev* __restrict__ patches, int p0,
                                                                     int cpp, int maxnz, double czw,
                                                                     double* __restrict__ buf, int nj) {
  extern __shared__ __align__(16) double csm[];
  const int nx = F->nx, ny = F->ny, m = ny / 2, hmax = ny - m;
  const int tid = threadIdx.x, q = tid >> 1, bot = tid & 1;
  const int pl = blockIdx.x / cpp, i0 = (blockIdx.x - pl * cpp) * MPC;
  const int i = i0 + q;
  const bool valid = i < nx;
  const PatchDev& P = patches[p0 + pl];
  const int nz = P.nz;
  constexpr int T = 2 * MPC;
  double* stg = csm;                               // [2][ny][MPC] transformed residuals
  double* X = stg + 2 * (size_t)ny * MPC + tid;    // [hmax][T] this thread's column
  double* fin = csm + 2 * (size_t)ny * MPC + (size_t)hmax * T;  // [nj+1][MPC] 1/m
  double* fcp = fin + (size_t)(nj + 1) * MPC;                    // [nj+1][MPC] c'
  for (int e = tid; e < (nj + 1) * MPC; e += T) {
    const int jj = e / MPC, ii = i0 + (e % MPC);
    const long long o = (long long)jj * nx + ii;
    fin[e] = ii < nx ? F->invm[o] : 1.0;
    fcp[e] = ii < nx ? F->cp[o] : 0.0;
  }
  const double lo = F->fy_lo;
  const int len = bot ? ny - m : m;
  const long long plane_cells = (long long)nx * ny;
  // this thread's rows: jj -> row0 + jj * drow
  const int row0 = bot ? ny - 1 : 0, drow = bot ? -1 : 1;
  auto load = [&](int k, int sidx) {
    if (valid && k < nz) {
      const double* src = buf + P.cell0 + (long long)k * plane_cells + i + (long long)row0 * nx;
      double* dst = stg + (size_t)sidx * ny * MPC + q + row0 * MPC;
      for (int jj = 0; jj < len; ++jj) async::cp8(dst + jj * drow * MPC, src + (long long)jj * drow * nx);
    }
    async::cp_commit();
  };
  __syncthreads();
  for (int jj = 0; jj < len; ++jj) X[jj * T] = 0.0;
  const double* finq = fin + q;
  const double* fcpq = fcp + q;
  const double c_own = len > 0 ? fcpq[min(len - 1, nj) * MPC] : 0.0;
  load(0, 0);
  for (int k = 0; k < maxnz; ++k) {
    load(k + 1, (k + 1) & 1);
    async::cp_wait<1>();  // plane k (this thread's own copies) landed
    const double* S = stg + (size_t)(k & 1) * ny * MPC + q + row0 * MPC;
    const bool act = valid && k < nz;
    const double cz = k > 0 ? czw : 0.0;  // xhat(-1) = 0: X starts zeroed
    double prev = 0.0;
    if (act) {
      // rows below nj use their own factors, the rest the converged ones
      const int jn = min(len, nj);
      const int sstep = drow * MPC;
      const double* sp = S;
      double* xp = X;
      const double* fp = finq;
#pragma unroll 4
      for (int jj = 0; jj < jn; ++jj, sp += sstep, xp += T, fp += MPC) {
        const double v = fma(-cz, *xp, *sp);
        prev = fma(-lo, prev, v) * *fp;
        *xp = prev;
      }
      const double finf = finq[nj * MPC];
#pragma unroll 8
      for (int jj = jn; jj < len; ++jj, sp += sstep, xp += T) {
        const double v = fma(-cz, *xp, *sp);
        prev = fma(-lo, prev, v) * finf;
        *xp = prev;
      }
    }
    const double y_oth = __shfl_xor_sync(0xffffffffu, prev, 1);
    const double c_oth = __shfl_xor_sync(0xffffffffu, c_own, 1);
    if (act && len > 0) {
      const double yT = bot ? y_oth : prev, yB = bot ? prev : y_oth;
      const double cT = bot ? c_oth : c_own, cB = bot ? c_own : c_oth;
      const double xT = (yT - cT * yB) / (1.0 - cT * cB);
      double next = bot ? yB - cB * xT : xT;
      const long long dstep = (long long)drow * nx;
      double* dp = buf + P.cell0 + (long long)k * plane_cells + i + (long long)row0 * nx + (len - 1) * dstep;
      double* xp = X + (len - 1) * T;
      *xp = next;
      *dp = next;
      int jj = len - 2;
      const double cinf = fcpq[nj * MPC];
#pragma unroll 8
      for (; jj >= nj; --jj) {
        xp -= T;
        dp -= dstep;
        next = fma(-cinf, next, *xp);
        *xp = next;
        *dp = next;
      }
      const double* fp = fcpq + jj * MPC;
#pragma unroll 4
      for (; jj >= 0; --jj, fp -= MPC) {
        xp -= T;
        dp -= dstep;
        next = fma(-*fp, next, *xp);
        *xp = next;
        *dp = next;
      }
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

template <int KSM, int EPI, bool QSM, bool BULK, int NG>
static cudaError_t dst_launch_t(const DstRun& R, const unsigned char* active, double omega, const double* in,
                                double* out, int nstage, int ustaged, long long rpp, int pp, cudaStream_t s) {
  const bool us = EPI != kEpiStore && ustaged;
  const DstSmem M = dst_smem(R.nx, QSM, us, nstage);
  const size_t smem = M.total(us) * sizeof(double);
  auto kern = dst_tile_kernel<KSM, EPI, QSM, BULK, NG>;
  // the opt-in is per device and this size depends on nx: set it per launch
  // (host-side, no stream work)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kDstAllThreads, smem);
  const long long ntiles = (R.nrows + kDstRows - 1) / kDstRows;
  const long long grid = std::max<long long>(1, std::min<long long>(ntiles, (long long)std::max(occ, 1) * sms));
  kern<<<(unsigned)grid, kDstAllThreads, smem, s>>>(R, active, omega, in, out, nstage, ustaged, rpp, pp);
  return cudaGetLastError();
}

template <int EPI>
static cudaError_t dst_launch_k(const DstRun& R, const unsigned char* active, double omega, const double* in,
                                double* out, long long rpp, cudaStream_t s) {
  const DstGeom G = dst_geom(R.nx);
  constexpr bool relax = EPI != kEpiStore;
  const size_t cap = 227 * 1024 - 2048;  // opt-in limit less the static shared memory
  // preference: split table on chip, three then two input stages, staged u
  // rows; dropped in the reverse order until the layout fits
  // Layout preference.  Store epilogue: split table on chip, three stages
  // (two ping-pong consumer groups plus one stage loading).  Relax
  // epilogues also stage the u rows (their direct loads are latency-bound):
  // table on chip, two stages, one consumer group (measured at C4: 1.14 ms,
  // against 1.29 with two groups on two stages and 2.15 with the table read
  // through L1/L2 to make room for three stages).
  bool qsm = true;
  int nstage = kDstStages, ustaged = relax ? 1 : 0, pp = 1;
  if (relax) {
    nstage = 2;
    pp = 0;
  }
  auto fits = [&] { return dst_smem(R.nx, qsm, ustaged, nstage).total(ustaged) * 8 <= cap; };
  if (!fits()) nstage = 2;
  if (!fits()) qsm = false;
  if (!fits()) nstage = kDstStages;
  if (!fits()) nstage = 2;
  if (!fits()) ustaged = 0;
  if (!fits()) nstage = 1;
  if (!fits()) return cudaErrorInvalidValue;
  // bulk copies need 16-byte aligned rows: even nx and an even workspace offset
  const bool bulk = (R.nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
  // eight independent DMMA accumulator chains per warp when the n-tiles
  // come in eights, else four
  const bool ng8 = G.nt % 8 == 0;
#define PSM_DST_NG(K_, Q_, B_) \
  return ng8 ? dst_launch_t<K_, EPI, Q_, B_, 8>(R, active, omega, in, out, nstage, ustaged, rpp, pp, s) \
             : dst_launch_t<K_, EPI, Q_, B_, 4>(R, active, omega, in, out, nstage, ustaged, rpp, pp, s)
#define PSM_DST(K_)                        \
  if (qsm) {                               \
    if (bulk) PSM_DST_NG(K_, true, true);  \
    PSM_DST_NG(K_, true, false);           \
  }                                        \
  if (bulk) PSM_DST_NG(K_, false, true);   \
  PSM_DST_NG(K_, false, false)
  if (G.ks <= 8) { PSM_DST(8); }
  if (G.ks <= 16) { PSM_DST(16); }
  if (G.ks <= 32) { PSM_DST(32); }
  PSM_DST(64);
#undef PSM_DST
#undef PSM_DST_NG
}

// rows -> transformed rows (EPI store), or relaxed into the patches
// rows_per_patch: ny * nz when every patch of the run has the same nz (row
// -> patch by division), else 0 (binary search over cell0)
cudaError_t launch_dst_rows(int epi, const PatchDev* patches, int p0, int p1, long long c0, long long nrows, int nx,
                            const double* qf, const unsigned char* active, double omega, const double* in,
                            double* out, long long rows_per_patch, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  if (nx > dst_max_nx()) return cudaErrorInvalidValue;
  DstRun R{patches, p0, p1, c0, nrows, nx, qf};
  if (epi == kEpiStore) return dst_launch_k<kEpiStore>(R, active, omega, in, out, rows_per_patch, s);
  if (epi == kEpiRelaxInPlace) return dst_launch_k<kEpiRelaxInPlace>(R, active, omega, in, out, rows_per_patch, s);
  if (epi == kEpiRelaxInto) return dst_launch_k<kEpiRelaxInto>(R, active, omega, in, out, rows_per_patch, s);
  return cudaErrorInvalidValue;
}

template <int MPC>
static size_t chain_smem_bytes(int ny, int nj) {
  return (2 * (size_t)ny * MPC + (size_t)(ny - ny / 2) * 2 * MPC + 2 * (size_t)(nj + 1) * MPC) * sizeof(double);
}

template <int MPC>
static cudaError_t chain_smem_launch(const PlaneFac* d_fac, int nx, int ny, const PatchDev* patches, int p0, int np,
                                    int maxnz, double czw, double* buf, int nj, cudaStream_t s) {
  const int cpp = (nx + MPC - 1) / MPC;
  const size_t smem = chain_smem_bytes<MPC>(ny, nj);
  auto kern = plane_gs_chain_smem_kernel<MPC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(np * cpp), 2 * MPC, smem, s>>>(d_fac, patches, p0, cpp, maxnz, czw, buf, nj);
  return cudaGetLastError();
}

// nj: rows from which the modal Thomas tables are bitwise constant (host
// check in psm_plane_build), or -1 when they are not within the limit
cudaError_t launch_plane_gs_chain(const PlaneFac* d_fac, int nx, int ny, int nj, const PatchDev* patches, int p0,
                                  int np, int maxnz, double czw, double* buf, cudaStream_t s) {
  const long long nlines = (long long)np * nx;
  if (nlines == 0) return cudaSuccess;
  // on-chip chains while their working set fits one SM: 32 modes per CTA
  // (two CTAs per SM at ny = 128), 64 when more CTAs would not fit anyway
  if (nj >= 0 && !getenv("PSM_PLANE_CHAIN_GLOBAL")) {
    const char* e = getenv("PSM_PLANE_CHAIN_MPC");
    const int mpc = e ? atoi(e) : 32;
    if (mpc == 32 && chain_smem_bytes<32>(ny, nj) <= 110 * 1024)
      return chain_smem_launch<32>(d_fac, nx, ny, patches, p0, np, maxnz, czw, buf, nj, s);
    if (chain_smem_bytes<64>(ny, nj) <= 220 * 1024)
      return chain_smem_launch<64>(d_fac, nx, ny, patches, p0, np, maxnz, czw, buf, nj, s);
  }
  plane_gs_chain_kernel<<<(unsigned)((2 * nlines + 127) / 128), 128, 0, s>>>(d_fac, patches, p0, nlines, maxnz, czw,
                                                                             buf);
  return cudaGetLastError();
}

}  // namespace psm
