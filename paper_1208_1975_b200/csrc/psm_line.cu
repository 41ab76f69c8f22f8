// Line-block (x-line) kernels: block Jacobi sweep, residual norm, and the
// generic full-Thomas fallback.
//
// Replaces, for block_dims (>=nx, 1, 1):
//   smoother._jacobi_step + work()        smoother.py:138-153
//   stencil.block_residual                 stencil.py:93-112
//   smoother.block_update -> matvec        smoother.py:90-93, blocklinalg.py:90-105
//   smoother.residual_norm (partials)      smoother.py:96-109
//
// Tile kernel structure (one CTA = R consecutive x-lines of one z-plane):
//   A  coalesced: r = f - A u for every cell (reference operation order),
//      x-neighbours by warp shuffle, y/z-neighbours straight from L2; r goes
//      to shared memory (one pad double per 32 so segment reads are
//      conflict-free) and r^2 into the tile's norm partial.
//   B  one lane per 32-cell segment: Thomas on the segment with constant
//      factors, result y back to smem, segment end values to an exchange row.
//   C  coalesced: interface 2x2 solves (redundantly per cell, broadcast smem
//      reads), spike correction, v = u + omega*x, store v and the physical
//      x-face ghosts of v (grid.py:321-322 rule, fused).
#include "psm_internal.cuh"

namespace psm {

constexpr int kMaxE = 8;  // cells per thread per tile

template <int MODE>  // 0: residual partials only, 1: Jacobi sweep, 2: residual to rbuf (plane path)
__global__ void __launch_bounds__(256, 2) line_tile_kernel(const PatchDev* __restrict__ patches, int npatch,
                                                        const unsigned char* __restrict__ active, StencilDev st,
                                                        double omega, double* __restrict__ partials,
                                                        double* __restrict__ rbuf, long long tile_base) {
  extern __shared__ double sm[];
  __shared__ double wsum[32];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31;
  const long long tile = tile_base + blockIdx.x;
  const int pi = find_patch(patches, npatch, tile);
  const PatchDev& P = patches[pi];
  const int nx = P.nx, ny = P.ny;
  const long long cell0 = P.cell0;
  const LineFac* __restrict__ L = P.lf;
  int k, j0, R;
  tile_coords(P, tile, k, j0, R);
  const long long px = nx + 2, pxy = px * (ny + 2);
  const int act = active[pi];
  const double* __restrict__ u = P.buf[act];
  double* __restrict__ v = P.buf[act ^ 1];
  const double* __restrict__ f = P.f;
  const long long ubase = (long long)(k + 1) * pxy + (long long)(j0 + 1) * px + 1;  // u(0, j0, k)
  const long long fbase = ((long long)k * ny + j0) * nx;
  const int nelem = R * nx;
  const int RS = row_stride(nx);
  double* rs = sm;

  double ssq = 0.0;
  double ucen[kMaxE];
#pragma unroll
  for (int h = 0; h < kMaxE; h += 4) {
    if (h * T >= nelem) break;
    double c[4], ym[4], yp[4], zm[4], zp[4], fv[4];
    int xr[4], rr[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = (h + q) * T + tid;
      ok[q] = e < nelem;
      rr[q] = ok[q] ? e / nx : 0;
      xr[q] = ok[q] ? e - rr[q] * nx : 0;
      const long long iu = ubase + (long long)rr[q] * px + xr[q];
      if (ok[q]) {
        c[q] = __ldg(u + iu);
        ym[q] = __ldg(u + iu - px);
        yp[q] = __ldg(u + iu + px);
        zm[q] = __ldg(u + iu - pxy);
        zp[q] = __ldg(u + iu + pxy);
        fv[q] = __ldg(f + fbase + e);
      } else {
        c[q] = ym[q] = yp[q] = zm[q] = zp[q] = fv[q] = 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double xl = __shfl_up_sync(0xffffffffu, c[q], 1);
      double xp_ = __shfl_down_sync(0xffffffffu, c[q], 1);
      ucen[h + q] = c[q];
      if (ok[q]) {
        const long long iu = ubase + (long long)rr[q] * px + xr[q];
        if (lane == 0 || xr[q] == 0) xl = __ldg(u + iu - 1);
        if (lane == 31 || xr[q] == nx - 1) xp_ = __ldg(u + iu + 1);
        const double res = residual7(st, fv[q], c[q], xl, xp_, ym[q], yp[q], zm[q], zp[q]);
        ssq = fma(res, res, ssq);
        if (MODE == 1) rs[rr[q] * RS + xr[q] + (xr[q] >> 5)] = res;
        if (MODE == 2) rbuf[cell0 + fbase + (h + q) * T + tid] = res;
      }
    }
  }
  // deterministic tile partial of sum(r^2): fixed shuffle tree, warps in order
#pragma unroll
  for (int o = 16; o; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
  if (lane == 0) wsum[tid >> 5] = ssq;
  __syncthreads();
  if (tid == 0 && partials) {
    double s = 0.0;
    for (int w = 0; w < (T >> 5); ++w) s += wsum[w];
    partials[tile] = s;
  }
  if (MODE != 1) return;

  // ---- B: local segment solves -------------------------------------------
  const int nseg = L->nseg, tail = L->tail;
  double* ex = sm + R * RS;
  const double lo = L->lo;
  for (int ln = tid; ln < R * nseg; ln += T) {
    const int r = ln / nseg, s = ln - r * nseg;
    const int len = (s == nseg - 1) ? tail : kSeg;
    double* seg = rs + r * RS + s * (kSeg + 1);
    // forward elimination and back substitution in place in shared memory
    double prev = 0.0;
#pragma unroll
    for (int i = 0; i < kSeg; ++i) {
      if (i < len) {
        prev = fma(-lo, prev, seg[i]) * __ldg(&L->invm[i]);
        seg[i] = prev;
      }
    }
    const double ylast = prev;  // y[len-1] is final after the forward pass
    double next = prev;
#pragma unroll
    for (int i = kSeg - 2; i >= 0; --i) {
      if (i < len - 1) {
        next = fma(-__ldg(&L->cp[i]), next, seg[i]);
        seg[i] = next;
      }
    }
    ex[2 * ln] = next;
    ex[2 * ln + 1] = ylast;
  }
  __syncthreads();

  // ---- C: interfaces, spike correction, relaxation, store ----------------
  const double up = L->up, up_h31 = L->up_h31;
  const bool yz_edge = j0 == 0 || j0 + R >= ny || k == 0 || k == P.nz - 1;  // tile touches a y/z face
#pragma unroll
  for (int h = 0; h < kMaxE; ++h) {
    const int e = h * T + tid;
    if (h * T >= nelem) break;
    if (e < nelem) {
      const int r = e / nx, x = e - r * nx;
      const int s = x >> 5, i = x & (kSeg - 1);
      const int ln = r * nseg + s;
      const bool last = (s == nseg - 1);
      const double y = rs[r * RS + x + s];
      double cl = 0.0, cr = 0.0;
      if (s > 0) {
        const double xl = (ex[2 * ln - 1] - up_h31 * ex[2 * ln]) * (last ? L->d_tail : L->d_full);
        cl = lo * xl;
      }
      if (!last) {
        const bool rlast = (s + 1 == nseg - 1);
        const double yfr = ex[2 * ln + 2];
        const double xl2 = (ex[2 * ln + 1] - up_h31 * yfr) * (rlast ? L->d_tail : L->d_full);
        const double xf = yfr - (rlast ? L->lo_gT0 : L->lo_g0) * xl2;
        cr = up * xf;
      }
      const double gi = last ? __ldg(&L->gT[i]) : __ldg(&L->g[i]);
      const double xs = fma(-cr, __ldg(&L->h[i]), fma(-cl, gi, y));
      const double nv = relax(ucen[h], omega, xs);
      const long long iu = ubase + (long long)r * px + x;
      v[iu] = nv;
      if (x == 0) v[iu - 1] = -nv;
      if (x == nx - 1) v[iu + 1] = -nv;
      if (yz_edge) {
        const int j = j0 + r;
        if (j == 0 || j == ny - 1 || k == 0 || k == P.nz - 1)
          fused_yz_ghosts(v, iu, nv, x, j, k, nx, ny, P.nz, px, pxy, P.iface);
      }
    }
  }
}

// Generic exact line sweep: one thread per x-line, full-length Thomas with
// per-position factors (any nx, any stencil with a nonsingular pivot chain).
// The forward pass stages y' in v's interior; the backward pass overwrites it
// with the relaxed value.  Tiles have R = 1 (one line per partial).
__global__ void line_generic_jacobi_kernel(const PatchDev* __restrict__ patches, int npatch,
                                           const unsigned char* __restrict__ active, StencilDev st,
                                           double omega, double* __restrict__ partials, long long tile_base,
                                           long long ntiles, int solve) {
  const long long tile = tile_base + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (tile >= tile_base + ntiles) return;
  const int pi = find_patch(patches, npatch, tile);
  const PatchDev& P = patches[pi];
  const int nx = P.nx, ny = P.ny;
  int k, j, rows_;
  tile_coords(P, tile, k, j, rows_);
  const long long px = nx + 2, pxy = px * (ny + 2);
  const int act = active[pi];
  const double* u = P.buf[act];
  double* v = P.buf[act ^ 1];
  const long long ub = (long long)(k + 1) * pxy + (long long)(j + 1) * px + 1;
  const double* fr = P.f + ((long long)k * ny + j) * nx;
  const LineFac* L = P.lf;
  double ssq = 0.0, prev = 0.0;
  for (int x = 0; x < nx; ++x) {
    const long long iu = ub + x;
    const double r = residual7(st, fr[x], u[iu], u[iu - 1], u[iu + 1], u[iu - px], u[iu + px], u[iu - pxy],
                               u[iu + pxy]);
    ssq = fma(r, r, ssq);
    if (solve) {
      prev = fma(-L->lo, prev, r) * L->invmN[x];
      v[iu] = prev;
    }
  }
  if (partials) partials[tile] = ssq;
  if (!solve) return;
  double next = 0.0;
  for (int x = nx - 1; x >= 0; --x) {
    const long long iu = ub + x;
    const double yx = (x == nx - 1) ? v[iu] : fma(-L->cpN[x], next, v[iu]);
    next = yx;
    v[iu] = relax(u[iu], omega, yx);
  }
  v[ub - 1] = -v[ub];
  v[ub + nx] = -v[ub + nx - 1];
  if (j == 0 || j == ny - 1 || k == 0 || k == P.nz - 1)
    for (int x = 0; x < nx; ++x) fused_yz_ghosts(v, ub + x, v[ub + x], x, j, k, nx, ny, P.nz, px, pxy, P.iface);
}

// Apply the exact line inverse to `count` contiguous vectors of length nx
// (psm_factors_apply): one thread per vector, full-length Thomas.
__global__ void line_apply_kernel(const LineFac* __restrict__ L, const double* __restrict__ r,
                                  double* __restrict__ x, long long count) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (b >= count) return;
  const int nx = L->nx;
  const double* rb = r + b * nx;
  double* xb = x + b * nx;
  double prev = 0.0;
  for (int i = 0; i < nx; ++i) {
    prev = fma(-L->lo, prev, rb[i]) * L->invmN[i];
    xb[i] = prev;
  }
  for (int i = nx - 2; i >= 0; --i) xb[i] = fma(-L->cpN[i], xb[i + 1], xb[i]);
}


// ---------------------------------------------------------------------------
// Specialised line-Jacobi sweep for power-of-two nx in [64, 1024].
//
// Persistent CTAs (256 threads) walk tiles of R = 2048/NX x-lines of one
// plane in plane-major order, so the planes k-1, k, k+1 that concurrent
// tiles touch stay in L2 and u streams from HBM about once.  Per tile:
//   A  8 cells per thread, coalesced LDG.64 of u (centre, y+-1, z+-1) and f,
//      x+-1 by warp shuffle; r (reference operation order) -> shared memory,
//      r^2 -> tile partial.
//   B  one lane per 32-cell segment (R*NX/32 = 64 lanes): Thomas on the
//      segment with the dependency chain shortened to one DFMA per cell
//      (y_i = r_i*invm_i - (lo*invm_i)*y_{i-1}), segment end values swapped
//      between neighbouring lanes by shuffle (a row's segments share a warp),
//      interface 2x2 solves -> per-segment coefficients cl, cr.
//   C  8 cells per thread: x = y - cl*g[i] - cr*h[i], v = u + omega*x,
//      store v and the physical x-face ghosts of v.
// Shared buffers are double-buffered across tiles: two barriers per tile.
// At small sizes a tile is a latency chain (tools/nx_timing_probe.py, built
// with -DPSM_NX_TIMING: A 3.5 us, B 0.8 us, C 1.7-2.7 us at 64^3), so every
// independent load of phase A is issued before the first use of any.
// ---------------------------------------------------------------------------
#ifndef PSM_NX_THREADS
#define PSM_NX_THREADS 512
#endif
constexpr int kNxT = PSM_NX_THREADS;  // threads per tile CTA (cells per thread: 2048 / kNxT)
template <int NX, int UNIT>
__global__ void __launch_bounds__(kNxT, 512 / kNxT) line_jacobi_nx_kernel(const __grid_constant__ PatchDev P, int act,
                                                                StencilDev st, double omega,
                                                                double* __restrict__ partials, long long tile_begin,
                                                                long long tile_end, const __grid_constant__ LineFac L) {
  constexpr int T = kNxT, R = kMaxTileCells / NX, NSEG = NX / kSeg, CELLS = R * NX, E = CELLS / T;
  constexpr int RS = NX + NSEG, PX = NX + 2, NSL = R * NSEG;
  static_assert((E == 8 || E == 4) && NSEG <= 32 && NSL <= T, "tile shape");
  __shared__ double rs[2][R * RS];
  __shared__ double cl[2][NSL], cr[2][NSL];
  __shared__ double wsum[2][T / 32];
  __shared__ double tab_invm[kSeg], tab_loinv[kSeg], tab_cp[kSeg], tab_g[kSeg], tab_h[kSeg];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the patch (one launch per patch), its active buffer and the line factors
  // come in as kernel parameters (constant bank): no global round trip
  // before the first tile's loads
  if (tid < kSeg) {
    const double im = L.invm[tid];
    tab_invm[tid] = im;
    tab_loinv[tid] = L.lo * im;
    tab_cp[tid] = L.cp[tid];
    tab_g[tid] = L.g[tid];
    tab_h[tid] = L.h[tid];
  }
  const double lo = L.lo, up = L.up, up_h31 = L.up_h31, lo_g0 = L.lo_g0, d_full = L.d_full;
  __syncthreads();
  int buf = 0;
#ifdef PSM_NX_TIMING
  unsigned long long tm0 = 0, tm1 = 0, tm2 = 0, tmA = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tmA));
#endif
  for (long long tile = tile_begin + blockIdx.x; tile < tile_end; tile += gridDim.x, buf ^= 1) {
#ifdef PSM_NX_TIMING
    if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm0));
#endif
    const int ny = P.ny;
    int k, j0, rows;
    tile_coords(P, tile, k, j0, rows);
    const long long pxy = (long long)PX * (ny + 2);
    const double* __restrict__ u = P.buf[act];
    double* __restrict__ v = P.buf[act ^ 1];
    const long long ubase = (long long)(k + 1) * pxy + (long long)(j0 + 1) * PX + 1;
    const double* __restrict__ fb = P.f + ((long long)k * ny + j0) * NX;
    double* __restrict__ rb = rs[buf];

    // ---- A ----------------------------------------------------------------
    double ssq = 0.0;
    double ucen[E];
#pragma unroll
    for (int h = 0; h < E; h += 4) {
      double c[4], ym[4], yp[4], zm[4], zp[4], fv[4], xe[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = (h + q) * T + tid;
        const int row = e / NX, x = e % NX;
        const long long iu = ubase + (long long)row * PX + x;
        if (row < rows) {
          c[q] = __ldg(u + iu);
          ym[q] = __ldg(u + iu - PX);
          yp[q] = __ldg(u + iu + PX);
          zm[q] = __ldg(u + iu - pxy);
          zp[q] = __ldg(u + iu + pxy);
          fv[q] = __ldg(fb + e);
          // the warp's outer x neighbours, issued with the rest
          xe[q] = lane == 0 ? __ldg(u + iu - 1) : lane == 31 ? __ldg(u + iu + 1) : 0.0;
        } else {
          c[q] = ym[q] = yp[q] = zm[q] = zp[q] = fv[q] = xe[q] = 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = (h + q) * T + tid;
        const int row = e / NX, x = e % NX;
        double xl = __shfl_up_sync(0xffffffffu, c[q], 1);
        double xr = __shfl_down_sync(0xffffffffu, c[q], 1);
        ucen[h + q] = c[q];
        if (row < rows) {
          if (lane == 0) xl = xe[q];
          if (lane == 31) xr = xe[q];
          double res;
          if (UNIT) {
            double acc = __dmul_rn(st.c, c[q]);
            acc = __dsub_rn(acc, xl);
            acc = __dsub_rn(acc, xr);
            acc = __dsub_rn(acc, ym[q]);
            acc = __dsub_rn(acc, yp[q]);
            acc = __dsub_rn(acc, zm[q]);
            acc = __dsub_rn(acc, zp[q]);
            res = __dsub_rn(fv[q], acc);
          } else {
            res = residual7(st, fv[q], c[q], xl, xr, ym[q], yp[q], zm[q], zp[q]);
          }
          ssq = fma(res, res, ssq);
          rb[row * RS + x + (x >> 5)] = res;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if (lane == 0) wsum[buf][warp] = ssq;
    __syncthreads();  // (1) r complete
#ifdef PSM_NX_TIMING
    if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm1));
#endif
    if (tid == 0 && partials) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < T / 32; ++w) t += wsum[buf][w];
      partials[tile] = t;
    }

    // ---- B: segment solves + interfaces (lanes 0..NSL-1) ---------------------
    if (tid < NSL) {
      const int r = tid / NSEG, s = tid % NSEG;
      double* seg = rb + r * RS + s * (kSeg + 1);
      double yv[kSeg];
#pragma unroll
      for (int i = 0; i < kSeg; ++i) yv[i] = seg[i] * tab_invm[i];
      double prev = yv[0];
#pragma unroll
      for (int i = 1; i < kSeg; ++i) {
        prev = fma(-tab_loinv[i], prev, yv[i]);
        yv[i] = prev;
      }
      const double ylast = prev;
#pragma unroll
      for (int i = kSeg - 2; i >= 0; --i) yv[i] = fma(-tab_cp[i], yv[i + 1], yv[i]);
#pragma unroll
      for (int i = 0; i < kSeg; ++i) seg[i] = yv[i];
      const double yfirst = yv[0];
      // neighbours' end values: lanes of one row are contiguous in a warp
      const double yl_left = __shfl_up_sync(0xffffffffu >> (32 - (NSL < 32 ? NSL : 32)), ylast, 1);
      const double yf_right = __shfl_down_sync(0xffffffffu >> (32 - (NSL < 32 ? NSL : 32)), yfirst, 1);
      double cl_v = 0.0, cr_v = 0.0;
      if (s > 0) cl_v = lo * ((yl_left - up_h31 * yfirst) * d_full);
      if (s < NSEG - 1) {
        const double xl2 = (ylast - up_h31 * yf_right) * d_full;
        cr_v = up * (yf_right - lo_g0 * xl2);
      }
      cl[buf][tid] = cl_v;
      cr[buf][tid] = cr_v;
    }
    __syncthreads();  // (2) y, cl, cr complete
#ifdef PSM_NX_TIMING
    if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm2));
#endif

    // ---- C ----------------------------------------------------------------
    const bool yz_edge = j0 == 0 || j0 + rows >= ny || k == 0 || k == P.nz - 1;  // tile touches a y/z face
#pragma unroll
    for (int h = 0; h < E; ++h) {
      const int e = h * T + tid;
      const int row = e / NX, x = e % NX;
      if (row < rows) {
        const int sl = row * NSEG + (x >> 5);
        const double y = rb[row * RS + x + (x >> 5)];
        const double xs = fma(-cr[buf][sl], tab_h[lane], fma(-cl[buf][sl], tab_g[lane], y));
        const double nv = relax(ucen[h], omega, xs);
        const long long iu = ubase + (long long)row * PX + x;
        v[iu] = nv;
        if (x == 0) v[iu - 1] = -nv;
        if (x == NX - 1) v[iu + 1] = -nv;
        if (yz_edge) {
          const int j = j0 + row;
          if (j == 0 || j == ny - 1 || k == 0 || k == P.nz - 1)
            fused_yz_ghosts(v, iu, nv, x, j, k, NX, ny, P.nz, PX, pxy, P.iface);
        }
      }
    }
#ifdef PSM_NX_TIMING
    if (tid == 0) {
      unsigned long long t3;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
      printf("nx-timing cta %d tile %lld: start %llu end %llu  A %llu  B %llu  C %llu ns\n", blockIdx.x, tile, tmA,
             t3, tm1 - tm0, tm2 - tm1, t3 - tm2);
    }
#endif
  }
}

template <int NX>
static cudaError_t launch_nx(int unit, const PatchDev& P, int act, const StencilDev& st, double omega,
                             double* partials, long long t0, long long t1, int grid, const LineFac& L,
                             cudaStream_t stream) {
  if (unit)
    line_jacobi_nx_kernel<NX, 1><<<grid, kNxT, 0, stream>>>(P, act, st, omega, partials, t0, t1, L);
  else
    line_jacobi_nx_kernel<NX, 0><<<grid, kNxT, 0, stream>>>(P, act, st, omega, partials, t0, t1, L);
  return cudaGetLastError();
}

// nx values with a specialised kernel
bool line_nx_specialised(int nx) {
  return nx == 64 || nx == 128 || nx == 256 || nx == 512 || nx == 1024;
}

template <int NX>
static int occ_nx() {  // (per process: every device of a run is the same sm_100a part)
  static const int occ = [] {
    int a = 0, b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, line_jacobi_nx_kernel<NX, 0>, kNxT, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, line_jacobi_nx_kernel<NX, 1>, kNxT, 0);
    return a < b ? a : b;
  }();
  return occ;
}

int line_nx_occupancy(int nx) {
  switch (nx) {
    case 64: return occ_nx<64>();
    case 128: return occ_nx<128>();
    case 256: return occ_nx<256>();
    case 512: return occ_nx<512>();
    default: return occ_nx<1024>();
  }
}

// tiles [t0, t1) of patch P (host copy of its descriptor), active buffer act
cudaError_t launch_line_nx(int nx, int unit, const PatchDev& P, int act, const StencilDev& st, double omega,
                           double* partials, long long t0, long long t1, int grid, const LineFac& L,
                           cudaStream_t stream) {
  if (t1 <= t0) return cudaSuccess;
  const long long n = t1 - t0;
  if (grid > n) grid = (int)n;
#define PSM_NX(N) \
  case N: return launch_nx<N>(unit, P, act, st, omega, partials, t0, t1, grid, L, stream);
  switch (nx) {
    PSM_NX(64)
    PSM_NX(128)
    PSM_NX(256)
    PSM_NX(512)
    PSM_NX(1024)
    default: return cudaErrorInvalidValue;
  }
#undef PSM_NX
}

// ---- host-side launchers ---------------------------------------------------
cudaError_t launch_line_tiles(int mode, const PatchDev* patches, int npatch, const unsigned char* active,
                              const StencilDev& st, double omega, double* partials, double* rbuf, long long tile_base,
                              long long ntiles, int threads, size_t smem, cudaStream_t stream) {
  if (ntiles <= 0) return cudaSuccess;
  if (mode == 0) {
    line_tile_kernel<0><<<(unsigned)ntiles, threads, 0, stream>>>(patches, npatch, active, st, omega, partials,
                                                                  nullptr, tile_base);
  } else if (mode == 1) {
    line_tile_kernel<1><<<(unsigned)ntiles, threads, smem, stream>>>(patches, npatch, active, st, omega, partials,
                                                                     nullptr, tile_base);
  } else {
    line_tile_kernel<2><<<(unsigned)ntiles, threads, 0, stream>>>(patches, npatch, active, st, omega, partials,
                                                                  rbuf, tile_base);
  }
  return cudaGetLastError();
}

cudaError_t launch_line_generic(int solve, const PatchDev* patches, int npatch, const unsigned char* active,
                                const StencilDev& st, double omega, double* partials, long long tile_base,
                                long long ntiles, cudaStream_t stream) {
  if (ntiles <= 0) return cudaSuccess;
  const int tpb = 128;
  line_generic_jacobi_kernel<<<(unsigned)((ntiles + tpb - 1) / tpb), tpb, 0, stream>>>(
      patches, npatch, active, st, omega, partials, tile_base, ntiles, solve);
  return cudaGetLastError();
}

cudaError_t launch_line_apply(const LineFac* L, const double* r, double* x, long long count, cudaStream_t stream) {
  if (count == 0) return cudaSuccess;
  line_apply_kernel<<<(unsigned)((count + 127) / 128), 128, 0, stream>>>(L, r, x, count);
  return cudaGetLastError();
}

cudaError_t line_tile_kernel_setup(size_t smem) {
  return cudaFuncSetAttribute(line_tile_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

}  // namespace psm
