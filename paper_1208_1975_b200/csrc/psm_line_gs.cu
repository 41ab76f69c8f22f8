// Line-block Gauss-Seidel sweeps, in place (smoother._gs_step,
// smoother.py:156-169; ghosts lagged until the step-end refresh).
//
// The serial strategy (runtime.py:164-168) visits x-lines (j,k) of a patch in
// lexicographic order, j fastest.  Line (j,k) reads the NEW lines (j-1,k) and
// (j,k-1) and the OLD lines (j+1,k), (j,k+1).  The pipeline below keeps that
// information flow exactly: a work unit is one z-plane of one patch; one warp
// owns a unit and walks its rows j = 0..ny-1 in order, so (j-1,k) is new by
// construction; before row j it waits until the warp on plane k-1 has
// published row j (acquire/release progress flag), so (j,k-1) is new, and
// plane k+1 cannot touch row j before this warp publishes it, so (j,k+1) is
// still old.  Every line therefore computes exactly the lexicographic
// arithmetic (the pipeline is a wavefront schedule over d = j + k).
//
// CHAOTIC mode drops the acquire/release ordering: the progress word is read
// and written relaxed, without fences, so a line may see old or new values of
// (j,k-1) -- in-place block updates without a global ordering, the contract of
// smooth_chaotic_gs_step under parallel strategies.
//
// Units are handed out by an atomic ticket in dependency order, so a unit's
// predecessor is always held by a running warp: no co-residency assumption.
#include "psm_internal.cuh"

namespace psm {

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int NC, int CHAOTIC>
__global__ void __launch_bounds__(128) line_gs_kernel(const PatchDev* __restrict__ patches, int npatch,
                                                      const unsigned char* __restrict__ active, StencilDev st,
                                                      double omega, int* __restrict__ flags, long long nunits,
                                                      const int* __restrict__ unit_patch,
                                                      const int* __restrict__ unit_plane) {
  extern __shared__ double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kRS = NC * kSeg + NC;  // padded row (nx <= 32*NC)
  double* rs = sm + wid * (kRS + 2 * NC);
  double* ex = rs + kRS;
  int* ticket = flags - 1;  // flags[-1] is the unit counter
  for (;;) {
    long long u = 0;
    if (lane == 0) u = atomicAdd(ticket, 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= nunits) return;
    const int p = unit_patch[u], k = unit_plane[u];
    const PatchDev& P = patches[p];
    const int nx = P.nx, ny = P.ny, nz = P.nz;
    const long long px = nx + 2, pxy = px * (ny + 2);
    double* U = P.buf[active[p]];
    const double* F = P.f + (long long)k * ny * nx;
    int* my_flag = flags + P.plane0 + k;
    const int* dep_flag = flags + P.plane0 + k - 1;
    const LineFac* __restrict__ L = P.lf;
    const int nseg = L->nseg, tail = L->tail;
    const double lo = L->lo, up = L->up, up_h31 = L->up_h31;
    // row base pointer: u(0, j, kk)
    auto rowp = [&](int j, int kk) -> double* {
      return U + (long long)(kk + 1) * pxy + (long long)(j + 1) * px + 1;
    };

    double cen[NC], ym[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int x = i * kSeg + lane;
      const bool ok = x < nx;
      cen[i] = ok ? rowp(0, k)[x] : 0.0;
      ym[i] = ok ? rowp(-1, k)[x] : 0.0;  // lagged physical/interface ghost row
    }
    for (int j = 0; j < ny; ++j) {
      double nxt[NC], zp[NC], zm[NC], fv[NC];
      double* rj = rowp(j, k);
      const double* rn = rowp(j + 1, k);       // old row j+1 (ghost row when j+1 == ny)
      const double* rz = rowp(j, k + 1);       // old plane k+1 (ghost plane when k+1 == nz)
      const double* rzm = rowp(j, k - 1);      // new plane k-1 (ghost plane when k == 0)
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int x = i * kSeg + lane;
        const bool ok = x < nx;
        nxt[i] = ok ? rn[x] : 0.0;
        zp[i] = ok ? __ldcg(rz + x) : 0.0;
        fv[i] = ok ? __ldg(F + (long long)j * nx + x) : 0.0;
      }
      const double gl = rj[-1], gr = rj[nx];
      if (k > 0) {
        if (lane == 0) {
          if (CHAOTIC) {
            while (ld_relaxed(dep_flag) <= j) {
            }
          } else {
            while (ld_acquire(dep_flag) <= j) {
            }
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int x = i * kSeg + lane;
        zm[i] = (x < nx) ? __ldcg(rzm + x) : 0.0;
      }
      // ---- residual (reference order), r to smem -------------------------
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int x = i * kSeg + lane;
        double xl = __shfl_up_sync(0xffffffffu, cen[i], 1);
        double xr = __shfl_down_sync(0xffffffffu, cen[i], 1);
        const double wrapl = (i > 0) ? __shfl_sync(0xffffffffu, cen[i > 0 ? i - 1 : 0], 31) : gl;
        const double wrapr = (i + 1 < NC) ? __shfl_sync(0xffffffffu, cen[i + 1 < NC ? i + 1 : i], 0) : gr;
        if (lane == 0) xl = (i > 0) ? wrapl : gl;
        if (lane == 31 || x + 1 >= nx) xr = (x + 1 >= nx) ? gr : wrapr;
        if (x < nx) {
          const double r = residual7(st, fv[i], cen[i], xl, xr, ym[i], nxt[i], zm[i], zp[i]);
          rs[x + (x >> 5)] = r;
        }
      }
      __syncwarp();
      // ---- segment solves ------------------------------------------------
      if (lane < nseg) {
        const int s = lane;
        const int len = (s == nseg - 1) ? tail : kSeg;
        double* seg = rs + s * (kSeg + 1);
        double prev = 0.0;
#pragma unroll
        for (int i = 0; i < kSeg; ++i) {
          if (i < len) {
            prev = fma(-lo, prev, seg[i]) * __ldg(&L->invm[i]);
            seg[i] = prev;
          }
        }
        const double ylast = prev;
        double next = prev;
#pragma unroll
        for (int i = kSeg - 2; i >= 0; --i) {
          if (i < len - 1) {
            next = fma(-__ldg(&L->cp[i]), next, seg[i]);
            seg[i] = next;
          }
        }
        ex[2 * s] = next;
        ex[2 * s + 1] = ylast;
      }
      __syncwarp();
      // ---- interfaces, correction, in-place update -------------------------
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int x = i * kSeg + lane;
        if (x < nx) {
          const int s = i;  // x >> 5
          const bool last = (s == nseg - 1);
          double cl = 0.0, cr = 0.0;
          if (s > 0) cl = lo * ((ex[2 * s - 1] - up_h31 * ex[2 * s]) * (last ? L->d_tail : L->d_full));
          if (!last) {
            const bool rlast = (s + 1 == nseg - 1);
            const double yfr = ex[2 * s + 2];
            const double xl2 = (ex[2 * s + 1] - up_h31 * yfr) * (rlast ? L->d_tail : L->d_full);
            cr = up * (yfr - (rlast ? L->lo_gT0 : L->lo_g0) * xl2);
          }
          const double gi = last ? __ldg(&L->gT[lane]) : __ldg(&L->g[lane]);
          const double xs = fma(-cr, __ldg(&L->h[lane]), fma(-cl, gi, rs[x + s]));
          const double nv = relax(cen[i], omega, xs);
          rj[x] = nv;
          ym[i] = nv;
          cen[i] = nxt[i];
        }
      }
      // ---- publish row j of plane k ----------------------------------------
      if (CHAOTIC) {
        __syncwarp();
        if (lane == 0) st_relaxed(my_flag, j + 1);
      } else {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(my_flag, j + 1);
      }
    }
    (void)nz;
  }
}

template <int NC, int CH>
static cudaError_t launch_gs_t(const PatchDev* patches, int npatch, const unsigned char* active,
                               const StencilDev& st, double omega, int* flags, long long nunits,
                               const int* unit_patch, const int* unit_plane, int threads, size_t smem, int grid,
                               cudaStream_t stream) {
  line_gs_kernel<NC, CH><<<grid, threads, smem, stream>>>(patches, npatch, active, st, omega, flags, nunits,
                                                           unit_patch, unit_plane);
  return cudaGetLastError();
}

int gs_chunks_for(int max_nx) {
  if (max_nx <= 32) return 1;
  if (max_nx <= 64) return 2;
  if (max_nx <= 128) return 4;
  if (max_nx <= 256) return 8;
  return 0;  // generic wavefront path
}

size_t gs_smem_per_warp(int nc) { return (size_t)(nc * kSeg + nc + 2 * nc) * sizeof(double); }

template <int NC>
static int occupancy_t(int threads, size_t smem) {
  int b0 = 0, b1 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, line_gs_kernel<NC, 0>, threads, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, line_gs_kernel<NC, 1>, threads, smem);
  return b0 < b1 ? b0 : b1;
}

int gs_occupancy(int nc, int threads, size_t smem) {
  switch (nc) {
    case 1: return occupancy_t<1>(threads, smem);
    case 2: return occupancy_t<2>(threads, smem);
    case 4: return occupancy_t<4>(threads, smem);
    default: return occupancy_t<8>(threads, smem);
  }
}

cudaError_t launch_line_gs(int mode, const PatchDev* patches, int npatch, const unsigned char* active,
                           const StencilDev& st, double omega, int* flags, long long nunits, const int* unit_patch,
                           const int* unit_plane, int threads, size_t smem, int grid_nc, cudaStream_t stream) {
  // grid_nc packs (grid << 4) | nc
  const int nc = grid_nc & 15, grid = grid_nc >> 4;
#define PSM_GS_CASE(N)                                                                                          \
  case N:                                                                                                       \
    return mode ? launch_gs_t<N, 1>(patches, npatch, active, st, omega, flags, nunits, unit_patch, unit_plane, \
                                    threads, smem, grid, stream)                                              \
                : launch_gs_t<N, 0>(patches, npatch, active, st, omega, flags, nunits, unit_patch, unit_plane, \
                                    threads, smem, grid, stream);
  switch (nc) {
    PSM_GS_CASE(1)
    PSM_GS_CASE(2)
    PSM_GS_CASE(4)
    PSM_GS_CASE(8)
    default:
      return cudaErrorInvalidValue;
  }
#undef PSM_GS_CASE
}

// Generic wavefront GS: one launch per wavefront d = j + k; one thread per
// line of the wavefront, full-length Thomas.  Any nx, any dominant stencil.
__global__ void line_gs_generic_kernel(const PatchDev* __restrict__ patches, int npatch,
                                       const unsigned char* __restrict__ active, StencilDev st, double omega,
                                       int wave, long long nlines_total) {
  // enumerate candidate lines j of every patch; k = wave - j
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long acc = 0;
  int p = -1;
  for (int q = 0; q < npatch; ++q) {
    if (t < acc + patches[q].ny) {
      p = q;
      break;
    }
    acc += patches[q].ny;
  }
  if (p < 0) return;
  const PatchDev& P = patches[p];
  const int j = (int)(t - acc), k = wave - j;
  if (k < 0 || k >= P.nz) return;
  const int nx = P.nx, ny = P.ny;
  const long long px = nx + 2, pxy = px * (ny + 2);
  double* U = P.buf[active[p]];
  const long long ub = (long long)(k + 1) * pxy + (long long)(j + 1) * px + 1;
  const double* fr = P.f + ((long long)k * ny + j) * nx;
  const LineFac* L = P.lf;
  // residual of the whole line first (it reads the line's old values), staged
  // in the other buffer's matching interior cells (scratch during GS)
  double* scratch = P.buf[active[p] ^ 1] + ub;
  double prev = 0.0;
  for (int x = 0; x < nx; ++x) {
    const long long iu = ub + x;
    const double r = residual7(st, fr[x], U[iu], U[iu - 1], U[iu + 1], U[iu - px], U[iu + px], U[iu - pxy],
                               U[iu + pxy]);
    prev = fma(-L->lo, prev, r) * L->invmN[x];
    scratch[x] = prev;
  }
  double next = 0.0;
  for (int x = nx - 1; x >= 0; --x) {
    const double yx = (x == nx - 1) ? scratch[x] : fma(-L->cpN[x], next, scratch[x]);
    next = yx;
    U[ub + x] = relax(U[ub + x], omega, yx);
  }
  (void)nlines_total;
}

cudaError_t launch_line_gs_generic(const PatchDev* patches, int npatch, const unsigned char* active,
                                   const StencilDev& st, double omega, int wave, long long nj_total,
                                   cudaStream_t stream) {
  if (nj_total == 0) return cudaSuccess;
  line_gs_generic_kernel<<<(unsigned)((nj_total + 127) / 128), 128, 0, stream>>>(patches, npatch, active, st,
                                                                                 omega, wave, nj_total);
  return cudaGetLastError();
}

}  // namespace psm
