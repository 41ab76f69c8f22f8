// Box blocks (bx, by, bz) with every extent <= 8: the paper's own cubic
// blocks (Algorithm 2; DEFAULT_BLOCK_SIZES 2^3 .. 8^3, analysis.py:38-46).
//
// Replaces, for those block_dims, InverseCache.get / invert_dense
// (blocklinalg.py:116-163, stencil.py:115-138), the dense matvec
// (blocklinalg.py:90-105) and the block loops of smoother._jacobi_step /
// _gs_step (smoother.py:138-169).
//
// Exact inverse, separable.  The closure-free block operator is
// c I + L_x + L_y + L_z with L_a = tridiag(lo_a, 0, up_a) along axis a.  When
// lo_a up_a > 0 (every physical stencil) the similarity D_a = diag(s_a^p),
// s_a = sqrt(lo_a/up_a), makes each L_a symmetric with off-diagonal
// sign(lo_a) sqrt(lo_a up_a), so A = D (Q Lambda Q) D^{-1} with Q the
// orthonormal DST-I of each extent and
//   lambda_ijk = c + 2 o_x cos(pi (i+1)/(ex+1)) + 2 o_y cos(..) + 2 o_z cos(..).
// A^{-1} r = D Q Lambda^{-1} Q D^{-1} r: three forward transforms
// F_a = Q diag(s_a^-p), a scaling, three backward transforms B_a = diag(s_a^p) Q,
// 2 (ex + ey + ez) FMAs per cell instead of the 2 ex ey ez of the dense
// matvec.  Tables cover every extent 1..8 per axis, so blocks truncated at
// patch edges (grid.py:298-306) need nothing extra.
//
// Kernel: one 128-thread CTA per region of <= 8^3 cells tiled by whole
// blocks (small blocks are batched, 2^3 blocks 64 to a region), persistent
// over a region list.  The region's u with a one-cell halo is staged in
// shared memory, the residual is formed in the reference operation order,
// each 1-D transform has one thread per block line (line in registers, padded
// rows: conflict-free), the 1/lambda scaling (host table per extent triple) is
// folded into the last forward pass and the relaxation into the last
// backward pass.  Jacobi writes v (and v's physical x-ghosts) for all
// blocks in one launch; GS updates u in place one wavefront
// (bi + bj + bk = w) of blocks per launch: face-adjacent blocks lie on
// neighbouring wavefronts, so the order is exactly the lexicographic one of
// runtime.py:164-168.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "psm_internal.cuh"

namespace psm {

constexpr int kBoxMax = 8;     // largest extent per axis
constexpr int kBoxT = 128;     // threads per block CTA
constexpr int kHs = 10;        // halo box row stride (ex + 2 <= 10)
constexpr int kHp = 100;       // halo box plane stride
#ifndef PSM_BOX_RS
#define PSM_BOX_RS 12
#define PSM_BOX_RP 100
#endif
// work cube strides: rows 12, planes 100 (both = 4 mod 8 doubles) make the
// DMMA B-fragment loads of all three axes bank-conflict free
constexpr int kRs = PSM_BOX_RS;
constexpr int kRp = PSM_BOX_RP;

__device__ __forceinline__ void box_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void box_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void box_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void box_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ const double* box_mat(const double* T, int axis, int e) {
  return T + ((axis * kBoxMax) + (e - 1)) * 64;
}
__device__ __forceinline__ const double* box_eig(const double* L, int axis, int e) {
  return L + ((axis * kBoxMax) + (e - 1)) * kBoxMax;
}

// y(out) = M x along one line of n <= 8 values: x strided by `stride` in the
// work cube; M row-major 8x8 (entry (i, p) at i*8+p).
__device__ __forceinline__ void box_line(double* __restrict__ w, int stride, int n, const double* __restrict__ M) {
  double x[kBoxMax];
#pragma unroll
  for (int p = 0; p < kBoxMax; ++p) x[p] = p < n ? w[p * stride] : 0.0;
#pragma unroll
  for (int i = 0; i < kBoxMax; ++i) {
    if (i < n) {
      double acc = 0.0;
#pragma unroll
      for (int p = 0; p < kBoxMax; ++p)
        if (p < n) acc = fma(__ldg(M + i * 8 + p), x[p], acc);
      w[i * stride] = acc;
    }
  }
}

// 1/lambda of cell (i, j, k) of a block with extents (ex, ey, ez)
__device__ __forceinline__ double box_ilam(const double* __restrict__ IL, int ex, int ey, int ez, int i, int j,
                                           int k) {
  return __ldg(IL + ((((ex - 1) * 8 + (ey - 1)) * 8 + (ez - 1)) * 512) + (k * 8 + j) * 8 + i);
}

// Work items are regions (patch, x0, y0, z0) of (bx*mx, by*my, bz*mz) <= 8^3
// cells, clipped to the patch and tiled by whole blocks (Jacobi: every block
// of the region at once; GS: m = 1, one block).  inplace = 0: Jacobi into the
// inactive buffer; 1: GS in the active buffer.
__global__ void __launch_bounds__(kBoxT) box_sweep_kernel(const PatchDev* __restrict__ patches,
                                                          const unsigned char* __restrict__ active, StencilDev st,
                                                          double omega, const int4* __restrict__ blocks,
                                                          int nblocks, int inplace, int mx, int my, int mz) {
  __shared__ double hb[kHp * kHs];      // u with halo, (rz+2) x (ry+2) x (rx+2)
  __shared__ double wc[kBoxMax * kRp];  // work cube
  const int tid = threadIdx.x;
  for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const int4 B = blocks[b];
    const PatchDev& P = patches[B.x];
    const BoxFac* __restrict__ F = P.bf;
    const int nx = P.nx, ny = P.ny, nz = P.nz;
    const int bx = F->bx, by = F->by, bz = F->bz;
    const int x0 = B.y, y0 = B.z, z0 = B.w;
    const int rx = min(bx * mx, nx - x0), ry = min(by * my, ny - y0), rz = min(bz * mz, nz - z0);
    const int qx = (rx + bx - 1) / bx, qy = (ry + by - 1) / by, qz = (rz + bz - 1) / bz;
    const long long px = nx + 2, pxy = px * (ny + 2);
    const int act = active[B.x];
    const double* __restrict__ u = P.buf[act];
    double* __restrict__ v = P.buf[inplace ? act : act ^ 1];
    // ---- stage u with its halo ---------------------------------------------
    const int hx = rx + 2, hy = ry + 2, hn = hx * hy * (rz + 2);
    const double* ub = u + (long long)z0 * pxy + (long long)y0 * px + x0;  // padded (x0-1, y0-1, z0-1) + 1
    for (int q = tid; q < hn; q += kBoxT) {
      const int c = q / (hx * hy), r = q - c * hx * hy, bb = r / hx, a = r - bb * hx;
      hb[c * kHp + bb * kHs + a] = ub[(long long)c * pxy + (long long)bb * px + a];
    }
    __syncthreads();
    // ---- residual, reference operation order (stencil.py:106-111) -----------
    const int ncell = rx * ry * rz;
    for (int q = tid; q < ncell; q += kBoxT) {
      const int k = q / (rx * ry), r = q - k * rx * ry, j = r / rx, i = r - j * rx;
      const int h = (k + 1) * kHp + (j + 1) * kHs + i + 1;
      const double fv = P.f[((long long)(z0 + k) * ny + (y0 + j)) * nx + x0 + i];
      wc[k * kRp + j * kRs + i] = residual7(st, fv, hb[h], hb[h - 1], hb[h + 1], hb[h - kHs], hb[h + kHs],
                                            hb[h - kHp], hb[h + kHp]);
    }
    __syncthreads();
    // ---- forward transforms F_x, F_y, F_z (z also scales by 1/lambda) -------
    for (int l = tid; l < qx * ry * rz; l += kBoxT) {  // x-lines: (block column, y, z)
      const int q = l % qx, yz = l / qx, j = yz % ry, k = yz / ry, i0 = q * bx, ex = min(bx, rx - i0);
      box_line(wc + k * kRp + j * kRs + i0, 1, ex, box_mat(F->F, 0, ex));
    }
    __syncthreads();
    for (int l = tid; l < qy * rx * rz; l += kBoxT) {  // y-lines: (x, block row, z)
      const int i = l % rx, r = l / rx, q = r % qy, k = r / qy, j0 = q * by, ey = min(by, ry - j0);
      box_line(wc + k * kRp + j0 * kRs + i, kRs, ey, box_mat(F->F, 1, ey));
    }
    __syncthreads();
    for (int l = tid; l < qz * rx * ry; l += kBoxT) {  // z-lines: (x, y, block layer)
      const int i = l % rx, r = l / rx, j = r % ry, q = r / ry, k0 = q * bz, ez = min(bz, rz - k0);
      double* w = wc + k0 * kRp + j * kRs + i;
      box_line(w, kRp, ez, box_mat(F->F, 2, ez));
      const int ib = i % bx, jb = j % by;
      const int ex = min(bx, rx - (i - ib)), ey = min(by, ry - (j - jb));
      for (int k = 0; k < ez; ++k) w[k * kRp] *= box_ilam(F->IL, ex, ey, ez, ib, jb, k);
    }
    __syncthreads();
    // ---- backward transforms B_z, B_y, B_x; relax in the last ---------------
    for (int l = tid; l < qz * rx * ry; l += kBoxT) {
      const int i = l % rx, r = l / rx, j = r % ry, q = r / ry, k0 = q * bz, ez = min(bz, rz - k0);
      box_line(wc + k0 * kRp + j * kRs + i, kRp, ez, box_mat(F->B, 2, ez));
    }
    __syncthreads();
    for (int l = tid; l < qy * rx * rz; l += kBoxT) {
      const int i = l % rx, r = l / rx, q = r % qy, k = r / qy, j0 = q * by, ey = min(by, ry - j0);
      box_line(wc + k * kRp + j0 * kRs + i, kRs, ey, box_mat(F->B, 1, ey));
    }
    __syncthreads();
    for (int l = tid; l < qx * ry * rz; l += kBoxT) {
      const int q = l % qx, yz = l / qx, j = yz % ry, k = yz / ry, i0 = q * bx, ex = min(bx, rx - i0);
      double* w = wc + k * kRp + j * kRs + i0;
      box_line(w, 1, ex, box_mat(F->B, 0, ex));
      double* vrow = v + (long long)(z0 + k + 1) * pxy + (long long)(y0 + j + 1) * px + x0 + i0 + 1;
      const double* hrow = hb + (k + 1) * kHp + (j + 1) * kHs + i0 + 1;
      for (int i = 0; i < ex; ++i) {
        const double nv = relax(hrow[i], omega, w[i]);
        vrow[i] = nv;
        if (!inplace) {  // v's physical x-ghosts (the step-end refresh skips x faces)
          if (x0 + i0 + i == 0) vrow[i - 1] = -nv;
          if (x0 + i0 + i == nx - 1) vrow[i + 1] = -nv;
        }
      }
    }
    __syncthreads();
  }
}

// ---- tensor-core (DMMA m8n8k4) transforms of interior 8^3 regions ---------
// One pass computes Y = M X for the 64 lines of one axis of the region: M is
// the 8x8 block-diagonal composition of the block transform (blockdiag of
// 8/B copies of the B x B matrix), X the 8 x 64 line matrix.  4 warps x 2
// line tiles x 2 k-steps: 16 DMMA per pass instead of 4,096 scalar FMAs.
__device__ __forceinline__ int box_addr(int axis, int n, int p) {
  return axis == 0 ? (n >> 3) * kRp + (n & 7) * kRs + p
                   : axis == 1 ? (n >> 3) * kRp + p * kRs + (n & 7) : p * kRp + (n >> 3) * kRs + (n & 7);
}
__device__ __forceinline__ void box_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// A fragments (m8n8k4: lane holds M[lane/4][4 ks + lane%4]) of blockdiag(T_B)
template <int BS>
__device__ __forceinline__ void box_afrag(const double* __restrict__ T, int lane, double (&a)[2]) {
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const int r = lane >> 2, c = 4 * ks + (lane & 3);
    a[ks] = (r / BS == c / BS) ? __ldg(T + (r % BS) * 8 + (c % BS)) : 0.0;
  }
}
template <int BX, int BY, int BZ>
__device__ __forceinline__ void box_pass_mma(double* wc, int axis, const double (&a)[2], int lane, int warp,
                                             const double* sc /* 4 per lane or null */) {
#pragma unroll
  for (int tt = 0; tt < 2; ++tt) {
    const int t = warp * 2 + tt;
    double d0 = 0.0, d1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
      box_dmma(d0, d1, a[ks], wc[box_addr(axis, 8 * t + (lane >> 2), 4 * ks + (lane & 3))]);
    const int p = lane >> 2, n0 = 8 * t + 2 * (lane & 3);
    if (sc) {  // forward z pass: scale by 1/lambda (p = k, line n = (i, j))
      d0 *= sc[2 * tt];
      d1 *= sc[2 * tt + 1];
    }
    __syncwarp();
    wc[box_addr(axis, n0, p)] = d0;
    wc[box_addr(axis, n0 + 1, p)] = d1;
  }
}

// The same sweep with compile-time block dims and region multipliers: a
// fixed thread-to-cell/line mapping replaces the runtime integer divisions
// that dominated the generic kernel's instruction count (ncu: 28% IMAD plus
// software division).  Regions are clipped at patch edges at run time.
// GS (gsdep != null): one persistent launch per sweep instead of one per
// wavefront.  Blocks are handed out by an atomic ticket in wavefront order
// (bi + bj + bk, the list the host built); a block waits until its three
// lexicographic predecessors (gsdep[b].y/z/w: flag indices, -1 at patch
// faces) have stored their new values, reads its halo (fresh: acquire fence,
// no prefetch across dependent blocks), relaxes in place and releases its own
// flag (gsdep[b].x).  Predecessors always hold smaller tickets, so the waits
// cannot deadlock; the arithmetic is the lexicographic sweep's exactly.
__device__ __forceinline__ int box_ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int BX, int BY, int BZ, int MX, int MY, int MZ>
__global__ void __launch_bounds__(kBoxT, 5) box_sweep_t(const PatchDev* __restrict__ patches,
                                                     const unsigned char* __restrict__ active, StencilDev st,
                                                     double omega, const int4* __restrict__ blocks, int nblocks,
                                                     int inplace, const int4* __restrict__ gsdep, int* flags,
                                                     int* ticket) {
  constexpr int RX = BX * MX, RY = BY * MY, RZ = BZ * MZ;
  constexpr int HX = RX + 2, HY = RY + 2, HN = HX * HY * (RZ + 2);
  constexpr int NC = RX * RY * RZ;
  // double-buffered staging: the next region's u halo and f stream in with
  // cp.async while this region computes (the sweep is otherwise latency-bound)
  __shared__ __align__(16) double hbuf[2][kHp * kHs];
  __shared__ __align__(16) double fbuf[2][NC];
  __shared__ double wc[kBoxMax * kRp];
  const int tid = threadIdx.x;
  auto stage = [&](int b, int slot) {
    if (b < nblocks) {
      const int4 B = blocks[b];
      const PatchDev& P = patches[B.x];
      const int nx = P.nx, ny = P.ny, nz = P.nz;
      const int x0 = B.y, y0 = B.z, z0 = B.w;
      const int rx = min(RX, nx - x0), ry = min(RY, ny - y0), rz = min(RZ, nz - z0);
      const long long px = nx + 2, pxy = px * (ny + 2);
      const double* ub = P.buf[active[B.x]] + (long long)z0 * pxy + (long long)y0 * px + x0;
      const double* fb0 = P.f + ((long long)z0 * ny + y0) * nx + x0;
      // 16-byte copies when every row start is 16-byte aligned (full rows of an
      // even-width patch at an even x0; the halo row stride kHs is even)
      const bool wide = (RX % 2 == 0) && rx == RX && ((nx | x0) & 1) == 0 &&
                        ((((uintptr_t)ub) | ((uintptr_t)fb0)) & 15) == 0;
      if (wide) {
        constexpr int HW = HX / 2, FW = RX / 2;  // 16-byte chunks per halo / f row
        for (int q = tid; q < HW * HY * (RZ + 2); q += kBoxT) {
          const int c = q / (HW * HY), r = q - c * (HW * HY), bb = r / HW, a = r - bb * HW;
          if (bb < ry + 2 && c < rz + 2)
            box_cp16(&hbuf[slot][c * kHp + bb * kHs + 2 * a], ub + (long long)c * pxy + (long long)bb * px + 2 * a);
        }
        for (int q = tid; q < FW * RY * RZ; q += kBoxT) {
          const int k = q / (FW * RY), r = q - k * (FW * RY), j = r / FW, a = r - j * FW;
          if (j < ry && k < rz)
            box_cp16(&fbuf[slot][(k * RY + j) * RX + 2 * a], fb0 + ((long long)k * ny + j) * nx + 2 * a);
        }
      } else {
        for (int q = tid; q < HN; q += kBoxT) {
          const int c = q / (HX * HY), r = q - c * (HX * HY), bb = r / HX, a = r - bb * HX;
          if (a < rx + 2 && bb < ry + 2 && c < rz + 2)
            box_cp8(&hbuf[slot][c * kHp + bb * kHs + a], ub + (long long)c * pxy + (long long)bb * px + a);
        }
        for (int q = tid; q < NC; q += kBoxT) {
          const int k = q / (RX * RY), r = q - k * (RX * RY), j = r / RX, i = r - j * RX;
          if (i < rx && j < ry && k < rz)
            box_cp8(&fbuf[slot][q], fb0 + ((long long)k * ny + j) * nx + i);
        }
      }
    }
    box_commit();
  };
  __shared__ int gs_b;
  const bool gsp = gsdep != nullptr;
  if (!gsp) stage(blockIdx.x, 0);
  int slot = 0;
  const BoxFac* afF = nullptr;  // factor object whose fragments af/scl hold
  double af[6][2], scl[4];
  for (int b = blockIdx.x;; b += gridDim.x, slot ^= 1) {
    if (gsp) {
      slot = 0;
      if (tid == 0) {
        const int tk = atomicAdd(ticket, 1);
        if (tk < nblocks) {
          const int4 d = gsdep[tk];
          const int pred[3] = {d.y, d.z, d.w};
          for (int q = 0; q < 3; ++q)
            if (pred[q] >= 0)
              while (box_ld_relaxed(flags + pred[q]) == 0) {
              }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        gs_b = tk;
      }
      __syncthreads();
      b = gs_b;
      if (b >= nblocks) break;
      stage(b, 0);
      box_wait<0>();
      __syncthreads();
    } else {
      if (b >= nblocks) break;
      stage(b + gridDim.x, slot ^ 1);
      box_wait<1>();
      __syncthreads();
    }
    const double* hb = hbuf[slot];
    const double* fb = fbuf[slot];
    const int4 B = blocks[b];
    const PatchDev& P = patches[B.x];
    const BoxFac* __restrict__ F = P.bf;
    const int nx = P.nx, ny = P.ny, nz = P.nz;
    const int x0 = B.y, y0 = B.z, z0 = B.w;
    const int rx = min(RX, nx - x0), ry = min(RY, ny - y0), rz = min(RZ, nz - z0);
    const long long px = nx + 2, pxy = px * (ny + 2);
    const int act = active[B.x];
    double* __restrict__ v = P.buf[inplace ? act : act ^ 1];
#pragma unroll
    for (int q0 = 0; q0 < NC; q0 += kBoxT) {
      const int q = q0 + tid;
      const int k = q / (RX * RY), r = q - k * (RX * RY), j = r / RX, i = r - j * RX;
      if (q < NC && i < rx && j < ry && k < rz) {
        const int h = (k + 1) * kHp + (j + 1) * kHs + i + 1;
        wc[k * kRp + j * kRs + i] = residual7(st, fb[q], hb[h], hb[h - 1], hb[h + 1], hb[h - kHs], hb[h + kHs],
                                              hb[h - kHp], hb[h + kHp]);
      }
    }
    __syncthreads();
    bool done = false;
    if constexpr (MX * BX == 8 && MY * BY == 8 && MZ * BZ == 8) {
      if (rx == 8 && ry == 8 && rz == 8) {  // interior region: tensor-core passes
        const int lane = tid & 31, warp = tid >> 5;
        if (F != afF) {  // A fragments of the six transforms and this lane's 1/lambda, per factor object
          afF = F;
          box_afrag<BX>(box_mat(F->F, 0, BX), lane, af[0]);
          box_afrag<BY>(box_mat(F->F, 1, BY), lane, af[1]);
          box_afrag<BZ>(box_mat(F->F, 2, BZ), lane, af[2]);
          box_afrag<BZ>(box_mat(F->B, 2, BZ), lane, af[3]);
          box_afrag<BY>(box_mat(F->B, 1, BY), lane, af[4]);
          box_afrag<BX>(box_mat(F->B, 0, BX), lane, af[5]);
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) {
            const int n0 = 8 * (warp * 2 + tt) + 2 * (lane & 3), pz = lane >> 2;
#pragma unroll
            for (int e = 0; e < 2; ++e)
              scl[2 * tt + e] = box_ilam(F->IL, BX, BY, BZ, ((n0 + e) & 7) % BX, ((n0 + e) >> 3) % BY, pz % BZ);
          }
        }
        box_pass_mma<BX, BY, BZ>(wc, 0, af[0], lane, warp, nullptr);
        __syncthreads();
        box_pass_mma<BX, BY, BZ>(wc, 1, af[1], lane, warp, nullptr);
        __syncthreads();
        box_pass_mma<BX, BY, BZ>(wc, 2, af[2], lane, warp, scl);
        __syncthreads();
        box_pass_mma<BX, BY, BZ>(wc, 2, af[3], lane, warp, nullptr);
        __syncthreads();
        box_pass_mma<BX, BY, BZ>(wc, 1, af[4], lane, warp, nullptr);
        __syncthreads();
        box_pass_mma<BX, BY, BZ>(wc, 0, af[5], lane, warp, nullptr);
        __syncthreads();
#pragma unroll
        for (int q0 = 0; q0 < 512; q0 += kBoxT) {  // relax, row-contiguous stores
          const int q = q0 + tid, k = q >> 6, j = (q >> 3) & 7, i = q & 7;
          const double nv = relax(hb[(k + 1) * kHp + (j + 1) * kHs + i + 1], omega, wc[k * kRp + j * kRs + i]);
          double* vp = v + (long long)(z0 + k + 1) * pxy + (long long)(y0 + j + 1) * px + x0 + i + 1;
          *vp = nv;
          if (!inplace) {
            if (x0 + i == 0) vp[-1] = -nv;
            if (x0 + i == nx - 1) vp[1] = -nv;
          }
        }
        done = true;
      }
    }
    if (!done) {
      // forward x: lines (q, j, k)
  #pragma unroll
      for (int l0 = 0; l0 < MX * RY * RZ; l0 += kBoxT) {
        const int l = l0 + tid, q = l % MX, j = (l / MX) % RY, k = l / (MX * RY), i0 = q * BX;
        if (l < MX * RY * RZ && i0 < rx && j < ry && k < rz) {
          const int ex = min(BX, rx - i0);
          box_line(wc + k * kRp + j * kRs + i0, 1, ex, box_mat(F->F, 0, ex));
        }
      }
      __syncthreads();
  #pragma unroll
      for (int l0 = 0; l0 < MY * RX * RZ; l0 += kBoxT) {  // y: lines (i, q, k)
        const int l = l0 + tid, i = l % RX, q = (l / RX) % MY, k = l / (RX * MY), j0 = q * BY;
        if (l < MY * RX * RZ && i < rx && j0 < ry && k < rz) {
          const int ey = min(BY, ry - j0);
          box_line(wc + k * kRp + j0 * kRs + i, kRs, ey, box_mat(F->F, 1, ey));
        }
      }
      __syncthreads();
  #pragma unroll
      for (int l0 = 0; l0 < MZ * RX * RY; l0 += kBoxT) {  // z: lines (i, j, q), then 1/lambda
        const int l = l0 + tid, i = l % RX, j = (l / RX) % RY, q = l / (RX * RY), k0 = q * BZ;
        if (l < MZ * RX * RY && i < rx && j < ry && k0 < rz) {
          const int ez = min(BZ, rz - k0);
          double* w = wc + k0 * kRp + j * kRs + i;
          box_line(w, kRp, ez, box_mat(F->F, 2, ez));
          const int ib = i % BX, jb = j % BY;
          const int ex = min(BX, rx - (i - ib)), ey = min(BY, ry - (j - jb));
  #pragma unroll
          for (int k = 0; k < BZ; ++k)
            if (k < ez) w[k * kRp] *= box_ilam(F->IL, ex, ey, ez, ib, jb, k);
        }
      }
      __syncthreads();
  #pragma unroll
      for (int l0 = 0; l0 < MZ * RX * RY; l0 += kBoxT) {
        const int l = l0 + tid, i = l % RX, j = (l / RX) % RY, q = l / (RX * RY), k0 = q * BZ;
        if (l < MZ * RX * RY && i < rx && j < ry && k0 < rz) {
          const int ez = min(BZ, rz - k0);
          box_line(wc + k0 * kRp + j * kRs + i, kRp, ez, box_mat(F->B, 2, ez));
        }
      }
      __syncthreads();
  #pragma unroll
      for (int l0 = 0; l0 < MY * RX * RZ; l0 += kBoxT) {
        const int l = l0 + tid, i = l % RX, q = (l / RX) % MY, k = l / (RX * MY), j0 = q * BY;
        if (l < MY * RX * RZ && i < rx && j0 < ry && k < rz) {
          const int ey = min(BY, ry - j0);
          box_line(wc + k * kRp + j0 * kRs + i, kRs, ey, box_mat(F->B, 1, ey));
        }
      }
      __syncthreads();
  #pragma unroll
      for (int l0 = 0; l0 < MX * RY * RZ; l0 += kBoxT) {
        const int l = l0 + tid, q = l % MX, j = (l / MX) % RY, k = l / (MX * RY), i0 = q * BX;
        if (l < MX * RY * RZ && i0 < rx && j < ry && k < rz) {
          const int ex = min(BX, rx - i0);
          double* w = wc + k * kRp + j * kRs + i0;
          box_line(w, 1, ex, box_mat(F->B, 0, ex));
          double* vrow = v + (long long)(z0 + k + 1) * pxy + (long long)(y0 + j + 1) * px + x0 + i0 + 1;
          const double* hrow = hb + (k + 1) * kHp + (j + 1) * kHs + i0 + 1;
  #pragma unroll
          for (int i = 0; i < BX; ++i) {  // (hb of this slot is not restaged before the loop-top barrier)
            if (i < ex) {
              const double nv = relax(hrow[i], omega, w[i]);
              vrow[i] = nv;
              if (!inplace) {
                if (x0 + i0 + i == 0) vrow[i - 1] = -nv;
                if (x0 + i0 + i == nx - 1) vrow[i + 1] = -nv;
              }
            }
          }
        }
      }
    }
    __syncthreads();
    if (gsp && tid == 0) {  // every thread's stores precede the barrier above: release them
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + gsdep[b].x), "r"(1) : "memory");
    }
  }
}

// x = Ainv r for `count` contiguous block vectors of one full box shape
// (x fastest), for BlockFactors.apply / dense().
__global__ void __launch_bounds__(kBoxT) box_apply_kernel(const BoxFac* __restrict__ F, const double* __restrict__ r,
                                                          double* __restrict__ out, long long count) {
  __shared__ double wc[kBoxMax * kRp];
  const int tid = threadIdx.x;
  const int ex = F->bx, ey = F->by, ez = F->bz, n = ex * ey * ez;
  for (long long b = blockIdx.x; b < count; b += gridDim.x) {
    for (int q = tid; q < n; q += kBoxT) {
      const int k = q / (ex * ey), rr = q - k * ex * ey, j = rr / ex, i = rr - j * ex;
      wc[k * kRp + j * kRs + i] = r[b * n + q];
    }
    __syncthreads();
    if (tid < ey * ez) box_line(wc + (tid / ey) * kRp + (tid % ey) * kRs, 1, ex, box_mat(F->F, 0, ex));
    __syncthreads();
    if (tid < ex * ez) box_line(wc + (tid / ex) * kRp + (tid % ex), kRs, ey, box_mat(F->F, 1, ey));
    __syncthreads();
    if (tid < ex * ey) {
      const int i = tid % ex, j = tid / ex;
      double* w = wc + j * kRs + i;
      box_line(w, kRp, ez, box_mat(F->F, 2, ez));
      for (int k = 0; k < ez; ++k) w[k * kRp] *= box_ilam(F->IL, ex, ey, ez, i, j, k);
    }
    __syncthreads();
    if (tid < ex * ey) box_line(wc + (tid / ex) * kRs + (tid % ex), kRp, ez, box_mat(F->B, 2, ez));
    __syncthreads();
    if (tid < ex * ez) box_line(wc + (tid / ex) * kRp + (tid % ex), kRs, ey, box_mat(F->B, 1, ey));
    __syncthreads();
    if (tid < ey * ez) box_line(wc + (tid / ey) * kRp + (tid % ey) * kRs, 1, ex, box_mat(F->B, 0, ex));
    __syncthreads();
    for (int q = tid; q < n; q += kBoxT) {
      const int k = q / (ex * ey), rr = q - k * ex * ey, j = rr / ex, i = rr - j * ex;
      out[b * n + q] = wc[k * kRp + j * kRs + i];
    }
    __syncthreads();
  }
}

// bx, by, bz: the launch's common block dims (0 if the blocks differ);
// shapes of the reference's DEFAULT_BLOCK_SIZES get the compile-time kernel.
cudaError_t launch_box_sweep(const PatchDev* patches, const unsigned char* active, const StencilDev& st,
                             double omega, const int4* blocks, int nblocks, int inplace, int mx, int my, int mz,
                             int bx, int by, int bz, cudaStream_t s, const int4* gsdep, int* flags, int* ticket) {
  if (nblocks <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(nblocks, 16 * sms);
  const bool region = mx * bx == 8 && my * by == 8 && mz * bz == 8;  // Jacobi regions of 8^3
  const bool single = mx == 1 && my == 1 && mz == 1;
#define PSM_BOXT(X, Y, Z)                                                                                      \
  if (bx == X && by == Y && bz == Z) {                                                                        \
    if (region) {                                                                                             \
      box_sweep_t<X, Y, Z, 8 / X, 8 / Y, 8 / Z><<<grid, kBoxT, 0, s>>>(patches, active, st, omega, blocks,    \
                                                                      nblocks, inplace, gsdep, flags, ticket); \
      return cudaGetLastError();                                                                              \
    }                                                                                                         \
    if (single) {                                                                                             \
      box_sweep_t<X, Y, Z, 1, 1, 1><<<grid, kBoxT, 0, s>>>(patches, active, st, omega, blocks, nblocks,       \
                                                           inplace, gsdep, flags, ticket);                    \
      return cudaGetLastError();                                                                              \
    }                                                                                                         \
  }
  PSM_BOXT(2, 2, 2)
  PSM_BOXT(4, 2, 2)
  PSM_BOXT(4, 4, 2)
  PSM_BOXT(4, 4, 4)
  PSM_BOXT(8, 4, 4)
  PSM_BOXT(8, 8, 4)
  PSM_BOXT(8, 8, 8)
#undef PSM_BOXT
  box_sweep_kernel<<<grid, kBoxT, 0, s>>>(patches, active, st, omega, blocks, nblocks, inplace, mx, my, mz);
  return cudaGetLastError();
}

cudaError_t launch_box_apply(const BoxFac* F, const double* r, double* x, long long count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const long long grid = std::min<long long>(count, 148LL * 16);
  box_apply_kernel<<<(unsigned)grid, kBoxT, 0, s>>>(F, r, x, count);
  return cudaGetLastError();
}

}  // namespace psm

using namespace psm;

int psm_set_error(int code, const char* msg);

// Host tables for box blocks up to (ex, ey, ez) of stencil st.
int psm_box_build(const psm_stencil* st, int ex, int ey, int ez, psm_factors* F) {
  const int ext[3] = {ex, ey, ez};
  for (int a = 0; a < 3; ++a)
    if (ext[a] < 1 || ext[a] > kBoxMax)
      return psm_set_error(PSM_EUNSUPPORTED, "box blocks need extents in [1, 8] per axis");
  const long double c = st->center;
  const long double pi = 3.141592653589793238462643383279502884L;
  const size_t nm = 3 * kBoxMax * 64, nl = 3 * kBoxMax * kBoxMax;
  std::vector<double> Fm(nm, 0.0), Bm(nm, 0.0), Lm(nl, 0.0);
  long double off[3], sr[3];
  for (int a = 0; a < 3; ++a) {
    const long double lo = st->faces[2 * a], up = st->faces[2 * a + 1];
    if (lo == 0 && up == 0) {
      off[a] = 0;
      sr[a] = 1;
    } else if (lo * up > 0) {
      off[a] = (lo < 0 ? -1.0L : 1.0L) * sqrtl(lo * up);
      sr[a] = sqrtl(lo / up);
    } else {
      return psm_set_error(PSM_EUNSUPPORTED,
                           "box blocks need the two faces of every axis to share a sign (or both be zero)");
    }
    for (int e = 1; e <= kBoxMax; ++e) {
      const long double sc = sqrtl(2.0L / (e + 1));
      for (int i = 0; i < e; ++i) {
        Lm[(a * kBoxMax + e - 1) * kBoxMax + i] = (double)(2.0L * off[a] * cosl(pi * (i + 1) / (e + 1)));
        for (int p = 0; p < e; ++p) {
          const long double q = sc * sinl(pi * (i + 1) * (p + 1) / (e + 1));
          Fm[(a * kBoxMax + e - 1) * 64 + i * 8 + p] = (double)(q * powl(sr[a], -p));  // Q diag(s^-p)
          Bm[(a * kBoxMax + e - 1) * 64 + p * 8 + i] = (double)(powl(sr[a], p) * q);   // diag(s^p) Q
        }
      }
    }
  }
  // every eigenvalue of every (truncated) shape up to the block must be safe
  for (int a0 = 1; a0 <= ex; ++a0)
    for (int a1 = 1; a1 <= ey; ++a1)
      for (int a2 = 1; a2 <= ez; ++a2)
        for (int i = 0; i < a0; ++i)
          for (int j = 0; j < a1; ++j)
            for (int k = 0; k < a2; ++k) {
              const long double lam = c + 2 * off[0] * cosl(pi * (i + 1) / (a0 + 1)) +
                                      2 * off[1] * cosl(pi * (j + 1) / (a1 + 1)) +
                                      2 * off[2] * cosl(pi * (k + 1) / (a2 + 1));
              if (fabsl(lam) < 1e-14L * fabsl(c))
                return psm_set_error(PSM_ESINGULAR, "box block operator is singular (eigenvalue below 1e-14*|A|)");
            }
  // 1/lambda for every extent combination (ex, ey, ez) in [1, 8]^3, cells (k, j, i) at stride 8
  const size_t ni = 512 * 512;
  std::vector<double> IL(ni, 0.0);
  for (int a0 = 1; a0 <= kBoxMax; ++a0)
    for (int a1 = 1; a1 <= kBoxMax; ++a1)
      for (int a2 = 1; a2 <= kBoxMax; ++a2)
        for (int k = 0; k < a2; ++k)
          for (int j = 0; j < a1; ++j)
            for (int i = 0; i < a0; ++i) {
              const long double lam = c + 2 * off[0] * cosl(pi * (i + 1) / (a0 + 1)) +
                                      2 * off[1] * cosl(pi * (j + 1) / (a1 + 1)) +
                                      2 * off[2] * cosl(pi * (k + 1) / (a2 + 1));
              if (fabsl(lam) >= 1e-14L * fabsl(c))  // unreachable shapes of a singular stencil stay 0
                IL[((((a0 - 1) * 8 + (a1 - 1)) * 8 + (a2 - 1)) * 512) + (k * 8 + j) * 8 + i] = (double)(1.0L / lam);
            }
  const size_t bytes = sizeof(BoxFac) + (2 * nm + nl + ni) * sizeof(double);
  if (cudaMalloc(&F->dev, bytes) != cudaSuccess) return psm_set_error(PSM_ENOMEM, "cudaMalloc for box factors");
  double* tab = (double*)((char*)F->dev + sizeof(BoxFac));
  BoxFac& H = F->h_box;
  memset(&H, 0, sizeof H);
  H.bx = ex;
  H.by = ey;
  H.bz = ez;
  H.c = st->center;
  H.F = tab;
  H.B = tab + nm;
  H.L = tab + 2 * nm;
  H.IL = tab + 2 * nm + nl;
  F->d_box = (BoxFac*)F->dev;
  if (cudaMemcpy(F->dev, &H, sizeof H, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tab, Fm.data(), nm * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tab + nm, Bm.data(), nm * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tab + 2 * nm, Lm.data(), nl * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tab + 2 * nm + nl, IL.data(), ni * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return psm_set_error(PSM_ECUDA, "uploading box factors");
  return PSM_OK;
}
