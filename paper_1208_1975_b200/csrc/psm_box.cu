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
// over a region list, six CTAs per SM.  The region's u with a one-cell halo
// and its f are staged in shared memory (TMA tensor copies, double-buffered;
// cp.async for odd widths), the residual is formed in the reference
// operation order.  Interior 8^3 regions run the six 1-D transforms as DMMA
// m8n8k4 passes with the data in fragment registers (box_sweep_t, below);
// edge regions run them with one thread per block line.  The 1/lambda
// scaling (host table per extent triple) is folded into the last forward
// pass and the relaxation into the last backward pass.  Jacobi writes v (and
// v's physical x-ghosts) for all blocks in one launch.  GS updates u in
// place in one persistent launch per sweep: blocks are handed out in
// wavefront order (bi + bj + bk = w; face-adjacent blocks lie on
// neighbouring wavefronts) and each waits for its three lexicographic
// predecessors' flags, so the order is exactly the lexicographic one of
// runtime.py:164-168 (PSM_BOX_GS_WAVES=1: one launch per wavefront).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <cuda.h>

#include <algorithm>
#include <vector>

#include "psm_async.cuh"
#include "psm_internal.cuh"

namespace psm {

constexpr int kBoxMax = 8;     // largest extent per axis
constexpr int kBoxT = 128;     // threads per block CTA
constexpr int kHs = 10;        // halo box row stride (ex + 2 <= 10)
constexpr int kHp = 100;       // halo box plane stride
constexpr int kHslot = 1008;   // halo staging slot (kHp * 10 rounded to 128 bytes, for TMA)
constexpr int kTmapBytes = 128;  // sizeof(CUtensorMap)
#ifndef PSM_BOX_MINB
// resident CTAs per SM the sweep kernel is register-limited to (6: 80
// registers; holding the DMMA A fragments in registers instead of shared
// memory needs 5 and measured 13% slower on F1)
#define PSM_BOX_MINB 6
#endif
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
// Interior 8^3 regions run the six transforms as DMMA m8n8k4 passes with the
// data in fragment registers: lane (r = lane/4, c = lane%4) of warp w holds,
// per tile tt (plane 2w+tt), the B operand X[4ks+c][r] and the result D[r][2c+e].
// Only the two axis changes that cross warps (y -> z, z -> y) go through the
// work cube; x -> y, z -> z' and y' -> x' are register shuffles.  The line
// orders below make every shared-memory access conflict-free (two wavefronts
// per 8-byte warp access; tools/box_lanes_sim.py checks the orders, the
// conflicts and the arithmetic):
//   x pass    line r -> row j = box_jx(r)       (residual loads from the halo)
//   y pass    line r -> column i = box_ip(r)    (results stored to the cube)
//   z, z'     line r -> i = r, i = box_ip(r)    (z' results stored to the cube)
//   y', x'    line r -> i = r, j = r            (x' results relaxed from registers)
__device__ __forceinline__ int box_jx(int n) { return 2 * (n & 3) + (n >> 2); }
__device__ __forceinline__ int box_ip(int n) { return (n >> 1) + 4 * (n & 1); }
__device__ __forceinline__ void box_mma2(const double (&a)[2], const double (&bq)[2], double (&d)[2]) {
  d[0] = 0.0;
  d[1] = 0.0;
  box_dmma(d[0], d[1], a[0], bq[0]);
  box_dmma(d[0], d[1], a[1], bq[1]);
}
// One register exchange between passes: every lane needs two of the 64
// values its warp holds (two per lane).  Two shuffles suffice: in each, every
// lane sends the element (pick ? d[1] : d[0], then the other) that its one
// reader needs and reads from src0 / src1; `swap` says which received value
// is the lane's ks = 0 operand.  tools/box_lanes_sim.py derives and checks
// the three schedules (x -> y, z -> z', y' -> x').
__device__ __forceinline__ void box_exchange(const double (&d)[2], bool pick, int src0, int src1, bool swap,
                                             double (&bq)[2]) {
  const double s0 = __shfl_sync(0xffffffffu, pick ? d[1] : d[0], src0);
  const double s1 = __shfl_sync(0xffffffffu, pick ? d[0] : d[1], src1);
  bq[0] = swap ? s1 : s0;
  bq[1] = swap ? s0 : s1;
}

template <int BX, int BY, int BZ, int MX, int MY, int MZ, int GS>
__global__ void __launch_bounds__(kBoxT, PSM_BOX_MINB) box_sweep_t(const PatchDev* __restrict__ patches,
                                                     const unsigned char* __restrict__ active, StencilDev st,
                                                     double omega, const int4* __restrict__ blocks, int nblocks,
                                                     int inplace, const int4* __restrict__ gsdep, int* flags,
                                                     int* ticket, const char* __restrict__ tmaps) {
  constexpr int RX = BX * MX, RY = BY * MY, RZ = BZ * MZ;
  constexpr int HX = RX + 2, HY = RY + 2, HN = HX * HY * (RZ + 2);
  constexpr int NC = RX * RY * RZ;
  // 8^3 regions: the halo box is staged dense (10^3: row stride kHs, plane
  // stride kHp) and f with row stride 10 (conflict-free fragment loads), so
  // two TMA tensor copies (one thread) replace ~760 cp.async requests
  constexpr bool kShape8 = RX == 8 && RY == 8 && RZ == 8;
  constexpr int FS = kShape8 ? 10 : RX;  // f staging row stride
  constexpr int FN = FS * RY * RZ;
  const bool tma = kShape8 && tmaps != nullptr;
  // double-buffered staging: the next region's u halo and f stream in
  // while this region computes (the sweep is otherwise latency-bound)
  __shared__ __align__(128) double hbuf[2][kHslot];
  __shared__ __align__(128) double fbuf[2][FN];
  __shared__ double wc[kBoxMax * kRp];
  __shared__ uint64_t tbar[2];
  const int tid = threadIdx.x;
  uint32_t tphase = 0;  // parity of each slot's next TMA completion
  if (tma) {
    if (tid == 0) {
      async::bar_init(&tbar[0], 1);
      async::bar_init(&tbar[1], 1);
      async::bar_fence_init();
    }
    __syncthreads();
  }
  // one thread: the TMA copies of region B (active buffer act) into a slot
  auto stage_tma = [&](int slot, int4 B, int act) {
    const char* m = tmaps + (size_t)(3 * B.x) * kTmapBytes;
    async::bar_expect(&tbar[slot], (uint32_t)((kHp * kHs + FN) * sizeof(double)));
    async::tensor3d_g2s(&hbuf[slot][0], m + act * kTmapBytes, B.y, B.z, B.w, &tbar[slot]);
    async::tensor3d_g2s(&fbuf[slot][0], m + 2 * kTmapBytes, B.y, B.z, B.w, &tbar[slot]);
  };
  auto stage = [&](int b, int slot) {
    if (tma) {
      if (tid == 0 && b < nblocks) {
        const int4 B = blocks[b];
        stage_tma(slot, B, active[B.x]);
      }
      return;
    }
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
            box_cp16(&fbuf[slot][(k * RY + j) * FS + 2 * a], fb0 + ((long long)k * ny + j) * nx + 2 * a);
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
            box_cp8(&fbuf[slot][(k * RY + j) * FS + i], fb0 + ((long long)k * ny + j) * nx + i);
        }
      }
    }
    box_commit();
  };
  __shared__ int gs_b, gs_nxt[2];
  const bool gsp = GS && gsdep != nullptr;  // (GS = 0: the persistent-GS code compiles away)
  // GS with TMA staging: the block's thread 0 runs a ticket pipeline off the
  // CTA's critical path.  Besides the block it computes it holds the next
  // ticket tA (whose halo goes to the other slot: its predecessors' flags are
  // loaded at the end of the previous block and checked after this block's
  // first and second barriers) and the one after, tB (taken at the end of
  // the previous block, its dependencies loaded after the first barrier).  Thread 0 only
  // ever blocks on tA after releasing the current block, and tB > tA: every
  // unfinished ticket's predecessors are held by CTAs that make progress.
  const bool gpre = gsp && tma;
  auto gs_acquire = [&]() {
    // acquire pattern with the relaxed flag loads (fence.acquire: an L1
    // invalidate only, no wait for this thread's own outstanding stores)
    asm volatile("fence.acquire.gpu;" ::: "memory");
    // the TMA reads of the halo go through the async proxy
    if (tma) asm volatile("fence.proxy.async.global;" ::: "memory");
  };
  auto gs_wait = [&](int4 d) {
    const int pred[3] = {d.y, d.z, d.w};
    for (int q = 0; q < 3; ++q)
      if (pred[q] >= 0)
        while (box_ld_relaxed(flags + pred[q]) == 0) {
        }
    gs_acquire();
  };
  const int4 kNoDeps = make_int4(-1, -1, -1, -1);
  int tA = 0, tB = 0, fA0 = 1, fA1 = 1, fA2 = 1, aA = 0;
  int4 dA = kNoDeps, dB = kNoDeps, bA = kNoDeps, bB = kNoDeps;  // deps and region of tA / tB
  bool stgA = false;
  auto poll_issue = [&]() {  // loads only: the values are checked later
    fA0 = dA.y >= 0 ? box_ld_relaxed(flags + dA.y) : 1;
    fA1 = dA.z >= 0 ? box_ld_relaxed(flags + dA.z) : 1;
    fA2 = dA.w >= 0 ? box_ld_relaxed(flags + dA.w) : 1;
  };
  auto gs_hook = [&](int slot, bool first) {  // thread 0, right after a barrier of the block
    if (tA < nblocks && !stgA) {
      if (fA0 && fA1 && fA2) {
        gs_acquire();
        stage_tma(slot ^ 1, bA, aA);
        stgA = true;
      } else {
        poll_issue();
      }
    }
    if (first && tB < nblocks) {  // loads for the ticket after next, used at the end of the block
      dB = gsdep[tB];
      bB = blocks[tB];
    }
  };
  if (!gsp) stage(blockIdx.x, 0);
  int slot = 0, gcur = 0;
  if (gpre) {
    if (tid == 0) {
      const int tk = atomicAdd(ticket, 1);
      if (tk < nblocks) {
        gs_wait(gsdep[tk]);
        stage(tk, 0);
      }
      gs_b = tk;
      tA = atomicAdd(ticket, 1);
      if (tA < nblocks) {
        dA = gsdep[tA];
        bA = blocks[tA];
        aA = active[bA.x];
      }
      tB = atomicAdd(ticket, 1);
      poll_issue();
    }
    __syncthreads();
    gcur = gs_b;
  }
  const BoxFac* afF = nullptr;  // factor object whose fragments afs/scl hold
  double scl[2][2];
  __shared__ double afs[6][2][32];  // A fragments of the six transforms (lane-indexed)
  const int lane = tid & 31, warp = tid >> 5, lr = lane >> 2, lc = lane & 3;
  for (int b = blockIdx.x;; b += gridDim.x, slot ^= 1) {
    if (gpre) {
      b = gcur;
      if (b >= nblocks) break;
      if (tid == 0) {
        gs_nxt[slot] = tA;
        stgA = false;
      }
      async::bar_wait(&tbar[slot], (tphase >> slot) & 1);
      tphase ^= 1u << slot;
    } else if (gsp) {
      slot = 0;
      if (tid == 0) {
        const int tk = atomicAdd(ticket, 1);
        if (tk < nblocks) gs_wait(gsdep[tk]);
        gs_b = tk;
      }
      __syncthreads();
      b = gs_b;
      if (b >= nblocks) break;
      stage(b, 0);
      if (tma) {
        async::bar_wait(&tbar[0], tphase & 1);
        tphase ^= 1;
      } else {
        box_wait<0>();
      }
      __syncthreads();
    } else {
      if (b >= nblocks) break;
      if (!tma) stage(b + gridDim.x, slot ^ 1);  // (TMA: issued after the first barrier below)
      if (tma) {
        async::bar_wait(&tbar[slot], (tphase >> slot) & 1);
        tphase ^= 1u << slot;
      } else {
        box_wait<1>();
        __syncthreads();
      }
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
    bool interior8 = false;
    if constexpr (MX * BX == 8 && MY * BY == 8 && MZ * BZ == 8) interior8 = rx == 8 && ry == 8 && rz == 8;
    if (!interior8) {
      // edge region (or a TMA-less launch still holding the other slot's copy):
      // the prefetch of the next region cannot wait for the first barrier
      // (an interior region before this one ends without a barrier)
      if (tma && !gsp) {
        __syncthreads();
        stage(b + gridDim.x, slot ^ 1);
      }
#pragma unroll
      for (int q0 = 0; q0 < NC; q0 += kBoxT) {
        const int q = q0 + tid;
        const int k = q / (RX * RY), r = q - k * (RX * RY), j = r / RX, i = r - j * RX;
        if (q < NC && i < rx && j < ry && k < rz) {
          const int h = (k + 1) * kHp + (j + 1) * kHs + i + 1;
          wc[k * kRp + j * kRs + i] = residual7(st, fb[(k * RY + j) * FS + i], hb[h], hb[h - 1], hb[h + 1],
                                                hb[h - kHs], hb[h + kHs], hb[h - kHp], hb[h + kHp]);
        }
      }
      __syncthreads();
      if (gpre && tid == 0) gs_hook(slot, true);
    }
    if constexpr (MX * BX == 8 && MY * BY == 8 && MZ * BZ == 8) {
      if (interior8) {
        if (F != afF) {  // A fragments of the six transforms and this lane's 1/lambda, per factor object
          afF = F;
          if (warp == 0) {
            double a[2];
            box_afrag<BX>(box_mat(F->F, 0, BX), lane, a);
            afs[0][0][lane] = a[0], afs[0][1][lane] = a[1];
            box_afrag<BY>(box_mat(F->F, 1, BY), lane, a);
            afs[1][0][lane] = a[0], afs[1][1][lane] = a[1];
            box_afrag<BZ>(box_mat(F->F, 2, BZ), lane, a);
            afs[2][0][lane] = a[0], afs[2][1][lane] = a[1];
            box_afrag<BZ>(box_mat(F->B, 2, BZ), lane, a);
            afs[3][0][lane] = a[0], afs[3][1][lane] = a[1];
            box_afrag<BY>(box_mat(F->B, 1, BY), lane, a);
            afs[4][0][lane] = a[0], afs[4][1][lane] = a[1];
            box_afrag<BX>(box_mat(F->B, 0, BX), lane, a);
            afs[5][0][lane] = a[0], afs[5][1][lane] = a[1];
          }
          // z-pass result (k = lr, i = 2 lc + e) of the plane j = 2 warp + tt
#pragma unroll
          for (int tt = 0; tt < 2; ++tt)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              scl[tt][e] = box_ilam(F->IL, BX, BY, BZ, (2 * lc + e) % BX, (2 * warp + tt) % BY, lr % BZ);
          __syncthreads();  // afs (F is uniform over the CTA)
        }
        double bq[2][2], d[2][2];
#define PSM_BOX_A(P) const double A##P[2] = {afs[P][0][lane], afs[P][1][lane]};
        // residual (reference operation order) straight into the x-pass B
        // fragments: cells (i = 4 ks + lc, j = box_jx(lr), k = 2 warp + tt)
        // (the two planes of a lane are each other's z neighbours)
        const int jr = box_jx(lr);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int k = 2 * warp, i = 4 * ks + lc;
          const int h = (k + 1) * kHp + (jr + 1) * kHs + i + 1, h1 = h + kHp;
          const double c0 = hb[h], c1 = hb[h1];
          bq[0][ks] = residual7(st, fb[(k * 8 + jr) * FS + i], c0, hb[h - 1], hb[h + 1], hb[h - kHs], hb[h + kHs],
                                hb[h - kHp], c1);
          bq[1][ks] = residual7(st, fb[((k + 1) * 8 + jr) * FS + i], c1, hb[h1 - 1], hb[h1 + 1], hb[h1 - kHs],
                                hb[h1 + kHs], c0, hb[h1 + kHp]);
        }
        // x pass; x -> y by shuffle: lane needs (i = box_ip(lr), j = 4 ks + lc)
PSM_BOX_A(0)
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) box_mma2(A0, bq[tt], d[tt]);
        {  // lane (lr, lc) reads lane (box_ip(lr), {0,2,1,3}[lc]) then (.., {1,3,0,2}[lc])
          const int s0 = box_ip(lr) * 4 + (((lc & 1) << 1) | (lc >> 1));
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) box_exchange(d[tt], lc & 1, s0, s0 ^ 1, lc >> 1, bq[tt]);
        }
        // y pass -> cube (k = 2 warp + tt, j = lr, i = box_ip(2 lc + e))
PSM_BOX_A(1)
        __syncwarp();  // the warp's y'-pass cube reads of the previous region precede these stores
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          box_mma2(A1, bq[tt], d[tt]);
#pragma unroll
          for (int e = 0; e < 2; ++e) wc[(2 * warp + tt) * kRp + lr * kRs + box_ip(2 * lc + e)] = d[tt][e];
        }
        __syncthreads();
        // every warp is past this region's halo reads of the previous slot:
        // prefetch the next region into it
        if (tma && !gsp) stage(b + gridDim.x, slot ^ 1);
        if (gpre && tid == 0) gs_hook(slot, true);
        // z pass (plane j = 2 warp + tt, line i = lr), scaled by 1/lambda;
        // z -> z' by shuffle: lane needs (k = 4 ks + lc, i = box_ip(lr))
PSM_BOX_A(2)
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) bq[tt][ks] = wc[(4 * ks + lc) * kRp + (2 * warp + tt) * kRs + lr];
          box_mma2(A2, bq[tt], d[tt]);
          d[tt][0] *= scl[tt][0];
          d[tt][1] *= scl[tt][1];
        }
        {  // lane reads row k = lc or 4 + lc (first the one of its own parity e) at column box_ip(lr) / 2
          const int ir = box_ip(lr), e = ir & 1;
          const int s0 = ((e ? 4 : 0) + lc) * 4 + (ir >> 1), s1 = ((e ? 0 : 4) + lc) * 4 + (ir >> 1);
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) box_exchange(d[tt], lr >= 4, s0, s1, e, bq[tt]);
        }
        // z' pass -> cube (k = lr, j = 2 warp + tt, i = box_ip(2 lc + e))
PSM_BOX_A(3)
        __syncwarp();  // the warp's z-pass cube reads precede these stores (WAR across lanes)
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          box_mma2(A3, bq[tt], d[tt]);
#pragma unroll
          for (int e = 0; e < 2; ++e) wc[lr * kRp + (2 * warp + tt) * kRs + box_ip(2 * lc + e)] = d[tt][e];
        }
        __syncthreads();
        if (gpre && tid == 0) gs_hook(slot, false);
        // y' pass (plane k = 2 warp + tt, line i = lr); y' -> x' by shuffle:
        // lane needs (j = lr, i = 4 ks + lc)
PSM_BOX_A(4)
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) bq[tt][ks] = wc[(2 * warp + tt) * kRp + (4 * ks + lc) * kRs + lr];
          box_mma2(A4, bq[tt], d[tt]);
        }
        {  // within the quad: columns (lc >> 1) + 2 (lc & 1), then (lc >> 1) + 2 (1 - (lc & 1))
          const int s0 = lr * 4 + (lc >> 1) + 2 * (lc & 1), s1 = lr * 4 + (lc >> 1) + 2 * ((lc & 1) ^ 1);
#pragma unroll
          for (int tt = 0; tt < 2; ++tt) box_exchange(d[tt], lc >> 1, s0, s1, lc & 1, bq[tt]);
        }
        // x' pass: result (i = lr, j = 2 lc + e, k = 2 warp + tt); relax and store
PSM_BOX_A(5)
        #pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          box_mma2(A5, bq[tt], d[tt]);
          const int k = 2 * warp + tt;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int j = 2 * lc + e;
            const double nv = relax(hb[(k + 1) * kHp + (j + 1) * kHs + lr + 1], omega, d[tt][e]);
            double* vp = v + (long long)(z0 + k + 1) * pxy + (long long)(y0 + j + 1) * px + x0 + lr + 1;
            *vp = nv;
            if (!inplace) {
              if (x0 + lr == 0) vp[-1] = -nv;
              if (x0 + lr == nx - 1) vp[1] = -nv;
            }
          }
        }
#undef PSM_BOX_A
      }
    }
    if (!interior8) {
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
          for (int i = 0; i < BX; ++i) {  // (hb of this slot is not restaged before the loop-end barrier)
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
    // the interior path needs no barrier here: its cube accesses after the
    // second barrier are warp-local and the next prefetch waited for the
    // first; edge regions, the cp.async staging and the GS release do
    if (!interior8 || !tma || gsp) __syncthreads();
    if (gsp && tid == 0)  // every thread's stores precede the barrier above: the release covers them
      asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + gsdep[b].x), "r"(1) : "memory");
    if (gpre) {
      if (tid == 0) {
        if (tA < nblocks && !stgA) {  // not prefetched: wait now (this block is released)
          gs_wait(dA);
          stage_tma(slot ^ 1, bA, aA);
        }
        tA = tB;
        dA = dB;
        bA = bB;
        if (tA < nblocks) aA = active[bA.x];
        poll_issue();  // checked after the next block's first barrier
        tB = atomicAdd(ticket, 1);
      }
      gcur = gs_nxt[slot];
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

// Tensor maps for the TMA staging of 8^3 regions, 3 per patch: buf[0] and
// buf[1] (padded (nx+2, ny+2, nz+2), box 10^3) and f ((nx, ny, nz), box
// 10 x 8 x 8: rows padded to the staging stride FS).  Needs 16-byte aligned bases and strides (nx even); *out stays null
// (cp.async staging) otherwise, or with PSM_BOX_TMA=0.
typedef CUresult (*EncodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
cudaError_t box_build_tmaps(const PatchDev* hp, int npatch, void** out) {
  *out = nullptr;
  const char* env = getenv("PSM_BOX_TMA");
  if (env && env[0] == '0') return cudaSuccess;
  static EncodeTiled_t encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (EncodeTiled_t)fn;
  }();
  if (!encode || npatch <= 0) return cudaSuccess;
  static_assert(sizeof(CUtensorMap) == kTmapBytes, "tensor map size");
  std::vector<CUtensorMap> maps(3 * (size_t)npatch);
  for (int p = 0; p < npatch; ++p) {
    const PatchDev& h = hp[p];
    if ((h.nx & 1) || (((uintptr_t)h.buf[0] | (uintptr_t)h.buf[1] | (uintptr_t)h.f) & 15)) return cudaSuccess;
    for (int k = 0; k < 3; ++k) {
      const bool fmap = k == 2;
      const cuuint64_t dims[3] = {(cuuint64_t)h.nx + (fmap ? 0 : 2), (cuuint64_t)h.ny + (fmap ? 0 : 2),
                                  (cuuint64_t)h.nz + (fmap ? 0 : 2)};
      const cuuint64_t strides[2] = {dims[0] * 8, dims[0] * dims[1] * 8};
      const cuuint32_t box[3] = {10u, fmap ? 8u : 10u, fmap ? 8u : 10u};  // f rows padded to 10 (FS)
      const cuuint32_t estr[3] = {1, 1, 1};
      void* base = fmap ? (void*)h.f : (void*)h.buf[k];
      if (encode(&maps[3 * p + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaSuccess;
    }
  }
  void* d = nullptr;
  cudaError_t e = cudaMalloc(&d, maps.size() * sizeof(CUtensorMap));
  if (e == cudaSuccess) e = cudaMemcpy(d, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(d);
    return e;
  }
  *out = d;
  return cudaSuccess;
}

// bx, by, bz: the launch's common block dims (0 if the blocks differ);
// shapes of the reference's DEFAULT_BLOCK_SIZES get the compile-time kernel.
cudaError_t launch_box_sweep(const PatchDev* patches, const unsigned char* active, const StencilDev& st,
                             double omega, const int4* blocks, int nblocks, int inplace, int mx, int my, int mz,
                             int bx, int by, int bz, cudaStream_t s, const int4* gsdep, int* flags, int* ticket,
                             const void* tmaps) {
  if (nblocks <= 0) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(nblocks, 16 * sms);  // persistent over the region list
  const bool region = mx * bx == 8 && my * by == 8 && mz * bz == 8;  // Jacobi regions of 8^3
  const bool single = mx == 1 && my == 1 && mz == 1;
  const char* tm = (const char*)tmaps;
#define PSM_BOXK(X, Y, Z, M1, M2, M3, G)                                                                     \
  {                                                                                                           \
    cudaFuncSetAttribute(box_sweep_t<X, Y, Z, M1, M2, M3, G>, cudaFuncAttributePreferredSharedMemoryCarveout, \
                         cudaSharedmemCarveoutMaxShared);                                                     \
    box_sweep_t<X, Y, Z, M1, M2, M3, G><<<grid, kBoxT, 0, s>>>(patches, active, st, omega, blocks, nblocks,   \
                                                               inplace, gsdep, flags, ticket, tm);            \
    return cudaGetLastError();                                                                                \
  }
#define PSM_BOXT(X, Y, Z)                                      \
  if (bx == X && by == Y && bz == Z) {                        \
    if (region && !gsdep) PSM_BOXK(X, Y, Z, 8 / X, 8 / Y, 8 / Z, 0) \
    if (single && gsdep) PSM_BOXK(X, Y, Z, 1, 1, 1, 1)        \
    if (single) PSM_BOXK(X, Y, Z, 1, 1, 1, 0)                 \
  }
  PSM_BOXT(2, 2, 2)
  PSM_BOXT(4, 2, 2)
  PSM_BOXT(4, 4, 2)
  PSM_BOXT(4, 4, 4)
  PSM_BOXT(8, 4, 4)
  PSM_BOXT(8, 8, 4)
  PSM_BOXT(8, 8, 8)
#undef PSM_BOXT
#undef PSM_BOXK
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
