// Line-block Jacobi sweep, z-marching TMA pipeline (sm_100a).
//
// Replaces smoother._jacobi_step + block_residual + block_update/matvec
// (smoother.py:138-153, stencil.py:93-112, blocklinalg.py:90-105) for line
// blocks (>=nx,1,1) and power-of-two nx in [64, 1024].
//
// Work unit: one column of R = 2048/nx consecutive x-lines (rows j0..j0+R-1)
// over a chunk of planes k0..k1-1 of one patch.  Persistent CTAs (one per SM)
// take units in (patch, chunk, column) order, so concurrently running CTAs
// march neighbouring columns through the same planes and the y-halo rows one
// CTA re-reads are L2 hits; u and f stream from HBM once (24 B/update).
//
// Warp roles (608 threads):
//   warp 18      producer: cp.async.bulk (TMA, 1-D) of each plane's u slab
//                (R+2 padded rows incl. both y-halo rows, contiguous in
//                memory) into a 4-slot ring and of f's R rows into a 2-slot
//                ring, completion via mbarrier transaction counts.
//   warps 0-15   A/C: each thread owns 4 cells of the column and keeps a
//                register queue u(k-1), u(k), u(k+1) for them, so per plane it
//                reads only the new plane's centre, u(j+-1) and f from shared
//                memory; x+-1 come by warp shuffle.  A(k): residual in the
//                reference operation order -> padded r buffer, r^2 partial.
//                C(k-1): x = y - cl*g - cr*h, v = u + omega*x, store v and
//                the physical x-face ghosts of v.
//   warps 16-17  solver: one lane per 32-cell segment (64 segments per tile):
//                Thomas with constant factors, segment ends exchanged by
//                shuffle, exact 2x2 interface solves -> cl, cr; also the
//                tile's r^2 partial.  B(k) overlaps A(k+1) of the A/C warps
//                (double-buffered r / y buffers, named barriers).
#include <stdint.h>
#include <string.h>

#include <type_traits>

#include "psm_internal.cuh"

namespace psm {

struct ZUnit {
  int patch, j0, k0, k1;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "MBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// f is read once: its bulk copies carry an L2 evict-first policy, so the
// u rows the neighbouring columns re-read as y-halos stay resident longer
__device__ __forceinline__ void tma_load_1d_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int NX>
struct ZCfg {
  static constexpr int R = kMaxTileCells / NX;  // rows per column
  static constexpr int PX = NX + 2;
  static constexpr int NSEG = NX / kSeg;
  static constexpr int NSL = R * NSEG;  // 64 segment lanes
  static constexpr int RS = NX + NSEG;  // padded r row
  // ring slots; deeper rings (4/3, 4/4, 5/3) measured no better on B200
  // (tools/ztune.sh: within +-3% run to run at 512^3 and 1024^3)
#ifdef PSM_ZNU
  static constexpr int NU = PSM_ZNU, NF = PSM_ZNF;  // tuning builds
#else
  static constexpr int NU = 4, NF = 2;
#endif
  static constexpr int US = (R + 2) * PX;  // doubles per u slot
  static constexpr int FS = R * NX;
  static constexpr int RB = R * RS;
  static constexpr int AC_WARPS = 16, SOLVER_WARPS = 2, THREADS = (AC_WARPS + SOLVER_WARPS + 1) * 32;
  static constexpr int ACT = AC_WARPS * 32;
  static constexpr int E = kMaxTileCells / ACT;  // cells per A/C thread (4)
  static constexpr size_t SMEM_DOUBLES = (size_t)NU * US + NF * FS + 2 * RB + 2 * AC_WARPS;
  static constexpr size_t SMEM_BYTES = SMEM_DOUBLES * 8 + (2 * NU + 2 * NF) * 8 + 16;
};

constexpr int kBarR = 1, kBarY = 3, kBarRes = 5;

// Factor tables passed by value: they live in the kernel-parameter constant
// bank, so the fully unrolled solver reads them as DFMA constant operands
// (no load instructions).
struct ZTab {
  double invm[kSeg], loinv[kSeg], cp[kSeg], g[kSeg], h[kSeg], g16[16], h16[16];
  double lo, up, up_h31, lo_g0, d_full, up_h16, lo_g16, d16;
};

// cell q of A/C thread tid (0..ACT-1) in a tile of 2048/NX rows: cells
// e = q*ACT + tid, row = e / NX, x = e % NX, folded at compile time
template <int NX, int ACT>
__device__ __forceinline__ int cell_row(int q, int tid) {
  if constexpr (NX >= ACT) return (q * ACT) / NX;
  else return q * (ACT / NX) + tid / NX;
}
template <int NX, int ACT>
__device__ __forceinline__ int cell_x(int q, int tid) {
  if constexpr (NX >= ACT) return (q * ACT) % NX + tid;
  else return tid % NX;
}  // named barriers 1,2 (r ready) and 3,4 (y ready)

// A/C warp role of the z-marching kernel.  Thread t owns NXP x-positions
// and RPT consecutive rows of the column (E = NXP*RPT = 4 cells), so the
// y-neighbours inside its rows come from its own registers; only the first
// row's y-1 and the last row's y+1 are read from the slab.  Three register
// arrays rotate through the roles u(k-1), u(k), u(k+1) (the plane loop is
// unrolled by three, so the queue never moves data).
template <int NX, int UNIT, int RES>
struct ZAC {
  using C = ZCfg<NX>;
  static constexpr int R = C::R, PX = C::PX, RS = C::RS, E = C::E, ACT = C::ACT;
  static constexpr bool NX_GE = NX >= ACT;
  static constexpr int NXP = NX_GE ? NX / ACT : 1;
  static constexpr int RPT = E / NXP;
  static constexpr int NBAR = (C::AC_WARPS + C::SOLVER_WARPS) * 32;

  int tid, lane, warp, tx, trow0, rows, j0, k0;
  StencilDev st;
  double omega;
  double *uring, *fring, *rbuf, *wsum, *v;
  double* peer_lo = nullptr;   // neighbour below: its v buffer (we fill its top ghost plane)
  double* peer_hi = nullptr;   // neighbour above: its v buffer (we fill its bottom ghost plane)
  long long peer_lo_off = 0, peer_hi_off = 0;  // added to our v index of plane 0 / nz-1
  int kw = 0, nz = 0;          // plane phaseC writes, planes of the patch
  double* rg = nullptr;        // RES: global residual of this patch (cell-major like f)
  double* partials = nullptr;  // RES: per (plane, tile) r^2 partials
  long long tslot0 = 0;        // RES: partial index of plane 0's tile
  int tpp = 0, ny = 0;
  uint64_t *full_u, *empty_u, *full_f, *empty_f;
  long long pxy, vbase_old = 0;
  uint32_t nu = 0, nf = 0;
  int b = 0, s_cur = 0;
  double A0[E], A1[E], A2[E];

  __device__ __forceinline__ void load_c(double (&dst)[E], const double* sl) const {
#pragma unroll
    for (int p = 0; p < NXP; ++p)
#pragma unroll
      for (int r = 0; r < RPT; ++r) dst[p * RPT + r] = sl[(trow0 + r + 1) * PX + tx + p * ACT + 1];
  }

  template <bool FULL>
  __device__ __forceinline__ void phaseC(const double (&cold)[E]) {
    const int bo = b ^ 1;
    named_sync(kBarY + bo, NBAR);
    const double* xb = rbuf + bo * C::RB;
#pragma unroll
    for (int p = 0; p < NXP; ++p)
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int row = trow0 + r, x = tx + p * ACT;
        if (FULL || row < rows) {
          const double nv = relax(cold[p * RPT + r], omega, xb[row * RS + x + (x >> 5)]);
          const long long iu = vbase_old + (long long)row * PX + x;
#ifdef PSM_ZMARCH_NO_HINT
          v[iu] = nv;
#else
          __stcs(v + iu, nv);  // streaming store: v is not re-read by this sweep
#endif
          if constexpr (NX_GE) {
            if (p == 0 && tid == 0) v[iu - 1] = -nv;
            if (p == NXP - 1 && tid == ACT - 1) v[iu + 1] = -nv;
          } else {
            if (x == 0) v[iu - 1] = -nv;
            if (x == NX - 1) v[iu + 1] = -nv;
          }
        }
      }
    // fused halo: a boundary plane also lands in the neighbour's ghost plane
    // (CTA-uniform and rare, kept out of the loop above)
    double* pl = kw == 0 ? peer_lo : nullptr;
    double* ph = kw == nz - 1 ? peer_hi : nullptr;
    if (RES == 2 && (pl != nullptr || ph != nullptr)) {
      if (pl) pl += peer_lo_off;
      if (ph) ph += peer_hi_off;
#pragma unroll
      for (int p = 0; p < NXP; ++p)
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int row = trow0 + r, x = tx + p * ACT;
          if (FULL || row < rows) {
            const double nv = relax(cold[p * RPT + r], omega, xb[row * RS + x + (x >> 5)]);
            const long long iu = vbase_old + (long long)row * PX + x;
            if (pl) pl[iu] = nv;
            if (ph) ph[iu] = nv;
          }
        }
    }
  }

  // plane k: A(k) then C(k-1)
  template <bool FULL>
  __device__ __forceinline__ void step(const double (&zm)[E], const double (&c)[E], double (&zp)[E], int k) {
    const int s_nxt = nu % C::NU;
    mbar_wait(&full_u[s_nxt], (nu / C::NU) & 1);
    ++nu;
    const int t = nf % C::NF;
    mbar_wait(&full_f[t], (nf / C::NF) & 1);
    ++nf;
    const double* cur = uring + s_cur * C::US;
    const double* fs = fring + t * C::FS;
    double* rb = rbuf + b * C::RB;
    load_c(zp, uring + s_nxt * C::US);
    double ssq = 0.0;
#pragma unroll
    for (int p = 0; p < NXP; ++p) {
      const int x = tx + p * ACT;
      const double ym0 = cur[trow0 * PX + x + 1];              // y-1 of the first owned row
      const double ypl = cur[(trow0 + RPT + 1) * PX + x + 1];  // y+1 of the last owned row
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = p * RPT + r, row = trow0 + r;
        double xl = __shfl_up_sync(0xffffffffu, c[i], 1);
        double xr = __shfl_down_sync(0xffffffffu, c[i], 1);
        if (lane == 0) xl = cur[(row + 1) * PX + x];
        if (lane == 31) xr = cur[(row + 1) * PX + x + 2];
        if (FULL || row < rows) {
          const double ym = r > 0 ? c[i - 1] : ym0;
          const double yp = r < RPT - 1 ? c[i + 1] : ypl;
          const double fv = fs[row * NX + x];
          double res;
          if (UNIT) {
            double acc = __dmul_rn(st.c, c[i]);
            acc = __dsub_rn(acc, xl);
            acc = __dsub_rn(acc, xr);
            acc = __dsub_rn(acc, ym);
            acc = __dsub_rn(acc, yp);
            acc = __dsub_rn(acc, zm[i]);
            acc = __dsub_rn(acc, zp[i]);
            res = __dsub_rn(fv, acc);
          } else {
            res = residual7(st, fv, c[i], xl, xr, ym, yp, zm[i], zp[i]);
          }
          ssq = fma(res, res, ssq);
          if (RES == 1)
            __stcs(rg + ((long long)k * ny + j0 + row) * NX + x, res);
          else
            rb[row * RS + x + (x >> 5)] = res;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if (lane == 0) wsum[b * C::AC_WARPS + warp] = ssq;
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty_u[s_cur]);
      mbar_arrive(&empty_f[t]);
    }
    if (RES == 1) {
      // residual-only (plane path): the A/C warps reduce the tile partial
      // themselves, in the solver warps' fixed order
      named_sync(kBarRes, ACT);
      if (tid == 0 && partials) {
        double tt = 0.0;
#pragma unroll
        for (int q = 0; q < C::AC_WARPS; ++q) tt += wsum[b * C::AC_WARPS + q];
        partials[tslot0 + (long long)k * tpp + j0 / R] = tt;
      }
    } else {
      named_arrive(kBarR + b, NBAR);
      if (k > k0) phaseC<FULL>(zm);  // u(k-1) is this plane's zm
    }
    vbase_old = (long long)(k + 1) * pxy + (long long)(j0 + 1) * PX + 1;
    kw = k;
    s_cur = s_nxt;
    b ^= 1;
  }

  template <bool FULL>
  __device__ __forceinline__ void run_unit(int ka, int kb) {
    {  // slab ka-1 -> A0
      const int sidx = nu % C::NU;
      mbar_wait(&full_u[sidx], (nu / C::NU) & 1);
      load_c(A0, uring + sidx * C::US);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_u[sidx]);
      ++nu;
    }
    s_cur = nu % C::NU;  // slab ka -> A1, slot kept for the halo rows
    mbar_wait(&full_u[s_cur], (nu / C::NU) & 1);
    ++nu;
    load_c(A1, uring + s_cur * C::US);
    int k = ka;
    for (;;) {
      step<FULL>(A0, A1, A2, k++);
      if (k >= kb) { if (RES != 1) phaseC<FULL>(A1); break; }
      step<FULL>(A1, A2, A0, k++);
      if (k >= kb) { if (RES != 1) phaseC<FULL>(A2); break; }
      step<FULL>(A2, A0, A1, k++);
      if (k >= kb) { if (RES != 1) phaseC<FULL>(A0); break; }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_u[s_cur]);  // the unit's last slab (plane kb)
  }
};

// RES = 1: residual only (plane path): r = f - A u to rglob plus the tile
// partials; no solver, no v.  RES = 2: the sweep plus the fused multi-GPU halo
// (boundary planes also stored into the z-neighbours' ghost planes).
template <int NX, int UNIT, int RES>
__global__ void __launch_bounds__(ZCfg<NX>::THREADS, 1)
    line_jacobi_zmarch_kernel(const PatchDev* __restrict__ patches, const unsigned char* __restrict__ active,
                              StencilDev st, double omega, double* __restrict__ partials,
                              const ZUnit* __restrict__ units, int nunits, const __grid_constant__ ZTab T,
                              double* __restrict__ rglob) {
  using C = ZCfg<NX>;
  constexpr int R = C::R, PX = C::PX, NSEG = C::NSEG, RS = C::RS;
  extern __shared__ __align__(128) double zsm[];
  double* uring = zsm;
  double* fring = uring + C::NU * C::US;
  double* rbuf = fring + C::NF * C::FS;
  double* wsum = rbuf + 2 * C::RB;
  uint64_t* bars = (uint64_t*)(wsum + 2 * C::AC_WARPS);
  uint64_t* full_u = bars;
  uint64_t* empty_u = full_u + C::NU;
  uint64_t* full_f = empty_u + C::NU;
  uint64_t* empty_f = full_f + C::NF;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::NU; ++s) {
      mbar_init(&full_u[s], 1);
      mbar_init(&empty_u[s], C::AC_WARPS);
    }
    for (int s = 0; s < C::NF; ++s) {
      mbar_init(&full_f[s], 1);
      mbar_init(&empty_f[s], C::AC_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ======================= producer warp =====================================
  if (warp == C::AC_WARPS + C::SOLVER_WARPS) {
    if (lane != 0) return;
    uint32_t nu = 0, nf = 0;
    for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
      const ZUnit U = units[w];
      const PatchDev& P = patches[U.patch];
      const int rows = min(R, P.ny - U.j0);
      const long long pxy = (long long)PX * (P.ny + 2);
      const double* u = P.buf[active[U.patch]];
      const uint32_t ubytes = (uint32_t)((rows + 2) * PX * 8);
      const uint32_t fbytes = (uint32_t)(rows * NX * 8);
      for (int kk = U.k0 - 1; kk <= U.k1; ++kk) {
        // u slab of plane kk: rows j0-1 .. j0+rows, contiguous
        const int s = nu % C::NU;
        mbar_wait(&empty_u[s], ((nu / C::NU) & 1) ^ 1);
        mbar_expect_tx(&full_u[s], ubytes);
        tma_load_1d(uring + s * C::US, u + (long long)(kk + 1) * pxy + (long long)U.j0 * PX, ubytes, &full_u[s]);
        ++nu;
        // f slab of plane kk-1 once its u(k+1) partner is queued
        const int kf = kk - 1;
        if (kf >= U.k0 && kf < U.k1) {
          const int t = nf % C::NF;
          mbar_wait(&empty_f[t], ((nf / C::NF) & 1) ^ 1);
          mbar_expect_tx(&full_f[t], fbytes);
#ifdef PSM_ZMARCH_NO_HINT
          tma_load_1d(fring + t * C::FS, P.f + ((long long)kf * P.ny + U.j0) * NX, fbytes, &full_f[t]);
#else
          tma_load_1d_evict_first(fring + t * C::FS, P.f + ((long long)kf * P.ny + U.j0) * NX, fbytes, &full_f[t]);
#endif
          ++nf;
        }
      }
    }
    return;
  }

  // ======================= solver warps ======================================
  if (warp >= C::AC_WARPS) {
    if (RES == 1) return;
    const int sl = tid - C::AC_WARPS * 32;  // 0..NSL-1
    const int r = sl / NSEG, s = sl % NSEG;
    const double lo = T.lo, up = T.up, up_h31 = T.up_h31, lo_g0 = T.lo_g0, d_full = T.d_full;
    const double up_h16 = T.up_h16, lo_g16 = T.lo_g16, d16 = T.d16;
    int b = 0;
    for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
      const ZUnit U = units[w];
      const PatchDev& P = patches[U.patch];
      for (int k = U.k0; k < U.k1; ++k, b ^= 1) {
        named_sync(kBarR + b, (C::AC_WARPS + C::SOLVER_WARPS) * 32);
        if (sl == 0 && partials) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < C::AC_WARPS; ++q) t += wsum[b * C::AC_WARPS + q];
          partials[P.tile0 + (long long)k * P.tpp + U.j0 / R] = t;
        }
        double* seg = rbuf + b * C::RB + r * RS + s * (kSeg + 1);
        // local solve of the 32-cell segment as two independent 16-cell
        // Thomas chains (same prefix factors) joined by an exact 2x2 system
        double ya[16], yb[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          ya[i] = seg[i] * T.invm[i];
          yb[i] = seg[16 + i] * T.invm[i];
        }
#pragma unroll
        for (int i = 1; i < 16; ++i) {
          ya[i] = fma(-T.loinv[i], ya[i - 1], ya[i]);
          yb[i] = fma(-T.loinv[i], yb[i - 1], yb[i]);
        }
#pragma unroll
        for (int i = 14; i >= 0; --i) {
          ya[i] = fma(-T.cp[i], ya[i + 1], ya[i]);
          yb[i] = fma(-T.cp[i], yb[i + 1], yb[i]);
        }
        const double xa15 = (ya[15] - up_h16 * yb[0]) * d16;
        const double xb0 = yb[0] - lo_g16 * xa15;
        const double ca = up * xb0, cb = lo * xa15;
        double yv[kSeg];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          yv[i] = fma(-ca, T.h16[i], ya[i]);
          yv[16 + i] = fma(-cb, T.g16[i], yb[i]);
        }
        const double ylast = yv[kSeg - 1];
        const double yfirst = yv[0];
        const double yl_left = __shfl_up_sync(0xffffffffu, ylast, 1);
        const double yf_right = __shfl_down_sync(0xffffffffu, yfirst, 1);
        double clv = 0.0, crv = 0.0;
        if (s > 0) clv = lo * ((yl_left - up_h31 * yfirst) * d_full);
        if (s < NSEG - 1) crv = up * (yf_right - lo_g0 * ((ylast - up_h31 * yf_right) * d_full));
        // exact solution of the segment: y - lo*x_left*g - up*x_right*h
#pragma unroll
        for (int i = 0; i < kSeg; ++i) seg[i] = fma(-crv, T.h[i], fma(-clv, T.g[i], yv[i]));
        named_arrive(kBarY + b, (C::AC_WARPS + C::SOLVER_WARPS) * 32);
      }
    }
    return;
  }

  // ======================= A/C warps =========================================
  ZAC<NX, UNIT, RES> ac;
  ac.tid = tid;
  ac.lane = lane;
  ac.warp = warp;
  ac.st = st;
  ac.omega = omega;
  ac.uring = uring;
  ac.fring = fring;
  ac.rbuf = rbuf;
  ac.wsum = wsum;
  ac.full_u = full_u;
  ac.empty_u = empty_u;
  ac.full_f = full_f;
  ac.empty_f = empty_f;
  ac.tx = ZAC<NX, UNIT, RES>::NX_GE ? tid : tid % NX;
  ac.trow0 = ZAC<NX, UNIT, RES>::NX_GE ? 0 : (tid / NX) * ZAC<NX, UNIT, RES>::RPT;
  ac.partials = partials;
  for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
    const ZUnit U = units[w];
    const PatchDev& P = patches[U.patch];
    ac.rows = min(R, P.ny - U.j0);
    ac.pxy = (long long)PX * (P.ny + 2);
    ac.v = P.buf[active[U.patch] ^ 1];
    ac.j0 = U.j0;
    ac.k0 = U.k0;
    if (RES == 2) {
      const int vo = active[U.patch] ^ 1;  // peers swap in lockstep: their v has our parity
      ac.nz = P.nz;
      ac.peer_lo = P.peer_lo[vo];
      ac.peer_hi = P.peer_hi[vo];
      ac.peer_lo_off = (long long)P.peer_lo_nz * ac.pxy;      // plane 0 -> their plane nz_lo + 1
      ac.peer_hi_off = -(long long)P.nz * ac.pxy;             // plane nz-1 -> their plane 0
    }
    if (RES == 1) {
      ac.rg = rglob + P.cell0;
      ac.tslot0 = P.tile0;
      ac.tpp = P.tpp;
      ac.ny = P.ny;
    }
    if (ac.rows == R)
      ac.template run_unit<true>(U.k0, U.k1);
    else
      ac.template run_unit<false>(U.k0, U.k1);
  }
}

template <int NX>
static cudaError_t zlaunch(int unit, const PatchDev* patches, const unsigned char* active, const StencilDev& st,
                           double omega, double* partials, const ZUnit* units, int nunits, int grid,
                           const ZTab& T, double* rglob, int peer, cudaStream_t stream) {
  using C = ZCfg<NX>;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
    cudaFuncSetAttribute(line_jacobi_zmarch_kernel<NX, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM_BYTES);
  }
#define PSM_ZL(U_, R_)                                                                                         \
  line_jacobi_zmarch_kernel<NX, U_, R_><<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(patches, active, st, omega, \
                                                                                      partials, units, nunits, T, \
                                                                                      rglob)
  if (rglob) {
    if (unit) PSM_ZL(1, 1); else PSM_ZL(0, 1);
  } else if (peer) {
    if (unit) PSM_ZL(1, 2); else PSM_ZL(0, 2);
  } else {
    if (unit) PSM_ZL(1, 0); else PSM_ZL(0, 0);
  }
#undef PSM_ZL
  return cudaGetLastError();
}

int zmarch_rows(int nx) { return kMaxTileCells / nx; }

cudaError_t launch_line_zmarch(int nx, int unit, const PatchDev* patches, const unsigned char* active,
                               const StencilDev& st, double omega, double* partials, const void* units, int nunits,
                               int grid, const LineFac& L, cudaStream_t stream, double* rglob, int peer) {
  if (nunits <= 0) return cudaSuccess;
  if (grid > nunits) grid = nunits;
  const ZUnit* u = (const ZUnit*)units;
  ZTab T;
  memset(&T, 0, sizeof T);
  if (!rglob)
  for (int i = 0; i < kSeg; ++i) {
    T.invm[i] = L.invm[i];
    T.loinv[i] = L.lo * L.invm[i];
    T.cp[i] = L.cp[i];
    T.g[i] = L.g[i];
    T.h[i] = L.h[i];
  }
  for (int i = 0; i < 16; ++i) {
    T.g16[i] = L.g16[i];
    T.h16[i] = L.h16[i];
  }
  if (!rglob) {
  T.lo = L.lo;
  T.up = L.up;
  T.up_h31 = L.up_h31;
  T.lo_g0 = L.lo_g0;
  T.d_full = L.d_full;
  T.up_h16 = L.up_h16;
  T.lo_g16 = L.lo_g16;
  T.d16 = L.d16;
  }
  switch (nx) {
    case 64: return zlaunch<64>(unit, patches, active, st, omega, partials, u, nunits, grid, T, rglob, peer, stream);
    case 128: return zlaunch<128>(unit, patches, active, st, omega, partials, u, nunits, grid, T, rglob, peer, stream);
    case 256: return zlaunch<256>(unit, patches, active, st, omega, partials, u, nunits, grid, T, rglob, peer, stream);
    case 512: return zlaunch<512>(unit, patches, active, st, omega, partials, u, nunits, grid, T, rglob, peer, stream);
    case 1024: return zlaunch<1024>(unit, patches, active, st, omega, partials, u, nunits, grid, T, rglob, peer, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace psm
