// Line-block Jacobi sweep for any even nx in [42, 1024]: the z-marching TMA
// pipeline of psm_line_tma.cu with the line length a launch parameter.
//
// Replaces smoother._jacobi_step + block_residual + block_update/matvec
// (smoother.py:138-153, stencil.py:93-112, blocklinalg.py:90-105) for line
// blocks on patches whose nx has no specialised kernel -- the AMR case of
// mixed patch sizes (reference bench.py:44, the paper's Table 2 set of
// 64^3..96^3 patches).
//
// Same work units, roles and ring protocol as line_jacobi_zmarch_kernel:
//   warp 19      producer: one 1-D bulk copy per plane of the unit's u slab
//                (rows j0-1 .. j0+R, contiguous; needs nx even for 16-byte
//                alignment) into a 4-slot ring, f's R rows into a 2-slot ring.
//   warps 0-15   A/C: thread t owns the cells e = q*512 + t (q < 4) of the
//                R x nx tile; their (row, x) are recomputed only when a unit's
//                patch has another nx (one launch covers patches of any mix of
//                line lengths; ring slots are sized for the largest).
//                Per plane: residual in the reference operation order from
//                the slab (x/y neighbours) and a register queue of the owned
//                cells' u(k-1), u(k), u(k+1) -> padded r buffer; then C(k-1):
//                v = u + omega * x, x ghosts of v fused.
//   warps 16-18  solver: one lane per 32-cell segment (R * ceil(nx/32) <= 96
//                lanes, whole rows per warp), Thomas with constant prefix
//                factors, the last segment of a row shorter (tail), segment
//                ends exchanged by shuffle, exact 2x2 interface solves (valid when the
//                dropped couplings are below 1e-18, LineFac::partitioned).
#include <stdint.h>
#include <string.h>

#include "psm_internal.cuh"

namespace psm {
namespace {

__device__ __forceinline__ uint32_t g_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void g_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(g_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void g_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(g_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void g_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(g_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void g_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "GMBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra GMBW_%=;\n"
      "}\n" ::"r"(g_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void g_tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          g_smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(g_smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void g_named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void g_named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

constexpr int kGAcWarps = 16, kGSolWarps = 3, kGThreads = (kGAcWarps + kGSolWarps + 1) * 32;
constexpr int kGAct = kGAcWarps * 32;          // A/C threads
constexpr int kGE = kMaxTileCells / kGAct;     // cells per A/C thread (4)
constexpr int kGNbar = (kGAcWarps + kGSolWarps) * 32;
constexpr int kGNU = 4, kGNF = 2;
constexpr int kGBarR = 1, kGBarY = 3;

// launch geometry of one nx (host and device agree through this struct)
struct GGeom {
  int nx, px, R, nseg, tail, rs;
  int us, fs, rb;  // doubles per u slot, f slot, r buffer
};

__host__ __device__ inline GGeom g_geom(int nx) {
  GGeom g;
  g.nx = nx;
  g.px = nx + 2;
  g.R = kMaxTileCells / nx;
  g.nseg = (nx + kSeg - 1) / kSeg;
  g.tail = nx - kSeg * (g.nseg - 1);
  g.rs = nx + g.nseg;
  g.us = (g.R + 2) * g.px;
  g.fs = g.R * nx;
  g.rb = g.R * g.rs;
  return g;
}

// factor tables in the kernel-parameter constant bank
struct GTab {
  double invm[kSeg], loinv[kSeg], cp[kSeg], g[kSeg], h[kSeg];  // full-segment factors: any nx
  double lo, up, up_h31, lo_g0, d_full;
};

struct GUnit {
  int patch, j0, k0, k1;
};

// A/C role: owned cells (row, x) fixed per launch, register queue of their
// u(k-1), u(k), u(k+1) rotated by unrolling the plane loop by three.
template <int UNIT>
struct GAC {
  int tid, lane, warp, nx = 0, R, PX, RS, rows, j0, k0;
  int su, sf, sb;  // slot strides (doubles) of the u ring, f ring, r buffers
  StencilDev st;
  double omega;
  double *uring, *fring, *rbuf, *wsum, *v;
  uint64_t *full_u, *empty_u, *full_f, *empty_f;
  GGeom G;
  long long pxy, vbase_old = 0;
  uint32_t nu = 0, nf = 0;
  int b = 0, s_cur = 0;
  int crow[kGE];                 // row of owned cell q (1<<20: none)
  int oc[kGE], orb[kGE], of[kGE];  // its offsets in a u slab (centre), the r buffer, an f slab
  int ov[kGE];                   // and in v relative to the tile's first cell
  int xedge;                     // bit q: x == 0, bit q + 8: x == nx - 1
  double A0[kGE], A1[kGE], A2[kGE];

  __device__ __forceinline__ void init(int tid_, int lane_, int warp_, int su_, int sf_, int sb_,
                                       const StencilDev& st_, double om, double* ur, double* fr, double* rb,
                                       double* ws, uint64_t* fu, uint64_t* eu, uint64_t* ff, uint64_t* ef) {
    tid = tid_;
    lane = lane_;
    warp = warp_;
    su = su_;
    sf = sf_;
    sb = sb_;
    st = st_;
    omega = om;
    uring = ur;
    fring = fr;
    rbuf = rb;
    wsum = ws;
    full_u = fu;
    empty_u = eu;
    full_f = ff;
    empty_f = ef;
  }

  // owned cells of an R x nx tile (recomputed when the line length changes)
  __device__ __forceinline__ void set_nx(int nx_) {
    if (nx_ == nx) return;
    nx = nx_;
    G = g_geom(nx);
    R = G.R;
    PX = G.px;
    RS = G.rs;
    xedge = 0;
#pragma unroll
    for (int q = 0; q < kGE; ++q) {
      const int e = q * kGAct + tid;
      const int row = e / nx, x = e - (e / nx) * nx;
      crow[q] = row < R ? row : 1 << 20;  // beyond the tile: never valid
      oc[q] = (row + 1) * PX + x + 1;
      orb[q] = row * RS + x + (x >> 5);
      of[q] = row * nx + x;
      ov[q] = row * PX + x;
      xedge |= (x == 0 ? 1 << q : 0) | (x == nx - 1 ? 256 << q : 0);
    }
  }

  __device__ __forceinline__ void load_c(double (&dst)[kGE], const double* sl) const {
#pragma unroll
    for (int q = 0; q < kGE; ++q) dst[q] = crow[q] < rows ? sl[oc[q]] : 0.0;
  }

  __device__ __forceinline__ void phaseC(const double (&cold)[kGE]) {
    const int bo = b ^ 1;
    g_named_sync(kGBarY + bo, kGNbar);
    const double* xb = rbuf + bo * sb;
#pragma unroll
    for (int q = 0; q < kGE; ++q) {
      if (crow[q] < rows) {
        const double nv = relax(cold[q], omega, xb[orb[q]]);
        double* vp = v + vbase_old + ov[q];
        *vp = nv;
        if (xedge & (1 << q)) vp[-1] = -nv;
        if (xedge & (256 << q)) vp[1] = -nv;
      }
    }
  }

  __device__ __forceinline__ void step(const double (&zm)[kGE], const double (&c)[kGE], double (&zp)[kGE], int k) {
    const int s_nxt = nu % kGNU;
    g_mbar_wait(&full_u[s_nxt], (nu / kGNU) & 1);
    ++nu;
    const int t = nf % kGNF;
    g_mbar_wait(&full_f[t], (nf / kGNF) & 1);
    ++nf;
    const double* cur = uring + s_cur * su;
    const double* fs = fring + t * sf;
    double* rb = rbuf + b * sb;
    load_c(zp, uring + s_nxt * su);
    double ssq = 0.0;
#pragma unroll
    for (int q = 0; q < kGE; ++q) {
      if (crow[q] < rows) {
        const double* cu = cur + oc[q];
        const double xl = cu[-1], xr = cu[1], ym = cu[-PX], yp = cu[PX];
        const double fv = fs[of[q]];
        double res;
        if (UNIT) {
          double acc = __dmul_rn(st.c, c[q]);
          acc = __dsub_rn(acc, xl);
          acc = __dsub_rn(acc, xr);
          acc = __dsub_rn(acc, ym);
          acc = __dsub_rn(acc, yp);
          acc = __dsub_rn(acc, zm[q]);
          acc = __dsub_rn(acc, zp[q]);
          res = __dsub_rn(fv, acc);
        } else {
          res = residual7(st, fv, c[q], xl, xr, ym, yp, zm[q], zp[q]);
        }
        ssq = fma(res, res, ssq);
        rb[orb[q]] = res;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if (lane == 0) wsum[b * kGAcWarps + warp] = ssq;
    __syncwarp();
    if (lane == 0) {
      g_mbar_arrive(&empty_u[s_cur]);
      g_mbar_arrive(&empty_f[t]);
    }
    g_named_arrive(kGBarR + b, kGNbar);
    if (k > k0) phaseC(zm);  // u(k-1) is this plane's zm
    vbase_old = (long long)(k + 1) * pxy + (long long)(j0 + 1) * PX + 1;
    s_cur = s_nxt;
    b ^= 1;
  }

  __device__ __forceinline__ void run_unit(int ka, int kb) {
    {  // slab ka-1 -> A0
      const int sidx = nu % kGNU;
      g_mbar_wait(&full_u[sidx], (nu / kGNU) & 1);
      load_c(A0, uring + sidx * su);
      __syncwarp();
      if (lane == 0) g_mbar_arrive(&empty_u[sidx]);
      ++nu;
    }
    s_cur = nu % kGNU;
    g_mbar_wait(&full_u[s_cur], (nu / kGNU) & 1);
    ++nu;
    load_c(A1, uring + s_cur * su);
    int k = ka;
    for (;;) {
      step(A0, A1, A2, k++);
      if (k >= kb) { phaseC(A1); break; }
      step(A1, A2, A0, k++);
      if (k >= kb) { phaseC(A2); break; }
      step(A2, A0, A1, k++);
      if (k >= kb) { phaseC(A0); break; }
    }
    __syncwarp();
    if (lane == 0) g_mbar_arrive(&empty_u[s_cur]);
  }
};

template <int UNIT>
__global__ void __launch_bounds__(kGThreads, 1)
    line_jacobi_zgen_kernel(const PatchDev* __restrict__ patches, const unsigned char* __restrict__ active,
                            StencilDev st, double omega, double* __restrict__ partials,
                            const GUnit* __restrict__ units, int nunits, const __grid_constant__ GTab T, int su,
                            int sf, int sb) {
  extern __shared__ __align__(128) double gsm[];
  double* uring = gsm;
  double* fring = uring + kGNU * su;
  double* rbuf = fring + kGNF * sf;
  double* wsum = rbuf + 2 * sb;
  uint64_t* bars = (uint64_t*)(wsum + 2 * kGAcWarps);
  uint64_t* full_u = bars;
  uint64_t* empty_u = full_u + kGNU;
  uint64_t* full_f = empty_u + kGNU;
  uint64_t* empty_f = full_f + kGNF;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kGNU; ++s) {
      g_mbar_init(&full_u[s], 1);
      g_mbar_init(&empty_u[s], kGAcWarps);
    }
    for (int s = 0; s < kGNF; ++s) {
      g_mbar_init(&full_f[s], 1);
      g_mbar_init(&empty_f[s], kGAcWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // ======================= producer warp =====================================
  if (warp == kGAcWarps + kGSolWarps) {
    if (lane != 0) return;
    uint32_t nu = 0, nf = 0;
    for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
      const GUnit U = units[w];
      const PatchDev& P = patches[U.patch];
      const int nx = P.nx, PX = nx + 2;
      const int rows = min(kMaxTileCells / nx, P.ny - U.j0);
      const long long pxy = (long long)PX * (P.ny + 2);
      const double* u = P.buf[active[U.patch]];
      const uint32_t ubytes = (uint32_t)((rows + 2) * PX * 8);
      const uint32_t fbytes = (uint32_t)(rows * nx * 8);
      for (int kk = U.k0 - 1; kk <= U.k1; ++kk) {
        const int s = nu % kGNU;
        g_mbar_wait(&empty_u[s], ((nu / kGNU) & 1) ^ 1);
        g_mbar_expect_tx(&full_u[s], ubytes);
        g_tma_load_1d(uring + s * su, u + (long long)(kk + 1) * pxy + (long long)U.j0 * PX, ubytes, &full_u[s]);
        ++nu;
        const int kf = kk - 1;
        if (kf >= U.k0 && kf < U.k1) {
          const int t = nf % kGNF;
          g_mbar_wait(&empty_f[t], ((nf / kGNF) & 1) ^ 1);
          g_mbar_expect_tx(&full_f[t], fbytes);
          g_tma_load_1d(fring + t * sf, P.f + ((long long)kf * P.ny + U.j0) * nx, fbytes, &full_f[t]);
          ++nf;
        }
      }
    }
    return;
  }

  // ======================= solver warps ======================================
  if (warp >= kGAcWarps) {
    const int sl = tid - kGAcWarps * 32;
    const double lo = T.lo, up = T.up, up_h31 = T.up_h31;
    int b = 0;
    for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
      const GUnit U = units[w];
      const PatchDev& P = patches[U.patch];
      const GGeom G = g_geom(P.nx);
      const int R = G.R, NSEG = G.nseg;
      // whole rows per solver warp, so a segment's neighbours are shuffles away
      const int rpw = 32 / NSEG, wl = sl & 31;
      const int r = (sl >> 5) * rpw + wl / NSEG, s = wl - (wl / NSEG) * NSEG;
      const bool live = wl < rpw * NSEG && r < R;
      const bool last = s == NSEG - 1;
      const int len = last ? G.tail : kSeg;
      // tail-segment factors depend on nx: from the patch's factor record
      const LineFac* __restrict__ L = P.lf;
      const double d_tail = L->d_tail, lo_gT0 = L->lo_gT0;
      for (int k = U.k0; k < U.k1; ++k, b ^= 1) {
        g_named_sync(kGBarR + b, kGNbar);
        if (sl == 0 && partials) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < kGAcWarps; ++q) t += wsum[b * kGAcWarps + q];
          partials[P.tile0 + (long long)k * P.tpp + U.j0 / R] = t;
        }
        double* seg = rbuf + b * sb + r * G.rs + s * (kSeg + 1);
        double yfirst = 0.0, ylast = 0.0;
        if (live) {
          double y[kSeg];
#pragma unroll
          for (int i = 0; i < kSeg; ++i) y[i] = i < len ? seg[i] * T.invm[i] : 0.0;
#pragma unroll
          for (int i = 1; i < kSeg; ++i)  // past a tail's end the input is 0: harmless, no select
            y[i] = fma(-T.loinv[i], y[i - 1], y[i]);
#pragma unroll
          for (int i = kSeg - 2; i >= 0; --i)
            if (i < len - 1) y[i] = fma(-T.cp[i], y[i + 1], y[i]);
#pragma unroll
          for (int i = 0; i < kSeg; ++i) {
            if (i < len) seg[i] = y[i];
            if (i == len - 1) ylast = y[i];
          }
          yfirst = y[0];
        }
        const double yl_left = __shfl_up_sync(0xffffffffu, ylast, 1);
        const double yf_right = __shfl_down_sync(0xffffffffu, yfirst, 1);
        if (live) {
          double clv = 0.0, crv = 0.0;
          if (s > 0) clv = lo * ((yl_left - up_h31 * yfirst) * (last ? d_tail : T.d_full));
          if (!last) {
            const bool rlast = s + 1 == NSEG - 1;
            const double yfr = yf_right;
            crv = up * (yfr - (rlast ? lo_gT0 : T.lo_g0) * ((ylast - up_h31 * yfr) * (rlast ? d_tail : T.d_full)));
          }
          if (last) {
#pragma unroll
            for (int i = 0; i < kSeg; ++i)
              if (i < len) seg[i] = fma(-crv, T.h[i], fma(-clv, __ldg(&L->gT[i]), seg[i]));
          } else {
#pragma unroll
            for (int i = 0; i < kSeg; ++i) seg[i] = fma(-crv, T.h[i], fma(-clv, T.g[i], seg[i]));
          }
        }
        g_named_arrive(kGBarY + b, kGNbar);
      }
    }
    return;
  }

  // ======================= A/C warps =========================================
  GAC<UNIT> ac;
  ac.init(tid, lane, warp, su, sf, sb, st, omega, uring, fring, rbuf, wsum, full_u, empty_u, full_f, empty_f);
  for (int w = blockIdx.x; w < nunits; w += gridDim.x) {
    const GUnit U = units[w];
    const PatchDev& P = patches[U.patch];
    ac.set_nx(P.nx);
    ac.rows = min(ac.R, P.ny - U.j0);
    ac.pxy = (long long)ac.PX * (P.ny + 2);
    ac.v = P.buf[active[U.patch] ^ 1];
    ac.j0 = U.j0;
    ac.k0 = U.k0;
    ac.run_unit(U.k0, U.k1);
  }
}

}  // namespace

// 20 warps (warp allocation comes in fours: 96 registers per thread), so
// three solver warps of whole rows: ceil(R / floor(32 / nseg)) <= 3 holds for
// every even nx in [42, 1024]
bool line_zgen_supported(int nx) {
  if (nx < 42 || nx > 1024 || (nx & 1)) return false;
  const GGeom g = g_geom(nx);
  const int rpw = 32 / g.nseg;
  return (g.R + rpw - 1) / rpw <= kGSolWarps;
}

cudaError_t launch_line_zgen(const int* nxs, int nnx, int unit, const PatchDev* patches, const unsigned char* active,
                             const StencilDev& st, double omega, double* partials, const void* units, int nunits,
                             int grid, const LineFac& L, cudaStream_t stream) {
  if (nunits <= 0) return cudaSuccess;
  if (grid > nunits) grid = nunits;
  int su = 0, sf = 0, sb = 0;
  for (int i = 0; i < nnx; ++i) {
    if (!line_zgen_supported(nxs[i])) return cudaErrorInvalidValue;
    const GGeom g = g_geom(nxs[i]);
    su = su > g.us ? su : g.us;
    sf = sf > g.fs ? sf : g.fs;
    sb = sb > g.rb ? sb : g.rb;
  }
  GTab T;
  memset(&T, 0, sizeof T);
  for (int i = 0; i < kSeg; ++i) {
    T.invm[i] = L.invm[i];
    T.loinv[i] = L.lo * L.invm[i];
    T.cp[i] = L.cp[i];
    T.g[i] = L.g[i];
    T.h[i] = L.h[i];
  }
  T.lo = L.lo;
  T.up = L.up;
  T.up_h31 = L.up_h31;
  T.lo_g0 = L.lo_g0;
  T.d_full = L.d_full;
  const size_t dbl = (size_t)kGNU * su + (size_t)kGNF * sf + 2 * (size_t)sb + 2 * kGAcWarps;
  const size_t smem = dbl * 8 + (2 * kGNU + 2 * kGNF) * 8 + 16;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // the opt-in is a per-device attribute and smem depends on the plan: set
  // it on every launch (a host-side call, no stream work, legal in capture)
  if (unit) {
    cudaFuncSetAttribute(line_jacobi_zgen_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    line_jacobi_zgen_kernel<1><<<grid, kGThreads, smem, stream>>>(patches, active, st, omega, partials,
                                                                  (const GUnit*)units, nunits, T, su, sf, sb);
  } else {
    cudaFuncSetAttribute(line_jacobi_zgen_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    line_jacobi_zgen_kernel<0><<<grid, kGThreads, smem, stream>>>(patches, active, st, omega, partials,
                                                                  (const GUnit*)units, nunits, T, su, sf, sb);
  }
  return cudaGetLastError();
}

}  // namespace psm
