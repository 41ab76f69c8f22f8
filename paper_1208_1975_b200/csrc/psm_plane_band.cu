// Plane blocks, factorised exact solve: block Thomas along y whose Schur
// complements are applied as short convolutions along x.
//
// Replaces, for block_dims (>=nx, >=ny, 1), the exact plane inverse of
// InverseCache.get / invert_dense (blocklinalg.py:116-163, stencil.py:115-138)
// and its dense matvec (blocklinalg.py:90-105) inside smoother._jacobi_step
// (smoother.py:138-153).
//
// The closure-free plane operator is block tridiagonal in y,
//   b_lo x_{j-1} + T x_j + b_up x_{j+1} = r_j,   T = tridiag(a, c, a) along x,
// so block LU gives  S_0 = T,  S_j = T - b_lo b_up S_{j-1}^{-1},
//   forward   z_j = S_j^{-1} (r_j - b_lo z_{j-1}),
//   backward  x_j = z_j - S_j^{-1} (b_up x_{j+1}).
// Every S_j^{-1} is a function F_j(T); with symmetric x faces it is
// diagonalised by the DST-I, so its entries are H_j(p-q) - H_j(p+q+2) with
//   H_j(m) = 1/(n+1) sum'_{i=0..n+1} cos(pi m i/(n+1)) F_j(lambda_i)
// (endpoint terms half weight; they cancel in the difference but make H_j
// the decaying Fourier series of the symbol).
// Applying it to a row is therefore a symmetric convolution with H_j over
// the row's odd extension (t_{-1} = t_n = 0, t_{-2-p} = t_{n+1+..} = -t_p).
// H_j decays geometrically (0.268^m for the default stencil) and S_j
// converges in j (ratio 0.072 per row), so the host keeps |m| <= BW and
// j < nj only where every dropped term is below 1e-17 of H(0): exact to
// rounding, like the line path's segment couplings.  Cost: 2(2BW+1) fp64
// FMAs per update instead of the 4 nx of the DST-GEMM form.
//
// Kernel: one 64-thread CTA per (patch, plane).  "S" phases own cells
// strided (p = t + 64 i: coalesced global traffic, conflict-free shared
// rows), "C" phases own K contiguous outputs (register-blocked convolution
// over a padded shared row).  Row inputs stream through cp.async rings two
// rows ahead; z_j goes to a scratch plane between the sweeps.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "psm_internal.cuh"

namespace psm {

#ifndef PSM_BAND_T
#define PSM_BAND_T 64
#endif
constexpr int kBandT = PSM_BAND_T;  // threads per plane CTA

__device__ __forceinline__ void band_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void band_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void band_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// The converged Schur-complement kernel H_nj (used by every row j >= nj):
// a kernel parameter, so the unrolled convolution reads it as DFMA
// constant-bank operands (no registers, no loads).
struct BandHinf {
  double h[49];
};

template <int K, int BW>
struct BandCfg {
  static constexpr int NMAX = kBandT * K;
  static constexpr int EXT = NMAX + 2 * BW;
  static constexpr int EXTP = EXT + EXT / K + 2;
  static constexpr int ROWP = NMAX + NMAX / K + 2;
  static constexpr int D = 2, P = D - 1;
  static constexpr size_t SMEM = (size_t)(2 * EXTP + ROWP + 2 * D * NMAX) * sizeof(double);
  __device__ static __forceinline__ int pos(int e) { return K > 1 ? e + e / K : e; }
};

// K contiguous outputs p = tK .. tK+K-1 of the convolution of the padded
// extended row `e` with the symmetric kernel h[0..BW] (registers or the
// constant bank, see BandHinf).
template <int K, int BW, typename HV>
__device__ __forceinline__ void band_conv(const double* __restrict__ e, const HV& h, int t, double (&acc)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  const double* w = e + (K > 1 ? t * (K + 1) : t);
#pragma unroll
  for (int d = 0; d < K + 2 * BW; ++d) {
    const double x = w[K > 1 ? d + d / K : d];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int m = d - k - BW;
      if (m >= -BW && m <= BW) acc[k] = fma(h[m < 0 ? -m : m], x, acc[k]);
    }
  }
}

// row j's kernel: the converged one from the constant bank, else table j
template <int K, int BW>
__device__ __forceinline__ void band_conv_row(const double* __restrict__ e, const BandHinf& Hinf,
                                              const double* __restrict__ Ht, int j, int nj, int t,
                                              double (&acc)[K]) {
  if (j >= nj) {
    band_conv<K, BW>(e, Hinf.h, t, acc);
  } else {
    double h[BW + 1];
#pragma unroll
    for (int m = 0; m <= BW; ++m) h[m] = __ldg(Ht + (long long)j * (BW + 1) + m);
    band_conv<K, BW>(e, h, t, acc);
  }
}

template <int K, int BW>
__global__ void __launch_bounds__(kBandT, 384 / kBandT) plane_band_jacobi_kernel(const PatchDev* __restrict__ patches,
                                                                  const unsigned char* __restrict__ active,
                                                                  double omega, const double* __restrict__ rbuf,
                                                                  double* __restrict__ zbuf,
                                                                  const int2* __restrict__ units, int nunits,
                                                                  const __grid_constant__ BandHinf Hinf) {
  using C = BandCfg<K, BW>;
  constexpr int NMAX = C::NMAX, EXTP = C::EXTP, D = C::D, P = C::P;
  extern __shared__ __align__(16) double bsm[];
  double* ext = bsm;                  // [2][EXTP] odd-extended rows (padded positions)
  double* crow = ext + 2 * EXTP;      // [ROWP] convolution outputs (padded positions)
  double* ringA = crow + C::ROWP;     // [D][NMAX] r rows (forward) / z rows (backward)
  double* ringB = ringA + D * NMAX;   // [D][NMAX] u rows (backward)
  const int t = threadIdx.x;

  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int2 U = units[u];
    const PatchDev& Pd = patches[U.x];
    const PlaneFac* F = Pd.pf;
    const int n = Pd.nx, ny = Pd.ny, k = U.y, nj = F->nj;
    const double* __restrict__ Ht = F->H;
    const double blo = F->fy_lo, bup = F->fy_up;
    const long long px = n + 2, pxy = px * (ny + 2);
    const int act = active[U.x];
    const double* ub = Pd.buf[act] + (long long)(k + 1) * pxy + px + 1;  // u(0, 0, k)
    double* vb = Pd.buf[act ^ 1] + (long long)(k + 1) * pxy + px + 1;
    const double* rk = rbuf + Pd.cell0 + (long long)k * ny * n;
    double* zk = zbuf + Pd.cell0 + (long long)k * ny * n;
    if (t < 2) {  // the odd extension's zeros t_{-1} = t_n = 0
      ext[t * EXTP + C::pos(BW - 1)] = 0.0;
      ext[t * EXTP + C::pos(n + BW)] = 0.0;
    }
    // ---------------- forward: z_j = S_j^{-1}(r_j - b_lo z_{j-1}) ----------
    auto issueF = [&](int j) {
      if (j < ny) {
        double* dst = ringA + (j % D) * NMAX;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int p = t + kBandT * i;
          if (p < n) band_cp8(dst + p, rk + (long long)j * n + p);
        }
      }
      band_commit();
    };
#pragma unroll
    for (int j = 0; j < P; ++j) issueF(j);
    for (int j = 0; j < ny; ++j) {
      issueF(j + P);
      band_wait<P>();
      const double* ra = ringA + (j % D) * NMAX;
      double* e = ext + (j & 1) * EXTP;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int p = t + kBandT * i;
        if (p < n) {
          double zp = 0.0;
          if (j > 0) {
            zp = crow[C::pos(p)];
            __stcg(zk + (long long)(j - 1) * n + p, zp);
          }
          const double tv = fma(-blo, zp, ra[p]);
          e[C::pos(p + BW)] = tv;
          if (p <= BW - 2) e[C::pos(BW - 2 - p)] = -tv;
          if (p >= n - BW + 1) e[C::pos(2 * n - p + BW)] = -tv;
        }
      }
      __syncthreads();
      double acc[K];
      band_conv_row<K, BW>(e, Hinf, Ht, j, nj, t, acc);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const int p = t * K + q;
        if (p < n) crow[C::pos(p)] = acc[q];
      }
      __syncthreads();
    }
    band_wait<0>();
    __threadfence_block();  // z rows stored above are re-read below by the same threads
    // ---------------- backward: x_j = z_j - S_j^{-1}(b_up x_{j+1}) --------
    auto issueB = [&](int b) {  // backward step b handles row j = ny-1-b
      const int j = ny - 1 - b;
      if (j >= 0) {
        double* dz = ringA + (b % D) * NMAX;
        double* du = ringB + (b % D) * NMAX;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int p = t + kBandT * i;
          if (p < n) {
            if (j < ny - 1) band_cp8(dz + p, zk + (long long)j * n + p);
            band_cp8(du + p, ub + (long long)j * px + p);
          }
        }
      }
      band_commit();
    };
#pragma unroll
    for (int b = 0; b < P; ++b) issueB(b);
    for (int b = 0; b < ny; ++b) {
      const int j = ny - 1 - b;
      issueB(b + P);
      band_wait<P>();
      const double* za = ringA + (b % D) * NMAX;
      const double* ua = ringB + (b % D) * NMAX;
      double* e = ext + (b & 1) * EXTP;
      double* vrow = vb + (long long)j * px;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int p = t + kBandT * i;
        if (p < n) {
          // j == ny-1: crow still holds z_{ny-1}; else it holds S_j^{-1} b_up x_{j+1}
          const double xv = (b == 0) ? crow[C::pos(p)] : za[p] - crow[C::pos(p)];
          const double nv = relax(ua[p], omega, xv);
          vrow[p] = nv;
          if (p == 0) vrow[-1] = -nv;
          if (p == n - 1) vrow[n] = -nv;
          if (j > 0) {
            const double w = bup * xv;
            e[C::pos(p + BW)] = w;
            if (p <= BW - 2) e[C::pos(BW - 2 - p)] = -w;
            if (p >= n - BW + 1) e[C::pos(2 * n - p + BW)] = -w;
          }
        }
      }
      __syncthreads();
      if (j > 0) {
        double acc[K];
        band_conv_row<K, BW>(e, Hinf, Ht, j - 1, nj, t, acc);
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const int p = t * K + q;
          if (p < n) crow[C::pos(p)] = acc[q];
        }
      }
      __syncthreads();
    }
    band_wait<0>();
  }
}

template <int K, int BW>
static cudaError_t band_launch_t(const PatchDev* patches, const unsigned char* active, double omega,
                                 const double* rbuf, double* zbuf, const int2* units, int nunits, int sms,
                                 const BandHinf& Hinf, cudaStream_t s) {
  using C = BandCfg<K, BW>;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(plane_band_jacobi_kernel<K, BW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  }
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, plane_band_jacobi_kernel<K, BW>, kBandT, C::SMEM);
  const int grid = std::max(1, std::min(nunits, std::max(1, occ) * sms));
  plane_band_jacobi_kernel<K, BW><<<grid, kBandT, C::SMEM, s>>>(patches, active, omega, rbuf, zbuf, units, nunits,
                                                                Hinf);
  return cudaGetLastError();
}

int band_k_for(int nx) {  // outputs per thread: kBandT * K >= nx
  for (int k = 1; k <= 16; k *= 2)
    if (nx <= kBandT * k) return k;
  return 0;
}

cudaError_t launch_plane_band_jacobi(int K, int BW, const PatchDev* patches, const unsigned char* active,
                                     double omega, const double* rbuf, double* zbuf, const int2* units,
                                     int nunits, const double* hinf_host, cudaStream_t s) {
  if (nunits <= 0) return cudaSuccess;
  BandHinf Hinf;
  memset(&Hinf, 0, sizeof Hinf);
  for (int m = 0; m <= BW && m < 49; ++m) Hinf.h[m] = hinf_host[m];
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#define PSM_BAND(KK, BB) \
  if (K == KK && BW == BB) return band_launch_t<KK, BB>(patches, active, omega, rbuf, zbuf, units, nunits, sms, Hinf, s);
#define PSM_BAND_K(KK) PSM_BAND(KK, 16) PSM_BAND(KK, 32) PSM_BAND(KK, 48)
  PSM_BAND_K(1)
  PSM_BAND_K(2)
  PSM_BAND_K(4)
  PSM_BAND_K(8)
  PSM_BAND_K(16)
#undef PSM_BAND_K
#undef PSM_BAND
  return cudaErrorInvalidValue;
}

// Host: band tables of the plane operator with x coefficient a (symmetric),
// center c and y couplings blo, bup, for an nx x ny plane.  On success
// *bw in {16, 32, 48} (<= nx), *nj = number of distinct leading S_j, and
// H holds (nj+1) x (bw+1) doubles; *bw = 0 when the banded form does not
// meet the 1e-17 truncation bound within 48 taps.
void plane_band_tables(long double c, long double a, long double blo, long double bup, int nx, int ny, int* bw_out,
                       int* nj_out, std::vector<double>& H) {
  *bw_out = 0;
  *nj_out = 0;
  H.clear();
  const int n = nx;
  if (band_k_for(n) == 0) return;
  const long double pi = 3.141592653589793238462643383279502884L;
  const int per = 2 * (n + 1);
  // Symbol sampled on the full circle i = 0..n+1 (endpoints half weight):
  // the i = 0 and i = n+1 terms only add c0 + c1 (-1)^m to H, which cancels
  // in H(p-q) - H(p+q+2), and they make H the geometrically decaying
  // Fourier series of the smooth symbol instead of a sequence with a
  // constant/alternating floor.
  std::vector<long double> cs(per), lam(n + 2), s(n + 2), Fj(n + 2);
  for (int q = 0; q < per; ++q) cs[q] = cosl(pi * q / (n + 1));
  for (int i = 0; i <= n + 1; ++i) lam[i] = c + 2.0L * a * cs[i];
  const int mmax = n + 1;
  auto tableH = [&](std::vector<long double>& out) {
    out.assign(mmax + 1, 0.0L);
    for (int m = 0; m <= mmax; ++m) {
      long double acc = 0, comp = 0;  // Kahan: keeps the summation noise near 1e-19 |F|
      for (int i = 0; i <= n + 1; ++i) {
        const long double wgt = (i == 0 || i == n + 1) ? 0.5L : 1.0L;
        const long double y = wgt * cs[(long long)m * i % per] * Fj[i] - comp;
        const long double tt = acc + y;
        comp = (tt - acc) - y;
        acc = tt;
      }
      out[m] = acc / (n + 1);
    }
  };
  std::vector<std::vector<long double>> tabs;
  std::vector<long double> cur;
  for (int i = 0; i <= n + 1; ++i) s[i] = lam[i];
  const int jmax = std::min(ny, 256);
  int nj = -1;
  bool converged = false;
  for (int j = 0; j < jmax; ++j) {
    if (j > 0)
      for (int i = 0; i <= n + 1; ++i) s[i] = lam[i] - blo * bup / s[i];
    for (int i = 0; i <= n + 1; ++i) {
      if (fabsl(s[i]) < 1e-14L * fabsl(c)) return;  // singular: leave to the DST path's diagnostics
      Fj[i] = 1.0L / s[i];
    }
    tableH(cur);
    if (!tabs.empty()) {
      long double dmax = 0;
      for (int m = 0; m <= mmax; ++m) dmax = fmaxl(dmax, fabsl(cur[m] - tabs.back()[m]));
      if (dmax <= 1e-18L * fabsl(cur[0])) {
        nj = j - 1;  // S_{j-1} already equals the limit to rounding
        converged = true;
        break;
      }
    }
    tabs.push_back(cur);
  }
  if (!converged) {
    if (ny > (int)tabs.size()) return;  // S_j still moving after 256 rows: DST path
    nj = (int)tabs.size() - 1;          // one table per row
  }
  // bandwidth: every dropped |H_j(m)| below 1e-17 |H_j(0)|; with the
  // geometric decay the dropped tail sums to < 1e-17 |H_j(0)| (the table
  // sums themselves carry ~1e-19 absolute noise, so a summed-tail test on the
  // computed values would only measure that noise)
  int need = 0;
  for (auto& Tb : tabs) {
    int b = mmax;
    while (b > 0 && fabsl(Tb[b]) <= 1e-17L * fabsl(Tb[0])) --b;
    need = std::max(need, b);
  }
  int bw = need <= 16 ? 16 : need <= 32 ? 32 : need <= 48 ? 48 : 0;
  if (bw == 0 || bw > n) return;
  *bw_out = bw;
  *nj_out = nj;
  H.resize((size_t)(nj + 1) * (bw + 1));
  for (int j = 0; j <= nj; ++j)
    for (int m = 0; m <= bw; ++m) H[(size_t)j * (bw + 1) + m] = (double)tabs[j][m];
}

}  // namespace psm

