// Line-block Gauss-Seidel, plane-pipelined CTAs with warp-level PCR solves.
//
// Replaces smoother._gs_step + block_residual + block_update/matvec for line
// blocks (smoother.py:156-169, stencil.py:93-112, blocklinalg.py:90-105) when
// nx is even and splits into nl <= 32 lane chunks of NC <= 8 cells (32, 64,
// 128, 256 with all 32 lanes; 72 = 24 x 3, 80 = 20 x 4, ...).  Ghosts are
// lagged until the step-end refresh, as in the reference.
//
// Order.  The serial strategy visits x-lines (j,k) of a patch
// lexicographically, j fastest (runtime.py:164-168): line (j,k) reads the NEW
// lines (j-1,k) and (j,k-1) and the OLD lines (j+1,k), (j,k+1).  Here a work
// unit is W consecutive planes k0..k0+W-1 of one patch; warp w of the CTA owns
// plane k0+w and walks its rows j = 0..ny-1 in order.  Row j of plane k waits
// for row j of plane k-1 (previous warp: shared-memory progress counter and a
// ring of new rows; previous CTA: a global acquire/release flag), so every
// line computes exactly the lexicographic arithmetic: a wavefront schedule over
// d = j + k.  CHAOTIC drops the acquire/release ordering on the cross-CTA flag
// (relaxed accesses, no fences): in-place block updates without a global
// memory ordering, the contract of smooth_chaotic_gs_step under parallel
// strategies.
//
// Line solve.  Lane L < nl owns the NC = nx/nl contiguous cells L*NC .. L*NC+NC-1
// (lanes nl..31 own none and carry identity rows of the interface system).
// Cells 0..NC-2 of a chunk are eliminated locally (constant Thomas factors and
// spikes g, h: one set serves every chunk), which leaves one tridiagonal
// interface system in the chunks' last cells a_L.  That 32-unknown system is
// solved exactly by five parallel-cyclic-reduction steps over warp shuffles
// with per-lane coefficients built once on the host in long double.  The
// chunk cells then follow as x = y - a_{L-1} g - a_L h.
//
// Data movement.  Per row a lane issues 8-byte cp.async copies (coalesced on
// the global side) of the old rows u(j+1,k), u(j,k+1), f(j,k) and the row's two
// x-ghosts into a 3-deep per-warp ring, two rows ahead of use; the shared
// layout pos(x) = (x % NC)*(32 + 16/NC) + x/NC makes both the coalesced copy
// and the lane-chunk reads bank-conflict free.  New rows go through a 2-deep
// per-warp ring: it feeds the next warp's u(j,k-1) and the coalesced global
// store of the row.
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <map>
#include <vector>

#include "psm_internal.cuh"

namespace psm {

constexpr int kGsW = 7;       // planes (compute warps) per CTA unit; + 1 publisher warp
constexpr int kGsThreads = (kGsW + 1) * 32;
constexpr int kGsTab = 18;    // per-lane table entries: q0,q1,q2 + 5 PCR steps x (p0,p1,p2)
#ifdef PSM_GS_PUB
constexpr int kGsPub = PSM_GS_PUB;  // tuning builds
#else
constexpr int kGsPub = 2;     // wavefront mode: rows per release of the cross-CTA flag (1: 0.78, 2: 0.77, 4: 0.82 ms at C2)
#endif

// uniform chunk-interior tables (passed by value: constant-bank operands)
struct GsUniform {
  double invm[8], loinv[8], cp[8], g[8], h[8];
  double tinv[8][8];  // explicit inverse of the chunk interior block (row i: y_i = sum_p tinv[i][p] r_p)
  int npcr;  // PCR steps until the remaining interface couplings are < 1e-20 (<= 5: exact)
};

template <int NC, int MS = 0>
struct GCfg {
  static constexpr int IS = 32 + 16 / NC;      // stride between the NC "i-rows" of a slot
  static constexpr int SLOT = (NC * IS + 3) / 2 * 2;  // doubles per ring slot (+ the two x-ghosts), even: 16-B bulk copies
#ifdef PSM_GS_D
  static constexpr int D = PSM_GS_D;           // tuning builds
#else
  static constexpr int D = 3;                  // prefetch ring depth
#endif
  static constexpr int P = D - 1;              // rows of prefetch ahead
  static constexpr int DH = 2;                 // new-row ring depth (warp -> next warp)
  static constexpr int DHL = 4;                // new-row ring depth (last warp -> publisher)
#ifdef PSM_GS_DM
  static constexpr int DM = PSM_GS_DM;         // tuning builds
#else
  static constexpr int DM = 3;                 // warp 0: rows of plane k0-1 in flight (TMA)
#endif
  static constexpr int MROW = 32 * NC + 2;     // padded row, contiguous
  static constexpr int NBAR = 2 * kGsW * DH + 2 * DHL + DM;  // mbarriers
  static constexpr int HEAD_DOUBLES = kGsTab * 32 + 8 + NBAR + (NBAR & 1);  // tables, ints, mbarriers
  static constexpr int WARP_DOUBLES = (3 * D + DH) * SLOT;
  static constexpr int LAST_DOUBLES = (3 * D + DHL) * SLOT;
  // warp 0's ring: the lagged ghost plane u(j,-1) when k0 == 0 (cp.async,
  // chunk layout), else the new rows of plane k0-1 (TMA bulk, padded rows)
  static constexpr int MR = (D * SLOT > DM * MROW) ? D * SLOT : DM * MROW;
  // multi-sweep mode (MS): the old rows travel beside the new ones (the
  // history residual of the previous sweep needs u^{s-1}(j, k-1)): one old
  // ring per warp hand-off, one for the publisher, one for warp 0's rows of
  // plane k0-1 (from the boundary buffer)
  static constexpr int OLD_DOUBLES = MS ? ((kGsW - 1) * DH * SLOT + DHL * SLOT + DM * MROW) : 0;
  static constexpr size_t SMEM =
      (size_t)(HEAD_DOUBLES + (kGsW - 1) * WARP_DOUBLES + LAST_DOUBLES + MR + OLD_DOUBLES) * sizeof(double);
  static constexpr int MINB = (NC >= 8 || MS) ? 1 : 2;
  __device__ static __forceinline__ int pos(int x) { return (x % NC) * IS + x / NC; }
};

__device__ __forceinline__ uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sm32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Deadlock guard for the progress spins: trap (a launch error, not a hung
// GPU) if one wait exceeds ~2^35 cycles (~17 s).
__device__ __forceinline__ long long clk64() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
struct SpinGuard {
  long long t0;
  __device__ __forceinline__ SpinGuard() : t0(clk64()) {}
  __device__ __forceinline__ void check() {
    if (clk64() - t0 > (1LL << 35)) __trap();
  }
};

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void gs_mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void gs_mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(sm32(bar)) : "memory");
}
__device__ __forceinline__ void gs_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm32(bar)) : "memory");
}
__device__ __forceinline__ void gs_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void gs_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "GMBW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra GMBW_%=;\n"
      "}\n" ::"r"(sm32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void gs_tma_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm32(dst)),
      "l"(src), "r"(bytes), "r"(sm32(bar))
      : "memory");
}

#ifdef PSM_GS_PROFILE
// phase timing of block 0, warp 0, lane 0 (tools/gs_phase_probe.py)
__device__ long long g_gs_prof[16];
#define GS_PROF(ph, dep)                                                   \
  do {                                                                     \
    if (prof_on) {                                                         \
      double _t;                                                           \
      asm volatile("mov.b64 %0, %1;" : "=d"(_t) : "d"((double)(dep)));     \
      (void)_t;                                                            \
      const long long _c = clk64();                                        \
      g_gs_prof[ph] += _c - prof_t;                                        \
      prof_t = _c;                                                         \
    }                                                                      \
  } while (0)
#else
#define GS_PROF(ph, dep) \
  do {                   \
  } while (0)
#endif

// Multi-sweep mode (MS = 1; one patch whose faces are all physical): the
// launch runs several GS steps, units (sweep s, k0) in s-major ticket order,
// so sweep s+1 trails sweep s by a few wavefronts instead of waiting for it
// to finish.  Every sweep has its own per-plane progress words (flags +
// s * flag_stride: a single word per plane would let a later sweep's
// progress stand in for an earlier one's); a unit of sweep s reads the old
// rows u(j+1, k) and u(j, k+1) only
// once sweep s-1 has published them (and, by the same wait, has consumed
// the values it overwrites), so the arithmetic is exactly that of s
// separate sweeps.  Ghost values are the step-end refresh's: every face is
// physical, ghost = -(the adjacent interior cell's value after the previous
// step), which each line has at hand as its own old value.  The history
// residual of sweep s-1's result is formed while sweep s passes over each
// cell (the old values of (j-1, k) and (j, k-1) travel beside the new ones;
// a unit's first plane gets them from the boundary buffer `oldb`, written
// by the previous unit's publisher) with the reference's operation order,
// and summed per plane into hist slot s-1.
template <int NC, int CHAOTIC, int UNIT, int MS>
__global__ void __launch_bounds__(kGsThreads, GCfg<NC, MS>::MINB)
    line_gs_pipe_kernel(const PatchDev* __restrict__ patches, const unsigned char* __restrict__ active,
                        StencilDev st, double omega, int* __restrict__ flags, int* __restrict__ ticket,
                        const int2* __restrict__ units, int nunits, const double* __restrict__ lane_tab,
                        const __grid_constant__ GsUniform T, int nl, double* __restrict__ hist,
                        long long hist_stride, double* __restrict__ oldb, int flag_stride) {
  using C = GCfg<NC, MS>;
  constexpr int M = NC - 1;  // locally eliminated cells per chunk
  const int nx = NC * nl;    // lanes nl..31 carry no cells (nx not 32*NC)
  constexpr int IS = C::IS, SLOT = C::SLOT, D = C::D, P = C::P, DH = C::DH, DHL = C::DHL, DM = C::DM;
  constexpr int MROW = C::MROW;
  extern __shared__ __align__(16) double gsm[];
  double* tab = gsm;                                   // [kGsTab][32]
  int* unit_sh = (int*)(gsm + kGsTab * 32);            // current unit
  uint64_t* bars = (uint64_t*)(gsm + kGsTab * 32 + 8);
  uint64_t* fullH = bars;                              // [kGsW][DH] warp w -> warp w+1
  uint64_t* emptyH = fullH + kGsW * DH;
  uint64_t* fullL = emptyH + kGsW * DH;                // [DHL] last warp -> publisher
  uint64_t* emptyL = fullL + DHL;
  uint64_t* mbarM = emptyL + DHL;                      // [DM] warp 0's TMA rows
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring = gsm + C::HEAD_DOUBLES;
  double* Ur = ring + warp * C::WARP_DOUBLES;          // old u(j+1,k) + x-ghosts of row j
  double* Zr = Ur + D * SLOT;                          // old u(j,k+1)
  double* Fr = Zr + D * SLOT;                          // f(j,k)
  double* Hr = Fr + D * SLOT;                          // new u(j,k)
  double* HL = ring + (kGsW - 1) * C::WARP_DOUBLES + 3 * D * SLOT;  // last warp's new rows (DHL)
  const double* Hprev = Hr - C::WARP_DOUBLES;          // previous warp's new rows
  double* Mr = ring + (kGsW - 1) * C::WARP_DOUBLES + C::LAST_DOUBLES;
  // MS: old-row rings (see GCfg::OLD_DOUBLES)
  double* oldr = Mr + C::MR;
  double* HO = oldr + (warp < kGsW - 1 ? warp : 0) * C::DH * SLOT;   // this warp's old rows -> next warp
  const double* HOprev = oldr + (warp > 0 ? warp - 1 : 0) * C::DH * SLOT;
  double* HLO = oldr + (kGsW - 1) * C::DH * SLOT;                     // last warp's old rows -> publisher
  double* MrO = HLO + C::DHL * SLOT;                                  // warp 0: old rows of plane k0-1
  uint32_t mbase = 0;  // warp 0: TMA row loads completed in earlier units

  for (int e = threadIdx.x; e < kGsTab * 32; e += blockDim.x) tab[e] = lane_tab[e];
  if (threadIdx.x == 0) {
    for (int i = 0; i < DM; ++i) gs_mbar_init(&mbarM[i], 1);
  }
  __syncthreads();
  const double* q = tab + lane;  // q[32*e]: this lane's table entry e
  int dpos[NC];  // shared-memory position of this lane's coalesced cell i*32+lane
#pragma unroll
  for (int i = 0; i < NC; ++i) dpos[i] = C::pos(i * 32 + lane);

  for (int first = 1;; first = 0) {
    if (threadIdx.x == 0) {
      unit_sh[0] = atomicAdd(ticket, 1);
      for (int i = 0; i < 2 * kGsW * DH + 2 * DHL; ++i) {
        if (!first) gs_mbar_inval(&bars[i]);
        gs_mbar_init(&bars[i], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int u = unit_sh[0];
    if (u >= nunits) return;
    const int2 U = units[u];
    const int sw = MS ? (U.x >> 16) : 0;   // sweep of this unit (MS)
    const int pidx = MS ? (U.x & 0xffff) : U.x;
    const PatchDev& Pd = patches[pidx];
    const int nz = Pd.nz, ny = Pd.ny;
    const long long px = nx + 2, pxy = px * (ny + 2);
    int* const fl = flags + (MS ? (long long)sw * flag_stride : 0);  // this sweep's progress words
    double* Ub = Pd.buf[active[pidx]];

    if (warp == kGsW) {
      // ======================= publisher ====================================
      const int kl = U.y + kGsW - 1;  // plane of the last compute warp
      if (kl < nz) {
        double* row0 = Ub + (long long)(kl + 1) * pxy + px + 1;
        int* my_flag = fl + Pd.plane0 + kl;
        const bool succ = kl + 1 < nz;
        // MS: the boundary buffer row of plane kl (old values, for the next
        // unit's history residual)
        double* ob = MS && succ ? oldb + (long long)(kl / kGsW) * ny * nx : nullptr;
        for (int j = 0; j < ny; ++j) {
          const int s = j % DHL;
          gs_mbar_wait(&fullL[s], (j / DHL) & 1);
          const double* hs = HL + s * SLOT;
          double* dst = row0 + (long long)j * px;
#pragma unroll
          for (int i = 0; i < NC; ++i)
            if (i * 32 + lane < nx) __stcg(dst + i * 32 + lane, hs[dpos[i]]);
          if (MS && ob) {
            const double* ho = HLO + s * SLOT;
#pragma unroll
            for (int i = 0; i < NC; ++i)
              if (i * 32 + lane < nx) __stcg(ob + (long long)j * nx + i * 32 + lane, ho[dpos[i]]);
          }
          __syncwarp();
          if (lane == 0) {
            gs_mbar_arrive(&emptyL[s]);
            // release: cumulative over the warp's stores (warp barrier above);
            // MS: every sweep's rows are published (the next sweep waits on them)
            if (MS) {
              if ((j + 1) % kGsPub == 0 || j == ny - 1) st_release_gpu(my_flag, j + 1);
            } else if (succ) {
              if (CHAOTIC) st_relaxed_gpu(my_flag, j + 1);
              else if ((j + 1) % kGsPub == 0 || j == ny - 1) st_release_gpu(my_flag, j + 1);
            }
          }
        }
      }
    } else if (U.y + warp < nz) {
      // ======================= compute warp: plane k ========================
      const int k = U.y + warp;
      const bool last = warp == kGsW - 1;
      const bool consumer = !last && (k + 1 < nz);
      double* row0 = Ub + (long long)(k + 1) * pxy + px + 1;  // u(0, 0, k)
      const double* Fk = Pd.f + (long long)k * ny * nx;
      const int* dep_flag = fl + Pd.plane0 + k - 1;
      // MS, sweep >= 1: old rows of plane k (row j+1) and k+1 (row j) must be
      // sweep sw-1's final values (lane 0 polls that sweep's words, caches
      // what it saw)
      const int* flag_k = fl - flag_stride + Pd.plane0 + k;
      const int* flag_k1 = flag_k + 1;
      int seen_k = 0, seen_k1 = 0;
      auto await_old = [&](int j) {
        if (!MS || sw == 0) return;
        if (lane == 0) {
          const int need_k = min(j + 2, ny), need_k1 = k + 1 < nz ? min(j + 1, ny) : 0;
          if (seen_k < need_k || seen_k1 < need_k1) {
            SpinGuard sg;
            while (seen_k < need_k) {
              seen_k = ld_relaxed_gpu(flag_k);
              if (seen_k < need_k) sg.check();
            }
            while (seen_k1 < need_k1) {
              seen_k1 = ld_relaxed_gpu(flag_k1);
              if (seen_k1 < need_k1) sg.check();
            }
            asm volatile("fence.acquire.gpu;" ::: "memory");  // acquire pattern with the relaxed loads
          }
        }
        __syncwarp();
      };

      auto issue = [&](int j) {
        if (j < ny) await_old(j);
        if (j < ny) {
          const int s = (j % D) * SLOT;
          const double* src_u = row0 + (long long)(j + 1) * px;
          const double* src_z = src_u - px + pxy;
          const double* src_f = Fk + (long long)j * nx;
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            const int x = i * 32 + lane;
            if (x < nx) {
              cp_async8(Ur + s + dpos[i], src_u + x);
              cp_async8(Zr + s + dpos[i], src_z + x);
              cp_async8(Fr + s + dpos[i], src_f + x);
            }
          }
          if (warp == 0 && k == 0) {
            const double* src_m = src_u - px - pxy;
#pragma unroll
            for (int i = 0; i < NC; ++i)
              if (i * 32 + lane < nx) cp_async8(Mr + s + dpos[i], src_m + i * 32 + lane);
          }
          if (lane < 2) cp_async8(Ur + s + NC * IS + lane, src_u - px + (lane ? nx : -1));
        }
        cp_commit();
      };

      double cen[NC], ym[NC];
      double ymo[NC];   // MS: old u(j-1, k) (the previous row's cen before the update)
      double hsum = 0.0;  // MS: sum of r^2 of sweep sw-1's result over this lane's cells of plane k
      await_old(0);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        cen[i] = lane < nl ? row0[lane * NC + i] : 0.0;
        // MS: the ghost row j = -1 after the previous step's refresh is -u(0, k)
        ym[i] = MS ? -cen[i] : (lane < nl ? row0[lane * NC + i - px] : 0.0);
        ymo[i] = ym[i];
      }
#pragma unroll
      for (int j = 0; j < P; ++j) issue(j);
      int avail = 0, issued = 0;  // warp 0, k > 0: rows of plane k-1 published / requested

#ifdef PSM_GS_PROFILE
      const bool prof_on = blockIdx.x == 0 && warp == 0 && lane == 0;
      long long prof_t = clk64();
#endif
      for (int j = 0; j < ny; ++j) {
        GS_PROF(0, 0.0);
        cp_wait<P - 1>();  // G(j) landed (G(j+1..j+P-1) may still fly)
        __syncwarp();
        GS_PROF(1, 0.0);
        const int s = (j % D) * SLOT;
        double nxt[NC], zp[NC], fv[NC], zm[NC], zmo[NC];
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          nxt[i] = Ur[s + i * IS + lane];
          zp[i] = Zr[s + i * IS + lane];
          fv[i] = Fr[s + i * IS + lane];
        }
        double gl = Ur[s + NC * IS], gr = Ur[s + NC * IS + 1];
        if (MS) {  // refreshed ghosts: -(own old end values), -(own old row / plane)
          gl = -__shfl_sync(0xffffffffu, cen[0], 0);
          gr = -__shfl_sync(0xffffffffu, cen[NC - 1], nl - 1);
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            if (j == ny - 1) nxt[i] = -cen[i];
            if (k == nz - 1) zp[i] = -cen[i];
          }
        }
        GS_PROF(2, 0.0);
        // ---- residual prefix, reference order (stencil.py:106-111): c u,
        // -x, +x, -y, +y need nothing from plane k-1, so they run before the
        // hand-off wait; -z (new) and +z follow it
        double acc[NC];
        {
          const double lft = __shfl_up_sync(0xffffffffu, cen[NC - 1], 1);
          const double rgt = __shfl_down_sync(0xffffffffu, cen[0], 1);
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            const double xl = i > 0 ? cen[i > 0 ? i - 1 : 0] : (lane == 0 ? gl : lft);
            const double xr = i < NC - 1 ? cen[i < NC - 1 ? i + 1 : 0] : (lane == nl - 1 ? gr : rgt);
            if (UNIT) {  // faces all -1: face*nbr is exactly -nbr, same roundings
              double a = __dmul_rn(st.c, cen[i]);
              a = __dsub_rn(a, xl);
              a = __dsub_rn(a, xr);
              a = __dsub_rn(a, ym[i]);
              acc[i] = __dsub_rn(a, nxt[i]);
            } else {
              double a = __dmul_rn(st.c, cen[i]);
              a = __dadd_rn(a, __dmul_rn(st.xm, xl));
              a = __dadd_rn(a, __dmul_rn(st.xp, xr));
              a = __dadd_rn(a, __dmul_rn(st.ym, ym[i]));
              acc[i] = __dadd_rn(a, __dmul_rn(st.yp, nxt[i]));
            }
          }
        }
        // ---- u(j, k-1), new ----------------------------------------------
        if (warp > 0) {
          const int hs = j % DH;
          gs_mbar_wait(&fullH[(warp - 1) * DH + hs], (j / DH) & 1);
          const double* h = Hprev + hs * SLOT;
#pragma unroll
          for (int i = 0; i < NC; ++i) zm[i] = h[i * IS + lane];
          if (MS) {
            const double* ho = HOprev + hs * SLOT;
#pragma unroll
            for (int i = 0; i < NC; ++i) zmo[i] = ho[i * IS + lane];
          }
          __syncwarp();
          if (lane == 0) gs_mbar_arrive(&emptyH[(warp - 1) * DH + hs]);
        } else if (k == 0) {
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            zm[i] = MS ? -cen[i] : Mr[s + i * IS + lane];  // MS: refreshed ghost plane
            zmo[i] = zm[i];
          }
        } else {
          // new rows of plane k0-1 (previous CTA's publisher): TMA bulk copies
          // through L2 (never a stale L1 line), issued once published
          if (lane == 0) {
            if (avail <= j) {
              SpinGuard sg;
              while ((avail = ld_relaxed_gpu(dep_flag)) <= j) sg.check();
              if (!CHAOTIC || MS) asm volatile("fence.acquire.gpu;" ::: "memory");  // (acquire pattern)
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const int lim = min(avail, j + DM);
            const double* ob = MS ? oldb + (long long)(k / kGsW - 1) * ny * nx : nullptr;
            for (; issued < lim; ++issued) {
              const uint32_t n = mbase + (uint32_t)issued;
              gs_mbar_expect_tx(&mbarM[n % DM], (uint32_t)(px * 8) + (MS && sw > 0 ? (uint32_t)(nx * 8) : 0u));
              gs_tma_row(Mr + (n % DM) * MROW, row0 + (long long)issued * px - pxy - 1, (uint32_t)(px * 8),
                         &mbarM[n % DM]);
              if (MS && sw > 0)
                gs_tma_row(MrO + (n % DM) * MROW, ob + (long long)issued * nx, (uint32_t)(nx * 8), &mbarM[n % DM]);
            }
          }
          __syncwarp();
          const uint32_t n = mbase + (uint32_t)j;
          gs_mbar_wait(&mbarM[n % DM], (n / DM) & 1);
          const double* mrow = Mr + (n % DM) * MROW + 1 + lane * NC;
#pragma unroll
          for (int i = 0; i < NC; ++i) zm[i] = mrow[i];
          if (MS && sw > 0) {
            const double* morow = MrO + (n % DM) * MROW + lane * NC;
#pragma unroll
            for (int i = 0; i < NC; ++i) zmo[i] = morow[i];
          }
        }
        GS_PROF(3, zm[NC - 1] + fv[NC - 1] + nxt[NC - 1] + zp[NC - 1]);
        if (MS && sw > 0 && hist) {
          // residual of sweep sw-1's result at this line (reference order:
          // c u, -x, +x, -y, +y, -z, +z, then f - acc), all old values
          const double lft = __shfl_up_sync(0xffffffffu, cen[NC - 1], 1);
          const double rgt = __shfl_down_sync(0xffffffffu, cen[0], 1);
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            const double xl = i > 0 ? cen[i > 0 ? i - 1 : 0] : (lane == 0 ? gl : lft);
            const double xr = i < NC - 1 ? cen[i < NC - 1 ? i + 1 : 0] : (lane == nl - 1 ? gr : rgt);
            double a;
            if (UNIT) {
              a = __dmul_rn(st.c, cen[i]);
              a = __dsub_rn(a, xl);
              a = __dsub_rn(a, xr);
              a = __dsub_rn(a, ymo[i]);
              a = __dsub_rn(a, nxt[i]);
              a = __dsub_rn(a, zmo[i]);
              a = __dsub_rn(a, zp[i]);
            } else {
              a = __dmul_rn(st.c, cen[i]);
              a = __dadd_rn(a, __dmul_rn(st.xm, xl));
              a = __dadd_rn(a, __dmul_rn(st.xp, xr));
              a = __dadd_rn(a, __dmul_rn(st.ym, ymo[i]));
              a = __dadd_rn(a, __dmul_rn(st.yp, nxt[i]));
              a = __dadd_rn(a, __dmul_rn(st.zm, zmo[i]));
              a = __dadd_rn(a, __dmul_rn(st.zp, zp[i]));
            }
            const double rr = lane < nl ? __dsub_rn(fv[i], a) : 0.0;
            hsum = fma(rr, rr, hsum);
          }
        }
        double r[NC];
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          if (UNIT) {
            r[i] = __dsub_rn(fv[i], __dsub_rn(__dsub_rn(acc[i], zm[i]), zp[i]));
          } else {
            const double a = __dadd_rn(acc[i], __dmul_rn(st.zm, zm[i]));
            r[i] = __dsub_rn(fv[i], __dadd_rn(a, __dmul_rn(st.zp, zp[i])));
          }
          if (lane >= nl) r[i] = 0.0;  // cell-less lanes: identity rows of the interface system
        }
        GS_PROF(4, r[NC - 1] + r[0]);
        // ---- exact line solve: local elimination + PCR ------------------
        // chunk interior: y = T_int^{-1} r as independent dot products (depth
        // M instead of the 2M-1 dependent steps of Thomas)
        double y[NC];
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double a = 0.0;
#pragma unroll
          for (int p = 0; p < M; ++p) a = fma(T.tinv[i][p], r[p], a);
          y[i] = a;
        }
        GS_PROF(5, y[0] + y[M > 0 ? M - 1 : 0]);
        double rho = q[0] * r[NC - 1];
        if (M > 0) {
          const double y0r = __shfl_down_sync(0xffffffffu, y[0], 1);
          rho = fma(-q[32], y[M > 0 ? M - 1 : 0], rho);
          rho = fma(-q[64], y0r, rho);
        }
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          if (t < T.npcr) {
            const int dd = 1 << t;
            const double rl = __shfl_up_sync(0xffffffffu, rho, dd);
            const double rr = __shfl_down_sync(0xffffffffu, rho, dd);
            rho = fma(-q[32 * (5 + 3 * t)], rr, fma(-q[32 * (4 + 3 * t)], rl, q[32 * (3 + 3 * t)] * rho));
          }
        }
        GS_PROF(6, rho);
        double al = __shfl_up_sync(0xffffffffu, rho, 1);
        if (lane == 0) al = 0.0;
        double nv[NC];
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const double xv = i < M ? fma(-rho, T.h[i], fma(-al, T.g[i], y[i])) : rho;
          nv[i] = relax(cen[i], omega, xv);
        }
        GS_PROF(7, nv[NC - 1] + nv[0]);
        // ---- hand the new row on -----------------------------------------
        if (last) {
          const int hs = j % DHL;
          if (j >= DHL) gs_mbar_wait(&emptyL[hs], ((j / DHL) - 1) & 1);
          double* h = HL + hs * SLOT;
#pragma unroll
          for (int i = 0; i < NC; ++i) h[i * IS + lane] = nv[i];
          if (MS) {
            double* ho = HLO + hs * SLOT;
#pragma unroll
            for (int i = 0; i < NC; ++i) ho[i * IS + lane] = cen[i];
          }
          __syncwarp();
          if (lane == 0) gs_mbar_arrive(&fullL[hs]);
        } else {
          const int hs = j % DH;
          if (consumer && j >= DH) gs_mbar_wait(&emptyH[warp * DH + hs], ((j / DH) - 1) & 1);
          double* h = Hr + hs * SLOT;
#pragma unroll
          for (int i = 0; i < NC; ++i) h[i * IS + lane] = nv[i];
          if (MS) {
            double* ho = HO + hs * SLOT;
#pragma unroll
            for (int i = 0; i < NC; ++i) ho[i * IS + lane] = cen[i];
          }
          __syncwarp();
          if (consumer && lane == 0) gs_mbar_arrive(&fullH[warp * DH + hs]);
          double* dst = row0 + (long long)j * px;
#pragma unroll
          for (int i = 0; i < NC; ++i)
            if (i * 32 + lane < nx) __stcg(dst + i * 32 + lane, h[dpos[i]]);
          if (MS) {  // publish this plane's progress for the next sweep
            __syncwarp();
            if (lane == 0 && ((j + 1) % kGsPub == 0 || j == ny - 1)) st_release_gpu(fl + Pd.plane0 + k, j + 1);
          }
        }
        issue(j + P);  // prefetch, off the hand-off critical path
        GS_PROF(8, 0.0);
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          ym[i] = nv[i];
          ymo[i] = cen[i];
          cen[i] = nxt[i];
        }
      }
      cp_wait<0>();
      if (warp == 0 && k > 0) mbase += (uint32_t)ny;
      if (MS && sw > 0 && hist) {
        // plane k's sum of sweep sw-1: fixed-order warp tree, into the first
        // history tile of the plane (the plane's other tiles hold zero)
#pragma unroll
        for (int o = 16; o; o >>= 1) hsum += __shfl_xor_sync(0xffffffffu, hsum, o);
        double* slot = hist + (long long)(sw - 1) * hist_stride + Pd.tile0 + (long long)k * Pd.tpp;
        for (int t = lane; t < Pd.tpp; t += 32) slot[t] = t == 0 ? hsum : 0.0;
      }
    }
    __syncthreads();
  }
}

template <int NC, int CH, int UN, int MS>
static int gs_pipe_occ1() {
  using C = GCfg<NC, MS>;
  cudaFuncSetAttribute(line_gs_pipe_kernel<NC, CH, UN, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, line_gs_pipe_kernel<NC, CH, UN, MS>, kGsThreads, C::SMEM);
  return b;
}
template <int NC>
static int gs_pipe_occupancy(int ms = 0) {
  if (ms)
    return std::min(std::min(gs_pipe_occ1<NC, 0, 0, 1>(), gs_pipe_occ1<NC, 0, 1, 1>()),
                    std::min(gs_pipe_occ1<NC, 1, 0, 1>(), gs_pipe_occ1<NC, 1, 1, 1>()));
  return std::min(std::min(gs_pipe_occ1<NC, 0, 0, 0>(), gs_pipe_occ1<NC, 0, 1, 0>()),
                  std::min(gs_pipe_occ1<NC, 1, 0, 0>(), gs_pipe_occ1<NC, 1, 1, 0>()));
}

template <int NC>
static cudaError_t gs_pipe_launch(int chaotic, int unit, int ms, int grid, const PatchDev* patches,
                                  const unsigned char* active, const StencilDev& st, double omega, int* flags,
                                  int* ticket, const int2* units, int nunits, const double* lane_tab,
                                  const GsUniform& T, int nl, double* hist, long long hist_stride, double* oldb,
                                  int flag_stride, cudaStream_t s) {
#define PSM_GSP(CH, UN, MS_)                                                                                 \
  line_gs_pipe_kernel<NC, CH, UN, MS_><<<grid, kGsThreads, GCfg<NC, MS_>::SMEM, s>>>(                        \
      patches, active, st, omega, flags, ticket, units, nunits, lane_tab, T, nl, hist, hist_stride, oldb, \
      flag_stride)
  if (ms) {
    if (chaotic) {
      if (unit) PSM_GSP(1, 1, 1); else PSM_GSP(1, 0, 1);
    } else {
      if (unit) PSM_GSP(0, 1, 1); else PSM_GSP(0, 0, 1);
    }
  } else if (chaotic) {
    if (unit) PSM_GSP(1, 1, 0); else PSM_GSP(1, 0, 0);
  } else {
    if (unit) PSM_GSP(0, 1, 0); else PSM_GSP(0, 0, 0);
  }
#undef PSM_GSP
  return cudaGetLastError();
}

}  // namespace psm

using namespace psm;

int psm_set_error(int code, const char* msg);
extern "C" cudaError_t psm_side_fork(psm_plan* P, cudaStream_t s, int n);  // psm_api.cu
extern "C" cudaError_t psm_side_join(psm_plan* P, cudaStream_t s, int n);

// One group of patches sharing nx (= NC * nl): units, tables, launch geometry.
struct GsPipeGroup {
  int nc = 0, nl = 32;
  int2* d_units = nullptr;
  int nunits = 0;
  double* d_tab = nullptr;  // [kGsTab][32]
  GsUniform T{};
  int grid = 0;
  int ticket = 0;  // index of this group's ticket in the plan's flag array
};

struct GsPipeState {
  std::vector<GsPipeGroup> groups;
  // multi-sweep launches (one patch): units per step count, boundary buffer
  std::map<int, std::pair<int2*, int>> ms_units;
  double* oldb = nullptr;
  int ms_occ = -1;
};

#ifdef PSM_GS_PROFILE
extern "C" int psm_debug_gs_profile(long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_gs_prof, sizeof(long long) * 16);
  if (reset) {
    long long z[16] = {0};
    cudaMemcpyToSymbol(g_gs_prof, z, sizeof z);
  }
  return 0;
}
#endif

// Chunk length for a line of nx cells: the smallest NC <= 8 dividing nx with
// nx / NC <= 32 lanes (32, 64, 128, 256 -> 1, 2, 4, 8 and all 32 lanes;
// e.g. 72 -> 3 x 24 lanes, 80 -> 4 x 20); 0 when there is none.  nx must be
// even: warp 0 pulls whole padded rows with 16-byte bulk copies.
static int gs_pipe_nc(int nx) {
  if (nx < 2 || (nx & 1)) return 0;
  for (int nc = 1; nc <= 8; ++nc)
    if (nx % nc == 0 && nx / nc <= 32) return nc;
  return 0;
}

bool gs_pipe_supported(int nx) { return gs_pipe_nc(nx) > 0; }

// Host tables (long double) for the chunked line solve of order nx = nc*nl
// with sub-diagonal lo, diagonal d and super-diagonal up; lanes nl..31 get
// identity rows.
static int gs_pipe_tables(int nc, int nl, long double lo, long double d, long double up, GsUniform& T,
                          double* lane_tab) {
  const int m = nc - 1;
  memset(&T, 0, sizeof T);
  long double invm[8] = {0}, cp[8] = {0}, g[8] = {0}, h[8] = {0};
  // Thomas factors of tridiag(lo, d, up) of order m
  long double prev_cp = 0;
  for (int i = 0; i < m; ++i) {
    const long double mi = d - (i > 0 ? lo * prev_cp : 0.0L);
    if (fabsl(mi) < 1e-14L * fabsl(d)) return psm_set_error(PSM_ESINGULAR, "line block pivot below 1e-14*|A|");
    invm[i] = 1.0L / mi;
    cp[i] = up * invm[i];
    prev_cp = cp[i];
  }
  auto solve = [&](const long double* rhs, long double* x) {
    long double y[8];
    for (int i = 0; i < m; ++i) y[i] = (rhs[i] - (i > 0 ? lo * y[i - 1] : 0.0L)) * invm[i];
    for (int i = m - 1; i >= 0; --i) x[i] = y[i] - (i < m - 1 ? cp[i] * x[i + 1] : 0.0L);
  };
  if (m > 0) {
    long double e[8] = {0};
    e[0] = lo;
    solve(e, g);
    e[0] = 0;
    e[m - 1] = up;
    solve(e, h);
  }
  for (int c = 0; c < m; ++c) {  // columns of the interior inverse
    long double e[8] = {0}, col[8];
    e[c] = 1.0L;
    solve(e, col);
    for (int i = 0; i < m; ++i) T.tinv[i][c] = (double)col[i];
  }
  for (int i = 0; i < m; ++i) {
    T.invm[i] = (double)invm[i];
    T.loinv[i] = (double)(lo * invm[i]);
    T.cp[i] = (double)cp[i];
    T.g[i] = (double)g[i];
    T.h[i] = (double)h[i];
  }
  // interface system  A_L a_{L-1} + B_L a_L + C_L a_{L+1} = rhs_L
  long double A[32], B[32], Cc[32];
  for (int L = 0; L < 32; ++L) {
    if (L >= nl) {  // no cells: a_L = 0
      A[L] = 0.0L;
      B[L] = 1.0L;
      Cc[L] = 0.0L;
    } else if (m == 0) {
      A[L] = L > 0 ? lo : 0.0L;
      B[L] = d;
      Cc[L] = L < nl - 1 ? up : 0.0L;
    } else {
      A[L] = L > 0 ? -lo * g[m - 1] : 0.0L;
      B[L] = d - lo * h[m - 1] - (L < nl - 1 ? up * g[0] : 0.0L);
      Cc[L] = L < nl - 1 ? -up * h[0] : 0.0L;
    }
    if (L < nl && fabsl(B[L]) < 1e-14L * fabsl(d))
      return psm_set_error(PSM_ESINGULAR, "line interface pivot below 1e-14*|A|");
  }
  long double al[32], ga[32];
  for (int L = 0; L < 32; ++L) {
    lane_tab[0 * 32 + L] = (double)(1.0L / B[L]);
    lane_tab[1 * 32 + L] = (m > 0 && L < nl) ? (double)(lo / B[L]) : 0.0;
    lane_tab[2 * 32 + L] = (m > 0 && L < nl - 1) ? (double)(up / B[L]) : 0.0;
    al[L] = A[L] / B[L];
    ga[L] = Cc[L] / B[L];
  }
  for (int t = 0; t < 5; ++t) {
    const int dd = 1 << t;
    long double na[32], ng[32];
    for (int L = 0; L < 32; ++L) {
      const long double gm = L - dd >= 0 ? ga[L - dd] : 0.0L, am = L - dd >= 0 ? al[L - dd] : 0.0L;
      const long double ap = L + dd < 32 ? al[L + dd] : 0.0L, gp = L + dd < 32 ? ga[L + dd] : 0.0L;
      const long double den = 1.0L - al[L] * gm - ga[L] * ap;
      if (fabsl(den) < 1e-14L) return psm_set_error(PSM_ESINGULAR, "line PCR pivot below 1e-14");
      lane_tab[(3 + 3 * t) * 32 + L] = (double)(1.0L / den);
      lane_tab[(4 + 3 * t) * 32 + L] = (double)(al[L] / den);
      lane_tab[(5 + 3 * t) * 32 + L] = (double)(ga[L] / den);
      na[L] = -al[L] * am / den;
      ng[L] = -ga[L] * gp / den;
    }
    memcpy(al, na, sizeof al);
    memcpy(ga, ng, sizeof ga);
    // couplings left after step t (normalised: unit diagonal); once they are
    // below 1e-20 the remaining steps change a_L by < 1e-20 max|a|
    long double cmax = 0;
    for (int L = 0; L < 32; ++L) cmax = fmaxl(cmax, fmaxl(fabsl(al[L]), fabsl(ga[L])));
    if (T.npcr == 0 && cmax < 1e-20L) T.npcr = t + 1;
  }
  if (T.npcr == 0) T.npcr = 5;
  return PSM_OK;
}

// Builds the groups of the plan (all patches must have a supported nx);
// flags: per global plane progress words, then one ticket per group.
int psm_gs_pipe_prepare(psm_plan* P, int* n_tickets) {
  if (P->gspipe) {
    *n_tickets = (int)P->gspipe->groups.size();
    return PSM_OK;
  }
  GsPipeState* S = new GsPipeState();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  std::vector<int> nxs;
  for (int p = 0; p < P->npatch; ++p) nxs.push_back(P->hp[p].nx);
  std::sort(nxs.begin(), nxs.end());
  nxs.erase(std::unique(nxs.begin(), nxs.end()), nxs.end());
  for (int nx : nxs) {
    const int nc = gs_pipe_nc(nx);
    if (nc == 0) {
      delete S;
      return psm_set_error(PSM_EUNSUPPORTED, "line GS pipeline: unsupported nx");
    }
    // units (patch, k0) plane-group-major: every patch's first group comes
    // before any second group, so independent patches fill the machine while
    // each patch's CTA chain (group k0 waits on group k0-W) stays in order
    std::vector<int> uv;
    int maxnz = 0;
    for (int p = 0; p < P->npatch; ++p) maxnz = std::max(maxnz, P->hp[p].nz);
    for (int k0 = 0; k0 < maxnz; k0 += kGsW)
      for (int p = 0; p < P->npatch; ++p) {
        if (P->hp[p].nx != nx || k0 >= P->hp[p].nz) continue;
        uv.push_back(p);
        uv.push_back(k0);
      }
    if (uv.empty()) continue;
    GsPipeGroup G;
    G.nc = nc;
    G.nl = nx / nc;
    G.nunits = (int)(uv.size() / 2);
    double tab[kGsTab * 32];
    int rc = gs_pipe_tables(nc, G.nl, (long double)P->st.xm, (long double)P->st.c, (long double)P->st.xp, G.T, tab);
    if (rc) {
      delete S;
      return rc;
    }
    if (cudaMalloc(&G.d_units, uv.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&G.d_tab, sizeof tab) != cudaSuccess) {
      delete S;
      return psm_set_error(PSM_ENOMEM, "cudaMalloc for line GS units");
    }
    cudaMemcpy(G.d_units, uv.data(), uv.size() * sizeof(int), cudaMemcpyHostToDevice);
    cudaMemcpy(G.d_tab, tab, sizeof tab, cudaMemcpyHostToDevice);
    int occ = 1;
    switch (nc) {
      case 1: occ = gs_pipe_occupancy<1>(); break;
      case 2: occ = gs_pipe_occupancy<2>(); break;
      case 3: occ = gs_pipe_occupancy<3>(); break;
      case 4: occ = gs_pipe_occupancy<4>(); break;
      case 5: occ = gs_pipe_occupancy<5>(); break;
      case 6: occ = gs_pipe_occupancy<6>(); break;
      case 7: occ = gs_pipe_occupancy<7>(); break;
      default: occ = gs_pipe_occupancy<8>(); break;
    }
    if (occ < 1) {
      delete S;
      return psm_set_error(PSM_ECUDA, "line GS pipeline kernel does not fit on an SM");
    }
    G.grid = std::min(G.nunits, occ * sms);
    G.ticket = (int)S->groups.size();
    S->groups.push_back(G);
  }
  P->gspipe = S;
  *n_tickets = (int)S->groups.size();
  return PSM_OK;
}

void psm_gs_pipe_free(psm_plan* P) {
  if (!P->gspipe) return;
  for (auto& G : P->gspipe->groups) {
    cudaFree(G.d_units);
    cudaFree(G.d_tab);
  }
  for (auto& kv : P->gspipe->ms_units) cudaFree(kv.second.first);
  cudaFree(P->gspipe->oldb);
  delete P->gspipe;
  P->gspipe = nullptr;
}

// flags: per-plane progress words (nplanes), tickets: one per group; both
// zeroed by the caller on the stream before the launch.
int psm_gs_pipe_sweep(psm_plan* P, const unsigned char* da, double omega, int chaotic, int* flags, int* tickets,
                      cudaStream_t s) {
  const bool unit = P->st.xm == -1.0 && P->st.xp == -1.0 && P->st.ym == -1.0 && P->st.yp == -1.0 &&
                    P->st.zm == -1.0 && P->st.zp == -1.0;
  // groups of different nx touch different patches: run them concurrently
  // (a group's persistent grid often leaves SMs free for the next)
  const int ng = (int)P->gspipe->groups.size();
  const bool fan = ng > 1;
  if (fan) {
    const cudaError_t e = psm_side_fork(P, s, ng);
    if (e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
  }
  int gi = 0;
  for (const GsPipeGroup& G : P->gspipe->groups) {
    cudaError_t e;
    int* tk = tickets + G.ticket;
    cudaStream_t s_main = s;
    if (fan) s = P->side[gi++ % psm_plan::kSide];
#define PSM_GSL(N)                                                                                                 \
  gs_pipe_launch<N>(chaotic, unit, 0, G.grid, P->d_patches, da, P->st, omega, flags, tk, G.d_units, G.nunits,       \
                    G.d_tab, G.T, G.nl, nullptr, 0, nullptr, 0, s)
    switch (G.nc) {
      case 1: e = PSM_GSL(1); break;
      case 2: e = PSM_GSL(2); break;
      case 3: e = PSM_GSL(3); break;
      case 4: e = PSM_GSL(4); break;
      case 5: e = PSM_GSL(5); break;
      case 6: e = PSM_GSL(6); break;
      case 7: e = PSM_GSL(7); break;
      default: e = PSM_GSL(8); break;
    }
#undef PSM_GSL
    if (e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
    P->launches += 1;
    s = s_main;
  }
  if (fan) {
    const cudaError_t e = psm_side_join(P, s, ng);
    if (e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
  }
  return PSM_OK;
}

// Several GS steps in one launch (multi-sweep mode of line_gs_pipe_kernel):
// one patch, every face physical, a prepared pipeline with one group.
// hist: history slots (slot s-1 gets the residual sums of step s's input,
// s = 1..steps-1; null: none); flags: steps * nplanes progress words and
// tickets, zeroed by the caller.
bool psm_gs_pipe_multi_ok(const psm_plan* P) {
  return P->gspipe && P->gspipe->groups.size() == 1 && P->npatch == 1 && P->ncopy == 0 &&
         P->hp[0].iface == 0 && !P->hp[0].peer_lo[0] && !P->hp[0].peer_hi[0];
}

int psm_gs_pipe_multi(psm_plan* P, const unsigned char* da, double omega, int chaotic, int steps, double* hist,
                      long long hist_stride, int* flags, int* tickets, cudaStream_t s) {
  if (!psm_gs_pipe_multi_ok(P) || steps < 1 || steps >= 0x7fff)
    return psm_set_error(PSM_EINVAL, "multi-sweep line GS needs one patch with physical faces");
  GsPipeState* S = P->gspipe;
  const GsPipeGroup& G = S->groups[0];
  const PatchDev& h = P->hp[0];
  auto it = S->ms_units.find(steps);
  if (it == S->ms_units.end()) {
    // ticket order: by k0 + (W+1) s, i.e. roughly the order in which units
    // become ready (sweep s+1 trails sweep s by about one plane group), so
    // CTAs do not sit on units far ahead of the wavefront.  Every unit a
    // unit waits on -- (s, k0-W), (s-1, k0), (s-1, k0+W) -- has a strictly
    // smaller key, so the order stays deadlock-free.
    std::vector<std::pair<long long, int2>> order;
    for (int sw = 0; sw < steps; ++sw)
      for (int k0 = 0; k0 < h.nz; k0 += kGsW)
        order.push_back({(long long)k0 + (long long)(kGsW + 1) * sw, make_int2(sw << 16, k0)});
    std::stable_sort(order.begin(), order.end(),
                     [](const std::pair<long long, int2>& a, const std::pair<long long, int2>& b) {
                       return a.first < b.first;
                     });
    std::vector<int> uv;
    for (auto& o : order) {
      uv.push_back(o.second.x);
      uv.push_back(o.second.y);
    }
    int2* d = nullptr;
    if (cudaMalloc(&d, uv.size() * sizeof(int)) != cudaSuccess)
      return psm_set_error(PSM_ENOMEM, "cudaMalloc for multi-sweep GS units");
    cudaMemcpy(d, uv.data(), uv.size() * sizeof(int), cudaMemcpyHostToDevice);
    it = S->ms_units.emplace(steps, std::make_pair(d, (int)(uv.size() / 2))).first;
  }
  if (!S->oldb) {
    const size_t n = (size_t)((h.nz + kGsW - 1) / kGsW) * h.ny * h.nx;
    if (cudaMalloc(&S->oldb, n * sizeof(double)) != cudaSuccess)
      return psm_set_error(PSM_ENOMEM, "cudaMalloc for the multi-sweep boundary rows");
  }
  if (S->ms_occ < 0) {
    switch (G.nc) {
      case 1: S->ms_occ = gs_pipe_occupancy<1>(1); break;
      case 2: S->ms_occ = gs_pipe_occupancy<2>(1); break;
      case 3: S->ms_occ = gs_pipe_occupancy<3>(1); break;
      case 4: S->ms_occ = gs_pipe_occupancy<4>(1); break;
      case 5: S->ms_occ = gs_pipe_occupancy<5>(1); break;
      case 6: S->ms_occ = gs_pipe_occupancy<6>(1); break;
      case 7: S->ms_occ = gs_pipe_occupancy<7>(1); break;
      default: S->ms_occ = gs_pipe_occupancy<8>(1); break;
    }
  }
  if (S->ms_occ < 1) return psm_set_error(PSM_ECUDA, "multi-sweep line GS kernel does not fit on an SM");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nunits = it->second.second;
  const int grid = std::min(nunits, S->ms_occ * sms);
  const bool unit = P->st.xm == -1.0 && P->st.xp == -1.0 && P->st.ym == -1.0 && P->st.yp == -1.0 &&
                    P->st.zm == -1.0 && P->st.zp == -1.0;
  cudaError_t e;
#define PSM_GSM(N)                                                                                             \
  gs_pipe_launch<N>(chaotic, unit, 1, grid, P->d_patches, da, P->st, omega, flags, tickets + G.ticket,          \
                    it->second.first, nunits, G.d_tab, G.T, G.nl, hist, hist_stride, S->oldb, P->nplanes, s)
  switch (G.nc) {
    case 1: e = PSM_GSM(1); break;
    case 2: e = PSM_GSM(2); break;
    case 3: e = PSM_GSM(3); break;
    case 4: e = PSM_GSM(4); break;
    case 5: e = PSM_GSM(5); break;
    case 6: e = PSM_GSM(6); break;
    case 7: e = PSM_GSM(7); break;
    default: e = PSM_GSM(8); break;
  }
#undef PSM_GSM
  if (e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
  P->launches += 1;
  return PSM_OK;
}
