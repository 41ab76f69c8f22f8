// Internal device-side data structures of libpsmooth (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/psmooth.h"

namespace psm {

// True the first time it is called for the current device with this mask
// (one bit per device ordinal): per-device one-time setup such as the
// dynamic-shared-memory opt-in, which is a per-device function attribute.
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  return (mask.fetch_or(bit) & bit) == 0;
}

constexpr int kSeg = 32;  // line segment owned by one solver lane

// Exact line-block inverse in partitioned form (built by psm_factors_create).
// The closure-free line operator tridiag(lo, c, up) of order nx
// (stencil.py:115-138 with extent (nx,1,1)) is split into segments of 32
// (the last one `tail` long).  Every segment is the same local block, so one
// set of Thomas factors and two spike columns serves all of them:
//   g = T_32^{-1} e_0, h = T_32^{-1} e_31, gT = T_tail^{-1} e_0.
// A segment's exact solution is y - lo*x_left*g - up*x_right*h where y solves
// the local block; the interface values follow from 2x2 systems whose
// couplings to farther segments are below lo*g[31], up*h[0] (checked < 1e-18
// at build time, else the plan uses the generic full-Thomas kernel).
struct LineFac {
  double cp[kSeg], invm[kSeg];  // Thomas factors (prefix-valid for the tail)
  double g[kSeg], h[kSeg];      // spikes of a full segment
  double gT[kSeg];              // left spike of the tail segment
  double lo, up;                // coefficient of x-1 and x+1
  double up_h31;                // up * h[31]
  double lo_g0, lo_gT0;         // lo * g[0], lo * gT[0]
  double d_full, d_tail;        // 1/(1 - up*lo*h31*g0), same with gT0
  double g16[16], h16[16];      // spikes of a 16-cell half segment
  double up_h16, lo_g16, d16;   // up*h16[15], lo*g16[0], 1/(1 - up*lo*h16[15]*g16[0])
  int nx, nseg, tail;
  int partitioned;              // 1: segment kernel valid; 0: generic kernel
  // generic full-length Thomas factors (device pointers into the same
  // allocation), used when partitioned == 0
  const double* cpN;
  const double* invmN;
};

// Exact plane-block inverse: DST-I along x, then one tridiagonal system in y
// per x-mode (diagonal center + 2*a*cos(pi i/(nx+1))).
struct PlaneFac {
  int nx, ny;
  double fy_lo, fy_up;
  const double* Q;     // nx*nx orthonormal DST-I basis, symmetric
  const double* Qf;    // parity-split basis in DMMA fragment order (psm_plane_dst.cu)
  int nconst;          // rows >= nconst of cp / invm equal row nconst bitwise (every mode)
  const double* cp;    // [mode][ny] Thomas factors
  const double* invm;  // [mode][ny]
  // banded factorised form (psm_plane_band.cu); bw == 0: not available
  int bw, nj;          // convolution half-width, distinct leading Schur complements
  const double* H;     // [nj+1][bw+1] symmetric kernels H_j(0..bw)
};

// Box-block tables (psm_box.cu): per axis a and extent e in 1..8, forward
// F = Q diag(s^-p), backward B = diag(s^p) Q (8x8 row-major) and the eigen
// components L; the block's eigenvalue is c + Lx[i] + Ly[j] + Lz[k].
struct BoxFac {
  const double* F;
  const double* B;
  const double* L;
  const double* IL;  // 1/lambda per (ex, ey, ez) in [1,8]^3: [((ex-1)*8+ey-1)*8+ez-1][k][j][i] (stride 8)
  double c;
  int bx, by, bz;  // block dims (already truncated to the patch)
};

struct PatchDev {
  double* buf[2];
  const double* f;
  int nx, ny, nz;
  int R;          // rows (x-lines) per tile (the last tile of a plane may be short)
  int tpp;        // tiles per plane = ceil(ny / R)
  int tiles;      // tpp * nz
  long long tile0;  // first global tile
  int plane0;     // first global plane (prefix of nz)
  long long cell0;  // first interior cell (prefix of nx*ny*nz), for plane workspaces
  const LineFac* lf;
  const PlaneFac* pf;
  const BoxFac* bf;
  // fused multi-GPU halo (z-slabs): the neighbours' two buffers, mapped over
  // peer memory; the line-Jacobi sweep stores its first / last plane straight
  // into their ghost planes.  iface bit 1 / 2: the interior of the z-lo / z-hi
  // ghost plane is an interface (the physical fill leaves it alone).
  double* peer_lo[2];
  double* peer_hi[2];
  int peer_lo_nz;
  int iface;
  // bit 2*axis+side: that face's interior is wholly rewritten by one interface
  // copy, so the physical fill only needs its perimeter (edges, corners)
  int covered;
};

struct CopyDev {
  int src, dst;
  int src_lo[3], dst_lo[3], ext[3];
  long long elem0;  // prefix of element counts
};

struct StencilDev {
  double c, xm, xp, ym, yp, zm, zp;
};

__host__ __device__ inline int row_stride(int nx) { return nx + (nx + kSeg - 1) / kSeg; }

// tile -> (plane k, first row j0, rows in this tile); tiles never straddle planes
__device__ __forceinline__ void tile_coords(const PatchDev& P, long long tile, int& k, int& j0, int& rows) {
  const int ti = (int)(tile - P.tile0);
  k = ti / P.tpp;
  j0 = (ti - k * P.tpp) * P.R;
  rows = min(P.R, P.ny - j0);
}

__device__ __forceinline__ int find_patch(const PatchDev* __restrict__ p, int n, long long tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].tile0 <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// reference residual order (stencil.py:106-111): acc = c*u; acc += face*nbr
// for -x,+x,-y,+y,-z,+z; r = f - acc.  No FMA contraction, so the value is
// bit-identical to the reference for the same u and f.
__device__ __forceinline__ double residual7(const StencilDev& s, double f, double c, double xm, double xp,
                                            double ym, double yp, double zm, double zp) {
  double acc = __dmul_rn(s.c, c);
  acc = __dadd_rn(acc, __dmul_rn(s.xm, xm));
  acc = __dadd_rn(acc, __dmul_rn(s.xp, xp));
  acc = __dadd_rn(acc, __dmul_rn(s.ym, ym));
  acc = __dadd_rn(acc, __dmul_rn(s.yp, yp));
  acc = __dadd_rn(acc, __dmul_rn(s.zm, zm));
  acc = __dadd_rn(acc, __dmul_rn(s.zp, zp));
  return __dsub_rn(f, acc);
}

// block_update (smoother.py:93): u + omega * x, two roundings like numpy
__device__ __forceinline__ double relax(double u, double omega, double x) {
  return __dadd_rn(u, __dmul_rn(omega, x));
}

constexpr int kMaxTileCells = 2048;  // cells per line tile (8 per thread at 256 threads)

// Physical ghosts of v fused into a line-Jacobi sweep (grid.py:311-330 in the
// closed form of physical_ghost_kernel): the cell (x, j, k) just written with
// value nv (v index iu) also fills every y/z ghost cell whose nearest interior
// cell it is, sign (-1)^(number of ghost coordinates).  The x-only ghosts are
// the caller's (it already writes them).  The interior of a z face flagged as
// a peer interface (PatchDev::iface) is left to the neighbour's stores; its
// edges are still filled.  Call only for cells on a y or z boundary.
__device__ __forceinline__ void fused_yz_ghosts(double* __restrict__ v, long long iu, double nv, int x, int j, int k,
                                                int nx, int ny, int nz, long long px, long long pxy, int iface) {
  const int xs[3] = {0, x == 0 ? -1 : 2, x == nx - 1 ? 1 : 2};
  const int ys[3] = {0, j == 0 ? -1 : 2, j == ny - 1 ? 1 : 2};
  const int zs[3] = {0, k == 0 ? -1 : 2, k == nz - 1 ? 1 : 2};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int sz = zs[c];
    if (sz == 2) continue;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int sy = ys[b];
      if (sy == 2) continue;
      if (sy == 0 && sz == 0) continue;  // x-only ghosts: the caller's
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int sx = xs[a];
        if (sx == 2) continue;
        if (sx == 0 && sy == 0 && ((sz < 0 && (iface & 1)) || (sz > 0 && (iface & 2)))) continue;
        const int flips = (sx != 0) + (sy != 0) + (sz != 0);
        v[iu + sx + sy * px + sz * pxy] = (flips & 1) ? -nv : nv;
      }
    }
  }
}

}  // namespace psm

#include <map>
#include <string>
#include <vector>

struct PlaneState;  // psm_plane.cu
struct GsPipeState;  // psm_line_gs_pipe.cu

struct psm_factors {
  // host handle for one block shape
  int kind;
  int nx, ny;
  void* dev;            // one allocation: struct + tables
  psm::LineFac* d_line;      // kind == line
  psm::PlaneFac* d_plane;    // kind == plane
  psm::BoxFac* d_box;        // kind == box
  psm::LineFac h_line;       // host copy (pointers refer to device memory)
  psm::PlaneFac h_plane;
  psm::BoxFac h_box;
  int nz;                    // box blocks: ez
  double center, faces[6];
};

struct psm_plan {
  int npatch = 0, ncopy = 0, kind = 0;
  psm::StencilDev st{};
  std::vector<psm::PatchDev> hp;
  std::vector<psm_factors*> fac;
  psm::PatchDev* d_patches = nullptr;
  psm::CopyDev* d_copies = nullptr;
  long long copy_total = 0;
  long long* d_gprefix = nullptr;
  long long ghost_total = 0;
  long long ghost_max_face = 0;  // largest face of any patch (ghost kernel grid)
  long long copy_max = 0;        // largest interface copy (copy kernel grid)
  long long ntiles = 0;
  int nplanes = 0;
  int threads = 256;
  size_t smem = 0;
  int tiled = 1;  // line tile kernel usable (else generic one-thread-per-line kernels)
  std::map<std::string, unsigned char*> active_cache;
  int cap_slots = 0;
  double* d_partials = nullptr;    // cap_slots * ntiles
  double* d_plane_sums = nullptr;  // cap_slots * nplanes
  double* d_sums = nullptr;        // cap_slots
  double* d_scratch = nullptr;     // ntiles, for unrecorded sweeps
  // line GS
  int* d_flags = nullptr;         // per (patch, plane) progress counters
  int* d_unit_patch = nullptr;    // GS work units (patch, plane) in dependency order
  int* d_unit_plane = nullptr;
  long long nunits = 0;
  int gs_threads = 0, gs_grid = 0;
  size_t gs_smem = 0;
  long long launches = 0;  // kernels this plan launched (bench evidence)
  std::map<int, int> nx_grid;  // persistent grid per specialised nx
  std::map<std::string, std::pair<void*, int>> unit_cache;  // z-marching units per plane range
  // pipelined line GS (psm_line_gs_pipe.cu)
  GsPipeState* gspipe = nullptr;
  int* d_gsflags = nullptr;  // nplanes progress words + one ticket per group
  int gs_ntickets = 0;
  int* d_msflags = nullptr;   // multi-sweep line GS: steps * nplanes progress words + tickets
  long long ms_flag_cap = 0;
  // physical ghosts the sweeps since the last refresh left to it: 0 none
  // (one-tile / generic line-Jacobi kernels: written in their epilogues), 1
  // the y/z faces (z-marching line Jacobi, plane and box Jacobi: x faces
  // written), 2 all (GS sweeps); consulted by a refresh with PSM_GHOST_SKIP_X
  int phys_pending = 2;
  // side streams for independent launches of one sweep (line-GS groups of
  // different nx): fork / join by events, captured as parallel graph branches
  static constexpr int kSide = 4;
  cudaStream_t side[kSide] = {};
  cudaEvent_t side_fork = nullptr, side_join[kSide] = {};
  // box path: blocks (patch, x0, y0, z0) sorted by wavefront bi+bj+bk (GS),
  // and Jacobi regions of (8/bx) x (8/by) x (8/bz) blocks
  int4* d_boxes = nullptr;
  int nboxes = 0;
  int4* d_box_regions = nullptr;
  int4* d_box_deps = nullptr;   // per block (wavefront order): own flag, -x, -y, -z predecessor flags
  int* d_box_flags = nullptr;   // GS: nboxes done-flags + one ticket
  void* d_box_tmaps = nullptr;  // TMA tensor maps of the 8^3 region staging, 3 per patch (or null)
  int nregions = 0, reg_m[3] = {1, 1, 1};
  int box_dims[3] = {0, 0, 0};  // common block dims of all patches (0: they differ)
  std::vector<int> box_wave_off;  // blocks of wavefront w: [off[w], off[w+1])
  // plane path
  PlaneState* plane = nullptr;
  // CUDA graphs of whole smooth() step sequences (psm_smooth_steps)
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    long long kernels = 0;  // launches recorded at capture, added per replay
    int seen = 0;           // eager runs so far (capture on the second call)
  };
  std::map<std::string, GraphEntry> graphs;
};

