// Ghost refresh and history reductions.
//
// Replaces Level.refresh_ghosts (grid.py:507-517):
//   fill_physical_ghosts       grid.py:311-330
//   exchange_interface_ghosts  grid.py:523-547
// and the summation of residual_norm (smoother.py:96-109).
#include "psm_internal.cuh"

namespace psm {

// Physical ghosts.  The reference fills whole faces axis by axis (x, then y
// reading the fresh x ghosts, then z), so every ghost cell ends up as
// (-1)^(number of ghost coordinates) * u(nearest interior cell).  Computing
// that closed form per cell gives the same bits with no pass ordering, so one
// launch covers all faces of all patches.  Face counts per patch: 2*py*pz (x),
// 2*px*pz (y), 2*px*py (z); edge cells are written by several faces with the
// same value.  With skip_x the x faces are left to the Jacobi sweep, which
// already stored them (their edges are rewritten by the y/z faces).
__global__ void physical_ghost_kernel(const PatchDev* __restrict__ patches, int npatch,
                                      const unsigned char* __restrict__ active,
                                      const long long* __restrict__ gprefix, long long total, int skip_x) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = npatch - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (gprefix[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const PatchDev& P = patches[lo];
    double* u = P.buf[active[lo]];
    const int px = P.nx + 2, py = P.ny + 2, pz = P.nz + 2;
    long long c = g - gprefix[lo];
    int i, j, k;
    const long long nxf = 2LL * py * pz, nyf = 2LL * px * pz;
    if (c < nxf) {
      const int side = (int)(c / ((long long)py * pz));
      const long long q = c - (long long)side * py * pz;
      j = (int)(q % py);
      k = (int)(q / py);
      i = side ? px - 1 : 0;
      if (skip_x && j > 0 && j < py - 1 && k > 0 && k < pz - 1) continue;
    } else if (c < nxf + nyf) {
      c -= nxf;
      const int side = (int)(c / ((long long)px * pz));
      const long long q = c - (long long)side * px * pz;
      i = (int)(q % px);
      k = (int)(q / px);
      j = side ? py - 1 : 0;
    } else {
      c -= nxf + nyf;
      const int side = (int)(c / ((long long)px * py));
      const long long q = c - (long long)side * px * py;
      i = (int)(q % px);
      j = (int)(q / px);
      k = side ? pz - 1 : 0;
    }
    const int ic = min(max(i, 1), px - 2), jc = min(max(j, 1), py - 2), kc = min(max(k, 1), pz - 2);
    const int flips = (i != ic) + (j != jc) + (k != kc);
    const double val = u[(long long)ic + (long long)px * (jc + (long long)py * kc)];
    u[(long long)i + (long long)px * (j + (long long)py * k)] = (flips & 1) ? -val : val;
  }
}

// Interface ghosts: dst ghost layer <- src interior layer.  Sources are
// interior cells and destinations ghost cells, so no copy reads what another
// writes: the snapshot semantics of grid.py:530-546 hold in one launch.
__global__ void interface_copy_kernel(const PatchDev* __restrict__ patches, const unsigned char* __restrict__ active,
                                      const CopyDev* __restrict__ copies, int ncopy, long long total) {
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = ncopy - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (copies[mid].elem0 <= g) lo = mid; else hi = mid - 1;
    }
    const CopyDev& C = copies[lo];
    const long long e = g - C.elem0;
    const int a = (int)(e % C.ext[0]);
    const long long t = e / C.ext[0];
    const int b = (int)(t % C.ext[1]);
    const int c = (int)(t / C.ext[1]);
    const PatchDev& S = patches[C.src];
    const PatchDev& D = patches[C.dst];
    const double* su = S.buf[active[C.src]];
    double* du = D.buf[active[C.dst]];
    const long long spx = S.nx + 2, spy = S.ny + 2, dpx = D.nx + 2, dpy = D.ny + 2;
    const long long si = (C.src_lo[0] + a + 1) + spx * ((C.src_lo[1] + b + 1) + spy * (C.src_lo[2] + c + 1));
    const long long di = (C.dst_lo[0] + a + 1) + dpx * ((C.dst_lo[1] + b + 1) + dpy * (C.dst_lo[2] + c + 1));
    du[di] = su[si];
  }
}

// Per-plane sums of tile partials, tiles of a plane in order.  One thread per
// global plane; plane gp belongs to the patch whose plane0 prefix covers it.
__global__ void plane_sums_kernel(const PatchDev* __restrict__ patches, int npatch, const double* __restrict__ partials,
                                  double* __restrict__ plane_sums, int nplanes) {
  const int gp = blockIdx.x * blockDim.x + threadIdx.x;
  if (gp >= nplanes) return;
  int lo = 0, hi = npatch - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (patches[mid].plane0 <= gp) lo = mid; else hi = mid - 1;
  }
  const PatchDev& P = patches[lo];
  const int k = gp - P.plane0;
  const int per = P.tpp;
  const double* src = partials + P.tile0 + (long long)k * per;
  double s = 0.0;
  for (int t = 0; t < per; ++t) s += src[t];
  plane_sums[gp] = s;
}

// Deterministic sum of n values: thread t adds a contiguous chunk in order,
// then a fixed pairwise tree over the 1024 chunk sums.  The association
// depends only on n, so equal vectors give equal bits on any device count.
__global__ void __launch_bounds__(1024) tree_sum_kernel(const double* __restrict__ in, long long n,
                                                        double* __restrict__ out) {
  __shared__ double buf[1024];
  const int t = threadIdx.x;
  const long long chunk = (n + 1023) / 1024;
  const long long b = t * chunk, e = min(n, b + chunk);
  double s = 0.0;
  for (long long i = b; i < e; ++i) s += in[i];
  buf[t] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (t < w) buf[t] = buf[t] + buf[t + w];
    __syncthreads();
  }
  if (t == 0) out[0] = buf[0];
}

// Interface ghosts from a remote rank: the interior (nx x ny) of a received
// contiguous padded plane goes into one z-ghost plane (grid.py:541-546 for a
// copy whose source lives on another GPU; edges stay physical as in the
// reference, whose InterfaceCopy extents never include edge cells).
__global__ void halo_unpack_kernel(double* __restrict__ dst_plane, const double* __restrict__ src_plane, int px,
                                   int py) {
  const long long n = (long long)(px - 2) * (py - 2);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (px - 2)) + 1, j = (int)(t / (px - 2)) + 1;
    const long long o = (long long)j * px + i;
    dst_plane[o] = src_plane[o];
  }
}

cudaError_t launch_halo_unpack(double* dst_plane, const double* src_plane, int px, int py, cudaStream_t stream) {
  const long long n = (long long)(px - 2) * (py - 2);
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  halo_unpack_kernel<<<(unsigned)blocks, 256, 0, stream>>>(dst_plane, src_plane, px, py);
  return cudaGetLastError();
}

cudaError_t launch_physical_ghosts(const PatchDev* patches, int npatch, const unsigned char* active,
                                   const long long* gprefix, long long total, int skip_x, cudaStream_t stream) {
  if (total == 0) return cudaSuccess;
  const int tpb = 256;
  long long blocks = (total + tpb - 1) / tpb;
  if (blocks > 148 * 64) blocks = 148 * 64;
  physical_ghost_kernel<<<(unsigned)blocks, tpb, 0, stream>>>(patches, npatch, active, gprefix, total, skip_x);
  return cudaGetLastError();
}

cudaError_t launch_interface_copies(const PatchDev* patches, const unsigned char* active, const CopyDev* copies,
                                    int ncopy, long long total, cudaStream_t stream) {
  if (total == 0 || ncopy == 0) return cudaSuccess;
  const int tpb = 256;
  long long blocks = (total + tpb - 1) / tpb;
  if (blocks > 148 * 64) blocks = 148 * 64;
  interface_copy_kernel<<<(unsigned)blocks, tpb, 0, stream>>>(patches, active, copies, ncopy, total);
  return cudaGetLastError();
}

cudaError_t launch_plane_sums(const PatchDev* patches, int npatch, const double* partials, double* plane_sums,
                              int nplanes, cudaStream_t stream) {
  if (nplanes == 0) return cudaSuccess;
  plane_sums_kernel<<<(nplanes + 127) / 128, 128, 0, stream>>>(patches, npatch, partials, plane_sums, nplanes);
  return cudaGetLastError();
}

cudaError_t launch_tree_sum(const double* in, long long n, double* out, cudaStream_t stream) {
  tree_sum_kernel<<<1, 1024, 0, stream>>>(in, n, out);
  return cudaGetLastError();
}

}  // namespace psm
