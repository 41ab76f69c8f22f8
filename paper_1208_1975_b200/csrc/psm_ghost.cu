// Ghost refresh and history reductions.
//
// Replaces Level.refresh_ghosts (grid.py:507-517):
//   fill_physical_ghosts       grid.py:311-330
//   exchange_interface_ghosts  grid.py:523-547
// and the summation of residual_norm (smoother.py:96-109).
#include <algorithm>

#include "psm_internal.cuh"

namespace psm {

// Physical ghosts.  The reference fills whole faces axis by axis (x, then y
// reading the fresh x ghosts, then z), so every ghost cell ends up as
// (-1)^(number of ghost coordinates) * u(nearest interior cell).  Computing
// that closed form per cell gives the same bits with no pass ordering, so one
// launch covers all faces of all patches: grid (chunk, patch, face), 32-bit
// index math, contiguous rows for the y and z faces.  Edge cells are written
// by several faces with the same value.  With skip_x the x faces are left to
// the Jacobi sweep, which already stored their interior; only their
// perimeter (edges shared with y/z faces) is rewritten here.
__global__ void __launch_bounds__(256) physical_ghost_kernel(const PatchDev* __restrict__ patches,
                                                             const unsigned char* __restrict__ active, int skip_x,
                                                             int use_covered, int pbase) {
  const int face = blockIdx.z, axis = face >> 1, side = face & 1;
  const int pi = pbase + blockIdx.y;
  const PatchDev& P = patches[pi];
  double* __restrict__ u = P.buf[active[pi]];
  const int px = P.nx + 2, py = P.ny + 2, pz = P.nz + 2;
  // face extent (A fastest, then B)
  const int A = axis == 0 ? py : px, B = axis == 2 ? py : pz;
  // faces whose interior something else writes (the Jacobi sweep's x faces,
  // a face one interface copy covers, a peer-halo z face): perimeter only
  // (covered faces only when this refresh also runs the interface copies:
  // a physical-only refresh must fill every face, grid.py:311-330)
  const bool perim = (axis == 0 && skip_x) || (use_covered && ((P.covered >> face) & 1)) ||
                     (axis == 2 && ((P.iface >> side) & 1));
  const int n = perim ? 2 * A + 2 * (B - 2) : A * B;
  for (int c = blockIdx.x * 1024 + threadIdx.x; c < min(n, (int)(blockIdx.x + 1) * 1024); c += 256) {
    int a, b;
    if (perim) {  // the face's border: rows b = 0 and B-1, then columns a = 0 and A-1
      if (c < 2 * A) {
        a = c % A;
        b = c < A ? 0 : B - 1;
      } else {
        const int q = c - 2 * A;
        a = (q & 1) ? A - 1 : 0;
        b = 1 + (q >> 1);
      }
    } else {
      b = c / A;
      a = c - b * A;
    }
    int i, j, k;
    if (axis == 0) { i = side ? px - 1 : 0; j = a; k = b; }
    else if (axis == 1) { i = a; j = side ? py - 1 : 0; k = b; }
    else { i = a; j = b; k = side ? pz - 1 : 0; }
    const int ic = min(max(i, 1), px - 2), jc = min(max(j, 1), py - 2), kc = min(max(k, 1), pz - 2);
    const int flips = (i != ic) + (j != jc) + (k != kc);
    const double val = u[(long long)ic + (long long)px * (jc + (long long)py * kc)];
    u[(long long)i + (long long)px * (j + (long long)py * k)] = (flips & 1) ? -val : val;
  }
}

// Cross-GPU step signals for the fused halo: after a sweep, publish "my
// boundary planes of step s are in your ghost planes" into the neighbour's
// flag word (system-scope release after the sweep's peer stores); before
// the next sweep, wait until both neighbours published step s.
__global__ void halo_signal_kernel(int* flag_a, int* flag_b, int value) {
  __threadfence_system();
  if (flag_a) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(flag_a), "r"(value) : "memory");
  if (flag_b) asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(flag_b), "r"(value) : "memory");
}

__global__ void halo_wait_kernel(const int* flags, int n, int value) {
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    int v;
    do {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + i) : "memory");
      if (clock64() - t0 > (1LL << 36)) __trap();  // a neighbour never signalled (~35 s)
    } while (v < value);
  }
  __threadfence_system();
}

cudaError_t launch_halo_signal(int* flag_a, int* flag_b, int value, cudaStream_t s) {
  halo_signal_kernel<<<1, 1, 0, s>>>(flag_a, flag_b, value);
  return cudaGetLastError();
}

cudaError_t launch_halo_wait(const int* flags, int n, int value, cudaStream_t s) {
  halo_wait_kernel<<<1, 1, 0, s>>>(flags, n, value);
  return cudaGetLastError();
}

// Interface ghosts: dst ghost layer <- src interior layer.  Sources are
// interior cells and destinations ghost cells, so no copy reads what another
// writes: the snapshot semantics of grid.py:530-546 hold in one launch.  Grid
// (chunk, copy), 32-bit index math, x fastest (contiguous runs).
__global__ void __launch_bounds__(256) interface_copy_kernel(const PatchDev* __restrict__ patches,
                                                             const unsigned char* __restrict__ active,
                                                             const CopyDev* __restrict__ copies, int cbase) {
  const CopyDev& C = copies[cbase + blockIdx.y];
  const int e0 = C.ext[0], e01 = C.ext[0] * C.ext[1], n = e01 * C.ext[2];
  const PatchDev& S = patches[C.src];
  const PatchDev& D = patches[C.dst];
  const double* __restrict__ su = S.buf[active[C.src]];
  double* __restrict__ du = D.buf[active[C.dst]];
  const long long spx = S.nx + 2, spy = S.ny + 2, dpx = D.nx + 2, dpy = D.ny + 2;
  const long long sb = (C.src_lo[0] + 1) + spx * ((C.src_lo[1] + 1) + spy * (C.src_lo[2] + 1));
  const long long db = (C.dst_lo[0] + 1) + dpx * ((C.dst_lo[1] + 1) + dpy * (C.dst_lo[2] + 1));
  for (int e = blockIdx.x * 1024 + threadIdx.x; e < min(n, (int)(blockIdx.x + 1) * 1024); e += 256) {
    const int c = e / e01, r = e - c * e01, b = r / e0, a = r - b * e0;
    du[db + a + dpx * (b + dpy * c)] = su[sb + a + spx * (b + spy * c)];
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

// max_face: largest face (cells) of any patch; 1024 cells per CTA
cudaError_t launch_physical_ghosts(const PatchDev* patches, int npatch, const unsigned char* active,
                                   long long max_face, int skip_x, int use_covered, cudaStream_t stream) {
  if (npatch == 0 || max_face == 0) return cudaSuccess;
  for (int base = 0; base < npatch; base += 65535) {
    const dim3 grid((unsigned)((max_face + 1023) / 1024), (unsigned)std::min(65535, npatch - base), 6);
    physical_ghost_kernel<<<grid, 256, 0, stream>>>(patches, active, skip_x, use_covered, base);
  }
  return cudaGetLastError();
}

// max_elems: largest copy (cells)
cudaError_t launch_interface_copies(const PatchDev* patches, const unsigned char* active, const CopyDev* copies,
                                    int ncopy, long long max_elems, cudaStream_t stream) {
  if (max_elems == 0 || ncopy == 0) return cudaSuccess;
  for (int base = 0; base < ncopy; base += 65535) {
    const dim3 grid((unsigned)((max_elems + 1023) / 1024), (unsigned)std::min(65535, ncopy - base), 1);
    interface_copy_kernel<<<grid, 256, 0, stream>>>(patches, active, copies, base);
  }
  return cudaGetLastError();
}

// All history slots at once: block s reduces slot s with exactly the
// arithmetic of plane_sums_kernel followed by tree_sum_kernel (each thread
// sums its chunk of planes in order, every plane's tiles in order, then the
// same pairwise tree), so the bits equal the two-launch path.
__global__ void __launch_bounds__(1024) history_reduce_kernel(const PatchDev* __restrict__ patches, int npatch,
                                                              const double* __restrict__ partials, long long tstride,
                                                              int nplanes, double* __restrict__ out) {
  __shared__ double buf[1024];
  const int t = threadIdx.x;
  const double* part = partials + (long long)blockIdx.x * tstride;
  const long long chunk = ((long long)nplanes + 1023) / 1024;
  const long long b = t * chunk, e = min((long long)nplanes, b + chunk);
  double s = 0.0;
  for (long long gp = b; gp < e; ++gp) {
    int lo = 0, hi = npatch - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (patches[mid].plane0 <= gp) lo = mid; else hi = mid - 1;
    }
    const PatchDev& P = patches[lo];
    const double* src = part + P.tile0 + (gp - P.plane0) * (long long)P.tpp;
    double ps = 0.0;
    for (int q = 0; q < P.tpp; ++q) ps += src[q];
    s += ps;
  }
  buf[t] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (t < w) buf[t] = buf[t] + buf[t + w];
    __syncthreads();
  }
  if (t == 0) out[blockIdx.x] = buf[0];
}

cudaError_t launch_history_reduce(const PatchDev* patches, int npatch, const double* partials, long long tstride,
                                  int nplanes, int nslots, double* out, cudaStream_t stream) {
  if (nslots <= 0) return cudaSuccess;
  history_reduce_kernel<<<nslots, 1024, 0, stream>>>(patches, npatch, partials, tstride, nplanes, out);
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
