// Per-block primitives of the reference API, on the device.
//
// The smoother never calls these (its sweeps fuse the residual, the exact
// block solve and the update into one kernel); they back the reference's
// public building blocks so code written against them runs unchanged:
//   psm_box_residual  -> block_residual   stencil.py:93-112  (f - A u on a box)
//                        apply_stencil    stencil.py:71-84   (A u, no f)
//   psm_matvec        -> matvec           blocklinalg.py:90-105
//                        block_update     smoother.py:90-93  (u + omega M r)
//   psm_invert_dense  -> invert_dense     blocklinalg.py:50-87
// Rounding: residual and matvec use separate multiply and add roundings
// (__dmul_rn / __dadd_rn, no FMA contraction) in the reference's order, so
// their results are bit-identical to the reference's numpy arithmetic.
#include <math.h>

#include <algorithm>

#include "psm_internal.cuh"

int psm_set_error(int code, const char* msg);

namespace psm {

// out[x + ex*(y + ey*z)] for the box [lo, lo+ext) of the interior:
// acc = c*u; acc += face_d * u[shift_d] for d = -x,+x,-y,+y,-z,+z; then
// out = f - acc (or acc when f is null).  One thread per cell, x fastest.
__global__ void box_residual_kernel(const double* __restrict__ u, const double* __restrict__ f, int nx, int ny,
                                    int lo0, int lo1, int lo2, int ex, int ey, long long n, StencilDev st,
                                    double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int x = (int)(t % ex);
  const long long q = t / ex;
  const int y = (int)(q % ey), z = (int)(q / ey);
  const long long px = nx + 2, pxy = px * (ny + 2);
  const int i = lo0 + x, j = lo1 + y, k = lo2 + z;
  const long long c = (i + 1) + px * (j + 1) + pxy * (k + 1);
  double acc = __dmul_rn(st.c, u[c]);
  acc = __dadd_rn(acc, __dmul_rn(st.xm, u[c - 1]));
  acc = __dadd_rn(acc, __dmul_rn(st.xp, u[c + 1]));
  acc = __dadd_rn(acc, __dmul_rn(st.ym, u[c - px]));
  acc = __dadd_rn(acc, __dmul_rn(st.yp, u[c + px]));
  acc = __dadd_rn(acc, __dmul_rn(st.zm, u[c - pxy]));
  acc = __dadd_rn(acc, __dmul_rn(st.zp, u[c + pxy]));
  out[t] = f ? __dsub_rn(f[i + (long long)nx * (j + (long long)ny * k)], acc) : acc;
}

// y = M x with M column-major, accumulated over ascending columns with one
// rounding per multiply and per add (the reference's axpy loop); with u:
// y = u + omega * y (block_update).  One thread per row: each column read is
// coalesced across the warp.
__global__ void matvec_kernel(const double* __restrict__ m, const double* __restrict__ x,
                              const double* __restrict__ u, double omega, double* __restrict__ y, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  const double* col = m + i;
  for (int j = 0; j < n; ++j, col += n) acc = __dadd_rn(acc, __dmul_rn(*col, __ldg(x + j)));
  y[i] = u ? __dadd_rn(u[i], __dmul_rn(omega, acc)) : acc;
}

// ---- Gauss-Jordan inverse with partial pivoting on W = [A | I] (n x 2n,
// column-major, leading dimension n).  Step k: one CTA picks the pivot row
// (largest |W[i,k]|, i >= k, first on ties), records the singular step,
// swaps rows k and p and stages the scaled pivot row and the column-k
// multipliers; a grid then eliminates column k from every other row.
struct GJState {
  double anorm;
  int singular_step;  // 0 = regular, else 1 + step of the first tiny pivot
  double tiny_pivot;
};

__global__ void __launch_bounds__(1024) gj_norm_kernel(const double* __restrict__ w, int n, GJState* S) {
  __shared__ double red[32];
  double best = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += fabs(w[i + (long long)j * n]);
    best = fmax(best, s);
  }
  for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (threadIdx.x == 0) {
      S->anorm = best;
      S->singular_step = 0;
      S->tiny_pivot = 0.0;
    }
  }
}

__global__ void __launch_bounds__(1024) gj_pivot_kernel(double* __restrict__ w, int n, int k, GJState* S,
                                                        double rtol, double* __restrict__ rowk,
                                                        double* __restrict__ colk) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ int piv;
  if (S->singular_step) return;
  // argmax |W[i,k]| over i >= k, smallest index on ties
  double bv = -1.0;
  int bi = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(w[i + (long long)k * n]);
    if (a > bv) { bv = a; bi = i; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = bv; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool have = threadIdx.x < (blockDim.x >> 5);
    bv = have ? sv[threadIdx.x] : -1.0;
    bi = have ? si[threadIdx.x] : n;
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (threadIdx.x == 0) piv = bi;
  }
  __syncthreads();
  const int p = piv;
  const double pivot = w[p + (long long)k * n];
  if (!(fabs(pivot) >= rtol * S->anorm)) {  // also catches NaN
    if (threadIdx.x == 0) { S->singular_step = k + 1; S->tiny_pivot = pivot; }
    return;
  }
  // swap rows k and p over every column >= k (the columns < k of the left
  // half are unit vectors e_j, j < k: zero in both rows)
  for (int j = k + threadIdx.x; j < 2 * n; j += blockDim.x) {
    double* c = w + (long long)j * n;
    const double a = c[k], b = c[p];
    c[k] = b;
    c[p] = a;
    rowk[j] = b / pivot;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) colk[i] = w[i + (long long)k * n];
}

__global__ void gj_eliminate_kernel(double* __restrict__ w, int n, int k, const GJState* __restrict__ S,
                                    const double* __restrict__ rowk, const double* __restrict__ colk) {
  if (S->singular_step) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = k + blockIdx.y;
  if (i >= n) return;
  const double r = rowk[j];
  double* c = w + (long long)j * n;
  c[i] = i == k ? r : c[i] - colk[i] * r;
}

}  // namespace psm

using namespace psm;

static StencilDev stencil_dev(const psm_stencil* st) {
  StencilDev s;
  s.c = st->center;
  s.xm = st->faces[0];
  s.xp = st->faces[1];
  s.ym = st->faces[2];
  s.yp = st->faces[3];
  s.zm = st->faces[4];
  s.zp = st->faces[5];
  return s;
}

extern "C" {

int psm_box_residual(const double* u, const double* f, int nx, int ny, int nz, const int* lo, const int* ext,
                     const psm_stencil* st, double* out, void* stream) {
  if (!u || !lo || !ext || !st || !out || nx < 1 || ny < 1 || nz < 1)
    return psm_set_error(PSM_EINVAL, "box_residual: bad arguments");
  const int dims[3] = {nx, ny, nz};
  for (int a = 0; a < 3; ++a)
    if (lo[a] < 0 || ext[a] < 1 || lo[a] + ext[a] > dims[a])
      return psm_set_error(PSM_EINVAL, "box_residual: box leaves the interior");
  const long long n = (long long)ext[0] * ext[1] * ext[2];
  box_residual_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      u, f, nx, ny, lo[0], lo[1], lo[2], ext[0], ext[1], n, stencil_dev(st), out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PSM_OK : psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
}

int psm_matvec(const double* m, const double* x, const double* u, double omega, double* y, int n, void* stream) {
  if (!m || !x || !y || n < 1) return psm_set_error(PSM_EINVAL, "matvec: bad arguments");
  matvec_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(m, x, u, omega, y, n);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PSM_OK : psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
}

int psm_invert_dense(double* w, int n, double* work, int* singular_step, double* tiny_pivot, void* stream) {
  if (!w || !work || !singular_step || n < 1 || n > 32767)
    return psm_set_error(PSM_EINVAL, "invert_dense: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  double* rowk = work;
  double* colk = work + 2 * (size_t)n;
  GJState* S = reinterpret_cast<GJState*>(work + 3 * (size_t)n);
  gj_norm_kernel<<<1, 1024, 0, s>>>(w, n, S);
  for (int k = 0; k < n; ++k) {
    gj_pivot_kernel<<<1, 1024, 0, s>>>(w, n, k, S, 1e-14, rowk, colk);
    const dim3 grid((unsigned)((n + 127) / 128), (unsigned)(2 * n - k));
    gj_eliminate_kernel<<<grid, 128, 0, s>>>(w, n, k, S, rowk, colk);
  }
  GJState h;
  cudaError_t e = cudaMemcpyAsync(&h, S, sizeof h, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return psm_set_error(PSM_ECUDA, cudaGetErrorString(e));
  *singular_step = h.singular_step;
  if (tiny_pivot) *tiny_pivot = h.tiny_pivot;
  if (h.anorm == 0.0) {
    *singular_step = -1;
    return psm_set_error(PSM_ESINGULAR, "matrix is exactly zero");
  }
  if (h.singular_step) return psm_set_error(PSM_ESINGULAR, "pivot below 1e-14 * ||A||_inf");
  return PSM_OK;
}

}  // extern "C"
