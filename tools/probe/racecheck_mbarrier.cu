// Does compute-sanitizer racecheck see mbarrier arrive/wait ordering?
// Warp 0 writes a shared-memory row, __syncwarp, lane 0 arrives on an
// mbarrier (release.cta); warp 1 waits on it (acquire.cta) and reads the row
// -- the same hand-off as psm_line_gs_pipe.cu (fullH / emptyH).  A correct
// program; any racecheck hazard reported here is the tool's blind spot.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/rc tools/probe/racecheck_mbarrier.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase)
      : "memory");
}

__global__ void handoff(double* out, int rounds) {
  __shared__ double row[32];
  __shared__ uint64_t full, empty;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&empty, 1);
  }
  __syncthreads();
  double acc = 0.0;
  for (int r = 0; r < rounds; ++r) {
    if (warp == 0) {
      if (r > 0) mbar_wait(&empty, (r - 1) & 1);
      row[lane] = r + lane;
      __syncwarp();
      if (lane == 0) mbar_arrive(&full);
    } else {
      mbar_wait(&full, r & 1);
      acc += row[lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty);
    }
  }
  if (warp == 1) out[lane] = acc;
}

int main() {
  double* d;
  cudaMalloc(&d, 32 * sizeof(double));
  handoff<<<1, 64>>>(d, 8);
  double h[32];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int l = 0; l < 32; ++l) bad += h[l] != 8.0 * l + 28.0;
  printf("mbarrier hand-off: %s\n", bad ? "WRONG" : "ok");
  return bad;
}
