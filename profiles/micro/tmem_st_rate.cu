// Microbenchmark: tcgen05.st (32x32b) throughput per SM vs. how many stores
// are in flight before tcgen05.wait::st (K4 stores P as 2 x .x16 then waits).
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_12201_b200/csrc/common.cuh"
using namespace omni;
void omni_set_last_error(const char*) {}

template <int NST, int X>  // NST stores of .xX (X = 16 or 32 columns) per wait
__global__ void k(uint32_t* out, int iters, unsigned long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  // 16 warps: 4 lane quarters x 4 column groups of 128 columns
  const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128u * ((warp >> 2) & 3);
  uint32_t r[32];
  for (int c = 0; c < 32; ++c) r[c] = threadIdx.x + c;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      if (X == 16) tmem_st16(tl + 16u * s, r);
      else tmem_st32(tl + 32u * s, r);
    }
    tmem_wait_st();
    r[it & 15] += 1;
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = r[5];
  if ((threadIdx.x & 31) == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
template <int NST, int X>
void run(int warps) {
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int iters = 1000;
  for (int r = 0; r < 2; ++r) { cudaMemset(cyc, 0, 8); k<NST, X><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); }
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double cyc_per_warp = (double)h / (148.0 * warps);
  const double bytes = (double)warps * iters * NST * X * 128;
  printf("st.x%d x%d per wait, warps=%2d: %.1f cycles per iteration, %.1f B/clk/SM\n", X, NST, warps,
         cyc_per_warp / iters, bytes / cyc_per_warp);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 16}) { run<1, 16>(w); run<2, 16>(w); run<4, 16>(w); run<1, 32>(w); run<4, 32>(w); }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
