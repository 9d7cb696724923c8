// Microbenchmark: TMEM -> register bandwidth (tcgen05.ld.32x32b.x32) per SM
// for 4, 8 and 16 warps, and tcgen05.st bandwidth.
#include <cstdio>
#include <cstdint>
#include "../../paper_2511_12201_b200/csrc/common.cuh"
using namespace omni;
void omni_set_last_error(const char*) {}

template <bool STORE>
__global__ void k(uint32_t* out, int iters, unsigned long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 32u * ((warp >> 2) & 15);
  uint32_t r[32];
  for (int c = 0; c < 32; ++c) r[c] = threadIdx.x + c;
  uint32_t x = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (STORE) {
      tmem_st32(tl, r);
      tmem_wait_st();
      r[it & 31] += 1;
    } else {
      tmem_ld32(tl, r);
      tmem_wait_ld();
      x += r[0] ^ r[31];
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + r[5];
  if ((threadIdx.x & 31) == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
template <bool STORE>
void run(int warps) {
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int r = 0; r < 2; ++r) { cudaMemset(cyc, 0, 8); k<STORE><<<148, warps * 32>>>(out, iters, cyc); cudaDeviceSynchronize(); }
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double cyc_per_warp = (double)h / (148.0 * warps);
  const double bytes_per_clk_sm = (double)warps * iters * 4096 / cyc_per_warp;
  printf("%s warps=%2d: %.1f cycles per 4 KB op per warp, %.1f B/clk/SM\n", STORE ? "st" : "ld", warps,
         cyc_per_warp / iters, bytes_per_clk_sm);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 4, 8, 16}) run<false>(w);
  for (int w : {1, 4, 8, 16}) run<true>(w);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
