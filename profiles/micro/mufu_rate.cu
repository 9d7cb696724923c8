// Microbenchmark: MUFU.EX2 element throughput per SM sub-partition for
// ex2.approx.ftz.f32, ex2.approx.f16x2 and ex2.approx.ftz.bf16x2.
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  if (KIND == 0) for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[i]));
      if (KIND == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (KIND == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
    }
  }
  const long long t1 = clock64();
  uint32_t x = 0;
  for (int i = 0; i < 16; ++i) x ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x % 32 == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}
template <int KIND>
void run(int wps) {
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 2048 * 4); cudaMalloc(&cyc, 8);
  int threads = 128 * wps, iters = 1000;
  for (int r = 0; r < 2; ++r) { cudaMemset(cyc, 0, 8); k<KIND><<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize(); }
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double per_warp = (double)h / (148.0 * threads / 32) / iters / 16;  // cycles per instruction per warp
  const int elems = KIND == 0 ? 1 : 2;
  printf("kind=%s warps/SMSP=%d: %.2f cycles per warp-instr -> %.2f elements/clk/SMSP\n",
         KIND == 0 ? "f32" : KIND == 1 ? "f16x2" : "bf16x2", wps, per_warp, 32.0 * elems * wps / (per_warp * wps));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 4, 8}) { run<0>(w); run<1>(w); run<2>(w); }
  return 0;
}
