// L2 fp32 reduction throughput: every CTA red.global.add.v4.f32's 64 KB tiles
// (128 rows x 128 floats, one row per thread, like a TMEM dQ drain) into a
// [tiles][128][128] fp32 buffer; tiles are shared by `share` CTAs (several key
// tiles reduce into one Q tile). Reports GB/s of reduction payload.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128) red_kernel(float* buf, int ntiles, int iters, int share) {
  const int row = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const int t = ((blockIdx.x / share) * 7 + it * 13) % ntiles;
    float4* dst = reinterpret_cast<float4*>(buf + ((size_t)t * 128 + row) * 128);
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      float4 v = make_float4(1.f, 2.f, 3.f, (float)c);
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + c), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
    }
  }
}
int main() {
  const int ntiles = 28 * 256;  // 28 heads x 256 Q tiles (32K tokens)
  float* buf;
  cudaMalloc(&buf, (size_t)ntiles * 128 * 128 * 4);
  cudaMemset(buf, 0, (size_t)ntiles * 128 * 128 * 4);
  for (int share : {1, 8}) {
    for (int blocks : {148 * 4, 148 * 8}) {
      const int iters = 64;
      red_kernel<<<blocks, 128>>>(buf, ntiles, 2, share);
      cudaEvent_t a, b;
      cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      red_kernel<<<blocks, 128>>>(buf, ntiles, iters, share);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)blocks * iters * 128 * 128 * 4;
      printf("share %d blocks %d: %.3f ms, %.1f GB/s reduction payload\n", share, blocks, ms, bytes / ms / 1e6);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
