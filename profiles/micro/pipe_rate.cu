// Microbenchmark: warp-instruction throughput per SM sub-partition of the
// instructions in the K4 softmax mix (F2FP bf16 pack, FFMA2, FADD2, FMNMX3,
// IMAD, FMNMX), 8 warps per SMSP, 16 independent chains per thread.
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(uint32_t* out, int iters, unsigned long long* cyc) {
  uint32_t v[16];
  for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(0.5f + 0.001f * (threadIdx.x + i));
  uint64_t w[16];
  for (int i = 0; i < 16; ++i) w[i] = ((uint64_t)v[i] << 32) | v[(i + 1) & 15];
  const uint64_t c = w[3];
  long long t0; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (KIND == 0) asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(v[i]) : "r"(v[(i + 3) & 15]) : "memory");
      if (KIND == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(w[i]) : "l"(c) : "memory");
      if (KIND == 2) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(c) : "memory");
      if (KIND == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+r"(v[i]) : "r"(v[(i + 3) & 15]), "r"(v[(i + 5) & 15]));
      if (KIND == 4) asm volatile("mad.lo.u32 %0, %0, 8388608, %1;" : "+r"(v[i]) : "r"(v[(i + 3) & 15]) : "memory");
      if (KIND == 5) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(v[i]) : "r"(v[(i + 3) & 15]) : "memory");
      if (KIND == 6) asm volatile("max.f32 %0, %0, %1;" : "+r"(v[i]) : "r"(v[(i + 3) & 15]) : "memory");
      if (KIND == 8) { if (i & 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[i]) : "l"(c) : "memory");
                       else asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(w[i]) : "l"(c) : "memory"); }
      if (KIND == 7) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[i]));
    }
  }
  long long t1; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) :: "memory");
  uint32_t x = 0;
  for (int i = 0; i < 16; ++i) x ^= v[i] ^ (uint32_t)w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
  if (threadIdx.x % 32 == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}
template <int KIND>
void run(const char* name) {
  uint32_t* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
  const int wps = 8, threads = 128 * wps, iters = 1000;
  for (int r = 0; r < 2; ++r) { cudaMemset(cyc, 0, 8); k<KIND><<<148, threads>>>(out, iters, cyc); cudaDeviceSynchronize(); }
  unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double cyc_per_warp = (double)h / (148.0 * threads / 32);
  const double instr_per_clk_smsp = (double)wps * iters * 16 / cyc_per_warp;
  printf("%-22s %.3f warp-instr/clk/SMSP (%.1f cycles per warp-instr at the pipe)\n", name, instr_per_clk_smsp, 1.0 / instr_per_clk_smsp);
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<0>("F2FP.BF16 pack");
  run<1>("FFMA2");
  run<2>("FADD2");
  run<3>("FMNMX3");
  run<4>("IMAD");
  run<5>("FFMA");
  run<6>("FMNMX");
  run<7>("MUFU.EX2");
  run<8>("FFMA2+FADD2 mix");
  return 0;
}
