// Microbenchmark: throughput of the K4 softmax instruction mix (scale+max,
// exp2 via MUFU or the FMA-pipe polynomial, row sum, bf16 pack) on register
// data, for W warps per SM sub-partition. Prints cycles per 32-column chunk
// per warp. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_2511_12201_b200/csrc
#include <cstdio>
#include "../../paper_2511_12201_b200/csrc/common.cuh"
using namespace omni;

void omni_set_last_error(const char*) {}

template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

template <int POLY, int MODE>
__global__ void mix(float* out, int iters, unsigned long long* cyc) {
  uint32_t sr[32];
  for (int c = 0; c < 32; ++c) sr[c] = __float_as_uint(0.01f * (threadIdx.x + c));
  const float sl2 = 0.1275f;
  const Exp2PolyConsts pc = exp2_poly_consts();
  float m = 1.0f, l = 0.f;
  uint32_t acc_pk = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      m0 = fmax3(m0, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
      m1 = fmax3(m1, __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
    }
    const float nmu = -m;
    const uint64_t c2 = f32x2(sl2, sl2), n2 = f32x2(nmu, nmu);
    uint64_t acc0 = f32x2(0.f, 0.f), acc1 = f32x2(0.f, 0.f);
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      const uint64_t xx = ffma2(f32x2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), c2, n2);
      uint64_t pp;
      if (use_poly<POLY>(c >> 1)) pp = exp2_poly_pair(xx, pc);
      else pp = f32x2(fast_exp2(f32x2_lo(xx)), fast_exp2(f32x2_hi(xx)));
      if (MODE == 0) { if ((c & 2) == 0) acc0 = fadd2(acc0, pp); else acc1 = fadd2(acc1, pp); }
      pk[c >> 1] = pack_bf16x2(f32x2_lo(pp), f32x2_hi(pp));
    }
    const uint64_t acc = fadd2(acc0, acc1);
    l += f32x2_lo(acc) + f32x2_hi(acc);
#pragma unroll
    for (int c = 0; c < 16; ++c) acc_pk ^= pk[c];
    m = fmaxf(m, fmaxf(m0, m1) * 1e-30f);
    // perturb inputs so the loop is not hoisted
#pragma unroll
    for (int c = 0; c < 32; ++c) sr[c] ^= (acc_pk & 1);
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + __uint_as_float(acc_pk);
  if (threadIdx.x % 32 == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
}

template <int POLY>
void run(int warps_per_smsp) {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  const int threads = 128 * warps_per_smsp;
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    mix<POLY, 0><<<148, threads>>>(out, iters, cyc);
    cudaDeviceSynchronize();
  }
  unsigned long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp = (double)h / (148.0 * threads / 32);
  printf("POLY=%d warps/SMSP=%d: %.1f cycles per 32-col chunk per warp (%.1f per chunk per SMSP)\n", POLY,
         warps_per_smsp, per_warp / iters, per_warp / iters / warps_per_smsp);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 4}) {
    run<0>(w);
    run<4>(w);
    run<6>(w);
    run<8>(w);
  }
  return 0;
}
