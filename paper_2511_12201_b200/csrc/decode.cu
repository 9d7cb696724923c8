// K7: slimmed decode attention (split-K flash decoding over the slim cache).
//
// Replaces classify_decode_query + _fetched_segments + decode_attention
// (decode.py:124-194) for a batch of sequences under GQA rule B. Work unit =
// (sequence, KV group, 256-key chunk) so 32 sequences x 4 groups x ~120
// chunks fill the 148 SMs many times over. Every CTA re-derives its group's
// lazy/active flags in float64 from the frozen probe keys (7 x 2 dot products
// — cheaper than a separate launch); a vision chunk of a group whose Q heads
// are all lazy exits before touching HBM, which is exactly the KV-fetch skip
// of decode.py:176-190. The kernel is HBM-bound: K and V of a chunk are read
// once into padded shared memory and reused by all Q heads of the group.
// A second kernel merges the per-chunk (max, sum, acc) partials per Q head.
#include <math.h>

#include "common.cuh"

namespace omni {
namespace dec {

constexpr int CHUNK = 256;
constexpr int D = 128;
constexpr int ROWB = D * 2 + 16;  // padded smem row (bytes): conflict-free 16B reads
constexpr int MAXREP = 16;

__global__ void __launch_bounds__(256) decode_partial_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ vk, const __nv_bfloat16* __restrict__ vv,
    const int32_t* __restrict__ vlen, const __nv_bfloat16* __restrict__ tk, const __nv_bfloat16* __restrict__ tv,
    int nt, const __nv_bfloat16* __restrict__ ak, const __nv_bfloat16* __restrict__ av, int na,
    const double* __restrict__ k_lazy, const double* __restrict__ k_act, int Hq, int Hkv, int vcap, int acap,
    double tau, int preserve, const uint8_t* __restrict__ flags_override, uint8_t* __restrict__ flags_out,
    int vis_chunks, float* __restrict__ part_ml, float* __restrict__ part_acc, int n_chunks) {
  extern __shared__ __align__(16) uint8_t sh[];
  uint8_t* sK = sh;                                   // [CHUNK][ROWB]
  uint8_t* sV = sh + CHUNK * ROWB;                    // [CHUNK][ROWB]
  float* sQ = reinterpret_cast<float*>(sh + 2 * CHUNK * ROWB);  // [rep][D]
  float* sP = sQ + MAXREP * D;                        // [rep][CHUNK]
  float* sRed = sP + MAXREP * CHUNK;                  // [8][rep] / [4][rep][D] reuse
  __shared__ int s_flag[MAXREP];
  __shared__ int s_any;

  const int c = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int rep = Hq / Hkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---- flags for this group's Q heads (f64, query_select.py:63-68)
  if (warp == 0) {
    const double scale = 1.0 / sqrt(static_cast<double>(D));
    for (int r = 0; r < rep; ++r) {
      const int h = g * rep + r;
      int f;
      if (flags_override) {
        f = flags_override[(size_t)s * Hq + h] ? 1 : 0;
      } else {
        double dl = 0.0, da = 0.0;
        for (int e = lane; e < D; e += 32) {
          const double x = static_cast<double>(__bfloat162float(q[((size_t)s * Hq + h) * D + e]));
          dl = fma(x, k_lazy[((size_t)s * Hkv + g) * D + e], dl);
          da = fma(x, k_act[((size_t)s * Hkv + g) * D + e], da);
        }
        dl = warp_sum(dl);
        da = warp_sum(da);
        const double l0 = dl * scale, l1 = da * scale, mx = fmax(l0, l1);
        const double e0 = exp(l0 - mx), e1 = exp(l1 - mx);
        f = (e1 / (e0 + e1) > tau) ? 1 : 0;
        if (preserve && h == 0) f = 1;
      }
      if (lane == 0) {
        s_flag[r] = f;
        if (c == 0) flags_out[(size_t)s * Hq + h] = static_cast<uint8_t>(f);
      }
    }
    if (lane == 0) {
      int any = 0;
      for (int r = 0; r < rep; ++r) any |= s_flag[r];
      s_any = any;
    }
  }
  __syncthreads();

  // ---- key range of this chunk
  const bool is_vis = c < vis_chunks;
  int k0, k1;
  const __nv_bfloat16 *kbase = nullptr, *vbase = nullptr;
  if (is_vis) {
    const int vl = vlen[s];
    k0 = c * CHUNK;
    k1 = min(vl, k0 + CHUNK);
    if (!s_any) k1 = k0;  // group lazy: no vision fetch
    kbase = vk + ((size_t)s * Hkv + g) * vcap * D;
    vbase = vv + ((size_t)s * Hkv + g) * vcap * D;
  } else {
    k0 = (c - vis_chunks) * CHUNK;
    k1 = min(nt + na, k0 + CHUNK);
  }
  const int nk = max(0, k1 - k0);
  float* ml = part_ml + (((size_t)s * Hq + g * rep) * n_chunks + c) * 2;
  float* acc_out = part_acc + (((size_t)s * Hq + g * rep) * n_chunks + c) * D;
  if (nk == 0) {
    if (tid < rep) {
      ml[(size_t)tid * n_chunks * 2 + 0] = -INFINITY;
      ml[(size_t)tid * n_chunks * 2 + 1] = 0.f;
    }
    return;
  }

  // ---- stage q (f32) and the K/V chunk (bf16) in smem
  for (int e = tid; e < rep * D; e += blockDim.x)
    sQ[e] = __bfloat162float(q[((size_t)s * Hq + g * rep) * D + e]);
  for (int e = tid; e < nk * 16; e += blockDim.x) {
    const int r = e >> 4, cc = e & 15;
    const int key = k0 + r;
    const uint4* ks;
    const uint4* vs;
    if (is_vis) {
      ks = reinterpret_cast<const uint4*>(kbase + (size_t)key * D);
      vs = reinterpret_cast<const uint4*>(vbase + (size_t)key * D);
    } else if (key < nt) {
      ks = reinterpret_cast<const uint4*>(tk + (((size_t)s * Hkv + g) * nt + key) * D);
      vs = reinterpret_cast<const uint4*>(tv + (((size_t)s * Hkv + g) * nt + key) * D);
    } else {
      ks = reinterpret_cast<const uint4*>(ak + (((size_t)s * Hkv + g) * acap + (key - nt)) * D);
      vs = reinterpret_cast<const uint4*>(av + (((size_t)s * Hkv + g) * acap + (key - nt)) * D);
    }
    *reinterpret_cast<uint4*>(sK + r * ROWB + cc * 16) = __ldg(ks + cc);
    *reinterpret_cast<uint4*>(sV + r * ROWB + cc * 16) = __ldg(vs + cc);
  }
  __syncthreads();

  // ---- scores: thread t <-> key t, all Q heads of the group
  const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
  float sc[MAXREP];
#pragma unroll
  for (int r = 0; r < MAXREP; ++r) sc[r] = 0.f;
  if (tid < nk) {
    for (int cc = 0; cc < 16; ++cc) {
      const uint4 u = *reinterpret_cast<const uint4*>(sK + tid * ROWB + cc * 16);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
      float kf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h2[i]);
        kf[2 * i] = f.x;
        kf[2 * i + 1] = f.y;
      }
#pragma unroll
      for (int r = 0; r < MAXREP; ++r) {
        if (r < rep) {
          const float4 qa = *reinterpret_cast<const float4*>(sQ + r * D + cc * 8);
          const float4 qb = *reinterpret_cast<const float4*>(sQ + r * D + cc * 8 + 4);
          sc[r] += qa.x * kf[0] + qa.y * kf[1] + qa.z * kf[2] + qa.w * kf[3] + qb.x * kf[4] + qb.y * kf[5] +
                   qb.z * kf[6] + qb.w * kf[7];
        }
      }
    }
  }
  // ---- per-head chunk max and exp (exclusion: lazy heads get no vision keys)
  float mx[MAXREP];
#pragma unroll
  for (int r = 0; r < MAXREP; ++r) {
    float x = -INFINITY;
    if (r < rep && tid < nk && (!is_vis || s_flag[r])) x = sc[r] * sl2;
    sc[r] = x;
    float m = x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    mx[r] = m;
  }
  if (lane == 0)
    for (int r = 0; r < rep; ++r) sRed[warp * MAXREP + r] = mx[r];
  __syncthreads();
  for (int r = 0; r < rep; ++r) {
    float m = -INFINITY;
    for (int w = 0; w < 8; ++w) m = fmaxf(m, sRed[w * MAXREP + r]);
    mx[r] = m;
  }
  __syncthreads();
  float ls[MAXREP];
  for (int r = 0; r < rep; ++r) {
    const float p = (mx[r] == -INFINITY || sc[r] == -INFINITY) ? 0.f : fast_exp2(sc[r] - mx[r]);
    sP[r * CHUNK + tid] = p;
    ls[r] = warp_sum(p);
  }
  if (lane == 0)
    for (int r = 0; r < rep; ++r) sRed[warp * MAXREP + r] = ls[r];
  __syncthreads();
  if (tid < rep) {
    float l = 0.f;
    for (int w = 0; w < 8; ++w) l += sRed[w * MAXREP + tid];
    ml[(size_t)tid * n_chunks * 2 + 0] = mx[tid];
    ml[(size_t)tid * n_chunks * 2 + 1] = l;
  }
  __syncthreads();

  // ---- acc[r][col] = sum_t p[r][t] V[t][col]; thread = (column pair, key quarter)
  const int cp = tid & 63, kq = tid >> 6;
  float a0[MAXREP], a1[MAXREP];
#pragma unroll
  for (int r = 0; r < MAXREP; ++r) a0[r] = a1[r] = 0.f;
  for (int t = kq * 64; t < min(nk, kq * 64 + 64); ++t) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sV + t * ROWB + cp * 4));
#pragma unroll
    for (int r = 0; r < MAXREP; ++r) {
      if (r < rep) {
        const float p = sP[r * CHUNK + t];
        a0[r] = fmaf(p, v.x, a0[r]);
        a1[r] = fmaf(p, v.y, a1[r]);
      }
    }
  }
  float* red = reinterpret_cast<float*>(sK);  // reuse: [4][rep][D]
  for (int r = 0; r < rep; ++r) {
    red[(kq * rep + r) * D + 2 * cp] = a0[r];
    red[(kq * rep + r) * D + 2 * cp + 1] = a1[r];
  }
  __syncthreads();
  for (int e = tid; e < rep * D; e += blockDim.x) {
    const int r = e / D, col = e % D;
    const float v = red[(0 * rep + r) * D + col] + red[(1 * rep + r) * D + col] + red[(2 * rep + r) * D + col] +
                    red[(3 * rep + r) * D + col];
    acc_out[(size_t)r * n_chunks * D + col] = v;
  }
}

__global__ void decode_combine_kernel(const float* __restrict__ part_ml, const float* __restrict__ part_acc,
                                      int n_chunks, float* __restrict__ out, int* __restrict__ degenerate) {
  const int h = blockIdx.x, s = blockIdx.y, Hq = gridDim.x;
  const size_t base = (size_t)s * Hq + h;
  const float* ml = part_ml + base * n_chunks * 2;
  const float* acc = part_acc + base * n_chunks * D;
  float M = -INFINITY;
  for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, ml[2 * c]);
  float L = 0.f, o = 0.f;
  const int col = threadIdx.x;
  for (int c = 0; c < n_chunks; ++c) {
    const float m = ml[2 * c];
    if (m == -INFINITY) continue;
    const float w = fast_exp2(m - M);
    L += w * ml[2 * c + 1];
    o += w * acc[(size_t)c * D + col];
  }
  if (L > 0.f) {
    out[base * D + col] = o / L;
  } else {
    out[base * D + col] = 0.f;
    if (col == 0) atomicExch(degenerate, 1);
  }
}

}  // namespace dec
}  // namespace omni

using namespace omni;

static int dec_chunks(int vcap, int n_text, int n_answer, int* vis_chunks) {
  *vis_chunks = (vcap + dec::CHUNK - 1) / dec::CHUNK;
  return *vis_chunks + (n_text + n_answer + dec::CHUNK - 1) / dec::CHUNK;
}

extern "C" size_t omni_decode_workspace(int batch, int n_q_heads, int vcap, int n_text, int acap, int head_dim) {
  int vc;
  const int nc = dec_chunks(vcap, n_text, acap, &vc);
  return sizeof(float) * (size_t)batch * n_q_heads * nc * (head_dim + 2) + 16;
}

extern "C" int omni_decode_step(const void* q, const void* vision_k, const void* vision_v, const int32_t* vision_len,
                                const void* text_k, const void* text_v, int n_text, const void* answer_k,
                                const void* answer_v, int n_answer, const double* k_lazy, const double* k_act,
                                int batch, int n_q_heads, int n_kv_heads, int head_dim, int vcap, int acap, double tau,
                                int preserve_first_head, const uint8_t* flags_override, uint8_t* flags, float* out,
                                void* workspace, void* stream) {
  OMNI_CHECK(head_dim == dec::D, OMNI_E_SHAPE, "decode kernel requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(n_q_heads / n_kv_heads <= dec::MAXREP, OMNI_E_SHAPE, "at most 16 Q heads per KV group");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  OMNI_CHECK(n_answer >= 0 && n_answer <= acap && n_text >= 0, OMNI_E_SHAPE, "answer segment overflow");
  OMNI_CHECK(batch >= 1, OMNI_E_SHAPE, "empty batch");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int vc;
  const int nc = dec_chunks(vcap, n_text, n_answer, &vc);
  const int ncap = dec_chunks(vcap, n_text, acap, &vc);
  (void)ncap;
  float* part_ml = static_cast<float*>(workspace);
  float* part_acc = part_ml + (size_t)batch * n_q_heads * nc * 2;
  int* degenerate = reinterpret_cast<int*>(part_acc + (size_t)batch * n_q_heads * nc * head_dim);
  OMNI_CUDA_TRY(cudaMemsetAsync(degenerate, 0, sizeof(int), st));
  const size_t shm = 2 * dec::CHUNK * dec::ROWB + sizeof(float) * (dec::MAXREP * dec::D + dec::MAXREP * dec::CHUNK +
                                                                    8 * dec::MAXREP);
  static bool attr = false;
  if (!attr) {
    OMNI_CUDA_TRY(cudaFuncSetAttribute(dec::decode_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)shm));
    attr = true;
  }
  dim3 grid(nc, n_kv_heads, batch);
  dec::decode_partial_kernel<<<grid, 256, shm, st>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(vision_k),
      static_cast<const __nv_bfloat16*>(vision_v), vision_len, static_cast<const __nv_bfloat16*>(text_k),
      static_cast<const __nv_bfloat16*>(text_v), n_text, static_cast<const __nv_bfloat16*>(answer_k),
      static_cast<const __nv_bfloat16*>(answer_v), n_answer, k_lazy, k_act, n_q_heads, n_kv_heads, vcap, acap, tau,
      preserve_first_head, flags_override, flags, vc, part_ml, part_acc, nc);
  dec::decode_combine_kernel<<<dim3(n_q_heads, batch), dec::D, 0, st>>>(part_ml, part_acc, nc, out, degenerate);
  int st_code = omni_launch_check();
  if (st_code) return st_code;
  if (n_text + n_answer == 0) {
    // Only reachable degenerate case (decode.py:152-153): read the flag back.
    int h = 0;
    OMNI_CUDA_TRY(cudaMemcpyAsync(&h, degenerate, sizeof(int), cudaMemcpyDeviceToHost, st));
    OMNI_CUDA_TRY(cudaStreamSynchronize(st));
    OMNI_CHECK(h == 0, OMNI_E_DEGENERATE_CONTEXT, "lazy head with no text and no answer KV");
  }
  return OMNI_OK;
}
