// Exact key scores (score_source = "exact"): column mass of the full causal
// attention map per Q head, float64 — replaces accumulated_key_scores over the
// dense oracle maps (kv_select.py:56-73, prefill.py:133-134) without ever
// materialising the N x N map. Two passes over the causal triangle:
//   rows:    m_i = max_{j<=i} s_ij,  l_i = sum_{j<=i} exp(s_ij - m_i)
//   columns: a_j = sum_{i>=j} exp(s_ij - m_i) / l_i
// s_ij = q_i . k_j / sqrt(d) in float64 on CUDA cores (SURVEY §8f "next":
// validation-scale path; the 64K hot path uses the block probe).
#include <float.h>
#include <math.h>

#include "common.cuh"

namespace omni {
namespace exact {

constexpr int T = 32;  // rows / keys per tile

template <typename X>
__device__ __forceinline__ void load_tile(double* dst, const X* src, int rows, int r0, int N, int d) {
  for (int e = threadIdx.x; e < T * d; e += blockDim.x) {
    const int r = e / d, c = e % d;
    dst[r * (d + 1) + c] = (r0 + r < N) ? to_f64(src[(size_t)(r0 + r) * d + c]) : 0.0;
  }
  (void)rows;
}

// CTA = 32 query rows of head h; thread (row = tid/8, part = tid%8) keeps the
// running max / sum of its row over a strided subset of keys, merged at the end.
template <typename X>
__global__ void __launch_bounds__(256) row_pass_kernel(const X* __restrict__ Q, const X* __restrict__ K, int N, int d,
                                                       int rep, double* __restrict__ stats) {
  extern __shared__ double sh[];
  double* sq = sh;                // [T][d+1]
  double* sk = sh + T * (d + 1);  // [T][d+1]
  __shared__ double red_m[T][8], red_l[T][8];
  const int h = blockIdx.y, g = h / rep;
  const int i0 = blockIdx.x * T;
  const X* Qh = Q + (size_t)h * N * d;
  const X* Kg = K + (size_t)g * N * d;
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  load_tile(sq, Qh, T, i0, N, d);
  const int r = threadIdx.x >> 3, part = threadIdx.x & 7;
  const int i = i0 + r;
  double m = -DBL_MAX, l = 0.0;
  for (int j0 = 0; j0 <= min(N - 1, i0 + T - 1); j0 += T) {
    __syncthreads();
    load_tile(sk, Kg, T, j0, N, d);
    __syncthreads();
    for (int jj = part; jj < T; jj += 8) {
      const int j = j0 + jj;
      if (i < N && j <= i) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) s = fma(sq[r * (d + 1) + c], sk[jj * (d + 1) + c], s);
        s *= scale;
        if (s > m) {
          l = l * exp(m - s) + 1.0;
          m = s;
        } else {
          l += exp(s - m);
        }
      }
    }
  }
  red_m[r][part] = m;
  red_l[r][part] = l;
  __syncthreads();
  if (part == 0 && i < N) {
    double M = -DBL_MAX;
    for (int k = 0; k < 8; ++k) M = fmax(M, red_m[r][k]);
    double L = 0.0;
    for (int k = 0; k < 8; ++k)
      if (red_l[r][k] > 0.0) L += red_l[r][k] * exp(red_m[r][k] - M);
    stats[((size_t)h * N + i) * 2 + 0] = M;
    stats[((size_t)h * N + i) * 2 + 1] = L;
  }
}

// CTA = 32 key columns of head h; thread (col = tid/8, part = tid%8) sums the
// probabilities of a strided subset of rows i >= j.
template <typename X>
__global__ void __launch_bounds__(256) col_pass_kernel(const X* __restrict__ Q, const X* __restrict__ K, int N, int d,
                                                       int rep, const double* __restrict__ stats,
                                                       double* __restrict__ mass) {
  extern __shared__ double sh[];
  double* sk = sh;                // [T][d+1] keys of this CTA
  double* sq = sh + T * (d + 1);  // [T][d+1] query tile
  __shared__ double red[T][8];
  const int h = blockIdx.y, g = h / rep;
  const int j0 = blockIdx.x * T;
  const X* Qh = Q + (size_t)h * N * d;
  const X* Kg = K + (size_t)g * N * d;
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  load_tile(sk, Kg, T, j0, N, d);
  const int cidx = threadIdx.x >> 3, part = threadIdx.x & 7;
  const int j = j0 + cidx;
  double a = 0.0;
  for (int i0 = j0; i0 < N; i0 += T) {
    __syncthreads();
    load_tile(sq, Qh, T, i0, N, d);
    __syncthreads();
    for (int ii = part; ii < T; ii += 8) {
      const int i = i0 + ii;
      if (j < N && i < N && j <= i) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) s = fma(sq[ii * (d + 1) + c], sk[cidx * (d + 1) + c], s);
        const double* st = stats + ((size_t)h * N + i) * 2;
        a += exp(s * scale - st[0]) / st[1];
      }
    }
  }
  red[cidx][part] = a;
  __syncthreads();
  if (part == 0 && j < N) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[cidx][k];
    mass[(size_t)h * N + j] = t;
  }
}

}  // namespace exact
}  // namespace omni

using namespace omni;

extern "C" size_t omni_exact_mass_workspace(int n_q_heads, int seq_len) {
  return sizeof(double) * 2 * (size_t)n_q_heads * seq_len;
}

extern "C" int omni_exact_mass(const void* Q, const void* K, int dtype, int n_q_heads, int n_kv_heads, int seq_len,
                               int head_dim, double* mass, void* workspace, void* stream) {
  omni_begin();
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim >= 1 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be in [1, 256]");
  OMNI_CHECK(seq_len >= 1, OMNI_E_SHAPE, "empty sequence");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t shm = sizeof(double) * 2 * exact::T * (head_dim + 1);
  const dim3 grid((seq_len + exact::T - 1) / exact::T, n_q_heads);
  const int rep = n_q_heads / n_kv_heads;
  double* stats = static_cast<double*>(workspace);
  if (dtype == OMNI_DTYPE_BF16) {
    auto q = static_cast<const __nv_bfloat16*>(Q);
    auto k = static_cast<const __nv_bfloat16*>(K);
    OMNI_CUDA_TRY(omni_smem_attr(exact::row_pass_kernel<__nv_bfloat16>, (int)shm));
    OMNI_CUDA_TRY(omni_smem_attr(exact::col_pass_kernel<__nv_bfloat16>, (int)shm));
    exact::row_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats);
    exact::col_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats, mass);
  } else if (dtype == OMNI_DTYPE_F32) {
    auto q = static_cast<const float*>(Q);
    auto k = static_cast<const float*>(K);
    OMNI_CUDA_TRY(omni_smem_attr(exact::row_pass_kernel<float>, (int)shm));
    OMNI_CUDA_TRY(omni_smem_attr(exact::col_pass_kernel<float>, (int)shm));
    exact::row_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats);
    exact::col_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats, mass);
  } else if (dtype == OMNI_DTYPE_F64) {
    auto q = static_cast<const double*>(Q);
    auto k = static_cast<const double*>(K);
    OMNI_CUDA_TRY(omni_smem_attr(exact::row_pass_kernel<double>, (int)shm));
    OMNI_CUDA_TRY(omni_smem_attr(exact::col_pass_kernel<double>, (int)shm));
    exact::row_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats);
    exact::col_pass_kernel<<<grid, 256, shm, s>>>(q, k, seq_len, head_dim, rep, stats, mass);
  } else {
    OMNI_CHECK(false, OMNI_E_PARAM, "unsupported dtype");
  }
  return omni_launch_check();
}
