// K1 (probe keys + pooled K), K2 (query classification + pooled Q + lazy-row
// zeroing), active-row compaction and K6 row gather.
//
// All four are HBM-bound streaming passes: K1 and K2 read K / Q exactly once
// with 16-byte (bf16 x 8) or 32-byte (f32 x 8) vector loads, accumulate in
// float64 (decision-critical, SURVEY §7 hard parts) and write only tiny
// outputs. One CTA per (probe block, head): grid = nb x H, which at 64K tokens
// is 256 x 28 = 7168 CTAs (48 waves of 148 SMs).
#include "common.cuh"

namespace omni {

template <typename T>
struct Vec8;  // 8 consecutive elements loaded with one (or two) vector loads
template <>
struct Vec8<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, double* out) {
    uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = static_cast<double>(__bfloat162float(h[i]));
  }
};
template <>
struct Vec8<float> {
  __device__ static void load(const float* p, double* out) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
    out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
  }
};

// Raw 8-element vector kept in registers until converted (keeps many rows in
// flight per thread without paying 16 f64 registers per row).
template <typename T>
struct Raw8;
template <>
struct Raw8<__nv_bfloat16> {
  uint4 u;
  __device__ void load(const __nv_bfloat16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ void zero() { u = make_uint4(0, 0, 0, 0); }
  __device__ double at(int i) const {
    return static_cast<double>(__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(&u)[i]));
  }
};
template <>
struct Raw8<float> {
  float4 a, b;
  __device__ void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ double at(int i) const {
    return static_cast<double>(i < 4 ? reinterpret_cast<const float*>(&a)[i] : reinterpret_cast<const float*>(&b)[i - 4]);
  }
};

// ------------------------------------------------------------------------ K1
// CTA (block J, kv head g): column sums of K[g, rows of J] (all rows) and of
// the rows < n_vision, in f64. 256 threads = (256 / (d/8)) row lanes x (d/8)
// column groups of 8.
template <typename T>
__global__ void __launch_bounds__(256) kv_probe_kernel(const T* __restrict__ K, int N, int d, int n_vision, int block,
                                                       double* __restrict__ pooled_k, double* __restrict__ vis_part) {
  extern __shared__ double sh[];  // [2][row_lanes][d]
  const int J = blockIdx.x, g = blockIdx.y, nb = gridDim.x;
  const int cg = d / 8, lanes = blockDim.x / cg;
  const int tc = threadIdx.x % cg, tr = threadIdx.x / cg;
  const int r0 = J * block, r1 = min(N, r0 + block);
  double all[8] = {0, 0, 0, 0, 0, 0, 0, 0}, vis[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const T* base = K + (size_t)g * N * d + tc * 8;
  for (int r = r0 + tr; r < r1; r += lanes) {
    double x[8];
    Vec8<T>::load(base + (size_t)r * d, x);
    const bool v = r < n_vision;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      all[i] += x[i];
      if (v) vis[i] += x[i];
    }
  }
  double* s_all = sh;
  double* s_vis = sh + lanes * d;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    s_all[tr * d + tc * 8 + i] = all[i];
    s_vis[tr * d + tc * 8 + i] = vis[i];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double a = 0.0, v = 0.0;
    for (int l = 0; l < lanes; ++l) {
      a += s_all[l * d + c];
      v += s_vis[l * d + c];
    }
    pooled_k[((size_t)g * nb + J) * d + c] = a / static_cast<double>(r1 - r0);
    vis_part[((size_t)g * nb + J) * d + c] = v;
  }
}

// k_act[g] = (sum over blocks of vision partial sums) / n_vision; k_lazy = K[sink].
template <typename T>
__global__ void probe_finish_kernel(const T* __restrict__ K, int N, int d, int nb, int n_vision, int sink,
                                    const double* __restrict__ vis_part, double* __restrict__ k_lazy,
                                    double* __restrict__ k_act) {
  // CTA (32-column slice, group g), 1024 threads = 32 columns x 32 block phases;
  // partial sums over blocks J = phase (mod 32), combined in a fixed order.
  __shared__ double part[32][33];
  const int g = blockIdx.y;
  const int col = threadIdx.x & 31, ph = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + col;
  double s = 0.0;
  if (c < d)
    for (int J = ph; J < nb; J += 32) s += vis_part[((size_t)g * nb + J) * d + c];
  part[ph][col] = s;
  __syncthreads();
  if (ph == 0 && c < d) {
    double t = 0.0;
    for (int k = 0; k < 32; ++k) t += part[k][col];
    k_act[(size_t)g * d + c] = t / static_cast<double>(n_vision);
    k_lazy[(size_t)g * d + c] = to_f64(K[((size_t)g * N + sink) * d + c]);
  }
}

// ------------------------------------------------------------------------ K2
// CTA (block J, q head h), 8 warps. A row is read by LPR = d/8 lanes with one
// 16-byte (bf16) vector load each (a coalesced 256-byte row segment); every
// lane keeps U = 4 rows in flight so the pass streams at HBM rate. Two f64 dot
// products per row (lazy / active probe keys) are butterfly-reduced over the
// LPR lanes, after which lane k of the row group finalises row k: the
// reference's max-subtracted two-way softmax (one of the two exponentials is
// exp(0) = 1) and the strict p_act > tau test (query_select.py:63-68). Column
// sums for the pooled query stay in registers until the end.
constexpr int QS_U = 4;

template <typename T>
__global__ void __launch_bounds__(256) q_score_kernel(const T* __restrict__ Q, int N, int d, int rep, int n_vision,
                                                      double tau, int preserve, int block,
                                                      const double* __restrict__ k_lazy,
                                                      const double* __restrict__ k_act, uint8_t* __restrict__ active,
                                                      double* __restrict__ p_act, double* __restrict__ pooled_q,
                                                      int32_t* __restrict__ block_active,
                                                      __nv_bfloat16* __restrict__ o_zero) {
  __shared__ double s_pool[2048];  // [row slot][column]: slots * d == 2048 for every d
  __shared__ int s_cnt[8];
  const int J = blockIdx.x, h = blockIdx.y, nb = gridDim.x;
  const int g = h / rep;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lpr = d / 8;                 // lanes per row
  const int rpw = 32 / lpr;              // rows per warp step
  const int sub = lane / lpr, cl = lane % lpr;
  const int slots = 8 * rpw;             // row slots per CTA
  const int slot = warp * rpw + sub;
  const int r0 = J * block, r1 = min(N, r0 + block);
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  double kl[8], ka[8], pool[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    kl[i] = k_lazy[(size_t)g * d + cl * 8 + i];
    ka[i] = k_act[(size_t)g * d + cl * 8 + i];
    pool[i] = 0.0;
  }
  int cnt = 0;
  const T* qh = Q + (size_t)h * N * d + cl * 8;
  for (int rb = r0; rb < r1; rb += slots * QS_U) {
    Raw8<T> x[QS_U];
#pragma unroll
    for (int u = 0; u < QS_U; ++u) {
      const int r = rb + u * slots + slot;
      if (r < r1) x[u].load(qh + (size_t)r * d); else x[u].zero();
    }
    double dl[QS_U], da[QS_U];
#pragma unroll
    for (int u = 0; u < QS_U; ++u) {
      dl[u] = 0.0;
      da[u] = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double v = x[u].at(i);
        pool[i] += v;
        dl[u] = fma(v, kl[i], dl[u]);
        da[u] = fma(v, ka[i], da[u]);
      }
    }
    for (int o = lpr >> 1; o > 0; o >>= 1) {
#pragma unroll
      for (int u = 0; u < QS_U; ++u) {
        dl[u] += __shfl_xor_sync(0xffffffffu, dl[u], o);
        da[u] += __shfl_xor_sync(0xffffffffu, da[u], o);
      }
    }
    // lane cl == u of the row group finalises row u of this step
    int my_act = 1;
    const int ur = cl < QS_U ? cl : 0;
    const int r_mine = rb + ur * slots + slot;
    if (cl < QS_U && r_mine < r1) {
      double l0 = dl[0], l1 = da[0];
#pragma unroll
      for (int u = 1; u < QS_U; ++u)
        if (u == cl) { l0 = dl[u]; l1 = da[u]; }
      if (r_mine < n_vision) {
        l0 *= scale;
        l1 *= scale;
        const double p = (l1 >= l0) ? 1.0 / (exp(l0 - l1) + 1.0) : (exp(l1 - l0) / (1.0 + exp(l1 - l0)));
        my_act = (p > tau) ? 1 : 0;
        if (p_act) p_act[(size_t)h * n_vision + r_mine] = p;
      }
      if (preserve && h == 0) my_act = 1;
      active[(size_t)h * N + r_mine] = static_cast<uint8_t>(my_act);
      cnt += my_act;
    }
    if (o_zero) {
#pragma unroll
      for (int u = 0; u < QS_U; ++u) {
        const int src_lane = sub * lpr + u;
        const int act_u = __shfl_sync(0xffffffffu, my_act, src_lane);
        const int r = rb + u * slots + slot;
        if (r < r1 && !act_u)
          *reinterpret_cast<uint4*>(o_zero + ((size_t)h * N + r) * d + cl * 8) = make_uint4(0, 0, 0, 0);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) s_pool[slot * d + cl * 8 + i] = pool[i];
  cnt = warp_sum(cnt);
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < slots; ++w) s += s_pool[w * d + c];
    pooled_q[((size_t)h * nb + J) * d + c] = s / static_cast<double>(r1 - r0);
  }
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += s_cnt[w];
    block_active[(size_t)h * nb + J] = t;
  }
}

// ------------------------------------------------------------- compaction
// CTA (block J, head h): offset = active rows in earlier blocks, then a
// block-wide exclusive scan of this block's flags.
__global__ void __launch_bounds__(256) compact_rows_kernel(const uint8_t* __restrict__ active,
                                                           const int32_t* __restrict__ block_active, int N, int block,
                                                           int32_t* __restrict__ rows, int32_t* __restrict__ counts) {
  __shared__ int s_warp[8];
  __shared__ int s_base;
  const int J = blockIdx.x, h = blockIdx.y, nb = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int part = 0;
  for (int i = threadIdx.x; i < J; i += blockDim.x) part += block_active[(size_t)h * nb + i];
  part = warp_sum(part);
  if (lane == 0) s_warp[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += s_warp[w];
    s_base = t;
  }
  __syncthreads();
  int base = s_base;
  const int r0 = J * block, r1 = min(N, r0 + block);
  for (int c0 = r0; c0 < r1; c0 += blockDim.x) {
    const int r = c0 + threadIdx.x;
    const int f = (r < r1) ? active[(size_t)h * N + r] : 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    const int within = __popc(m & ((1u << lane) - 1u));
    __syncthreads();
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += s_warp[w];
    if (f) rows[(size_t)h * N + off + within] = r;
    int tot = 0;
    for (int w = 0; w < 8; ++w) tot += s_warp[w];
    base += tot;
  }
  if (J == nb - 1 && threadIdx.x == 0) counts[h] = base;
}

// ------------------------------------------------------------------ gather
// One warp per destination row: 16-byte lane copies of a bf16/f32 row.
__global__ void __launch_bounds__(256) gather_rows_kernel(const uint8_t* __restrict__ src, int src_rows,
                                                          int row_bytes, const int32_t* __restrict__ idx,
                                                          int idx_stride, const int32_t* __restrict__ counts,
                                                          int count_const, uint8_t* __restrict__ dst, int dst_rows,
                                                          int pad_rows) {
  const int g = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int cnt = counts ? counts[g] : count_const;
  const int lim = min(dst_rows, ((cnt + pad_rows - 1) / pad_rows) * pad_rows);
  if (r >= lim) return;
  uint8_t* o = dst + ((size_t)g * dst_rows + r) * row_bytes;
  if (r < cnt) {
    const int s = __ldg(idx + (size_t)g * idx_stride + r);
    const uint8_t* i = src + ((size_t)g * src_rows + s) * row_bytes;
    for (int c = lane * 16; c < row_bytes; c += 512)
      *reinterpret_cast<uint4*>(o + c) = __ldg(reinterpret_cast<const uint4*>(i + c));
  } else {
    for (int c = lane * 16; c < row_bytes; c += 512) *reinterpret_cast<uint4*>(o + c) = make_uint4(0, 0, 0, 0);
  }
}

}  // namespace omni

using namespace omni;

static inline int nblocks(int n, int b) { return (n + b - 1) / b; }

extern "C" size_t omni_kv_probe_workspace(int n_kv_heads, int seq_len, int head_dim, int block_size) {
  if (block_size < 1) return 0;
  return sizeof(double) * (size_t)n_kv_heads * nblocks(seq_len, block_size) * head_dim;
}

extern "C" int omni_kv_probe(const void* K, int dtype, int n_kv_heads, int seq_len, int head_dim, int n_vision,
                             int sink_index, int block_size, double* k_lazy, double* k_act, double* pooled_k,
                             void* workspace, void* stream) {
  OMNI_CHECK(n_vision >= 1, OMNI_E_LAYOUT, "probe keys need at least one vision token");
  OMNI_CHECK(n_vision <= seq_len, OMNI_E_LAYOUT, "n_vision exceeds seq_len");
  OMNI_CHECK(sink_index >= 0 && sink_index < seq_len, OMNI_E_LAYOUT, "sink_index outside the sequence");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(head_dim % 8 == 0 && head_dim >= 8 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be a multiple of 8 in [8, 256]");
  OMNI_CHECK(n_kv_heads >= 1 && seq_len >= 1, OMNI_E_SHAPE, "empty K");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = nblocks(seq_len, block_size);
  const int lanes = 256 / (head_dim / 8);
  const size_t shm = sizeof(double) * 2 * lanes * head_dim;
  dim3 grid(nb, n_kv_heads);
  double* vis = static_cast<double*>(workspace);
  if (dtype == OMNI_DTYPE_BF16) {
    kv_probe_kernel<__nv_bfloat16><<<grid, 256, shm, s>>>(static_cast<const __nv_bfloat16*>(K), seq_len, head_dim,
                                                            n_vision, block_size, pooled_k, vis);
    probe_finish_kernel<__nv_bfloat16><<<dim3((head_dim + 31) / 32, n_kv_heads), 1024, 0, s>>>(static_cast<const __nv_bfloat16*>(K), seq_len,
                                                                   head_dim, nb, n_vision, sink_index, vis, k_lazy,
                                                                   k_act);
  } else if (dtype == OMNI_DTYPE_F32) {
    kv_probe_kernel<float><<<grid, 256, shm, s>>>(static_cast<const float*>(K), seq_len, head_dim, n_vision,
                                                    block_size, pooled_k, vis);
    probe_finish_kernel<float><<<dim3((head_dim + 31) / 32, n_kv_heads), 1024, 0, s>>>(static_cast<const float*>(K), seq_len, head_dim, nb,
                                                           n_vision, sink_index, vis, k_lazy, k_act);
  } else {
    OMNI_CHECK(false, OMNI_E_PARAM, "unsupported dtype");
  }
  return omni_launch_check();
}

extern "C" int omni_q_score(const void* Q, int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim,
                            int n_vision, double tau, int preserve_first_head, int block_size, const double* k_lazy,
                            const double* k_act, uint8_t* active, double* p_act, double* pooled_q,
                            int32_t* block_active, void* O_zero, void* stream) {
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(n_vision >= 0 && n_vision <= seq_len, OMNI_E_LAYOUT, "n_vision outside the sequence");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim == 32 || head_dim == 64 || head_dim == 128 || head_dim == 256, OMNI_E_SHAPE,
             "head_dim must be 32, 64, 128 or 256");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 grid(nblocks(seq_len, block_size), n_q_heads);
  const int rep = n_q_heads / n_kv_heads;
  __nv_bfloat16* oz = static_cast<__nv_bfloat16*>(O_zero);
  if (dtype == OMNI_DTYPE_BF16)
    q_score_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(Q), seq_len, head_dim, rep,
                                                       n_vision, tau, preserve_first_head, block_size, k_lazy, k_act,
                                                       active, p_act, pooled_q, block_active, oz);
  else if (dtype == OMNI_DTYPE_F32)
    q_score_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(Q), seq_len, head_dim, rep, n_vision, tau,
                                               preserve_first_head, block_size, k_lazy, k_act, active, p_act,
                                               pooled_q, block_active, oz);
  else
    OMNI_CHECK(false, OMNI_E_PARAM, "unsupported dtype");
  return omni_launch_check();
}

extern "C" int omni_compact_rows(const uint8_t* active, const int32_t* block_active, int n_q_heads, int seq_len,
                                 int block_size, int32_t* rows, int32_t* counts, void* stream) {
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  dim3 grid(nblocks(seq_len, block_size), n_q_heads);
  compact_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(active, block_active, seq_len, block_size,
                                                                           rows, counts);
  return omni_launch_check();
}

extern "C" int omni_gather_rows(const void* src, int dtype, int n_groups, int src_rows, int head_dim,
                                const int32_t* idx, int idx_stride, const int32_t* counts, int count_const, void* dst,
                                int dst_rows, int pad_rows, void* stream) {
  OMNI_CHECK(pad_rows >= 1, OMNI_E_PARAM, "pad_rows must be >= 1");
  const int esz = dtype == OMNI_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = head_dim * esz;
  OMNI_CHECK(row_bytes % 16 == 0, OMNI_E_SHAPE, "row bytes must be a multiple of 16");
  dim3 grid(nblocks(dst_rows, 8), n_groups);
  if (grid.x == 0 || n_groups == 0) return OMNI_OK;
  gather_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), src_rows, row_bytes, idx, idx_stride, counts, count_const,
      static_cast<uint8_t*>(dst), dst_rows, pad_rows);
  return omni_launch_check();
}
