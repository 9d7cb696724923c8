// K1 (probe keys + pooled K), K2 (query classification + pooled Q + lazy-row
// zeroing), active-row compaction and K6 row gather.
//
// All four are HBM-bound streaming passes that read K / Q exactly once and
// accumulate the decision-critical sums in float64 (SURVEY §7 hard parts).
// The bf16 / d = 128 hot path (K1 kv_probe_stream_kernel, K2
// q_score_stream_kernel) runs one persistent CTA per SM over a 3-stage
// bulk-copy ring of probe blocks; the generic kernels (one CTA per (probe
// block, head)) serve other dtypes, head sizes, the want_prob path and the
// A/B switch OMNI_QSCORE_F64. Measured at 64K tokens (28 / 4 heads, one
// B200, device time in a CUDA graph, profiles/r02_notes.md): K1 0.016 ms
// (with probe_finish; 4.2 TB/s, 0.65 of the measured copy bandwidth), K2
// 0.172 ms (4.05 TB/s, 0.62; the float64 column sums of the pooled queries
// keep it issue-bound) vs 0.028 / 0.194 ms (eager) for the generic kernels.
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

template <>
struct Vec8<double> {
  __device__ static void load(const double* p, double* out) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(p) + i);
      out[2 * i] = v.x;
      out[2 * i + 1] = v.y;
    }
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

template <>
struct Raw8<double> {  // the reference's own precision (drop-in float64 workloads)
  double2 v[4];
  __device__ void load(const double* p) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __ldg(reinterpret_cast<const double2*>(p) + i);
  }
  __device__ void zero() {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = make_double2(0.0, 0.0);
  }
  __device__ double at(int i) const { return (i & 1) ? v[i >> 1].y : v[i >> 1].x; }
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
  // four rows per lane in flight per pass (raw loads first, then the f64 sums)
  for (int rb = r0 + tr; rb < r1; rb += 4 * lanes) {
    Raw8<T> x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rb + u * lanes;
      if (r < r1) x[u].load(base + (size_t)r * d); else x[u].zero();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rb + u * lanes;
      const bool v = r < n_vision;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double xi = x[u].at(i);
        all[i] += xi;
        if (v) vis[i] += xi;
      }
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
  if (c < d) {
    // eight independent loads in flight, added in ascending J (fixed order)
    int J = ph;
    for (; J + 7 * 32 < nb; J += 8 * 32) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = vis_part[((size_t)g * nb + J + 32 * k) * d + c];
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; J < nb; J += 32) s += vis_part[((size_t)g * nb + J) * d + c];
  }
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

// query_select.py:63-68: active iff p_act > tau with p_act the max-subtracted
// two-way softmax of (l0, l1). p is monotone in delta = l1 - l0, so away from
// the boundary the decision is delta > T = ln(tau / (1 - tau)) without the
// float64 exponential; within 1e-9 of T (the computed p can only disagree
// within ~1e-14) and whenever p itself is wanted, the reference's expression
// decides. Both paths use the same rounded l0 - l1, so decisions are
// identical to evaluating the expression for every row.
__device__ __forceinline__ int two_way_active(double l0, double l1, double tau, double T, double* p_out) {
  if (p_out == nullptr && tau > 0.0) {
    const double dlt = (l1 - l0) - T;
    if (fabs(dlt) > 1e-9 * (1.0 + fabs(T))) return dlt > 0.0 ? 1 : 0;
  }
  const double p = (l1 >= l0) ? 1.0 / (exp(l0 - l1) + 1.0) : (exp(l1 - l0) / (1.0 + exp(l1 - l0)));
  if (p_out) *p_out = p;
  return (p > tau) ? 1 : 0;
}

template <typename T>
__global__ void __launch_bounds__(256) q_score_kernel(const T* __restrict__ Q, int N, int d, int rep, int n_vision,
                                                      double tau, double tau_logit, int preserve, int block,
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
        my_act = two_way_active(l0, l1, tau, tau_logit, p_act ? p_act + (size_t)h * n_vision + r_mine : nullptr);
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

// K2 bulk variant (bf16, d = 128, 64 <= block <= 256 rows: the hot path).
// The CTA's whole probe block of Q (block x 256 B, up to 64 KB) is brought into
// shared memory by four cp.async.bulk copies on mbarriers issued by one
// thread; three CTAs per SM keep up to ~192 KB of reads in flight. Rows are
// consumed from shared memory (16 lanes per row, 16 B each) with the float64
// dot products, two-way softmax and lazy-row zeroing of q_score_kernel.
// Measured at 64K (28 heads): 223 us vs 332 us for q_score_kernel; a
// persistent double-buffered variant (one CTA of 16 warps per SM) measured
// 343 us — the float64 instruction stream, not HBM, is the limit.
constexpr int QSB_MAX_ROWS = 256;
constexpr int QSB_CHUNKS = 2;  // bulk-copy pieces per block (2: 0.194 ms vs 4: 0.198, 8: 0.207 at 64K)

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__global__ void __launch_bounds__(256, 3) q_score_bulk_kernel(const __nv_bfloat16* __restrict__ Q, int N, int rep,
                                                               int n_vision, double tau, double tau_logit,
                                                               int preserve, int block,
                                                               const double* __restrict__ k_lazy,
                                                               const double* __restrict__ k_act,
                                                               uint8_t* __restrict__ active, double* __restrict__ p_act,
                                                               double* __restrict__ pooled_q,
                                                               int32_t* __restrict__ block_active,
                                                               __nv_bfloat16* __restrict__ o_zero) {
  constexpr int d = 128;
  extern __shared__ __align__(16) uint8_t qsm[];  // [rows][256 B]
  __shared__ __align__(8) uint64_t bars[QSB_CHUNKS];
  __shared__ double s_pool[8][d];
  __shared__ int s_cnt[8];
  const int J = blockIdx.x, h = blockIdx.y, nb = gridDim.x;
  const int g = h / rep;
  const int r0 = J * block, nr = min(N, r0 + block) - r0;
  const int rpc = (nr + QSB_CHUNKS - 1) / QSB_CHUNKS;  // rows per chunk
  const uint32_t sq = smem_u32(qsm);
  if (threadIdx.x == 0) {
    for (int c = 0; c < QSB_CHUNKS; ++c) mbar_init(smem_u32(&bars[c]), 1);
    fence_mbar_init();
    const uint8_t* src = reinterpret_cast<const uint8_t*>(Q + ((size_t)h * N + r0) * d);
    for (int c = 0; c < QSB_CHUNKS; ++c) {
      const int lo = c * rpc, hi = min(nr, lo + rpc);
      if (hi <= lo) continue;
      const uint32_t bytes = (uint32_t)(hi - lo) * (d * 2);
      mbar_expect_tx(smem_u32(&bars[c]), bytes);
      bulk_g2s(sq + lo * (d * 2), src + (size_t)lo * (d * 2), bytes, smem_u32(&bars[c]));
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 4, cl = lane & 15;
  double kl[8], ka[8], pool[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    kl[i] = k_lazy[(size_t)g * d + cl * 8 + i];
    ka[i] = k_act[(size_t)g * d + cl * 8 + i];
    pool[i] = 0.0;
  }
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  __syncthreads();  // barrier initialisation visible before anyone waits
  // Each half-warp takes QSB_U consecutive rows per step (independent f64
  // chains), then a reduce-scatter over its 16 lanes (xor 8, 4, then a
  // butterfly over xor 2, 1): 5 shuffles per 4 rows and value instead of 16,
  // and four lanes finalise the four rows in parallel.
  constexpr int QSB_U = 4;
  const int b3 = (cl >> 3) & 1, b2 = (cl >> 2) & 1;
  const int my_u = b3 * 2 + b2;  // row of this lane after the reduce-scatter
  int cnt = 0, waited = -1;
  for (int base = warp * 2 * QSB_U; base < nr; base += 8 * 2 * QSB_U) {
    const int rb = base + sub * QSB_U;  // this half-warp's first row
    const int last = min(nr, base + 2 * QSB_U) - 1;
    const int c = last / rpc;
    for (int cc = waited + 1; cc <= c; ++cc) mbar_wait(smem_u32(&bars[cc]), 0);
    waited = max(waited, c);
    double dl[QSB_U], da[QSB_U];
#pragma unroll
    for (int u = 0; u < QSB_U; ++u) {
      dl[u] = 0.0;
      da[u] = 0.0;
      if (rb + u < nr) {
        const uint4 q = *reinterpret_cast<const uint4*>(qsm + (size_t)(rb + u) * (d * 2) + cl * 16);
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double v = static_cast<double>(__bfloat162float(hv[i]));
          pool[i] += v;
          dl[u] = fma(v, kl[i], dl[u]);
          da[u] = fma(v, ka[i], da[u]);
        }
      }
    }
    auto rs_step = [&](double* v, int n, int bit, int mask) {
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const double lo = v[k], hi = v[k + n];
        const double send = bit ? lo : hi, keep = bit ? hi : lo;
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
      }
    };
    rs_step(dl, 2, b3, 8); rs_step(da, 2, b3, 8);
    rs_step(dl, 1, b2, 4); rs_step(da, 1, b2, 4);
    double sl = dl[0] + __shfl_xor_sync(0xffffffffu, dl[0], 2);
    double sa = da[0] + __shfl_xor_sync(0xffffffffu, da[0], 2);
    sl += __shfl_xor_sync(0xffffffffu, sl, 1);
    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
    const int rr = rb + my_u, r = r0 + rr;
    int act = 1;
    const bool fin = (cl & 3) == 0 && rr < nr;
    if (fin) {
      if (r < n_vision) {
        const double l0 = sl * scale, l1 = sa * scale;
        act = two_way_active(l0, l1, tau, tau_logit, p_act ? p_act + (size_t)h * n_vision + r : nullptr);
      }
      if (preserve && h == 0) act = 1;
      active[(size_t)h * N + r] = static_cast<uint8_t>(act);
      cnt += act;
    }
    // lazy rows of this half-warp -> zero output rows (16 B per lane per row)
    const unsigned lazy = __ballot_sync(0xffffffffu, fin && !act);
    if (o_zero) {
#pragma unroll
      for (int u = 0; u < QSB_U; ++u) {
        const int src_lane = sub * 16 + ((u >> 1) & 1) * 8 + (u & 1) * 4;
        if ((lazy >> src_lane) & 1u)
          *reinterpret_cast<uint4*>(o_zero + ((size_t)h * N + r0 + rb + u) * d + cl * 8) = make_uint4(0, 0, 0, 0);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) pool[i] += __shfl_xor_sync(0xffffffffu, pool[i], 16);
  if (sub == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) s_pool[warp][cl * 8 + i] = pool[i];
  }
  cnt = warp_sum(cnt);
  if (lane == 0) s_cnt[warp] = cnt;
  __syncthreads();
  if (threadIdx.x < d) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += s_pool[w][threadIdx.x];
    pooled_q[((size_t)h * nb + J) * d + threadIdx.x] = t / static_cast<double>(nr);
  }
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += s_cnt[w];
    block_active[(size_t)h * nb + J] = t;
  }
}

// ------------------------------------------------- K1 / K2 persistent streams
// The hot-path instances (bf16, d = 128, probe blocks of <= 256 rows): one
// CTA per SM walks the (head, block) items c, c + G, c + 2G, ... and streams
// each item's rows (<= 64 KB) into a 3-stage shared-memory ring with one
// cp.async.bulk per item, so two items' reads are always in flight while the
// third is consumed. The per-item column sums (pooled Q / K, float64) are
// reduced through a double-buffered shared-memory slab in a fixed order.
constexpr int SP_STAGES = 3;
constexpr uint32_t SP_STAGE = 256 * 256;  // one probe block of bf16 rows, d = 128

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }


// item -> (head, block) and its row span
struct SpItem {
  int h, J, r0, nr;
};
__device__ __forceinline__ SpItem sp_item(int i, int nb, int block, int N) {
  SpItem it;
  it.h = i / nb;
  it.J = i - it.h * nb;
  it.r0 = it.J * block;
  it.nr = min(N, it.r0 + block) - it.r0;
  return it;
}
__device__ __forceinline__ void sp_issue(const __nv_bfloat16* src, int nb, int block, int N, int i, uint32_t dst,
                                         uint32_t bar) {
  const SpItem it = sp_item(i, nb, block, N);
  const uint32_t bytes = (uint32_t)it.nr * 256u;
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, reinterpret_cast<const uint8_t*>(src + ((size_t)it.h * N + it.r0) * 128), bytes, bar);
}

// K2: the decision needs only the sign of l1 - l0 - T with l1 - l0 = q . kd,
// kd = (k_act - k_lazy) / sqrt(d): one fp32 dot product (FFMA2 pairs) per row
// instead of two float64 ones, with a rigorous error bound. kd is rounded to
// fp32 once (relative error u = 2^-24 per component), q is exact in fp32, and
// every partial sum is a chain of at most 8 roundings (the pair FMA, the pair
// add, 5 cross-lane adds), so
//   |d32 - q . kd| <= 9 u sum_i |q_i kd_i| <= 9 u ||q||_2 ||kd||_2
// (Cauchy-Schwarz; ||q||^2 is accumulated alongside in fp32 and the bound
// taken as 13 u and inflated by 1 %). Rows with |d32 - T| beyond that bound
// plus q_score_bulk_kernel's own 1e-9 band get the decision
// q_score_bulk_kernel's float64 path takes (its l1 - l0 differs from q . kd
// by far less than the band); the rest (a few rows per million) are
// re-evaluated from shared memory with q_score_bulk_kernel's float64
// arithmetic, operation for operation.
//
// Layout: lane L owns columns 4L..4L+3 (one 8-byte load per row: a warp reads
// a whole 256-byte row, conflict-free) and a warp owns 16 rows of the item.
// The 16 per-row partials are reduce-scattered over the lanes (xor 16, 8, 4,
// 2, then a butterfly on xor 1) without selects: register slot k of lane L
// holds row k ^ m(L), m(L) = the lane bits 4..1 reversed into 8/4/2/1, so at
// every level each lane keeps its low slots and sends its high ones, and
// lanes 2j, 2j + 1 end with row m(2j). Pooled Q column sums (float64) need no
// cross-lane work: each lane owns its columns.
#ifndef OMNI_QP_WARPS
#define OMNI_QP_WARPS 16
#endif
constexpr int QP_WARPS = OMNI_QP_WARPS;
constexpr int QP_ROWS = 256 / QP_WARPS;  // rows per warp and item
constexpr int QP_LEVELS = QP_ROWS == 16 ? 4 : QP_ROWS == 8 ? 3 : 2;
constexpr int QP_SHARE = 32 / QP_ROWS;   // lanes that end with the same row
constexpr int QP_SLABS = QP_WARPS <= 16 ? 2 : 1;  // double-buffered column-sum slab when it fits
constexpr uint32_t QP_SMEM = SP_STAGES * SP_STAGE + QP_SLABS * QP_WARPS * 128 * 8;

// slot k of lane L holds row k ^ m(L): lane bits 4, 3, ... reversed
__device__ __forceinline__ int sp_row_mask(int lane) {
  int m = 0;
#pragma unroll
  for (int l = 0; l < QP_LEVELS; ++l) m |= ((lane >> (4 - l)) & 1) << (QP_LEVELS - 1 - l);
  return m;
}

__global__ void __launch_bounds__(QP_WARPS * 32, 1) q_score_stream_kernel(
    const __nv_bfloat16* __restrict__ Q, int N, int nb, int n_items, int rep, int n_vision, double tau,
    double tau_logit, int preserve, int block, const double* __restrict__ k_lazy, const double* __restrict__ k_act,
    uint8_t* __restrict__ active, double* __restrict__ pooled_q, int32_t* __restrict__ block_active,
    __nv_bfloat16* __restrict__ o_zero) {
  constexpr int d = 128;
  extern __shared__ __align__(1024) uint8_t sp_smem[];
  static_assert(QP_SLABS == 2, "the mbarrier hand-off needs the double-buffered slab");
  __shared__ __align__(8) uint64_t bars[SP_STAGES];
  // done[sl]: every thread has consumed its rows of the item and written its
  // slab column sums (one arrival per thread, so each thread's own accesses
  // are released by its own arrive); sfree[sl]: the 128 reducer threads have
  // read the slab. No CTA-wide barrier per item: warps drift across items,
  // bounded by the ring and the slab double buffer.
  __shared__ __align__(8) uint64_t done[2], sfree[2];
  __shared__ int s_cnt[QP_SLABS][QP_WARPS];
  double* s_pool = reinterpret_cast<double*>(sp_smem + SP_STAGES * SP_STAGE);  // [slabs][warps][128]
  const uint32_t ring = smem_u32(sp_smem);
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_STAGES; ++s) mbar_init(smem_u32(&bars[s]), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&done[b]), QP_WARPS * 32);
      mbar_init(smem_u32(&sfree[b]), 128);
    }
    fence_mbar_init();
    for (int k = 0; k < SP_STAGES; ++k) {
      const int i = blockIdx.x + k * G;
      if (i < n_items) sp_issue(Q, nb, block, N, i, ring + k * SP_STAGE, smem_u32(&bars[k]));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = sp_row_mask(lane);
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  const double band = 1e-9 * (1.0 + fabs(tau_logit));
  uint64_t kd01 = 0, kd23 = 0;
  double kbound = 0.0;
  float kboundf = 0.f;
  int cur_g = -1;
  for (int k = 0;; ++k) {
    const int i = blockIdx.x + k * G;
    if (i >= n_items) break;
    const int s = k % SP_STAGES;
    const SpItem it = sp_item(i, nb, block, N);
    const int h = it.h, g = h / rep, r0 = it.r0, nr = it.nr;
    if (g != cur_g) {  // kd of this lane's 4 columns; ||kd||_2 over the warp
      cur_g = g;
      double v[4], kdn2 = 0.0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const size_t o = (size_t)g * d + 4 * lane + e;
        v[e] = (__ldg(k_act + o) - __ldg(k_lazy + o)) * scale;
        kdn2 = fma(v[e], v[e], kdn2);
      }
      kd01 = f32x2(static_cast<float>(v[0]), static_cast<float>(v[1]));
      kd23 = f32x2(static_cast<float>(v[2]), static_cast<float>(v[3]));
      kdn2 = warp_sum(kdn2);
      kbound = 13.0 * 0x1p-24 * sqrt(kdn2) * 1.02;  // 13 u ||kd||, inflated for fp32 ||q||^2 and sqrtf
      kboundf = static_cast<float>(kbound) * 1.0001f;
    }
    const uint8_t* qsm = sp_smem + s * SP_STAGE;
    double pool[4] = {0.0, 0.0, 0.0, 0.0};
    int cnt = 0;
    mbar_wait(smem_u32(&bars[s]), (k / SP_STAGES) & 1);
    const int rbase = warp * QP_ROWS;
    if (rbase < nr) {
      float dv[QP_ROWS], nv[QP_ROWS];
#pragma unroll
      for (int kk = 0; kk < QP_ROWS; ++kk) {
        const int rr = rbase + (kk ^ m);
        uint2 w = make_uint2(0u, 0u);
        if (rr < nr) w = *reinterpret_cast<const uint2*>(qsm + (size_t)rr * (d * 2) + lane * 8);
        const float a0 = bf_lo(w.x), a1 = bf_hi(w.x), a2 = bf_lo(w.y), a3 = bf_hi(w.y);
        const uint64_t x01 = f32x2(a0, a1), x23 = f32x2(a2, a3);
        const uint64_t acc = ffma2(x23, kd23, ffma2(x01, kd01, f32x2(0.f, 0.f)));
        const uint64_t nrm = ffma2(x23, x23, ffma2(x01, x01, f32x2(0.f, 0.f)));
        dv[kk] = f32x2_lo(acc) + f32x2_hi(acc);
        nv[kk] = f32x2_lo(nrm) + f32x2_hi(nrm);
        pool[0] += static_cast<double>(a0);
        pool[1] += static_cast<double>(a1);
        pool[2] += static_cast<double>(a2);
        pool[3] += static_cast<double>(a3);
      }
      // reduce-scatter: keep the low half of the slots, send the high half
#pragma unroll
      for (int half = QP_ROWS / 2, msk = 16; half >= 1; half >>= 1, msk >>= 1) {
#pragma unroll
        for (int kk = 0; kk < half; ++kk) {
          dv[kk] += __shfl_xor_sync(0xffffffffu, dv[kk + half], msk);
          nv[kk] += __shfl_xor_sync(0xffffffffu, nv[kk + half], msk);
        }
      }
#pragma unroll
      for (int msk = QP_SHARE / 2; msk >= 1; msk >>= 1) {
        dv[0] += __shfl_xor_sync(0xffffffffu, dv[0], msk);
        nv[0] += __shfl_xor_sync(0xffffffffu, nv[0], msk);
      }
      // the QP_SHARE lanes of row m decide it identically
      const int rr = rbase + m, r = r0 + rr;
      const bool mine = rr < nr;
      int act = 1;
      bool near = false;
      if (mine && r < n_vision && !(preserve && h == 0)) {
        const double dd = static_cast<double>(dv[0]);
        if (fabs(dd - tau_logit) > static_cast<double>(kboundf * sqrtf(nv[0])) + band) act = dd > tau_logit ? 1 : 0;
        else near = (lane & (QP_SHARE - 1)) == 0;
      }
      unsigned nearm = __ballot_sync(0xffffffffu, near);
      while (nearm) {
        // rare: q_score_bulk_kernel's float64 evaluation, operation for
        // operation (16 lanes x 8 columns, FMA chains in column order, the
        // xor 8 / 4 / 2 / 1 tree), so verdict and p agree with the want_prob path
        const int fl = __ffs(nearm) - 1;
        nearm &= nearm - 1;
        const int ru = rbase + sp_row_mask(fl);
        const int cl = lane & 15;
        const uint4 q = *reinterpret_cast<const uint4*>(qsm + (size_t)ru * (d * 2) + cl * 16);
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&q);
        double sl = 0.0, sa = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double v = static_cast<double>(__bfloat162float(hv[e]));
          sl = fma(v, __ldg(k_lazy + (size_t)g * d + cl * 8 + e), sl);
          sa = fma(v, __ldg(k_act + (size_t)g * d + cl * 8 + e), sa);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          sl += __shfl_xor_sync(0xffffffffu, sl, o);
          sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        const int a = two_way_active(sl * scale, sa * scale, tau, tau_logit, nullptr);
        if ((lane / QP_SHARE) == (fl / QP_SHARE)) act = a;
      }
      if (mine && (lane & (QP_SHARE - 1)) == 0) {
        active[(size_t)h * N + r] = static_cast<uint8_t>(act);
        cnt += act;
      }
      // a lazy row's output row is zeroed by its QP_SHARE lanes
      if (o_zero && mine && !act) {
        constexpr int per = 16 / QP_SHARE;  // 16-byte stores per lane
        uint4* orow = reinterpret_cast<uint4*>(o_zero + ((size_t)h * N + r) * d) + (lane & (QP_SHARE - 1)) * per;
#pragma unroll
        for (int c = 0; c < per; ++c) orow[c] = make_uint4(0, 0, 0, 0);
      }
    }
    const int sl = k & 1;
    double* slab = s_pool + (size_t)sl * QP_WARPS * d;
    cnt = warp_sum(cnt);
    if (k >= 2) mbar_wait(smem_u32(&sfree[sl]), ((k >> 1) - 1) & 1);  // item k - 2's slab read
    *reinterpret_cast<double2*>(slab + warp * d + 4 * lane) = make_double2(pool[0], pool[1]);
    *reinterpret_cast<double2*>(slab + warp * d + 4 * lane + 2) = make_double2(pool[2], pool[3]);
    if (lane == 0) s_cnt[sl][warp] = cnt;
    mbar_arrive(smem_u32(&done[sl]));  // releases this thread's slab writes and stage reads
    if (warp < 4) {  // reducers: the item's column sums over the warps in a fixed order
      mbar_wait(smem_u32(&done[sl]), (k >> 1) & 1);
      if (threadIdx.x == 0 && i + SP_STAGES * G < n_items)  // every warp is done with stage s
        sp_issue(Q, nb, block, N, i + SP_STAGES * G, ring + s * SP_STAGE, smem_u32(&bars[s]));
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < QP_WARPS; ++w) t += slab[w * d + threadIdx.x];
      pooled_q[((size_t)h * nb + it.J) * d + threadIdx.x] = t / static_cast<double>(nr);
      if (threadIdx.x == 0) {
        int c = 0;
        for (int w = 0; w < QP_WARPS; ++w) c += s_cnt[sl][w];
        block_active[(size_t)h * nb + it.J] = c;
      }
      mbar_arrive(smem_u32(&sfree[sl]));
    }
  }
}

// K1: pooled K (all rows) and the vision partial (rows < n_vision, summed
// separately only on blocks that reach past the vision span) per block,
// float64. Lane L owns columns 4L..4L+3 (8-byte loads, a warp reads whole
// rows) and a warp owns 32 rows of the item: no cross-lane reduction.
constexpr int KP_WARPS = 8;
constexpr uint32_t KP_SMEM = SP_STAGES * SP_STAGE + 2 * 2 * KP_WARPS * 128 * 8;

__global__ void __launch_bounds__(KP_WARPS * 32, 1) kv_probe_stream_kernel(const __nv_bfloat16* __restrict__ K, int N,
                                                                           int nb, int n_items, int n_vision, int block,
                                                                           double* __restrict__ pooled_k,
                                                                           double* __restrict__ vis_part) {
  constexpr int d = 128;
  extern __shared__ __align__(1024) uint8_t sp_smem[];
  __shared__ __align__(8) uint64_t bars[SP_STAGES];
  double* s_red = reinterpret_cast<double*>(sp_smem + SP_STAGES * SP_STAGE);  // [2][all|vis][warps][128]
  const uint32_t ring = smem_u32(sp_smem);
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SP_STAGES; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
    for (int k = 0; k < SP_STAGES; ++k) {
      const int i = blockIdx.x + k * G;
      if (i < n_items) sp_issue(K, nb, block, N, i, ring + k * SP_STAGE, smem_u32(&bars[k]));
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0;; ++k) {
    const int i = blockIdx.x + k * G;
    if (i >= n_items) break;
    const int s = k % SP_STAGES;
    const SpItem it = sp_item(i, nb, block, N);
    const bool split = it.r0 + it.nr > n_vision;
    const uint8_t* ksm = sp_smem + s * SP_STAGE;
    double all[4] = {0.0, 0.0, 0.0, 0.0}, vis[4] = {0.0, 0.0, 0.0, 0.0};
    mbar_wait(smem_u32(&bars[s]), (k / SP_STAGES) & 1);
    const int rend = min(it.nr, (warp + 1) * 32);
#pragma unroll 8
    for (int rr = warp * 32; rr < rend; ++rr) {
      const uint2 w = *reinterpret_cast<const uint2*>(ksm + (size_t)rr * (d * 2) + lane * 8);
      const double a0 = bf_lo(w.x), a1 = bf_hi(w.x), a2 = bf_lo(w.y), a3 = bf_hi(w.y);
      all[0] += a0;
      all[1] += a1;
      all[2] += a2;
      all[3] += a3;
      if (split && it.r0 + rr < n_vision) {
        vis[0] += a0;
        vis[1] += a1;
        vis[2] += a2;
        vis[3] += a3;
      }
    }
    double* slab = s_red + (size_t)(k & 1) * 2 * KP_WARPS * d;
    *reinterpret_cast<double2*>(slab + warp * d + 4 * lane) = make_double2(all[0], all[1]);
    *reinterpret_cast<double2*>(slab + warp * d + 4 * lane + 2) = make_double2(all[2], all[3]);
    if (split) {
      *reinterpret_cast<double2*>(slab + (KP_WARPS + warp) * d + 4 * lane) = make_double2(vis[0], vis[1]);
      *reinterpret_cast<double2*>(slab + (KP_WARPS + warp) * d + 4 * lane + 2) = make_double2(vis[2], vis[3]);
    }
    __syncthreads();  // stage s consumed, slab complete
    if (threadIdx.x == 0 && i + SP_STAGES * G < n_items)
      sp_issue(K, nb, block, N, i + SP_STAGES * G, ring + s * SP_STAGE, smem_u32(&bars[s]));
    if (threadIdx.x < d) {
      double a = 0.0, v = 0.0;
#pragma unroll
      for (int w = 0; w < KP_WARPS; ++w) {
        a += slab[w * d + threadIdx.x];
        if (split) v += slab[(KP_WARPS + w) * d + threadIdx.x];
      }
      const size_t o = ((size_t)it.h * nb + it.J) * d + threadIdx.x;
      pooled_k[o] = a / static_cast<double>(it.nr);
      vis_part[o] = split ? v : a;
    }
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
// dst[g, r] = src[g, idx[g, r]]: each warp moves GR_ROWS rows per pass with
// 16-byte lane copies (256-byte bf16 rows: two rows per warp instruction),
// all loads of a pass issued before the stores so several KB are in flight
// per warp; rows [count, roundup(count, pad)) are zero-filled.
constexpr int GR_ROWS = 8;

__global__ void __launch_bounds__(256) gather_rows_kernel(const uint8_t* __restrict__ src, int src_rows,
                                                          int row_bytes, const int32_t* __restrict__ idx,
                                                          int idx_stride, const int32_t* __restrict__ counts,
                                                          int count_const, uint8_t* __restrict__ dst, int dst_rows,
                                                          int pad_rows) {
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = counts ? counts[g] : count_const;
  const int lim = min(dst_rows, ((cnt + pad_rows - 1) / pad_rows) * pad_rows);
  const int chunks = row_bytes >> 4;  // 16-byte chunks per row
  const int r0 = (blockIdx.x * 8 + warp) * GR_ROWS;
  if (r0 >= lim) return;
  const int total = GR_ROWS * chunks;  // chunks this warp moves
  for (int base = 0; base < total; base += 32 * 4) {
    uint4 v[4];
    int rr[4], cc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = base + u * 32 + lane;
      rr[u] = r0 + e / chunks;
      cc[u] = e % chunks;
      v[u] = make_uint4(0, 0, 0, 0);
      if (e < total && rr[u] < cnt) {
        const int sidx = __ldg(idx + (size_t)g * idx_stride + rr[u]);
        v[u] = __ldg(reinterpret_cast<const uint4*>(src + ((size_t)g * src_rows + sidx) * row_bytes) + cc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = base + u * 32 + lane;
      if (e < total && rr[u] < lim)
        reinterpret_cast<uint4*>(dst + ((size_t)g * dst_rows + rr[u]) * row_bytes)[cc[u]] = v[u];
    }
  }
}

// dst[g, idx[g, r]] = src[g, r] for r < counts[g] (the inverse of the gather:
// compacted key gradients back to original positions), 16-byte lane copies.
__global__ void __launch_bounds__(256) scatter_rows_kernel(const uint8_t* __restrict__ src, int src_rows,
                                                           int row_bytes, const int32_t* __restrict__ idx,
                                                           int idx_stride, const int32_t* __restrict__ counts,
                                                           uint8_t* __restrict__ dst, int dst_rows) {
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = min(__ldg(counts + g), src_rows);
  const int chunks = row_bytes >> 4;
  for (int r = blockIdx.x * 8 + warp; r < cnt; r += gridDim.x * 8) {
    const int d = __ldg(idx + (size_t)g * idx_stride + r);
    if (d < 0 || d >= dst_rows) continue;
    const uint4* s = reinterpret_cast<const uint4*>(src + ((size_t)g * src_rows + r) * row_bytes);
    uint4* o = reinterpret_cast<uint4*>(dst + ((size_t)g * dst_rows + d) * row_bytes);
    for (int c = lane; c < chunks; c += 32) o[c] = __ldg(s + c);
  }
}

// Key-gradient epilogue (training): compacted fp32 dK / dV rows to their
// original positions in the leaves' dtype, the sink row's extra dV (rows
// whose forward copied V[sink]) folded in before the rounding.
__global__ void __launch_bounds__(256) scatter_key_grads_kernel(const float* __restrict__ src, int src_rows, int d,
                                                                const int32_t* __restrict__ idx, int idx_stride,
                                                                const int32_t* __restrict__ counts, int sink,
                                                                const float* __restrict__ sink_add, void* dst,
                                                                int bf16, int dst_rows) {
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = min(__ldg(counts + g), src_rows);
  const int32_t* ig = idx + (size_t)g * idx_stride;
  auto store = [&](int p, int c, float4 v) {
    if (bf16) {
      uint2* o = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(dst) + ((size_t)g * dst_rows + p) * d + c);
      *o = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    } else {
      *reinterpret_cast<float4*>(static_cast<float*>(dst) + ((size_t)g * dst_rows + p) * d + c) = v;
    }
  };
  if (sink_add && blockIdx.x == 0 && warp == 0) {
    // sink row not among the selected keys: it receives only the extra dV
    const bool member = count_le(ig, cnt, sink) > (sink > 0 ? count_le(ig, cnt, sink - 1) : 0);
    if (!member && sink >= 0 && sink < dst_rows)
      for (int c = lane * 4; c < d; c += 128)
        store(sink, c, __ldg(reinterpret_cast<const float4*>(sink_add + (size_t)g * d + c)));
  }
  for (int r = blockIdx.x * 8 + warp; r < cnt; r += gridDim.x * 8) {
    const int p = __ldg(ig + r);
    if (p < 0 || p >= dst_rows) continue;
    const float* s = src + ((size_t)g * src_rows + r) * d;
    for (int c = lane * 4; c < d; c += 128) {
      float4 v = __ldg(reinterpret_cast<const float4*>(s + c));
      if (sink_add && p == sink) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(sink_add + (size_t)g * d + c));
        v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
      }
      store(p, c, v);
    }
  }
}

}  // namespace omni

using namespace omni;

static inline int nblocks(int n, int b) { return (n + b - 1) / b; }

extern "C" int omni_scatter_key_grads(const float* src, int n_groups, int src_rows, int head_dim, const int32_t* idx,
                                      int idx_stride, const int32_t* counts, int sink_index, const float* sink_add,
                                      void* dst, int dst_dtype, int dst_rows, void* stream) {
  omni_begin();
  OMNI_CHECK(dst_dtype == OMNI_DTYPE_F32 || dst_dtype == OMNI_DTYPE_BF16, OMNI_E_PARAM, "key gradients must be f32 or bf16");
  OMNI_CHECK(head_dim % 4 == 0 && head_dim >= 4, OMNI_E_SHAPE, "head_dim must be a multiple of 4");
  OMNI_CHECK(counts != nullptr, OMNI_E_PARAM, "scatter needs device counts");
  if (n_groups == 0 || src_rows == 0) return OMNI_OK;
  dim3 grid(min(nblocks(src_rows, 8), 1024), n_groups);
  scatter_key_grads_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, src_rows, head_dim, idx, idx_stride, counts, sink_index, sink_add, dst, dst_dtype == OMNI_DTYPE_BF16 ? 1 : 0,
      dst_rows);
  return omni_launch_check();
}

// OMNI_QSCORE_F64=1 (tests / A-B): the float64 q_score_bulk_kernel for every
// row instead of the fp32-with-bound fast kernel.
static int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

static bool fast_off() {
  static const bool off = [] {
    const char* e = getenv("OMNI_QSCORE_F64");
    return e && atoi(e) != 0;
  }();
  return off;
}

extern "C" size_t omni_kv_probe_workspace(int n_kv_heads, int seq_len, int head_dim, int block_size) {
  if (block_size < 1) return 0;
  return sizeof(double) * (size_t)n_kv_heads * nblocks(seq_len, block_size) * head_dim;
}

extern "C" int omni_kv_probe(const void* K, int dtype, int n_kv_heads, int seq_len, int head_dim, int n_vision,
                             int sink_index, int block_size, double* k_lazy, double* k_act, double* pooled_k,
                             void* workspace, void* stream) {
  omni_begin();
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
  if (dtype == OMNI_DTYPE_BF16 && head_dim == 128 && block_size <= QSB_MAX_ROWS) {
    const int items = nb * n_kv_heads;
    OMNI_CUDA_TRY(omni_smem_attr(kv_probe_stream_kernel, (int)KP_SMEM));
    kv_probe_stream_kernel<<<std::min(items, num_sms()), KP_WARPS * 32, KP_SMEM, s>>>(
        static_cast<const __nv_bfloat16*>(K), seq_len, nb, items, n_vision, block_size, pooled_k, vis);
    probe_finish_kernel<__nv_bfloat16><<<dim3(4, n_kv_heads), 1024, 0, s>>>(
        static_cast<const __nv_bfloat16*>(K), seq_len, head_dim, nb, n_vision, sink_index, vis, k_lazy, k_act);
  } else if (dtype == OMNI_DTYPE_BF16) {
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
  } else if (dtype == OMNI_DTYPE_F64) {
    kv_probe_kernel<double><<<grid, 256, shm, s>>>(static_cast<const double*>(K), seq_len, head_dim, n_vision,
                                                     block_size, pooled_k, vis);
    probe_finish_kernel<double><<<dim3((head_dim + 31) / 32, n_kv_heads), 1024, 0, s>>>(
        static_cast<const double*>(K), seq_len, head_dim, nb, n_vision, sink_index, vis, k_lazy, k_act);
  } else {
    OMNI_CHECK(false, OMNI_E_PARAM, "unsupported dtype");
  }
  return omni_launch_check();
}

extern "C" int omni_q_score(const void* Q, int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim,
                            int n_vision, double tau, int preserve_first_head, int block_size, const double* k_lazy,
                            const double* k_act, uint8_t* active, double* p_act, double* pooled_q,
                            int32_t* block_active, void* O_zero, void* stream) {
  omni_begin();
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(n_vision >= 0 && n_vision <= seq_len, OMNI_E_LAYOUT, "n_vision outside the sequence");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim == 32 || head_dim == 64 || head_dim == 128 || head_dim == 256, OMNI_E_SHAPE,
             "head_dim must be 32, 64, 128 or 256");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 grid(nblocks(seq_len, block_size), n_q_heads);
  const int rep = n_q_heads / n_kv_heads;
  const double T = tau > 0.0 ? log(tau / (1.0 - tau)) : -INFINITY;  // decision threshold on l1 - l0
  __nv_bfloat16* oz = static_cast<__nv_bfloat16*>(O_zero);
  if (dtype == OMNI_DTYPE_BF16 && head_dim == 128 && block_size >= 64 && block_size <= QSB_MAX_ROWS &&
      p_act == nullptr && tau > 0.0 && !fast_off()) {
    const int items = (int)grid.x * n_q_heads;
    OMNI_CUDA_TRY(omni_smem_attr(q_score_stream_kernel, (int)QP_SMEM));
    q_score_stream_kernel<<<std::min(items, num_sms()), QP_WARPS * 32, QP_SMEM, s>>>(
        static_cast<const __nv_bfloat16*>(Q), seq_len, (int)grid.x, items, rep, n_vision, tau, T, preserve_first_head,
        block_size, k_lazy, k_act, active, pooled_q, block_active, oz);
  } else if (dtype == OMNI_DTYPE_BF16 && head_dim == 128 && block_size >= 64 && block_size <= QSB_MAX_ROWS) {
    const int shm = block_size * head_dim * 2;
    OMNI_CUDA_TRY(omni_smem_attr(q_score_bulk_kernel, QSB_MAX_ROWS * 128 * 2));  // one limit for every block size
    q_score_bulk_kernel<<<grid, 256, shm, s>>>(static_cast<const __nv_bfloat16*>(Q), seq_len, rep, n_vision, tau, T,
                                               preserve_first_head, block_size, k_lazy, k_act, active, p_act, pooled_q,
                                               block_active, oz);
  } else if (dtype == OMNI_DTYPE_BF16)
    q_score_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(Q), seq_len, head_dim, rep,
                                                       n_vision, tau, T, preserve_first_head, block_size, k_lazy,
                                                       k_act, active, p_act, pooled_q, block_active, oz);
  else if (dtype == OMNI_DTYPE_F32)
    q_score_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(Q), seq_len, head_dim, rep, n_vision, tau, T,
                                               preserve_first_head, block_size, k_lazy, k_act, active, p_act,
                                               pooled_q, block_active, oz);
  else if (dtype == OMNI_DTYPE_F64)
    q_score_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(Q), seq_len, head_dim, rep, n_vision, tau,
                                                T, preserve_first_head, block_size, k_lazy, k_act, active, p_act,
                                                pooled_q, block_active, oz);
  else
    OMNI_CHECK(false, OMNI_E_PARAM, "unsupported dtype");
  return omni_launch_check();
}

extern "C" int omni_compact_rows(const uint8_t* active, const int32_t* block_active, int n_q_heads, int seq_len,
                                 int block_size, int32_t* rows, int32_t* counts, void* stream) {
  omni_begin();
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  dim3 grid(nblocks(seq_len, block_size), n_q_heads);
  compact_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(active, block_active, seq_len, block_size,
                                                                           rows, counts);
  return omni_launch_check();
}

extern "C" int omni_gather_rows(const void* src, int dtype, int n_groups, int src_rows, int head_dim,
                                const int32_t* idx, int idx_stride, const int32_t* counts, int count_const, void* dst,
                                int dst_rows, int pad_rows, void* stream) {
  omni_begin();
  OMNI_CHECK(pad_rows >= 1, OMNI_E_PARAM, "pad_rows must be >= 1");
  const int esz = dtype == OMNI_DTYPE_BF16 ? 2 : dtype == OMNI_DTYPE_F64 ? 8 : 4;
  const int row_bytes = head_dim * esz;
  OMNI_CHECK(row_bytes % 16 == 0, OMNI_E_SHAPE, "row bytes must be a multiple of 16");
  dim3 grid(nblocks(dst_rows, 8 * GR_ROWS), n_groups);
  if (grid.x == 0 || n_groups == 0) return OMNI_OK;
  gather_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), src_rows, row_bytes, idx, idx_stride, counts, count_const,
      static_cast<uint8_t*>(dst), dst_rows, pad_rows);
  return omni_launch_check();
}

extern "C" int omni_scatter_rows(const void* src, int dtype, int n_groups, int src_rows, int head_dim,
                                 const int32_t* idx, int idx_stride, const int32_t* counts, void* dst, int dst_rows,
                                 void* stream) {
  omni_begin();
  const int esz = dtype == OMNI_DTYPE_BF16 ? 2 : dtype == OMNI_DTYPE_F64 ? 8 : 4;
  const int row_bytes = head_dim * esz;
  OMNI_CHECK(row_bytes % 16 == 0, OMNI_E_SHAPE, "row bytes must be a multiple of 16");
  OMNI_CHECK(counts != nullptr, OMNI_E_PARAM, "scatter needs device counts");
  if (n_groups == 0 || src_rows == 0) return OMNI_OK;
  dim3 grid(min(nblocks(src_rows, 8), 1024), n_groups);
  scatter_rows_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), src_rows, row_bytes, idx, idx_stride, counts, static_cast<uint8_t*>(dst),
      dst_rows);
  return omni_launch_check();
}

// SURVEY §8b's minimum export set names the cache slimming entry point
// omni_slim_cache: build_cache's pruning + regrouping (decode.py:92-107) of one
// sequence — the budget selected vision rows of K and V per KV group into the
// slim cache segments [Hkv, vcap, d], rows past the budget zero-filled (the
// TMA-staged decode reads whole 64-row tiles).
extern "C" int omni_slim_cache(const void* K, const void* V, int dtype, int n_kv_heads, int seq_len, int head_dim,
                               const int32_t* vision_selected, int sel_stride, int budget, int vcap, void* vision_k,
                               void* vision_v, void* stream) {
  omni_begin();
  OMNI_CHECK(budget >= 1 && budget <= vcap, OMNI_E_INTEGRITY, "budget outside [1, vision capacity]");
  int rc = omni_gather_rows(K, dtype, n_kv_heads, seq_len, head_dim, vision_selected, sel_stride, nullptr, budget,
                            vision_k, vcap, vcap, stream);
  if (rc) return rc;
  return omni_gather_rows(V, dtype, n_kv_heads, seq_len, head_dim, vision_selected, sel_stride, nullptr, budget,
                          vision_v, vcap, vcap, stream);
}
