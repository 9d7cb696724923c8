// K3: block-probe column mass (K3a) and shared-budget KV selection (K3b).
//
// K3a is the (N/B)^2 d probe of block_probe.py:44-64 in float64 — at 64K
// tokens that is 28 heads x 256 x 256 pooled scores, latency-bound (µs), not a
// roofline kernel. K3b is a single-CTA selection: per-group token scores,
// length-weighted kurtosis, argmin (flattest head), top-p budget on the
// flattest group and one top-b block table per group, written out as
// ascending index lists (kv_select.py:49-195). Scores on the probe path are
// constant within a probe block, so every sort/scan runs over nb blocks
// instead of N tokens; block_size = 1 degenerates to the token-exact path.
#include <float.h>
#include <limits.h>

#include "common.cuh"

namespace omni {

constexpr int kSelMaxBlocks = 8192;

// ----------------------------------------------------------------------- K3a
// Scores S[h, I, J] = pq[h, I] . pk[g, J] / sqrt(d) for J <= I (block-causal
// tril). CTA = 16 query blocks x all visible key blocks, staged through smem in
// tiles of 32 key blocks (rows padded by one double: conflict-free f64 reads).
__global__ void __launch_bounds__(256) probe_scores_kernel(const double* __restrict__ pq,
                                                           const double* __restrict__ pk, int nb, int d, int rep,
                                                           double* __restrict__ S) {
  extern __shared__ double sh[];
  const int ld = d + 1;
  double* sq = sh;            // [16][ld]
  double* sk = sh + 16 * ld;  // [32][ld]
  const int h = blockIdx.y, g = h / rep;
  const int I0 = blockIdx.x * 16;
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  for (int e = threadIdx.x; e < 16 * d; e += blockDim.x) {
    const int i = e / d, c = e % d;
    sq[i * ld + c] = (I0 + i < nb) ? pq[((size_t)h * nb + I0 + i) * d + c] : 0.0;
  }
  const int jmax = min(nb, I0 + 16);
  const int ti = threadIdx.x / 16, tj = threadIdx.x % 16;
  const int I = I0 + ti;
  for (int jt = 0; jt < jmax; jt += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * d; e += blockDim.x) {
      const int j = e / d, c = e % d;
      sk[j * ld + c] = (jt + j < nb) ? pk[((size_t)g * nb + jt + j) * d + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int jj = tj + 16 * u, J = jt + jj;
      if (I < nb && J <= I) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
        for (; c + 4 <= d; c += 4) {
          a0 = fma(sq[ti * ld + c], sk[jj * ld + c], a0);
          a1 = fma(sq[ti * ld + c + 1], sk[jj * ld + c + 1], a1);
          a2 = fma(sq[ti * ld + c + 2], sk[jj * ld + c + 2], a2);
          a3 = fma(sq[ti * ld + c + 3], sk[jj * ld + c + 3], a3);
        }
        for (; c < d; ++c) a0 = fma(sq[ti * ld + c], sk[jj * ld + c], a0);
        S[((size_t)h * nb + I) * nb + J] = ((a0 + a1) + (a2 + a3)) * scale;
      }
    }
  }
}

// Row max and sum of exp(S - max) over the visible prefix J <= I (warp/row).
__global__ void probe_rowstats_kernel(const double* __restrict__ S, int nb, double* __restrict__ stats) {
  const int I = blockIdx.x, h = blockIdx.y, lane = threadIdx.x;
  const double* row = S + ((size_t)h * nb + I) * nb;
  double mx = -DBL_MAX;
  for (int J = lane; J <= I; J += 32) mx = fmax(mx, row[J]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double s = 0.0;
  for (int J = lane; J <= I; J += 32) s += exp(row[J] - mx);
  s = warp_sum(s);
  if (lane == 0) {
    stats[((size_t)h * nb + I) * 2 + 0] = mx;
    stats[((size_t)h * nb + I) * 2 + 1] = s;
  }
}

// mass[h, J] = sum over rows I >= J of exp(S[I, J] - max_I) / sum_I. Block of
// 32 columns x 8 row-phases: each thread sums the rows I = J + phase mod 8 (8
// independent loads in flight), partials are combined in a fixed order.
__global__ void __launch_bounds__(256) probe_colsum_kernel(const double* __restrict__ S,
                                                           const double* __restrict__ stats, int nb,
                                                           double* __restrict__ mass) {
  __shared__ double part[8][33];
  const int h = blockIdx.y;
  const int cj = threadIdx.x & 31, ph = threadIdx.x >> 5;
  const int J = blockIdx.x * 32 + cj;
  double acc = 0.0;
  if (J < nb) {
    const double* Sh = S + (size_t)h * nb * nb;
    const double* st = stats + (size_t)h * nb * 2;
    for (int I = J + ph; I < nb; I += 8) acc += exp(Sh[(size_t)I * nb + J] - st[2 * I]) / st[2 * I + 1];
  }
  part[ph][cj] = acc;
  __syncthreads();
  if (ph == 0 && J < nb) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += part[k][cj];
    mass[(size_t)h * nb + J] = t;
  }
}

// Fused K3a (hot path, nb <= 512): CTA = 16 query blocks of one Q head. The
// pooled scores of its 16 rows against every visible key block are computed
// into shared memory (2 x 2 register micro-tiles over 64-key-block tiles of
// pooled K), the row max / sum of the masked softmax follow in place, and the
// CTA writes its 16-row partial column sums; probe_colsum_partials_kernel adds
// the partials of all CTAs in ascending row-tile order (deterministic). No
// nb x nb map in HBM, three launches -> two.
constexpr int PF_ROWS = 16, PF_JT = 64, PF_MAXNB = 512;

__global__ void __launch_bounds__(256) probe_mass_fused_kernel(const double* __restrict__ pq,
                                                               const double* __restrict__ pk, int nb, int rep,
                                                               double* __restrict__ partial) {
  constexpr int d = 128, ld = d + 2;  // +2 doubles: 16-byte aligned rows, staggered banks
  extern __shared__ double psm[];
  double* sq = psm;                   // [16][ld]
  double* skb = sq + PF_ROWS * ld;    // [2][64][ld]: key tiles, double-buffered
  double* S = skb + 2 * PF_JT * ld;   // [16][nb]
  __shared__ double s_m[PF_ROWS], s_l[PF_ROWS];
  const int h = blockIdx.y, g = h / rep;
  const int I0 = blockIdx.x * PF_ROWS;
  const int jmax = min(nb, I0 + PF_ROWS);  // key blocks visible to the CTA's last row
  const double scale = 1.0 / sqrt(static_cast<double>(d));
  // global -> shared copies as 16-byte cp.async (all of a thread's chunks in
  // flight at once; padded rows keep the micro-tile reads conflict-free), one
  // commit group per call
  auto copy_rows = [&](double* dst, const double* src, int rows, int valid) {
    for (int e = threadIdx.x; e < rows * (d / 2); e += blockDim.x) {
      const int i = e / (d / 2), c2 = e % (d / 2);
      double* dp = dst + i * ld + 2 * c2;
      if (i < valid) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dp)), "l"(src + (size_t)i * d + 2 * c2)
                     : "memory");
      } else {
        dp[0] = 0.0;
        dp[1] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  copy_rows(sq, pq + ((size_t)h * nb + I0) * d, PF_ROWS, min(PF_ROWS, nb - I0));
  copy_rows(skb, pk + (size_t)g * nb * d, PF_JT, min(PF_JT, nb));
  // thread -> rows {ti, ti + 8}, key blocks {tj, tj + 32} of the 64-wide tile
  const int ti = threadIdx.x >> 5, tj = threadIdx.x & 31;
  for (int jt = 0, it = 0; jt < jmax; jt += PF_JT, ++it) {
    double* sk = skb + (it & 1) * PF_JT * ld;
    if (jt + PF_JT < jmax) {  // the next key tile streams in while this one is used
      copy_rows(skb + ((it + 1) & 1) * PF_JT * ld, pk + ((size_t)g * nb + jt + PF_JT) * d, PF_JT,
                min(PF_JT, nb - jt - PF_JT));
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
    const double* q0 = sq + ti * ld;
    const double* q1 = sq + (ti + 8) * ld;
    const double* k0 = sk + tj * ld;
    const double* k1 = sk + (tj + 32) * ld;
#pragma unroll 4
    for (int c = 0; c < d; c += 2) {
      const double2 x0 = *reinterpret_cast<const double2*>(q0 + c), x1 = *reinterpret_cast<const double2*>(q1 + c);
      const double2 y0 = *reinterpret_cast<const double2*>(k0 + c), y1 = *reinterpret_cast<const double2*>(k1 + c);
      a00 = fma(x0.x, y0.x, a00); a00 = fma(x0.y, y0.y, a00);
      a01 = fma(x0.x, y1.x, a01); a01 = fma(x0.y, y1.y, a01);
      a10 = fma(x1.x, y0.x, a10); a10 = fma(x1.y, y0.y, a10);
      a11 = fma(x1.x, y1.x, a11); a11 = fma(x1.y, y1.y, a11);
    }
    const int J0 = jt + tj, J1 = jt + tj + 32;
    if (J0 < nb) { S[ti * nb + J0] = a00 * scale; S[(ti + 8) * nb + J0] = a10 * scale; }
    if (J1 < nb) { S[ti * nb + J1] = a01 * scale; S[(ti + 8) * nb + J1] = a11 * scale; }
    __syncthreads();  // every thread is done with this buffer before it is refilled
  }
  __syncthreads();
  // masked softmax statistics of each row over J <= I (warp per two rows)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int ii = warp; ii < PF_ROWS; ii += 8) {
    const int I = I0 + ii;
    double mx = -DBL_MAX, sum = 0.0;
    if (I < nb) {
      for (int J = lane; J <= I; J += 32) mx = fmax(mx, S[ii * nb + J]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int J = lane; J <= I; J += 32) {  // keep exp(S - max) for the column pass
        const double e = exp(S[ii * nb + J] - mx);
        S[ii * nb + J] = e;
        sum += e;
      }
      sum = warp_sum(sum);
    }
    if (lane == 0) { s_m[ii] = mx; s_l[ii] = sum; }
  }
  __syncthreads();
  // partial column sums of the normalised rows (fixed row order)
  double* out = partial + ((size_t)h * gridDim.x + blockIdx.x) * nb;
  for (int J = threadIdx.x; J < jmax; J += blockDim.x) {
    double t = 0.0;
    for (int ii = max(0, J - I0); ii < PF_ROWS; ++ii) {
      const int I = I0 + ii;
      if (I < nb) t += S[ii * nb + J] / s_l[ii];
    }
    out[J] = t;
  }
}

// mass[h, J] = sum over row tiles T with 16 T + 15 >= J of partial[h, T, J].
__global__ void probe_colsum_partials_kernel(const double* __restrict__ partial, int nb, int ntiles,
                                             double* __restrict__ mass) {
  const int h = blockIdx.y;
  const int J = blockIdx.x * blockDim.x + threadIdx.x;
  if (J >= nb) return;
  double t = 0.0;
  for (int T = J / PF_ROWS; T < ntiles; ++T) t += partial[((size_t)h * ntiles + T) * nb + J];
  mass[(size_t)h * nb + J] = t;
}

// ----------------------------------------------------------------------- K3b
struct SelShared {
  double key[kSelMaxBlocks];
  double pre[kSelMaxBlocks];
  int idx[kSelMaxBlocks];
  int take[kSelMaxBlocks];
  int ipre[kSelMaxBlocks];
  double wtot[32];
  int itot[32];
  int cross;
  double red[32];
  double kurt[64];
  int flat;
  int budget;
  double retained, total;
};

__device__ __forceinline__ int block_len(int J, int N, int B) { return min(B, N - J * B); }

__device__ double block_reduce_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// In-place inclusive prefix sum of a[0..n) (smem) with the whole block:
// contiguous per-thread runs, warp shuffles, then warp totals.
template <typename T>
__device__ void block_inclusive_scan(T* a, int n, T* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int beg = min(n, threadIdx.x * per), end = min(n, beg + per);
  T run = 0;
  for (int i = beg; i < end; ++i) {
    run += a[i];
    a[i] = run;
  }
  T v = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < nw) ? tot[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    tot[lane] = w;
  }
  __syncthreads();
  const T off = (v - run) + (warp > 0 ? tot[warp - 1] : T(0));
  for (int i = beg; i < end; ++i) a[i] += off;
  __syncthreads();
}

// Ascending bitonic sort of (key, idx) pairs, ties broken by idx: with
// key = -score this is the reference's lexsort((arange, -a)) order.
__device__ void bitonic_sort(double* key, int* idx, int n_pow2) {
  for (int k = 2; k <= n_pow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n_pow2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const bool up = (i & k) == 0;
          const double ki = key[i], kp = key[p];
          const int ii = idx[i], ip = idx[p];
          const bool gt = (ki > kp) || (ki == kp && ii > ip);
          if (gt == up) {
            key[i] = kp; key[p] = ki;
            idx[i] = ip; idx[p] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(1024) select_kernel(const double* __restrict__ mass, int hq, int hkv, int N, int B,
                                                      double p, int gran, int vision_limit, int budget_override,
                                                      int32_t* __restrict__ selected, int32_t* __restrict__ info,
                                                      double* __restrict__ stats, double* __restrict__ gscores) {
  extern __shared__ __align__(16) unsigned char sel_raw[];
  SelShared& S = *reinterpret_cast<SelShared*>(sel_raw);
  const int nb = (N + B - 1) / B;
  const int rep = hq / hkv;
  int np2 = 1;
  while (np2 < nb) np2 <<= 1;

  // Phase 1: per-group per-token scores (block-constant) and kurtosis.
  for (int g = 0; g < hkv; ++g) {
    double part = 0.0;
    for (int J = threadIdx.x; J < nb; J += blockDim.x) {
      const double len = static_cast<double>(block_len(J, N, B));
      double s = mass[(size_t)(g * rep) * nb + J] / len;
      for (int r = 1; r < rep; ++r) s += mass[(size_t)(g * rep + r) * nb + J] / len;
      gscores[(size_t)g * nb + J] = s;
      part += len * s;
    }
    __syncthreads();
    const double mean = block_reduce_sum(part, S.red) / static_cast<double>(N);
    double p2 = 0.0, p4 = 0.0;
    for (int J = threadIdx.x; J < nb; J += blockDim.x) {
      const double len = static_cast<double>(block_len(J, N, B));
      const double dv = gscores[(size_t)g * nb + J] - mean;
      const double d2 = dv * dv;
      p2 += len * d2;
      p4 += len * d2 * d2;
    }
    const double m2 = block_reduce_sum(p2, S.red) / static_cast<double>(N);
    const double m4 = block_reduce_sum(p4, S.red) / static_cast<double>(N);
    if (threadIdx.x == 0) S.kurt[g] = (m2 == 0.0) ? 0.0 : m4 / (m2 * m2);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int f = 0;
    for (int g = 1; g < hkv; ++g)
      if (S.kurt[g] < S.kurt[f]) f = g;  // argmin, ties to the lowest index
    S.flat = f;
  }
  __syncthreads();
  const int flat = S.flat;

  // Phase 2: budget on the flattest group (descending cumsum over tokens,
  // evaluated block-wise: within a block of equal values cum = C + k * s).
  if (budget_override > 0) {
    if (threadIdx.x == 0) { S.budget = budget_override; S.retained = 0.0; S.total = 0.0; }
  } else {
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
      S.key[i] = (i < nb) ? -gscores[(size_t)flat * nb + i] : DBL_MAX;
      S.idx[i] = (i < nb) ? i : INT_MAX;
    }
    __syncthreads();
    bitonic_sort(S.key, S.idx, np2);
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      S.pre[i] = static_cast<double>(block_len(S.idx[i], N, B)) * (-S.key[i]);
    if (threadIdx.x == 0) S.cross = nb - 1;
    __syncthreads();
    block_inclusive_scan(S.pre, nb, S.wtot);  // descending-sorted cumulative mass, block-wise
    const double total = S.pre[nb - 1];
    const double thr = fmin(p * total, total);
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (S.pre[i] >= thr) atomicMin(&S.cross, i);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int i = S.cross;
      const double s = -S.key[i];
      const int len = block_len(S.idx[i], N, B);
      const double C = i > 0 ? S.pre[i - 1] : 0.0;
      int T = 0;
      for (int t = 0; t < i; ++t) T += block_len(S.idx[t], N, B);
      int k = len;
      if (s > 0.0) {
        const double kk = ceil((thr - C) / s);
        k = (kk < 1.0) ? 1 : (kk > len ? len : static_cast<int>(kk));
        while (k > 1 && C + static_cast<double>(k - 1) * s >= thr) --k;
        while (k < len && C + static_cast<double>(k) * s < thr) ++k;
      } else {
        k = 1;
      }
      S.budget = T + k;
      S.retained = C + static_cast<double>(k) * s;
      S.total = total;
    }
  }
  __syncthreads();
  int b = S.budget;
  const int span = (vision_limit >= 0) ? vision_limit : N;
  if (b > span) b = span;

  // Phase 3: per-group top-b block table -> ascending index list.
  for (int g = 0; g < hkv; ++g) {
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
      if (i < nb) {
        const double s = gscores[(size_t)g * nb + i];
        const double rank = (gran == OMNI_GRAN_BLOCK) ? s * static_cast<double>(block_len(i, N, B)) : s;
        S.key[i] = -rank;
        S.idx[i] = i;
      } else {
        S.key[i] = DBL_MAX;
        S.idx[i] = INT_MAX;
      }
      if (i < nb) S.take[i] = 0;
    }
    __syncthreads();
    bitonic_sort(S.key, S.idx, np2);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const int lo = S.idx[i] * B;
      S.ipre[i] = max(0, min(lo + block_len(S.idx[i], N, B), span) - lo);  // vision-clipped length
    }
    __syncthreads();
    block_inclusive_scan(S.ipre, nb, S.itot);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
      const int len = S.ipre[i] - (i > 0 ? S.ipre[i - 1] : 0);
      const int before = S.ipre[i] - len;
      S.take[S.idx[i]] = max(0, min(len, b - before));  // whole blocks in rank order, marginal prefix
    }
    __syncthreads();
    for (int J = threadIdx.x; J < nb; J += blockDim.x) S.ipre[J] = S.take[J];
    __syncthreads();
    block_inclusive_scan(S.ipre, nb, S.itot);
    for (int J = threadIdx.x; J < nb; J += blockDim.x) S.idx[J] = S.ipre[J] - S.take[J];  // exclusive offsets
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int J = warp; J < nb; J += nw) {
      const int t = S.take[J], off = S.idx[J];
      for (int k = lane; k < t; k += 32) selected[(size_t)g * N + off + k] = J * B + k;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    info[0] = b;
    info[1] = flat;
    info[2] = hkv;
    info[3] = nb;
    for (int g = 0; g < hkv; ++g) {
      info[4 + g] = b;  // per-group selected counts (all equal: shared budget)
      stats[g] = S.kurt[g];
    }
    stats[hkv] = S.retained;
    stats[hkv + 1] = S.total;
  }
}

// K3b, cluster variant (hot path: Hkv <= 8 groups, nb <= 1024 blocks). One
// CTA per KV group in a thread-block cluster: per-group scores, kurtosis and a
// one-pass rank sort run in parallel; the kurtoses and the flattest group's
// budget are exchanged through distributed shared memory with two cluster
// barriers. Same arithmetic and tie rules as select_kernel (kv_select.py:
// 49-195): argmin with ties to the lowest group, lexsort((arange, -a)) order.
constexpr int SC_MAXNB = 1024;
struct SelCl {
  double score[SC_MAXNB];  // per-token score of each block (this group)
  double skey[SC_MAXNB];   // sorted keys (ascending -rank)
  int sidx[SC_MAXNB];      // sorted block ids
  double pre[SC_MAXNB];
  int ipre[SC_MAXNB];
  int take[SC_MAXNB];
  double wtot[32];
  int itot[32];
  double red[32];
  double kurt;
  int budget;
  double retained, total;
  int cross;
};

// Ascending (key, index) order of key[0..n) by rank counting (n <= blockDim).
__device__ void rank_sort(const double* key, int n, double* skey, int* sidx) {
  const int i = threadIdx.x;
  if (i < n) {
    const double k = key[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double kj = key[j];
      r += (kj < k) || (kj == k && j < i);
    }
    skey[r] = k;
    sidx[r] = i;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024) select_cluster_kernel(const double* __restrict__ mass, int hq, int hkv, int N,
                                                              int B, double p, int gran, int vision_limit,
                                                              int budget_override, int32_t* __restrict__ selected,
                                                              int32_t* __restrict__ info, double* __restrict__ stats,
                                                              double* __restrict__ gscores) {
  extern __shared__ __align__(16) unsigned char sc_raw[];
  SelCl& S = *reinterpret_cast<SelCl*>(sc_raw);
  const int g = (int)cluster_ctarank();
  const int nb = (N + B - 1) / B;
  const int rep = hq / hkv;
  // per-group per-token scores (block-constant) and kurtosis
  double part = 0.0;
  for (int J = threadIdx.x; J < nb; J += blockDim.x) {
    const double len = static_cast<double>(block_len(J, N, B));
    double sc = mass[(size_t)(g * rep) * nb + J] / len;
    for (int r = 1; r < rep; ++r) sc += mass[(size_t)(g * rep + r) * nb + J] / len;
    S.score[J] = sc;
    gscores[(size_t)g * nb + J] = sc;
    part += len * sc;
  }
  __syncthreads();
  const double mean = block_reduce_sum(part, S.red) / static_cast<double>(N);
  double p2 = 0.0, p4 = 0.0;
  for (int J = threadIdx.x; J < nb; J += blockDim.x) {
    const double len = static_cast<double>(block_len(J, N, B));
    const double dv = S.score[J] - mean;
    const double d2 = dv * dv;
    p2 += len * d2;
    p4 += len * d2 * d2;
  }
  const double m2 = block_reduce_sum(p2, S.red) / static_cast<double>(N);
  const double m4 = block_reduce_sum(p4, S.red) / static_cast<double>(N);
  if (threadIdx.x == 0) S.kurt = (m2 == 0.0) ? 0.0 : m4 / (m2 * m2);
  // descending token-score order of this group (ties to the lower block)
  for (int J = threadIdx.x; J < nb; J += blockDim.x) S.pre[J] = -S.score[J];
  __syncthreads();
  rank_sort(S.pre, nb, S.skey, S.sidx);
  cluster_sync_all();  // kurtoses visible cluster-wide
  int flat = 0;
  {
    double best = 0.0;
    for (int q = 0; q < hkv; ++q) {
      const uint32_t a = mapa_shared(smem_u32(&S.kurt), (uint32_t)q);
      double kq;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(kq) : "r"(a) : "memory");
      if (q == 0 || kq < best) { best = kq; flat = q; }  // argmin, ties to the lowest index
    }
  }
  // budget on the flattest group (its CTA only), as in select_kernel phase 2
  if (g == flat) {
    if (budget_override > 0) {
      if (threadIdx.x == 0) { S.budget = budget_override; S.retained = 0.0; S.total = 0.0; }
    } else {
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        S.pre[i] = static_cast<double>(block_len(S.sidx[i], N, B)) * (-S.skey[i]);
        S.ipre[i] = block_len(S.sidx[i], N, B);
      }
      if (threadIdx.x == 0) S.cross = nb - 1;
      __syncthreads();
      block_inclusive_scan(S.pre, nb, S.wtot);
      block_inclusive_scan(S.ipre, nb, S.itot);
      const double total = S.pre[nb - 1];
      const double thr = fmin(p * total, total);
      for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (S.pre[i] >= thr) atomicMin(&S.cross, i);
      __syncthreads();
      if (threadIdx.x == 0) {
        const int i = S.cross;
        const double sv = -S.skey[i];
        const int len = block_len(S.sidx[i], N, B);
        const double C = i > 0 ? S.pre[i - 1] : 0.0;
        const int T = i > 0 ? S.ipre[i - 1] : 0;
        int k = len;
        if (sv > 0.0) {
          const double kk = ceil((thr - C) / sv);
          k = (kk < 1.0) ? 1 : (kk > len ? len : static_cast<int>(kk));
          while (k > 1 && C + static_cast<double>(k - 1) * sv >= thr) --k;
          while (k < len && C + static_cast<double>(k) * sv < thr) ++k;
        } else {
          k = 1;
        }
        S.budget = T + k;
        S.retained = C + static_cast<double>(k) * sv;
        S.total = total;
      }
    }
  }
  cluster_sync_all();  // budget visible cluster-wide
  const uint32_t fb = mapa_shared(smem_u32(&S.budget), (uint32_t)flat);
  int b = (int)ld_shared_cluster_u32(fb);
  const int span = (vision_limit >= 0) ? vision_limit : N;
  if (b > span) b = span;
  // this group's top-b block table -> ascending index list
  if (gran == OMNI_GRAN_BLOCK) {  // rank = per-token score x block length
    for (int J = threadIdx.x; J < nb; J += blockDim.x)
      S.pre[J] = -(S.score[J] * static_cast<double>(block_len(J, N, B)));
    __syncthreads();
    rank_sort(S.pre, nb, S.skey, S.sidx);
  }
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int lo = S.sidx[i] * B;
    S.ipre[i] = max(0, min(lo + block_len(S.sidx[i], N, B), span) - lo);  // vision-clipped length
    S.take[i] = 0;
  }
  __syncthreads();
  block_inclusive_scan(S.ipre, nb, S.itot);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int len = S.ipre[i] - (i > 0 ? S.ipre[i - 1] : 0);
    const int before = S.ipre[i] - len;
    S.take[S.sidx[i]] = max(0, min(len, b - before));  // whole blocks in rank order, marginal prefix
  }
  __syncthreads();
  for (int J = threadIdx.x; J < nb; J += blockDim.x) S.ipre[J] = S.take[J];
  __syncthreads();
  block_inclusive_scan(S.ipre, nb, S.itot);
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int J = warp; J < nb; J += nw) {
      const int t = S.take[J], off = S.ipre[J] - t;
      for (int k = lane; k < t; k += 32) selected[(size_t)g * N + off + k] = J * B + k;
    }
  }
  if (threadIdx.x == 0) {
    info[4 + g] = b;  // per-group selected counts (all equal: shared budget)
    stats[g] = S.kurt;
    if (g == 0) {
      info[0] = b;
      info[1] = flat;
      info[2] = hkv;
      info[3] = nb;
      double v;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa_shared(smem_u32(&S.retained), (uint32_t)flat)) : "memory");
      stats[hkv] = v;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa_shared(smem_u32(&S.total), (uint32_t)flat)) : "memory");
      stats[hkv + 1] = v;
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
}

}  // namespace omni

using namespace omni;

extern "C" size_t omni_probe_mass_workspace(int n_q_heads, int n_blocks) {
  return sizeof(double) * (size_t)n_q_heads * n_blocks * (n_blocks + 2);
}

// Materialising path (reference-named probe_attention needs the map): scores
// S [Hq, nb, nb] and row statistics [Hq, nb, 2] are left in the workspace.
extern "C" int omni_probe_mass_map(const double* pooled_q, const double* pooled_k, int n_q_heads, int n_kv_heads,
                                   int n_blocks, int head_dim, double* mass, void* workspace, void* stream) {
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim >= 1 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be in [1, 256]");
  OMNI_CHECK(n_blocks >= 1, OMNI_E_SHAPE, "no probe blocks");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* S = static_cast<double*>(workspace);
  double* st = S + (size_t)n_q_heads * n_blocks * n_blocks;
  const size_t shm = sizeof(double) * 48 * (head_dim + 1);
  if (shm > 48 * 1024)
    OMNI_CUDA_TRY(cudaFuncSetAttribute(probe_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  probe_scores_kernel<<<dim3((n_blocks + 15) / 16, n_q_heads), 256, shm, s>>>(pooled_q, pooled_k, n_blocks, head_dim,
                                                                            n_q_heads / n_kv_heads, S);
  probe_rowstats_kernel<<<dim3(n_blocks, n_q_heads), 32, 0, s>>>(S, n_blocks, st);
  probe_colsum_kernel<<<dim3((n_blocks + 31) / 32, n_q_heads), 256, 0, s>>>(S, st, n_blocks, mass);
  return omni_launch_check();
}

// Hot path: fused scores + statistics + partial column sums (d = 128,
// nb <= 512, i.e. up to 128K tokens at B = 256), else the materialising path.
extern "C" int omni_probe_mass(const double* pooled_q, const double* pooled_k, int n_q_heads, int n_kv_heads,
                               int n_blocks, int head_dim, double* mass, void* workspace, void* stream) {
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim >= 1 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be in [1, 256]");
  OMNI_CHECK(n_blocks >= 1, OMNI_E_SHAPE, "no probe blocks");
  if (head_dim != 128 || n_blocks > PF_MAXNB)
    return omni_probe_mass_map(pooled_q, pooled_k, n_q_heads, n_kv_heads, n_blocks, head_dim, mass, workspace, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int ntiles = (n_blocks + PF_ROWS - 1) / PF_ROWS;
  double* partial = static_cast<double*>(workspace);  // [Hq, ntiles, nb] <= [Hq, nb, nb + 2]
  const int shm = (int)sizeof(double) * ((PF_ROWS + 2 * PF_JT) * (128 + 2) + PF_ROWS * n_blocks);
  static int attr = 0;
  if (shm > attr) {
    OMNI_CUDA_TRY(cudaFuncSetAttribute(probe_mass_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    attr = shm;
  }
  probe_mass_fused_kernel<<<dim3(ntiles, n_q_heads), 256, shm, s>>>(pooled_q, pooled_k, n_blocks,
                                                                     n_q_heads / n_kv_heads, partial);
  probe_colsum_partials_kernel<<<dim3((n_blocks + 127) / 128, n_q_heads), 128, 0, s>>>(partial, n_blocks, ntiles,
                                                                                       mass);
  return omni_launch_check();
}

extern "C" int omni_select(const double* block_mass, int n_q_heads, int n_kv_heads, int seq_len, int block_size,
                           double p, int granularity, int vision_limit, int budget_override, int32_t* selected,
                           int32_t* info, double* stats, double* group_scores, void* stream) {
  OMNI_CHECK(p > 0.0 && p <= 1.0, OMNI_E_PARAM, "retention p must be in (0, 1]");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(n_kv_heads >= 1 && n_kv_heads <= 64 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE,
             "need 1 <= n_kv_heads <= 64 dividing n_q_heads");
  OMNI_CHECK(granularity == OMNI_GRAN_TOKEN || granularity == OMNI_GRAN_BLOCK, OMNI_E_PARAM, "granularity must be token or block");
  const int nb = (seq_len + block_size - 1) / block_size;
  OMNI_CHECK(nb >= 1 && nb <= kSelMaxBlocks, OMNI_E_PARAM, "selection supports at most 8192 probe blocks");
  OMNI_CHECK(vision_limit != 0, OMNI_E_PARAM, "vision span is empty");
  OMNI_CHECK(budget_override <= seq_len, OMNI_E_PARAM, "budget exceeds the sequence");
  OMNI_CHECK(group_scores != nullptr, OMNI_E_PARAM, "group_scores buffer required");
  if (n_kv_heads <= 8 && nb <= SC_MAXNB) {
    // one CTA per KV group in a cluster (distributed-shared-memory exchange)
    const size_t shm = sizeof(SelCl);
    OMNI_CUDA_TRY(cudaFuncSetAttribute(select_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_kv_heads);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = n_kv_heads;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    OMNI_CUDA_TRY(cudaLaunchKernelEx(&cfg, select_cluster_kernel, block_mass, n_q_heads, n_kv_heads, seq_len,
                                     block_size, p, granularity, vision_limit, budget_override, selected, info, stats,
                                     group_scores));
    return omni_launch_check();
  }
  const size_t shm = sizeof(SelShared);
  OMNI_CUDA_TRY(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  select_kernel<<<1, 1024, shm, static_cast<cudaStream_t>(stream)>>>(block_mass, n_q_heads, n_kv_heads, seq_len,
                                                                      block_size, p, granularity, vision_limit,
                                                                      budget_override, selected, info, stats,
                                                                      group_scores);
  return omni_launch_check();
}
