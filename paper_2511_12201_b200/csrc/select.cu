// K3: block-probe column mass (K3a) and shared-budget KV selection (K3b).
//
// K3a is the (N/B)^2 d probe of block_probe.py:44-64 in float64 — at 64K
// tokens that is 28 heads x 256 x 256 pooled scores, latency-bound (µs), not a
// roofline kernel. K3b is the selection: per-group token scores, kurtosis,
// argmin (flattest head), top-p budget on the flattest group and one top-b
// block table per group, written out as ascending index lists
// (kv_select.py:49-195); one cluster of Hkv CTAs on the hot path, a
// four-launch general path beyond it. Scores on the probe path are constant
// within a probe block, so every sort/scan runs over nb blocks instead of N
// tokens; block_size = 1 degenerates to the token-exact path.
#include <float.h>
#include <limits.h>

#include "common.cuh"

namespace omni {

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
  // heaviest row tiles (most visible key blocks) first across all heads: the
  // light tiles fill the tail of the launch (longest-processing-time order)
  const int hq = gridDim.y, ntiles = gridDim.x;
  const int t = ntiles - 1 - (int)((blockIdx.y * gridDim.x + blockIdx.x) / hq);
  const int h = (int)((blockIdx.y * gridDim.x + blockIdx.x) % hq), g = h / rep;
  const int I0 = t * PF_ROWS;
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
  double* out = partial + ((size_t)h * ntiles + t) * nb;
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
//
// Parity by construction. The reference decides the flattest group and the
// budget with float64 arithmetic in a fixed order; where its inputs are
// identical (the kv_select operators called on user vectors, the decode
// hand-off) the GPU reproduces that order bit for bit, and where it cannot
// afford to (a 64K-step serial cumsum) it proves the decision safe first:
//  * kurtosis (kv_select.py:49-53 -> _core_py.kurtosis, the NumPy backend the
//    golden fixtures pin): mu = v.mean(), m2 = mean(d*d), m4 = mean(d*d*d*d),
//    each mean a NumPy pairwise sum emulated exactly (np_pairwise_sum, every
//    op rounded individually, no FMA contraction) over the per-token vector;
//  * budget (kv_select.py:83-120): the block-wise scan C + k s finds the
//    crossing in parallel; when the distance of the two neighbouring
//    cumulative masses from the threshold is within a rigorous bound on the
//    rounding difference between that scan and the reference's sequential
//    np.cumsum of the sorted per-token vector ((4N + 16) u total), one thread
//    replays the reference's cumsum token by token and its b is used;
//  * block ranks (select_top_blocks, kv_select.py:160): np.add.reduceat
//    block sums of the per-token vector (first element + pairwise rest);
//  * argmin / lexsort tie rules as before (lowest group, lowest index).

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

// ------------------------------------------------------------ NumPy order
// numpy's pairwise summation (np.sum / np.mean of a contiguous float64
// vector; numpy/_core/src/umath/loops_utils.h.src, pairwise_sum): a run of
// n < 8 elements is summed sequentially from 0; a run of 8 <= n <= 128 with 8
// strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
// sequential tail; a longer run splits at n2 = n/2 - (n/2) % 8. The
// restatement was checked bit for bit against NumPy 2.3 np.sum for every
// length up to 300 and lengths up to 200000 (tests/test_oracle_golden.py).
constexpr int PW_LEAF = 128;

template <typename F>
__device__ double pw_leaf(const F& f, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, f(lo + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
  return res;
}

__host__ __device__ inline int pw_depth(int n) {
  // every node at depth D is a leaf: node sizes at depth d are at most
  // n / 2^d + 16 (a right child holds at most half its parent plus 8)
  int D = 0;
  while ((n >> D) + 16 > PW_LEAF) ++D;
  return D;
}

// One thread: pairwise sum of f(lo .. lo+n) (short runs: block sums).
template <typename F>
__device__ double pw_serial(const F& f, int lo, int n) {
  if (n <= PW_LEAF) return pw_leaf(f, lo, n);
  // explicit post-order over the split tree (depth <= 24)
  int st_lo[32], st_n[32], st_state[32];
  double st_val[32];
  int sp = 0;
  st_lo[0] = lo; st_n[0] = n; st_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int m = st_n[sp];
    if (m <= PW_LEAF) {
      ret = pw_leaf(f, st_lo[sp], m);
      --sp;
      continue;
    }
    const int h = m / 2, n2 = h - h % 8;
    if (st_state[sp] == 0) {         // descend left
      st_state[sp] = 1;
      st_lo[sp + 1] = st_lo[sp]; st_n[sp + 1] = n2; st_state[sp + 1] = 0;
      ++sp;
    } else if (st_state[sp] == 1) {  // left done: keep it, descend right
      st_val[sp] = ret;
      st_state[sp] = 2;
      st_lo[sp + 1] = st_lo[sp] + n2; st_n[sp + 1] = m - n2; st_state[sp + 1] = 0;
      ++sp;
    } else {                         // both done
      ret = __dadd_rn(st_val[sp], ret);
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat segment sum: out = a[lo] + pairwise(a[lo+1 .. lo+n)).
template <typename F>
__device__ double reduceat_sum(const F& f, int lo, int n) {
  if (n == 1) return f(lo);
  return __dadd_rn(f(lo), pw_serial(f, lo + 1, n - 1));
}

// Leaf of the pairwise sum over a block-constant vector v(t) = vals[t / B]:
// the elements are consumed in increasing t with a running block index, so
// the additions happen in exactly pw_leaf's order without a division per
// element.
__device__ __forceinline__ double pw_leaf_blocks(const double* vals, int B, int nb, int lo, int n) {
  int J = lo / B, rem = lo - J * B;
  double cur = vals[J];
  auto next = [&]() {
    const double v = cur;
    if (++rem == B) {
      rem = 0;
      if (++J < nb) cur = vals[J];
    }
    return v;
  };
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, next());
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = next();
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], next());
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, next());
  return res;
}

// CTA-wide pairwise sum of n elements whose leaf sums leaf(lo, m) computes:
// leaves in parallel (path p of the depth-D split tree; a leaf reached early
// is computed by the path whose remaining bits are zero and kept at slot p),
// then internal nodes bottom up (node (d, q) at slot q << (D - d), right child
// at (2q + 1) << (D - d - 1)). buf: 2^pw_depth(n) doubles. Every thread
// returns the sum.
template <typename Leaf>
__device__ double np_pairwise_sum(const Leaf& leaf, int n, double* buf) {
  const int D = pw_depth(n);
  const int L = 1 << D;
  for (int p = threadIdx.x; p < L; p += blockDim.x) {
    int lo = 0, m = n, d = 0;
    while (d < D && m > PW_LEAF) {
      const int h = m / 2, n2 = h - h % 8;
      if ((p >> (D - 1 - d)) & 1) { lo += n2; m -= n2; } else { m = n2; }
      ++d;
    }
    if ((p & ((1 << (D - d)) - 1)) == 0) buf[p] = leaf(lo, m);
  }
  __syncthreads();
  for (int d = D - 1; d >= 0; --d) {
    for (int q = threadIdx.x; q < (1 << d); q += blockDim.x) {
      int m = n;
      bool live = true;
      for (int e = 0; e < d; ++e) {
        if (m <= PW_LEAF) { live = false; break; }  // an ancestor is a leaf: no such node
        const int h = m / 2, n2 = h - h % 8;
        m = ((q >> (d - 1 - e)) & 1) ? m - n2 : n2;
      }
      if (live && m > PW_LEAF) {
        const int s = D - d;
        buf[q << s] = __dadd_rn(buf[q << s], buf[(2 * q + 1) << (s - 1)]);
      }
    }
    __syncthreads();
  }
  const double r = buf[0];
  __syncthreads();
  return r;
}

// _core_py.kurtosis (kv_select.py:49-53) of the per-token vector v(t) =
// score[t / B], t < N, in NumPy's order: mu = v.mean(), d = v - mu,
// m2 = mean(d * d), m4 = mean(d * d * d * d) (left to right), m4 / m2^2.
// d and its powers are per block (the same rounded value for every token of
// a block), staged in tmp[nb]; the means are pairwise sums over the tokens.
// CTA-wide; score / tmp in shared or global memory.
__device__ double kurtosis_np(const double* score, double* tmp, int N, int B, double* buf) {
  const int nb = (N + B - 1) / B;
  const double n = static_cast<double>(N);
  const double mu = __ddiv_rn(np_pairwise_sum([&](int lo, int m) { return pw_leaf_blocks(score, B, nb, lo, m); },
                                              N, buf), n);
  for (int J = threadIdx.x; J < nb; J += blockDim.x) {
    const double d = __dsub_rn(score[J], mu);
    tmp[J] = __dmul_rn(d, d);
  }
  __syncthreads();
  const double m2 = __ddiv_rn(np_pairwise_sum([&](int lo, int m) { return pw_leaf_blocks(tmp, B, nb, lo, m); },
                                              N, buf), n);
  if (m2 == 0.0) return 0.0;  // uniform across the CTA (every thread holds the same m2)
  for (int J = threadIdx.x; J < nb; J += blockDim.x) {
    const double d = __dsub_rn(score[J], mu);
    tmp[J] = __dmul_rn(__dmul_rn(__dmul_rn(d, d), d), d);
  }
  __syncthreads();
  const double m4 = __ddiv_rn(np_pairwise_sum([&](int lo, int m) { return pw_leaf_blocks(tmp, B, nb, lo, m); },
                                              N, buf), n);
  return __ddiv_rn(m4, __dmul_rn(m2, m2));
}

struct BudgetResult {
  int budget;
  double retained, total, margin;
  int replayed;
};

// Thread 0 after the parallel crossing search: the crossing lies in sorted
// block i (value s per token, len tokens, C = cumulative mass and T = tokens of
// the blocks before it). Finds k, checks the decision margin against the
// rounding bound and replays the reference's sequential cumsum when needed.
// sval(i) / slen(i): per-token value and token count of the i-th block in
// descending value order.
template <typename SV, typename SL>
__device__ BudgetResult budget_finish(const SV& sval, const SL& slen, int nb, int N, double p, int i, double C, int T,
                                      double total, double thr) {
  BudgetResult r;
  const double s = sval(i);
  const int len = slen(i);
  int k = len;
  if (s > 0.0) {
    const double kk = ceil((thr - C) / s);
    k = (kk < 1.0) ? 1 : (kk > len ? len : static_cast<int>(kk));
    while (k > 1 && C + static_cast<double>(k - 1) * s >= thr) --k;
    while (k < len && C + static_cast<double>(k) * s < thr) ++k;
  } else {
    k = 1;
  }
  r.budget = T + k;
  r.retained = C + static_cast<double>(k) * s;
  r.total = total;
  r.replayed = 0;
  const double hi = r.retained - thr;  // >= 0: the cumulative mass at b reaches thr
  const double lo = (r.budget == 1) ? INFINITY : thr - (k > 1 ? C + static_cast<double>(k - 1) * s : C);
  const double m = fmin(hi, lo);
  const double bound = 1.01 * (4.0 * static_cast<double>(N) + 16.0) * 1.1102230246251565e-16 * fabs(total);
  r.margin = total != 0.0 ? m / fabs(total) : 0.0;
  if (!(m > bound)) {
    // reference order (kv_select.py:83-84,116-119): cum = np.cumsum of the
    // descending per-token vector, thr = min(p * cum[-1], cum[-1]),
    // b = searchsorted(cum, thr, 'left') + 1, retained = cum[b - 1]
    double cum = 0.0;
    for (int j = 0; j < nb; ++j) {
      const double v = sval(j);
      for (int t = slen(j); t > 0; --t) cum = __dadd_rn(cum, v);
    }
    const double tot = cum;
    const double th = fmin(__dmul_rn(p, tot), tot);
    cum = 0.0;
    int cnt = 0;
    bool done = false;
    for (int j = 0; j < nb && !done; ++j) {
      const double v = sval(j);
      for (int t = slen(j); t > 0; --t) {
        cum = __dadd_rn(cum, v);
        ++cnt;
        if (cum >= th) { done = true; break; }
      }
    }
    r.budget = cnt;
    r.retained = cum;
    r.total = tot;
    r.replayed = 1;
  }
  return r;
}

// K3b, cluster variant (hot path: Hkv <= 8 groups, nb <= 1024 blocks, N <=
// 2^12 * 112 tokens). One CTA per KV group in a thread-block cluster:
// per-group scores, kurtosis and a one-pass rank sort run in parallel; the
// kurtoses and the flattest group's budget are exchanged through distributed
// shared memory with two cluster barriers (kv_select.py:49-195).
constexpr int SC_MAXNB = 1024;
constexpr int SC_PW = 4096;  // pairwise-sum slots: N <= 112 * 4096 tokens
struct SelCl {
  double score[SC_MAXNB];  // per-token score of each block (this group)
  double skey[SC_MAXNB];   // sorted keys (ascending -rank)
  int sidx[SC_MAXNB];      // sorted block ids
  double pre[SC_MAXNB];
  int ipre[SC_MAXNB];
  int take[SC_MAXNB];
  double pw[SC_PW];
  double wtot[32];
  int itot[32];
  double red[32];
  double kurt;
  int budget;
  double retained, total, margin;
  int replayed;
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

__device__ __forceinline__ double ld_cluster_f64(const double* local, uint32_t rank) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(mapa_shared(smem_u32(local), rank)) : "memory");
  return v;
}

// Per-token score of block J of group g: sum over the group's Q heads (in
// ascending head order) of block mass / block length (block_probe.py:76-77
// + rule-B composition).
__device__ __forceinline__ double group_token_score(const double* mass, int g, int rep, int nb, int J, int N, int B) {
  const double len = static_cast<double>(block_len(J, N, B));
  double sc = __ddiv_rn(mass[(size_t)(g * rep) * nb + J], len);
  for (int r = 1; r < rep; ++r) sc = __dadd_rn(sc, __ddiv_rn(mass[(size_t)(g * rep + r) * nb + J], len));
  return sc;
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
  for (int J = threadIdx.x; J < nb; J += blockDim.x) {
    const double sc = group_token_score(mass, g, rep, nb, J, N, B);
    S.score[J] = sc;
    gscores[(size_t)g * nb + J] = sc;
  }
  __syncthreads();
  const double kurt = kurtosis_np(S.score, S.pre, N, B, S.pw);
  if (threadIdx.x == 0) S.kurt = kurt;
  // descending token-score order of this group (ties to the lower block)
  for (int J = threadIdx.x; J < nb; J += blockDim.x) S.pre[J] = -S.score[J];
  __syncthreads();
  rank_sort(S.pre, nb, S.skey, S.sidx);
  cluster_sync_all();  // kurtoses visible cluster-wide
  int flat = 0;
  {
    double best = 0.0;
    for (int q = 0; q < hkv; ++q) {
      const double kq = ld_cluster_f64(&S.kurt, (uint32_t)q);
      if (q == 0 || kq < best) { best = kq; flat = q; }  // argmin, ties to the lowest index
    }
  }
  // budget on the flattest group (its CTA only)
  if (g == flat) {
    if (budget_override > 0) {
      if (threadIdx.x == 0) {
        S.budget = budget_override; S.retained = 0.0; S.total = 0.0; S.margin = 0.0; S.replayed = 0;
      }
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
        const BudgetResult r = budget_finish([&](int j) { return -S.skey[j]; },
                                             [&](int j) { return block_len(S.sidx[j], N, B); }, nb, N, p, i,
                                             i > 0 ? S.pre[i - 1] : 0.0, i > 0 ? S.ipre[i - 1] : 0, total, thr);
        S.budget = r.budget;
        S.retained = r.retained;
        S.total = r.total;
        S.margin = r.margin;
        S.replayed = r.replayed;
      }
    }
  }
  cluster_sync_all();  // budget visible cluster-wide
  int b = (int)ld_shared_cluster_u32(mapa_shared(smem_u32(&S.budget), (uint32_t)flat));
  const int span = (vision_limit >= 0) ? vision_limit : N;
  if (b > span) b = span;
  // this group's top-b block table -> ascending index list
  if (gran == OMNI_GRAN_BLOCK) {  // rank = np.add.reduceat block sum of the per-token vector
    for (int J = threadIdx.x; J < nb; J += blockDim.x) {
      const double s = S.score[J];
      S.pre[J] = -reduceat_sum([s](int) { return s; }, 0, block_len(J, N, B));
    }
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
      stats[hkv] = ld_cluster_f64(&S.retained, (uint32_t)flat);
      stats[hkv + 1] = ld_cluster_f64(&S.total, (uint32_t)flat);
      stats[hkv + 2] = ld_cluster_f64(&S.margin, (uint32_t)flat);
      stats[hkv + 3] = static_cast<double>(ld_shared_cluster_u32(mapa_shared(smem_u32(&S.replayed), (uint32_t)flat)));
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still read its shared memory
}

// ------------------------------------------------ K3b, general path
// Any Hkv (<= 64) and nb (token-level selection over long sequences, the
// exact score source at >= 32K): per-group scores + kurtosis (one CTA per
// group), a segmented bitonic sort of the per-group (key, block) pairs, the
// budget on the flattest group (one CTA, chunked scan + the same gate and
// replay), then per group the top-b table and its ascending index list (one
// CTA per group, chunked scans over global memory).
struct SelWs {
  int stride;        // npow2: sort rows padded to a power of two
  double* key_tok;   // [Hkv, stride] -score, sorted in place (ascending (key, id) = descending score)
  int* idx_tok;      // [Hkv, stride] block ids, permuted with the keys
  double* key_blk;   // [Hkv, stride] -reduceat block sum
  int* idx_blk;
  double* tmp;       // [Hkv, nb] kurtosis scratch
  int* take;         // [Hkv, nb] keys taken per block id
  int* rpre;         // [Hkv, nb] scan scratch
  double* pre;       // [nb]
  int* ipre;         // [nb]
};

// Segmented bitonic sort of (key, id) rows in ascending (key, id) order —
// a total order (ids are unique within a row), so the reference's
// lexsort((arange, -a)) order needs no stable sort. Rows are padded to a
// power of two with (+DBL_MAX, INT_MAX). Tiles of BS_T elements sort in
// shared memory; larger strides are global compare-exchange passes.
constexpr int BS_T = 2048;

__device__ __forceinline__ bool bs_gt(double ka, int ia, double kb, int ib) {
  return ka > kb || (ka == kb && ia > ib);
}

// kk == 0: sort every tile completely (stages 2 .. T); kk > 0: the strides
// j < T of stage kk.
__global__ void __launch_bounds__(1024) bsort_tile_kernel(double* __restrict__ key, int* __restrict__ idx,
                                                          int stride, int T, int kk) {
  __shared__ double sk[BS_T];
  __shared__ int si[BS_T];
  const int base = blockIdx.x * T;
  double* K = key + (size_t)blockIdx.y * stride;
  int* I = idx + (size_t)blockIdx.y * stride;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    sk[t] = K[base + t];
    si[t] = I[base + t];
  }
  __syncthreads();
  const int k0 = kk ? kk : 2, k1 = kk ? kk : T;
  for (int k = k0; k <= k1; k <<= 1) {
    for (int j = min(k, T) >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < T; t += blockDim.x) {
        const int l = t ^ j;
        if (l > t) {
          const bool up = ((base + t) & k) == 0;
          if (bs_gt(sk[t], si[t], sk[l], si[l]) == up) {
            const double kt = sk[t];
            const int it = si[t];
            sk[t] = sk[l]; si[t] = si[l];
            sk[l] = kt; si[l] = it;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    K[base + t] = sk[t];
    I[base + t] = si[t];
  }
}

__global__ void bsort_global_kernel(double* __restrict__ key, int* __restrict__ idx, int stride, int k, int j) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= stride) return;
  const int l = i ^ j;
  if (l <= i) return;
  double* K = key + (size_t)blockIdx.y * stride;
  int* I = idx + (size_t)blockIdx.y * stride;
  const bool up = (i & k) == 0;
  const double ki = K[i], kl = K[l];
  const int ii = I[i], il = I[l];
  if (bs_gt(ki, ii, kl, il) == up) {
    K[i] = kl; I[i] = il;
    K[l] = ki; I[l] = ii;
  }
}

static inline int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

static void seg_sort(double* key, int* idx, int rows, int stride, cudaStream_t st) {
  const int T = stride < BS_T ? stride : BS_T;
  bsort_tile_kernel<<<dim3(stride / T, rows), 1024, 0, st>>>(key, idx, stride, T, 0);
  for (int k = 2 * T; k <= stride; k <<= 1) {
    for (int j = k >> 1; j >= T; j >>= 1)
      bsort_global_kernel<<<dim3((stride + 255) / 256, rows), 256, 0, st>>>(key, idx, stride, k, j);
    bsort_tile_kernel<<<dim3(stride / T, rows), 1024, 0, st>>>(key, idx, stride, T, k);
  }
}

__global__ void __launch_bounds__(1024) sel_scores_kernel(const double* __restrict__ mass, int hq, int hkv, int N,
                                                          int B, int gran, double* __restrict__ gscores,
                                                          double* __restrict__ stats, SelWs ws) {
  extern __shared__ double pwbuf[];
  const int g = blockIdx.x, nb = (N + B - 1) / B, rep = hq / hkv;
  const size_t row = (size_t)g * ws.stride;
  for (int J = threadIdx.x; J < ws.stride; J += blockDim.x) {
    if (J < nb) {
      const double sc = group_token_score(mass, g, rep, nb, J, N, B);
      gscores[(size_t)g * nb + J] = sc;
      ws.key_tok[row + J] = -sc;
      ws.idx_tok[row + J] = J;
      if (gran == OMNI_GRAN_BLOCK) {
        ws.key_blk[row + J] = -reduceat_sum([sc](int) { return sc; }, 0, block_len(J, N, B));
        ws.idx_blk[row + J] = J;
      }
    } else {  // padding sorts last
      ws.key_tok[row + J] = DBL_MAX;
      ws.idx_tok[row + J] = INT_MAX;
      if (gran == OMNI_GRAN_BLOCK) {
        ws.key_blk[row + J] = DBL_MAX;
        ws.idx_blk[row + J] = INT_MAX;
      }
    }
  }
  __syncthreads();
  const double kurt = kurtosis_np(gscores + (size_t)g * nb, ws.tmp + (size_t)g * nb, N, B, pwbuf);
  if (threadIdx.x == 0) stats[g] = kurt;
}

// Chunked block-wide inclusive scan of f(0..n) into out (global), returning
// the total; 1024 elements per chunk, running carry.
template <typename T, typename F>
__device__ T chunked_scan(const F& f, int n, T* out, T* tot) {
  __shared__ T carry_s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) carry_s = T(0);
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const T x = i < n ? f(i) : T(0);
    T v = x;
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
    const T carry = carry_s;
    const T incl = carry + v + (warp > 0 ? tot[warp - 1] : T(0));
    if (i < n) out[i] = incl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = incl;
    __syncthreads();
  }
  const T r = carry_s;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024) sel_budget_kernel(int hkv, int N, int B, double p, int vision_limit,
                                                          int budget_override, int32_t* __restrict__ info,
                                                          double* __restrict__ stats, SelWs ws) {
  __shared__ double dtot[32];
  __shared__ int itot[32];
  __shared__ int cross;
  const int nb = (N + B - 1) / B;
  int flat = 0;
  for (int q = 1; q < hkv; ++q)
    if (stats[q] < stats[flat]) flat = q;  // argmin, ties to the lowest index
  BudgetResult r{budget_override, 0.0, 0.0, 0.0, 0};
  if (budget_override <= 0) {
    const double* sk = ws.key_tok + (size_t)flat * ws.stride;
    const int* si = ws.idx_tok + (size_t)flat * ws.stride;
    const double total = chunked_scan<double>(
        [&](int i) { return static_cast<double>(block_len(si[i], N, B)) * (-sk[i]); }, nb, ws.pre, dtot);
    chunked_scan<int>([&](int i) { return block_len(si[i], N, B); }, nb, ws.ipre, itot);
    const double thr = fmin(p * total, total);
    if (threadIdx.x == 0) cross = nb - 1;
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (ws.pre[i] >= thr) atomicMin(&cross, i);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int i = cross;
      r = budget_finish([&](int j) { return -sk[j]; }, [&](int j) { return block_len(si[j], N, B); }, nb, N, p, i,
                        i > 0 ? ws.pre[i - 1] : 0.0, i > 0 ? ws.ipre[i - 1] : 0, total, thr);
    }
  }
  if (threadIdx.x == 0) {
    const int span = (vision_limit >= 0) ? vision_limit : N;
    info[0] = min(r.budget, span);
    info[1] = flat;
    info[2] = hkv;
    info[3] = nb;
    stats[hkv] = r.retained;
    stats[hkv + 1] = r.total;
    stats[hkv + 2] = r.margin;
    stats[hkv + 3] = static_cast<double>(r.replayed);
  }
}

__global__ void __launch_bounds__(1024) sel_take_kernel(int N, int B, int gran, int vision_limit, int b_const,
                                                        int32_t* __restrict__ selected, int32_t* __restrict__ info,
                                                        SelWs ws) {
  __shared__ int itot[32];
  const int g = blockIdx.x, nb = (N + B - 1) / B;
  const int b = b_const > 0 ? b_const : info[0];
  const int span = (vision_limit >= 0) ? vision_limit : N;
  const int* si = (gran == OMNI_GRAN_BLOCK ? ws.idx_blk : ws.idx_tok) + (size_t)g * ws.stride;
  int* take = ws.take + (size_t)g * nb;  // per block id
  int* rpre = ws.rpre + (size_t)g * nb;  // scan scratch
  auto clen = [&](int i) {  // vision-clipped length of the i-th ranked block
    const int lo = si[i] * B;
    return max(0, min(lo + block_len(si[i], N, B), span) - lo);
  };
  // whole blocks in rank order, the marginal block's lowest indices
  chunked_scan<int>(clen, nb, rpre, itot);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const int len = clen(i);
    take[si[i]] = max(0, min(len, b - (rpre[i] - len)));
  }
  __syncthreads();
  // ascending index list: exclusive offsets over block ids
  chunked_scan<int>([&](int J) { return take[J]; }, nb, rpre, itot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int J = warp; J < nb; J += nw) {
    const int t = take[J], off = rpre[J] - t;
    for (int k = lane; k < t; k += 32) selected[(size_t)g * N + off + k] = J * B + k;
  }
  if (threadIdx.x == 0) info[4 + g] = b;
}

}  // namespace omni

namespace omni {

// np.add.reduceat(x[r], arange(0, n, block)) per row (select_top_blocks'
// block mass, kv_select.py:160; the exact-path block granularity).
__global__ void block_sums_kernel(const double* __restrict__ x, int n, int block, double* __restrict__ out) {
  const int r = blockIdx.y, nb = (n + block - 1) / block;
  const int J = blockIdx.x * blockDim.x + threadIdx.x;
  if (J >= nb) return;
  const double* row = x + (size_t)r * n;
  out[(size_t)r * nb + J] = reduceat_sum([row](int t) { return row[t]; }, J * block, block_len(J, n, block));
}

// The materialised BlockProbeMap (block_probe.py:60-63): map[h, I, J] =
// exp(S[I, J] - max_I) / sum_I for J <= I, 0 above the diagonal, from the
// scores and row statistics omni_probe_mass_map leaves in its workspace.
__global__ void probe_map_kernel(const double* __restrict__ S, const double* __restrict__ st, int nb,
                                 double* __restrict__ map) {
  const int I = blockIdx.x, h = blockIdx.y;
  const double* row = S + ((size_t)h * nb + I) * nb;
  const double mx = st[((size_t)h * nb + I) * 2], sum = st[((size_t)h * nb + I) * 2 + 1];
  double* out = map + ((size_t)h * nb + I) * nb;
  for (int J = threadIdx.x; J < nb; J += blockDim.x) out[J] = (J <= I) ? exp(row[J] - mx) / sum : 0.0;
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
  omni_begin();
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim >= 1 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be in [1, 256]");
  OMNI_CHECK(n_blocks >= 1, OMNI_E_SHAPE, "no probe blocks");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* S = static_cast<double*>(workspace);
  double* st = S + (size_t)n_q_heads * n_blocks * n_blocks;
  const size_t shm = sizeof(double) * 48 * (head_dim + 1);
  if (shm > 48 * 1024)
    OMNI_CUDA_TRY(omni_smem_attr(probe_scores_kernel, (int)shm));
  probe_scores_kernel<<<dim3((n_blocks + 15) / 16, n_q_heads), 256, shm, s>>>(pooled_q, pooled_k, n_blocks, head_dim,
                                                                            n_q_heads / n_kv_heads, S);
  probe_rowstats_kernel<<<dim3(n_blocks, n_q_heads), 32, 0, s>>>(S, n_blocks, st);
  probe_colsum_kernel<<<dim3((n_blocks + 31) / 32, n_q_heads), 256, 0, s>>>(S, st, n_blocks, mass);
  return omni_launch_check();
}

extern "C" int omni_probe_map(const void* workspace, int n_q_heads, int n_blocks, double* map, void* stream) {
  omni_begin();
  OMNI_CHECK(n_q_heads >= 1 && n_blocks >= 1, OMNI_E_SHAPE, "empty probe map");
  const double* S = static_cast<const double*>(workspace);
  const double* st = S + (size_t)n_q_heads * n_blocks * n_blocks;
  probe_map_kernel<<<dim3(n_blocks, n_q_heads), 128, 0, static_cast<cudaStream_t>(stream)>>>(S, st, n_blocks, map);
  return omni_launch_check();
}

// Hot path: fused scores + statistics + partial column sums (d = 128,
// nb <= 512, i.e. up to 128K tokens at B = 256), else the materialising path.
extern "C" int omni_probe_mass(const double* pooled_q, const double* pooled_k, int n_q_heads, int n_kv_heads,
                               int n_blocks, int head_dim, double* mass, void* workspace, void* stream) {
  omni_begin();
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(head_dim >= 1 && head_dim <= 256, OMNI_E_SHAPE, "head_dim must be in [1, 256]");
  OMNI_CHECK(n_blocks >= 1, OMNI_E_SHAPE, "no probe blocks");
  if (head_dim != 128 || n_blocks > PF_MAXNB)
    return omni_probe_mass_map(pooled_q, pooled_k, n_q_heads, n_kv_heads, n_blocks, head_dim, mass, workspace, stream);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int ntiles = (n_blocks + PF_ROWS - 1) / PF_ROWS;
  double* partial = static_cast<double*>(workspace);  // [Hq, ntiles, nb] <= [Hq, nb, nb + 2]
  const int shm = (int)sizeof(double) * ((PF_ROWS + 2 * PF_JT) * (128 + 2) + PF_ROWS * n_blocks);
  OMNI_CUDA_TRY(omni_smem_attr(probe_mass_fused_kernel,
                               (int)sizeof(double) * ((PF_ROWS + 2 * PF_JT) * (128 + 2) + PF_ROWS * PF_MAXNB)));
  probe_mass_fused_kernel<<<dim3(ntiles, n_q_heads), 256, shm, s>>>(pooled_q, pooled_k, n_blocks,
                                                                     n_q_heads / n_kv_heads, partial);
  probe_colsum_partials_kernel<<<dim3((n_blocks + 127) / 128, n_q_heads), 128, 0, s>>>(partial, n_blocks, ntiles,
                                                                                       mass);
  return omni_launch_check();
}

extern "C" int omni_block_sums(const double* x, int rows, int n, int block_size, double* out, void* stream) {
  omni_begin();
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(rows >= 0 && n >= 0, OMNI_E_SHAPE, "negative extent");
  if (rows == 0 || n == 0) return OMNI_OK;
  const int nb = (n + block_size - 1) / block_size;
  block_sums_kernel<<<dim3((nb + 127) / 128, rows), 128, 0, static_cast<cudaStream_t>(stream)>>>(x, n, block_size,
                                                                                                out);
  return omni_launch_check();
}

// ------------------------------------------------------------- K3b host side
static constexpr int kSelMaxTokens = PW_LEAF * (1 << 14) - 16 * (1 << 14);  // pairwise depth <= 14

static bool sel_cluster_ok(int n_kv_heads, int nb, int seq_len) {
  return n_kv_heads <= 8 && nb <= SC_MAXNB && (1 << pw_depth(seq_len)) <= SC_PW;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static SelWs sel_layout(void* base, int n_kv_heads, int nb, size_t* total) {
  SelWs w{};
  char* p = static_cast<char*>(base);
  size_t off = 0;
  w.stride = pow2_at_least(nb);
  const size_t hs = (size_t)n_kv_heads * w.stride, hn = (size_t)n_kv_heads * nb;
  auto take = [&](size_t bytes) { char* r = p ? p + off : nullptr; off += align256(bytes); return r; };
  w.key_tok = reinterpret_cast<double*>(take(hs * 8));
  w.idx_tok = reinterpret_cast<int*>(take(hs * 4));
  w.key_blk = reinterpret_cast<double*>(take(hs * 8));
  w.idx_blk = reinterpret_cast<int*>(take(hs * 4));
  w.tmp = reinterpret_cast<double*>(take(hn * 8));
  w.take = reinterpret_cast<int*>(take(hn * 4));
  w.rpre = reinterpret_cast<int*>(take(hn * 4));
  w.pre = reinterpret_cast<double*>(take((size_t)nb * 8));
  w.ipre = reinterpret_cast<int*>(take((size_t)nb * 4));
  if (total) *total = off;
  return w;
}

extern "C" size_t omni_select_workspace(int n_kv_heads, int seq_len, int block_size) {
  if (n_kv_heads < 1 || seq_len < 1 || block_size < 1) return 0;
  const int nb = (seq_len + block_size - 1) / block_size;
  if (sel_cluster_ok(n_kv_heads, nb, seq_len)) return 0;
  size_t total = 0;
  sel_layout(nullptr, n_kv_heads, nb, &total);
  return total;
}

extern "C" int omni_select_ex(const double* block_mass, int n_q_heads, int n_kv_heads, int seq_len, int block_size,
                              double p, int granularity, int vision_limit, int budget_override, int32_t* selected,
                              int32_t* info, double* stats, double* group_scores, void* workspace, void* stream) {
  omni_begin();
  OMNI_CHECK(p > 0.0 && p <= 1.0, OMNI_E_PARAM, "retention p must be in (0, 1]");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(n_kv_heads >= 1 && n_kv_heads <= 64 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE,
             "need 1 <= n_kv_heads <= 64 dividing n_q_heads");
  OMNI_CHECK(granularity == OMNI_GRAN_TOKEN || granularity == OMNI_GRAN_BLOCK, OMNI_E_PARAM, "granularity must be token or block");
  OMNI_CHECK(seq_len >= 1 && seq_len <= kSelMaxTokens, OMNI_E_PARAM, "selection supports 1 .. 1,835,008 tokens");
  const int nb = (seq_len + block_size - 1) / block_size;
  OMNI_CHECK(vision_limit != 0, OMNI_E_PARAM, "vision span is empty");
  OMNI_CHECK(budget_override <= seq_len, OMNI_E_PARAM, "budget exceeds the sequence");
  OMNI_CHECK(group_scores != nullptr, OMNI_E_PARAM, "group_scores buffer required");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (sel_cluster_ok(n_kv_heads, nb, seq_len)) {
    // one CTA per KV group in a cluster (distributed-shared-memory exchange)
    const size_t shm = sizeof(SelCl);
    OMNI_CUDA_TRY(omni_smem_attr(select_cluster_kernel, (int)shm));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_kv_heads);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = shm;
    cfg.stream = st;
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
  OMNI_CHECK(workspace != nullptr, OMNI_E_PARAM,
             "this selection (more than 8 KV groups or 1024 blocks) needs omni_select_workspace() bytes");
  SelWs ws = sel_layout(workspace, n_kv_heads, nb, nullptr);
  const int pw_bytes = (int)sizeof(double) << pw_depth(seq_len);
  OMNI_CUDA_TRY(omni_smem_attr(sel_scores_kernel, pw_bytes));
  sel_scores_kernel<<<n_kv_heads, 1024, pw_bytes, st>>>(block_mass, n_q_heads, n_kv_heads, seq_len, block_size,
                                                        granularity, group_scores, stats, ws);
  seg_sort(ws.key_tok, ws.idx_tok, n_kv_heads, ws.stride, st);
  if (granularity == OMNI_GRAN_BLOCK) seg_sort(ws.key_blk, ws.idx_blk, n_kv_heads, ws.stride, st);
  sel_budget_kernel<<<1, 1024, 0, st>>>(n_kv_heads, seq_len, block_size, p, vision_limit, budget_override, info,
                                        stats, ws);
  sel_take_kernel<<<n_kv_heads, 1024, 0, st>>>(seq_len, block_size, granularity, vision_limit, 0, selected, info,
                                                ws);
  return omni_launch_check();
}

namespace omni {
__global__ void top_blocks_keys_kernel(const double* __restrict__ block_mass, int groups, int nb,
                                       SelWs ws) {
  const int g = blockIdx.y, J = blockIdx.x * blockDim.x + threadIdx.x;
  if (J >= ws.stride) return;
  const size_t row = (size_t)g * ws.stride;
  ws.key_blk[row + J] = J < nb ? -block_mass[(size_t)g * nb + J] : DBL_MAX;
  ws.idx_blk[row + J] = J < nb ? J : INT_MAX;
}
}  // namespace omni

extern "C" size_t omni_top_blocks_workspace(int groups, int seq_len, int block_size) {
  if (groups < 1 || seq_len < 1 || block_size < 1) return 0;
  size_t total = 0;
  sel_layout(nullptr, groups, (seq_len + block_size - 1) / block_size, &total);
  return total;
}

extern "C" int omni_top_blocks(const double* block_mass, int groups, int seq_len, int block_size, int budget,
                               int32_t* selected, int32_t* info, void* workspace, void* stream) {
  omni_begin();
  OMNI_CHECK(groups >= 1 && seq_len >= 1, OMNI_E_SHAPE, "empty score rows");
  OMNI_CHECK(block_size >= 1, OMNI_E_PARAM, "block size must be >= 1");
  OMNI_CHECK(budget >= 1 && budget <= seq_len, OMNI_E_PARAM, "budget must be in [1, seq_len]");
  OMNI_CHECK(workspace != nullptr, OMNI_E_PARAM, "omni_top_blocks needs omni_top_blocks_workspace() bytes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = (seq_len + block_size - 1) / block_size;
  SelWs ws = sel_layout(workspace, groups, nb, nullptr);
  top_blocks_keys_kernel<<<dim3((ws.stride + 255) / 256, groups), 256, 0, st>>>(block_mass, groups, nb, ws);
  seg_sort(ws.key_blk, ws.idx_blk, groups, ws.stride, st);
  sel_take_kernel<<<groups, 1024, 0, st>>>(seq_len, block_size, OMNI_GRAN_BLOCK, -1, budget, selected, info, ws);
  return omni_launch_check();
}

extern "C" int omni_select(const double* block_mass, int n_q_heads, int n_kv_heads, int seq_len, int block_size,
                           double p, int granularity, int vision_limit, int budget_override, int32_t* selected,
                           int32_t* info, double* stats, double* group_scores, void* stream) {
  omni_begin();
  return omni_select_ex(block_mass, n_q_heads, n_kv_heads, seq_len, block_size, p, granularity, vision_limit,
                        budget_override, selected, info, stats, group_scores, nullptr, stream);
}
