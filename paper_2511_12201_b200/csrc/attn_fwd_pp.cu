// K4 (CTA-pair ping-pong variant, OMNI_FWD_IMPL=pp): the single-CTA kernel's
// two-Q-tile ping-pong and softmax organisation (attn_fwd.cu, fwd_tile) on a
// pair of SMs with tcgen05.mma.cta_group::2.
//
// Contract as sparse_head_attention (prefill.py:89-122), see attn_fwd.cu. A
// cluster of two CTAs owns 512 compacted rows of one Q head as two M = 256
// tiles (A = rows [0, 256), B = [256, 512)); CTA r holds rows [128 r, 128 r +
// 128) of each tile in its TMEM lanes and its shared memory. Every MMA is
// issued once, by the leader, for both SMs:
//   S_X = Q_X K_j^T : A = Q_X (each CTA's smem), B = K_j split by key (CTA r
//                     stages keys [64 r, 64 r + 64) of the tile)
//   O_X += P_X V_j  : A = P_X (TMEM), B = V_j split by column (CTA r stages
//                     d columns [64 r, 64 r + 64))
// so a K / V tile is fetched from L2 once per 256 rows of each tile and each
// SM's shared-memory operand traffic for S = Q K^T drops from 128 B/clk (A +
// B of an M = 128 SS MMA) to 96 B/clk. TMEM per CTA is the single-CTA
// kernel's: S_A | O_A | S_B | O_B. K / V rings are 4 stages of half tiles.
//
// Warp roles per CTA (576 threads): warp 0 TMA (its CTA's halves, completing
// on the leader's barriers), warp 1 TMEM allocation (pair) and, on the leader,
// the MMA issue schedule PV_A(j), QK_A(j+1), PV_B(j), QK_B(j+1); warps 2-17
// softmax exactly as fwd_tile (two warps per TMEM lane quarter and tile, 64
// key columns each, deferred agreement in FAST mode). "P ready" is one
// arrival per softmax warp of both CTAs on the leader's barrier.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace fwdpp {

constexpr int BM = 128, BN = 128, D = 128, NST = 4;
constexpr int NTHREADS = 576;
constexpr int HC = 64;
constexpr uint32_t ATOM = 128 * 128;     // 128 rows x 128 B swizzle atom (Q tile: two)
constexpr uint32_t TILE = 2 * ATOM;      // 128 x 128 bf16
constexpr uint32_t KATOM = 64 * 128;     // 64 rows x 128 B (K half tile: two)
constexpr uint32_t KH = 2 * KATOM;       // this CTA's half of a K tile (64 keys x 128 d)
constexpr uint32_t VH = BN * 64 * 2;     // this CTA's half of a V tile (128 keys x 64 d)
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = OFF_Q + 2 * TILE;
constexpr uint32_t OFF_V = OFF_K + NST * KH;
constexpr uint32_t OFF_BAR = OFF_V + NST * VH;
enum {
  B_QF = 0,             // [2] Q tile X in smem, both CTAs (leader; 2 x 256 thread arrivals)
  B_KF = 2,             // [NST] K stage full (leader; both CTAs' bytes)
  B_KE = 2 + NST,       // [NST] K stage free (both CTAs; pair commit)
  B_VF = 2 + 2 * NST,   // [NST]
  B_VE = 2 + 3 * NST,   // [NST]
  B_SF = 2 + 4 * NST,   // [2] S_X(j) ready (both CTAs; pair commit)
  B_PF = 4 + 4 * NST,   // [2] P_X(j) written in both CTAs (leader; 2 x 8 warp arrivals)
  B_PV = 6 + 4 * NST,   // [2] PV_X(j) done (both CTAs; pair commit)
  B_COUNT = 8 + 4 * NST
};
constexpr uint32_t OFF_MISC = OFF_BAR + 8 * B_COUNT;  // tmem slot, nt[2]
constexpr uint32_t SMEM_BYTES = OFF_MISC + 16 + 1024;
constexpr uint32_t TMEM_COLS = 512;
__device__ __forceinline__ uint32_t col_s(int x) { return 256u * x; }
__device__ __forceinline__ uint32_t col_o(int x) { return 256u * x + 128u; }
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

template <int POLY, bool FAST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
sparse_fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                     const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                     const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep, int N,
                     int cap, int sel_stride, int sink, __nv_bfloat16* __restrict__ O, float* __restrict__ lse,
                     int* __restrict__ status) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = blockIdx.x >> 1;
  const int h = cid % Hq;
  // heaviest (latest rows) 512-row groups first, counted down from the
  // largest active-row count over the heads (as fwd_tile)
  int cmax = 0;
  for (int k = threadIdx.x & 31; k < Hq; k += 32) cmax = max(cmax, __ldg(counts + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  const int quad = (cmax + 4 * BM - 1) / (4 * BM) - 1 - cid / Hq;
  const int cnt = __ldg(counts + h);
  const int qrow0 = quad * 4 * BM;
  if (quad < 0 || qrow0 >= cnt) return;  // both CTAs of the cluster take this branch together

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_MISC);
  int* s_nt = reinterpret_cast<int*>(smem + OFF_MISC + 4);
  __shared__ float s_xch[2][BM][2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;

  const int sidx = warp - 2;
  const int xs = sidx >> 3;
  const int hf = (sidx >> 2) & 1;
  const int is = (warp & 3) * 32 + lane;
  const int rbase = qrow0 + xs * 2 * BM + (int)rank * BM;  // this CTA's first row of tile xs
  const int nrows_s = min(BM, cnt - rbase);
  const bool rvalid = warp >= 2 && is < nrows_s;
  const int pos = rvalid ? __ldg(rows + (size_t)h * N + rbase + is) : 0;
  uint4 qv[8];
  if (warp >= 2) {
    const uint4* qrow = reinterpret_cast<const uint4*>(Q + ((size_t)h * N + pos) * D) + hf * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) qv[c] = rvalid ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
  }
  int vis = warp >= 2 ? count_le_warp(selg, nsel, pos, rvalid) : 0;
  if (!rvalid) vis = 0;
  if (warp >= 2 && hf == 0) {
    if (is == nrows_s - 1) s_nt[xs] = (vis + BN - 1) / BN;
    if (nrows_s <= 0 && is == 0) s_nt[xs] = 0;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    for (int x = 0; x < 2; ++x) {
      mbar_init(B(B_QF + x), 4 * BM);
      mbar_init(B(B_SF + x), 1);
      mbar_init(B(B_PF + x), 2 * 8);
      mbar_init(B(B_PV + x), 1);
    }
    for (int s = 0; s < NST; ++s) {
      mbar_init(B(B_KF + s), 1);
      mbar_init(B(B_KE + s), 1);
      mbar_init(B(B_VF + s), 1);
      mbar_init(B(B_VE + s), 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(smem_u32(tmem_slot), TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs; s_nt published
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // both CTAs run a tile's key tiles up to its last row over the pair
  const int ntA = max(s_nt[0], (int)ld_shared_cluster_u32(mapa_shared(smem_u32(s_nt), rank ^ 1u)));
  const int ntB = max(s_nt[1], (int)ld_shared_cluster_u32(mapa_shared(smem_u32(s_nt + 1), rank ^ 1u)));
  const int ntm = max(ntA, ntB);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0 && ntm > 0) {
      const int kr0 = g * cap;
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NST;
        const uint32_t ph = ((j / NST) - 1) & 1;
        if (j >= NST) mbar_wait(B(B_KE + s), ph);
        if (leader) mbar_expect_tx(B(B_KF + s), 2 * KH);
        const int krow = kr0 + j * BN + (int)rank * 64;
        tma_load_2d_pair(sbase + OFF_K + s * KH, &tm_k, B(B_KF + s), 0, krow);
        tma_load_2d_pair(sbase + OFF_K + s * KH + KATOM, &tm_k, B(B_KF + s), 64, krow);
        if (j >= NST) mbar_wait(B(B_VE + s), ph);
        if (leader) mbar_expect_tx(B(B_VF + s), 2 * VH);
        tma_load_2d_pair(sbase + OFF_V + s * VH, &tm_v, B(B_VF + s), (int)rank * 64, kr0 + j * BN);
      }
      for (int j = ntm > NST ? ntm - NST : 0; j < ntm; ++j) {
        mbar_wait(B(B_KE + j % NST), (j / NST) & 1);
        mbar_wait(B(B_VE + j % NST), (j / NST) & 1);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer (leader)
    if (leader && ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(2 * BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(2 * BM, D, 0, 1);
      const int nt[2] = {ntA, ntB};
      const uint64_t dq0 = sdesc_sw128(sbase + OFF_Q, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, 16, 1024);
      auto qk = [&](int x, int j) {  // S_X(j) = Q_X K_j^T
        const uint64_t qd = dq0 + ((x * TILE) >> 4), kd = dk0 + (((j % NST) * KH) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offq = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          const uint32_t offk = ((kk >> 2) * KATOM + (kk & 3) * 32) >> 4;
          umma_pair_ss_ws(tmem + col_s(x), qd + offq, kd + offk, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_pair_ws(B(B_SF + x));
      };
      mbar_wait(B(B_KF), 0);
      for (int x = 0; x < 2; ++x) {
        if (nt[x] == 0) continue;
        mbar_wait_cluster(B(B_QF + x), 0);  // Q_X in both CTAs' smem
        tc_fence_after();
        qk(x, 0);
      }
      umma_commit_pair_ws(B(B_KE + 0));
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NST;
        mbar_wait(B(B_VF + s), (j / NST) & 1);
        bool kwaited = false;
        const uint64_t vd = dv0 + ((s * VH) >> 4);
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          mbar_wait_cluster(B(B_PF + x), j & 1);  // P_X(j) written (and O_X corrected) in both CTAs
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_pair_ts_ws(tmem + col_o(x), tmem + col_s(x) + (kk >> 2) * HC + (kk & 3) * 8,
                            vd + ((kk * 2048) >> 4), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit_pair_ws(B(B_PV + x));
          if (j + 1 < nt[x]) {
            if (!kwaited) {
              mbar_wait(B(B_KF + (j + 1) % NST), ((j + 1) / NST) & 1);
              tc_fence_after();
              kwaited = true;
            }
            qk(x, j + 1);
          }
        }
        umma_commit_pair_ws(B(B_VE + s));
        if (kwaited) umma_commit_pair_ws(B(B_KE + (j + 1) % NST));
      }
    }
  } else {
    // ------------------------------------------------------ softmax warps (fwd_tile's)
    const int x = xs;
    const int quarter = warp & 3;
    const int i = is;
    const int cb = hf * HC;
    const uint32_t bid = 1 + x * 4 + quarter;
    const int nt = x ? ntB : ntA;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t pf_bar = mapa_shared(B(B_PF + x), 0);
    const uint32_t qf_bar = mapa_shared(B(B_QF + x), 0);
    auto arrive_p = [&]() {  // one arrival per warp on the leader's barrier (TMEM stores complete)
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(B(B_PF + x)); else mbar_arrive_cluster_relaxed(pf_bar);
      }
    };
    float m_run = -INFINITY, l_run = 0.f;
    float pend_alpha = 1.f;
    if (nt > 0) {
      uint8_t* q_gen = smem + OFF_Q + x * TILE + hf * ATOM;
#pragma unroll
      for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(q_gen + swz(i, c)) = qv[c];
      fence_proxy_async_smem();
      mbar_arrive_cluster(qf_bar);

      const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
      const Exp2PolyConsts pc = exp2_poly_consts();
      for (int j = 0; j < nt; ++j) {
        mbar_wait(B(B_SF + x), j & 1);
        if (j > 0) mbar_wait(B(B_PV + x), (j - 1) & 1);
        tc_fence_after();
        if constexpr (POLY < 0) {
          tc_fence_before();
          arrive_p();
          l_run = 1.f;
          continue;
        }
        const int lim_row = vis - j * BN;
        const int lim = lim_row - cb;
        const bool full = __all_sync(0xffffffffu, lim >= HC);
        auto exps = [&](auto full_c, const uint32_t* sr, float nmu, uint32_t* pk) -> float {
          constexpr bool FULL = decltype(full_c)::value;
          const uint64_t c2 = f32x2(sl2, sl2), n2 = f32x2(nmu, nmu);
          uint64_t acc0 = f32x2(0.f, 0.f), acc1 = f32x2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const uint64_t xx = ffma2(f32x2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), c2, n2);
            uint64_t pp;
            if (FULL && use_poly<POLY>(c >> 1)) {
              pp = exp2_poly2_pair(xx, pc);
            } else {
              pp = f32x2(fast_exp2(f32x2_lo(xx)), fast_exp2(f32x2_hi(xx)));
            }
            if ((c & 2) == 0) acc0 = fadd2(acc0, pp); else acc1 = fadd2(acc1, pp);
            pk[c >> 1] = pack_bf16x2(f32x2_lo(pp), f32x2_hi(pp));
          }
          const uint64_t acc = fadd2(acc0, acc1);
          return f32x2_lo(acc) + f32x2_hi(acc);
        };
        auto chunk = [&](int q, float& m_cur, float& cmax, float& mu) -> float {
          uint32_t sr[32], pk[16];
          __syncwarp();
          tmem_ld32(tl + col_s(x) + cb + q * 32, sr);
          tmem_wait_ld();
          if (!full) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
          }
          float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            m0 = fmax3(m0, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
            m1 = fmax3(m1, __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
          }
          float rs = full ? exps(std::true_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk)
                          : exps(std::false_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk);
          const float cm = fmaxf(m0, m1) * sl2;
          cmax = fmaxf(cmax, cm);
          const bool hard = cm > m_cur + 64.0f;
          if (__any_sync(0xffffffffu, hard)) {
            if (hard) m_cur = ceilf(cm);
            rs = full ? exps(std::true_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk)
                      : exps(std::false_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk);
          }
          mu = m_cur;
          tmem_st16(tl + col_s(x) + cb + q * 16, pk);
          return rs;
        };
        auto chunk_fast = [&](int q, float m_cur) -> float {
          uint32_t sr[32], pk[16];
          __syncwarp();
          tmem_ld32(tl + col_s(x) + cb + q * 32, sr);
          tmem_wait_ld();
          if (!full) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
          }
          const float rs = full ? exps(std::true_type{}, sr, -m_cur, pk) : exps(std::false_type{}, sr, -m_cur, pk);
          tmem_st16(tl + col_s(x) + cb + q * 16, pk);
          return rs;
        };
        if constexpr (FAST) {
          if (__any_sync(0xffffffffu, pend_alpha != 1.f)) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t o[32];
              __syncwarp();
              tmem_ld32(tl + col_o(x) + cb + q * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * pend_alpha);
              tmem_st32(tl + col_o(x) + cb + q * 32, o);
            }
            pend_alpha = 1.f;
          }
          if (!__any_sync(0xffffffffu, m_run == -INFINITY && lim_row > 0)) {
            const float rs = chunk_fast(0, m_run) + chunk_fast(1, m_run);
            tmem_wait_st();
            tc_fence_before();
            arrive_p();
            if (m_run != -INFINITY && !(rs <= 0x1p64f)) atomicExch(status, 1);
            const float tgt = (m_run != -INFINITY && rs > 256.f) ? m_run + ceilf(__log2f(rs)) : m_run;
            if (named_bar_red_or(bid, 2 * 32, tgt != m_run)) {
              s_xch[x][i][hf] = tgt;
              named_bar_sync(bid, 2 * 32);
              const float m_fin = fmaxf(tgt, s_xch[x][i][hf ^ 1]);
              named_bar_sync(bid, 2 * 32);
              const float alpha = pow2_int(m_run - m_fin);
              l_run = (l_run + rs) * alpha;
              pend_alpha = alpha;
              m_run = m_fin;
            } else {
              l_run += rs;
            }
            continue;
          }
        }
        float m_cur = m_run, cmax = -INFINITY, mu0, mu1;
        const float rs0 = chunk(0, m_cur, cmax, mu0);
        const float rs1 = chunk(1, m_cur, cmax, mu1);
        const float tgt = cmax > mu1 + 8.0f ? ceilf(cmax) : mu1;
        if (named_bar_red_or(bid, 2 * 32, tgt != m_run)) {
          s_xch[x][i][hf] = tgt;
          named_bar_sync(bid, 2 * 32);
          const float m_fin = fmaxf(tgt, s_xch[x][i][hf ^ 1]);
          named_bar_sync(bid, 2 * 32);
          float f0 = 1.f, f1 = 1.f, alpha = 1.f;
          if (m_fin != -INFINITY) {
            f0 = pow2_int(mu0 - m_fin);
            f1 = pow2_int(mu1 - m_fin);
            alpha = pow2_int(m_run - m_fin);
          }
          l_run = l_run * alpha + rs0 * f0 + rs1 * f1;
          m_run = m_fin;
          if (__any_sync(0xffffffffu, f0 != 1.f)) {
            uint32_t pw[32];
            tmem_wait_st();
            __syncwarp();
            tmem_ld32(tl + col_s(x) + cb, pw);
            tmem_wait_ld();
            const uint32_t a0 = pack_bf16x2(f0, f0), a1 = pack_bf16x2(f1, f1);
#pragma unroll
            for (int c = 0; c < 16; ++c) pw[c] = mul_bf16x2(pw[c], a0);
#pragma unroll
            for (int c = 16; c < 32; ++c) pw[c] = mul_bf16x2(pw[c], a1);
            tmem_st32(tl + col_s(x) + cb, pw);
          }
          if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t o[32];
              __syncwarp();
              tmem_ld32(tl + col_o(x) + cb + q * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              tmem_st32(tl + col_o(x) + cb + q * 32, o);
            }
          }
        } else {
          l_run += rs0 + rs1;
        }
        tmem_wait_st();
        tc_fence_before();
        arrive_p();
      }
      mbar_wait(B(B_PV + x), (nt - 1) & 1);
      tc_fence_after();
      s_xch[x][i][hf] = l_run;
      named_bar_sync(bid, 2 * 32);
      l_run += s_xch[x][i][hf ^ 1];
    }
    // ------------------------------------------------------ epilogue
    uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)h * N + pos) * D + cb);
    if (nt > 0) {
      const float inv = l_run > 0.f ? pend_alpha / l_run : 0.f;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t o[32];
        __syncwarp();
        tmem_ld32(tl + col_o(x) + cb + q * 32, o);
        tmem_wait_ld();
        if (rvalid && l_run > 0.f) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float* f = reinterpret_cast<const float*>(o + 8 * c);
            dst[q * 4 + c] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                                        pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
          }
        }
      }
    }
    if (rvalid) {
      if (l_run > 0.f) {
        if (lse && hf == 0) lse[(size_t)h * N + pos] = static_cast<float>(M_LN2) * (m_run + log2f(l_run));
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(Vorig + ((size_t)g * N + sink) * D + cb);
#pragma unroll
        for (int c = 0; c < 8; ++c) dst[c] = __ldg(src + c);
        if (lse && hf == 0) lse[(size_t)h * N + pos] = -INFINITY;
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, TMEM_COLS);
  }
}

}  // namespace fwdpp
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

// Called by omni_sparse_attn_fwd_ex (attn_fwd.cu) after argument validation.
// status != nullptr: the FAST kernel (the caller launches the safe single-CTA
// redo behind it); else the safe kernel.
int omni_sparse_attn_fwd_pp(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream) {
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 64);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwdpp::BN);
  if (st) return st;
  const bool fast = status != nullptr;
  auto kern = poly == -1 ? fwdpp::sparse_fwd_pp_kernel<-1, false>
            : fast ? (poly == 4 ? fwdpp::sparse_fwd_pp_kernel<4, true> : fwdpp::sparse_fwd_pp_kernel<6, true>)
                   : (poly == 4 ? fwdpp::sparse_fwd_pp_kernel<4, false> : fwdpp::sparse_fwd_pp_kernel<6, false>);
  OMNI_CUDA_TRY(omni_smem_attr(kern, (int)fwdpp::SMEM_BYTES));
  const int n_quads = (seq_len + 4 * fwdpp::BM - 1) / (4 * fwdpp::BM);
  dim3 grid(2 * n_quads * n_q_heads);
  kern<<<grid, fwdpp::NTHREADS, fwdpp::SMEM_BYTES, stream>>>(
      tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
      sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index,
      static_cast<__nv_bfloat16*>(O), lse, status);
  return omni_launch_check();
}
