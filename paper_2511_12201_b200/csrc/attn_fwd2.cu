// K4 (CTA-pair variant): gathered sparse flash-attention forward on a pair of
// SMs with tcgen05.mma.cta_group::2 — the default forward kernel.
//
// Same contract as the single-CTA kernel in attn_fwd.cu (sparse_head_attention,
// prefill.py:89-122: row rows[h, i] attends to the selected keys j with
// selected[g, j] <= rows[h, i], softmax renormalised, V[sink] for rows with no
// visible key). What changes is the pipeline shape:
//
// * A cluster of two CTAs owns 256 compacted rows of one Q head; each CTA
//   holds 128 of them. Every MMA is M = 256 (one 128-row half per SM) and each
//   SM stages only HALF of every K / V tile (the B operand is split across the
//   pair), so a K/V tile read from L2 serves 256 query rows while each SM's
//   shared-memory operand traffic stays at ~64 B/clk.
// * Q lives in TMEM (A operand of S = Q K^T, TS mode), written straight from
//   registers; P is written over its own S columns (A operand of O += P V).
// * TMEM per CTA: Q [0, 64) | S buffer 0 [128, 256) | S buffer 1 [256, 384) |
//   O [384, 512). With S double-buffered, QK(j+2) is computed while the
//   softmax of tile j+1 runs, so the softmax of consecutive key tiles runs
//   back to back and the tensor core only waits for P (one tile per CTA; no
//   ping-pong between two Q tiles is needed).
//
// Warp roles (576 threads per CTA):
//   warp 0      TMA producer (both CTAs): this CTA's halves of K_j (64 keys x
//               128 d) and V_j (128 keys x 64 d) into NS-stage rings; the
//               transaction bytes complete on the leader's barriers.
//   warp 1      TMEM allocator (both CTAs); MMA issuer (leader only).
//   warps 2-17  softmax: four warps per TMEM lane quarter, each owning 32 key
//               columns of its 32 rows (thread <-> row <-> lane). Integral
//               running max shared by a row's four threads; optimistic
//               exponentials against it; one OR-barrier per quarter settles
//               the rare growth beyond 2^8 (exact power-of-two rescale of P,
//               l and O).
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace omni {
namespace fwd2 {

constexpr int BM = 128;   // rows per CTA (256 per pair)
constexpr int BN = 128;   // keys per tile
constexpr int D = 128;
constexpr int NS = 4;     // K / V ring stages
constexpr int CW = 32;    // key columns per softmax thread
constexpr int NTHREADS = 576;
constexpr uint32_t KH = 64 * D * 2;    // this CTA's half of a K tile (64 keys x 128 d), bytes
constexpr uint32_t VH = BN * 64 * 2;   // this CTA's half of a V tile (128 keys x 64 d), bytes
constexpr uint32_t KATOM = 64 * 128;   // 64 rows x 128 B swizzle atom (K half tile: two of them)
constexpr uint32_t OFF_K = 0;
constexpr uint32_t OFF_V = OFF_K + NS * KH;
constexpr uint32_t OFF_BAR = OFF_V + NS * VH;
enum {
  B_KF = 0,            // [NS] K stage full (leader; both CTAs' bytes)
  B_KE = NS,           // [NS] K stage free (both CTAs; pair commit)
  B_VF = 2 * NS,       // [NS]
  B_VE = 3 * NS,       // [NS]
  B_SF = 4 * NS,       // [2] S buffer ready (both CTAs; pair commit)
  B_PF = 4 * NS + 2,   // [2] P of tile j written, by j & 1 (leader; 32 warp arrivals). Two
                       // barriers: a fast warp may already arrive for tile j+1 (its S is
                       // double-buffered) before every warp has arrived for tile j.
  B_QF = 4 * NS + 4,   // Q in TMEM (leader; 32 warp arrivals)
  B_PVD = 4 * NS + 5,  // PV of the current tile done (both CTAs; pair commit)
  B_OD = 4 * NS + 6,   // last PV done: O final (both CTAs; pair commit)
  B_COUNT = 4 * NS + 7
};
constexpr uint32_t OFF_MISC = OFF_BAR + 8 * B_COUNT;  // tmem slot, nt
constexpr uint32_t SMEM_BYTES = OFF_MISC + 16 + 1024;  // + alignment slack
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_Q = 0, COL_S = 128, COL_O = 384;
constexpr int SOFT_WARPS_PER_CTA = 16;

// POLY: exponential pairs per 16 on the FMA-pipe polynomial (full tiles only).
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

// Profiling-only cycle accounting (OMNI_FWD_TRACE=1): leader MMA warp waits on
// P / V / K, its issue time, the key-tile steps, softmax S-waits and busy time.
__device__ unsigned long long g_trace[8];

template <int POLY, int TRACE = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
sparse_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                       const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                       const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                       const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep,
                       int N, int cap, int sel_stride, int sink, int n_pairs_per_head, __nv_bfloat16* __restrict__ O,
                       float* __restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ float s_xch[BM][4];  // per (row, column quarter): maxima, then partial sums
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int h = pair % Hq;
  const int tile = n_pairs_per_head - 1 - pair / Hq;  // heaviest (latest rows) pairs first
  const int cnt = __ldg(counts + h);
  const int prow0 = tile * 2 * BM;
  if (prow0 >= cnt) return;  // both CTAs of the pair take this branch together
  const int row0 = prow0 + (int)rank * BM;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_MISC);
  int* s_nt = reinterpret_cast<int*>(smem + OFF_MISC + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;
  const int nrows = min(BM, cnt - row0);  // may be <= 0 for the second CTA of the last pair

  // Softmax threads: row, visible-key count and this thread's 32 Q columns,
  // fetched before the barriers; the owner of the CTA's last row publishes its
  // key-tile count.
  const int sidx = warp - 2;
  const int cc = sidx >> 2;                 // column quarter 0..3
  const int quarter = warp & 3;             // TMEM lane quarter
  const int i = quarter * 32 + lane;        // row within the CTA tile == TMEM lane
  const bool rvalid = warp >= 2 && i < nrows;
  const int pos = rvalid ? __ldg(rows + (size_t)h * N + row0 + i) : 0;
  uint4 qv[4];
  if (warp >= 2) {
    const uint4* qrow = reinterpret_cast<const uint4*>(Q + ((size_t)h * N + pos) * D) + cc * 4;
#pragma unroll
    for (int c = 0; c < 4; ++c) qv[c] = rvalid ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
  }
  int vis = warp >= 2 ? count_le_warp(selg, nsel, pos, rvalid) : 0;
  if (!rvalid) vis = 0;
  if (warp >= 2 && cc == 0) {
    if (i == nrows - 1) *s_nt = (vis + BN - 1) / BN;
    if (nrows <= 0 && i == 0) *s_nt = 0;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    for (int s = 0; s < NS; ++s) {
      mbar_init(B(B_KF + s), 1);
      mbar_init(B(B_KE + s), 1);
      mbar_init(B(B_VF + s), 1);
      mbar_init(B(B_VE + s), 1);
    }
    mbar_init(B(B_SF + 0), 1);
    mbar_init(B(B_SF + 1), 1);
    mbar_init(B(B_PF + 0), 2 * SOFT_WARPS_PER_CTA);
    mbar_init(B(B_PF + 1), 2 * SOFT_WARPS_PER_CTA);
    mbar_init(B(B_QF), 2 * SOFT_WARPS_PER_CTA);
    mbar_init(B(B_PVD), 1);
    mbar_init(B(B_OD), 1);
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
  const int nt_own = *s_nt;
  const int nt_peer = (int)ld_shared_cluster_u32(mapa_shared(smem_u32(s_nt), rank ^ 1u));
  const int ntm = max(nt_own, nt_peer);  // both CTAs run the same number of key tiles

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0 && ntm > 0) {
      const int kr0 = g * cap;
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NS;
        const uint32_t ph = ((j / NS) - 1) & 1;
        if (j >= NS) mbar_wait(B(B_KE + s), ph);
        if (leader) mbar_expect_tx(B(B_KF + s), 2 * KH);
        const int krow = kr0 + j * BN + (int)rank * 64;
        tma_load_2d_pair(sbase + OFF_K + s * KH, &tm_k, B(B_KF + s), 0, krow);
        tma_load_2d_pair(sbase + OFF_K + s * KH + KATOM, &tm_k, B(B_KF + s), 64, krow);
        if (j >= NS) mbar_wait(B(B_VE + s), ph);
        if (leader) mbar_expect_tx(B(B_VF + s), 2 * VH);
        tma_load_2d_pair(sbase + OFF_V + s * VH, &tm_v, B(B_VF + s), (int)rank * 64, kr0 + j * BN);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer (leader)
    if (leader && ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(2 * BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(2 * BM, D, 0, 1);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, 16, 1024);
      uint32_t tw[4] = {0, 0, 0, 0};
      auto timed = [&](int k, auto&& fn) {
        if constexpr ((TRACE & 5) != 0) {
          const uint32_t t0 = clock();
          fn();
          tw[k] += clock() - t0;
        } else {
          fn();
        }
      };
      auto qk = [&](int jj) {  // S[jj & 1] = Q K_jj^T (A = Q from TMEM)
        const int s = jj % NS;
        timed(2, [&] { mbar_wait(B(B_KF + s), (jj / NS) & 1); });
        tc_fence_after();
        const uint64_t kd = dk0 + ((s * KH) >> 4);
        const uint32_t sc = tmem + COL_S + 128u * (jj & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * KATOM + (kk & 3) * 32) >> 4;
          umma_pair_ts_ws(sc, tmem + COL_Q + kk * 8, kd + off, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_pair_ws(B(B_KE + s));
        umma_commit_pair_ws(B(B_SF + (jj & 1)));
      };
      mbar_wait_cluster(B(B_QF), 0);  // Q of both CTAs in TMEM
      tc_fence_after();
      qk(0);
      if (ntm > 1) qk(1);
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NS;
        timed(0, [&] { mbar_wait_cluster(B(B_PF + (j & 1)), (j >> 1) & 1); });  // P_j of both CTAs (and O rescaled)
        timed(1, [&] { mbar_wait(B(B_VF + s), (j / NS) & 1); });
        tc_fence_after();
        const uint64_t vd = dv0 + ((s * VH) >> 4);
        const uint32_t pc = tmem + COL_S + 128u * (j & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_pair_ts_ws(tmem + COL_O, pc + 32u * (kk >> 1) + 8u * (kk & 1), vd + ((kk * 2048) >> 4), idesc_pv,
                          (j > 0 || kk > 0) ? 1u : 0u);
        umma_commit_pair_ws(B(B_VE + s));
        umma_commit_pair_ws(B(B_PVD));
        if (j + 1 == ntm) umma_commit_pair_ws(B(B_OD));
        if (j + 2 < ntm) qk(j + 2);  // reuses S[j & 1] after PV_j (in order in the tensor pipe)
      }
      if constexpr ((TRACE & 1) != 0) {
        if (lane == 0) {
          for (int k = 0; k < 3; ++k) atomicAdd(&g_trace[k], (unsigned long long)tw[k]);
          atomicAdd(&g_trace[4], (unsigned long long)ntm);
        }
      }
    }
  } else {
    // ------------------------------------------------------ softmax warps
    const uint32_t bid = 1 + quarter;          // named barrier of the four threads of these rows
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    const int cb = cc * CW;                    // first key column of this thread
    const uint32_t pf_bar0 = leader ? B(B_PF) : mapa_shared(B(B_PF), 0);
    const uint32_t qf_bar = leader ? B(B_QF) : mapa_shared(B(B_QF), 0);
    auto warp_arrive = [&](uint32_t b) {  // one arrival per warp on the leader's barrier
      __syncwarp();
      if (lane == 0) {
        // the TMEM writes being signalled are complete (tcgen05.wait::st):
        // a relaxed remote arrive avoids a cluster-scope release per step
        if (leader) mbar_arrive(b); else mbar_arrive_cluster_relaxed(b);
      }
    };
    float m_run = -INFINITY, l_run = 0.f;
    if (ntm > 0) {
      // Q columns [cb, cb + 32) of this row -> TMEM (bf16 pairs, A operand of QK).
      {
        const uint32_t* qw = reinterpret_cast<const uint32_t*>(qv);
        uint32_t qr[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) qr[c] = qw[c];
        __syncwarp();
        tmem_st16(tl + COL_Q + cc * 16, qr);
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(qf_bar);
      }
      const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
      const Exp2PolyConsts pc = exp2_poly_consts();
      uint32_t tsw = 0, tsb = 0, tcur = clock();
      for (int j = 0; j < ntm; ++j) {
        if constexpr ((TRACE & 3) != 0) {
          const uint32_t t = clock();
          tsb += t - tcur;
          tcur = t;
        }
        mbar_wait(B(B_SF + (j & 1)), (j >> 1) & 1);
        if constexpr ((TRACE & 3) != 0) {
          const uint32_t t = clock();
          tsw += t - tcur;
          tcur = t;
        }
        tc_fence_after();
        if constexpr (POLY < 0) {  // profiling only: MMA / TMA pipeline without softmax work
          tc_fence_before();
          warp_arrive(pf_bar0 + 8u * (j & 1));
          l_run = 1.f;
          continue;
        }
        const uint32_t scol = COL_S + 128u * (j & 1) + cb;
        const int lim = vis - j * BN - cb;  // visible keys of this row among this thread's columns
        const bool full = __all_sync(0xffffffffu, lim >= CW);
        auto exps = [&](auto full_c, const uint32_t* sr, float nmu, uint32_t* pk) -> float {
          constexpr bool FULL = decltype(full_c)::value;
          const uint64_t c2 = f32x2(sl2, sl2), n2 = f32x2(nmu, nmu);
          uint64_t acc0 = f32x2(0.f, 0.f), acc1 = f32x2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const uint64_t xx = ffma2(f32x2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), c2, n2);
            uint64_t pp;
            if (FULL && use_poly<POLY>(c >> 1)) {
              pp = exp2_poly_pair(xx, pc);
            } else {
              pp = f32x2(fast_exp2(f32x2_lo(xx)), fast_exp2(f32x2_hi(xx)));
            }
            if ((c & 2) == 0) acc0 = fadd2(acc0, pp); else acc1 = fadd2(acc1, pp);
            pk[c >> 1] = pack_bf16x2(f32x2_lo(pp), f32x2_hi(pp));
          }
          const uint64_t acc = fadd2(acc0, acc1);
          return f32x2_lo(acc) + f32x2_hi(acc);
        };
        uint32_t sr[32], pk[16];
        __syncwarp();
        tmem_ld32(tl + scol, sr);
        tmem_wait_ld();
        if (!full) {  // staircase tile: masked keys -> -inf -> exactly 0
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c >= lim) sr[c] = __float_as_uint(-INFINITY);
        }
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          m0 = fmax3(m0, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
          m1 = fmax3(m1, __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
        }
        // optimistic exponentials against the shared running max (no max -> exp dependency)
        float m_cur = m_run;
        float rs = full ? exps(std::true_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk)
                        : exps(std::false_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk);
        const float cm = fmaxf(m0, m1) * sl2;
        if (__any_sync(0xffffffffu, cm > m_cur + 64.0f)) {  // first visible tile / extreme jump: redo
          if (cm > m_cur + 64.0f) m_cur = ceilf(cm);
          rs = full ? exps(std::true_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk)
                    : exps(std::false_type{}, sr, m_cur == -INFINITY ? 0.f : -m_cur, pk);
        }
        tmem_st16(tl + scol, pk);  // P over this thread's own, already-read S columns
        const float tgt = cm > m_cur + 8.0f ? ceilf(cm) : m_cur;
        if (named_bar_red_or(bid, 4 * 32, tgt != m_run)) {
          // rare: some row's max grew by more than 2^8 — agree on the new max
          s_xch[i][cc] = tgt;
          named_bar_sync(bid, 4 * 32);
          const float m_fin = fmaxf(fmaxf(s_xch[i][0], s_xch[i][1]), fmaxf(s_xch[i][2], s_xch[i][3]));
          named_bar_sync(bid, 4 * 32);  // all read before the slots are reused
          float f = 1.f, alpha = 1.f;
          if (m_fin != -INFINITY) {
            f = pow2_int(m_cur - m_fin);
            alpha = pow2_int(m_run - m_fin);
          }
          l_run = l_run * alpha + rs * f;
          m_run = m_fin;
          if (__any_sync(0xffffffffu, f != 1.f)) {
            tmem_wait_st();
            const uint32_t a2 = pack_bf16x2(f, f);
#pragma unroll
            for (int c = 0; c < 16; ++c) pk[c] = mul_bf16x2(pk[c], a2);
            __syncwarp();
            tmem_st16(tl + scol, pk);
          }
          if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
            mbar_wait(B(B_PVD), (j - 1) & 1);  // O stable: PV_{j-1} complete
            tc_fence_after();
            uint32_t o[32];
            __syncwarp();
            tmem_ld32(tl + COL_O + cb, o);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
            tmem_st32(tl + COL_O + cb, o);
          }
        } else {
          l_run += rs;
        }
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(pf_bar0 + 8u * (j & 1));
      }
      if constexpr ((TRACE & 1) != 0) {
        tsb += clock() - tcur;
        if (lane == 0) {
          atomicAdd(&g_trace[5], (unsigned long long)tsw);
          atomicAdd(&g_trace[6], (unsigned long long)tsb);
          atomicAdd(&g_trace[7], (unsigned long long)ntm);
        }
      }
      mbar_wait(B(B_OD), 0);  // (PVD parity alone is ambiguous once phases have been skipped)
      tc_fence_after();
    }
    // ------------------------------------------------------ epilogue
    s_xch[i][cc] = l_run;
    named_bar_sync(bid, 4 * 32);
    const float l_tot = (s_xch[i][0] + s_xch[i][1]) + (s_xch[i][2] + s_xch[i][3]);
    uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)h * N + pos) * D + cb);
    if (ntm > 0) {
      const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
      uint32_t o[32];
      __syncwarp();
      tmem_ld32(tl + COL_O + cb, o);
      tmem_wait_ld();
      if (rvalid && l_tot > 0.f) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float* f = reinterpret_cast<const float*>(o + 8 * c);
          dst[c] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                              pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
        }
      }
    }
    if (rvalid) {
      if (l_tot > 0.f) {
        if (lse && cc == 0) lse[(size_t)h * N + pos] = static_cast<float>(M_LN2) * (m_run + log2f(l_tot));
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(Vorig + ((size_t)g * N + sink) * D + cb);
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = __ldg(src + c);
        if (lse && cc == 0) lse[(size_t)h * N + pos] = -INFINITY;
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

}  // namespace fwd2
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

// Called by omni_sparse_attn_fwd (attn_fwd.cu) after argument validation.
int omni_sparse_attn_fwd_pair(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                              const int32_t* counts, const int32_t* selected, const int32_t* sel_counts,
                              int n_q_heads, int n_kv_heads, int seq_len, int cap, int sink_index, void* O,
                              float* lse, int poly, cudaStream_t stream) {
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 64);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd2::BN);
  if (st) return st;
  static const bool trace = [] {
    const char* e = getenv("OMNI_FWD_TRACE");
    return e && atoi(e) != 0;
  }();
  static const int trace_mode = [] {
    const char* e = getenv("OMNI_FWD_TRACE");
    return e ? atoi(e) : 0;
  }();
  auto kern = trace ? (trace_mode == 2   ? fwd2::sparse_fwd_pair_kernel<4, 2>
                       : trace_mode == 4 ? fwd2::sparse_fwd_pair_kernel<4, 4>
                       : poly == -1      ? fwd2::sparse_fwd_pair_kernel<-1, 1>
                                         : fwd2::sparse_fwd_pair_kernel<4, 1>)
            : poly == -1 ? fwd2::sparse_fwd_pair_kernel<-1>  // profiling: no softmax work
            : poly == 0 ? fwd2::sparse_fwd_pair_kernel<0>
            : poly == 6 ? fwd2::sparse_fwd_pair_kernel<6>
            : poly == 8 ? fwd2::sparse_fwd_pair_kernel<8>
                        : fwd2::sparse_fwd_pair_kernel<4>;
  OMNI_CUDA_TRY(omni_smem_attr(kern, (int)fwd2::SMEM_BYTES));
  const int n_pairs = (seq_len + 2 * fwd2::BM - 1) / (2 * fwd2::BM);
  dim3 grid(2 * n_pairs * n_q_heads);
  kern<<<grid, fwd2::NTHREADS, fwd2::SMEM_BYTES, stream>>>(
      tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
      sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index, n_pairs,
      static_cast<__nv_bfloat16*>(O), lse);
  return omni_launch_check();
}

extern "C" int omni_debug_fwd_pair_trace(unsigned long long* host8) {
  omni_begin();
  OMNI_CUDA_TRY(cudaMemcpyFromSymbol(host8, fwd2::g_trace, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  OMNI_CUDA_TRY(cudaMemcpyToSymbol(fwd2::g_trace, z, sizeof(z)));
  return OMNI_OK;
}
