// K4 (shared-S / separate-P variant, OMNI_FWD_IMPL=sp): the single-CTA
// kernel's two Q tiles with the softmax taken off the tensor core's critical
// path.
//
// Contract as sparse_head_attention (prefill.py:89-122), see attn_fwd.cu. In
// the single-CTA kernel P is written over S, so QK_X(j+1) cannot start before
// PV_X(j) has read P_X(j): per Q tile the chain softmax -> PV -> QK ->
// softmax sets the period (1,024 tensor cycles + the softmax latency, ~1,700
// cycles, per 128-key step against 2,048 cycles of tensor work for both
// tiles; profiles/r02_notes.md). Here P has its own TMEM columns and one S
// buffer is shared by the two tiles:
//   TMEM: S [0, 128) | P_A [128, 192) | P_B [192, 256) | O_A [256, 384) |
//         O_B [384, 512)
// A tile's softmax threads load their S row into registers and release S at
// once (one arrival per thread), so the other tile's QK follows after the
// TMEM load latency; P_X(j) is stored once PV_X(j-1) has read P_X(j-1). The
// issue order per round r is QK_A(r), PV_A(r-1), QK_B(r), PV_B(r-1): each PV
// is issued a full round (2,048 tensor cycles) after its tile's S became
// ready, so the tensor core waits for neither softmax while the softmax
// latency stays below ~1,900 cycles.
//
// Warps (576 threads): 0 TMA (K / V 128-key tiles, 2-stage rings), 1 TMEM
// allocation + MMA issue, 2-17 softmax as in fwd_tile (two warps per TMEM lane
// quarter and tile, 64 key columns each; FAST: exponentials against the
// running max, growth beyond 2^8 settled after P is released, a jump beyond
// 2^64 flags *status for the single-CTA redo; safe: chunk maxima and
// agreement before P is stored).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace fwdsp {

constexpr int BM = 128, BN = 128, D = 128, NST = 2;
constexpr int NTHREADS = 576;
constexpr int HC = 64;
constexpr uint32_t ATOM = 128 * 128;
constexpr uint32_t TILE = 2 * ATOM;
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = OFF_Q + 2 * TILE;
constexpr uint32_t OFF_V = OFF_K + NST * TILE;
constexpr uint32_t OFF_BAR = OFF_V + NST * TILE;
enum {
  B_QF = 0,             // [2] Q tile X in smem (256 thread arrivals)
  B_KF = 2,             // [NST]
  B_KE = 2 + NST,       // [NST]
  B_VF = 2 + 2 * NST,   // [NST]
  B_VE = 2 + 3 * NST,   // [NST]
  B_SF = 2 + 4 * NST,   // [2] S_X(j) ready (MMA commit)
  B_SE = 4 + 4 * NST,   // [2] S_X(j) loaded by tile X's threads: S free (8 warp arrivals)
  B_PF = 6 + 4 * NST,   // [2] P_X(j) stored (+ O_X corrected) (8 warp arrivals)
  B_PD = 8 + 4 * NST,   // [2] PV_X(j) done: P_X free, O_X stable (MMA commit)
  B_COUNT = 10 + 4 * NST
};
constexpr uint32_t OFF_MISC = OFF_BAR + 8 * B_COUNT;
constexpr uint32_t SMEM_BYTES = OFF_MISC + 16 + 1024;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_S = 0;
__device__ __forceinline__ uint32_t col_p(int x) { return 128u + 64u * x; }
__device__ __forceinline__ uint32_t col_o(int x) { return 256u + 128u * x; }
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}
// One arrival per warp once every lane's TMEM accesses being signalled are
// complete (tcgen05.wait::ld / wait::st + fence::before_thread_sync).
__device__ __forceinline__ void warp_arrive(uint32_t b) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(b);
}
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

// Profiling (OMNI_FWD_TRACE=1 with OMNI_FWD_IMPL=sp): cycle sums read back by
// omni_debug_fwd_sp_trace: [0] MMA waits on S free, [1] on P ready, [2] on
// K / V / Q, [3] MMA loop, [4] softmax waits on S ready, [5] on PV done, [6]
// softmax loop, [7] MMA rounds.
__device__ unsigned long long g_sp_trace[8];

template <int POLY, bool FAST, bool TRACE = false>
__global__ void __launch_bounds__(NTHREADS, 1)
sparse_fwd_sp_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                     const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                     const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                     const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep, int N,
                     int cap, int sel_stride, int sink, __nv_bfloat16* __restrict__ O, float* __restrict__ lse,
                     int* __restrict__ status) {
  extern __shared__ uint8_t smem_raw[];
  const int L = blockIdx.x;
  const int h = L % Hq;
  int cmax = 0;
  for (int k = threadIdx.x & 31; k < Hq; k += 32) cmax = max(cmax, __ldg(counts + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  const int tile = (cmax + 2 * BM - 1) / (2 * BM) - 1 - L / Hq;  // heaviest tile pairs first
  const int cnt = __ldg(counts + h);
  const int row0 = tile * 2 * BM;
  if (tile < 0 || row0 >= cnt) return;

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
  const int32_t* rows_t = rows + (size_t)h * N + row0;

  const int sidx = warp - 2;
  const int xs = sidx >> 3;
  const int hf = (sidx >> 2) & 1;
  const int is = (warp & 3) * 32 + lane;
  const int nrows_s = min(BM, cnt - row0 - xs * BM);
  const bool rvalid = warp >= 2 && is < nrows_s;
  const int pos = rvalid ? __ldg(rows_t + xs * BM + is) : 0;
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
      mbar_init(B(B_QF + x), 2 * BM);
      mbar_init(B(B_SF + x), 1);
      mbar_init(B(B_SE + x), 8);
      mbar_init(B(B_PF + x), 8);
      mbar_init(B(B_PD + x), 1);
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
    tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ntA = s_nt[0], ntB = s_nt[1];
  const int ntm = max(ntA, ntB);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0 && ntm > 0) {
      const int kr0 = g * cap;
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NST;
        const uint32_t ph = ((j / NST) - 1) & 1;
        if (j >= NST) mbar_wait(B(B_KE + s), ph);
        mbar_expect_tx(B(B_KF + s), TILE);
        tma_load_2d(sbase + OFF_K + s * TILE, &tm_k, B(B_KF + s), 0, kr0 + j * BN);
        tma_load_2d(sbase + OFF_K + s * TILE + ATOM, &tm_k, B(B_KF + s), 64, kr0 + j * BN);
        if (j >= NST) mbar_wait(B(B_VE + s), ph);
        mbar_expect_tx(B(B_VF + s), TILE);
        tma_load_2d(sbase + OFF_V + s * TILE, &tm_v, B(B_VF + s), 0, kr0 + j * BN);
        tma_load_2d(sbase + OFF_V + s * TILE + ATOM, &tm_v, B(B_VF + s), 64, kr0 + j * BN);
      }
      for (int j = ntm > NST ? ntm - NST : 0; j < ntm; ++j) {
        mbar_wait(B(B_KE + j % NST), (j / NST) & 1);
        mbar_wait(B(B_VE + j % NST), (j / NST) & 1);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, D, 0, 1);
      const int nt[2] = {ntA, ntB};
      const uint64_t dq0 = sdesc_sw128(sbase + OFF_Q, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, ATOM, 1024);
      int last_x = -1, last_j = 0;  // the QK whose S the next QK overwrites
      unsigned long long tw[3] = {0, 0, 0};
      const long long t_loop = clock64();
      auto twait = [&](int k, uint32_t b, uint32_t ph) {
        if constexpr (TRACE) {
          const long long t0 = clock64();
          mbar_wait(b, ph);
          tw[k] += clock64() - t0;
        } else {
          mbar_wait(b, ph);
        }
      };
      for (int r = 0; r <= ntm; ++r) {
        bool kwaited = false, vwaited = false;
        for (int x = 0; x < 2; ++x) {
          if (r < nt[x]) {  // QK_X(r) into the shared S
            if (last_x >= 0) twait(0, B(B_SE + last_x), last_j & 1);  // previous S loaded by its tile
            if (!kwaited) {
              twait(2, B(B_KF + r % NST), (r / NST) & 1);
              kwaited = true;
            }
            if (r == 0) twait(2, B(B_QF + x), 0);
            tc_fence_after();
            const uint64_t qd = dq0 + ((x * TILE) >> 4), kd = dk0 + (((r % NST) * TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
              umma_bf16_ws(tmem + COL_S, qd + off, kd + off, idesc_qk, kk > 0 ? 1u : 0u);
            }
            umma_commit_ws(B(B_SF + x));
            last_x = x;
            last_j = r;
          }
          if (r >= 1 && r <= nt[x]) {  // PV_X(r - 1)
            const int j = r - 1, s = j % NST;
            if (!vwaited) {
              twait(2, B(B_VF + s), (j / NST) & 1);
              vwaited = true;
            }
            twait(1, B(B_PF + x), j & 1);
            tc_fence_after();
            const uint64_t vd = dv0 + ((s * TILE) >> 4);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              umma_bf16_ts_ws(tmem + col_o(x), tmem + col_p(x) + kk * 8, vd + ((kk * 2048) >> 4), idesc_pv,
                              (j > 0 || kk > 0) ? 1u : 0u);
            umma_commit_ws(B(B_PD + x));
          }
        }
        if (kwaited) umma_commit_ws(B(B_KE + r % NST));
        if (vwaited) umma_commit_ws(B(B_VE + (r - 1) % NST));
      }
      if constexpr (TRACE) {
        if (lane == 0) {
          for (int k = 0; k < 3; ++k) atomicAdd(&g_sp_trace[k], tw[k]);
          atomicAdd(&g_sp_trace[3], (unsigned long long)(clock64() - t_loop));
          atomicAdd(&g_sp_trace[7], (unsigned long long)(ntm + 1));
        }
      }
    }
  } else {
    // ------------------------------------------------------ softmax warps
    const int x = xs;
    const int quarter = warp & 3;
    const int i = is;
    const int cb = hf * HC;
    const uint32_t bid = 1 + x * 4 + quarter;
    const int nt = x ? ntB : ntA;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t tS = tl + COL_S + cb;          // this thread's 64 S columns
    const uint32_t tP = tl + col_p(x) + hf * 32;  // ... and their 32 packed P columns
    float m_run = -INFINITY, l_run = 0.f;
    float pend_alpha = 1.f;
    auto rescale_o = [&](float a) {  // this thread's 64 O columns, 16 at a time (register pressure)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t o[16];
        __syncwarp();
        tmem_ld16(tl + col_o(x) + cb + q * 16, o);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * a);
        tmem_st16(tl + col_o(x) + cb + q * 16, o);
      }
    };
    if (nt > 0) {
      uint8_t* q_gen = smem + OFF_Q + x * TILE + hf * ATOM;
#pragma unroll
      for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(q_gen + swz(i, c)) = qv[c];
      fence_proxy_async_smem();
      mbar_arrive(B(B_QF + x));

      const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
      const Exp2PolyConsts pc = exp2_poly_consts();
      auto exps = [&](auto full_c, const uint32_t* sr, float nmu, uint32_t* pk) -> float {
        constexpr bool FULL = decltype(full_c)::value;
        const uint64_t c2 = f32x2(sl2, sl2), n2 = f32x2(nmu, nmu);
        uint64_t acc0 = f32x2(0.f, 0.f), acc1 = f32x2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const uint64_t xx = ffma2(f32x2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), c2, n2);
          uint64_t pp;
          if (FULL && use_poly<POLY>(c >> 1)) pp = exp2_poly2_pair(xx, pc);
          else pp = f32x2(fast_exp2(f32x2_lo(xx)), fast_exp2(f32x2_hi(xx)));
          if ((c & 2) == 0) acc0 = fadd2(acc0, pp); else acc1 = fadd2(acc1, pp);
          pk[c >> 1] = pack_bf16x2(f32x2_lo(pp), f32x2_hi(pp));
        }
        const uint64_t acc = fadd2(acc0, acc1);
        return f32x2_lo(acc) + f32x2_hi(acc);
      };
      auto cmax32 = [&](const uint32_t* sr) -> float {
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          m0 = fmax3(m0, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
          m1 = fmax3(m1, __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
        }
        return fmaxf(m0, m1) * sl2;
      };
      unsigned long long tsw = 0, tpw = 0;
      const long long t_sm = clock64();
      for (int j = 0; j < nt; ++j) {
        if constexpr (TRACE) {
          const long long t0 = clock64();
          mbar_wait(B(B_SF + x), j & 1);
          tsw += clock64() - t0;
        } else {
          mbar_wait(B(B_SF + x), j & 1);
        }
        tc_fence_after();
        const int lim_row = vis - j * BN;
        const int lim = lim_row - cb;
        const bool full = __all_sync(0xffffffffu, lim >= HC);
        auto mask = [&](int q, uint32_t* sr) {
          if (!full) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
          }
        };
        auto wait_pd = [&]() {  // P_X free, O_X holds every P up to j - 1
          if (j > 0) {
            if constexpr (TRACE) {
              const long long t0 = clock64();
              mbar_wait(B(B_PD + x), (j - 1) & 1);
              tpw += clock64() - t0;
            } else {
              mbar_wait(B(B_PD + x), (j - 1) & 1);
            }
            tc_fence_after();
          }
        };
        if (FAST && !__any_sync(0xffffffffu, m_run == -INFINITY && lim_row > 0)) {
          // one 32-column chunk in registers at a time; S is released after the
          // second load (its latency hides under PV_A(r-1) in the issue order)
          const float nmu = -m_run;
          uint32_t sr[32], pk[16];
          __syncwarp();
          tmem_ld32(tS, sr);
          tmem_wait_ld();
          mask(0, sr);
          float rs = full ? exps(std::true_type{}, sr, nmu, pk) : exps(std::false_type{}, sr, nmu, pk);
          __syncwarp();
          tmem_ld32(tS + 32, sr);
          tmem_wait_ld();
          tc_fence_before();
          warp_arrive(B(B_SE + x));  // S may now be overwritten by the next QK
          wait_pd();
          if (__any_sync(0xffffffffu, pend_alpha != 1.f)) {
            rescale_o(pend_alpha);
            pend_alpha = 1.f;
          }
          __syncwarp();
          tmem_st16(tP, pk);
          mask(1, sr);
          rs += full ? exps(std::true_type{}, sr, nmu, pk) : exps(std::false_type{}, sr, nmu, pk);
          tmem_st16(tP + 16, pk);
          tmem_wait_st();
          tc_fence_before();
          warp_arrive(B(B_PF + x));
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
        uint32_t s0[32], s1[32];
        __syncwarp();
        tmem_ld32(tS, s0);
        tmem_ld32(tS + 32, s1);
        tmem_wait_ld();
        tc_fence_before();
        warp_arrive(B(B_SE + x));
        mask(0, s0);
        mask(1, s1);
        // agreement before P is stored: exponentials against the running max,
        // or against ceil(row max) where that is more than 2^64 above it (a
        // row's first visible keys, or a jump)
        const float cm = fmaxf(cmax32(s0), cmax32(s1));
        float m_cur = m_run;
        if (cm > m_cur + 64.0f) m_cur = ceilf(cm);
        const float nmu = m_cur == -INFINITY ? 0.f : -m_cur;
        uint32_t pk0[16], pk1[16];
        const float rs = (full ? exps(std::true_type{}, s0, nmu, pk0) : exps(std::false_type{}, s0, nmu, pk0)) +
                         (full ? exps(std::true_type{}, s1, nmu, pk1) : exps(std::false_type{}, s1, nmu, pk1));
        const float tgt = cm > m_cur + 8.0f ? ceilf(cm) : m_cur;
        float alpha = 1.f;
        if (named_bar_red_or(bid, 2 * 32, tgt != m_run)) {
          s_xch[x][i][hf] = tgt;
          named_bar_sync(bid, 2 * 32);
          const float m_fin = fmaxf(tgt, s_xch[x][i][hf ^ 1]);
          named_bar_sync(bid, 2 * 32);
          float f = 1.f;
          if (m_fin != -INFINITY) {
            f = pow2_int(m_cur - m_fin);
            alpha = pow2_int(m_run - m_fin);
          }
          l_run = l_run * alpha + rs * f;
          m_run = m_fin;
          if (__any_sync(0xffffffffu, f != 1.f)) {
            const uint32_t a2 = pack_bf16x2(f, f);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              pk0[c] = mul_bf16x2(pk0[c], a2);
              pk1[c] = mul_bf16x2(pk1[c], a2);
            }
          }
        } else {
          l_run += rs;
        }
        wait_pd();
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) rescale_o(alpha);
        __syncwarp();
        tmem_st16(tP, pk0);
        tmem_st16(tP + 16, pk1);
        tmem_wait_st();
        tc_fence_before();
        warp_arrive(B(B_PF + x));
      }
      if constexpr (TRACE) {
        if (lane == 0) {
          atomicAdd(&g_sp_trace[4], tsw);
          atomicAdd(&g_sp_trace[5], tpw);
          atomicAdd(&g_sp_trace[6], (unsigned long long)(clock64() - t_sm));
        }
      }
      mbar_wait(B(B_PD + x), (nt - 1) & 1);
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
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace fwdsp
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

// Called by omni_sparse_attn_fwd_ex (attn_fwd.cu) after argument validation.
// status != nullptr: the FAST kernel (the caller launches the safe single-CTA
// redo behind it); else the safe kernel.
int omni_sparse_attn_fwd_sp(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream) {
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwdsp::BN);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwdsp::BN);
  if (st) return st;
  const bool fast = status != nullptr;
  static const bool trace = [] {
    const char* e = getenv("OMNI_FWD_TRACE");
    return e && atoi(e) != 0;
  }();
  auto kern = (fast && trace) ? fwdsp::sparse_fwd_sp_kernel<6, true, true>
            : fast ? (poly == 4   ? fwdsp::sparse_fwd_sp_kernel<4, true>
                      : poly == 8 ? fwdsp::sparse_fwd_sp_kernel<8, true>
                      : poly == 0 ? fwdsp::sparse_fwd_sp_kernel<0, true>
                                  : fwdsp::sparse_fwd_sp_kernel<6, true>)
                   : fwdsp::sparse_fwd_sp_kernel<6, false>;
  OMNI_CUDA_TRY(omni_smem_attr(kern, (int)fwdsp::SMEM_BYTES));
  const int n_tiles = (seq_len + 2 * fwdsp::BM - 1) / (2 * fwdsp::BM);
  kern<<<n_tiles * n_q_heads, fwdsp::NTHREADS, fwdsp::SMEM_BYTES, stream>>>(
      tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
      sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index,
      static_cast<__nv_bfloat16*>(O), lse, status);
  return omni_launch_check();
}

extern "C" int omni_debug_fwd_sp_trace(unsigned long long* host8) {
  omni_begin();
  OMNI_CUDA_TRY(cudaMemcpyFromSymbol(host8, fwdsp::g_sp_trace, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  OMNI_CUDA_TRY(cudaMemcpyToSymbol(fwdsp::g_sp_trace, z, sizeof(z)));
  return OMNI_OK;
}
