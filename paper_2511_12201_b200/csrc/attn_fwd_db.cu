// K4 (double-buffered S variant, OMNI_FWD_IMPL=db): the single-CTA kernel's
// two Q tiles with 64-key sub-tiles and two S buffers per Q tile, so the
// softmax of a tile's consecutive sub-tiles runs back to back and the tensor
// core waits only for P.
//
// Contract as sparse_head_attention (prefill.py:89-122), see attn_fwd.cu. One
// CTA owns 256 compacted rows of one Q head (tiles A, B of 128 rows) and
// streams its group's compacted selected keys in 64-key sub-tiles j:
//   S_X(j) = Q_X K_j^T  (SS, M = 128, N = 64)   -> S buffer (j & 1) of tile X
//   O_X += P_X(j) V_j   (TS, M = 128, N = 128, K = 64; P written over S)
// TMEM per tile X (256 columns): S buffers [256X, +64), [256X + 64, +64),
// O [256X + 128, +128). QK_X(j + 2) is issued right behind PV_X(j) (same S
// buffer; the tensor pipe is in order), i.e. one sub-tile ahead of the
// softmax, which therefore never waits for the tensor core's PV / QK latency
// of its own previous sub-tile — in the single-CTA kernel that chain (softmax
// -> PV -> QK -> softmax) sets the period (profiles/r02_notes.md).
//
// Warps (320 threads): 0 TMA (K, V sub-tiles, 64 keys x 128 d, 4-stage
// rings), 1 TMEM allocation + MMA issue, 2-9 softmax: warps 2-5 tile A, 6-9
// tile B, thread = row = TMEM lane, 64 columns per sub-tile, so the row
// maximum and sum need no exchange between threads. Online softmax in the
// exp2 domain with an integral running max; FAST mode exponentiates against
// the running max, releases P and settles growth beyond 2^8 afterwards (O
// rescaled before the next sub-tile's P is released, after that tile's
// previous PV has completed); a logit jump beyond 2^64 flags *status and the
// single-CTA safe kernel redoes the launch. A warp in which some row meets its
// first visible keys takes the two-pass path (row max, then exponentials).
//
// Barriers that a waiter could otherwise see complete twice before it waits
// (S ready, P ready, PV done) are per S buffer: a waiter is never more than
// one phase behind on any of them.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace fwddb {

constexpr int BM = 128, BK = 64, D = 128, NS = 4;
constexpr int NTHREADS = 320;
constexpr uint32_t ATOM = 128 * 128;    // 128 rows x 128 B (Q tile: two)
constexpr uint32_t TILE = 2 * ATOM;     // 128 x 128 bf16
constexpr uint32_t KATOM = 64 * 128;    // 64 rows x 128 B
constexpr uint32_t SUB = 2 * KATOM;     // one K or V sub-tile: 64 keys x 128 d
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = OFF_Q + 2 * TILE;
constexpr uint32_t OFF_V = OFF_K + NS * SUB;
constexpr uint32_t OFF_BAR = OFF_V + NS * SUB;
enum {
  B_QF = 0,             // [2] Q tile X in smem (128 thread arrivals)
  B_KF = 2,             // [NS]
  B_KE = 2 + NS,        // [NS]
  B_VF = 2 + 2 * NS,    // [NS]
  B_VE = 2 + 3 * NS,    // [NS]
  B_SF = 2 + 4 * NS,    // [2][2] S_X(j) in buffer b ready (MMA commit)
  B_PF = 6 + 4 * NS,    // [2][2] P_X(j) in buffer b written (+ O_X corrected) (128 thread arrivals)
  B_PV = 10 + 4 * NS,   // [2][2] PV_X(j) of buffer b done (MMA commit)
  B_COUNT = 14 + 4 * NS
};
constexpr uint32_t OFF_MISC = OFF_BAR + 8 * B_COUNT;  // tmem slot, nt[2]
constexpr uint32_t SMEM_BYTES = OFF_MISC + 16 + 1024;
constexpr uint32_t TMEM_COLS = 512;
__device__ __forceinline__ uint32_t col_s(int x, int b) { return 256u * x + 64u * b; }
__device__ __forceinline__ uint32_t col_o(int x) { return 256u * x + 128u; }
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

template <int POLY, bool FAST>
__global__ void __launch_bounds__(NTHREADS, 1)
sparse_fwd_db_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;
  const int32_t* rows_t = rows + (size_t)h * N + row0;

  const int xs = (warp - 2) >> 2;         // Q tile of a softmax warp
  const int is = (warp & 3) * 32 + lane;  // its row == TMEM lane
  const int nrows_s = min(BM, cnt - row0 - xs * BM);
  const bool rvalid = warp >= 2 && is < nrows_s;
  const int pos = rvalid ? __ldg(rows_t + xs * BM + is) : 0;
  uint4 qv[16];
  if (warp >= 2) {
    const uint4* qrow = reinterpret_cast<const uint4*>(Q + ((size_t)h * N + pos) * D);
#pragma unroll
    for (int c = 0; c < 16; ++c) qv[c] = rvalid ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
  }
  int vis = warp >= 2 ? count_le_warp(selg, nsel, pos, rvalid) : 0;
  if (!rvalid) vis = 0;
  if (warp >= 2) {
    if (is == nrows_s - 1) s_nt[xs] = (vis + BK - 1) / BK;
    if (nrows_s <= 0 && is == 0) s_nt[xs] = 0;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    for (int x = 0; x < 2; ++x) mbar_init(B(B_QF + x), BM);
    for (int k = 0; k < 4; ++k) {
      mbar_init(B(B_SF + k), 1);
      mbar_init(B(B_PF + k), BM);
      mbar_init(B(B_PV + k), 1);
    }
    for (int s = 0; s < NS; ++s) {
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
        const int s = j % NS;
        const uint32_t ph = ((j / NS) - 1) & 1;
        if (j >= NS) mbar_wait(B(B_KE + s), ph);
        mbar_expect_tx(B(B_KF + s), SUB);
        tma_load_2d(sbase + OFF_K + s * SUB, &tm_k, B(B_KF + s), 0, kr0 + j * BK);
        tma_load_2d(sbase + OFF_K + s * SUB + KATOM, &tm_k, B(B_KF + s), 64, kr0 + j * BK);
        if (j >= NS) mbar_wait(B(B_VE + s), ph);
        mbar_expect_tx(B(B_VF + s), SUB);
        tma_load_2d(sbase + OFF_V + s * SUB, &tm_v, B(B_VF + s), 0, kr0 + j * BK);
        tma_load_2d(sbase + OFF_V + s * SUB + KATOM, &tm_v, B(B_VF + s), 64, kr0 + j * BK);
      }
      for (int j = ntm > NS ? ntm - NS : 0; j < ntm; ++j) {
        mbar_wait(B(B_KE + j % NS), (j / NS) & 1);
        mbar_wait(B(B_VE + j % NS), (j / NS) & 1);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BK, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, D, 0, 1);
      const int nt[2] = {ntA, ntB};
      const uint64_t dq0 = sdesc_sw128(sbase + OFF_Q, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, KATOM, 1024);
      auto qk = [&](int x, int j) {  // S_X(j) = Q_X K_j^T -> S buffer j & 1
        const uint64_t qd = dq0 + ((x * TILE) >> 4), kd = dk0 + (((j % NS) * SUB) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offq = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          const uint32_t offk = ((kk >> 2) * KATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + col_s(x, j & 1), qd + offq, kd + offk, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_ws(B(B_SF + 2 * x + (j & 1)));
      };
      // prologue: S(0) and S(1) of both tiles
      for (int j = 0; j < 2 && j < ntm; ++j) {
        mbar_wait(B(B_KF + j), 0);
        tc_fence_after();
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          if (j == 0) {
            mbar_wait(B(B_QF + x), 0);
            tc_fence_after();
          }
          qk(x, j);
        }
        umma_commit_ws(B(B_KE + j));
      }
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NS, b = j & 1;
        mbar_wait(B(B_VF + s), (j / NS) & 1);
        bool kwaited = false;
        const uint64_t vd = dv0 + ((s * SUB) >> 4);
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          mbar_wait(B(B_PF + 2 * x + b), (j >> 1) & 1);  // P_X(j) written (and O_X corrected)
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ts_ws(tmem + col_o(x), tmem + col_s(x, b) + kk * 8, vd + ((kk * 2048) >> 4), idesc_pv,
                            (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit_ws(B(B_PV + 2 * x + b));
          if (j + 2 < nt[x]) {
            if (!kwaited) {
              mbar_wait(B(B_KF + (j + 2) % NS), ((j + 2) / NS) & 1);
              tc_fence_after();
              kwaited = true;
            }
            qk(x, j + 2);  // into S buffer b, after PV_X(j) has read P from it (in-order pipe)
          }
        }
        umma_commit_ws(B(B_VE + s));
        if (kwaited) umma_commit_ws(B(B_KE + (j + 2) % NS));
      }
    }
  } else {
    // ------------------------------------------------------ softmax warps
    const int x = xs, i = is;
    const int nt = x ? ntB : ntA;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f, pend_alpha = 1.f;
    if (nt > 0) {
      uint8_t* q_gen = smem + OFF_Q + x * TILE;
#pragma unroll
      for (int c = 0; c < 16; ++c) *reinterpret_cast<uint4*>(q_gen + (c >> 3) * ATOM + swz(i, c & 7)) = qv[c];
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
      auto mask = [&](int q, int lim, uint32_t* sr) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
      };
      auto wait_pv = [&](int jj) {  // PV_X(jj) (and, in order, every earlier one) complete
        mbar_wait(B(B_PV + 2 * x + (jj & 1)), (jj >> 1) & 1);
        tc_fence_after();
      };
      auto rescale_o = [&](float a) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[32];
          __syncwarp();
          tmem_ld32(tl + col_o(x) + q * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * a);
          tmem_st32(tl + col_o(x) + q * 32, o);
        }
      };
      for (int j = 0; j < nt; ++j) {
        const int b = j & 1;
        const uint32_t sc = tl + col_s(x, b);
        mbar_wait(B(B_SF + 2 * x + b), (j >> 1) & 1);
        tc_fence_after();
        const int lim = vis - j * BK;
        const bool full = __all_sync(0xffffffffu, lim >= BK);
        if (FAST && __any_sync(0xffffffffu, pend_alpha != 1.f)) {
          wait_pv(j - 1);  // O holds every P up to j - 1 (computed against the old max)
          rescale_o(pend_alpha);
          pend_alpha = 1.f;
        }
        if (FAST && !__any_sync(0xffffffffu, m_run == -INFINITY && lim > 0)) {
          const float nmu = m_run == -INFINITY ? 0.f : -m_run;
          uint32_t s0[32], s1[32], pk[16];
          __syncwarp();
          tmem_ld32(sc, s0);
          tmem_ld32(sc + 32, s1);
          tmem_wait_ld();
          if (!full) {
            mask(0, lim, s0);
            mask(1, lim, s1);
          }
          float rs = full ? exps(std::true_type{}, s0, nmu, pk) : exps(std::false_type{}, s0, nmu, pk);
          tmem_st16(sc, pk);
          rs += full ? exps(std::true_type{}, s1, nmu, pk) : exps(std::false_type{}, s1, nmu, pk);
          tmem_st16(sc + 16, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(B(B_PF + 2 * x + b));
          if (m_run != -INFINITY && !(rs <= 0x1p64f)) atomicExch(status, 1);
          if (m_run != -INFINITY && rs > 256.f) {
            const float m_new = m_run + ceilf(__log2f(rs));
            const float alpha = pow2_int(m_run - m_new);
            l_run = (l_run + rs) * alpha;
            pend_alpha = alpha;
            m_run = m_new;
          } else {
            l_run += rs;
          }
          continue;
        }
        // two-pass path: the row maximum over this sub-tile's visible keys first
        uint32_t s0[32], s1[32];
        __syncwarp();
        tmem_ld32(sc, s0);
        tmem_ld32(sc + 32, s1);
        tmem_wait_ld();
        if (!full) {
          mask(0, lim, s0);
          mask(1, lim, s1);
        }
        float cm = -INFINITY;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          cm = fmax3(cm, __uint_as_float(s0[c]), __uint_as_float(s0[c + 1]));
          cm = fmax3(cm, __uint_as_float(s1[c]), __uint_as_float(s1[c + 1]));
        }
        cm *= sl2;
        float m_fin = m_run;
        if (cm != -INFINITY && (m_run == -INFINITY || cm > m_run + 8.f)) m_fin = ceilf(cm);
        const float alpha = (m_run == -INFINITY || m_fin == -INFINITY) ? 1.f : pow2_int(m_run - m_fin);
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          wait_pv(j - 1);
          rescale_o(alpha);
        }
        l_run *= alpha;
        m_run = m_fin;
        const float nmu = m_run == -INFINITY ? 0.f : -m_run;
        uint32_t pk[16];
        float rs = exps(std::false_type{}, s0, nmu, pk);
        tmem_st16(sc, pk);
        rs += exps(std::false_type{}, s1, nmu, pk);
        tmem_st16(sc + 16, pk);
        l_run += rs;
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(B(B_PF + 2 * x + b));
      }
      wait_pv(nt - 1);
    }
    // ------------------------------------------------------ epilogue
    uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)h * N + pos) * D);
    if (nt > 0) {
      const float inv = l_run > 0.f ? pend_alpha / l_run : 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t o[32];
        __syncwarp();
        tmem_ld32(tl + col_o(x) + q * 32, o);
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
        if (lse) lse[(size_t)h * N + pos] = static_cast<float>(M_LN2) * (m_run + log2f(l_run));
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(Vorig + ((size_t)g * N + sink) * D);
#pragma unroll
        for (int c = 0; c < 16; ++c) dst[c] = __ldg(src + c);
        if (lse) lse[(size_t)h * N + pos] = -INFINITY;
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

}  // namespace fwddb
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

// Called by omni_sparse_attn_fwd_ex (attn_fwd.cu) after argument validation.
// status != nullptr: the FAST kernel (the caller launches the safe single-CTA
// redo behind it); else the two-pass kernel.
int omni_sparse_attn_fwd_db(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream) {
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwddb::BK);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwddb::BK);
  if (st) return st;
  const bool fast = status != nullptr;
  auto kern = fast ? (poly == 4   ? fwddb::sparse_fwd_db_kernel<4, true>
                      : poly == 8 ? fwddb::sparse_fwd_db_kernel<8, true>
                      : poly == 0 ? fwddb::sparse_fwd_db_kernel<0, true>
                                  : fwddb::sparse_fwd_db_kernel<6, true>)
                   : fwddb::sparse_fwd_db_kernel<6, false>;
  OMNI_CUDA_TRY(omni_smem_attr(kern, (int)fwddb::SMEM_BYTES));
  const int n_tiles = (seq_len + 2 * fwddb::BM - 1) / (2 * fwddb::BM);
  kern<<<n_tiles * n_q_heads, fwddb::NTHREADS, fwddb::SMEM_BYTES, stream>>>(
      tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
      sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index,
      static_cast<__nv_bfloat16*>(O), lse, status);
  return omni_launch_check();
}
