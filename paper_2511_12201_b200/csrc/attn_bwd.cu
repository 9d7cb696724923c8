// K5: backward of the gathered sparse flash attention (tcgen05 / TMEM / TMA).
//
// The reference has no autograd; gradients are checked against a float64
// torch-autograd restatement of sparse_head_attention (oracle/grad.py). With
// compacted active rows (per Q head) and compacted selected keys (per group):
//   P_ij  = exp(s_ij - lse_i) for j < vis_i (original-position staircase)
//   dV_j  = sum_i P_ij dO_i            dP_ij = dO_i . V_j
//   dS_ij = P_ij (dP_ij - D_i)          D_i   = dO_i . O_i
//   dQ_i  = scale sum_j dS_ij K_j       dK_j  = scale sum_i dS_ij Q_i
// Rows with no visible key copied V[sink] in the forward: their dO goes to
// dV[sink] (dV_sink). Three kernels, no atomics on the hot path:
//   prep  (HBM-bound): gathers Q / dO rows into compact bf16 tiles, computes
//         D_i, log2-domain LSE and vis_i per compact row;
//   dq    Q-tile CTAs (like the forward): S = Q K^T, dP = dO V^T, dS -> smem,
//         dQ += dS K (TMEM accumulator);
//   dkv   KV-tile CTAs looping over every Q tile of the group's Q heads that
//         can see the tile: S^T = K Q^T, dP^T = V dO^T, P^T / dS^T -> smem,
//         dV += P^T dO, dK += dS^T Q (TMEM accumulators). One CTA per (key
//         tile, Q head); the group's Q heads reduce into the zero-initialised
//         fp32 dK / dV with vector atomics (red.global.add.v4.f32), so the
//         fp32 summation order over a group's heads varies run to run.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace bwd {

constexpr int D = 128;
// Exponential pairs (of 16 per 32-column chunk) evaluated by the FMA-pipe
// polynomial instead of MUFU.EX2 in the dS math (masked entries are discarded
// by a select, so the polynomial's behaviour on them does not matter).
// Measured at C4: dq 4 of 16 (MUFU co-bottleneck); dkv 0 since P^T is formed
// off the critical path (4 of 16 was best before that change).
#ifndef OMNI_BWD_POLY
#define OMNI_BWD_POLY 0
#endif
#ifndef OMNI_DQ_POLY
#define OMNI_DQ_POLY 4
#endif
__device__ __forceinline__ constexpr bool bwd_poly(int pair) {
  return OMNI_BWD_POLY > 0 && ((pair * OMNI_BWD_POLY) % 16) < OMNI_BWD_POLY;
}
__device__ __forceinline__ constexpr bool dq_poly(int pair) {
  return OMNI_DQ_POLY > 0 && ((pair * OMNI_DQ_POLY) % 16) < OMNI_DQ_POLY;
}
constexpr uint32_t ATOM = 128 * 128;  // 128 rows x 128 B swizzle region
constexpr uint32_t TILE = 2 * ATOM;   // 128 x 128 bf16

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}

// ------------------------------------------------------------------ prep
__global__ void __launch_bounds__(256) bwd_prep_kernel(
    const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ dO,
    const float* __restrict__ lse, const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
    const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int N, int rep, int capq,
    __nv_bfloat16* __restrict__ Qc, __nv_bfloat16* __restrict__ dOc, float* __restrict__ lse2c,
    float* __restrict__ Dc, int32_t* __restrict__ visc, float* __restrict__ dv_sink) {
  // one warp per 32 consecutive compacted rows: their visible-key counts by a
  // warp-cooperative search (ascending rows), then the rows one by one
  const int h = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int i0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32;
  const int cnt = __ldg(counts + h);
  const int lim = ((cnt + 127) / 128) * 128;
  if (i0 >= lim) return;
  const int g = h / rep;
  const int il = i0 + lane;
  const bool lvalid = il < cnt;
  const int lpos = lvalid ? __ldg(rows + (size_t)h * N + il) : 0;
  int lvis = count_le_warp(sel + (size_t)g * N, __ldg(sel_counts + g), lpos, lvalid);
  if (!lvalid) lvis = 0;
  if (il < lim) {
    const size_t ci = (size_t)h * capq + il;
    lse2c[ci] = lvalid ? __ldg(lse + (size_t)h * N + lpos) * static_cast<float>(kLog2e) : 0.f;
    visc[ci] = lvis;
  }
#pragma unroll 8
  for (int r = 0; r < 32; ++r) {
    const int i = i0 + r;
    if (i >= lim) break;
    const size_t ci = (size_t)h * capq + i;
    uint2* qd = reinterpret_cast<uint2*>(Qc + ci * D);
    uint2* dd = reinterpret_cast<uint2*>(dOc + ci * D);
    if (i >= cnt) {
      qd[lane] = make_uint2(0, 0);
      dd[lane] = make_uint2(0, 0);
      if (lane == 0) Dc[ci] = 0.f;
      continue;
    }
    const int pos = __shfl_sync(0xffffffffu, lpos, r);
    const int vis = __shfl_sync(0xffffffffu, lvis, r);
    const size_t src = ((size_t)h * N + pos) * D;
    const uint2 qv = __ldg(reinterpret_cast<const uint2*>(Q + src) + lane);
    const uint2 ov = __ldg(reinterpret_cast<const uint2*>(O + src) + lane);
    const uint2 gv = __ldg(reinterpret_cast<const uint2*>(dO + src) + lane);
    qd[lane] = qv;
    dd[lane] = gv;
    const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
    float dsum = 0.f;
    float gf[4];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const float2 a2 = __bfloat1622float2(o2[k]), b2 = __bfloat1622float2(g2[k]);
      dsum += a2.x * b2.x + a2.y * b2.y;
      gf[2 * k] = b2.x;
      gf[2 * k + 1] = b2.y;
    }
    dsum = warp_sum(dsum);
    if (lane == 0) Dc[ci] = dsum;
    if (vis == 0) {  // forward copied V[sink] for this row: dV[sink] += dO
#pragma unroll
      for (int k = 0; k < 4; ++k) atomicAdd(dv_sink + (size_t)g * D + lane * 4 + k, gf[k]);
    }
  }
}

// ------------------------------------------------------------------ dq
namespace dq {
// K ring 3 deep: K_j is held until dQ_j completes, which is just before
// S_{j+2} needs K_{j+2} (a 2-deep ring exposed the TMA latency there); V_j is
// free once dP_j is done, so 2 stages suffice.
constexpr int NSK = 3;
constexpr uint32_t OFF_Q = 0, OFF_DO = TILE, OFF_K = 2 * TILE, OFF_V = OFF_K + NSK * TILE;
constexpr uint32_t OFF_BAR = OFF_V + 2 * TILE;
enum { B_QD = 0, B_KF = 1, B_KE = 1 + NSK, B_VF = 1 + 2 * NSK, B_VE = 3 + 2 * NSK, B_SF = 5 + 2 * NSK, B_SE, B_DSF,
       B_DSE, B_QT, B_N };
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * B_N;
constexpr uint32_t SMEM = OFF_TMEM + 16 + 1024;
// dS (bf16 pairs, 64 columns) lives in TMEM: dQ += dS K is a TS MMA, so
// the only shared-memory operand traffic of a key tile is S / dP's and K's
// (the SS dS product made the kernel shared-memory-bandwidth bound)
constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DQ = 256, COL_DS = 384;
// QT: the Q tile also lives in TMEM (bf16 pairs, columns 448..511), so
// S = Q K^T is a TS MMA too and only K crosses the shared-memory operand
// path for it (the SS S / dP MMAs bound the MMA pipeline at 128 B/clk)
constexpr uint32_t COL_Q = 448;
}  // namespace dq

// PROBE (profiling only, OMNI_DQ_PROBE=1): the gradient warps release dS
// without computing it (the MMA / TMA pipeline floor).
template <int PROBE, bool QT = true>
__global__ void __launch_bounds__(576, 1)
dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
          const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
          const int32_t* __restrict__ rows, const int32_t* __restrict__ counts, const float* __restrict__ lse2c,
          const float* __restrict__ Dc, const int32_t* __restrict__ visc, int Hq, int rep, int N, int cap, int capq,
          int n_tiles, void* __restrict__ dQ, int dq_bf16) {
  using namespace dq;
  extern __shared__ uint8_t smem_raw[];
  const int L = blockIdx.x;
  const int h = L % Hq;
  const int tile = n_tiles - 1 - L / Hq;
  const int cnt = __ldg(counts + h);
  const int r0 = tile * 128;
  if (r0 >= cnt) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar = sb + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ int s_nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nrows = min(128, cnt - r0);
  const size_t crow0 = (size_t)h * capq + r0;
  if (threadIdx.x == 0) {
    s_nt = (__ldg(visc + crow0 + nrows - 1) + 127) / 128;
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(B(B_QD), 1);
    for (int s = 0; s < NSK; ++s) {
      mbar_init(B(B_KF + s), 1);
      mbar_init(B(B_KE + s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(B(B_VF + s), 1);
      mbar_init(B(B_VE + s), 1);
    }
    mbar_init(B(B_SF), 1);
    mbar_init(B(B_SE), 512);
    mbar_init(B(B_DSF), 512);
    mbar_init(B(B_DSE), 1);
    mbar_init(B(B_QT), 512);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nt = s_nt;

  if (warp == 0) {
    if (lane == 0 && nt > 0) {
      mbar_expect_tx(B(B_QD), 2 * TILE);
      tma_load_2d(sb + OFF_Q, &tm_q, B(B_QD), 0, (int)crow0);
      tma_load_2d(sb + OFF_Q + ATOM, &tm_q, B(B_QD), 64, (int)crow0);
      tma_load_2d(sb + OFF_DO, &tm_do, B(B_QD), 0, (int)crow0);
      tma_load_2d(sb + OFF_DO + ATOM, &tm_do, B(B_QD), 64, (int)crow0);
      const int kr0 = g * cap;
      for (int j = 0; j < nt; ++j) {
        const int sk = j % NSK, s = j & 1;
        if (j >= NSK) mbar_wait(B(B_KE + sk), ((j / NSK) - 1) & 1);
        mbar_expect_tx(B(B_KF + sk), TILE);
        tma_load_2d(sb + OFF_K + sk * TILE, &tm_k, B(B_KF + sk), 0, kr0 + j * 128);
        tma_load_2d(sb + OFF_K + sk * TILE + ATOM, &tm_k, B(B_KF + sk), 64, kr0 + j * 128);
        if (j >= 2) mbar_wait(B(B_VE + s), ((j >> 1) - 1) & 1);
        mbar_expect_tx(B(B_VF + s), TILE);
        tma_load_2d(sb + OFF_V + s * TILE, &tm_v, B(B_VF + s), 0, kr0 + j * 128);
        tma_load_2d(sb + OFF_V + s * TILE + ATOM, &tm_v, B(B_VF + s), 64, kr0 + j * 128);
      }
      // observe the last ring phases (every mbarrier phase is waited on)
      for (int j = nt > NSK ? nt - NSK : 0; j < nt; ++j) mbar_wait(B(B_KE + j % NSK), (j / NSK) & 1);
      for (int j = nt > 2 ? nt - 2 : 0; j < nt; ++j) mbar_wait(B(B_VE + (j & 1)), (j >> 1) & 1);
    }
  } else if (warp == 1) {
    // whole warp runs the schedule; elect.sync picks the issuing lane
    if (nt > 0) {
      constexpr uint32_t id_kk = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t id_mn = idesc_bf16_f32(128, 128, 0, 1);
      const uint64_t dq0 = sdesc_sw128(sb + OFF_Q, 16, 1024), ddo0 = sdesc_sw128(sb + OFF_DO, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sb + OFF_K, 16, 1024), dv0 = sdesc_sw128(sb + OFF_V, 16, 1024);
      const uint64_t dkmn0 = sdesc_sw128(sb + OFF_K, ATOM, 1024);
      auto issue_s = [&](int j) {
        const int s = j & 1, sk = j % NSK;
        mbar_wait(B(B_KF + sk), (j / NSK) & 1);
        mbar_wait(B(B_VF + s), (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          if constexpr (QT) umma_bf16_ts_ws(tmem + COL_S, tmem + COL_Q + kk * 8, dk0 + ((sk * TILE) >> 4) + off, id_kk, kk > 0);
          else umma_bf16_ws(tmem + COL_S, dq0 + off, dk0 + ((sk * TILE) >> 4) + off, id_kk, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + COL_DP, ddo0 + off, dv0 + ((s * TILE) >> 4) + off, id_kk, kk > 0);
        }
        umma_commit_ws(B(B_VE + s));
        umma_commit_ws(B(B_SF));
      };
      mbar_wait(B(B_QD), 0);
      if constexpr (QT) mbar_wait(B(B_QT), 0);  // Q copied into TMEM by the gradient warps
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nt; ++j) {
        mbar_wait(B(B_SE), j & 1);
        if (j + 1 < nt) issue_s(j + 1);
        mbar_wait(B(B_DSF), j & 1);
        tc_fence_after();
        const uint64_t kb = dkmn0 + (((j % NSK) * TILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          umma_bf16_ts_ws(tmem + COL_DQ, tmem + COL_DS + kk * 8, kb + ((kk * 2048) >> 4),
                       id_mn, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_ws(B(B_KE + j % NSK));
        umma_commit_ws(B(B_DSE));
      }
    }
  } else if (warp >= 2) {
    // 16 warps: four per TMEM lane quarter, each thread 32 key columns of its
    // row. S and dP are read into registers first and released at once (the
    // S / dP MMAs of the next key tile overlap this tile's dS math).
    const int hf = (warp - 2) >> 2;  // column quarter 0..3
    const int i = (warp & 3) * 32 + lane;
    const int cb = hf * 32;
    const bool valid = i < nrows;
    const size_t ci = crow0 + i;
    const int vis = valid ? __ldg(visc + ci) : 0;
    const float l2 = valid ? __ldg(lse2c + ci) : 0.f;
    const float Dv = valid ? __ldg(Dc + ci) : 0.f;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
    const uint64_t c2 = f32x2(sl2, sl2), nl2 = f32x2(-l2, -l2), nD2 = f32x2(-Dv, -Dv);
    const Exp2PolyConsts pc = exp2_poly_consts();
    if (QT && nt > 0) {
      // row i of the Q tile (swizzled smem, TMA) -> TMEM lane i: this warp's
      // 32 elements 32 hf .. 32 hf + 31 as 16 bf16-pair columns
      mbar_wait(B(B_QD), 0);
      uint32_t qw[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 v = *reinterpret_cast<const uint4*>(smem + OFF_Q + (hf >> 1) * ATOM + swz(i, (hf & 1) * 4 + c));
        qw[4 * c] = v.x; qw[4 * c + 1] = v.y; qw[4 * c + 2] = v.z; qw[4 * c + 3] = v.w;
      }
      __syncwarp();
      tmem_st16(tl + COL_Q + hf * 16, qw);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(B(B_QT));
    }
    for (int j = 0; j < nt; ++j) {
      mbar_wait(B(B_SF), j & 1);
      tc_fence_after();
      uint32_t s[32], p[32];
      __syncwarp();
      tmem_ld32(tl + COL_S + cb, s);
      tmem_ld32(tl + COL_DP + cb, p);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(B(B_SE));  // S / dP of this tile consumed: the next tile's MMAs may overwrite them
      if constexpr (PROBE == 1) {
        if (j > 0) mbar_wait(B(B_DSE), (j - 1) & 1);
        mbar_arrive(B(B_DSF));
        continue;
      }
      const int lim = vis - j * 128;
      // paired FP32 ops: x = s log2e/sqrt(d) - lse2, dS = 2^x (dP - D); the
      // visibility compare only on staircase tiles
      const bool full = __all_sync(0xffffffffu, lim >= cb + 32);
      uint32_t pk[16];
      auto math = [&](auto full_c) {  // separate full / staircase code (issue-bound loop)
        constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const uint64_t xl = ffma2(f32x2(__uint_as_float(s[c]), __uint_as_float(s[c + 1])), c2, nl2);
          float p0, p1;
          if (dq_poly(c >> 1)) {
            const uint64_t ex = exp2_poly_pair(xl, pc);
            p0 = f32x2_lo(ex);
            p1 = f32x2_hi(ex);
          } else {
            p0 = fast_exp2(f32x2_lo(xl));
            p1 = fast_exp2(f32x2_hi(xl));
          }
          if constexpr (!FULL) {
            p0 = (cb + c < lim) ? p0 : 0.f;
            p1 = (cb + c + 1 < lim) ? p1 : 0.f;
          }
          const uint64_t ds =
              fmul2(f32x2(p0, p1), fadd2(f32x2(__uint_as_float(p[c]), __uint_as_float(p[c + 1])), nD2));
          pk[c / 2] = pack_bf16x2(f32x2_lo(ds), f32x2_hi(ds));
        }
      };
      if (full) math(std::true_type{}); else math(std::false_type{});
      if (j > 0) mbar_wait(B(B_DSE), (j - 1) & 1);  // dQ MMA of j-1 finished reading dS
      tc_fence_after();
      // dS of keys [cb, cb + 32) as 16 packed columns: keys 16kk .. 16kk + 15
      // are TMEM columns COL_DS + 8kk, the A operand of dQ K-step kk
      __syncwarp();
      tmem_st16(tl + COL_DS + hf * 16, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(B(B_DSF));
    }
    if (nt > 0) {
      mbar_wait(B(B_DSE), (nt - 1) & 1);
      tc_fence_after();
      const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(D)));
      const int pos = valid ? __ldg(rows + (size_t)h * N + r0 + i) : 0;
      uint32_t o[32];
      __syncwarp();
      tmem_ld32(tl + COL_DQ + cb, o);
      tmem_wait_ld();
      if (valid) {
        if (dq_bf16) {  // the training dtype directly: no fp32 round trip through HBM
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(dQ) + ((size_t)h * N + pos) * D + cb);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float* f = reinterpret_cast<const float*>(o + 8 * q);
            dst[q] = make_uint4(pack_bf16x2(f[0] * scale, f[1] * scale), pack_bf16x2(f[2] * scale, f[3] * scale),
                                pack_bf16x2(f[4] * scale, f[5] * scale), pack_bf16x2(f[6] * scale, f[7] * scale));
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(dQ) + ((size_t)h * N + pos) * D + cb);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            dst[q] = make_float4(__uint_as_float(o[4 * q]) * scale, __uint_as_float(o[4 * q + 1]) * scale,
                                 __uint_as_float(o[4 * q + 2]) * scale, __uint_as_float(o[4 * q + 3]) * scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#ifdef OMNI_VARIANTS  // the shared-memory P^T dkv kernel (v1), kept for A/B measurements
// ------------------------------------------------------------------ dkv
namespace dkv {
constexpr int BR = 64;                     // Q rows per inner tile
constexpr uint32_t QATOM = BR * 128;       // 64 rows x 128 B
constexpr uint32_t QTILE = 2 * QATOM;      // 64 x 128 bf16
constexpr uint32_t OFF_K = 0, OFF_V = TILE, OFF_Q = 2 * TILE, OFF_DO = OFF_Q + 2 * QTILE;
constexpr uint32_t OFF_PT = OFF_DO + 2 * QTILE;  // [128 keys][64 rows] bf16, one swizzle atom wide
constexpr uint32_t OFF_DST = OFF_PT + 128 * 128;
constexpr uint32_t OFF_INFO = OFF_DST + 128 * 128;  // [2][3][64] f32/i32
constexpr uint32_t OFF_BAR = OFF_INFO + 2 * 3 * BR * 4;
enum { B_KV = 0, B_QF = 1, B_QE = 3, B_IF = 5, B_IE = 7, B_SF = 9, B_SE = 10, B_PF = 11, B_PE = 12, B_N = 13 };
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * B_N;
constexpr uint32_t SMEM = OFF_TMEM + 16 + 1024;
constexpr uint32_t COL_S = 0, COL_DP = 64, COL_DV = 128, COL_DK = 256;
}  // namespace dkv

// Iteration space of one KV tile: for each Q head of the group, the 64-row
// compact Q tiles from the first row that can see the tile's first key.
struct DkvIter {
  int h0, rep, first_tile[16], n_tiles[16], total;
};

__global__ void __launch_bounds__(384, 1)
dkv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
           const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
           const int32_t* __restrict__ rows, const int32_t* __restrict__ counts, const int32_t* __restrict__ sel,
           const int32_t* __restrict__ sel_counts, const float* __restrict__ lse2c, const float* __restrict__ Dc,
           const int32_t* __restrict__ visc, int rep, int N, int cap, int capq, float* __restrict__ dK,
           float* __restrict__ dV) {
  using namespace dkv;
  extern __shared__ uint8_t smem_raw[];
  // CTA = (key tile t, group g, Q head g*rep + rs): one Q head per CTA keeps
  // the per-CTA work balanced (early key tiles are seen by every later row);
  // the group's heads accumulate into dK/dV with vector fp32 reductions.
  const int t = blockIdx.x, g = blockIdx.y / rep, rs = blockIdx.y % rep;
  const int nsel = __ldg(sel_counts + g);
  const int k0 = t * 128;
  if (k0 >= nsel) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar = sb + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ DkvIter it;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    const int first_key = __ldg(sel + (size_t)g * N + k0);
    it.h0 = g * rep;
    it.rep = rep;
    int tot = 0;
    for (int r = 0; r < rep; ++r) {
      if (r != rs) {
        it.first_tile[r] = 0;
        it.n_tiles[r] = 0;
        continue;
      }
      const int h = g * rep + r;
      const int cnt = __ldg(counts + h);
      // first compact row whose position >= first_key (it sees key k0)
      const int32_t* rh = rows + (size_t)h * N;
      int lo = 0, hi = cnt;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(rh + mid) < first_key) lo = mid + 1; else hi = mid;
      }
      it.first_tile[r] = lo / BR;
      it.n_tiles[r] = max(0, (cnt + BR - 1) / BR - lo / BR);
      tot += it.n_tiles[r];
    }
    it.total = tot;
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(B(B_KV), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(B(B_QF + s), 1);
      mbar_init(B(B_QE + s), 1);
      mbar_init(B(B_IF + s), 64);
      mbar_init(B(B_IE + s), 256);
    }
    mbar_init(B(B_SF), 1);
    mbar_init(B(B_SE), 256);
    mbar_init(B(B_PF), 256);
    mbar_init(B(B_PE), 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = it.total;
  // iteration index -> (head, compact Q tile)
  auto decode_it = [&](int k, int& h, int& qt) {
    int r = 0;
    while (k >= it.n_tiles[r]) { k -= it.n_tiles[r]; ++r; }
    h = it.h0 + r;
    qt = it.first_tile[r] + k;
  };

  if (warp == 0) {
    if (lane == 0 && total > 0) {
      mbar_expect_tx(B(B_KV), 2 * TILE);
      const int kr = g * cap + k0;
      tma_load_2d(sb + OFF_K, &tm_k, B(B_KV), 0, kr);
      tma_load_2d(sb + OFF_K + ATOM, &tm_k, B(B_KV), 64, kr);
      tma_load_2d(sb + OFF_V, &tm_v, B(B_KV), 0, kr);
      tma_load_2d(sb + OFF_V + ATOM, &tm_v, B(B_KV), 64, kr);
      for (int k = 0; k < total; ++k) {
        const int s = k & 1;
        int h, qt;
        decode_it(k, h, qt);
        const int row = h * capq + qt * BR;
        if (k >= 2) mbar_wait(B(B_QE + s), ((k >> 1) - 1) & 1);
        mbar_expect_tx(B(B_QF + s), 2 * QTILE);
        tma_load_2d(sb + OFF_Q + s * QTILE, &tm_q, B(B_QF + s), 0, row);
        tma_load_2d(sb + OFF_Q + s * QTILE + QATOM, &tm_q, B(B_QF + s), 64, row);
        tma_load_2d(sb + OFF_DO + s * QTILE, &tm_do, B(B_QF + s), 0, row);
        tma_load_2d(sb + OFF_DO + s * QTILE + QATOM, &tm_do, B(B_QF + s), 64, row);
      }
    }
  } else if (warp == 1) {
    // whole warp runs the schedule; elect.sync picks the issuing lane
    if (total > 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, BR, 0, 0);
      constexpr uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);
      const uint64_t dk0 = sdesc_sw128(sb + OFF_K, 16, 1024), dv0 = sdesc_sw128(sb + OFF_V, 16, 1024);
      const uint64_t dqs0 = sdesc_sw128(sb + OFF_Q, 16, 1024), ddos0 = sdesc_sw128(sb + OFF_DO, 16, 1024);
      const uint64_t dqm0 = sdesc_sw128(sb + OFF_Q, QATOM, 1024), ddom0 = sdesc_sw128(sb + OFF_DO, QATOM, 1024);
      const uint64_t dpt0 = sdesc_sw128(sb + OFF_PT, 16, 1024), ddst0 = sdesc_sw128(sb + OFF_DST, 16, 1024);
      auto issue_s = [&](int k) {
        const int s = k & 1;
        mbar_wait(B(B_QF + s), (k >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t oa = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((s * QTILE + (kk >> 2) * QATOM + (kk & 3) * 32)) >> 4;
          umma_bf16_ws(tmem + COL_S, dk0 + oa, dqs0 + ob, id_s, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t oa = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((s * QTILE + (kk >> 2) * QATOM + (kk & 3) * 32)) >> 4;
          umma_bf16_ws(tmem + COL_DP, dv0 + oa, ddos0 + ob, id_s, kk > 0);
        }
        umma_commit_ws(B(B_SF));
      };
      mbar_wait(B(B_KV), 0);
      issue_s(0);
      for (int k = 0; k < total; ++k) {
        const int s = k & 1;
        mbar_wait(B(B_SE), k & 1);
        if (k + 1 < total) issue_s(k + 1);
        mbar_wait(B(B_PF), k & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // K = 64 rows, 16 per MMA
          umma_bf16_ws(tmem + COL_DV, dpt0 + ((kk * 32) >> 4), ddom0 + ((s * QTILE + kk * 2048) >> 4), id_acc,
                       (k > 0 || kk > 0) ? 1u : 0u);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          umma_bf16_ws(tmem + COL_DK, ddst0 + ((kk * 32) >> 4), dqm0 + ((s * QTILE + kk * 2048) >> 4), id_acc,
                       (k > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_ws(B(B_QE + s));
        umma_commit_ws(B(B_PE));
      }
    }
  } else if (warp == 2 || warp == 3) {
    // row-info loader: lse2 / D / vis of the 64 rows of each Q tile -> smem ring
    const int r = threadIdx.x - 64;
    float* info = reinterpret_cast<float*>(smem + OFF_INFO);
    for (int k = 0; k < total; ++k) {
      const int s = k & 1;
      int h, qt;
      decode_it(k, h, qt);
      if (k >= 2) mbar_wait(B(B_IE + s), ((k >> 1) - 1) & 1);
      const size_t ci = (size_t)h * capq + qt * BR + r;
      info[(s * 3 + 0) * BR + r] = __ldg(lse2c + ci);
      info[(s * 3 + 1) * BR + r] = __ldg(Dc + ci);
      reinterpret_cast<int*>(info)[(s * 3 + 2) * BR + r] = __ldg(visc + ci);
      mbar_arrive(B(B_IF + s));
    }
  } else if (warp >= 4) {
    // softmax-gradient warps: thread j <-> key k0 + j <-> TMEM lane j; two
    // warps per lane quarter, each 32 of the 64 Q-row columns
    const int hf = (warp - 4) >> 2;
    const int j = (warp & 3) * 32 + lane;
    const int kj = k0 + j;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
    const float* info = reinterpret_cast<const float*>(smem + OFF_INFO);
    uint8_t* pt_gen = smem + OFF_PT;
    uint8_t* dst_gen = smem + OFF_DST;
    const int cb = hf * 32;
    for (int k = 0; k < total; ++k) {
      const int s = k & 1;
      mbar_wait(B(B_SF), k & 1);
      tc_fence_after();
      uint32_t sv[32], dp[32];
      __syncwarp();
      tmem_ld32(tl + COL_S + cb, sv);
      tmem_ld32(tl + COL_DP + cb, dp);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(B(B_SE));
      mbar_wait(B(B_IF + s), (k >> 1) & 1);
      const float* l2 = info + (s * 3 + 0) * BR + cb;
      const float* dd = info + (s * 3 + 1) * BR + cb;
      const int* vv = reinterpret_cast<const int*>(info) + (s * 3 + 2) * BR + cb;
      uint32_t pp[16], pd[16];
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const float p0 = (kj < vv[c]) ? fast_exp2(__uint_as_float(sv[c]) * sl2 - l2[c]) : 0.f;
        const float p1 = (kj < vv[c + 1]) ? fast_exp2(__uint_as_float(sv[c + 1]) * sl2 - l2[c + 1]) : 0.f;
        pp[c / 2] = pack_bf16x2(p0, p1);
        pd[c / 2] = pack_bf16x2(p0 * (__uint_as_float(dp[c]) - dd[c]), p1 * (__uint_as_float(dp[c + 1]) - dd[c + 1]));
      }
      mbar_arrive(B(B_IE + s));
      if (k > 0) mbar_wait(B(B_PE), (k - 1) & 1);  // previous dV/dK MMAs done with P^T / dS^T
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        *reinterpret_cast<uint4*>(pt_gen + swz(j, hf * 4 + q)) =
            make_uint4(pp[4 * q], pp[4 * q + 1], pp[4 * q + 2], pp[4 * q + 3]);
        *reinterpret_cast<uint4*>(dst_gen + swz(j, hf * 4 + q)) =
            make_uint4(pd[4 * q], pd[4 * q + 1], pd[4 * q + 2], pd[4 * q + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(B(B_PF));
    }
    const bool valid = kj < nsel;
    const int dcb = hf * 64;  // this thread's 64 head-dim columns of dK / dV
    float4* dvr = reinterpret_cast<float4*>(dV + ((size_t)g * cap + kj) * D + dcb);
    float4* dkr = reinterpret_cast<float4*>(dK + ((size_t)g * cap + kj) * D + dcb);
    if (total > 0) {
      mbar_wait(B(B_PE), (total - 1) & 1);
      tc_fence_after();
      const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(D)));
#pragma unroll
      for (int c4 = 0; c4 < 2; ++c4) {
        uint32_t a[32], b[32];
        __syncwarp();
        tmem_ld32(tl + COL_DV + dcb + c4 * 32, a);
        tmem_ld32(tl + COL_DK + dcb + c4 * 32, b);
        tmem_wait_ld();
        if (valid) {  // heads of the group reduce into the zero-initialised dK / dV
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            red_add_v4(dvr + c4 * 8 + q, __uint_as_float(a[4 * q]), __uint_as_float(a[4 * q + 1]),
                       __uint_as_float(a[4 * q + 2]), __uint_as_float(a[4 * q + 3]));
            red_add_v4(dkr + c4 * 8 + q, __uint_as_float(b[4 * q]) * scale, __uint_as_float(b[4 * q + 1]) * scale,
                       __uint_as_float(b[4 * q + 2]) * scale, __uint_as_float(b[4 * q + 3]) * scale);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

#endif  // OMNI_VARIANTS

// ------------------------------------------------------------------ dkv v2
// dkv with 128-row Q tiles and P^T / dS^T kept in TMEM. Per (key tile, Q
// tile k): S^T = K Q^T and dP^T = V dO^T (SS, M = 128 keys, N = 128 rows) into
// TMEM; 16 gradient warps (four per lane quarter, 32 row columns each) read
// their S^T / dP^T columns, release them, and write P^T and dS^T as bf16
// pairs over their own dP^T columns; dV += P^T dO and dK += dS^T Q are
// TS-mode MMAs (A from TMEM). No P^T / dS^T round trip through shared memory
// (the old kernel's bandwidth limit), and S^T(k+1) is computed while tile k's
// gradients are formed (only dP^T(k+1) waits for dV / dK(k)).
namespace dkv2 {
constexpr int BR = 128;
constexpr uint32_t OFF_K = 0, OFF_V = TILE, OFF_Q = 2 * TILE, OFF_DO = 4 * TILE;  // Q, dO: 2 stages each
constexpr int NI = 4;                                                             // row-info ring depth
constexpr uint32_t OFF_INFO = 6 * TILE;                                           // [NI][3][128]
constexpr uint32_t OFF_BAR = OFF_INFO + NI * 3 * BR * 4;
// B_TF: S^T(k) ready; B_SF: dP^T(k) ready; B_SE: S^T(k) read by every gradient thread
// Q and dO have separate rings (B_QF/B_QE, B_DF/B_DE): dK(k), the last use
// of Q(k), runs before dV(k), so the Q stage the next S^T needs frees early.
enum { B_KV = 0, B_QF = 1, B_QE = 3, B_IF = 5, B_IE = 5 + NI, B_SF = 5 + 2 * NI, B_SE, B_PF, B_PE, B_TF, B_DF,
       B_DE = B_DF + 2, B_N = B_DE + 2 };
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * B_N;
constexpr uint32_t SMEM = OFF_TMEM + 16 + 1024;
constexpr uint32_t COL_S = 0, COL_DP = 128, COL_DV = 256, COL_DK = 384;
constexpr int NTHREADS = 640;  // TMA, MMA, 2 row-info warps, 16 gradient warps
}  // namespace dkv2

// PROBE (profiling only, OMNI_BWD_PROBE): 1 = gradient warps release P^T /
// dS^T without computing them (the MMA / TMA pipeline floor); 2 = the
// gradient arithmetic without the exponentials (MUFU share); 3 = per-phase
// cycle sums (lane 0 of each gradient warp and of the MMA warp) into
// g_bwd_trace, read back with omni_debug_bwd_trace.
__device__ unsigned long long g_bwd_trace[8];
template <int PROBE>
__global__ void __launch_bounds__(dkv2::NTHREADS, 1)
dkv2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
            const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
            const int32_t* __restrict__ rows, const int32_t* __restrict__ counts, const int32_t* __restrict__ sel,
            const int32_t* __restrict__ sel_counts, const float* __restrict__ lse2c, const float* __restrict__ Dc,
            const int32_t* __restrict__ visc, int rep, int N, int cap, int capq, float* __restrict__ dK,
            float* __restrict__ dV) {
  using namespace dkv2;
  extern __shared__ uint8_t smem_raw[];
  // CTA = (key tile t, group g, Q head g*rep + rs), as dkv_kernel.
  const int t = blockIdx.x, g = blockIdx.y / rep, rs = blockIdx.y % rep;
  const int nsel = __ldg(sel_counts + g);
  const int k0 = t * 128;
  if (k0 >= nsel) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  const uint32_t bar = sb + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ int s_first, s_total;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = g * rep + rs;
  if (warp == 0) {
    // first compact row whose position >= first_key (it sees key k0): the
    // rows below it, by a warp-cooperative search (32 pivots per level; a
    // per-thread binary search is ~14 dependent L2 loads, ~0.5 us each while
    // the other SMs stream)
    const int first_key = __ldg(sel + (size_t)g * N + k0);
    const int cnt = __ldg(counts + h);
    const int lo = count_le_warp(rows + (size_t)h * N, cnt, first_key - 1, true);
    if (lane == 0) {
      s_first = lo / BR;
      s_total = max(0, (cnt + BR - 1) / BR - lo / BR);
    }
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(B(B_KV), 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(B(B_QF + s), 1);
      mbar_init(B(B_QE + s), 1);
      mbar_init(B(B_DF + s), 1);
      mbar_init(B(B_DE + s), 1);
    }
    for (int s = 0; s < NI; ++s) {
      mbar_init(B(B_IF + s), 64);
      mbar_init(B(B_IE + s), 512);
    }
    mbar_init(B(B_SF), 1);
    mbar_init(B(B_TF), 1);
    mbar_init(B(B_SE), 512);
    mbar_init(B(B_PF), 512);
    mbar_init(B(B_PE), 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = s_total, first = s_first;

  if (warp == 0) {
    if (lane == 0 && total > 0) {
      mbar_expect_tx(B(B_KV), 2 * TILE);
      const int kr = g * cap + k0;
      tma_load_2d(sb + OFF_K, &tm_k, B(B_KV), 0, kr);
      tma_load_2d(sb + OFF_K + ATOM, &tm_k, B(B_KV), 64, kr);
      tma_load_2d(sb + OFF_V, &tm_v, B(B_KV), 0, kr);
      tma_load_2d(sb + OFF_V + ATOM, &tm_v, B(B_KV), 64, kr);
      for (int k = 0; k < total; ++k) {
        const int s = k & 1;
        const int row = h * capq + (first + k) * BR;
        if (k >= 2) mbar_wait(B(B_QE + s), ((k >> 1) - 1) & 1);
        mbar_expect_tx(B(B_QF + s), TILE);
        tma_load_2d(sb + OFF_Q + s * TILE, &tm_q, B(B_QF + s), 0, row);
        tma_load_2d(sb + OFF_Q + s * TILE + ATOM, &tm_q, B(B_QF + s), 64, row);
        if (k >= 2) mbar_wait(B(B_DE + s), ((k >> 1) - 1) & 1);
        mbar_expect_tx(B(B_DF + s), TILE);
        tma_load_2d(sb + OFF_DO + s * TILE, &tm_do, B(B_DF + s), 0, row);
        tma_load_2d(sb + OFF_DO + s * TILE + ATOM, &tm_do, B(B_DF + s), 64, row);
      }
      // observe the last ring phases (every mbarrier phase is waited on)
      for (int k = total > 2 ? total - 2 : 0; k < total; ++k) {
        mbar_wait(B(B_QE + (k & 1)), (k >> 1) & 1);
        mbar_wait(B(B_DE + (k & 1)), (k >> 1) & 1);
      }
    }
  } else if (warp == 1) {
    // whole warp runs the schedule; elect.sync picks the issuing lane
    if (total > 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, BR, 0, 0);
      constexpr uint32_t id_acc = idesc_bf16_f32(128, 128, 0, 1);
      const uint64_t dk0 = sdesc_sw128(sb + OFF_K, 16, 1024), dv0 = sdesc_sw128(sb + OFF_V, 16, 1024);
      const uint64_t dq0 = sdesc_sw128(sb + OFF_Q, 16, 1024), ddo0 = sdesc_sw128(sb + OFF_DO, 16, 1024);
      const uint64_t dqm0 = sdesc_sw128(sb + OFF_Q, ATOM, 1024), ddom0 = sdesc_sw128(sb + OFF_DO, ATOM, 1024);
      uint32_t tw_qf = 0;
      auto issue_st = [&](int k) {  // S^T(k) = K Q(k)^T -> COL_S
        const int s = k & 1;
        const uint32_t q0 = clock();
        mbar_wait(B(B_QF + s), (k >> 1) & 1);
        if constexpr (PROBE == 3) tw_qf += clock() - q0;
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + COL_S, dk0 + off, dq0 + ((s * TILE) >> 4) + off, id_s, kk > 0);
        }
        umma_commit_ws(B(B_TF));
      };
      auto issue_dpt = [&](int k) {  // dP^T(k) = V dO(k)^T -> COL_DP
        const int s = k & 1;
        mbar_wait(B(B_DF + s), (k >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + COL_DP, dv0 + off, ddo0 + ((s * TILE) >> 4) + off, id_s, kk > 0);
        }
        umma_commit_ws(B(B_SF));
      };
      mbar_wait(B(B_KV), 0);
      issue_st(0);
      issue_dpt(0);
      uint32_t tw_se = 0, tw_pf = 0;
      for (int k = 0; k < total; ++k) {
        const int s = k & 1;
        const uint32_t t0 = clock();
        mbar_wait(B(B_SE), k & 1);  // S^T(k) read by every gradient thread
        tc_fence_after();
        const uint32_t t1 = clock();
        if (k + 1 < total) issue_st(k + 1);
        const uint32_t t2 = clock();
        mbar_wait(B(B_PF), k & 1);  // P^T(k), dS^T(k) in TMEM
        if constexpr (PROBE == 3) {
          tw_se += t1 - t0;
          tw_pf += clock() - t2;
        }
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dK += dS^T Q, K = 128 rows, 16 per MMA
          const uint32_t ac = COL_DP + 32u * (kk >> 1) + 16u + 8u * (kk & 1);
          umma_bf16_ts_ws(tmem + COL_DK, tmem + ac, dqm0 + ((s * TILE + kk * 2048) >> 4), id_acc,
                          (k > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_ws(B(B_QE + s));  // Q(k) free: the Q(k + 2) load starts under dV(k)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dV += P^T dO
          const uint32_t ac = COL_DP + 32u * (kk >> 1) + 8u * (kk & 1);
          umma_bf16_ts_ws(tmem + COL_DV, tmem + ac, ddom0 + ((s * TILE + kk * 2048) >> 4), id_acc,
                          (k > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit_ws(B(B_DE + s));
        umma_commit_ws(B(B_PE));
        if (k + 1 < total) issue_dpt(k + 1);  // after dV / dK(k): they read the dP^T region
      }
      if constexpr (PROBE == 3) {
        if (lane == 0) {
          (void)tw_se;
          (void)tw_pf;
          atomicAdd(&g_bwd_trace[3], (unsigned long long)tw_qf);  // (overrides the gradient st slot)
          atomicAdd(&g_bwd_trace[7], (unsigned long long)total);
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // row-info loader: lse2 / D / vis of the 128 rows of each Q tile -> smem ring
    const int r = threadIdx.x - 64;  // rows r and r + 64
    float* info = reinterpret_cast<float*>(smem + OFF_INFO);
    for (int k = 0; k < total; ++k) {
      const int s = k % NI;  // loaded NI - 1 Q tiles ahead of its use (global latency)
      if (k >= NI) mbar_wait(B(B_IE + s), ((k / NI) - 1) & 1);
      for (int rr = r; rr < BR; rr += 64) {
        const size_t ci = (size_t)h * capq + (first + k) * BR + rr;
        info[(s * 3 + 0) * BR + rr] = -__ldg(lse2c + ci);  // negated: one FFMA2 / FADD2 per pair
        info[(s * 3 + 1) * BR + rr] = -__ldg(Dc + ci);
        reinterpret_cast<int*>(info)[(s * 3 + 2) * BR + rr] = __ldg(visc + ci);
      }
      mbar_arrive(B(B_IF + s));
    }
  } else {
    // gradient warps: thread j <-> key k0 + j <-> TMEM lane j; four warps per
    // lane quarter, each 32 of the 128 Q-row columns
    const int cq = (warp - 4) >> 2;
    const int j = (warp & 3) * 32 + lane;
    const int kj = k0 + j;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
    const float* info = reinterpret_cast<const float*>(smem + OFF_INFO);
    const int cb = cq * 32;
    uint32_t tg[5] = {0, 0, 0, 0, 0};
    for (int k = 0; k < total; ++k) {
      // Two phases: P^T from S^T as soon as S^T(k) is ready — it overlaps
      // dV / dK(k-1) and dP^T(k) on the tensor core — then only the cheap
      // dS^T = P^T (dP^T - D) waits for dP^T(k).
      const uint32_t c0 = clock();
      mbar_wait(B(B_TF), k & 1);
      tc_fence_after();
      const uint32_t c1 = clock();
      uint32_t sv[32];
      __syncwarp();
      tmem_ld32(tl + COL_S + cb, sv);
      tmem_wait_ld();
      const uint32_t c2c = clock();
      tc_fence_before();
      mbar_arrive(B(B_SE));
      if constexpr (PROBE == 1) {
        mbar_wait(B(B_IF + k % NI), (k / NI) & 1);
        mbar_arrive(B(B_IE + k % NI));
        mbar_wait(B(B_SF), k & 1);
        mbar_arrive(B(B_PF));
        continue;
      }
      const int si = k % NI;
      mbar_wait(B(B_IF + si), (k / NI) & 1);
      const uint32_t c2i = clock();
      if constexpr (PROBE == 3) tg[4] += c2i - c2c;
      // pairs of rows on the paired FP32 pipe: x = s log2e/sqrt(d) - lse2,
      // P = 2^x (0 beyond a row's visible keys), dS = P (dP - D)
      const uint32_t a_l2 = smem_u32(info + (si * 3 + 0) * BR + cb), a_dd = smem_u32(info + (si * 3 + 1) * BR + cb);
      const uint32_t a_vv = smem_u32(info + (si * 3 + 2) * BR + cb);
      // rows ascend, so do their visible-key counts: every one of this
      // thread's 32 rows sees key kj iff the first one does
      const bool full = __all_sync(0xffffffffu, kj < lds_i4(a_vv).x);
      const uint64_t c2 = f32x2(sl2, sl2);
      const Exp2PolyConsts pc = exp2_poly_consts();
      uint32_t pp[16], pd[16];
      // phase 1 (P^T, bf16 pairs). Separate instantiations for full and
      // staircase tiles: predicated-off selects would still take issue slots
      auto pmath = [&](auto full_c) {
        constexpr bool FULL = decltype(full_c)::value;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 L = lds_f4(a_l2 + 16 * c4);
          int4 Vi;
          if constexpr (!FULL) Vi = lds_i4(a_vv + 16 * c4);
#pragma unroll
          for (int hp = 0; hp < 2; ++hp) {
            const int c = 4 * c4 + 2 * hp;
            const uint64_t xl = ffma2(f32x2(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), c2,
                                      hp ? f32x2(L.z, L.w) : f32x2(L.x, L.y));
            float p0 = f32x2_lo(xl), p1 = f32x2_hi(xl);
            if constexpr (PROBE != 2) {
              if (bwd_poly(c >> 1)) {
                const uint64_t ex = exp2_poly_pair(xl, pc);
                p0 = f32x2_lo(ex);
                p1 = f32x2_hi(ex);
              } else {
                p0 = fast_exp2(p0);
                p1 = fast_exp2(p1);
              }
            }
            if constexpr (!FULL) {
              p0 = kj < (hp ? Vi.z : Vi.x) ? p0 : 0.f;
              p1 = kj < (hp ? Vi.w : Vi.y) ? p1 : 0.f;
            }
            pp[c / 2] = pack_bf16x2(p0, p1);
          }
        }
      };
      if (full) pmath(std::true_type{}); else pmath(std::false_type{});
      // phase 2: dS^T = P^T (dP^T - D) with the bf16 P^T (the values dV uses)
      const uint32_t cs0 = clock();
      mbar_wait(B(B_SF), k & 1);
      // observe the dV / dK(k-1) phase (complete: dP^T(k) was issued after it)
      if (k > 0) mbar_wait(B(B_PE), (k - 1) & 1);
      const uint32_t cs1 = clock();
      tc_fence_after();
      uint32_t dp[32];
      __syncwarp();
      tmem_ld32(tl + COL_DP + cb, dp);
      tmem_wait_ld();
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 Dn = lds_f4(a_dd + 16 * c4);
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
          const int c = 4 * c4 + 2 * hp;
          const uint32_t w = pp[c / 2];
          const uint64_t pv = f32x2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
          const uint64_t ds = fmul2(pv, fadd2(f32x2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])),
                                              hp ? f32x2(Dn.z, Dn.w) : f32x2(Dn.x, Dn.y)));
          pd[c / 2] = pack_bf16x2(f32x2_lo(ds), f32x2_hi(ds));
        }
      }
      mbar_arrive(B(B_IE + si));
      const uint32_t c3 = clock();
      // P^T / dS^T over this thread's own (already read) dP^T columns; dV / dK(k-1)
      // finished reading the region before dP^T(k) was computed (in-order tensor pipe)
      __syncwarp();
      tmem_st16(tl + COL_DP + cb, pp);
      tmem_st16(tl + COL_DP + cb + 16, pd);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(B(B_PF));
      if constexpr (PROBE == 3) {
        const uint32_t c4 = clock();
        tg[0] += c1 - c0;      // wait S^T
        tg[1] += cs0 - c2c;    // ld S^T + info + P^T phase
        tg[2] += cs1 - cs0;    // wait dP^T
        tg[3] += c4 - cs1;     // ld dP^T, dS^T, stores, release
      }
    }
    if constexpr (PROBE == 3) {
      if (lane == 0) {
        for (int q = 0; q < 3; ++q) atomicAdd(&g_bwd_trace[q], (unsigned long long)tg[q]);
        atomicAdd(&g_bwd_trace[4], (unsigned long long)tg[3]);  // (overrides the MMA SE wait slot)
        atomicAdd(&g_bwd_trace[6], (unsigned long long)total);
        atomicAdd(&g_bwd_trace[5], (unsigned long long)tg[4]);  // (overrides the MMA PF wait slot)
      }
    }
    const bool valid = kj < nsel;
    const int dcb = cq * 32;  // this thread's 32 head-dim columns of dK / dV
    float4* dvr = reinterpret_cast<float4*>(dV + ((size_t)g * cap + kj) * D + dcb);
    float4* dkr = reinterpret_cast<float4*>(dK + ((size_t)g * cap + kj) * D + dcb);
    if (total > 0) {
      mbar_wait(B(B_PE), (total - 1) & 1);
      tc_fence_after();
      const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(D)));
      uint32_t a[32], b[32];
      __syncwarp();
      tmem_ld32(tl + COL_DV + dcb, a);
      tmem_ld32(tl + COL_DK + dcb, b);
      tmem_wait_ld();
      if (valid) {  // heads of the group reduce into the zero-initialised dK / dV
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          red_add_v4(dvr + q, __uint_as_float(a[4 * q]), __uint_as_float(a[4 * q + 1]), __uint_as_float(a[4 * q + 2]),
                     __uint_as_float(a[4 * q + 3]));
          red_add_v4(dkr + q, __uint_as_float(b[4 * q]) * scale, __uint_as_float(b[4 * q + 1]) * scale,
                     __uint_as_float(b[4 * q + 2]) * scale, __uint_as_float(b[4 * q + 3]) * scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace bwd
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

static inline int capq_of(int n) { return ((n + 127) / 128) * 128; }

extern "C" size_t omni_sparse_attn_bwd_workspace(int n_q_heads, int seq_len) {
  const size_t rows = (size_t)n_q_heads * capq_of(seq_len);
  return rows * bwd::D * 2 * 2 + rows * 4 * 3 + 1024;
}

extern "C" int omni_sparse_attn_bwd_ex(const void* Q, const void* K_sel, const void* V_sel, const void* O,
                                       const void* dO, const float* lse, const int32_t* rows, const int32_t* counts,
                                       const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                                       int n_kv_heads, int seq_len, int head_dim, int cap, int dq_dtype, void* dQ,
                                       float* dK_sel, float* dV_sel, float* dV_sink, void* workspace, void* stream) {
  omni_begin();
  OMNI_CHECK(dq_dtype == OMNI_DTYPE_F32 || dq_dtype == OMNI_DTYPE_BF16, OMNI_E_PARAM, "dQ must be f32 or bf16");
  OMNI_CHECK(head_dim == 128, OMNI_E_SHAPE, "sparse attention backward requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(n_q_heads / n_kv_heads <= 16, OMNI_E_SHAPE, "at most 16 Q heads per KV group");
  OMNI_CHECK(cap >= 128 && cap % 128 == 0, OMNI_E_SHAPE, "cap must be a positive multiple of 128");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rep = n_q_heads / n_kv_heads;
  const int capq = capq_of(seq_len);
  const size_t crow = (size_t)n_q_heads * capq;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  __nv_bfloat16* Qc = reinterpret_cast<__nv_bfloat16*>(ws);
  __nv_bfloat16* dOc = Qc + crow * bwd::D;
  float* lse2c = reinterpret_cast<float*>(dOc + crow * bwd::D);
  float* Dc = lse2c + crow;
  int32_t* visc = reinterpret_cast<int32_t*>(Dc + crow);
  const size_t dq_esz = dq_dtype == OMNI_DTYPE_BF16 ? 2 : 4;
  OMNI_CUDA_TRY(cudaMemsetAsync(dQ, 0, dq_esz * (size_t)n_q_heads * seq_len * head_dim, st));
  OMNI_CUDA_TRY(cudaMemsetAsync(dK_sel, 0, sizeof(float) * (size_t)n_kv_heads * cap * head_dim, st));
  OMNI_CUDA_TRY(cudaMemsetAsync(dV_sel, 0, sizeof(float) * (size_t)n_kv_heads * cap * head_dim, st));
  OMNI_CUDA_TRY(cudaMemsetAsync(dV_sink, 0, sizeof(float) * (size_t)n_kv_heads * head_dim, st));
  bwd::bwd_prep_kernel<<<dim3((capq + 255) / 256, n_q_heads), 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(O),
      static_cast<const __nv_bfloat16*>(dO), lse, rows, counts, selected, sel_counts, seq_len, rep, capq, Qc, dOc,
      lse2c, Dc, visc, dV_sink);
  int rc = omni_launch_check();
  if (rc) return rc;
  CUtensorMap tq128, tdo128, tq64, tdo64, tk, tv;
  if ((rc = omni_make_tmap_rows(&tq128, Qc, crow, 128, 2, 64, 128))) return rc;
  if ((rc = omni_make_tmap_rows(&tdo128, dOc, crow, 128, 2, 64, 128))) return rc;
  if ((rc = omni_make_tmap_rows(&tq64, Qc, crow, 128, 2, 64, 64))) return rc;
  if ((rc = omni_make_tmap_rows(&tdo64, dOc, crow, 128, 2, 64, 64))) return rc;
  if ((rc = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 128))) return rc;
  if ((rc = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 128))) return rc;
  const int n_tiles = capq / 128;
#ifdef OMNI_VARIANTS
  OMNI_CUDA_TRY(omni_smem_attr(bwd::dq_kernel<1>, (int)bwd::dq::SMEM));
  OMNI_CUDA_TRY(omni_smem_attr(bwd::dq_kernel<0, false>, (int)bwd::dq::SMEM));
  OMNI_CUDA_TRY(omni_smem_attr(bwd::dkv_kernel, (int)bwd::dkv::SMEM));
  static const int dq_probe = [] {
    const char* e = getenv("OMNI_DQ_PROBE");
    return e ? atoi(e) : 0;
  }();
  static const bool dq_qt = [] {  // OMNI_DQ_QT=0: Q read from shared memory by the S MMA
    const char* e = getenv("OMNI_DQ_QT");
    return !(e && atoi(e) == 0);
  }();
  auto dq_kern = dq_probe == 1 ? bwd::dq_kernel<1> : dq_qt ? bwd::dq_kernel<0> : bwd::dq_kernel<0, false>;
#else
  auto dq_kern = bwd::dq_kernel<0>;
#endif
  OMNI_CUDA_TRY(omni_smem_attr(bwd::dq_kernel<0>, (int)bwd::dq::SMEM));
  dq_kern<<<n_tiles * n_q_heads, 576, bwd::dq::SMEM, st>>>(tq128, tdo128, tk, tv, rows, counts, lse2c, Dc,
                                                                    visc, n_q_heads, rep, seq_len, cap, capq, n_tiles,
                                                                    dQ, dq_dtype == OMNI_DTYPE_BF16 ? 1 : 0);
  if ((rc = omni_launch_check())) return rc;
#ifdef OMNI_VARIANTS
  // dkv implementation: TMEM-resident P^T / dS^T kernel by default;
  // OMNI_BWD_DKV=v1 selects the shared-memory P^T kernel, OMNI_BWD_PROBE the
  // profiling instances of dkv2.
  static const bool dkv_v1 = [] {
    const char* e = getenv("OMNI_BWD_DKV");
    return e && strcmp(e, "v1") == 0;
  }();
  if (dkv_v1) {
    bwd::dkv_kernel<<<dim3(cap / 128, n_kv_heads * rep), 384, bwd::dkv::SMEM, st>>>(
        tq64, tdo64, tk, tv, rows, counts, selected, sel_counts, lse2c, Dc, visc, rep, seq_len, cap, capq, dK_sel,
        dV_sel);
    return omni_launch_check();
  }
  static const int probe = [] {
    const char* e = getenv("OMNI_BWD_PROBE");
    return e ? atoi(e) : 0;
  }();
  auto kern = probe == 1   ? bwd::dkv2_kernel<1>
              : probe == 2 ? bwd::dkv2_kernel<2>
              : probe == 3 ? bwd::dkv2_kernel<3>
                           : bwd::dkv2_kernel<0>;
#else
  (void)tq64;
  (void)tdo64;
  auto kern = bwd::dkv2_kernel<0>;
#endif
  OMNI_CUDA_TRY(omni_smem_attr(kern, (int)bwd::dkv2::SMEM));
  kern<<<dim3(cap / 128, n_kv_heads * rep), bwd::dkv2::NTHREADS, bwd::dkv2::SMEM, st>>>(
      tq128, tdo128, tk, tv, rows, counts, selected, sel_counts, lse2c, Dc, visc, rep, seq_len, cap, capq, dK_sel,
      dV_sel);
  return omni_launch_check();
}

#ifdef OMNI_VARIANTS
// Profiling support (OMNI_BWD_PROBE=3): copies the 8 dkv phase-cycle sums to
// host memory and resets them.
extern "C" int omni_debug_bwd_trace(unsigned long long* host8) {
  omni_begin();
  OMNI_CUDA_TRY(cudaMemcpyFromSymbol(host8, bwd::g_bwd_trace, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  OMNI_CUDA_TRY(cudaMemcpyToSymbol(bwd::g_bwd_trace, z, sizeof(z)));
  return OMNI_OK;
}
#endif  // OMNI_VARIANTS

extern "C" int omni_sparse_attn_bwd(const void* Q, const void* K_sel, const void* V_sel, const void* O, const void* dO,
                                    const float* lse, const int32_t* rows, const int32_t* counts,
                                    const int32_t* selected, const int32_t* sel_counts, int n_q_heads, int n_kv_heads,
                                    int seq_len, int head_dim, int cap, float* dQ, float* dK_sel, float* dV_sel,
                                    float* dV_sink, void* workspace, void* stream) {
  omni_begin();
  return omni_sparse_attn_bwd_ex(Q, K_sel, V_sel, O, dO, lse, rows, counts, selected, sel_counts, n_q_heads,
                                 n_kv_heads, seq_len, head_dim, cap, OMNI_DTYPE_F32, dQ, dK_sel, dV_sel, dV_sink,
                                 workspace, stream);
}
