// K4: gathered sparse flash-attention forward on tcgen05 / TMEM / TMA.
//
// Replaces sparse_head_attention (prefill.py:89-122). One CTA owns 128
// compacted active query rows of one Q head (rows[h, 128t : 128t+128]) and
// streams its GQA group's compacted selected keys (K_sel / V_sel, produced by
// omni_gather_rows) in tiles of 128. Visibility is the reference's
// `selected[j] <= row` in ORIGINAL positions; since both index lists are
// ascending this is a per-row prefix j < vis(row) = #{selected <= row}, so the
// mask costs one compare per score and the tile loop stops at
// ceil(vis(last row) / 128) (the causal staircase skips the rest).
//
// Operands: Q and P live in TMEM and feed tcgen05.mma as the A operand
// (".kind::f16 [d], [a_tmem], b_desc"); only K and V stream through shared
// memory. With M = 128 SS-mode MMAs both GEMMs sit at the 128 B/clk shared-
// memory operand limit; TMEM A operands halve that traffic.
// Warp roles (384 threads, 1 CTA / SM, ~193 KB smem, 512 TMEM columns):
//   warp 0      TMA producer: K_j, V_j tiles (2 x 64-column SW128 boxes each)
//               into 3-stage K and V rings.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_j = Q K_j^T  (M=128, N=128, K=128; S double-buffered in
//                 TMEM columns [0,128) / [128,256); Q bf16 in [448,512))
//                 O  += P_j V_j  (M=128, N=128, K=128; O in [256,384), P bf16
//                 in [384,448))
//               issue order QK_j, PV_{j-1} so the tensor core computes the
//               next scores while the softmax warps work on the current ones.
//   warps 4-11  softmax / correction / epilogue, two warps per TMEM lane
//               quarter (one per 64-key half; row max exchanged in smem). exp2-domain online softmax with lazy rescaling (the
//               O accumulator is corrected only when the running max grows by
//               more than 2^8), P written bf16 into TMEM (tcgen05.st; the A
//               operand of the PV MMA).
// Epilogue: O / l -> bf16 rows scattered to their original positions; rows
// with no visible key copy V[g, sink] (prefill.py:119-120); LSE side output
// for the backward kernel.
#include <math.h>

#include "common.cuh"

namespace omni {
namespace fwd {

constexpr int BM = 128, BN = 128, D = 128;
constexpr uint32_t ATOM = 128 * 128;  // one 128-row x 128-byte swizzle region
constexpr uint32_t TILE = 2 * ATOM;   // 128 x 128 bf16
constexpr int NST = 3;
constexpr uint32_t OFF_K = 0;                   // NST stages
constexpr uint32_t OFF_V = OFF_K + NST * TILE;  // NST stages
constexpr uint32_t OFF_XCH = OFF_V + NST * TILE;  // row max / sum exchange [3][2][128] f32
constexpr uint32_t OFF_BAR = OFF_XCH + 3 * 2 * 128 * 4;
// barrier slots (8 bytes each)
enum { B_QFULL = 0, B_KFULL = 1, B_KEMPTY = 1 + NST, B_VFULL = 1 + 2 * NST, B_VEMPTY = 1 + 3 * NST,
       B_SFULL = 1 + 4 * NST, B_SEMPTY = 3 + 4 * NST, B_PFULL = 5 + 4 * NST, B_PVDONE = 6 + 4 * NST,
       B_COUNT = 7 + 4 * NST };
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * B_COUNT;
constexpr uint32_t SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + alignment slack
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_O = 256, COL_P = 384, COL_Q = 448;

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  // byte offset of 16-byte chunk `chunk16` (0..7) of `row` in a SW128 atom
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}

__global__ void __launch_bounds__(384, 1)
sparse_fwd_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                  const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                  const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep, int N,
                  int cap, int sel_stride, int sink, int n_tiles_max, __nv_bfloat16* __restrict__ O,
                  float* __restrict__ lse) {
  extern __shared__ uint8_t smem_raw[];
  const int L = blockIdx.x;
  const int h = L % Hq;
  const int tile = n_tiles_max - 1 - L / Hq;  // heaviest (latest rows) tiles first
  const int cnt = __ldg(counts + h);
  const int row0 = tile * BM;
  if (row0 >= cnt) return;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sK = sbase + OFF_K, sV = sbase + OFF_V;
  const uint32_t bar = sbase + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ int s_nt;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;
  const int nrows = min(BM, cnt - row0);
  const int32_t* rows_t = rows + (size_t)h * N + row0;

  if (threadIdx.x == 0) {
    const int last = __ldg(rows_t + nrows - 1);
    s_nt = (count_le(selg, nsel, last) + BN - 1) / BN;
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    mbar_init(B(B_QFULL), 256);
    for (int s = 0; s < NST; ++s) {
      mbar_init(B(B_KFULL + s), 1);
      mbar_init(B(B_KEMPTY + s), 1);
      mbar_init(B(B_VFULL + s), 1);
      mbar_init(B(B_VEMPTY + s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(B(B_SFULL + s), 1);
      mbar_init(B(B_SEMPTY + s), 256);
    }
    mbar_init(B(B_PFULL), 256);
    mbar_init(B(B_PVDONE), 1);
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
  const int nt = s_nt;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0 && nt > 0) {
      const int kr0 = g * cap;
      for (int j = 0; j < nt; ++j) {
        const int s = j % NST;
        const uint32_t ph = ((j / NST) - 1) & 1;
        if (j >= NST) mbar_wait(B(B_KEMPTY + s), ph);
        mbar_expect_tx(B(B_KFULL + s), TILE);
        tma_load_2d(sK + s * TILE, &tm_k, B(B_KFULL + s), 0, kr0 + j * BN);
        tma_load_2d(sK + s * TILE + ATOM, &tm_k, B(B_KFULL + s), 64, kr0 + j * BN);
        if (j >= NST) mbar_wait(B(B_VEMPTY + s), ph);
        mbar_expect_tx(B(B_VFULL + s), TILE);
        tma_load_2d(sV + s * TILE, &tm_v, B(B_VFULL + s), 0, kr0 + j * BN);
        tma_load_2d(sV + s * TILE + ATOM, &tm_v, B(B_VFULL + s), 64, kr0 + j * BN);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    if (lane == 0 && nt > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, D, 0, 1);
      auto pv = [&](int t) {
        const int s = t % NST;
        mbar_wait(B(B_PFULL), t & 1);
        mbar_wait(B(B_VFULL + s), (t / NST) & 1);
        tc_fence_after();
        const uint32_t vb = sV + s * TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t b = sdesc_sw128(vb + kk * 2048, ATOM, 1024);
          umma_bf16_ts(tmem + COL_O, tmem + COL_P + kk * 8, b, idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(B(B_VEMPTY + s));
        umma_commit(B(B_PVDONE));
      };
      mbar_wait(B(B_QFULL), 0);
      tc_fence_after();
      for (int j = 0; j < nt; ++j) {
        const int sb = j & 1;
        const int ks = j % NST;
        if (j >= 2) mbar_wait(B(B_SEMPTY + sb), ((j >> 1) - 1) & 1);
        mbar_wait(B(B_KFULL + ks), (j / NST) & 1);
        tc_fence_after();
        const uint32_t kb = sK + ks * TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t b = sdesc_sw128(kb + (kk >> 2) * ATOM + (kk & 3) * 32, 16, 1024);
          umma_bf16_ts(tmem + sb * BN, tmem + COL_Q + kk * 8, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit(B(B_KEMPTY + ks));
        umma_commit(B(B_SFULL + sb));
        if (j >= 1) pv(j - 1);
      }
      pv(nt - 1);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ softmax warps
    // Two warps per TMEM lane quarter: warp w owns rows 32*(w%4) .. +31 and the
    // key half hf = (w-4)/4 of every tile (columns hf*64 .. +63). The row max is
    // exchanged between the pair through smem + a 64-thread named barrier.
    const int q4 = warp & 3, hf = (warp - 4) >> 2;
    const int i = q4 * 32 + lane;  // row within the tile == TMEM lane
    const bool rvalid = i < nrows;
    const int pos = rvalid ? __ldg(rows_t + i) : 0;
    const int vis = rvalid ? count_le(selg, nsel, pos) : 0;
    const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
    const uint32_t bar_id = 1 + q4;
    float* xch = reinterpret_cast<float*>(smem + OFF_XCH);  // [2 parity][2 halves][128 rows]
    float m_run = -INFINITY, l_run = 0.f;
    if (nt > 0) {
      // Q row half -> TMEM (bf16 pairs, the A operand of S = Q K^T).
      const uint4* qrow = reinterpret_cast<const uint4*>(Q + ((size_t)h * N + pos) * D) + hf * 8;
      uint32_t qv[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 v = rvalid ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
        qv[4 * c] = v.x;
        qv[4 * c + 1] = v.y;
        qv[4 * c + 2] = v.z;
        qv[4 * c + 3] = v.w;
      }
      __syncwarp();
      tmem_st32(tl + COL_Q + hf * 32, qv);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(B(B_QFULL));

      const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
      for (int j = 0; j < nt; ++j) {
        const int sb = j & 1;
        mbar_wait(B(B_SFULL + sb), (j >> 1) & 1);
        tc_fence_after();
        uint32_t sr[64];
        __syncwarp();
        tmem_ld32(tl + sb * BN + hf * 64, sr);
        tmem_ld32(tl + sb * BN + hf * 64 + 32, sr + 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(B(B_SEMPTY + sb));

        // raw-score max over this half (mask only on the staircase boundary)
        const int lim = vis - j * BN - hf * 64;
        if (!__all_sync(0xffffffffu, lim >= 64)) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= lim) sr[c] = __float_as_uint(-INFINITY);
        }
        float mt = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; c += 2) mt = fmax3(mt, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        xch[((j & 1) * 2 + hf) * 128 + i] = mt;
        named_bar_sync(bar_id, 64);
        mt = fmaxf(mt, xch[((j & 1) * 2 + (hf ^ 1)) * 128 + i]);
        const float m_new = fmaxf(m_run, mt * sl2);
        const bool resc = m_new > m_run + 8.0f;
        float alpha = 1.f;
        if (resc) {
          alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
          m_run = m_new;
        }
        const float nmu = (m_run == -INFINITY) ? 0.f : -m_run;
        float rs0 = 0.f, rs1 = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float x0 = fmaf(__uint_as_float(sr[c]), sl2, nmu);
          const float x1 = fmaf(__uint_as_float(sr[c + 1]), sl2, nmu);
          // a quarter of the exponentials on the FMA pipe (MUFU relief)
          const float p0 = ((c & 15) >= 12) ? exp2_poly(x0) : fast_exp2(x0);
          const float p1 = ((c & 15) >= 12) ? exp2_poly(x1) : fast_exp2(x1);
          rs0 += p0;
          rs1 += p1;
          pk[c >> 1] = pack_bf16x2(p0, p1);
        }
        l_run = l_run * alpha + (rs0 + rs1);

        if (j > 0) {
          mbar_wait(B(B_PVDONE), (j - 1) & 1);  // PV_{j-1} finished: O stable, P buffer free
          tc_fence_after();
          if (__any_sync(0xffffffffu, resc)) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              uint32_t o[32];
              __syncwarp();
              tmem_ld32(tl + COL_O + hf * 64 + q * 32, o);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * alpha);
              tmem_st32(tl + COL_O + hf * 64 + q * 32, o);
            }
            tmem_wait_st();
          }
        }
        __syncwarp();
        tmem_st32(tl + COL_P + hf * 32, pk);  // P (bf16 pairs) -> TMEM, A operand of PV
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(B(B_PFULL));
      }
      mbar_wait(B(B_PVDONE), (nt - 1) & 1);
      tc_fence_after();
    }
    // ------------------------------------------------------ epilogue
    xch[(2 * 2 + hf) * 128 + i] = l_run;  // third slot pair holds the row-sum halves
    named_bar_sync(bar_id, 64);
    const float l_tot = l_run + xch[(2 * 2 + (hf ^ 1)) * 128 + i];
    uint32_t o[64];
    if (nt > 0) {
      __syncwarp();
      tmem_ld32(tl + COL_O + hf * 64, o);
      tmem_ld32(tl + COL_O + hf * 64 + 32, o + 32);
      tmem_wait_ld();
    }
    if (rvalid) {
      uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)h * N + pos) * D) + hf * 8;
      if (l_tot > 0.f) {
        const float inv = 1.f / l_tot;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float* f = reinterpret_cast<const float*>(o + 8 * c);
          dst[c] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                              pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
        }
        if (lse && hf == 0) lse[(size_t)h * N + pos] = static_cast<float>(M_LN2) * (m_run + log2f(l_tot));
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(Vorig + ((size_t)g * N + sink) * D) + hf * 8;
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

}  // namespace fwd
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

extern "C" int omni_sparse_attn_fwd(const void* Q, const void* K_sel, const void* V_sel, const void* V,
                                    const int32_t* rows, const int32_t* counts, const int32_t* selected,
                                    const int32_t* sel_counts, int n_q_heads, int n_kv_heads, int seq_len,
                                    int head_dim, int cap, int sink_index, void* O, float* lse, void* stream) {
  OMNI_CHECK(head_dim == 128, OMNI_E_SHAPE, "sparse attention kernel requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(cap >= 128 && cap % 128 == 0, OMNI_E_SHAPE, "cap must be a positive multiple of 128");
  OMNI_CHECK(sink_index >= 0 && sink_index < seq_len, OMNI_E_LAYOUT, "sink_index outside the sequence");
  OMNI_CHECK(seq_len >= 1, OMNI_E_SHAPE, "empty sequence");
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 128);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, 128);
  if (st) return st;
  static bool attr_set = false;
  if (!attr_set) {
    OMNI_CUDA_TRY(cudaFuncSetAttribute(fwd::sparse_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)fwd::SMEM_BYTES));
    attr_set = true;
  }
  const int n_tiles = (seq_len + fwd::BM - 1) / fwd::BM;
  dim3 grid(n_tiles * n_q_heads);
  fwd::sparse_fwd_kernel<<<grid, 384, fwd::SMEM_BYTES, static_cast<cudaStream_t>(stream)>>>(
      tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
      sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index, n_tiles,
      static_cast<__nv_bfloat16*>(O), lse);
  return omni_launch_check();
}
