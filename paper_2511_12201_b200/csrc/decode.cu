// K7: slimmed decode attention over the slim cache (split-K flash decoding).
//
// Replaces classify_decode_query + _fetched_segments + decode_attention
// (decode.py:124-194) for a batch of sequences under GQA rule B.
//
//   decode_flags_kernel   one warp per (sequence, Q head): float64
//                         two-logit classification against the frozen probe
//                         keys (query_select.py:63-68), head 0 forced active.
//   decode_partial_kernel CTA = (2048-key chunk, KV group, sequence), 4 warps x
//                         512 keys. A group's key list is [vision (only if any
//                         of its Q heads is active — the fetch skip of
//                         decode.py:176-190), text, answer]; lazy Q heads see
//                         -inf on vision keys (exclusion, decode.py:12-16).
//                         The group's <= 16 Q heads form the M=16 rows of
//                         mma.sync.m16n8k16 tiles, so each K / V row is read
//                         from HBM exactly once and feeds every head. Head-dim
//                         and key orders inside a tile are permuted so every
//                         lane issues contiguous 16-byte loads straight into
//                         MMA fragments (no shared-memory staging).
//   decode_combine_kernel merges the per-chunk (max, sum, acc) partials.
// HBM-bound: bytes = fetched vision + text + answer K/V rows, once each.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace dec {

constexpr int D = 128;
constexpr int WARP_KEYS = 512;
constexpr int CTA_KEYS = 4 * WARP_KEYS;
constexpr int MAXREP = 8;  // rows of the m16 tile used (rows 8..15 stay zero)

// Text / answer segment lengths: one value for the whole batch, or per
// sequence (serving batches of ragged prompts and answers). The text segment
// of (sequence s, group g) starts at row (s * Hkv + g) * tcap.
struct SegLens {
  const int32_t* tlen;  // nullable: per-sequence text lengths
  const int32_t* alen;  // nullable: per-sequence answer lengths
  int nt, na, tcap;
  __device__ __forceinline__ int text(int s) const { return tlen ? tlen[s] : nt; }
  __device__ __forceinline__ int answer(int s) const { return alen ? alen[s] : na; }
};

__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Classification of the Q heads of KV group g of sequence s, one warp:
// lane l takes head r = l / 4 and head dims (l % 4) * 32 .. +31 (float64,
// query_select.py:63-68 with the decode probe keys), the four partial dots
// meet in a 2-step butterfly (identical on the four lanes). Returns the
// group's active mask (bit r = head g * rep + r) on every lane; head 0 is
// forced active under preserve; flags_override (decode.py:170-173) wins.
__device__ __forceinline__ uint32_t group_flag_mask(const __nv_bfloat16* __restrict__ q,
                                                    const double* __restrict__ k_lazy,
                                                    const double* __restrict__ k_act, int s, int g, int Hq, int Hkv,
                                                    double tau, int preserve,
                                                    const uint8_t* __restrict__ flags_override, double* sk) {
  // sk: 2 x D doubles of shared memory owned by this warp (the group's probe
  // keys, staged with coalesced loads so the float64 dot chains read them at
  // shared-memory latency)
  const int lane = threadIdx.x & 31, rep = Hq / Hkv;
  const int r = lane >> 2, qd = (lane & 3) * 32;
  const int h = g * rep + (r < rep ? r : 0);
  int f = 0;
  if (flags_override) {
    f = (r < rep && flags_override[(size_t)s * Hq + h]) ? 1 : 0;
  } else {
    uint4 qv[4];
    const uint4* qp = reinterpret_cast<const uint4*>(q + ((size_t)s * Hq + h) * D + qd);
#pragma unroll
    for (int v = 0; v < 4; ++v) qv[v] = __ldg(qp + v);
    {
      const double2* kl2 = reinterpret_cast<const double2*>(k_lazy + ((size_t)s * Hkv + g) * D);
      const double2* ka2 = reinterpret_cast<const double2*>(k_act + ((size_t)s * Hkv + g) * D);
      double2 a = __ldg(kl2 + lane), b = __ldg(kl2 + 32 + lane), c = __ldg(ka2 + lane), d = __ldg(ka2 + 32 + lane);
      __syncwarp();
      reinterpret_cast<double2*>(sk)[lane] = a;
      reinterpret_cast<double2*>(sk)[32 + lane] = b;
      reinterpret_cast<double2*>(sk + D)[lane] = c;
      reinterpret_cast<double2*>(sk + D)[32 + lane] = d;
      __syncwarp();
    }
    double dl = 0.0, da = 0.0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&qv[v]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double x = static_cast<double>(__bfloat162float(hv[e]));
        dl = fma(x, sk[qd + v * 8 + e], dl);
        da = fma(x, sk[D + qd + v * 8 + e], da);
      }
    }
    dl += __shfl_xor_sync(0xffffffffu, dl, 1);
    da += __shfl_xor_sync(0xffffffffu, da, 1);
    dl += __shfl_xor_sync(0xffffffffu, dl, 2);
    da += __shfl_xor_sync(0xffffffffu, da, 2);
    const double scale = 1.0 / sqrt(static_cast<double>(D));
    const double l0 = dl * scale, l1 = da * scale, mx = fmax(l0, l1);
    const double e0 = exp(l0 - mx), e1 = exp(l1 - mx);
    f = (r < rep && e1 / (e0 + e1) > tau) ? 1 : 0;
    if (preserve && h == 0 && r == 0) f = 1;
  }
  const uint32_t b = __ballot_sync(0xffffffffu, f && (lane & 3) == 0);  // bit 4r
  uint32_t mask = 0;
#pragma unroll
  for (int k = 0; k < MAXREP; ++k) mask |= ((b >> (4 * k)) & 1u) << k;
  return mask;
}

__global__ void decode_flags_kernel(const __nv_bfloat16* __restrict__ q, const double* __restrict__ k_lazy,
                                    const double* __restrict__ k_act, int Hq, int Hkv, double tau, int preserve,
                                    const uint8_t* __restrict__ flags_override, uint8_t* __restrict__ flags) {
  __shared__ __align__(16) double sk[2 * D];
  const int g = blockIdx.x, s = blockIdx.y, lane = threadIdx.x, rep = Hq / Hkv;
  const uint32_t mask = group_flag_mask(q, k_lazy, k_act, s, g, Hq, Hkv, tau, preserve, flags_override, sk);
  if (lane < rep) flags[(size_t)s * Hq + g * rep + lane] = static_cast<uint8_t>((mask >> lane) & 1u);
}

__global__ void __launch_bounds__(128) decode_partial_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ vk, const __nv_bfloat16* __restrict__ vv,
    const int32_t* __restrict__ vlen, const __nv_bfloat16* __restrict__ tk, const __nv_bfloat16* __restrict__ tv,
    const __nv_bfloat16* __restrict__ ak, const __nv_bfloat16* __restrict__ av, SegLens sl, int Hq, int Hkv,
    int vcap, int acap, const uint8_t* __restrict__ flags, float* __restrict__ part_ml, float* __restrict__ part_acc,
    int n_chunks, int* __restrict__ degenerate) {
  __shared__ float s_ml[4][MAXREP][2];
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) *degenerate = 0;  // for the merge
  __shared__ float s_acc[4][MAXREP][D];
  const int c = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int rep = Hq / Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane & 3, gid = lane >> 2;  // thread-in-group, group id (row / key / column index)

  // per-row (Q head) vision visibility; row gid (< rep) is this thread's A/C row
  int any = 0;
  for (int r = 0; r < rep; ++r) any |= flags[(size_t)s * Hq + g * rep + r];
  const bool row_valid = gid < rep;
  const bool row_vis = row_valid && flags[(size_t)s * Hq + g * rep + (row_valid ? gid : 0)];
  const int vl = vlen[s], nt = sl.text(s), tcap = sl.tcap;
  const int k_start = any ? 0 : vl;       // skip the vision segment when every head is lazy
  const int k_end = vl + nt + sl.answer(s);
  const int w0 = k_start + c * CTA_KEYS + warp * WARP_KEYS;
  const int w1 = min(k_end, w0 + WARP_KEYS);

  // Q A-fragments with the head-dim permutation: lane r4 owns dims r4*32 .. +31;
  // k-step ks uses dims r4*32 + ks*4 + {0,1} (a0a1) and {2,3} (a4a5).
  uint32_t qa[8][4];
  {
    uint4 qv[4];
    const uint4* qrow = reinterpret_cast<const uint4*>(q + ((size_t)s * Hq + g * rep + (row_valid ? gid : 0)) * D) + r4 * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) qv[i] = row_valid ? __ldg(qrow + i) : make_uint4(0, 0, 0, 0);
    const uint32_t* qw = reinterpret_cast<const uint32_t*>(qv);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      qa[ks][0] = qw[2 * ks];      // row gid, dims +0,+1
      qa[ks][1] = 0u;              // row gid+8 (padding)
      qa[ks][2] = qw[2 * ks + 1];  // row gid, dims +2,+3
      qa[ks][3] = 0u;
    }
  }
  const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
  float m_run = -INFINITY, l_run = 0.f;
  float acc[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

  const size_t sg = (size_t)s * Hkv + g;
  auto krow = [&](int v) -> const uint4* {
    const __nv_bfloat16* p;
    if (v < vl) p = vk + (sg * vcap + v) * D;
    else if (v < vl + nt) p = tk + (sg * tcap + (v - vl)) * D;
    else p = ak + (sg * acap + (v - vl - nt)) * D;
    return reinterpret_cast<const uint4*>(p);
  };
  auto vrow = [&](int v) -> const uint4* {
    const __nv_bfloat16* p;
    if (v < vl) p = vv + (sg * vcap + v) * D;
    else if (v < vl + nt) p = tv + (sg * tcap + (v - vl)) * D;
    else p = av + (sg * acap + (v - vl - nt)) * D;
    return reinterpret_cast<const uint4*>(p);
  };

  for (int kb = w0; kb < w1; kb += 16) {
    // ---- K fragments: n-tile t covers keys kb + 8t + gid; lane loads dims r4*32 .. +31
    uint4 kf[2][4];
    bool kvalid[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int key = kb + 8 * t + gid;
      kvalid[t] = key < w1;
      const uint4* p = krow(kvalid[t] ? key : kb) + r4 * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) kf[t][i] = __ldg(p + i);
    }
    // ---- V rows for the B fragments of P V: keys kb + 2*r4 + {0,1,8,9}, dims gid*16 .. +15
    uint4 vf[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int key = kb + 2 * r4 + (u & 1) + 8 * (u >> 1);
      const uint4* p = vrow(key < w1 ? key : kb) + gid * 2;
      vf[u][0] = __ldg(p);
      vf[u][1] = __ldg(p + 1);
    }
    // ---- S = Q K^T (rows = heads, cols = 16 keys)
    float sc[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      sc[t][0] = sc[t][1] = sc[t][2] = sc[t][3] = 0.f;
      const uint32_t* kw = reinterpret_cast<const uint32_t*>(kf[t]);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) mma_bf16_16816(sc[t], qa[ks], kw[2 * ks], kw[2 * ks + 1]);
    }
    // ---- mask (keys beyond the range; vision keys for lazy heads) and online softmax
    float x[4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = kb + 8 * t + 2 * r4 + e;  // C fragment column of this thread
        const bool ok = row_valid && key < w1 && (key >= vl || row_vis);
        x[2 * t + e] = ok ? sc[t][e] * sl2 : -INFINITY;
      }
    }
    float mt = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
    mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
    const float m_new = fmaxf(m_run, mt);
    if (m_new > m_run + 8.0f) {  // lazy rescale of this row's accumulator
      const float alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
      l_run *= alpha;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        acc[i][0] *= alpha;
        acc[i][1] *= alpha;
      }
      m_run = m_new;
    }
    const float mu = (m_run == -INFINITY) ? 0.f : m_run;
    float p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      p[e] = fast_exp2(x[e] - mu);
      l_run += p[e];
    }
    // P as the A fragment: a0a1 = keys 2r4,+1 (n-tile 0), a4a5 = keys 8+2r4,+1 (n-tile 1)
    uint32_t pa[4] = {pack_bf16x2(p[0], p[1]), 0u, pack_bf16x2(p[2], p[3]), 0u};
    // ---- O += P V over 16 d n-tiles; n-tile nt, column gid <-> dim gid*16 + nt
#pragma unroll
    for (int ntl = 0; ntl < 16; ++ntl) {
      const int w = ntl >> 1, hi = ntl & 1;
      const uint32_t* v0 = reinterpret_cast<const uint32_t*>(&vf[0][w >> 2]);
      const uint32_t* v1 = reinterpret_cast<const uint32_t*>(&vf[1][w >> 2]);
      const uint32_t* v2 = reinterpret_cast<const uint32_t*>(&vf[2][w >> 2]);
      const uint32_t* v3 = reinterpret_cast<const uint32_t*>(&vf[3][w >> 2]);
      const int wi = w & 3;
      const uint32_t sel = hi ? 0x7632u : 0x5410u;
      const uint32_t b0 = __byte_perm(v0[wi], v1[wi], sel);
      const uint32_t b1 = __byte_perm(v2[wi], v3[wi], sel);
      float* cc = acc[ntl];
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(cc[0]), "+f"(cc[1]), "+f"(cc[2]), "+f"(cc[3])
          : "r"(pa[0]), "r"(pa[1]), "r"(pa[2]), "r"(pa[3]), "r"(b0), "r"(b1));
    }
  }
  // ---- per-warp row results -> smem; row gid's l is spread over the 4 lanes of its group
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
  l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
  if (row_valid) {
    if (r4 == 0) {
      s_ml[warp][gid][0] = m_run;
      s_ml[warp][gid][1] = l_run;
    }
    // C fragment: acc[nt][0/1] = O[row gid][n = 2*r4 + {0,1}] -> dim n*16 + nt
#pragma unroll
    for (int ntl = 0; ntl < 16; ++ntl) {
      s_acc[warp][gid][(2 * r4) * 16 + ntl] = acc[ntl][0];
      s_acc[warp][gid][(2 * r4 + 1) * 16 + ntl] = acc[ntl][1];
    }
  }
  __syncthreads();
  // ---- combine the 4 warps, write this chunk's partial per Q head
  for (int e = threadIdx.x; e < rep * D; e += blockDim.x) {
    const int r = e / D, col = e % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, s_ml[w][r][0]);
    float L = 0.f, o = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float m = s_ml[w][r][0];
      if (m == -INFINITY) continue;
      const float wt = fast_exp2(m - M);
      L += wt * s_ml[w][r][1];
      o += wt * s_acc[w][r][col];
    }
    const size_t base = ((size_t)s * Hq + g * rep + r) * n_chunks + c;
    part_acc[base * D + col] = o;
    if (col == 0) {
      part_ml[base * 2 + 0] = M;
      part_ml[base * 2 + 1] = L;
    }
  }
}

__global__ void decode_combine_kernel(const float* __restrict__ part_ml, const float* __restrict__ part_acc,
                                      int n_chunks, float* __restrict__ out, int* __restrict__ degenerate) {
  const int h = blockIdx.x, s = blockIdx.y, Hq = gridDim.x;
  const size_t base = (size_t)s * Hq + h;
  const float* ml = part_ml + base * n_chunks * 2;
  const float* acc = part_acc + base * n_chunks * D;
  float M = -INFINITY;
#pragma unroll 8
  for (int c = 0; c < n_chunks; ++c) M = fmaxf(M, ml[2 * c]);
  float L = 0.f, o = 0.f;
  const int col = threadIdx.x;
#pragma unroll 8
  for (int c = 0; c < n_chunks; ++c) {
    const float m = ml[2 * c];
    if (m == -INFINITY) continue;
    const float w = fast_exp2(m - M);
    L += w * ml[2 * c + 1];
    o += w * acc[(size_t)c * D + col];
  }
  if (L > 0.f) {
    out[base * D + col] = o / L;
  } else {
    out[base * D + col] = 0.f;
    if (col == 0) atomicExch(degenerate, 1);
  }
}

// ---------------------------------------------------------------- K7 v3
// TMA-staged variant (default): persistent CTAs (one per SM) walk the
// (chunk, KV group, sequence) work items; a producer warp streams 64-key K and
// V tiles of each segment (vision / text / answer, 2-D tensor maps with
// SWIZZLE_128B) into an NSTG-stage shared-memory ring that runs ahead across
// work items, so each SM keeps up to NSTG x 32 KB of HBM reads in flight with
// no register staging. Four consumer warps take 16 keys of each tile: B
// fragments of S = Q K^T come from ldmatrix.x4 and of O += P V from
// ldmatrix.x4.trans (conflict-free on the swizzled tiles), the MMA and softmax
// math is that of decode_partial_kernel.
constexpr int TK = 64, NSTG = 4, NCW = 4;
constexpr uint32_t TATOM = TK * 128;      // 64 rows x 128 B
constexpr uint32_t TTILE = 2 * TATOM;     // 64 keys x 128 d bf16 = 16 KB
constexpr uint32_t TSTAGE = 2 * TTILE;    // K + V
constexpr uint32_t TSMEM = NSTG * TSTAGE + 1024;

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
// byte offset of 16-byte chunk c (0..15 over d = 128) of key row r in a tile
__device__ __forceinline__ uint32_t toff(int r, int c) {
  return (uint32_t)(c >> 3) * TATOM + (uint32_t)r * 128u + ((uint32_t)((c & 7) ^ (r & 7)) << 4);
}

struct DecItem {
  int s, g, c, lo, hi, vl, nt, any;
};

__device__ __forceinline__ DecItem dec_item(int t, int nc, int Hq, int Hkv, const SegLens& sl,
                                            const int32_t* __restrict__ vlen, const uint8_t* __restrict__ flags) {
  DecItem it;
  it.c = t % nc;
  it.g = (t / nc) % Hkv;
  it.s = t / (nc * Hkv);
  const int rep = Hq / Hkv;
  int any = 0;
  for (int r = 0; r < rep; ++r) any |= flags[(size_t)it.s * Hq + it.g * rep + r];
  it.any = any;
  it.vl = vlen[it.s];
  it.nt = sl.text(it.s);
  const int k_start = any ? 0 : it.vl;  // skip the vision segment when every head is lazy
  const int k_end = it.vl + it.nt + sl.answer(it.s);
  it.lo = k_start + it.c * CTA_KEYS;
  it.hi = min(k_end, it.lo + CTA_KEYS);
  return it;
}

// FUSED: the item's key range from the group's active mask (computed by the
// producer warp, handed to the consumers through a shared-memory ring)
__device__ __forceinline__ DecItem dec_item_mask(int t, int nc, int Hkv, const SegLens& sl,
                                                 const int32_t* __restrict__ vlen, uint32_t mask) {
  DecItem it;
  it.c = t % nc;
  it.g = (t / nc) % Hkv;
  it.s = t / (nc * Hkv);
  it.any = mask != 0u;
  it.vl = vlen[it.s];
  it.nt = sl.text(it.s);
  const int k_start = it.any ? 0 : it.vl;
  const int k_end = it.vl + it.nt + sl.answer(it.s);
  it.lo = k_start + it.c * CTA_KEYS;
  it.hi = min(k_end, it.lo + CTA_KEYS);
  return it;
}

// tile starting at key k of item `it`: segment, local row, valid keys
__device__ __forceinline__ void dec_tile(const DecItem& it, int k, int& seg, int& row, int& nvalid) {
  const int nt = it.nt;
  int seg_lo, seg_hi;
  if (k < it.vl) { seg = 0; seg_lo = 0; seg_hi = it.vl; }
  else if (k < it.vl + nt) { seg = 1; seg_lo = it.vl; seg_hi = it.vl + nt; }
  else { seg = 2; seg_lo = it.vl + nt; seg_hi = it.hi; }
  row = k - seg_lo;
  nvalid = min(TK, min(seg_hi, it.hi) - k);
}

// FUSED (default): the producer warp classifies each item's Q heads
// (group_flag_mask, the arithmetic of decode_flags_kernel) and hands the
// item's active mask to the consumers through a small shared-memory ring —
// no separate classification launch. (Merging the partials in the CTA that
// finishes a group's last chunk measured 3.7x slower than the separate merge
// kernel: the merge lands on few CTAs at the tail.)
struct FuseArgs {
  const double* k_lazy;
  const double* k_act;
  double tau;
  int preserve;
  const uint8_t* flags_override;
  uint8_t* flags_out;
};
constexpr int NIT = 4;  // item ring depth

template <bool FUSED>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) decode_partial_tma_kernel(
    const __grid_constant__ CUtensorMap tm_vk, const __grid_constant__ CUtensorMap tm_vv,
    const __grid_constant__ CUtensorMap tm_tk, const __grid_constant__ CUtensorMap tm_tv,
    const __grid_constant__ CUtensorMap tm_ak, const __grid_constant__ CUtensorMap tm_av,
    const __nv_bfloat16* __restrict__ q, const int32_t* __restrict__ vlen, SegLens sl, int Hq, int Hkv,
    int vcap, int acap, const uint8_t* __restrict__ flags, float* __restrict__ part_ml,
    float* __restrict__ part_acc, int n_chunks, int total_items, FuseArgs fa, int* __restrict__ degenerate) {
  extern __shared__ uint8_t dsm_raw[];
  __shared__ __align__(8) uint64_t full_bar[NSTG], empty_bar[NSTG];
  __shared__ __align__(8) uint64_t item_full[NIT], item_empty[NIT];
  __shared__ uint32_t s_mask[NIT];
  __shared__ __align__(16) double s_kstage[2 * D];  // producer: the item group's probe keys
  __shared__ float s_ml[NCW][MAXREP][2];
  __shared__ float s_acc[NCW][MAXREP][D];
  uint8_t* dsm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(dsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *degenerate = 0;  // reset for the merge kernel that follows
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTG; ++i) {
      mbar_init(smem_u32(&full_bar[i]), 1);
      mbar_init(smem_u32(&empty_bar[i]), NCW);
    }
    for (int i = 0; i < NIT; ++i) {
      mbar_init(smem_u32(&item_full[i]), 1);
      mbar_init(smem_u32(&item_empty[i]), NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int rep = Hq / Hkv;

  if (warp == NCW) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_vk); tma_prefetch_desc(&tm_vv);
      tma_prefetch_desc(&tm_tk); tma_prefetch_desc(&tm_tv);
      tma_prefetch_desc(&tm_ak); tma_prefetch_desc(&tm_av);
    }
    uint32_t n = 0, ni = 0;
    for (int t = blockIdx.x; t < total_items; t += gridDim.x, ++ni) {
      DecItem it;
      if constexpr (FUSED) {
        const int s_ = t / (n_chunks * Hkv), g_ = (t / n_chunks) % Hkv;
        const uint32_t mask = group_flag_mask(q, fa.k_lazy, fa.k_act, s_, g_, Hq, Hkv, fa.tau, fa.preserve,
                                              fa.flags_override, s_kstage);
        it = dec_item_mask(t, n_chunks, Hkv, sl, vlen, mask);
        if (it.c == 0 && lane < rep) fa.flags_out[(size_t)it.s * Hq + it.g * rep + lane] = (mask >> lane) & 1u;
        const int slot = ni % NIT;
        if (ni >= NIT) mbar_wait(smem_u32(&item_empty[slot]), ((ni / NIT) - 1) & 1);
        if (lane == 0) {
          s_mask[slot] = mask;
          mbar_arrive(smem_u32(&item_full[slot]));  // release: the mask write precedes it
        }
      } else {
        it = dec_item(t, n_chunks, Hq, Hkv, sl, vlen, flags);
      }
      if (lane == 0) {
        const int sg = it.s * Hkv + it.g;
        for (int k = it.lo; k < it.hi; k += TK) {
          int seg, row, nv;
          dec_tile(it, k, seg, row, nv);
          k += nv - TK;  // next tile starts after this tile's valid keys (segment-aligned)
          const int st = n % NSTG;
          if (n >= NSTG) mbar_wait(smem_u32(&empty_bar[st]), ((n / NSTG) - 1) & 1);
          const uint32_t fb = smem_u32(&full_bar[st]);
          mbar_expect_tx(fb, TSTAGE);
          const CUtensorMap* mk = seg == 0 ? &tm_vk : seg == 1 ? &tm_tk : &tm_ak;
          const CUtensorMap* mv = seg == 0 ? &tm_vv : seg == 1 ? &tm_tv : &tm_av;
          const int base = seg == 0 ? sg * vcap : seg == 1 ? sg * sl.tcap : sg * acap;
          const uint32_t kd = sbase + st * TSTAGE, vd = kd + TTILE;
          tma_load_2d(kd, mk, fb, 0, base + row);
          tma_load_2d(kd + TATOM, mk, fb, 64, base + row);
          tma_load_2d(vd, mv, fb, 0, base + row);
          tma_load_2d(vd + TATOM, mv, fb, 64, base + row);
          ++n;
        }
      }
      __syncwarp();
    }
    return;
  }
  // ------------------------------------------------------ consumers
  const int r4 = lane & 3, gid = lane >> 2;
  const bool row_valid = gid < rep;
  const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
  uint32_t n = 0, ni = 0;
  for (int t = blockIdx.x; t < total_items; t += gridDim.x, ++ni) {
    DecItem it;
    bool row_vis;
    if constexpr (FUSED) {
      const int slot = ni % NIT;
      mbar_wait(smem_u32(&item_full[slot]), (ni / NIT) & 1);
      const uint32_t mask = s_mask[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&item_empty[slot]));
      it = dec_item_mask(t, n_chunks, Hkv, sl, vlen, mask);
      row_vis = row_valid && ((mask >> gid) & 1u);
    } else {
      it = dec_item(t, n_chunks, Hq, Hkv, sl, vlen, flags);
      row_vis = row_valid && flags[(size_t)it.s * Hq + it.g * rep + (row_valid ? gid : 0)];
    }
    // Q A-fragments, natural head-dim order: k-step ks covers d = 16 ks .. +15
    uint32_t qa[8][4];
    {
      const uint32_t* qw =
          reinterpret_cast<const uint32_t*>(q + ((size_t)it.s * Hq + it.g * rep + (row_valid ? gid : 0)) * D);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qa[ks][0] = row_valid ? __ldg(qw + ks * 8 + r4) : 0u;      // d 16ks + 2 r4, +1
        qa[ks][1] = 0u;                                             // rows 8..15: padding
        qa[ks][2] = row_valid ? __ldg(qw + ks * 8 + 4 + r4) : 0u;  // d 16ks + 8 + 2 r4, +1
        qa[ks][3] = 0u;
      }
    }
    float m_run = -INFINITY, l_run = 0.f;
    float acc[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    for (int k = it.lo; k < it.hi; k += TK) {
      int seg, row, nv;
      dec_tile(it, k, seg, row, nv);
      const int key0 = k;
      k += nv - TK;
      const int st = n % NSTG;
      mbar_wait(smem_u32(&full_bar[st]), (n / NSTG) & 1);
      const uint32_t kt = sbase + st * TSTAGE, vt = kt + TTILE;
      const int w0 = warp * 16;  // this warp's first key of the tile
      if (w0 < nv) {
        // ---- S = Q K^T over 16 keys (two n-tiles of 8)
        float sc[2][4];
#pragma unroll
        for (int u = 0; u < 2; ++u) sc[u][0] = sc[u][1] = sc[u][2] = sc[u][3] = 0.f;
        const int mi = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b[4];
          // matrices: (keys 0-7, d lo) (keys 0-7, d hi) (keys 8-15, d lo) (keys 8-15, d hi)
          ldsm_x4(kt + toff(w0 + (mi >> 1) * 8 + rr, 2 * ks + (mi & 1)), b);
          mma_bf16_16816(sc[0], qa[ks], b[0], b[1]);
          mma_bf16_16816(sc[1], qa[ks], b[2], b[3]);
        }
        // ---- mask (keys beyond the tile; vision keys for lazy heads), online softmax
        float x[4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kk = w0 + 8 * u + 2 * r4 + e;  // key within the tile
            const bool ok = row_valid && kk < nv && (seg != 0 || row_vis);
            x[2 * u + e] = ok ? sc[u][e] * sl2 : -INFINITY;
          }
        }
        float mt = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 1));
        mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, 2));
        const float m_new = fmaxf(m_run, mt);
        if (m_new > m_run + 8.0f) {  // lazy rescale of this row's accumulator
          const float alpha = (m_run == -INFINITY) ? 0.f : fast_exp2(m_run - m_new);
          l_run *= alpha;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            acc[i][0] *= alpha;
            acc[i][1] *= alpha;
          }
          m_run = m_new;
        }
        const float mu = (m_run == -INFINITY) ? 0.f : m_run;
        float p[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          p[e] = fast_exp2(x[e] - mu);
          l_run += p[e];
        }
        uint32_t pa[4] = {pack_bf16x2(p[0], p[1]), 0u, pack_bf16x2(p[2], p[3]), 0u};
        // ---- O += P V over 16 d n-tiles (pairs from one ldmatrix.x4.trans)
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          uint32_t b[4];
          // matrices: (keys 0-7, d 8j) (keys 8-15, d 8j) (keys 0-7, d 8j+8) (keys 8-15, d 8j+8)
          ldsm_x4_t(vt + toff(w0 + (mi & 1) * 8 + rr, j + (mi >> 1)), b);
          mma_bf16_16816(acc[j], pa, b[0], b[1]);
          mma_bf16_16816(acc[j + 1], pa, b[2], b[3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty_bar[st]));
      ++n;
    }
    // ---- combine the consumer warps, write this item's partial per Q head
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    if (row_valid) {
      if (r4 == 0) {
        s_ml[warp][gid][0] = m_run;
        s_ml[warp][gid][1] = l_run;
      }
      // C fragment of n-tile j: acc[j][0/1] = O[row gid][d = 8 j + 2 r4 + {0,1}]
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        s_acc[warp][gid][8 * j + 2 * r4] = acc[j][0];
        s_acc[warp][gid][8 * j + 2 * r4 + 1] = acc[j][1];
      }
    }
    named_bar_sync(1, NCW * 32);
    for (int e = threadIdx.x; e < rep * D; e += NCW * 32) {
      const int r = e / D, col = e % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NCW; ++w) M = fmaxf(M, s_ml[w][r][0]);
      float L = 0.f, o = 0.f;
#pragma unroll
      for (int w = 0; w < NCW; ++w) {
        const float m = s_ml[w][r][0];
        if (m == -INFINITY) continue;
        const float wt = fast_exp2(m - M);
        L += wt * s_ml[w][r][1];
        o += wt * s_acc[w][r][col];
      }
      const size_t pb = ((size_t)it.s * Hq + it.g * rep + r) * n_chunks + it.c;
      part_acc[pb * D + col] = o;
      if (col == 0) {
        part_ml[pb * 2 + 0] = M;
        part_ml[pb * 2 + 1] = L;
      }
    }
    named_bar_sync(1, NCW * 32);  // partial slots free for the next item
  }
}

}  // namespace dec
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

static int dec_chunks(int vcap, int n_text, int n_answer) {
  return (vcap + n_text + n_answer + dec::CTA_KEYS - 1) / dec::CTA_KEYS;
}

extern "C" size_t omni_decode_workspace(int batch, int n_q_heads, int vcap, int n_text, int acap, int head_dim) {
  const int nc = dec_chunks(vcap, n_text, acap);
  return sizeof(float) * (size_t)batch * n_q_heads * nc * (head_dim + 2) + 16;
}

static int decode_step_impl(const void* q, const void* vision_k, const void* vision_v, const int32_t* vision_len,
                            const void* text_k, const void* text_v, const void* answer_k, const void* answer_v,
                            dec::SegLens sl, const double* k_lazy, const double* k_act, int batch, int n_q_heads,
                            int n_kv_heads, int head_dim, int vcap, int acap, double tau, int preserve_first_head,
                            const uint8_t* flags_override, uint8_t* flags, float* out, void* workspace,
                            int32_t* status, void* stream) {
  OMNI_CHECK(head_dim == dec::D, OMNI_E_SHAPE, "decode kernel requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(n_q_heads / n_kv_heads <= dec::MAXREP, OMNI_E_SHAPE, "at most 8 Q heads per KV group");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  OMNI_CHECK(batch >= 1, OMNI_E_SHAPE, "empty batch");
  const int n_text = sl.tcap;
  const int n_answer = sl.alen ? acap : sl.na;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nc = dec_chunks(vcap, n_text, n_answer);
  float* part_ml = static_cast<float*>(workspace);
  float* part_acc = part_ml + (size_t)batch * n_q_heads * nc * 2;
  int* degenerate = status ? reinterpret_cast<int*>(status)
                           : reinterpret_cast<int*>(part_acc + (size_t)batch * n_q_heads * nc * head_dim);
  // K7 implementation: the TMA-staged persistent kernel with the query
  // classification fused in by default, then the split-K merge;
  // OMNI_DECODE_IMPL=split classifies in a separate kernel first,
  // OMNI_DECODE_IMPL=regs uses the register-staged partial kernel.
  static const int impl = [] {
    const char* e = getenv("OMNI_DECODE_IMPL");
    return (e && strcmp(e, "regs") == 0) ? 2 : (e && strcmp(e, "split") == 0) ? 1 : 0;
  }();
  const bool regs = impl == 2, fused = impl == 0;
  if (!fused)
    dec::decode_flags_kernel<<<dim3(n_kv_heads, batch), 32, 0, st>>>(static_cast<const __nv_bfloat16*>(q), k_lazy,
                                                                      k_act, n_q_heads, n_kv_heads, tau,
                                                                      preserve_first_head, flags_override, flags);
  if (regs) {
    dec::decode_partial_kernel<<<dim3(nc, n_kv_heads, batch), 128, 0, st>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(vision_k),
        static_cast<const __nv_bfloat16*>(vision_v), vision_len, static_cast<const __nv_bfloat16*>(text_k),
        static_cast<const __nv_bfloat16*>(text_v), static_cast<const __nv_bfloat16*>(answer_k),
        static_cast<const __nv_bfloat16*>(answer_v), sl, n_q_heads, n_kv_heads, vcap, acap, flags, part_ml,
        part_acc, nc, degenerate);
  } else {
    CUtensorMap m[6];
    const uint64_t vrows = (uint64_t)batch * n_kv_heads * vcap;
    const void* bases[6] = {vision_k, vision_v, n_text > 0 ? text_k : vision_k, n_text > 0 ? text_v : vision_v,
                            acap > 0 ? answer_k : vision_k, acap > 0 ? answer_v : vision_v};
    const uint64_t rows[6] = {vrows, vrows, n_text > 0 ? (uint64_t)batch * n_kv_heads * n_text : vrows,
                              n_text > 0 ? (uint64_t)batch * n_kv_heads * n_text : vrows,
                              acap > 0 ? (uint64_t)batch * n_kv_heads * acap : vrows,
                              acap > 0 ? (uint64_t)batch * n_kv_heads * acap : vrows};
    for (int i = 0; i < 6; ++i) {
      const int rc = omni_make_tmap_rows(&m[i], bases[i], rows[i], dec::D, 2, 64, dec::TK);
      if (rc) return rc;
    }
    auto kern = fused ? dec::decode_partial_tma_kernel<true> : dec::decode_partial_tma_kernel<false>;
    static bool attr[2] = {false, false};
    if (!attr[fused]) {
      OMNI_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dec::TSMEM));
      attr[fused] = true;
    }
    int dev = 0, sms = 148;
    OMNI_CUDA_TRY(cudaGetDevice(&dev));
    OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int items = nc * n_kv_heads * batch;
    const dec::FuseArgs fa{k_lazy, k_act, tau, preserve_first_head, flags_override, flags};
    kern<<<min(sms, items), (dec::NCW + 1) * 32, dec::TSMEM, st>>>(
        m[0], m[1], m[2], m[3], m[4], m[5], static_cast<const __nv_bfloat16*>(q), vision_len, sl, n_q_heads,
        n_kv_heads, vcap, acap, flags, part_ml, part_acc, nc, items, fa, degenerate);
  }
  dec::decode_combine_kernel<<<dim3(n_q_heads, batch), dec::D, 0, st>>>(part_ml, part_acc, nc, out, degenerate);
  int st_code = omni_launch_check();
  if (st_code) return st_code;
  if (!status && n_text + n_answer == 0) {
    // Only reachable degenerate case (decode.py:152-153): read the flag back.
    int h = 0;
    OMNI_CUDA_TRY(cudaMemcpyAsync(&h, degenerate, sizeof(int), cudaMemcpyDeviceToHost, st));
    OMNI_CUDA_TRY(cudaStreamSynchronize(st));
    OMNI_CHECK(h == 0, OMNI_E_DEGENERATE_CONTEXT, "lazy head with no text and no answer KV");
  }
  return OMNI_OK;
}

extern "C" int omni_decode_step(const void* q, const void* vision_k, const void* vision_v, const int32_t* vision_len,
                                const void* text_k, const void* text_v, int n_text, const void* answer_k,
                                const void* answer_v, int n_answer, const double* k_lazy, const double* k_act,
                                int batch, int n_q_heads, int n_kv_heads, int head_dim, int vcap, int acap, double tau,
                                int preserve_first_head, const uint8_t* flags_override, uint8_t* flags, float* out,
                                void* workspace, void* stream) {
  OMNI_CHECK(n_answer >= 0 && n_answer <= acap && n_text >= 0, OMNI_E_SHAPE, "answer segment overflow");
  const dec::SegLens sl{nullptr, nullptr, n_text, n_answer, n_text};
  return decode_step_impl(q, vision_k, vision_v, vision_len, text_k, text_v, answer_k, answer_v, sl, k_lazy, k_act,
                          batch, n_q_heads, n_kv_heads, head_dim, vcap, acap, tau, preserve_first_head,
                          flags_override, flags, out, workspace, nullptr, stream);
}

extern "C" int omni_decode_step_varlen(const void* q, const void* vision_k, const void* vision_v,
                                       const int32_t* vision_len, const void* text_k, const void* text_v,
                                       const int32_t* text_len, int tcap, const void* answer_k, const void* answer_v,
                                       const int32_t* answer_len, const double* k_lazy, const double* k_act,
                                       int batch, int n_q_heads, int n_kv_heads, int head_dim, int vcap, int acap,
                                       double tau, int preserve_first_head, const uint8_t* flags_override,
                                       uint8_t* flags, float* out, void* workspace, int32_t* status, void* stream) {
  OMNI_CHECK(text_len && answer_len && status, OMNI_E_PARAM, "varlen decode needs text_len, answer_len and status");
  OMNI_CHECK(tcap >= 0 && acap >= 0 && tcap + acap > 0, OMNI_E_SHAPE, "text and answer capacities are both zero");
  const dec::SegLens sl{text_len, answer_len, 0, 0, tcap};
  return decode_step_impl(q, vision_k, vision_v, vision_len, text_k, text_v, answer_k, answer_v, sl, k_lazy, k_act,
                          batch, n_q_heads, n_kv_heads, head_dim, vcap, acap, tau, preserve_first_head,
                          flags_override, flags, out, workspace, status, stream);
}

// SURVEY §8b's minimum export set names the decode entry point omni_decode;
// it is omni_decode_step.
extern "C" int omni_decode(const void* q, const void* vision_k, const void* vision_v, const int32_t* vision_len,
                           const void* text_k, const void* text_v, int n_text, const void* answer_k,
                           const void* answer_v, int n_answer, const double* k_lazy, const double* k_act, int batch,
                           int n_q_heads, int n_kv_heads, int head_dim, int vcap, int acap, double tau,
                           int preserve_first_head, const uint8_t* flags_override, uint8_t* flags, float* out,
                           void* workspace, void* stream) {
  return omni_decode_step(q, vision_k, vision_v, vision_len, text_k, text_v, n_text, answer_k, answer_v, n_answer,
                          k_lazy, k_act, batch, n_q_heads, n_kv_heads, head_dim, vcap, acap, tau, preserve_first_head,
                          flags_override, flags, out, workspace, stream);
}

// append_answer (decode.py:111-121) for a batch, one launch: the new K / V row
// of every (sequence, KV group) goes to answer row pos_s = answer_len[s]
// (ragged batches; incremented here) or n_answer (answer_len NULL). One CTA
// per sequence, so the position is read before it is advanced.
__global__ void append_answer_kernel(const uint4* __restrict__ k_rows, const uint4* __restrict__ v_rows,
                                     uint4* __restrict__ ak, uint4* __restrict__ av, int Hkv, int acap, int n_answer,
                                     int32_t* __restrict__ answer_len) {
  constexpr int RV = dec::D * 2 / 16;  // uint4 per bf16 row
  const int s = blockIdx.x;
  const int pos = answer_len ? answer_len[s] : n_answer;
  for (int e = threadIdx.x; e < Hkv * RV; e += blockDim.x) {
    const int g = e / RV, c = e % RV;
    const size_t src = ((size_t)s * Hkv + g) * RV + c;
    const size_t dst = (((size_t)s * Hkv + g) * acap + pos) * RV + c;
    ak[dst] = k_rows[src];
    av[dst] = v_rows[src];
  }
  __syncthreads();
  if (answer_len && threadIdx.x == 0) answer_len[s] = pos + 1;
}

extern "C" int omni_append_answer(const void* k_rows, const void* v_rows, void* answer_k, void* answer_v, int batch,
                                  int n_kv_heads, int head_dim, int acap, int n_answer, int32_t* answer_len,
                                  void* stream) {
  OMNI_CHECK(head_dim == dec::D, OMNI_E_SHAPE, "answer rows must have head_dim 128");
  OMNI_CHECK(answer_len != nullptr || (n_answer >= 0 && n_answer < acap), OMNI_E_SHAPE, "answer capacity exhausted");
  if (batch == 0) return OMNI_OK;
  append_answer_kernel<<<batch, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_rows), static_cast<const uint4*>(v_rows), static_cast<uint4*>(answer_k),
      static_cast<uint4*>(answer_v), n_kv_heads, acap, n_answer, answer_len);
  return omni_launch_check();
}

// classify_decode_query (decode.py:124-140) alone: flags u8 [B, Hq] for one
// decode token per sequence (the classification K7 also fuses).
extern "C" int omni_decode_flags(const void* q, const double* k_lazy, const double* k_act, int batch, int n_q_heads,
                                 int n_kv_heads, int head_dim, double tau, int preserve_first_head, uint8_t* flags,
                                 void* stream) {
  OMNI_CHECK(head_dim == dec::D, OMNI_E_SHAPE, "decode classification requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0 && n_q_heads / n_kv_heads <= dec::MAXREP, OMNI_E_SHAPE,
             "need Hq a multiple of Hkv with at most 8 Q heads per group");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  if (batch == 0) return OMNI_OK;
  dec::decode_flags_kernel<<<dim3(n_kv_heads, batch), 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), k_lazy, k_act, n_q_heads, n_kv_heads, tau, preserve_first_head, nullptr,
      flags);
  return omni_launch_check();
}
