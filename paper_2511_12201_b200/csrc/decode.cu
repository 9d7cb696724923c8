// K7: slimmed decode attention over a PAGED slim cache (split-K flash decoding).
//
// Replaces classify_decode_query + _fetched_segments + decode_attention
// (decode.py:124-194) for a batch of sequences under GQA rule B.
//
// Cache layout (serving): one pool of 64-row pages per
// layer, K and V each [P, 64, 128] bf16. Sequence slot s, KV group g owns the
// page list table[(s * Hkv + g) * max_pages + j]: ceil(b / 64) vision pages,
// then ceil(n_text / 64) text pages, then ceil(n_answer / 64) answer pages
// (the segment order of _fetched_segments, decode.py:143-154). Admitting a
// sequence writes only its own pages, evicting one returns its pages, growing
// an answer takes a page every 64 tokens: no operation copies other
// sequences' KV (the reference grows one Python list per head,
// decode.py:111-121).
//
//   decode_partial_tma_kernel  persistent CTAs over (32-page chunk, KV group,
//       sequence) items. A producer warp classifies the item's Q heads
//       (float64 two-logit rule against the frozen probe keys, head 0 forced
//       active) and streams its pages with SWIZZLE_128B TMA (one 64-row box
//       per page and half-row) into a 4-stage ring; a group's vision pages
//       are skipped when all its Q heads are lazy (the fetch skip of
//       decode.py:176-190), lazy heads see -inf on vision keys (exclusion,
//       decode.py:12-16). Four consumer warps: the group's <= 8 Q heads as the
//       M rows of mma.sync m16n8k16 (ldmatrix B fragments), online softmax.
//   decode_combine_kernel merges the per-chunk (max, sum, acc) partials.
// HBM-bound: bytes = fetched vision + text + answer pages, once each.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace dec {

constexpr int D = 128;
constexpr int PAGE = 64;                       // rows per page = TMA box rows = keys per tile
constexpr int CHUNK_PAGES = 32;                // pages per work item (2048 keys)
constexpr int MAXREP = 8;  // rows of the m16 tile used (rows 8..15 stay zero)

// Per-sequence lengths (device i32 [B], rows) and the page table.
struct Paged {
  const int32_t* table;  // [B, Hkv, max_pages]
  int max_pages;
  const int32_t* vlen;   // vision rows (= budget b)
  const int32_t* tlen;   // text rows
  const int32_t* alen;   // answer rows
  double scale;          // 1 / sqrt(head_dim); rows stored with D columns (zero-padded past head_dim)
};

__device__ __forceinline__ int pages_of(int rows) { return (rows + PAGE - 1) / PAGE; }

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
                                                    double tau, double scale, int preserve,
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
                                    const double* __restrict__ k_act, int Hq, int Hkv, double tau, double scale,
                                    int preserve,
                                    const uint8_t* __restrict__ flags_override, uint8_t* __restrict__ flags) {
  __shared__ __align__(16) double sk[2 * D];
  const int g = blockIdx.x, s = blockIdx.y, lane = threadIdx.x, rep = Hq / Hkv;
  const uint32_t mask = group_flag_mask(q, k_lazy, k_act, s, g, Hq, Hkv, tau, scale, preserve, flags_override, sk);
  if (lane < rep) flags[(size_t)s * Hq + g * rep + lane] = static_cast<uint8_t>((mask >> lane) & 1u);
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

constexpr int NSTG = 4, NCW = 4;
constexpr uint32_t TATOM = PAGE * 128;    // 64 rows x 128 B
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
  int s, g, c, t0, t1, tv, tt, vl, nt, na;
};

// Item t = (chunk c, group g, sequence s): page slots [t0, t1) of the group's
// page list, the vision pages skipped when no Q head of the group is active.
__device__ __forceinline__ DecItem dec_item(int t, int nc, int Hkv, const Paged& pg, uint32_t mask) {
  DecItem it;
  it.c = t % nc;
  it.g = (t / nc) % Hkv;
  it.s = t / (nc * Hkv);
  it.vl = pg.vlen[it.s];
  it.nt = pg.tlen[it.s];
  it.na = pg.alen[it.s];
  it.tv = pages_of(it.vl);
  it.tt = pages_of(it.nt);
  const int first = mask ? 0 : it.tv;
  const int end = it.tv + it.tt + pages_of(it.na);
  it.t0 = first + it.c * CHUNK_PAGES;
  it.t1 = min(end, it.t0 + CHUNK_PAGES);
  return it;
}

// page slot j of item `it`: segment (0 vision, 1 text, 2 answer) and valid rows
__device__ __forceinline__ void dec_tile(const DecItem& it, int j, int& seg, int& nvalid) {
  if (j < it.tv) { seg = 0; nvalid = min(PAGE, it.vl - j * PAGE); }
  else if (j < it.tv + it.tt) { seg = 1; nvalid = min(PAGE, it.nt - (j - it.tv) * PAGE); }
  else { seg = 2; nvalid = min(PAGE, it.na - (j - it.tv - it.tt) * PAGE); }
}

// The producer warp classifies each item's Q heads (group_flag_mask) and
// hands the item's active mask to the consumers through a small shared-memory
// ring — no separate classification launch.
struct FuseArgs {
  const double* k_lazy;
  const double* k_act;
  double tau;
  int preserve;
  const uint8_t* flags_override;
  uint8_t* flags_out;
};
constexpr int NIT = 4;  // item ring depth

__global__ void __launch_bounds__((NCW + 1) * 32, 1) decode_partial_tma_kernel(
    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
    const __nv_bfloat16* __restrict__ q, Paged pg, int Hq, int Hkv, float* __restrict__ part_ml,
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
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
    }
    uint32_t n = 0, ni = 0;
    for (int t = blockIdx.x; t < total_items; t += gridDim.x, ++ni) {
      const int s_ = t / (n_chunks * Hkv), g_ = (t / n_chunks) % Hkv;
      const uint32_t mask = group_flag_mask(q, fa.k_lazy, fa.k_act, s_, g_, Hq, Hkv, fa.tau, pg.scale, fa.preserve,
                                            fa.flags_override, s_kstage);
      const DecItem it = dec_item(t, n_chunks, Hkv, pg, mask);
      if (it.c == 0 && lane < rep) fa.flags_out[(size_t)it.s * Hq + it.g * rep + lane] = (mask >> lane) & 1u;
      const int slot = ni % NIT;
      if (ni >= NIT) mbar_wait(smem_u32(&item_empty[slot]), ((ni / NIT) - 1) & 1);
      if (lane == 0) {
        s_mask[slot] = mask;
        mbar_arrive(smem_u32(&item_full[slot]));  // release: the mask write precedes it
      }
      if (lane == 0) {
        const int32_t* pages = pg.table + (size_t)(it.s * Hkv + it.g) * pg.max_pages;
        for (int j = it.t0; j < it.t1; ++j) {
          const int row = __ldg(pages + j) * PAGE;
          const int st = n % NSTG;
          if (n >= NSTG) mbar_wait(smem_u32(&empty_bar[st]), ((n / NSTG) - 1) & 1);
          const uint32_t fb = smem_u32(&full_bar[st]);
          mbar_expect_tx(fb, TSTAGE);
          const uint32_t kd = sbase + st * TSTAGE, vd = kd + TTILE;
          tma_load_2d(kd, &tm_k, fb, 0, row);
          tma_load_2d(kd + TATOM, &tm_k, fb, 64, row);
          tma_load_2d(vd, &tm_v, fb, 0, row);
          tma_load_2d(vd + TATOM, &tm_v, fb, 64, row);
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
  const float sl2 = static_cast<float>(kLog2e * pg.scale);
  uint32_t n = 0, ni = 0;
  for (int t = blockIdx.x; t < total_items; t += gridDim.x, ++ni) {
    const int slot = ni % NIT;
    mbar_wait(smem_u32(&item_full[slot]), (ni / NIT) & 1);
    const uint32_t mask = s_mask[slot];
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&item_empty[slot]));
    const DecItem it = dec_item(t, n_chunks, Hkv, pg, mask);
    const bool row_vis = row_valid && ((mask >> gid) & 1u);
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
    for (int j = it.t0; j < it.t1; ++j) {
      int seg, nv;
      dec_tile(it, j, seg, nv);
      const int st = n % NSTG;
      mbar_wait(smem_u32(&full_bar[st]), (n / NSTG) & 1);
      const uint32_t kt = sbase + st * TSTAGE, vt = kt + TTILE;
      const int w0 = warp * 16;  // this warp's first key of the page
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
        // ---- mask (rows past the page's valid rows; vision keys for lazy heads), online softmax
        float x[4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kk = w0 + 8 * u + 2 * r4 + e;  // key within the page
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
        for (int jj = 0; jj < 16; jj += 2) {
          uint32_t b[4];
          // matrices: (keys 0-7, d 8jj) (keys 8-15, d 8jj) (keys 0-7, d 8jj+8) (keys 8-15, d 8jj+8)
          ldsm_x4_t(vt + toff(w0 + (mi & 1) * 8 + rr, jj + (mi >> 1)), b);
          mma_bf16_16816(acc[jj], pa, b[0], b[1]);
          mma_bf16_16816(acc[jj + 1], pa, b[2], b[3]);
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
      // C fragment of n-tile jj: acc[jj][0/1] = O[row gid][d = 8 jj + 2 r4 + {0,1}]
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        s_acc[warp][gid][8 * jj + 2 * r4] = acc[jj][0];
        s_acc[warp][gid][8 * jj + 2 * r4 + 1] = acc[jj][1];
      }
    }
    named_bar_sync(1, NCW * 32);
    for (int e = threadIdx.x; e < rep * D; e += NCW * 32) {
      const int r = e / D, col = e % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NCW; ++w) M = fmaxf(M, s_ml[w][r][0]);
      float Lsum = 0.f, o = 0.f;
#pragma unroll
      for (int w = 0; w < NCW; ++w) {
        const float m = s_ml[w][r][0];
        if (m == -INFINITY) continue;
        const float wt = fast_exp2(m - M);
        Lsum += wt * s_ml[w][r][1];
        o += wt * s_acc[w][r][col];
      }
      const size_t pb = ((size_t)it.s * Hq + it.g * rep + r) * n_chunks + it.c;
      part_acc[pb * D + col] = o;
      if (col == 0) {
        part_ml[pb * 2 + 0] = M;
        part_ml[pb * 2 + 1] = Lsum;
      }
    }
    named_bar_sync(1, NCW * 32);  // partial slots free for the next item
  }
}

// append_answer (decode.py:111-121) for a batch, one launch: the new K / V
// row of every (sequence, KV group) goes to answer row a = alen[s] — page slot
// pages(vlen) + pages(tlen) + a / 64 of the group's list (allocated by the
// host beforehand), row a % 64 — and alen[s] advances. One CTA per sequence,
// so the position is read before it is advanced.
__global__ void append_paged_kernel(const uint4* __restrict__ k_rows, const uint4* __restrict__ v_rows,
                                    uint4* __restrict__ pool_k, uint4* __restrict__ pool_v, Paged pg, int Hkv,
                                    int32_t* __restrict__ alen) {
  constexpr int RV = D * 2 / 16;  // uint4 per bf16 row
  const int s = blockIdx.x;
  const int a = alen[s];
  const int slot = pages_of(pg.vlen[s]) + pages_of(pg.tlen[s]) + a / PAGE;
  for (int e = threadIdx.x; e < Hkv * RV; e += blockDim.x) {
    const int g = e / RV, c = e % RV;
    const int page = pg.table[((size_t)s * Hkv + g) * pg.max_pages + slot];
    const size_t src = ((size_t)s * Hkv + g) * RV + c;
    const size_t dst = ((size_t)page * PAGE + a % PAGE) * RV + c;
    pool_k[dst] = k_rows[src];
    pool_v[dst] = v_rows[src];
  }
  __syncthreads();
  if (threadIdx.x == 0) alen[s] = a + 1;
}

// Rows into pages (K6 for the paged cache): for group g and r < count,
// pool[page(g, first_slot + (row0 + r) / 64) * 64 + (row0 + r) % 64] =
// src[g, idx ? idx[g, r] : r]; the rest of the last page is zero-filled.
__global__ void page_write_kernel(const uint4* __restrict__ src, int src_rows, const int32_t* __restrict__ idx,
                                  int idx_stride, int count, const int32_t* __restrict__ table, int max_pages,
                                  int first_slot, uint4* __restrict__ pool) {
  constexpr int RV = D * 2 / 16;
  const int g = blockIdx.y;
  const int r = blockIdx.x * (blockDim.x / RV) + threadIdx.x / RV, c = threadIdx.x % RV;
  const int padded = pages_of(count) * PAGE;
  if (r >= padded) return;
  const int page = table[(size_t)g * max_pages + first_slot + r / PAGE];
  const size_t dst = ((size_t)page * PAGE + r % PAGE) * RV + c;
  if (r < count) {
    const int sr = idx ? idx[(size_t)g * idx_stride + r] : r;
    pool[dst] = src[((size_t)g * src_rows + sr) * RV + c];
  } else {
    pool[dst] = make_uint4(0, 0, 0, 0);
  }
}

}  // namespace dec
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

extern "C" size_t omni_decode_workspace(int batch, int n_q_heads, int n_chunks) {
  return sizeof(float) * (size_t)batch * n_q_heads * n_chunks * (dec::D + 2) + 16;
}

extern "C" int omni_decode(const void* q, const void* pool_k, const void* pool_v, int n_pages, const int32_t* table,
                           int max_pages, const int32_t* vision_len, const int32_t* text_len,
                           const int32_t* answer_len, int n_chunks, const double* k_lazy, const double* k_act,
                           int batch, int n_q_heads, int n_kv_heads, int head_dim, double tau,
                           int preserve_first_head, const uint8_t* flags_override, uint8_t* flags, float* out,
                           void* workspace, int32_t* status, void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim >= 1 && head_dim <= dec::D, OMNI_E_SHAPE,
             "decode rows are stored with 128 columns: head_dim must be in [1, 128] (zero-pad shorter rows)");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(n_q_heads / n_kv_heads <= dec::MAXREP, OMNI_E_SHAPE, "at most 8 Q heads per KV group");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  OMNI_CHECK(batch >= 1 && n_pages >= 1 && max_pages >= 1 && n_chunks >= 1, OMNI_E_SHAPE, "empty batch or pool");
  OMNI_CHECK(vision_len && text_len && answer_len && status && table, OMNI_E_PARAM,
             "decode needs the page table, the three length vectors and a status word");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float* part_ml = static_cast<float*>(workspace);
  float* part_acc = part_ml + (size_t)batch * n_q_heads * n_chunks * 2;
  CUtensorMap mk, mv;
  int rc = omni_make_tmap_rows(&mk, pool_k, (uint64_t)n_pages * dec::PAGE, dec::D, 2, 64, dec::PAGE);
  if (rc) return rc;
  rc = omni_make_tmap_rows(&mv, pool_v, (uint64_t)n_pages * dec::PAGE, dec::D, 2, 64, dec::PAGE);
  if (rc) return rc;
  OMNI_CUDA_TRY(omni_smem_attr(dec::decode_partial_tma_kernel, (int)dec::TSMEM));
  int dev = 0, sms = 148;
  OMNI_CUDA_TRY(cudaGetDevice(&dev));
  OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int items = n_chunks * n_kv_heads * batch;
  const dec::Paged pg{table, max_pages, vision_len, text_len, answer_len, 1.0 / sqrt(static_cast<double>(head_dim))};
  const dec::FuseArgs fa{k_lazy, k_act, tau, preserve_first_head, flags_override, flags};
  dec::decode_partial_tma_kernel<<<min(sms, items), (dec::NCW + 1) * 32, dec::TSMEM, st>>>(
      mk, mv, static_cast<const __nv_bfloat16*>(q), pg, n_q_heads, n_kv_heads, part_ml, part_acc, n_chunks, items,
      fa, status);
  dec::decode_combine_kernel<<<dim3(n_q_heads, batch), dec::D, 0, st>>>(part_ml, part_acc, n_chunks, out, status);
  return omni_launch_check();
}

extern "C" int omni_append_answer(const void* k_rows, const void* v_rows, void* pool_k, void* pool_v,
                                  const int32_t* table, int max_pages, const int32_t* vision_len,
                                  const int32_t* text_len, int32_t* answer_len, int batch, int n_kv_heads,
                                  int head_dim, void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim >= 1 && head_dim <= dec::D, OMNI_E_SHAPE, "answer rows are stored with 128 columns");
  OMNI_CHECK(table && vision_len && text_len && answer_len, OMNI_E_PARAM, "append needs the page table and lengths");
  if (batch == 0) return OMNI_OK;
  const dec::Paged pg{table, max_pages, vision_len, text_len, answer_len, 0.0};
  dec::append_paged_kernel<<<batch, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_rows), static_cast<const uint4*>(v_rows), static_cast<uint4*>(pool_k),
      static_cast<uint4*>(pool_v), pg, n_kv_heads, answer_len);
  return omni_launch_check();
}

extern "C" int omni_page_write(const void* src, int n_groups, int src_rows, int head_dim, const int32_t* idx,
                               int idx_stride, int count, const int32_t* table, int max_pages, int first_slot,
                               void* pool, void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim == dec::D, OMNI_E_SHAPE, "page rows are 128 bf16 columns (zero-pad shorter rows first)");
  OMNI_CHECK(count >= 0 && n_groups >= 0 && first_slot >= 0, OMNI_E_SHAPE, "negative extent");
  if (count == 0 || n_groups == 0) return OMNI_OK;
  const int rows_per_cta = 256 / (dec::D * 2 / 16);  // 16
  const int padded = (count + dec::PAGE - 1) / dec::PAGE * dec::PAGE;
  dec::page_write_kernel<<<dim3((padded + rows_per_cta - 1) / rows_per_cta, n_groups), 256, 0,
                           static_cast<cudaStream_t>(stream)>>>(static_cast<const uint4*>(src), src_rows, idx,
                                                                idx_stride, count, table, max_pages, first_slot,
                                                                static_cast<uint4*>(pool));
  return omni_launch_check();
}

// classify_decode_query (decode.py:124-140) alone: flags u8 [B, Hq] for one
// decode token per sequence (the classification K7 also fuses).
extern "C" int omni_decode_flags(const void* q, const double* k_lazy, const double* k_act, int batch, int n_q_heads,
                                 int n_kv_heads, int head_dim, double tau, int preserve_first_head, uint8_t* flags,
                                 void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim >= 1 && head_dim <= dec::D, OMNI_E_SHAPE, "decode queries are stored with 128 columns");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0 && n_q_heads / n_kv_heads <= dec::MAXREP, OMNI_E_SHAPE,
             "need Hq a multiple of Hkv with at most 8 Q heads per group");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  if (batch == 0) return OMNI_OK;
  dec::decode_flags_kernel<<<dim3(n_kv_heads, batch), 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), k_lazy, k_act, n_q_heads, n_kv_heads, tau,
      1.0 / sqrt(static_cast<double>(head_dim)), preserve_first_head, nullptr, flags);
  return omni_launch_check();
}

namespace omni {
namespace dec {
// classify_decode_query (decode.py:124-140) on float64 queries (the
// reference's own precision, for the reference-signature operators): one warp
// per (sequence, Q head), logits q . k / sqrt(head_dim) over the logical head
// dims, the max-subtracted two-way softmax and the strict p_act > tau.
__global__ void decode_flags_f64_kernel(const double* __restrict__ q, const double* __restrict__ k_lazy,
                                        const double* __restrict__ k_act, int Hq, int Hkv, int dl, int ldk,
                                        double tau, int preserve, uint8_t* __restrict__ flags) {
  const int h = blockIdx.x, s = blockIdx.y, lane = threadIdx.x, g = h / (Hq / Hkv);
  const double* qr = q + ((size_t)s * Hq + h) * dl;
  const double* kl = k_lazy + ((size_t)s * Hkv + g) * ldk;
  const double* ka = k_act + ((size_t)s * Hkv + g) * ldk;
  double a = 0.0, b = 0.0;
  for (int c = lane; c < dl; c += 32) {
    a = fma(qr[c], kl[c], a);
    b = fma(qr[c], ka[c], b);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    const double scale = 1.0 / sqrt(static_cast<double>(dl));
    const double l0 = a * scale, l1 = b * scale, mx = fmax(l0, l1);
    const double e0 = exp(l0 - mx), e1 = exp(l1 - mx);
    int f = (e1 / (e0 + e1) > tau) ? 1 : 0;
    if (preserve && h == 0) f = 1;
    flags[(size_t)s * Hq + h] = static_cast<uint8_t>(f);
  }
}
}  // namespace dec
}  // namespace omni

extern "C" int omni_decode_flags_f64(const double* q, const double* k_lazy, const double* k_act, int batch,
                                     int n_q_heads, int n_kv_heads, int head_dim, int probe_stride, double tau,
                                     int preserve_first_head, uint8_t* flags, void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim >= 1 && head_dim <= probe_stride, OMNI_E_SHAPE, "head_dim exceeds the probe-key row stride");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(tau >= 0.0 && tau < 1.0, OMNI_E_PARAM, "tau must be in [0, 1)");
  if (batch == 0) return OMNI_OK;
  dec::decode_flags_f64_kernel<<<dim3(n_q_heads, batch), 32, 0, static_cast<cudaStream_t>(stream)>>>(
      q, k_lazy, k_act, n_q_heads, n_kv_heads, head_dim, probe_stride, tau, preserve_first_head, flags);
  return omni_launch_check();
}
