// K4: gathered sparse flash-attention forward on tcgen05 / TMEM / TMA.
//
// Replaces sparse_head_attention (prefill.py:89-122). One CTA owns 256
// compacted active query rows of one Q head as two 128-row tiles (A, B) and
// streams its GQA group's compacted selected keys (K_sel / V_sel from
// omni_gather_rows) in 128-key tiles. Visibility is the reference's
// `selected[j] <= row` in ORIGINAL positions; both index lists are ascending,
// so it is a per-row prefix j < vis(row) = #{selected <= row}: one compare on
// staircase tiles only, and each Q tile stops after ceil(vis(last row) / 128)
// key tiles (the causal staircase skips the rest).
//
// Operand placement (smem operand bandwidth is the limit of M=128 SS MMAs):
//   S = Q K^T : A = Q (smem, SW128), B = K (smem)        -> S in TMEM (fp32)
//   O += P V  : A = P (TMEM, bf16 pairs written over S),  B = V (smem)
// TMEM per tile X: S/P columns [256X, 256X+128), O [256X+128, 256X+256).
//
// Warp roles (576 threads, 1 CTA / SM, ~197 KB smem, 512 TMEM columns):
//   warp 0      TMA producer: K_j, V_j (two 64-column SWIZZLE_128B boxes each)
//               into 2-stage rings.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, ping-pong
//               per key tile j: PV_A(j), QK_A(j+1), PV_B(j), QK_B(j+1) — the
//               tensor core runs one tile's GEMMs while the other tile's
//               softmax warps work.
//   warps 2-17  softmax / correction / epilogue: warps 2-9 own tile A, 10-17
//               tile B. Two warps per TMEM lane quarter and tile split the 128
//               key columns (64 each), so every row is served by two threads
//               in different warps: the per-tile softmax latency, which bounds
//               the ping-pong (S -> P -> PV/QK -> S), is halved while the issue
//               slots of each SM sub-partition are shared by four softmax
//               warps. Row maxima are exchanged through shared memory with a
//               64-thread named barrier per (tile, lane quarter); exp2-domain
//               online softmax with lazy rescaling (O corrected only when the
//               running max grows by more than 2^8).
// Epilogue: O / l -> bf16 rows scattered to their original positions; rows
// with no visible key copy V[g, sink] (prefill.py:119-120); LSE side output
// for the backward kernel.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace omni {
namespace fwd {

constexpr int BM = 128, BN = 128, D = 128, NST = 2;
constexpr int NTHREADS = 576;  // TMA warp + MMA warp + 16 softmax warps
constexpr int HC = 64;         // key columns per softmax thread (half a tile row)
constexpr uint32_t ATOM = 128 * 128;  // 128 rows x 128 B swizzle region
constexpr uint32_t TILE = 2 * ATOM;   // 128 x 128 bf16
constexpr uint32_t OFF_Q = 0;                     // 2 Q tiles
constexpr uint32_t OFF_K = OFF_Q + 2 * TILE;      // NST stages
constexpr uint32_t OFF_V = OFF_K + NST * TILE;    // NST stages
constexpr uint32_t OFF_BAR = OFF_V + NST * TILE;
enum {
  B_QF = 0,             // [2] Q tile X in smem (128 arrivals)
  B_KF = 2,             // [NST]
  B_KE = 2 + NST,       // [NST]
  B_VF = 2 + 2 * NST,   // [NST]
  B_VE = 2 + 3 * NST,   // [NST]
  B_SF = 2 + 4 * NST,   // [2] S_X(j) ready (MMA commit)
  B_PF = 4 + 4 * NST,   // [2] P_X(j) in TMEM + O_X corrected (128 arrivals)
  B_PV = 6 + 4 * NST,   // [2] PV_X(j) done (MMA commit)
  B_COUNT = 8 + 4 * NST
};
constexpr uint32_t OFF_TMEM = OFF_BAR + 8 * B_COUNT;
constexpr uint32_t SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + alignment slack
constexpr uint32_t TMEM_COLS = 512;
#ifdef OMNI_FWD_WARP_PF
// Variants build flag: "P ready" as one arrival per softmax warp (after a
// __syncwarp; the TMEM stores being signalled are complete, tcgen05.wait::st)
// instead of one per thread.
constexpr uint32_t PF_COUNT = 2 * BM / 32;
__device__ __forceinline__ void arrive_pf(uint32_t b) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(b);
}
#else
constexpr uint32_t PF_COUNT = 2 * BM;
__device__ __forceinline__ void arrive_pf(uint32_t b) { mbar_arrive(b); }
#endif
__device__ __forceinline__ uint32_t col_s(int x) { return 256u * x; }
__device__ __forceinline__ uint32_t col_o(int x) { return 256u * x + 128u; }

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk16) {
  // byte offset of 16-byte chunk `chunk16` (0..7) of `row` in a SW128 atom
  return row * 128u + ((chunk16 ^ (row & 7u)) << 4);
}

// POLY: number of the 16 exponential pairs of a 32-column chunk evaluated by
// the FMA-pipe polynomial (degree 2, relative error <= 1.7e-3, about the
// bf16 half ulp P is rounded to anyway) instead of MUFU.EX2 (full tiles only;
// staircase tiles, whose masked entries must be exactly 0, stay on MUFU). The
// chosen pairs are spread evenly so ptxas can interleave them with the MUFU
// stream. Default 6 (measured: degree 2 with 6 pairs ~2 % faster than degree
// 3 with 4).
template <int POLY>
__device__ __forceinline__ constexpr bool use_poly(int pair) {
  return POLY > 0 && ((pair * POLY) % 16) < POLY;
}

// Profiling-only cycle accounting (OMNI_FWD_TRACE=1): per-phase clock sums of
// lane 0 of every softmax / MMA warp, read back with omni_debug_fwd_trace.
__device__ unsigned long long g_fwd_trace[8];

#ifdef OMNI_FWD_CTA_TIMING
// Profiling build only (VFLAGS=-DOMNI_FWD_CTA_TIMING, profiles/k4_cta_timing.py):
// per-CTA wall-clock phases of the fast kernel in ns (globaltimer), summed
// into g_fwd_trace: [0] start -> first QK issued (prologue), [1] tile A's
// last PV complete -> exit (epilogue), [2] start -> exit, [3] CTAs, [4] SM
// cycles over the CTA (with [2]: the effective SM clock), [5] start -> set-up
// barrier, [6] start -> thread 64's row / Q loads done, [7] start -> its
// visible-key count done.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// FAST: deferred agreement between the two halves of a row (see the tile loop);
// a tile whose logits jump by more than 2^64 over the running max sets
// *status and the launch is redone by the FAST = false kernel (only_if).
// One CTA's work: 256 compacted rows (tile pair L) of one Q head. `reuse`:
// the CTA runs further tiles after this one (mbarriers invalidated at exit).
template <int POLY, bool TRACE, bool FAST>
__device__ __forceinline__ void fwd_tile(int L, bool reuse, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                         const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                                         const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                                         const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts,
                                         int Hq, int rep, int N, int cap, int sel_stride, int sink, int n_tiles_max,
                                         __nv_bfloat16* __restrict__ O, float* __restrict__ lse,
                                         int* __restrict__ status) {
  extern __shared__ uint8_t smem_raw[];
#ifdef OMNI_FWD_CTA_TIMING
  const unsigned long long t_start = gtimer();
  const long long c_start = clock64();
  __shared__ unsigned long long s_t_first, s_t_last, s_t_vis;
#endif
  const int h = L % Hq;
  // Heaviest (latest rows) tile pairs first, counted down from the largest
  // active-row count over the heads (device-side: the grid is sized for N
  // rows, so the tile pairs beyond every head's count come last and cost
  // nothing, instead of opening the launch with waves of empty CTAs).
  int cmax = 0;
  for (int k = threadIdx.x & 31; k < Hq; k += 32) cmax = max(cmax, __ldg(counts + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  const int tile = (cmax + 2 * BM - 1) / (2 * BM) - 1 - L / Hq;
  const int cnt = __ldg(counts + h);
  const int row0 = tile * 2 * BM;
  if (tile < 0 || row0 >= cnt) return;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ int s_nt[2];
  __shared__ float s_xch[2][BM][2];  // per (tile, row, half): partial row max, then l

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;
  const int32_t* rows_t = rows + (size_t)h * N + row0;

  // Softmax threads: row position, visible-key count and the Q half-row
  // are fetched before the CTA barrier (the binary searches of all rows run in
  // parallel); the thread owning a tile's last row publishes its key-tile count.
  const int sidx = warp - 2;                            // softmax warp index 0..15
  const int xs = sidx >> 3;                             // its Q tile
  const int hf = (sidx >> 2) & 1;                       // its key-column half
  const int is = (warp & 3) * 32 + lane;                // its row == TMEM lane
  const int nrows_s = min(BM, cnt - row0 - xs * BM);
  const bool rvalid = warp >= 2 && is < nrows_s;
  const int pos = rvalid ? __ldg(rows_t + xs * BM + is) : 0;
  uint4 qv[8];
  if (warp >= 2) {
    const uint4* qrow = reinterpret_cast<const uint4*>(Q + ((size_t)h * N + pos) * D) + hf * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) qv[c] = rvalid ? __ldg(qrow + c) : make_uint4(0, 0, 0, 0);
  }
#ifdef OMNI_FWD_CTA_TIMING
  const unsigned long long t_loaded = gtimer();  // row position and Q half-row loaded
#endif
  // visible-key counts: a warp's 32 rows are consecutive compacted rows, so
  // one warp-cooperative search (32 pivots per level, then a scan of the
  // window between its smallest and largest row) replaces 32 binary searches
  // of ~15 dependent L2 loads each (6.8 of the 10.7 us CTA prologue at 64K)
  int vis = warp >= 2 ? count_le_warp(selg, nsel, pos, rvalid) : 0;
  if (!rvalid) vis = 0;
#ifdef OMNI_FWD_CTA_TIMING
  if (FAST && threadIdx.x == 64) {
    s_t_vis = gtimer();
    atomicAdd(&g_fwd_trace[6], t_loaded - t_start);
  }
#endif
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
      mbar_init(B(B_PF + x), PF_COUNT);
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
    tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
    if (!reuse) tmem_relinquish();  // a reusing CTA allocates again for its next tile
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#ifdef OMNI_FWD_CTA_TIMING
  if (FAST && threadIdx.x == 0) atomicAdd(&g_fwd_trace[5], gtimer() - t_start);  // start -> set-up barrier
#endif
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
      // observe the last "stage free" phases too (each K / V tile's stage is
      // committed once; every mbarrier phase is waited on)
      for (int j = ntm > NST ? ntm - NST : 0; j < ntm; ++j) {
        mbar_wait(B(B_KE + j % NST), (j / NST) & 1);
        mbar_wait(B(B_VE + j % NST), (j / NST) & 1);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    // The whole warp runs the schedule (warp-uniform control and descriptor
    // arithmetic in uniform registers); elect.sync picks the issuing lane.
    if (ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, D, 0, 1);
      const int nt[2] = {ntA, ntB};
      // Descriptor bases; per-K-step offsets are added to the 14-bit start
      // address field (addresses < 256 KB, no carry out of the field).
      const uint64_t dq0 = sdesc_sw128(sbase + OFF_Q, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, ATOM, 1024);
      auto qk = [&](int x, int j) {  // S_X(j) = Q_X K_j^T
        const uint64_t qd = dq0 + ((x * TILE) >> 4), kd = dk0 + (((j % NST) * TILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + col_s(x), qd + off, kd + off, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_ws(B(B_SF + x));
      };
      // prologue: S(0) for both tiles
      mbar_wait(B(B_KF), 0);
      for (int x = 0; x < 2; ++x) {
        if (nt[x] == 0) continue;
        mbar_wait(B(B_QF + x), 0);
        tc_fence_after();
#ifdef OMNI_FWD_CTA_TIMING
        if (x == 0 && lane == 0) s_t_first = gtimer();
#endif
        qk(x, 0);
      }
      umma_commit_ws(B(B_KE + 0));
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NST;
        mbar_wait(B(B_VF + s), (j / NST) & 1);
        bool kwaited = false;
        const uint64_t vd = dv0 + ((s * TILE) >> 4);
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          if constexpr (TRACE) {
            const uint32_t t0 = clock();
            mbar_wait(B(B_PF + x), j & 1);
            if (lane == 0) atomicAdd(&g_fwd_trace[6], (unsigned long long)(clock() - t0));
          } else {
            mbar_wait(B(B_PF + x), j & 1);  // P_X(j) written (and O_X corrected)
          }
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts_ws(tmem + col_o(x), tmem + col_s(x) + (kk >> 2) * HC + (kk & 3) * 8, vd + ((kk * 2048) >> 4), idesc_pv,
                            (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit_ws(B(B_PV + x));
          if (j + 1 < nt[x]) {
            if (!kwaited) {
              mbar_wait(B(B_KF + (j + 1) % NST), ((j + 1) / NST) & 1);
              tc_fence_after();
              kwaited = true;
            }
            qk(x, j + 1);  // executes after PV_X(j): the tensor pipe is in order, so P is consumed first
          }
        }
        umma_commit_ws(B(B_VE + s));
        if (kwaited) umma_commit_ws(B(B_KE + (j + 1) % NST));
      }
    }
  } else {
    // ------------------------------------------------------ softmax warps
    const int x = xs;                            // Q tile of this warp
    const int quarter = warp & 3;                // TMEM lane quarter of this warp
    const int i = is;                            // row within the tile == TMEM lane
    const int cb = hf * HC;                      // first key column of this thread
    const uint32_t bid = 1 + x * 4 + quarter;    // named barrier of the two halves of these rows
    const int nt = x ? ntB : ntA;
    const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16);
    float m_run = -INFINITY, l_run = 0.f;
    float pend_alpha = 1.f;  // FAST: O rescale agreed after the previous tile's release
    if (nt > 0) {
      // Q half-row -> swizzled K-major smem tile (A operand of S = Q K^T).
      uint8_t* q_gen = smem + OFF_Q + x * TILE + hf * ATOM;
#pragma unroll
      for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(q_gen + swz(i, c)) = qv[c];
      fence_proxy_async_smem();
      mbar_arrive(B(B_QF + x));

      const float sl2 = static_cast<float>(kLog2e / sqrt(static_cast<double>(D)));
      const Exp2PolyConsts pc = exp2_poly_consts();
      uint32_t tr[5] = {0, 0, 0, 0, 0};
      uint32_t tc0 = clock();
      auto tick = [&](int k) {
        if constexpr (TRACE) {
          const uint32_t t = clock();
          tr[k] += t - tc0;
          tc0 = t;
        }
      };
      for (int j = 0; j < nt; ++j) {
        tick(4);
        mbar_wait(B(B_SF + x), j & 1);  // S_X(j) ready (and, in order, PV_X(j-1) done)
        // observe PV_X(j-1)'s phase (complete already: the commit of S_X(j)
        // covers every earlier MMA), so every phase of B_PV is waited on
        if (j > 0) mbar_wait(B(B_PV + x), (j - 1) & 1);
        tc_fence_after();
        tick(0);
        if constexpr (POLY < 0) {  // profiling only: the MMA / TMA pipeline without softmax work
          tc_fence_before();
          arrive_pf(B(B_PF + x));
          l_run = 1.f;
          continue;
        }
        const int lim_row = vis - j * BN;  // visible keys of this row in key tile j
        const int lim = lim_row - cb;      // ... within this thread's 64 columns
        const bool full = __all_sync(0xffffffffu, lim >= HC);
        // exp2(s * sl2 - m) of a 32-column chunk -> packed bf16 pk[16], row sum
        auto exps = [&](auto full_c, const uint32_t* sr, float nmu, uint32_t* pk) -> float {
          constexpr bool FULL = decltype(full_c)::value;
          const uint64_t c2 = f32x2(sl2, sl2), n2 = f32x2(nmu, nmu);
          uint64_t acc0 = f32x2(0.f, 0.f), acc1 = f32x2(0.f, 0.f);
#pragma unroll
          for (int c = 0; c < 32; c += 2) {
            const uint64_t xx = ffma2(f32x2(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), c2, n2);
            uint64_t pp;
            if (FULL && use_poly<POLY>(c >> 1)) {
              pp = exp2_poly2_pair(xx, pc);  // FMA-pipe share (MUFU relief), degree 2
            } else {
              pp = f32x2(fast_exp2(f32x2_lo(xx)), fast_exp2(f32x2_hi(xx)));
            }
            if ((c & 2) == 0) acc0 = fadd2(acc0, pp); else acc1 = fadd2(acc1, pp);
            pk[c >> 1] = pack_bf16x2(f32x2_lo(pp), f32x2_hi(pp));
          }
          const uint64_t acc = fadd2(acc0, acc1);
          return f32x2_lo(acc) + f32x2_hi(acc);
        };
        // The running max m_run (log2 domain) is integral and shared by both
        // halves of a row. Chunks are exponentiated optimistically against
        // the current max m_cur while the chunk max is reduced alongside (no
        // max -> exp dependency); only a chunk exceeding m_cur by more than
        // 2^64 (the first visible tile, or an extreme logit jump) is redone
        // from registers against ceil(chunk max), so P <= 2^64 always.
        // Growth beyond 2^8 is settled after both chunks: one OR-barrier
        // between the halves; on the (rare) true branch they exchange their
        // maxima and rescale P, l and O by exact powers of two.
        auto chunk = [&](int q, float& m_cur, float& cmax, float& mu) -> float {
          uint32_t sr[32], pk[16];
          __syncwarp();
          tmem_ld32(tl + col_s(x) + cb + q * 32, sr);
          tmem_wait_ld();
          if (!full) {  // staircase tile: masked keys -> -inf -> exactly 0
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
          tmem_st16(tl + col_s(x) + cb + q * 16, pk);  // P over this thread's own, already-read S columns
          return rs;
        };
        // FAST path chunk: exponentials against the shared running max only.
        // No chunk maximum: every P <= 2^8 unless the half-row sum exceeds
        // 2^8, and log2 of the sum bounds the growth when it does.
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
          // Deferred agreement: unless some row of the warp sees its first
          // visible keys (both halves evaluate this identically), exponentiate
          // against the shared running max, release P at once, and settle any
          // growth beyond 2^8 afterwards, off the S -> P -> MMA critical path:
          // the OR-barrier and max exchange then run while the tensor core
          // works, and O is rescaled at the next tile (or in the epilogue).
          // A jump beyond 2^64 (P could overflow) flags the launch for a redo.
          {
            if (__any_sync(0xffffffffu, pend_alpha != 1.f)) {  // PV_X(j-1) complete (it precedes QK_X(j))
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
          }
          if (!__any_sync(0xffffffffu, m_run == -INFINITY && lim_row > 0)) {
            const float rs = chunk_fast(0, m_run) + chunk_fast(1, m_run);
            tmem_wait_st();
            tc_fence_before();
            arrive_pf(B(B_PF + x));
            // rows that have seen no visible key yet (m_run = -inf; their
            // masked P are NaN and never used) are excluded from both tests
            if (m_run != -INFINITY && !(rs <= 0x1p64f)) atomicExch(status, 1);  // some P may exceed 2^64
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
            tick(3);
            continue;
          }
        }
        float m_cur = m_run, cmax = -INFINITY, mu0, mu1;
        const float rs0 = chunk(0, m_cur, cmax, mu0);
        tick(1);
        const float rs1 = chunk(1, m_cur, cmax, mu1);
        tick(2);
        // target max of this half: its P max, raised when the tile grew > 2^8
        const float tgt = cmax > mu1 + 8.0f ? ceilf(cmax) : mu1;
        if (named_bar_red_or(bid, 2 * 32, tgt != m_run)) {
          s_xch[x][i][hf] = tgt;
          named_bar_sync(bid, 2 * 32);
          const float m_fin = fmaxf(tgt, s_xch[x][i][hf ^ 1]);
          named_bar_sync(bid, 2 * 32);  // both read before the slots are reused
          float f0 = 1.f, f1 = 1.f, alpha = 1.f;
          if (m_fin != -INFINITY) {
            f0 = pow2_int(mu0 - m_fin);
            f1 = pow2_int(mu1 - m_fin);
            alpha = pow2_int(m_run - m_fin);
          }
          l_run = l_run * alpha + rs0 * f0 + rs1 * f1;
          m_run = m_fin;
          if (__any_sync(0xffffffffu, f0 != 1.f)) {  // (f1 != 1 implies f0 != 1)
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
            // O_X(j-1) is stable: PV_X(j-1) precedes QK_X(j) in the tensor pipe
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
        tick(3);
        tmem_wait_st();
        tc_fence_before();
        arrive_pf(B(B_PF + x));
      }
      tick(4);
      if constexpr (TRACE) {
        if (lane == 0) {
          for (int k = 0; k < 5; ++k) atomicAdd(&g_fwd_trace[k], (unsigned long long)tr[k]);
          atomicAdd(&g_fwd_trace[5], (unsigned long long)nt);
        }
      }
      mbar_wait(B(B_PV + x), (nt - 1) & 1);
      tc_fence_after();
#ifdef OMNI_FWD_CTA_TIMING
      if (threadIdx.x == 64) s_t_last = gtimer();  // (a tile-A thread)
#endif
      // the row normaliser is the sum of both halves' partial sums
      s_xch[x][i][hf] = l_run;
      named_bar_sync(bid, 2 * 32);
      l_run += s_xch[x][i][hf ^ 1];
    }
    // ------------------------------------------------------ epilogue
    uint4* dst = reinterpret_cast<uint4*>(O + ((size_t)h * N + pos) * D + cb);
    if (nt > 0) {
      // (a rescale agreed after the last tile applies to O, already to l)
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
#ifdef OMNI_FWD_CTA_TIMING
  if (FAST && threadIdx.x == 0 && ntm > 0) {
    const unsigned long long t_end = gtimer();
    atomicAdd(&g_fwd_trace[0], s_t_first - t_start);
    atomicAdd(&g_fwd_trace[1], t_end - s_t_last);
    atomicAdd(&g_fwd_trace[2], t_end - t_start);
    atomicAdd(&g_fwd_trace[3], 1ull);
    atomicAdd(&g_fwd_trace[4], (unsigned long long)(clock64() - c_start));  // SM cycles over the CTA
    atomicAdd(&g_fwd_trace[7], s_t_vis - t_start);  // start -> thread 64's visible-key count
  }
#endif
  if (reuse) {  // the next tile re-initialises the barriers
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < B_COUNT; ++k) mbar_inval(B(k));
    __syncthreads();
  }
}

// REDO: the fallback instance behind a FAST launch (only_if = its status word).
template <int POLY, bool TRACE = false, bool FAST = false, bool REDO = false>
__global__ void __launch_bounds__(NTHREADS, 1)
sparse_fwd_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                  const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                  const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep, int N,
                  int cap, int sel_stride, int sink, int n_tiles_max, __nv_bfloat16* __restrict__ O,
                  float* __restrict__ lse, int* __restrict__ status, const int* __restrict__ only_if) {
  if constexpr (REDO) {
    // fallback launch (one CTA per SM): nothing to do unless the fast kernel
    // flagged a jump; then redo every tile pair, grid-stride
    if (*(volatile const int*)only_if == 0) return;
    const int total = n_tiles_max * Hq;
    for (int L = blockIdx.x; L < total; L += gridDim.x)
      fwd_tile<POLY, TRACE, false>(L, true, tm_k, tm_v, Q, Vorig, rows, counts, sel, sel_counts, Hq, rep, N, cap,
                                   sel_stride, sink, n_tiles_max, O, lse, status);
    return;
  }
  fwd_tile<POLY, TRACE, FAST>(blockIdx.x, false, tm_k, tm_v, Q, Vorig, rows, counts, sel, sel_counts, Hq, rep, N, cap,
                              sel_stride, sink, n_tiles_max, O, lse, status);
}

#ifdef OMNI_VARIANTS
// ---------------------------------------------------------------------------
// Row-per-thread variant (OMNI_FWD_IMPL=rpt): 8 softmax warps, 4 per Q tile,
// each thread owns one full row of S / P / O (128 key columns), so the row
// maximum, sum and the lazy-rescale decision need no exchange or named
// barrier between threads. Same TMA / MMA schedule as fwd_tile; P of a key
// tile is stored packed over the first 64 columns of the tile's S region
// (K-step kk of PV reads columns 8kk..8kk+7). Fast path: exponentials
// against the running max, growth settled from the row sum afterwards (as in
// fwd_tile's FAST mode, a jump beyond 2^64 flags *status for the redo
// launch); a warp whose rows see their first visible keys takes the two-pass
// path (row max, then exponentials).
namespace rpt {
constexpr int NTHREADS = 320;
}

template <int POLY>
__device__ __forceinline__ void fwd_tile_rpt(int L, const CUtensorMap& tm_k, const CUtensorMap& tm_v,
                                             const __nv_bfloat16* __restrict__ Q,
                                             const __nv_bfloat16* __restrict__ Vorig,
                                             const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                                             const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts,
                                             int Hq, int rep, int N, int cap, int sel_stride, int sink,
                                             __nv_bfloat16* __restrict__ O, float* __restrict__ lse,
                                             int* __restrict__ status) {
  extern __shared__ uint8_t smem_raw[];
  const int h = L % Hq;
  int cmax = 0;
  for (int k = threadIdx.x & 31; k < Hq; k += 32) cmax = max(cmax, __ldg(counts + k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  const int tile = (cmax + 2 * BM - 1) / (2 * BM) - 1 - L / Hq;
  const int cnt = __ldg(counts + h);
  const int row0 = tile * 2 * BM;
  if (tile < 0 || row0 >= cnt) return;

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar = sbase + OFF_BAR;
  auto B = [&](int i) { return bar + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  __shared__ int s_nt[2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = h / rep;
  const int nsel = __ldg(sel_counts + g);
  const int32_t* selg = sel + (size_t)g * sel_stride;
  const int32_t* rows_t = rows + (size_t)h * N + row0;

  const int xs = (warp - 2) >> 2;          // Q tile of a softmax warp
  const int is = (warp & 3) * 32 + lane;   // its row == TMEM lane
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
    if (is == nrows_s - 1) s_nt[xs] = (vis + BN - 1) / BN;
    if (nrows_s <= 0 && is == 0) s_nt[xs] = 0;
  }
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    for (int x = 0; x < 2; ++x) {
      mbar_init(B(B_QF + x), BM);
      mbar_init(B(B_SF + x), 1);
      mbar_init(B(B_PF + x), BM);
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
    if (ntm > 0) {
      constexpr uint32_t idesc_qk = idesc_bf16_f32(BM, BN, 0, 0);
      constexpr uint32_t idesc_pv = idesc_bf16_f32(BM, D, 0, 1);
      const int nt[2] = {ntA, ntB};
      const uint64_t dq0 = sdesc_sw128(sbase + OFF_Q, 16, 1024);
      const uint64_t dk0 = sdesc_sw128(sbase + OFF_K, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sbase + OFF_V, ATOM, 1024);
      auto qk = [&](int x, int j) {
        const uint64_t qd = dq0 + ((x * TILE) >> 4), kd = dk0 + (((j % NST) * TILE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          umma_bf16_ws(tmem + col_s(x), qd + off, kd + off, idesc_qk, kk > 0 ? 1u : 0u);
        }
        umma_commit_ws(B(B_SF + x));
      };
      mbar_wait(B(B_KF), 0);
      for (int x = 0; x < 2; ++x) {
        if (nt[x] == 0) continue;
        mbar_wait(B(B_QF + x), 0);
        tc_fence_after();
        qk(x, 0);
      }
      umma_commit_ws(B(B_KE + 0));
      for (int j = 0; j < ntm; ++j) {
        const int s = j % NST;
        mbar_wait(B(B_VF + s), (j / NST) & 1);
        bool kwaited = false;
        const uint64_t vd = dv0 + ((s * TILE) >> 4);
        for (int x = 0; x < 2; ++x) {
          if (j >= nt[x]) continue;
          mbar_wait(B(B_PF + x), j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts_ws(tmem + col_o(x), tmem + col_s(x) + kk * 8, vd + ((kk * 2048) >> 4), idesc_pv,
                            (j > 0 || kk > 0) ? 1u : 0u);
          umma_commit_ws(B(B_PV + x));
          if (j + 1 < nt[x]) {
            if (!kwaited) {
              mbar_wait(B(B_KF + (j + 1) % NST), ((j + 1) / NST) & 1);
              tc_fence_after();
              kwaited = true;
            }
            qk(x, j + 1);
          }
        }
        umma_commit_ws(B(B_VE + s));
        if (kwaited) umma_commit_ws(B(B_KE + (j + 1) % NST));
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
      auto load_chunk = [&](int q, int lim, bool full, uint32_t* sr) {
        __syncwarp();
        tmem_ld32(tl + col_s(x) + q * 32, sr);
        tmem_wait_ld();
        if (!full) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
        }
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
        mbar_wait(B(B_SF + x), j & 1);
        if (j > 0) mbar_wait(B(B_PV + x), (j - 1) & 1);
        tc_fence_after();
        const int lim = vis - j * BN;
        const bool full = __all_sync(0xffffffffu, lim >= BN);
        if (__any_sync(0xffffffffu, pend_alpha != 1.f)) {  // O(j-1) complete
          rescale_o(pend_alpha);
          pend_alpha = 1.f;
        }
        if (!__any_sync(0xffffffffu, m_run == -INFINITY && lim > 0)) {
          const float nmu = m_run == -INFINITY ? 0.f : -m_run;
          float rs = 0.f;
          // chunk q + 1's TMEM load is in flight while chunk q is exponentiated
          uint32_t sbuf[2][32];
          __syncwarp();
          tmem_ld32(tl + col_s(x), sbuf[0]);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t* sr = sbuf[q & 1];
            reg_fence32(sr);
            if (q < 3) tmem_ld32(tl + col_s(x) + (q + 1) * 32, sbuf[(q + 1) & 1]);
            if (!full) {
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (q * 32 + c >= lim) sr[c] = __float_as_uint(-INFINITY);
            }
            uint32_t pk[16];
            rs += full ? exps(std::true_type{}, sr, nmu, pk) : exps(std::false_type{}, sr, nmu, pk);
            tmem_st16(tl + col_s(x) + q * 16, pk);
            if (q < 3) tmem_wait_ld();
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(B(B_PF + x));
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
        // two-pass path: the row maximum over the visible keys of this tile first
        float cm = -INFINITY;
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          uint32_t sr[32];
          load_chunk(q, lim, full, sr);
#pragma unroll
          for (int c = 0; c < 32; c += 2) cm = fmax3(cm, __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        }
        cm *= sl2;
        float m_fin = m_run;
        if (cm != -INFINITY && (m_run == -INFINITY || cm > m_run + 8.f)) m_fin = ceilf(cm);
        const float alpha = (m_run == -INFINITY || m_fin == -INFINITY) ? 1.f : pow2_int(m_run - m_fin);
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) rescale_o(alpha);  // O(j-1) is stable
        l_run *= alpha;
        m_run = m_fin;
        const float nmu = m_run == -INFINITY ? 0.f : -m_run;
        float rs = 0.f;
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
          uint32_t sr[32], pk[16];
          load_chunk(q, lim, full, sr);
          rs += exps(std::false_type{}, sr, nmu, pk);
          tmem_st16(tl + col_s(x) + q * 16, pk);
        }
        l_run += rs;
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(B(B_PF + x));
      }
      mbar_wait(B(B_PV + x), (nt - 1) & 1);
      tc_fence_after();
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

template <int POLY>
__global__ void __launch_bounds__(rpt::NTHREADS, 1)
sparse_fwd_rpt_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                      const __nv_bfloat16* __restrict__ Q, const __nv_bfloat16* __restrict__ Vorig,
                      const int32_t* __restrict__ rows, const int32_t* __restrict__ counts,
                      const int32_t* __restrict__ sel, const int32_t* __restrict__ sel_counts, int Hq, int rep, int N,
                      int cap, int sel_stride, int sink, __nv_bfloat16* __restrict__ O, float* __restrict__ lse,
                      int* __restrict__ status) {
  fwd_tile_rpt<POLY>(blockIdx.x, tm_k, tm_v, Q, Vorig, rows, counts, sel, sel_counts, Hq, rep, N, cap, sel_stride,
                     sink, O, lse, status);
}
#endif  // OMNI_VARIANTS

}  // namespace fwd
}  // namespace omni

using namespace omni;

int omni_make_tmap_rows(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols_elems, int elem_bytes,
                        uint32_t box_cols, uint32_t box_rows);

static constexpr int kDefaultPoly = 6;

#ifdef OMNI_VARIANTS
int omni_sparse_attn_fwd_pair(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                              const int32_t* counts, const int32_t* selected, const int32_t* sel_counts,
                              int n_q_heads, int n_kv_heads, int seq_len, int cap, int sink_index, void* O,
                              float* lse, int poly, cudaStream_t stream);
int omni_sparse_attn_fwd_pp(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream);
int omni_sparse_attn_fwd_sp(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream);
int omni_sparse_attn_fwd_db(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int cap, int sink_index, void* O, float* lse, int32_t* status,
                            int poly, cudaStream_t stream);
#endif

// status: device int workspace (nullable). With it the FAST kernel runs first
// and the safe kernel is launched behind it, exiting at once unless a tile's
// logits jumped beyond 2^64 over the running max (then it redoes everything).
extern "C" int omni_sparse_attn_fwd_ex(const void* Q, const void* K_sel, const void* V_sel, const void* V,
                                       const int32_t* rows, const int32_t* counts, const int32_t* selected,
                                       const int32_t* sel_counts, int n_q_heads, int n_kv_heads, int seq_len,
                                       int head_dim, int cap, int sink_index, void* O, float* lse, int32_t* status,
                                       void* stream) {
  omni_begin();
  OMNI_CHECK(head_dim == 128, OMNI_E_SHAPE, "sparse attention kernel requires head_dim == 128");
  OMNI_CHECK(n_kv_heads >= 1 && n_q_heads % n_kv_heads == 0, OMNI_E_SHAPE, "n_q_heads must be a multiple of n_kv_heads");
  OMNI_CHECK(cap >= 128 && cap % 128 == 0, OMNI_E_SHAPE, "cap must be a positive multiple of 128");
  OMNI_CHECK(sink_index >= 0 && sink_index < seq_len, OMNI_E_LAYOUT, "sink_index outside the sequence");
  OMNI_CHECK(seq_len >= 1, OMNI_E_SHAPE, "empty sequence");
  cudaStream_t st_ = static_cast<cudaStream_t>(stream);
#ifdef OMNI_VARIANTS
  // Kernel choice: the single-CTA two-Q-tile ping-pong kernel below by
  // default (measured fastest at the 64K bench workload); OMNI_FWD_IMPL=pair
  // selects the CTA-pair kernel of attn_fwd2.cu (faster MMA/TMA pipeline, 6.8
  // vs 7.2 ms without softmax work, but its one-tile-per-SM softmax is the
  // bottleneck; profiles/r01_k4_notes.md).
  static const bool single = [] {
    const char* e = getenv("OMNI_FWD_IMPL");
    return !(e && strcmp(e, "pair") == 0);
  }();
  static const int poly_env = [] {
    const char* e = getenv("OMNI_FWD_POLY");
    return e ? atoi(e) : kDefaultPoly;
  }();
  static const bool rpt_impl = [] {
    const char* e = getenv("OMNI_FWD_IMPL");
    return e && strcmp(e, "rpt") == 0;
  }();
  if (rpt_impl && status != nullptr) {
    CUtensorMap tk, tv;
    int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
    if (st) return st;
    st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
    if (st) return st;
    auto kern = fwd::sparse_fwd_rpt_kernel<kDefaultPoly>;
    auto redo = fwd::sparse_fwd_kernel<kDefaultPoly, false, false, true>;
    OMNI_CUDA_TRY(omni_smem_attr(kern, (int)fwd::SMEM_BYTES));
    OMNI_CUDA_TRY(omni_smem_attr(redo, (int)fwd::SMEM_BYTES));
    const int n_tiles = (seq_len + 2 * fwd::BM - 1) / (2 * fwd::BM);
    const int rep = n_q_heads / n_kv_heads;
    OMNI_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st_));
    kern<<<n_tiles * n_q_heads, fwd::rpt::NTHREADS, fwd::SMEM_BYTES, st_>>>(
        tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
        sel_counts, n_q_heads, rep, seq_len, cap, seq_len, sink_index, static_cast<__nv_bfloat16*>(O), lse, status);
    int dev = 0, sms = 148;
    OMNI_CUDA_TRY(cudaGetDevice(&dev));
    OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    redo<<<std::min<unsigned>(n_tiles * n_q_heads, (unsigned)sms), fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(
        tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
        sel_counts, n_q_heads, rep, seq_len, cap, seq_len, sink_index, n_tiles, static_cast<__nv_bfloat16*>(O), lse,
        nullptr, status);
    return omni_launch_check();
  }
  // 1: CTA-pair ping-pong (attn_fwd_pp.cu), 2: double-buffered S (attn_fwd_db.cu),
  // 3: shared S / separate P (attn_fwd_sp.cu)
  static const int alt_impl = [] {
    const char* e = getenv("OMNI_FWD_IMPL");
    return !e ? 0 : strcmp(e, "pp") == 0 ? 1 : strcmp(e, "db") == 0 ? 2 : strcmp(e, "sp") == 0 ? 3 : 0;
  }();
  if (alt_impl) {
    static const bool pp_fast = [] {
      const char* e = getenv("OMNI_FWD_FAST");
      return !(e && atoi(e) == 0);
    }();
    int32_t* pst = (pp_fast && poly_env >= 0) ? status : nullptr;
    if (pst) OMNI_CUDA_TRY(cudaMemsetAsync(pst, 0, sizeof(int32_t), st_));
    int st = (alt_impl == 1 ? omni_sparse_attn_fwd_pp : alt_impl == 2 ? omni_sparse_attn_fwd_db : omni_sparse_attn_fwd_sp)(
        Q, K_sel, V_sel, V, rows, counts, selected, sel_counts, n_q_heads, n_kv_heads, seq_len, cap, sink_index, O,
        lse, pst, poly_env, st_);
    if (st || !pst) return st;
    // the single-CTA safe kernel redoes the launch if a tile's logits jumped beyond 2^64
    CUtensorMap tk, tv;
    st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
    if (st) return st;
    st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
    if (st) return st;
    auto redo = fwd::sparse_fwd_kernel<kDefaultPoly, false, false, true>;
    OMNI_CUDA_TRY(omni_smem_attr(redo, (int)fwd::SMEM_BYTES));
    const int n_tiles = (seq_len + 2 * fwd::BM - 1) / (2 * fwd::BM);
    int dev = 0, sms = 148;
    OMNI_CUDA_TRY(cudaGetDevice(&dev));
    OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    redo<<<std::min<unsigned>(n_tiles * n_q_heads, (unsigned)sms), fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(
        tk, tv, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(V), rows, counts, selected,
        sel_counts, n_q_heads, n_q_heads / n_kv_heads, seq_len, cap, seq_len, sink_index, n_tiles,
        static_cast<__nv_bfloat16*>(O), lse, nullptr, pst);
    return omni_launch_check();
  }
  if (!single)
    return omni_sparse_attn_fwd_pair(Q, K_sel, V_sel, V, rows, counts, selected, sel_counts, n_q_heads, n_kv_heads,
                                     seq_len, cap, sink_index, O, lse, poly_env, st_);
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
  if (st) return st;
  // Tuning knobs: OMNI_FWD_POLY = number of the 16 exponential pairs per
  // 32-column chunk on the FMA-pipe polynomial (0, 4, 6 or 8; full tiles
  // only); OMNI_FWD_FAST=0 disables the deferred-agreement kernel.
  static const int poly = [] {
    const char* e = getenv("OMNI_FWD_POLY");
    const int v = e ? atoi(e) : kDefaultPoly;
    return (v == -1 || v == 0 || v == 4 || v == 6 || v == 8) ? v : kDefaultPoly;
  }();
  static const bool trace = [] {
    const char* e = getenv("OMNI_FWD_TRACE");
    return e && atoi(e) != 0;
  }();
  static const bool fast_env = [] {
    const char* e = getenv("OMNI_FWD_FAST");
    return !(e && atoi(e) == 0);
  }();
  auto safe = trace ? fwd::sparse_fwd_kernel<4, true>  // profiling: per-phase cycle accounting
            : poly == -1 ? fwd::sparse_fwd_kernel<-1>  // profiling: MMA pipeline only, no softmax
            : poly == 0 ? fwd::sparse_fwd_kernel<0>
            : poly == 4 ? fwd::sparse_fwd_kernel<4>
            : poly == 8 ? fwd::sparse_fwd_kernel<8>
                        : fwd::sparse_fwd_kernel<6>;
  auto fast = poly == 0 ? fwd::sparse_fwd_kernel<0, false, true>
            : poly == 8 ? fwd::sparse_fwd_kernel<8, false, true>
            : poly == 6 ? fwd::sparse_fwd_kernel<6, false, true>
                        : fwd::sparse_fwd_kernel<4, false, true>;
  auto redo = poly == 0 ? fwd::sparse_fwd_kernel<0, false, false, true>
            : poly == 8 ? fwd::sparse_fwd_kernel<8, false, false, true>
            : poly == 6 ? fwd::sparse_fwd_kernel<6, false, false, true>
                        : fwd::sparse_fwd_kernel<4, false, false, true>;
  const bool use_fast = status != nullptr && fast_env && !trace && poly >= 0;
  OMNI_CUDA_TRY(omni_smem_attr(safe, (int)fwd::SMEM_BYTES));
  if (use_fast) {
    OMNI_CUDA_TRY(omni_smem_attr(fast, (int)fwd::SMEM_BYTES));
    OMNI_CUDA_TRY(omni_smem_attr(redo, (int)fwd::SMEM_BYTES));
  }
#else
  // Product build: the single-CTA two-Q-tile ping-pong kernel with 6 of 16
  // exponential pairs on the FMA-pipe polynomial, fast (deferred agreement)
  // with the safe kernel as its fallback. The measured alternatives (CTA
  // pair, other splits, per-phase tracing) live in the OMNI_VARIANTS build
  // (libomnisparse_variants.so, profiles/r01_k4_notes.md).
  CUtensorMap tk, tv;
  int st = omni_make_tmap_rows(&tk, K_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
  if (st) return st;
  st = omni_make_tmap_rows(&tv, V_sel, (uint64_t)n_kv_heads * cap, 128, 2, 64, fwd::BN);
  if (st) return st;
  auto safe = fwd::sparse_fwd_kernel<kDefaultPoly>;
  auto fast = fwd::sparse_fwd_kernel<kDefaultPoly, false, true>;
  auto redo = fwd::sparse_fwd_kernel<kDefaultPoly, false, false, true>;
  const bool use_fast = status != nullptr;
  OMNI_CUDA_TRY(omni_smem_attr(safe, (int)fwd::SMEM_BYTES));
  if (use_fast) {
    OMNI_CUDA_TRY(omni_smem_attr(fast, (int)fwd::SMEM_BYTES));
    OMNI_CUDA_TRY(omni_smem_attr(redo, (int)fwd::SMEM_BYTES));
  }
#endif
  const int n_tiles = (seq_len + 2 * fwd::BM - 1) / (2 * fwd::BM);
  dim3 grid(n_tiles * n_q_heads);
  const int rep = n_q_heads / n_kv_heads;
  auto qp = static_cast<const __nv_bfloat16*>(Q);
  auto vp = static_cast<const __nv_bfloat16*>(V);
  auto op = static_cast<__nv_bfloat16*>(O);
#ifdef OMNI_VARIANTS
  // profiling (OMNI_FWD_PERSIST_SAFE=1): the safe kernel as a persistent
  // grid-stride loop (the redo instance, one CTA per SM) instead of one CTA
  // per tile pair — isolates the per-CTA launch cost
  static const bool persist_safe = [] {
    const char* e = getenv("OMNI_FWD_PERSIST_SAFE");
    return e && atoi(e) != 0;
  }();
  if (persist_safe && status != nullptr) {
    const int one = 1;
    OMNI_CUDA_TRY(cudaMemcpyAsync(status, &one, sizeof(int32_t), cudaMemcpyHostToDevice, st_));
    int dev = 0, sms = 148;
    OMNI_CUDA_TRY(cudaGetDevice(&dev));
    OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    redo<<<std::min<unsigned>(grid.x, (unsigned)sms), fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(
        tk, tv, qp, vp, rows, counts, selected, sel_counts, n_q_heads, rep, seq_len, cap, seq_len, sink_index, n_tiles,
        op, lse, nullptr, status);
    return omni_launch_check();
  }
#endif
  if (use_fast) {
    OMNI_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), st_));
    fast<<<grid, fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(tk, tv, qp, vp, rows, counts, selected, sel_counts, n_q_heads,
                                                        rep, seq_len, cap, seq_len, sink_index, n_tiles, op, lse,
                                                        status, nullptr);
    int dev = 0, sms = 148;
    OMNI_CUDA_TRY(cudaGetDevice(&dev));
    OMNI_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const dim3 fb_grid(std::min<unsigned>(grid.x, (unsigned)sms));  // exits at once in the common case
    redo<<<fb_grid, fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(tk, tv, qp, vp, rows, counts, selected, sel_counts,
                                                           n_q_heads, rep, seq_len, cap, seq_len, sink_index, n_tiles,
                                                           op, lse, nullptr, status);
  } else {
    safe<<<grid, fwd::NTHREADS, fwd::SMEM_BYTES, st_>>>(tk, tv, qp, vp, rows, counts, selected, sel_counts, n_q_heads,
                                                        rep, seq_len, cap, seq_len, sink_index, n_tiles, op, lse,
                                                        nullptr, nullptr);
  }
  return omni_launch_check();
}

extern "C" int omni_sparse_attn_fwd(const void* Q, const void* K_sel, const void* V_sel, const void* V,
                                    const int32_t* rows, const int32_t* counts, const int32_t* selected,
                                    const int32_t* sel_counts, int n_q_heads, int n_kv_heads, int seq_len,
                                    int head_dim, int cap, int sink_index, void* O, float* lse, void* stream) {
  omni_begin();
  return omni_sparse_attn_fwd_ex(Q, K_sel, V_sel, V, rows, counts, selected, sel_counts, n_q_heads, n_kv_heads,
                                 seq_len, head_dim, cap, sink_index, O, lse, nullptr, stream);
}

#ifdef OMNI_VARIANTS
// Profiling support (OMNI_FWD_TRACE=1): copies the 8 per-phase cycle sums
// of the traced K4 launches to host memory and resets them.
extern "C" int omni_debug_fwd_trace(unsigned long long* host8) {
  omni_begin();
  OMNI_CUDA_TRY(cudaMemcpyFromSymbol(host8, fwd::g_fwd_trace, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  OMNI_CUDA_TRY(cudaMemcpyToSymbol(fwd::g_fwd_trace, z, sizeof(z)));
  return OMNI_OK;
}
#endif  // OMNI_VARIANTS
