/*
 * omnisparse.h — C ABI of libomnisparse, the B200 (sm_100a) implementation of
 * the OmniSparse sparse-attention hot path.
 *
 * Conventions (all entry points):
 *  - Plain device pointers and sizes; `stream` is a cudaStream_t (NULL = the
 *    legacy default stream). No allocation inside: outputs and workspaces are
 *    caller-owned. Kernels are stream-ordered and reentrant.
 *  - Return 0 (OMNI_OK) or an OMNI_E_* status. The codes map 1:1 onto the
 *    reference exception classes of slimattn/errors.py:4-37 (the Python layer
 *    raises them); omni_last_error() gives a message for the calling thread.
 *  - Tensor layouts are row-major: Q [Hq, N, d], K/V [Hkv, N, d] with GQA
 *    group g = h / (Hq / Hkv) (rule B). Decision-critical
 *    arithmetic (probe keys, classification, pooled probe, column mass,
 *    kurtosis, budget) is float64; attention uses bf16 operands with fp32
 *    accumulation on tcgen05 tensor cores.
 *
 * The reference's own native boundary is the kernel-core plugin selected in
 * backend.py:19-35 (softmax_rows / mean_pool_rows / kurtosis / colsum,
 * _core_cy.pyx:17,60,83,103). Its hot-path callers are fused here into the
 * K1..K7 entry points below; each cites the reference interface it replaces.
 */
#ifndef OMNISPARSE_H
#define OMNISPARSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OMNI_ABI_VERSION 3

enum omni_status {
  OMNI_OK = 0,
  OMNI_E_SHAPE = 1,              /* ShapeError            errors.py:8  */
  OMNI_E_PARAM = 2,              /* ParameterError        errors.py:12 */
  OMNI_E_DEGENERATE_ROW = 3,     /* DegenerateRowError    errors.py:16 */
  OMNI_E_INTEGRITY = 4,          /* IntegrityError        errors.py:20 */
  OMNI_E_LAYOUT = 5,             /* LayoutError           errors.py:24 */
  OMNI_E_DEGENERATE_CONTEXT = 6, /* DegenerateContextError errors.py:28 */
  OMNI_E_CUDA = 7                /* CUDA runtime failure                */
};

/* F64 inputs are accepted by the selection-side entry points (K1, K2, K3x,
 * gather): the reference's own precision, for drop-in callers holding
 * float64 workloads. Attention (K4/K5/K7) is bf16. */
enum omni_dtype { OMNI_DTYPE_BF16 = 0, OMNI_DTYPE_F32 = 1, OMNI_DTYPE_F64 = 2 };
enum omni_granularity { OMNI_GRAN_TOKEN = 0, OMNI_GRAN_BLOCK = 1 };

int omni_abi_version(void);
const char* omni_last_error(void);
/* OMNI_OK when the current device is sm_100 (B200); OMNI_E_CUDA otherwise. */
int omni_device_check(void);

/* ---------------------------------------------------------------- K1
 * Probe keys and pooled keys, one pass over K.
 * Replaces build_probe_keys (query_select.py:41-47) and mean_pool_rows(K)
 * inside probe_attention (block_probe.py:58; _core_cy.pyx:60-80).
 * K: [Hkv, N, d] (dtype); outputs f64: k_lazy, k_act [Hkv, d],
 * pooled_k [Hkv, nb, d] with nb = ceil(N / block_size).
 * workspace: omni_kv_probe_workspace() bytes.
 * Errors: LAYOUT if n_vision < 1 or sink_index outside [0, N).            */
size_t omni_kv_probe_workspace(int n_kv_heads, int seq_len, int head_dim, int block_size);
int omni_kv_probe(const void* K, int dtype, int n_kv_heads, int seq_len, int head_dim, int n_vision,
                  int sink_index, int block_size, double* k_lazy, double* k_act, double* pooled_k,
                  void* workspace, void* stream);

/* ---------------------------------------------------------------- K2
 * Lazy/active query classification + pooled queries, one pass over Q.
 * Replaces classify_queries / build_query_masks (query_select.py:50-92) and
 * mean_pool_rows(Q) (block_probe.py:57). Rows < n_vision are classified
 * (p_act > tau, strict), other rows active, head 0 all-active when
 * preserve_first_head. Outputs: active u8 [Hq, N]; p_act f64 [Hq, n_vision]
 * (nullable); pooled_q f64 [Hq, nb, d]; block_active i32 [Hq, nb] (active
 * rows per probe block, feeds omni_compact_rows). When O_zero (bf16
 * [Hq, N, d]) is non-NULL the lazy rows of the attention output are zeroed
 * here (prefill.py:105: lazy rows output zero vectors).
 * Errors: PARAM if tau outside [0, 1) (the reference raises ValueError).   */
int omni_q_score(const void* Q, int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim,
                 int n_vision, double tau, int preserve_first_head, int block_size, const double* k_lazy,
                 const double* k_act, uint8_t* active, double* p_act, double* pooled_q, int32_t* block_active,
                 void* O_zero, void* stream);

/* Active-row compaction: rows i32 [Hq, N] (ascending original positions of
 * active rows, the np.flatnonzero(active) of prefill.py:106), counts [Hq]. */
int omni_compact_rows(const uint8_t* active, const int32_t* block_active, int n_q_heads, int seq_len,
                      int block_size, int32_t* rows, int32_t* counts, void* stream);

/* ---------------------------------------------------------------- K3a
 * Block-probe column mass: per Q head h, softmax over the block-causal
 * pooled scores pq_h pk_g^T / sqrt(d), summed over rows (colsum).
 * Replaces probe_attention (block_probe.py:44-64) + the colsum of
 * block_scores_to_token_scores (block_probe.py:76).
 * mass f64 [Hq, nb]; workspace f64 [Hq, nb, nb] + [Hq, nb, 2].             */
size_t omni_probe_mass_workspace(int n_q_heads, int n_blocks);
int omni_probe_mass(const double* pooled_q, const double* pooled_k, int n_q_heads, int n_kv_heads, int n_blocks,
                    int head_dim, double* mass, void* workspace, void* stream);
/* Same result, additionally leaving the pooled scores S [Hq, nb, nb] and the
 * row statistics (max, sum) [Hq, nb, 2] in the workspace — the materialised
 * BlockProbeMap of block_probe.py:44-64 (validation / probe_attention API). */
int omni_probe_mass_map(const double* pooled_q, const double* pooled_k, int n_q_heads, int n_kv_heads, int n_blocks,
                        int head_dim, double* mass, void* workspace, void* stream);

/* ---------------------------------------------------------------- K3x
 * Exact key scores (score_source = "exact"): per Q head the column mass of the
 * full causal attention map softmax(q k^T / sqrt(d)), float64, in two passes
 * over the causal triangle without materialising it. Replaces
 * accumulated_key_scores over the dense oracle maps (kv_select.py:56-73,
 * prefill.py:133-134, attention.py:99-108). Q [Hq, N, d], K [Hkv, N, d]
 * (dtype); mass f64 [Hq, N]; workspace omni_exact_mass_workspace() bytes.
 * O(N^2 d) float64 work: a validation-scale path (the hot path is K3a).     */
size_t omni_exact_mass_workspace(int n_q_heads, int seq_len);
int omni_exact_mass(const void* Q, const void* K, int dtype, int n_q_heads, int n_kv_heads, int seq_len, int head_dim,
                    double* mass, void* workspace, void* stream);

/* ---------------------------------------------------------------- K3b
 * Shared-budget KV selection from per-Q-head block column mass.
 * Replaces block_scores_to_token_scores (block_probe.py:67-78, per-token =
 * mass / block length), rule-B group sums, key_scores_from_vectors /
 * kurtosis (kv_select.py:49-53), flattest_head (kv_select.py:76-80),
 * budget_with_retained_mass (kv_select.py:104-120), build_key_masks /
 * top_b_indices (kv_select.py:123-144) or select_top_blocks (:147-176), and
 * select_vision_keys (:179-195) when vision_limit >= 0.
 * block_mass f64 [Hq, nb] (block_size = 1 gives the exact token path);
 * budget_override > 0 skips the budget search (decode hand-off).
 * Outputs: selected i32 [Hkv, seq_len] (ascending, first b valid per group),
 * info i32 [4 + Hkv] = {budget, flattest, Hkv, nb, per-group counts...},
 * stats f64 [Hkv + 4] = {kurtoses..., retained, total, margin, replayed}:
 * margin = distance of the budget decision from the threshold / total,
 * replayed = 1.0 when that margin was inside the rounding bound and the
 * reference's sequential cumsum decided; group_scores f64 [Hkv, nb] =
 * per-token score of each block.
 * Kurtosis is computed in NumPy's pairwise order and the budget is replayed
 * in the reference's order whenever the fast scan could disagree with it, so
 * for identical score vectors flattest group, budget and index sets equal the
 * reference's bit for bit.
 * workspace: omni_select_workspace() bytes (0 on the hot path: Hkv <= 8 and
 * nb <= 1024; otherwise the general path needs it; seq_len <= 1,835,008).
 * Errors: PARAM for p outside (0, 1], empty vision span, missing workspace. */
size_t omni_select_workspace(int n_kv_heads, int seq_len, int block_size);
int omni_select_ex(const double* block_mass, int n_q_heads, int n_kv_heads, int seq_len, int block_size, double p,
                   int granularity, int vision_limit, int budget_override, int32_t* selected, int32_t* info,
                   double* stats, double* group_scores, void* workspace, void* stream);
/* omni_select: SURVEY §8b's name; omni_select_ex without a workspace.      */
int omni_select(const double* block_mass, int n_q_heads, int n_kv_heads, int seq_len, int block_size, double p,
                int granularity, int vision_limit, int budget_override, int32_t* selected, int32_t* info,
                double* stats, double* group_scores, void* stream);

/* Block sums of per-token score rows in np.add.reduceat order (first element
 * + pairwise sum of the rest): x f64 [rows, n] -> out f64 [rows, nb]. The
 * block mass of select_top_blocks (kv_select.py:160). */
int omni_block_sums(const double* x, int rows, int n, int block_size, double* out, void* stream);

/* select_top_blocks (kv_select.py:147-176) from given block masses: per
 * group, blocks ranked by mass (ties to the lower block), whole blocks taken
 * in rank order and the marginal block's lowest indices, exactly `budget`
 * keys. block_mass f64 [G, nb]; selected i32 [G, seq_len] (ascending, first
 * budget valid); info i32 [4 + G] (entries 4.. = per-group counts).
 * workspace: omni_top_blocks_workspace() bytes.                           */
size_t omni_top_blocks_workspace(int groups, int seq_len, int block_size);
int omni_top_blocks(const double* block_mass, int groups, int seq_len, int block_size, int budget,
                    int32_t* selected, int32_t* info, void* workspace, void* stream);

/* The materialised BlockProbeMap (block_probe.py:60-63) from the workspace
 * omni_probe_mass_map left: map f64 [Hq, nb, nb], zero above the diagonal. */
int omni_probe_map(const void* workspace, int n_q_heads, int n_blocks, double* map, void* stream);

/* ---------------------------------------------------------------- K6
 * Row gather / KV regrouping: dst[g, r, :] = src[g, idx[g, r], :] for
 * r < count_g, zero rows for r in [count_g, roundup(count_g, pad_rows)).
 * Replaces the k[selected]/v[selected] gathers of prefill.py:109-110 and the
 * cache pruning + regrouping of build_cache (decode.py:92-107).
 * counts: device i32 [G] or NULL (then count_const for every group).       */
int omni_gather_rows(const void* src, int dtype, int n_groups, int src_rows, int head_dim, const int32_t* idx,
                     int idx_stride, const int32_t* counts, int count_const, void* dst, int dst_rows, int pad_rows,
                     void* stream);

/* Cache slimming for one sequence (build_cache, decode.py:82-108; the
 * omni_slim_cache of SURVEY §8b): vision_k/v [Hkv, vcap, d] = K/V rows
 * vision_selected[g, :budget] (ascending, inside the vision span), rows
 * [budget, vcap) zero. Errors: INTEGRITY when budget is outside [1, vcap]. */
int omni_slim_cache(const void* K, const void* V, int dtype, int n_kv_heads, int seq_len, int head_dim,
                    const int32_t* vision_selected, int sel_stride, int budget, int vcap, void* vision_k,
                    void* vision_v, void* stream);

/* Inverse of omni_gather_rows: dst[g, idx[g, r]] = src[g, r] for
 * r < counts[g] (device i32 [G]); other dst rows are untouched. Used to put
 * compacted key gradients back at their original positions. */
int omni_scatter_rows(const void* src, int dtype, int n_groups, int src_rows, int head_dim, const int32_t* idx,
                      int idx_stride, const int32_t* counts, void* dst, int dst_rows, void* stream);

/* Key-gradient epilogue of the training backward (autograd glue, no
 * reference counterpart: slimattn has no backward): dst[g, idx[g, r]] =
 * cast(src[g, r] + (idx[g, r] == sink_index ? sink_add[g] : 0)) for
 * r < counts[g], src fp32 [G, src_rows, head_dim], dst (dst_dtype f32 or
 * bf16) [G, dst_rows, head_dim] zero-initialised by the caller; when
 * sink_add (fp32 [G, head_dim], nullable) is given and sink_index is not
 * among a group's indices, dst[g, sink_index] = cast(sink_add[g]). idx rows
 * ascending. One pass replaces scatter + sink add + dtype cast. */
int omni_scatter_key_grads(const float* src, int n_groups, int src_rows, int head_dim, const int32_t* idx,
                           int idx_stride, const int32_t* counts, int sink_index, const float* sink_add, void* dst,
                           int dst_dtype, int dst_rows, void* stream);

/* ---------------------------------------------------------------- K4
 * Gathered sparse flash-attention forward (tcgen05 + TMEM + TMA).
 * Replaces sparse_head_attention (prefill.py:89-122) for every Q head:
 * active row rows[h, i] attends to the group's selected keys j with
 * selected[g, j] <= rows[h, i] (original positions), softmax renormalised;
 * rows with no visible key copy V[g, sink]; lazy rows are untouched (zeroed
 * by omni_q_score). Q, V bf16 original layout; K_sel / V_sel bf16
 * [Hkv, cap, d] compacted by omni_gather_rows with pad_rows = 128.
 * O bf16 [Hq, N, d]; lse f32 [Hq, N] (nullable; natural-log normaliser of the
 * row's softmax, -inf for fallback rows). head_dim must be 128.           */
int omni_sparse_attn_fwd(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                         const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                         int n_kv_heads, int seq_len, int head_dim, int cap, int sink_index, void* O, float* lse,
                         void* stream);
/* Same, with a device int32 status word (caller-owned, 4 bytes): enables the
 * deferred-agreement fast kernel, backed by the safe kernel that re-runs the
 * launch only when the fast one flagged a logit jump beyond 2^64 (status is
 * left 1 in that case). status == NULL is omni_sparse_attn_fwd. */
int omni_sparse_attn_fwd_ex(const void* Q, const void* K_sel, const void* V_sel, const void* V, const int32_t* rows,
                            const int32_t* counts, const int32_t* selected, const int32_t* sel_counts, int n_q_heads,
                            int n_kv_heads, int seq_len, int head_dim, int cap, int sink_index, void* O, float* lse,
                            int32_t* status, void* stream);

/* ---------------------------------------------------------------- K5
 * Backward of K4 (no reference counterpart: the reference has no autograd).
 * dO bf16 [Hq, N, d]; O, lse from K4. Outputs (fp32, zero-initialised by
 * the callee): dQ [Hq, N, d] (lazy rows 0), dK_sel / dV_sel [Hkv, cap, d]
 * over the compacted keys; fallback rows add dO into dV_sink [Hkv, d].
 * workspace: omni_sparse_attn_bwd_workspace() bytes.                      */
size_t omni_sparse_attn_bwd_workspace(int n_q_heads, int seq_len);
int omni_sparse_attn_bwd(const void* Q, const void* K_sel, const void* V_sel, const void* O, const void* dO,
                         const float* lse, const int32_t* rows, const int32_t* counts, const int32_t* selected,
                         const int32_t* sel_counts, int n_q_heads, int n_kv_heads, int seq_len, int head_dim, int cap,
                         float* dQ, float* dK_sel, float* dV_sel, float* dV_sink, void* workspace, void* stream);
/* As omni_sparse_attn_bwd with dQ in dtype dq_dtype (OMNI_DTYPE_F32 or
 * OMNI_DTYPE_BF16: the training dtype written directly by the dq kernel). */
int omni_sparse_attn_bwd_ex(const void* Q, const void* K_sel, const void* V_sel, const void* O, const void* dO,
                            const float* lse, const int32_t* rows, const int32_t* counts, const int32_t* selected,
                            const int32_t* sel_counts, int n_q_heads, int n_kv_heads, int seq_len, int head_dim,
                            int cap, int dq_dtype, void* dQ, float* dK_sel, float* dV_sel, float* dV_sink,
                            void* workspace, void* stream);

/* ---------------------------------------------------------------- K7
 * One slimmed decode step for a batch of sequences over a PAGED slim cache.
 * Replaces classify_decode_query + _fetched_segments + decode_attention
 * (decode.py:124-194) under rule B: Q head h is classified (f64) against its
 * group's frozen probe keys (head 0 forced active when preserve_first_head);
 * a group's vision segment is read iff any of its Q heads is active; lazy Q
 * heads attend over text + answer only (exclusion semantics, decode.py:12-16).
 * Cache: pool_k / pool_v bf16 [n_pages, 64, 128]; table i32
 * [B, Hkv, max_pages] lists each (sequence, group)'s pages: ceil(vision/64)
 * vision pages, then ceil(text/64) text pages, then ceil(answer/64) answer
 * pages; vision_len / text_len / answer_len i32 [B] rows per sequence.
 * Rows are stored with 128 columns; head_dim <= 128 is the logical width
 * (rows zero-padded past it) and sets the softmax scale 1 / sqrt(head_dim).
 * n_chunks = max over sequences of ceil(pages / 32). q bf16 [B, Hq, 128];
 * k_lazy / k_act f64 [B, Hkv, 128]; flags_override u8 [B, Hq] (nullable: the
 * flags hook of decode.py:170-173). Outputs: flags u8 [B, Hq]; out f32
 * [B, Hq, 128]; status i32 (device, required) = 1 when a lazy head had no
 * text and no answer key (DegenerateContextError, decode.py:152-153),
 * without a host synchronisation. workspace: omni_decode_workspace().       */
size_t omni_decode_workspace(int batch, int n_q_heads, int n_chunks);
int omni_decode(const void* q, const void* pool_k, const void* pool_v, int n_pages, const int32_t* table,
                int max_pages, const int32_t* vision_len, const int32_t* text_len, const int32_t* answer_len,
                int n_chunks, const double* k_lazy, const double* k_act, int batch, int n_q_heads, int n_kv_heads,
                int head_dim, double tau, int preserve_first_head, const uint8_t* flags_override, uint8_t* flags,
                float* out, void* workspace, int32_t* status, void* stream);

/* append_answer (decode.py:111-121) for a batch in one launch: bf16 k/v_rows
 * [B, Hkv, 128] go to answer row answer_len[s] of every (sequence, group) —
 * its page must already be in the table (the host allocates one every 64
 * tokens) — and answer_len[s] advances on the device.                      */
int omni_append_answer(const void* k_rows, const void* v_rows, void* pool_k, void* pool_v, const int32_t* table,
                       int max_pages, const int32_t* vision_len, const int32_t* text_len, int32_t* answer_len,
                       int batch, int n_kv_heads, int head_dim, void* stream);

/* Rows into pages (cache building for the paged layout, K6): for group g <
 * n_groups and r < count, the row src[g, idx ? idx[g, r] : r] ([G, src_rows,
 * 128] bf16) goes to page table[g, first_slot + r / 64], row r % 64, of
 * `pool`; the rest of the last page is zero-filled. `table` points at the
 * sequence's [Hkv, max_pages] rows. The gather of build_cache
 * (decode.py:92-107) straight into the serving pool.                      */
int omni_page_write(const void* src, int n_groups, int src_rows, int head_dim, const int32_t* idx, int idx_stride,
                    int count, const int32_t* table, int max_pages, int first_slot, void* pool, void* stream);

/* classify_decode_query (decode.py:124-140) for a batch: q bf16 [B, Hq, d],
 * k_lazy / k_act f64 [B, Hkv, d] -> flags u8 [B, Hq] (float64 two-logit
 * rule, head 0 forced active under preserve_first_head).                   */
int omni_decode_flags(const void* q, const double* k_lazy, const double* k_act, int batch, int n_q_heads,
                      int n_kv_heads, int head_dim, double tau, int preserve_first_head, uint8_t* flags,
                      void* stream);

/* classify_decode_query (decode.py:124-140) on float64 queries, the
 * reference's precision (reference-signature operators): q f64
 * [B, Hq, head_dim]; k_lazy / k_act f64 [B, Hkv, probe_stride] (the probe
 * keys of a cache whose rows are zero-padded to probe_stride columns).     */
int omni_decode_flags_f64(const double* q, const double* k_lazy, const double* k_act, int batch, int n_q_heads,
                          int n_kv_heads, int head_dim, int probe_stride, double tau, int preserve_first_head,
                          uint8_t* flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OMNISPARSE_H */
