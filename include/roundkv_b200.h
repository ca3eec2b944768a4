/*
 * roundkv_b200.h — C ABI of librk.so, the B200-native (sm_100a) hot path of
 * Round Attention (arXiv 2502.15294).
 *
 * Each entry point replaces one interface of the reference package
 * (/root/reference/pkg/src/roundkv/...), cited beside it.  Conventions follow
 * the reference's only FFI (the Cython kernel, _attn_ext.pyx:84-116):
 *   - the caller allocates every output and scratch buffer (device memory,
 *     torch-allocated on the Python side); the library never allocates;
 *   - all pointers are device pointers unless the name says `host`;
 *   - every call is asynchronous on `stream` (a cudaStream_t);
 *   - the return value is a status: RK_OK, or a negative RK_ERR_* code whose
 *     message is available from rk_last_error() (thread-local).  The Python
 *     layer maps the codes onto roundkv.errors (errors.py:28-41):
 *       RK_ERR_DOMAIN -> DomainError, RK_ERR_CAPACITY -> CapacityError,
 *       RK_ERR_CONSISTENCY -> ConsistencyError, RK_ERR_INVARIANT -> InvariantError.
 *     Row-level invariants found on the device (a query row with no visible
 *     key, _attn_ext.pyx:49-50,110-111) are reported through a device int32
 *     `bad_row` (INT32_MAX = none) that the caller reads back.
 *
 * Layouts (row-major, element = float32 or bf16 per `kv_dtype`):
 *   q            [rows][hq][d]            float32
 *   KV cache     [keys][hkv][d]           token-major, as the reference's
 *                                          per-layer payload (store.py:225-242)
 *   out          [rows][hq][d]            float32 (== reference (n, H*d))
 * GQA: query head h reads key head h / (hq/hkv) (HF repeat_kv convention).
 */
#ifndef ROUNDKV_B200_H
#define ROUNDKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* rk_stream_t; /* identical to cudaStream_t */

#define RK_ABI_VERSION 1

#define RK_F32 0
#define RK_BF16 1

#define RK_OK 0
#define RK_ERR_DOMAIN -1
#define RK_ERR_CAPACITY -2
#define RK_ERR_CONSISTENCY -3
#define RK_ERR_INVARIANT -4
#define RK_ERR_CUDA -5
#define RK_ERR_UNSUPPORTED -6

/* selection kinds (selection.py:20) */
#define RK_SEL_FIXED 0
#define RK_SEL_TOP_PERCENT 1
#define RK_SEL_ADAPTIVE 2
#define RK_SEL_ALL 3

int rk_abi_version(void);
const char* rk_last_error(void);

/* ------------------------------------------------------------------------
 * 1. Kernel contract: attention_forward(q, k, v, q_pos, k_pos, allowed, capture)
 *    Replaces backend.attention_forward (backend.py:46-47) ->
 *    _attn_ext.attention_forward (_attn_ext.pyx:84-116) / _attn_np.py:50-92.
 *    scores (nullable): [n][s] float64, head-summed and row-normalised
 *    (capture=True).  allowed (nullable): [s] uint8.  hq % hkv == 0.
 * ---------------------------------------------------------------------- */
size_t rk_attention_workspace_bytes(int n, int hq, int hkv, int s, int d);
int rk_attention_forward(const float* q, int n, int hq, int d,
                         const void* k, const void* v, int kv_dtype, int s, int hkv,
                         const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed,
                         float* out, double* scores, int32_t* bad_row,
                         void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* ------------------------------------------------------------------------
 * 2. Sparse decode attention over a round-spliced cache (the decode loop,
 *    pipeline.py:298-313 -> engine.forward_range:244-267 with one new row).
 *    Dialogue b's cache starts at k_cache + b*cache_stride elements and holds
 *    seq_len[b] keys (device int32).  If k_new/v_new ([batch][hkv][d]) are
 *    given, the row is appended at index seq_len[b] and attended (seq_len is
 *    NOT advanced; see rk_advance_lengths).  max_seq_len bounds seq_len[b]+1
 *    and sizes the split-K grid.
 *    items (nullable): round-aligned work items [batch][items_stride][3] =
 *    (key_lo, key_hi, bin) with n_items[batch]; with items the per-item
 *    softmax statistics are left in `workspace` for rk_round_scores_finalize
 *    (fused watershed scoring; items_stride <= 512).
 *    advance_len (nullable): advance_len[b] += 1 after the layer completes
 *    (pass it on the last layer that reads a length array).
 *    Successive calls on one stream overlap through programmatic dependent
 *    launch: the next call may prefetch its K/V tiles and read seq_len while
 *    the previous call's merge runs, so a length array must not be advanced
 *    by the call immediately preceding a reader of the same array.
 *    Workspace: rk_decode_workspace_bytes(batch, hq, hkv, d, max_splits)
 *    (max_splits = max(items_stride * 8/hkv, 592)); no zeroing needed.
 * ---------------------------------------------------------------------- */
size_t rk_decode_workspace_bytes(int batch, int hq, int hkv, int d, int max_splits);
int rk_decode_attention(const float* q, int batch, int hq, int d,
                        void* k_cache, void* v_cache, int kv_dtype, int hkv,
                        int64_t cache_stride, const int32_t* seq_len, int max_seq_len,
                        const void* k_new, const void* v_new,
                        const int32_t* items, const int32_t* n_items, int items_stride,
                        float* out, int32_t* advance_len,
                        void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* Row-masked decode for a batch whose rows are not all in the decode loop
 * (cohort serving): rows with row_active[b] == 0 are skipped entirely — no
 * append, no output, no length advance.  Runs the cluster decode (one CTA per
 * (dialogue, kv-head) in several waves beyond one wave of pairs); RK_ERR_DOMAIN
 * for shapes it does not serve. */
int rk_decode_attention_rows(const float* q, int batch, int hq, int d, void* k_cache, void* v_cache,
                             int kv_dtype, int hkv, int64_t cache_stride, const int32_t* seq_len,
                             int max_seq_len, const void* k_new, const void* v_new, const int32_t* row_active,
                             float* out, int32_t* advance_len, rk_stream_t stream);

/* seq_len[i] += delta for i < n (advance one decode step) */
int rk_advance_lengths(int32_t* seq_len, int n, int delta, rk_stream_t stream);

/* Which decode kernel rk_decode_attention runs for this shape (no launch).
 * The cluster decode reads the caches through 2-D TMA tensor maps spanning the
 * batch, so it also needs cache_stride to be a multiple of hkv*d when batch > 1
 * (else the persistent kernel runs); bf16 or fp32 KV; the rest of the contract
 * (append, lengths, PDL ordering, workspace) is the same for every kernel:
 * C > 0  one thread-block cluster of C CTAs per (dialogue, kv-head), split-K
 *        merged in distributed shared memory (small batches: batch*hkv <= SMs,
 *        bf16 or fp32 (128-key / 64-key TMA stages), d 64/128, no item table);
 * 0      persistent split-K over the concatenated key ranges + merge kernel;
 * -1     the generic split kernel (other dtypes / head shapes). */
int rk_decode_plan(int batch, int hq, int hkv, int d, int kv_dtype, int max_seq_len, int64_t cache_stride,
                   int has_items);

/* ------------------------------------------------------------------------
 * 3. Watershed round scoring: the fused equivalent of
 *      capture = attention_forward(q, K_{Lw-1}, ..., capture=True)[1]
 *      raw = aggregate_round_attention(capture, rounds, "question", n,
 *                                      active_rounds, row_offset=q_start)
 *    (pipeline.py:225-245, stats.py:59-94, _attn_ext.pyx:75-76,113-114).
 *    Keys [0, s) of layer Lw-1 are grouped into round-aligned work items
 *    (key_lo, key_hi, bin); bin in [0, n_bins) is a prior round, bin ==
 *    n_bins is the current question (denominator only).  Only the softmax
 *    statistics are produced (no capture matrix).  raw_out has one float64 per
 *    ACTIVE bin, in ascending bin order (active: [n_bins] uint8, nullable).
 * ---------------------------------------------------------------------- */
size_t rk_round_scores_workspace_bytes(int n_q, int hq, int hkv, int n_items, int d, int n_bins);
int rk_round_scores(const float* q, int n_q, int hq, int d,
                    const void* k, int kv_dtype, int s, int hkv,
                    const int64_t* q_pos, const int64_t* k_pos,
                    const int32_t* items, int n_items, int n_bins, const uint8_t* active,
                    double* raw_out, void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* Finalise scores left by rk_decode_attention(items != NULL): one dialogue
 * row per batch entry; raw_out [batch][n_bins] (inactive bins -> 0). */
int rk_round_scores_finalize(int batch, int hq, int hkv, int d, int kv_dtype, int items_stride,
                             const int32_t* items, const int32_t* n_items, int n_bins, const uint8_t* active,
                             double* raw_out, void* workspace, rk_stream_t stream);

/* Eq. 1 on a materialised capture matrix (stats.py:59-94 on the device):
 * raw[a] = sum over rows [row_lo,row_hi) of scores[row][col] for the columns
 * of active round a, given as two half-open spans per round (q_span, a_span). */
int rk_aggregate_rounds(const double* scores, int64_t ld, int row_lo, int row_hi,
                        const int64_t* spans /* [n_active][4] */, int n_active,
                        double* raw_out, rk_stream_t stream);

/* ------------------------------------------------------------------------
 * 4. normalize + select (stats.py:97-115, selection.py:63-126), one block.
 *    masses = raw / sum(raw) with NumPy's pairwise summation order, uniform
 *    when the sum is 0 (degenerate).  Kept positions are ascending indices
 *    into raw.  top_percent keeps the k_top largest masses, ties to the lower
 *    index (stable argsort); k_top is computed by the caller with the
 *    reference expression (selection.py:93-94).  fixed / adaptive fall back to
 *    the first argmax when nothing passes.  status_out: 0 ok, RK_ERR_DOMAIN if
 *    any raw < 0.  Bit-exact against the reference for the same raw.
 * ---------------------------------------------------------------------- */
int rk_select(const double* raw, int n, int normalize, int kind, double v, int k_top, double kappa,
              double* masses_out, int32_t* kept_out, int32_t* n_kept_out,
              int32_t* degenerate_out, int32_t* status_out, rk_stream_t stream);

/* Batched form for B independent dialogues: row b of raw/masses/kept starts
 * at b*ld; n_kept/degenerate/status are [batch]. One block per dialogue. */
int rk_select_batch(const double* raw, int n, int ld, int batch, int normalize, int kind, double v,
                    int k_top, double kappa, double* masses_out, int32_t* kept_out, int32_t* n_kept_out,
                    int32_t* degenerate_out, int32_t* status_out, rk_stream_t stream);

/* Selection over each dialogue's ACTIVE rounds (the inactivity drop policy:
 * selection.py:183-204 ActivityLedger + pipeline.py:238-245 active_rounds).
 * raw [batch][ld] float64 holds the Eq. 1 mass of every one of the n rounds
 * (inactive ones included); active [batch][ld] uint8 (NULL = all active).  Per
 * dialogue the active rounds are taken in ascending order, normalized and
 * selected as rk_select_batch; kept_out receives ROUND IDS (ascending),
 * masses_out the normalized masses at the compacted positions.  top_percent
 * with k_top <= 0 sizes k per dialogue from fraction / min_rounds and the
 * dialogue's active count (selection.py:87-97).  margin_out [batch] (nullable)
 * as rk_selection_margin.  n <= 2048. */
int rk_select_batch_active(const double* raw, int n, int ld, int batch, const uint8_t* active, int normalize,
                           int kind, double v, int k_top, double fraction, int min_rounds, double kappa,
                           double* masses_out, int32_t* kept_out, int32_t* n_kept_out, int32_t* degenerate_out,
                           int32_t* status_out, double* margin_out, rk_stream_t stream);

/* Decision margin of the selection made from `masses` (rows ld apart):
 * top_percent (m_(K) - m_(K+1)) / m_(K) of the K-th / (K+1)-th largest masses;
 * fixed min |m - v| / v; adaptive min |m - cut| / |cut|; all +inf.
 * margin_out [batch] float64.  The fp32-class scorers (rk_round_scores, the
 * fused decode / prefill scoring) reproduce the reference's kept set whenever
 * the margin exceeds twice their relative error; below that the caller
 * re-scores with rk_round_scores_exact (the engines use 1e-5 for multi-row
 * questions; 1-row questions are always scored exactly). */
int rk_selection_margin(const double* masses, int n, int ld, int batch, int kind, double v, int k_top,
                        double kappa, double* margin_out, rk_stream_t stream);

/* ------------------------------------------------------------------------
 * 4b. Exact (fp64) watershed round scoring with the reference kernel's
 *    arithmetic (_attn_ext.pyx:52-76,113-114 + stats.py:59-94): logits are fp64
 *    dot products of exact fp64 products (q fp32 x k bf16/fp32), summed on the
 *    FP64 tensor pipe for bf16 keys with d 64/128 (~1e-16 from the reference's
 *    sequential sum) and sequentially otherwise; softmax statistics per (row,
 *    head, round-aligned item) in fp64, Eq. 1 masses in fp64 — the kept set is
 *    the reference's up to fp64 rounding (~1e-16 relative), and identical rounds
 *    tie exactly (a key's logit never depends on its position).
 *    batch dialogues: q [batch][n_q][hq][d] f32; dialogue b's keys start at
 *    k + b*k_batch_stride elements, [s_b][hkv][d] (s_b = seq_len[b], or s when
 *    seq_len is NULL); q_pos [n_q] int64 (shared), k_pos [s] int64 or NULL
 *    (key j at position j); key j is visible to row i iff k_pos[j] <= q_pos[i].
 *    items [batch][items_stride][3] = (key_lo, key_hi, bin), round-aligned,
 *    sorted by bin, covering every visible key (bin n_bins = the current
 *    question); n_items [batch] device or NULL (= items_stride).
 *    raw_out [batch][n_out]: one float64 per ACTIVE bin (active [n_bins] uint8,
 *    nullable; n_out = number of active bins).  hq/hkv <= 8, d % 8 == 0.
 * ---------------------------------------------------------------------- */
size_t rk_round_scores_exact_workspace_bytes(int batch, int n_q, int hq, int items_stride, int n_bins);
int rk_round_scores_exact(const float* q, int batch, int n_q, int hq, int d,
                          const void* k, int kv_dtype, int hkv, int64_t k_batch_stride,
                          const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                          const int32_t* items, int items_stride, const int32_t* n_items,
                          int n_bins, const uint8_t* active, int n_out, double* raw_out,
                          void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* capture_mode="pre" (engine.py:187-200, Model._capture_pre): the same Eq. 1
 * masses from ONE softmax per query row over the head-summed logits
 * sum_h q_h . k_kv(h) / (Hq * sqrt(d)) (fp64; einsum "nhd,shd->ns"), instead of
 * the head-summed per-head probabilities.  Arguments, workspace and outputs as
 * rk_round_scores_exact (hq*d*8 bytes of shared memory per row, <= 200 KB). */
int rk_round_scores_exact_pre(const float* q, int batch, int n_q, int hq, int d,
                              const void* k, int kv_dtype, int hkv, int64_t k_batch_stride,
                              const int32_t* seq_len, int s, const int64_t* q_pos, const int64_t* k_pos,
                              const int32_t* items, int items_stride, const int32_t* n_items,
                              int n_bins, const uint8_t* active, int n_out, double* raw_out,
                              void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* ------------------------------------------------------------------------
 * 5. Batched host->HBM gather of kept rounds' upper-layer blocks
 *    (store.fetch_upper store.py:254-263 + pipeline._assemble :158-169).
 *    Copy i moves `height[i]` rows of `width[i]` bytes from pinned host
 *    memory (src_host[i], row pitch src_pitch[i]) to device memory
 *    (dst[i], pitch dst_pitch[i]) as DMA on `stream`; one call = one ledger
 *    h2d event.  If done_event (a cudaEvent_t) is given it is recorded after
 *    the last copy.
 * ---------------------------------------------------------------------- */
int rk_h2d_gather(int n, const void* const* src_host, const size_t* src_pitch,
                  void* const* dst, const size_t* dst_pitch,
                  const size_t* width, const size_t* height,
                  rk_stream_t stream, void* done_event);

/* The peer-HBM tier: the same batched gather when the kept
 * rounds' upper blocks live in GPU memory — another GPU's HBM over NVLink
 * (after rk_enable_peer_access) or this GPU's — instead of pinned host memory
 * (cudaMemcpyDefault: unified addressing picks the path). */
int rk_peer_gather(int n, const void* const* src, const size_t* src_pitch,
                   void* const* dst, const size_t* dst_pitch,
                   const size_t* width, const size_t* height,
                   rk_stream_t stream, void* done_event);

/* Enable direct loads / copies from peer_device's memory on the current device
 * (no-op for the current device; RK_ERR_CUDA when the topology forbids it). */
int rk_enable_peer_access(int peer_device);

/* D2H counterpart for the new round's upper block (writeback_upper :265-278). */
int rk_d2h_scatter(int n, const void* const* src, const size_t* src_pitch,
                   void* const* dst_host, const size_t* dst_pitch,
                   const size_t* width, const size_t* height,
                   rk_stream_t stream, void* done_event);

/* ------------------------------------------------------------------------
 * 6. Question prefill attention on the tensor cores (tcgen05), with the
 *    watershed round scoring fused in.  The multi-row form of section 1
 *    (forward_range over the question rows, pipeline.py:225-230 lower layers
 *    over the full history, :292-296 upper layers over kept + current; the
 *    kernel contract _attn_ext.pyx:20-81) for bf16 K/V, head_dim 128 and
 *    n_q * hq/hkv >= 64; rk_attention_forward uses the same kernel for those
 *    shapes.  If raw_out is given, items [n_items][3] = (key_lo, key_hi, bin)
 *    must be round-aligned and cover the keys (as for rk_round_scores) and
 *    raw_out receives the Eq. 1 masses of the active bins
 *    (aggregate_round_attention, stats.py:59-94) from the same pass — no
 *    capture matrix, no second pass over K.  Without raw_out, items may be
 *    NULL (uniform split).  bad_row: INT32_MAX or the first row with no
 *    visible key (-> InvariantError).
 * ---------------------------------------------------------------------- */
/* flags: RK_PREFILL_SINGLE_PASS = the bf16 path (q and softmax P rounded to
 * bf16, one MMA pass each; outputs ~1e-2 relative instead of ~1e-6; not with
 * raw_out).  0 = the default two-pass fp32-class path. */
#define RK_PREFILL_SINGLE_PASS 1
size_t rk_prefill_workspace_bytes(int n_q, int hq, int hkv, int s, int d, int n_items, int n_bins);
int rk_prefill_attention(const float* q, int n_q, int hq, int d,
                         const void* k, const void* v, int kv_dtype, int s, int hkv,
                         const int64_t* q_pos, const int64_t* k_pos, const uint8_t* allowed,
                         const int32_t* items, int n_items, int n_bins, const uint8_t* active,
                         float* out, double* raw_out, int32_t* bad_row,
                         void* workspace, size_t workspace_bytes, int flags, rk_stream_t stream);

/* ------------------------------------------------------------------------
 * 7. The decode step's layer body (engine.py:244-251,267-271 of the reference:
 *    q, k = RoPE(x W_q), RoPE(x W_k); v = x W_v; append; attention;
 *    x += out W_o; logits = x E^T; greedy argmax, pipeline.py:308), GQA
 *    (W_k, W_v: d_model x hkv*d) with bf16 weights and fp32 activations.
 *    Weights are stored once for the tensor cores: rk_pack_weight(W [k][n]
 *    row-major (x @ W), fp32 or bf16) -> 16 KB tiles [n_pad/128][k/64] of
 *    W^T (128 features x 64 k, bf16, each in the 128-byte-swizzled K-major
 *    shared-memory image of a tcgen05 A operand; rk_packed_weight_bytes(k, n),
 *    n padded to 128 with zero rows, k % 64 == 0).  The projections are persistent tcgen05 kernels
 *    (M = 128 features, N = the rows padded to 16/32/64) that split K across
 *    the CTAs; `workspace` (rk_proj_workspace_bytes(m, k, n), ZEROED once at
 *    allocation — the kernels leave their tickets at zero) holds the split-K
 *    partials, added in a fixed order (deterministic).  One workspace per
 *    stream: concurrent launches must not share it.
 *    rk_qkv_rope: x [m][d_model] f32 (m rows: one per dialogue in decode, the
 *    question rows in prefill) times the packed [W_q | W_k | W_v]; RoPE on q
 *    and k at pos [m] (int32) with rope_freq [d/2] (float64, the reference's
 *    theta ** (-2i/d)); q_out [m][hq][d] f32; k/v rows (bf16) at
 *    k_out / v_out + row * kv_row_stride elements.
 *    rk_out_proj: resid [m][d_model] += a [m][k] W_o.
 *    rk_lm_head: logits of x [m][d_model] against the packed embedding
 *    (vocab rows; m <= 64) into workspace, the first argmax per row -> tokens [m]
 *    (and tokens_log[row * log_stride] when given), x_next [m][d_model] =
 *    emb[token] (bf16 table [vocab][d_model]), pos[row] += 1 when given.
 *    rk_embed: x [m][d_model] = emb[tokens[row]].
 *    All launch as programmatic dependents: their weight loads start before
 *    the previous kernel on the stream completes.
 * ---------------------------------------------------------------------- */
size_t rk_packed_weight_bytes(int k, int n);
int rk_pack_weight(const void* w, int w_dtype, int k, int n, void* packed, rk_stream_t stream);
size_t rk_proj_workspace_bytes(int m, int k, int n);
int rk_qkv_rope(const float* x, int m, int d_model, const void* w_qkv_packed, int hq, int hkv, int d,
                const int32_t* pos, const double* rope_freq, float* q_out, void* k_out, void* v_out,
                int64_t kv_row_stride, void* workspace, size_t workspace_bytes, rk_stream_t stream);

/* rk_qkv_rope with the cache's dtype: kv_dtype RK_BF16 (rk_qkv_rope) or RK_F32
 * (the reference's float32 KV, _attn_np.py:26-28); kv_row_stride in elements. */
int rk_qkv_rope_kv(const float* x, int m, int d_model, const void* w_qkv_packed, int hq, int hkv, int d,
                   const int32_t* pos, const double* rope_freq, float* q_out, void* k_out, void* v_out,
                   int kv_dtype, int64_t kv_row_stride, void* workspace, size_t workspace_bytes,
                   rk_stream_t stream);
int rk_out_proj(const float* a, int m, int k, const void* w_o_packed, int d_model, float* resid,
                void* workspace, size_t workspace_bytes, rk_stream_t stream);
size_t rk_lm_head_workspace_bytes(int m, int vocab, int d_model);
int rk_lm_head(const float* x, int m, int d_model, const void* emb_packed, int vocab, const void* emb,
               float* x_next, int32_t* tokens, int32_t* pos, int32_t* tokens_log, int log_stride,
               void* workspace, size_t workspace_bytes, rk_stream_t stream);
int rk_embed(const int32_t* tokens, int m, const void* emb, int d_model, float* x, rk_stream_t stream);
/* Row-masked forms for a decode batch whose rows (dialogues) are not all in the
 * decode loop (cohort serving): rows with row_active[t] == 0 keep their
 * residual (rk_out_proj_rows) / token, position and input row (rk_lm_head_rows).
 * rk_lm_head_rows with log_pos_base >= 0 logs row t's token at
 * tokens_log[t * log_stride + pos[t] - log_pos_base + 1] (rows at different steps). */
int rk_out_proj_rows(const float* a, int m, int k, const void* w_o_packed, int d_model, float* resid,
                     const int32_t* row_active, void* workspace, size_t workspace_bytes, rk_stream_t stream);
int rk_lm_head_rows(const float* x, int m, int d_model, const void* emb_packed, int vocab, const void* emb,
                    float* x_next, int32_t* tokens, int32_t* pos, int32_t* tokens_log, int log_stride,
                    const int32_t* row_active, int log_pos_base, void* workspace, size_t workspace_bytes,
                    rk_stream_t stream);
/* ---- the drop-in model's layer body (engine.Model: the reference's toy
 * transformer, float32 weights [d_model][d_model] row-major, x @ W) ----
 * rk_small_qkv_rope: q, k = RoPE(x W_q), RoPE(x W_k), v = x W_v for n rows
 *   (engine.py:244-251; RoPE with float64 angles / trig, engine.py:175-185),
 *   outputs [n][d_model] float32 (q as [n][heads][d_k]).
 * rk_small_out_proj: x_out = x + a W_o (engine.py:267); x_out may not alias a.
 * rk_small_logits: logits = x E^T ([n][vocab], nullable) and the first maximum
 *   per row (engine.py:270-271, pipeline.py:308 np.argmax). d_model <= 4096. */
int rk_small_qkv_rope(const float* x, int n, int d_model, const float* w_q, const float* w_k, const float* w_v,
                      int heads, const int64_t* pos, const double* rope_freq, float* q_out, float* k_out,
                      float* v_out, rk_stream_t stream);
int rk_small_out_proj(const float* a, int n, int d_model, const float* w_o, const float* x, float* x_out,
                      rk_stream_t stream);
int rk_small_logits(const float* x, int n, int d_model, const float* emb, int vocab, float* logits,
                    int32_t* argmax, rk_stream_t stream);
/* capture_mode="pre" capture matrix (engine.py:187-200): out[i][j] = softmax_j over the
 * visible keys (k_pos[j] <= q_pos[i], allowed[j] when given) of
 * sum_h q[i][h] . k[j][h] / (heads sqrt(d_k)), float64; q [n][heads][d_k], k [s][heads][d_k]
 * float32; a row without a visible key is NaN (as the reference). */
int rk_capture_pre(const float* q, int n, int heads, int d_k, const float* k, int s, const int64_t* q_pos,
                   const int64_t* k_pos, const uint8_t* allowed, double* out, rk_stream_t stream);

/* ---- the whole decode token step in one persistent launch (small batches) ----
 * One answer token of every dialogue through all num_layers layers + the tied
 * logits and first-max argmax (reference engine.py:244-271 forward_range per
 * layer, pipeline.py:298-313 the greedy decode loop body): for each layer
 * x -> RoPE(x W_q), RoPE(x W_k), x W_v (rows appended at lower_len / upper_len),
 * attention over the cached keys + the new one, x += attn W_o; then
 * tokens = argmax(x E^T), x = E[tokens], pos / lower_len / upper_len += 1 and
 * tokens_log[b * log_stride] = token (when tokens_log is given).
 * Layout as the layered entries: lower [batch][watershed][2][lower_seq][hkv][head_dim]
 * and upper [batch][num_layers - watershed][2][upper_seq][hkv][head_dim] bf16;
 * w_qkv / w_o: DEVICE arrays of num_layers rk_pack_weight images (W_q|W_k|W_v,
 * W_o); emb_packed = rk_pack_weight(E^T), emb = E [vocab][d_model] bf16.
 * One CTA per SM for the whole step (producer warp streaming every weight tile
 * and cached K/V box of the step through a shared-memory ring; consumers
 * synchronised by device-scope counters), so nothing else may occupy the GPU's
 * SMs concurrently.  The workspace (rk_decode_step_workspace_bytes) is zeroed
 * once and then reused by every launch (monotonic counters, epoch in word 0).
 * Supported: rk_decode_step_supported() (batch <= 16, group <= 8, head_dim 128,
 * bf16 KV). */
typedef struct rk_decode_step_args {
  int batch, num_layers, watershed, hq, hkv, head_dim, vocab;
  float* x;                        /* [batch][hq * head_dim] residual in; next token's embedding out */
  void* lower;
  int64_t lower_seq;
  void* upper;
  int64_t upper_seq;
  int32_t* lower_len;
  int32_t* upper_len;
  int32_t* pos;
  const double* rope_freq;         /* [head_dim / 2] (engine.py:162-164) */
  const void* const* w_qkv;
  const void* const* w_o;
  const void* emb_packed;
  const void* emb;
  int32_t* tokens;                 /* nullable */
  int32_t* tokens_log;             /* nullable */
  int log_stride;
  void* workspace;
  size_t workspace_bytes;
} rk_decode_step_args;
size_t rk_decode_step_workspace_bytes(int batch, int num_layers, int hq, int hkv, int head_dim, int vocab);
int rk_decode_step_supported(int batch, int hq, int hkv, int head_dim, int kv_dtype);
int rk_decode_step(const rk_decode_step_args* args, rk_stream_t stream);
/* the code a bounded wait left in the workspace before trapping (0 = none) */
int rk_decode_step_watchdog(const void* workspace, unsigned* code_out, rk_stream_t stream);

/* RoPE + cache append for projections computed by a library GEMM (the multi-row
 * question prefill): qkv [m][(hq + 2 hkv) d] f32 -> q_out [m][hq][d]; k / v rows
 * of row r at k_out / v_out + (r / rows_per_group) * kv_group_stride +
 * (r % rows_per_group) * kv_row_stride elements (bf16). */
int rk_rope_rows(const float* qkv, int m, int hq, int hkv, int d, const int32_t* pos, const double* rope_freq,
                 float* q_out, void* k_out, void* v_out, int64_t kv_row_stride, int rows_per_group,
                 int64_t kv_group_stride, rk_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* ROUNDKV_B200_H */
