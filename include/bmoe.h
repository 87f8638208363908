/*
 * bmoe.h — C-ABI of libbmoe.so, the B200 (sm_100a) BuddyMoE hot path.
 *
 * The reference (arxiv 2511.10054, package `buddysim`, pure Python/numpy)
 * has no FFI: its "operator API" is a set of Python functions. Each entry
 * point below replaces one of them; the reference function it stands in for
 * is cited as file:line relative to the reference's pkg/src/buddysim/.
 * INTEGRATION.md shows the ctypes binding a buddysim maintainer would add.
 *
 * Conventions
 *   - All sizes are int64_t. All pointers are DEVICE pointers unless the
 *     parameter name ends in `_host`.
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as
 *     void*); no call synchronises the device unless documented.
 *   - The caller owns every buffer; kernels never allocate. Handles
 *     (bm_cache) own only what their create call documents.
 *   - Return value: BM_OK or an error code; no exceptions cross the ABI.
 *     bm_last_error() returns the thread-local message of the last failure.
 *     Codes map onto the reference taxonomy (errors.py:9-38):
 *       BM_EINVAL->InputError, BM_ECONFIG->ConfigurationError,
 *       BM_EDEGENERATE->DegeneratePivotError, BM_EINVARIANT->InvariantViolation,
 *       BM_ECUDA->InternalError.
 *   - Plans use kind codes 0 kept / 1 substituted / 2 ondemand_fallback /
 *     3 dropped (substitution.py:25-28).
 *   - Buddy tables are dense: ids[E][K] int32 (-1 padded, stored rank order),
 *     weights[E][K] float64, lens[E] int32 (buddies.py:35-76).
 */
#ifndef BMOE_H
#define BMOE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BM_ABI_VERSION 1

enum { BM_OK = 0, BM_EINVAL = 1, BM_ECONFIG = 2, BM_EDEGENERATE = 3, BM_EINVARIANT = 4, BM_ECUDA = 5 };
enum { BM_KIND_KEPT = 0, BM_KIND_SUBSTITUTED = 1, BM_KIND_ONDEMAND = 2, BM_KIND_DROPPED = 3 };
enum { BM_FALLBACK_PREFETCH = 0, BM_FALLBACK_DROP = 1 };                 /* substitution.py:30-31 */
enum { BM_METHOD_BUDDY = 0, BM_METHOD_ORIGINAL = 1, BM_METHOD_IDENTITY = 2, BM_METHOD_RANDOM = 3 };
enum { BM_ACT_TANH = 0, BM_ACT_SWIGLU = 1 };
enum { BM_POLICY_LRU = 0, BM_POLICY_LFU = 1, BM_POLICY_FREQ_STATIC = 2 };  /* memtier.py:31-34 */
enum { BM_EV_HIT = 0, BM_EV_MISS_ONDEMAND = 1, BM_EV_MISS_SUBSTITUTED = 2, BM_EV_PREFETCH_ISSUE = 3,
       BM_EV_PREFETCH_COMPLETE = 4, BM_EV_EVICT = 5, BM_EV_DROP = 6 };  /* memtier.py:20-26 */

typedef void *bm_stream_t;

int bm_abi_version(void);
const char *bm_last_error(void);
/* Number of SMs of the current device (grid sizing); -1 without a device. */
int bm_device_sm_count(void);

/* ---------------------------------------------------------------- K1 router
 * Fused fp32 gate: z = x Wg^T + b; top-k of z by value desc, expert id asc;
 * p~ = softmax(z/T) restricted to the selected set and renormalised (f64
 * math, stored f32); TAE = -sum p~ ln p~ / ln k clamped to [0,1] (k=1 -> 0);
 * margin = p~[0]-p~[1] (k=1 -> 1); token_allowed = !(TAE <= tau) &&
 * !(gamma >= 0 && margin >= gamma). tau < 0 never forbids; gamma < 0
 * disables the margin check. logits/tae/margin may be NULL.
 * Replaces model.route_batch (model.py:231-280) and gating.tae/margin/
 * token_gate (gating.py:71-108). x[B,d], wg[E,d], bias[E] fp32 row-major.
 * Limits: E <= 256, k <= 32, k <= E. */
int bm_gate_topk(const float *x, const float *wg, const float *bias, int64_t B, int64_t E, int64_t d,
                 int64_t k, double temperature, double tau, double gamma, float *logits, int32_t *topk,
                 float *probs, double *tae, double *margin, uint8_t *token_allowed, bm_stream_t stream);

/* Selection + gates from given float64 logits[B,E] (the "identical logits
 * give identical indices" parity boundary, model.py:259-263). probs64 may be
 * NULL; probs (f32) may be NULL. */
int bm_select_topk_f64(const double *logits, int64_t B, int64_t E, int64_t k, double temperature, double tau,
                       double gamma, int32_t *topk, float *probs, double *probs64, double *tae, double *margin,
                       uint8_t *token_allowed, bm_stream_t stream);

/* ------------------------------------------------------- K2 buddy remap
 * One warp per token; Alg. 1 of the paper as implemented by
 * substitution.substitute_token (substitution.py:146-190) under one
 * residency snapshot, with the batch distribution gate of
 * gating.distribution_gate/evaluate_gates (gating.py:126-165):
 *   delta = #non-resident requested slots / (B*k) (duplicates counted),
 *   batch_allowed = !(delta >= beta); a token may substitute iff
 *   token_allowed[b] && batch_allowed.
 * method BUDDY: slot order; a resident original is kept; else, if allowed and
 *   used < rho (rho < 0 = unlimited), the first of ids[orig][0:min(len,H)]
 *   (Psi-ordered when eta or kappa > 0, substitution.py:107-143) that is
 *   resident and not yet assigned to the token; else fallback kind.
 * method ORIGINAL: substitution.ondemand_plan (substitution.py:217-224).
 * method IDENTITY: substitution.identity_plan (substitution.py:211-214).
 * resident_bitmap: ceil(E/32) words, bit e of word e/32 = resident.
 * logits (for eta/kappa z-scores, :98-104) are float64 when logits_f64 != 0,
 * else float32; may be NULL when eta == kappa == 0. partition_of may be NULL.
 * delta_out / batch_allowed_out: single device scalars (may be NULL).
 * Limits: E <= 256, k <= 32, H <= 256. */
int bm_buddy_remap(const int32_t *topk, const uint8_t *token_allowed, const void *logits, int32_t logits_f64,
                   int64_t B, int64_t k, int64_t E, const uint32_t *resident_bitmap, const int32_t *tbl_ids,
                   const double *tbl_w, const int32_t *tbl_len, int64_t tbl_stride, int64_t H, int64_t rho,
                   int32_t fallback, int32_t method, double beta, double eta, double kappa,
                   int32_t use_local_logit, const int32_t *partition_of, double hop, int32_t *executed,
                   uint8_t *kind, int32_t *used, double *delta_out, uint8_t *batch_allowed_out,
                   bm_stream_t stream);

/* ------------------------------------------------ adaptive distribution-gate beta (host)
 * gating.derive_beta (gating.py:173-186): the largest grid value whose
 * estimated admitted volume nhat * expert_bytes fits the budget, else the
 * current beta. BetaController (gating.py:189-221): per record an EMA of the
 * would-be misses admitted at every candidate (delta < candidate), beta
 * re-derived every `period` records. The engine drives the same state. */
#define BM_BETA_MAX_GRID 64
typedef struct {
    double budget_bytes, expert_bytes, beta, decay;
    int64_t period, steps;
    int32_t n_grid, pad_;
    double grid[BM_BETA_MAX_GRID], ema[BM_BETA_MAX_GRID];
} bm_beta_state;
int bm_derive_beta(double budget_bytes, double expert_bytes, const double *grid_host, const double *nhat_host,
                   int32_t n, double current_beta, double *beta_out);
int bm_beta_init(bm_beta_state *state_host, double budget_bytes, double expert_bytes, double initial_beta,
                 const double *grid_host, int32_t n, double decay, int64_t period);
int bm_beta_record(bm_beta_state *state_host, double delta, int64_t miss_count, double *beta_out);

/* ------------------------------------------------ Random baseline (host)
 * numpy's PCG64 bit generator state (Generator.bit_generator.state: the
 * 128-bit state and increment, has_uint32 / uinteger), so host code can make
 * the same draws as the reference and hand the advanced state back. */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int32_t has_uint32;
    uint32_t uinteger;
} bm_pcg64;
/* substitution.random_plan (substitution.py:227-248) for B tokens in order,
 * sharing one generator (harness.py:358-359): a resident expert is kept; a
 * missing one is replaced by pool[rng.integers(0, pool.size)], pool = the
 * resident experts (ascending) not yet assigned to the token, or falls back to
 * ondemand when the pool is empty. Host memory; mask_host[E] = the snapshot. */
int bm_random_plan(const int32_t *topk_host, int64_t B, int64_t k, const uint8_t *mask_host, int64_t E,
                   bm_pcg64 *rng_host, int32_t *executed_host, uint8_t *kind_host, int32_t *used_host);
/* Generator.integers(0, n) drawn `count` times (n <= 2^32), for tests. */
int bm_pcg64_integers(bm_pcg64 *rng_host, int64_t n, int64_t count, int64_t *out_host);

/* ------------------------------------------ K3 permute / K5 combine
 * bm_permute: stable grouping of the executed (token, slot) pairs by expert
 * (dropped slots excluded, model.py:294-305). Outputs expert_count[E] (real
 * rows), expert_offset[E+1] (segment starts, each segment padded to a
 * multiple of row_align rows; offset[E] = total padded rows), row_token[r]
 * (-1 on padding rows; caller sizes it bmoe_permute_rows_max()), slot_row[B*k]
 * (-1 for dropped). Single CTA; deterministic. */
int64_t bm_permute_rows_max(int64_t B, int64_t k, int64_t E, int64_t row_align);
int bm_permute(const int32_t *executed, const uint8_t *kind, int64_t B, int64_t k, int64_t E, int64_t row_align,
               int32_t *expert_count, int32_t *expert_offset, int32_t *row_token, int32_t *slot_row,
               bm_stream_t stream);
/* The same permute with a caller-owned chunk scratch of
 * bm_permute_scratch_elems(B, k, E) int32: plans of 4+ chunks of 1024 slots
 * (prefill) then run as three multi-CTA kernels (chunk histograms, chunk
 * bases + offsets, scatter) with bitwise the same rows; without it (or below
 * 4 chunks) one CTA walks the chunks. */
int bm_permute_scratch_elems(int64_t B, int64_t k, int64_t E);
int bm_permute_ws(const int32_t *executed, const uint8_t *kind, int64_t B, int64_t k, int64_t E, int64_t row_align,
                  int32_t *expert_count, int32_t *expert_offset, int32_t *row_token, int32_t *slot_row,
                  int32_t *chunk_scratch, int64_t scratch_elems, bm_stream_t stream);

/* Extend a plan [B][k] with S always-executed shared experts E..E+S-1 (kind
 * kept, weight 1): outputs [B][k+S] (DeepSeek-V2-style shared experts). */
int bm_append_shared(const int32_t *executed, const uint8_t *kind, const float *probs, int64_t B, int64_t k,
                     int64_t E, int64_t S, int32_t *executed_ext, uint8_t *kind_ext, float *probs_ext,
                     bm_stream_t stream);

/* count_a[e] = mask[e] ? 0 : count[e], count_b[e] = mask[e] ? count[e] : 0 —
 * splits one grouped FFN into experts already in HBM (run while the
 * others are still being fetched) and the fetched ones. */
int bm_split_counts(const int32_t *expert_count, const int32_t *mask, int64_t E, int32_t *count_a, int32_t *count_b,
                    bm_stream_t stream);

/* Gather token rows into the permuted activation buffer (128-bit loads).
 * layout 0: plain row-major fp32 x_perm[r_max][d].
 * layout 1: bf16 "UMMA K-major SW128" planes: x_perm[d/64][r_max][64] with
 *           the 16-byte chunk j of row r stored at chunk (j ^ (r & 7)) —
 *           the exact shared-memory image the tcgen05 GEMM consumes.
 * Padding rows are zero-filled. */
int bm_gather_rows(const float *x, int64_t B, int64_t d, const int32_t *row_token, const int32_t *expert_offset,
                   int64_t E, int64_t r_max, int32_t layout, void *x_perm, bm_stream_t stream);

/* y[b] = sum_s p~[b,s] * [kind != dropped] * y_perm[slot_row[b,s]]  (model.py:334-340,
 * original weights, no renormalisation of dropped mass); then, if h_in is
 * not NULL, out = layer_update(h_in, y) = (h + scale*y)/max(rms, 1e-12)
 * (model.py:343-347), else out = y. Fixed slot order: deterministic. */
int bm_combine(const float *y_perm, const int32_t *slot_row, const float *probs, const uint8_t *kind, int64_t B,
               int64_t k, int64_t d, const float *h_in, float residual_scale, float *out, bm_stream_t stream);
/* The same K3 gather / K5 combine + layer_update in float64 (the reference's
 * precision; model.forward_batch / layer_update of the Python API). */
int bm_gather_rows_f64(const double *x, int64_t B, int64_t d, const int32_t *row_token, const int32_t *expert_offset,
                       int64_t E, int64_t r_max, double *x_perm, bm_stream_t stream);
int bm_combine_f64(const double *y_perm, const int32_t *slot_row, const double *probs, const uint8_t *kind, int64_t B,
                   int64_t k, int64_t d, const double *h_in, double residual_scale, double *out, bm_stream_t stream);

/* ------------------------------------------------- K4 grouped expert FFN
 * Expert weights live in an "arena" of equally sized buffers; buffer b holds
 *   SWIGLU: [W1 (f x d) | W3 (f x d) | W2 (d x f)]   y = (silu(x W1^T) * (x W3^T)) W2^T
 *   TANH:   [Win^T (f x d) | Wout^T (d x f)]         y = tanh(x Win) Wout (model.py:85-99)
 * row-major; buf_of_expert[E] (device) maps an expert id to its buffer.
 *
 * fp32 parity mode (SIMT FFMA, fp32 weights and activations): x_perm is
 * layout 0 [r_max][d]; h_ws is fp32 [r_max][f]; y_perm fp32 [r_max][d]. */
int bm_expert_ffn_f32(const float *x_perm, const int32_t *expert_count, const int32_t *expert_offset, int64_t E,
                      int64_t d, int64_t f, int32_t act, const float *w_arena, int64_t buf_elems,
                      const int32_t *buf_of_expert, int64_t r_max, float *h_ws, float *y_perm,
                      bm_stream_t stream);
/* float64 SIMT tiles of the same grouped FFN (reference precision). */
int bm_expert_ffn_f64(const double *x_perm, const int32_t *expert_count, const int32_t *expert_offset, int64_t E,
                      int64_t d, int64_t f, int32_t act, const double *w_arena, int64_t buf_elems,
                      const int32_t *buf_of_expert, int64_t r_max, double *h_ws, double *y_perm, bm_stream_t stream);

/* bf16 tensor-core mode: persistent stream-K tcgen05/TMEM/TMA GEMMs with
 * weights as the M=128 operand ("swap-AB": decode token counts are the N
 * dimension), fused SwiGLU/tanh, deterministic (split tiles are summed in
 * fixed CTA order, never with float atomics). x_perm is layout 1 (bf16 SW128 planes over d). Workspace from
 * bm_expert_ffn_bf16_workspace(): the persistent state of the decode kernel
 * (grid-barrier and launch counts, per-expert H readiness, split-tile
 * arrival counters; at offsets that do not depend on n_tile, so a workspace
 * sized for one n_tile serves every smaller one), the fp32 partial tiles and
 * the SW128 bf16 intermediate H. It must be ZEROED ONCE when allocated, and
 * serves one stream at a time (calls on it must be stream-ordered).
 * y_perm fp32 [r_max][d]. Decode-width tiles (n_tile <= 64) run as ONE
 * cooperative launch (GEMM1 -> activation -> GEMM2, split tiles reduced in
 * kernel, each expert's GEMM2 waiting only for its own H); wider tiles run
 * data-parallel GEMM kernels.
 * Requires d % 128 == 0, f % 128 == 0. n_tile (16..256, multiple of 16)
 * caps the per-tile token count; larger expert segments are chunked. */
/* bf16 expert buffers use the HBM-native "UMMA-tiled" layout: each weight
 * matrix W[M][K] is stored as 16 KB blocks (128 rows x 64 columns, rows in
 * the 128-byte-swizzled K-major shared-memory image), ordered
 * [m-tile][k-block][matrix], with W1/W3 interleaved per block for SwiGLU:
 *   SWIGLU buffer: [W1|W3 interleaved blocks (2*f*d) | W2 blocks (d*f)]
 *   TANH buffer:   [Win^T blocks (f*d) | Wout^T blocks (d*f)]
 * so one k-step of every matrix is one contiguous bulk copy. bm_pack_expert_bf16
 * converts row-major matrices (w1,w3: [f][d], w2: [d][f]; TANH: w1 = Win^T,
 * w2 = Wout^T, w3 = NULL) into one buffer. */
int bm_pack_expert_bf16(const void *w1, const void *w3, const void *w2, int64_t d, int64_t f, int32_t act, void *dst,
                        bm_stream_t stream);
int64_t bm_expert_ffn_bf16_workspace(int64_t E, int64_t d, int64_t f, int64_t r_max, int64_t n_tile);
int bm_expert_ffn_bf16(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset, int64_t E,
                       int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                       const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                       int64_t workspace_bytes, float *y_perm, bm_stream_t stream);

/* bm_expert_ffn_bf16 followed by bm_combine(y_perm, slot_row, probs, kind, B,
 * k, d, h, residual_scale, h): the gate-weighted combine + layer_update of
 * forward_batch / layer_update (model.py:334-347) in place on h [B][d] fp32.
 * At decode widths (n_tile <= 64) both run in ONE launch (the combine after a
 * second grid barrier of the fused FFN), bit-identical to the two calls. */
int bm_expert_ffn_bf16_combine(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset,
                               int64_t E, int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                               const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                               int64_t workspace_bytes, float *y_perm, const int32_t *slot_row, const float *probs,
                               const uint8_t *kind, int64_t B, int64_t k, float *h, float residual_scale,
                               bm_stream_t stream);
/* Diagnostics: with BMOE_FFN_TRACE=1 in the environment the fused decode FFN
 * records 12 globaltimer stamps (ns) per CTA of its last call (entry, setup,
 * GEMM1 loads issued, GEMM1 MMAs committed, GEMM1 epilogue done, H ready /
 * barrier seen, GEMM2 epilogue done, exit, last GEMM1 accumulator ready, last
 * split-tile arrival seen, first GEMM2 stage landed, GEMM2 MMAs committed);
 * copies up to cap of them, returns the count. */
int64_t bm_ffn_trace_read(uint64_t *out_host, int64_t cap);
/* Kernel timing for the bench's roofline: after bm_set_kernel_timing(1)
 * every bm_expert_ffn_bf16 call records CUDA events on its stream around its
 * two GEMM kernels; bm_kernel_times() waits for them and writes 2 floats per
 * call (GEMM1 ms, GEMM2 ms; a fused decode call is one kernel and reports
 * (kernel ms, 0)), returning the count written (-1 on error).
 * bm_set_kernel_timing() clears the record. */
int bm_set_kernel_timing(int32_t enable);
int bm_kernel_timing_enabled(void);
int64_t bm_kernel_times(float *out_host, int64_t cap);
/* One float per timed call: the fused decode kernel's on-device span in ms
 * (first CTA's entry to last CTA's exit, globaltimer), 0 for calls without
 * one; a cross-check of the events, which also see the launch. */
int64_t bm_kernel_spans(float *out_host, int64_t cap);

/* ------------------------------------- K6/K7 co-activation and buddy ranking
 * bm_coact_count: topk[N][k] int32 accumulated into counts[E] and the
 * symmetric pair matrix pairs[E][E] as uint64 (binary mode: each present pair
 * adds 1, profiler.py:86-92). Rows with an id outside [0, E) or a repeated id
 * are rejected like observe() rejects them (profiler.py:76-80): they are not
 * counted and *invalid_rows (device int32, accumulated) is incremented, so
 * the caller raises InputError after reading it back.
 * For E <= 128, k <= 16 (default BMOE_COACT_TC=2) the count is X^T X on the
 * FP4 tensor cores (tcgen05.mma kind::mxf4 over e2m1 one-hot tiles, exact f32
 * accumulation per CTA); otherwise (or BMOE_COACT_TC=0) shared-memory-
 * privatised per-CTA counters, flushed with 64-bit adds, with the diagonal
 * derived as rowsum/(k-1) for k >= 2 (exact for distinct ids). Every path
 * gives the same counts bit for bit.
 * Warm-up down-weighting is applied by the caller by counting the warm-up
 * token range separately (the weights are exact dyadic scalars).
 * Accumulates (does not clear). Limits: E <= 256, k <= 32. */
int bm_coact_count(const int32_t *topk, int64_t N, int64_t k, int64_t E, unsigned long long *counts,
                   unsigned long long *pairs, int32_t *invalid_rows, bm_stream_t stream);
/* Weighted mass (profiler.py:93-95): pw[i][j] += w * min(p~_a, p~_b), f64
 * atomics (order-dependent: tolerance-level parity only). */
int bm_coact_weighted(const int32_t *topk, const float *probs, int64_t N, int64_t k, int64_t E, double w,
                      double *pair_weights, bm_stream_t stream);
/* out[i] = w_warm * warm[i] + main[i] as float64 (exact for counts < 2^53). */
int bm_counts_to_f64(const unsigned long long *warm, const unsigned long long *main_, int64_t n, double w_warm,
                     double *out, bm_stream_t stream);
/* bm_buddy_rank: per pivot (one warp), bit-exact with buddies.build_table
 * (buddies.py:79-129) over profiler.conditional_row (profiler.py:98-119):
 * row = M[p] + eps, row[p] = 0, total = numpy pairwise sum, q = row/total,
 * order = sort by (-q, id), t = first r with sequential cumsum >= alpha-1e-9
 * (else nnz), len = min(t, nnz, k_max); total <= 0 -> empty list.
 * Writes ids[E][k_max] (-1 padded), weights[E][k_max], lens[E]. E <= 1024. */
int bm_buddy_rank(const double *pair_matrix, int64_t E, double eps, double alpha, int64_t k_max, int32_t *ids,
                  double *weights, int32_t *lens, bm_stream_t stream);
/* profiler.conditional_row for every pivot (profiler.py:98-119): q_out[E][E],
 * degenerate_out[E] = 1 where the row has no mass (caller raises). */
int bm_conditional_rows(const double *pair_matrix, int64_t E, double eps, double *q_out, uint8_t *degenerate_out,
                        bm_stream_t stream);
/* buddies.cft_prefix (buddies.py:79-95) on R given rows q[R][E]: t_out[R] =
 * min(t, nnz), order_out[R][E] = stable descending order (-1 past t),
 * degenerate_out[R] = 1 where the row sums to <= 0. */
int bm_cft_prefix(const double *q_rows, int64_t R, int64_t E, double alpha, int32_t *t_out, int32_t *order_out,
                  uint8_t *degenerate_out, bm_stream_t stream);
/* gating.tae / margin / token_gate from given renormalised probabilities
 * p[B][k] f64 (gating.py:71-108). */
int bm_gate_from_probs(const double *probs, int64_t B, int64_t k, double tau, double gamma, double *tae,
                       double *margin, uint8_t *token_allowed, bm_stream_t stream);
/* gating.distribution_gate (gating.py:126-145): delta over n requested ids
 * (duplicates counted) against the residency bitmap; allowed = !(delta >= beta). */
int bm_distribution_gate(const int32_t *requested, int64_t n, const uint32_t *resident_bitmap, double beta,
                         double *delta_out, uint8_t *allowed_out, bm_stream_t stream);

/* ----------------------------------------------- expert cache control plane
 * Exact replica of memtier.ResidencyState/access/prefetch/settle
 * (memtier.py:96-300) for all layers, one shared transfer channel and
 * simulated clock (memtier.py:72-93), plus the next-layer predictor
 * (harness.py:209-218). Host-only C++; decisions are bit-exact with the
 * reference (same f64 clock arithmetic). */
typedef struct bm_cache bm_cache;
typedef struct {
    double time_ms;
    int32_t kind, layer, token, expert;
    int64_t bytes;
    double stall_ms;
} bm_event;

int bm_cache_create(int32_t num_layers, int32_t num_experts, int32_t capacity, int32_t policy,
                    const int32_t *initial_host /* [L][capacity], -1 padded, ascending */,
                    const double *static_freq_host /* [L][E] or NULL */, double expert_load_ms, double hit_ms,
                    double prefetch_ms, int64_t expert_bytes, bm_cache **out);
void bm_cache_destroy(bm_cache *c);
/* mode 0 ondemand / 1 substituted_away (memtier.py:217-254). */
int bm_cache_access(bm_cache *c, int32_t layer, int32_t expert, int32_t mode, int32_t token, bm_event *ev_out_host);
/* The plan replay of harness.py:363-378 for one batch-layer: dropped -> drop
 * event; substituted -> access(orig, substituted_away) then access(executed);
 * else access(executed). Returns through out_host[4]: executed slots,
 * ondemand misses, substitutions, read bytes. */
int bm_cache_apply_plan(bm_cache *c, int32_t layer, int64_t B, int64_t k, const int32_t *tokens_host,
                        const int32_t *topk_host, const int32_t *executed_host, const uint8_t *kind_host,
                        int64_t *out_host);
int bm_cache_prefetch(bm_cache *c, int32_t layer, const int32_t *experts_host, int64_t n);
int bm_cache_settle(bm_cache *c, int32_t layer);
int bm_cache_advance(bm_cache *c, double ms);
int bm_cache_now(const bm_cache *c, double *now_host);
int bm_cache_snapshot(const bm_cache *c, int32_t layer, uint8_t *mask_host, uint32_t *bitmap_host);
/* Top-m of counts[E] (count desc, id asc), m = capacity - #nonzero. */
int bm_cache_predict(const bm_cache *c, int32_t layer, const int32_t *counts_host, int32_t *out_host,
                     int64_t *n_out_host);
int64_t bm_cache_num_events(const bm_cache *c);
int bm_cache_events(const bm_cache *c, int64_t start, int64_t n, bm_event *out_host);
void bm_cache_clear_events(bm_cache *c);
/* Per-layer state for inspection: last_use[E] int64, freq[E] f64, pending
 * count, waste evictions, unused-prefetch residents. */
int bm_cache_layer_state(const bm_cache *c, int32_t layer, int64_t *last_use_host, double *freq_host,
                         int64_t *scalars_host /* [tick, n_pending, waste, unused_resident] */);
int bm_cache_pending(const bm_cache *c, int32_t layer, double *done_host, int32_t *expert_host, int64_t cap);
/* Clock / cost model accessors (SimClock + PcieChannel state, CostModel),
 * so a caller that owns the clock (memtier's free functions take it as an
 * argument) can drive the replica. */
int bm_cache_set_clock(bm_cache *c, double now, double free_at);
int bm_cache_get_clock(const bm_cache *c, double *now_host, double *free_at_host);
int bm_cache_set_costs(bm_cache *c, double expert_load_ms, double hit_ms, double prefetch_ms, int64_t expert_bytes);
/* ResidencyState.insert (memtier.py:172-195); *victim_host = evicted id or -1. */
int bm_cache_insert(bm_cache *c, int32_t layer, int32_t expert, int32_t via_prefetch, int32_t *victim_host);

/* ------------------------------------------------ offloaded decode engine
 * The run_simulation inner loop (harness.py:315-393) over real memory: the
 * control plane above decides hits/misses/evictions/prefetches exactly as
 * the reference; the data plane keeps every layer's resident experts in a
 * pool of fixed HBM buffers (capacity per layer + `staging` transient
 * buffers), fetches misses from a pinned host mirror with cudaMemcpyAsync on
 * copy streams, and orders buffer reuse with CUDA events. Per layer-step:
 * prefetch(l+1) -> settle(l) -> K1 gate -> K2 remap on the residency
 * snapshot -> plan readback -> control-plane replay -> H2D fetch of
 * executed-but-absent experts -> K3 permute -> K4 grouped FFN -> K5 combine
 * + layer_update (in place on h). */
typedef struct bm_engine bm_engine;
typedef struct {
    int32_t num_layers, num_experts, top_k, d, f, act;
    int32_t max_batch, capacity, staging; /* staging <= 0: automatic */
    int32_t method, policy, search_rank_h, fallback, prefetch_enabled, n_tile;
    int32_t fp32_weights; /* 1: fp32 arena + SIMT FFN (parity), 0: bf16 + tcgen05 */
    int64_t rho;          /* < 0 unlimited */
    double beta, temperature, gamma; /* gamma < 0: margin gate off */
    double load_ms, hit_ms, compute_ms, prefetch_ms; /* control-plane cost model (memtier.py:39-58) */
    int64_t expert_bytes;                            /* reported per miss (CostModel.expert_bytes) */
    int32_t num_shared; /* always-resident shared experts per layer (DeepSeek-V2-style), outside the budget:
                           host_mirror[l] then holds num_experts + num_shared buffers, the shared ones are
                           uploaded once and added to every token with weight 1 */
    int32_t fetch_codec; /* 0: host_mirror[l] = raw buffers back to back; 1 (bf16 only): host_mirror[l] is an
                            exponent-coded layer image (bm_xfer_layer_header + one blob per expert), fetched
                            piece by piece through a staging ring and rebuilt in HBM by bm_xfer_decode_piece */
    double pcie_budget_bytes; /* >= 0: adaptive distribution-gate beta (gating.BetaController, gating.py:189-221,
                                 gate.pcie_budget_bytes config.py:94) starting at `beta`; < 0: fixed beta */
    bm_pcg64 rng; /* method RANDOM: the generator of harness.py:299-300 (SeedSequence([run.seed, 31])) */
    int32_t beta_wire_bytes; /* adaptive beta's bytes per admitted miss: 0 = expert_bytes (the reference's
                                cost model, gating.py:189-221), 1 = the measured mean of the bytes a
                                physical fetch moved over PCIe so far (coded size with fetch_codec) */
} bm_engine_config;

typedef struct {
    int64_t tokens, executed_slots, ondemand_misses, substitutions, drops;
    int64_t physical_fetches, prefetch_copies, h2d_bytes, gate_forbidden, batch_bypassed;
    int64_t ffn_calls, ffn_experts, ffn_rows; /* grouped-FFN launches, sum of distinct executed experts / rows */
    double sim_now_ms;   /* control-plane clock */
    double stall_ms;     /* measured: compute stream waiting on expert fetches (CUDA events) */
    double copy_ms;      /* measured: copy-stream time spent in expert H2D copies (CUDA events; only while
                            bm_engine_set_copy_timing is on) */
    int64_t kernel_launches; /* libbmoe kernels launched (graph nodes included) */
    int64_t wire_bytes;      /* bytes actually moved host -> device for expert fetches (coded or raw) */
    double beta;             /* the distribution-gate beta in force (adaptive when pcie_budget_bytes >= 0) */
    int64_t inflight_releases; /* buffers released while their speculative fetch was still in flight */
} bm_engine_stats;

/* host_mirror[l]: pinned host memory, num_experts buffers of the arena
 * layout (bf16 or fp32 per fp32_weights). gate_w [L][E][d], gate_b [L][E]
 * fp32 device. Table (method BUDDY): tbl_ids [L][E][K] int32, tbl_len [L][E]
 * device. tau_host [L] (token gate thresholds; < 0 never forbids).
 * initial_host [L][capacity] residents (-1 padded); static_freq_host [L][E]
 * for freq_static (else NULL). */
int bm_engine_create(const bm_engine_config *cfg, const void *const *host_mirror, const float *gate_w,
                     const float *gate_b, const int32_t *tbl_ids, const int32_t *tbl_len, int32_t tbl_k,
                     const double *tau_host, const int32_t *initial_host, const double *static_freq_host,
                     bm_engine **out);
void bm_engine_destroy(bm_engine *e);
/* One decode step over all layers, h [B][d] fp32 device, updated in place.
 * tokens_host[B]: global token ids (events). Enqueues on `stream`; returns
 * after the last layer's kernels are enqueued. */
int bm_engine_step(bm_engine *e, float *h, int64_t B, const int32_t *tokens_host, bm_stream_t stream);
/* Accumulated stats (synchronises the engine's events); reset clears them. */
int bm_engine_stats_get(bm_engine *e, bm_engine_stats *out_host, int32_t reset);
bm_cache *bm_engine_cache(bm_engine *e);
/* Optional per-layer-step trace for parity checks: layer, batch size, the
 * residency bitmap the remap saw, batch gate, and per token/slot topk,
 * token gate, executed id and kind (all host memory; set_trace clears). */
int bm_engine_set_trace(bm_engine *e, int32_t enable);
/* Bracket every expert fetch's copies with timing events (stats.copy_ms, the
 * PCIe roofline). Off by default: a timing event on the copy stream costs the
 * copy engine ~6 us per fetch (measured), 5% of a 6.5 MB Qwen3 expert copy. */
int bm_engine_set_copy_timing(bm_engine *e, int32_t enable);
int bm_engine_trace_size(const bm_engine *e, int64_t *records_host, int64_t *tokens_host);
int bm_engine_trace_get(const bm_engine *e, int32_t *layer_host, int32_t *B_host, uint32_t *bitmaps_host,
                        uint8_t *batch_ok_host, int32_t *topk_host, uint8_t *allowed_host, int32_t *executed_host,
                        uint8_t *kind_host);
/* Gate-record fields of the trace (harness.py:345-350): per token f64 TAE and
 * margin (K1), per record the distribution-gate delta (K2). */
int bm_engine_trace_gates(const bm_engine *e, double *tae_host, double *margin_host, double *delta_host);
/* Psi ordering of the buddy candidates inside the engine's remap
 * (substitution.py:107-143; sub.eta / sub.kappa / sub.use_local_logit,
 * topology.partitions / topology.hop): tbl_w [L][E][K] f64 device table
 * weights, partition_of [E] int32 device (NULL: no topology). The z-scores
 * use K1's fp32 logits. eta = kappa = 0 restores the stored order. */
int bm_engine_set_psi(bm_engine *e, const double *tbl_w, double eta, double kappa, int32_t use_local_logit,
                      const int32_t *partition_of, double hop);
/* Bytes of device memory held by the engine (arena + workspaces). */
int64_t bm_engine_device_bytes(const bm_engine *e);

/* ------------------------------------------------ synthetic weights (bench inputs)
 * out[i] = lut[(mix64(base + i/4) >> 16*(i%4)) & 0xFFFF], mix64 = the splitmix64
 * finaliser (z += 0x9E3779B97F4A7C15; two xor-shift-multiply rounds). lut: 65,536
 * bf16 values in device memory (16-byte aligned), out: n bf16. Integer-only, so
 * the numpy twin (synth.py) reproduces the bits on the host. */
int bm_synth_bf16(const uint16_t *lut, uint64_t base, int64_t n, uint16_t *out, bm_stream_t stream);
/* Clustered experts (model.py:161-171 recipe): out[i] = bf16_rn(b + spread * e) in
 * fp32 (rounded per operation), b = value i of the cluster's base matrix
 * (key base_key), e = value i of the expert's delta matrix (key delta_key). */
int bm_synth_mix_bf16(const uint16_t *lut, uint64_t base_key, uint64_t delta_key, float spread, int64_t n,
                      uint16_t *out, bm_stream_t stream);

/* ------------------------------------------------ fetch codec (expert transfer)
 * Lossless exponent coding of bf16 expert buffers for the H2D fetch (no
 * reference counterpart: the reference's transfer is an analytic cost,
 * memtier.py:41-58; this only changes how many bytes cross PCIe, never the
 * bytes that land in HBM). A value keeps its sign+mantissa byte; its exponent
 * is coded. Piece format v3 ("BXP3", the default): one canonical Huffman code
 * of the exponent per piece (<= 12 bits per code), 32 lane streams per
 * 8192-value chunk, ~10.7 bits per value for N(0, s) weights (xfer_v3.cuh
 * documents the layout). Format v2 ("BXP2", BMOE_XFER_FORMAT=2; the layout
 * struct below): a 2-bit code for the chunk's (2048 values) three most
 * frequent exponents, or an escape followed by a 3-bit code for the next seven
 * (code 7: the exponent byte in the piece's raw list), ~10.9 bits per value.
 * The decoders dispatch on the piece magic. Blobs are split into
 * self-contained pieces of BM_XFER_PIECE_VALUES values (the fetch pipeline's
 * unit). */
#define BM_XFER_PIECE_VALUES (32 * 1024 * 1024)
typedef struct {
    uint32_t magic;        /* "BXC1" */
    uint32_t n_pieces;
    uint64_t n_values;
    uint32_t piece_values; /* BM_XFER_PIECE_VALUES */
    uint32_t reserved;
    uint64_t piece_off[1]; /* [n_pieces + 1] byte offsets from the blob start; the last = blob bytes */
} bm_xfer_blob_header;
typedef struct {
    uint32_t magic; /* "BXP2" (v3 pieces: "BXP3", n_chunks of 8192 values at the same offset,
                       bytes at the same offset; the rest per xfer_v3.cuh) */
    uint32_t n_chunks, n_raw;
    uint32_t off_planes, off_meta, off_l2, off_raw, bytes; /* from the piece start; low bytes at 32 */
} bm_xfer_piece_header;
typedef struct {
    uint32_t magic; /* "BXL1" */
    uint32_t count; /* experts in the layer image (num_experts + num_shared) */
    uint64_t raw_bytes;    /* decoded bytes per expert */
    uint64_t blob_off[1];  /* [count + 1], 256-byte aligned offsets from the image start */
} bm_xfer_layer_header;
/* Upper bound of a blob for n_values (a positive multiple of 2048), -1 otherwise. */
int64_t bm_xfer_blob_bound(int64_t n_values);
/* Encode n_values bf16 at src (device) into blob (device, 256-byte aligned,
 * blob_cap bytes). Synchronises `stream`; *blob_bytes_host = blob size. */
int bm_xfer_encode(const uint16_t *src, int64_t n_values, uint8_t *blob, int64_t blob_cap, int64_t *blob_bytes_host,
                   bm_stream_t stream);
/* Decode a whole blob (device) into dst [n_values] bf16 (device). */
int bm_xfer_decode(const uint8_t *blob, uint16_t *dst, int64_t n_values, bm_stream_t stream);
/* Decode one piece (device copy, 256-byte aligned) into dst (the piece's
 * first value); n_chunks = the piece header's (sizes the grid only). */
int bm_xfer_decode_piece(const uint8_t *piece, uint16_t *dst, int64_t n_chunks, bm_stream_t stream);
/* The same on at most max_ctas CTAs (0: the full grid). The engine decodes the
 * pieces that are not on its critical path (all but an expert's last) on a
 * narrow grid, so they stream alongside the copies instead of taking HBM and
 * issue slots from the FFN running at the same time. */
int bm_xfer_decode_piece_ctas(const uint8_t *piece, uint16_t *dst, int64_t n_chunks, int32_t max_ctas,
                              bm_stream_t stream);

/* Pinned host allocation of exact size (cudaHostAlloc, portable). */
int bm_host_alloc(int64_t bytes, void **out);
int bm_host_free(void *p);
/* Page-lock an existing host mapping for DMA (cudaHostRegister, portable;
 * read_only != 0 adds cudaHostRegisterReadOnly). Replicas on one node share
 * one expert mirror this way: a shared-memory file mapped by every rank. */
int bm_host_register(void *p, int64_t bytes, int32_t read_only);
int bm_host_unregister(void *p);
int bm_memcpy(void *dst, const void *src, int64_t bytes, bm_stream_t stream); /* cudaMemcpyAsync default kind */

#ifdef __cplusplus
}
#endif
#endif /* BMOE_H */
