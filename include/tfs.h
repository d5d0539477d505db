/*
 * tfs.h -- C ABI of libtfs, the B200 (sm_100a) hot path of the large-vocabulary language-model
 * training step of Abadi et al., "TensorFlow: A system for large-scale machine learning"
 * (arXiv 1605.08695): the sharded embedding lookup Part -> Gather -> Stitch (§4.2),
 * the sampled-softmax output layer (§6.4) and the sparse ScatterAdd/SGD
 * update.  "P:n" cites /root/reference/PAPER.md line n; "R-k" cites
 * reading k of DESIGN.md §3 (where the paper is silent or garbled).
 *
 * CONVENTIONS (every entry point)
 *  - Buffers are DEVICE pointers owned by the caller (e.g. torch CUDA tensors), unless a
 *    parameter says "host".  The library never allocates device memory and never synchronises
 *    the stream, except tfs_sampler_init and the stepper / communicator setup calls.  Scratch
 *    comes from a caller-provided workspace `ws` of at least the bytes the matching
 *    *_workspace_bytes() query returns; ws must be 256-byte aligned.  Workspaces of the calls
 *    that sum gradient rows per id (tfs_sort_reduce, tfs_scatter_add_sgd*, tfs_scatter_opt_*,
 *    tfs_route_reduce*) hold arrival counters: zero-fill them once before the first call
 *    (every call leaves them zero).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Calls are
 *    stream-ordered and asynchronous.
 *  - The returned tfs_status reports ARGUMENT errors only, detected on the host before any
 *    launch (nothing is launched then).  DATA errors (an id outside its table, a bad stitch
 *    permutation, an exhausted sampler) are written to the caller's device-resident
 *    tfs_device_error: `code` and the SMALLEST offending input position in `index`
 *    (deterministic).  Offending elements are skipped (never read or written out of bounds);
 *    the output rows they would have produced are unspecified.  The caller zeroes the error
 *    slot (code 0, index INT64_MAX) before use; `err` may be NULL to skip reporting.
 *  - Ids are int64 at the boundary.  Integer outputs are bit-exact and run-to-run
 *    deterministic; floating-point outputs are run-to-run bit-identical (no float atomics:
 *    every reduction has a fixed order).
 *  - sm_100a only: on any other device every compute call returns TFS_ERR_UNSUPPORTED.
 *    There is no CPU fallback.
 */
#ifndef TFS_H
#define TFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TFS_OK = 0,
  TFS_ERR_INVALID_ARGUMENT = 1,
  TFS_ERR_OUT_OF_RANGE = 2,
  TFS_ERR_BAD_POSITIONS = 3,
  TFS_ERR_WORKSPACE_TOO_SMALL = 4,
  TFS_ERR_CUDA = 5,
  TFS_ERR_UNSUPPORTED = 7,
  TFS_ERR_SAMPLER_EXHAUSTED = 8,
  TFS_ERR_CAPACITY = 9, /* a fixed-capacity route slot overflowed (tfs_route_plan) */
  TFS_ERR_COMM_TIMEOUT = 10 /* a device barrier waited longer than its timeout (tfs_comm) */
} tfs_status;

typedef enum { TFS_F32 = 0, TFS_BF16 = 1 } tfs_dtype;

/* Device-resident data-error slot.  index = smallest offending input position. */
typedef struct {
  int32_t code;
  int32_t _pad;
  int64_t index;
} tfs_device_error;

/* Library version (major*10000 + minor*100 + patch) and status strings. */
int32_t tfs_version(void);
const char* tfs_status_string(int32_t status);
/* Message of the last TFS_ERR_CUDA on this host thread (copied into buf, NUL-terminated). */
int32_t tfs_last_error_detail(char* buf, size_t len);
/* TFS_OK if `device` is an sm_100 (B200-class) GPU, TFS_ERR_UNSUPPORTED otherwise. */
int32_t tfs_device_check(int32_t device);

/* ==== Part =========================================================================
 * "The dynamic partition (Part) operation divides the incoming indices into variable-sized
 * tensors that contain the indices destined for each shard."
 * Default (assignments == NULL): owner = ids[i] mod num_shards, out_local = ids[i] div
 * num_shards (R-1); ids must lie in [0, vocab) (else TFS_ERR_OUT_OF_RANGE at i, R-5).
 * Explicit mode (assignments != NULL, int32[n]): owner = assignments[i] in [0, num_shards),
 * out_local = ids[i] unchanged; vocab is ignored.
 * Output is shard-major and STABLE (original order within a shard, R-2): out_local[j] and
 * out_positions[j] (original index i of the element placed at slot j) for j < n;
 * out_counts[s] = number of elements of shard s (int64[num_shards]).
 * 1 <= num_shards <= 256.  n == 0 writes zero counts. */
size_t tfs_partition_workspace_bytes(int64_t n, int32_t num_shards);
int32_t tfs_partition(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                      const int32_t* assignments, int64_t* out_local, int64_t* out_positions,
                      int64_t* out_counts, void* ws, size_t ws_bytes, tfs_device_error* err,
                      void* stream);

/* ==== Gather =======================================================================
 * "Gather, which extracts a sparse set of rows from a tensor", colocated with the variable.
 * out[j, :] = table[ids[j], :] for j < n; duplicates allowed; table is row-major [rows x dim].
 * table_dtype must be TFS_F32.  out_dtype TFS_F32 copies bits; TFS_BF16 rounds to nearest
 * even.  ids outside [0, rows) -> TFS_ERR_OUT_OF_RANGE at the smallest j, except id -1, which
 * marks padding (its output row is left unwritten, no error).  dim >= 1; rows are read with
 * 16-byte vectors when dim % 4 == 0 and the pointers are 16-byte aligned. */
int32_t tfs_gather(const void* table, int64_t rows, int32_t dim, int32_t table_dtype,
                   const int64_t* ids, int64_t n, void* out, int32_t out_dtype,
                   tfs_device_error* err, void* stream);
/* tfs_gather2: the same Gather of a row table plus its width-1 companion in one pass (the
 * softmax rows W with their bias b, R-11): out as tfs_gather; out2[j] = table2[ids[j]] (fp32,
 * [n]); table2 has the same `rows`.  Same error and padding behaviour. */
int32_t tfs_gather2(const float* table, int64_t rows, int32_t dim, const float* table2,
                    const int64_t* ids, int64_t n, void* out, int32_t out_dtype, float* out2,
                    tfs_device_error* err, void* stream);

/* ==== Stitch =======================================================================
 * The "dynamic static" (read: dynamic stitch, R-3) op "reassembles the partial results from
 * each shard into a single result tensor": out[positions[j], :] = rows[j, :] for j < n.
 * Rows are opaque: row_bytes bytes each (a multiple of 4).  positions must be a permutation
 * of 0..n-1; when err != NULL it is validated (TFS_ERR_BAD_POSITIONS at the smallest j whose
 * position is out of range or already claimed by an earlier j, R-4) using ws.  With
 * err == NULL no workspace is needed and the permutation is trusted. */
size_t tfs_stitch_workspace_bytes(int64_t n);
int32_t tfs_stitch(const int64_t* positions, const void* rows, int64_t n, int64_t row_bytes,
                   void* out, void* ws, size_t ws_bytes, tfs_device_error* err, void* stream);

/* ==== Log-uniform candidate sampler (R-6..R-10, R-17, R-24) ==========
 * "a set of randomly sampled false classes"; "We sample 512 classes for each batch".
 * Distribution P(k) = ln((k+2)/(k+1)) / ln(V+1) over frequency-ranked ids (R-6), drawn by
 * Philox4x32-10 (ctr = (i, step_hi, step_lo, replica), key = (seed_lo, seed_hi)) -> 53-bit
 * m = ((w0 << 32) | w1) >> 11 -> k = min{k : m < Thr[k]}, Thr[k] = floor(2^53 ln(k+2)/ln(V+1))
 * evaluated in host long double, Thr[V-1] = 2^53 (R-17).
 * unique != 0: the first S DISTINCT draws in draw order, num_tries T = draws consumed (R-8);
 * unique == 0: s_j = draw j, T = S.  Expected counts ec(k) = -expm1(T log1p(-p_k)) (unique) or
 * S p_k; the log of ec is written (as fp32) for every sampled id and every label (R-10, R-24).
 *
 * Setup: `state` is a device buffer of tfs_sampler_state_bytes(vocab) bytes.
 * tfs_sampler_init fills it (threshold table computed on the host, uploaded synchronously;
 * per-id scratch initialised) and returns in *out_max_draws (host) a draw budget for
 * (vocab, S): the smallest N whose expected number of distinct draws exceeds S by 10 standard
 * deviations (Chernoff; failure probability < 1e-21).  Sampling with that budget never needs
 * the host; if the budget is ever exhausted the error slot gets TFS_ERR_SAMPLER_EXHAUSTED.
 * The state is reused across calls (each call restores its scratch); calls sharing a state
 * must be stream-ordered.  step_dev (device, nullable): if given, the step counter is read
 * from device memory when the kernels run (so a captured CUDA graph can advance it between
 * replays) and `step` is ignored.  out_sampled int64[S]; out_log_ec_sampled f32[S];
 * out_log_ec_labels f32[n_labels]; out_num_tries int64[1] (device). */
size_t tfs_sampler_state_bytes(int64_t vocab);
int32_t tfs_sampler_init(int64_t vocab, int32_t num_sampled, int32_t unique, void* state,
                         int64_t* out_max_draws /* host */, void* stream);
size_t tfs_sampler_workspace_bytes(int64_t max_draws);
int32_t tfs_log_uniform_sample(const void* state, int64_t vocab, int32_t num_sampled,
                               int32_t unique, int64_t max_draws, uint64_t seed, uint64_t step,
                               const uint64_t* step_dev, uint32_t replica,
                               const int64_t* labels, int64_t n_labels,
                               int64_t* out_sampled, float* out_log_ec_sampled,
                               float* out_log_ec_labels, int64_t* out_num_tries, void* ws,
                               size_t ws_bytes, tfs_device_error* err, void* stream);

/* tfs_sample_commit: the step draws each step's candidates one step AHEAD (the draws depend on
 * (seed, step, replica) only, not on the batch), off the critical path; at the step it commits
 * them: out_sampled / out_log_ec_sampled / out_num_tries = copies of a tfs_log_uniform_sample
 * result (drawn with n_labels = 0), and out_log_ec_labels[t] = log ec(labels[t]) with that T --
 * identical to one tfs_log_uniform_sample call with the labels.  Bad labels as there. */
int32_t tfs_sample_commit(int64_t vocab, int32_t num_sampled, int32_t unique,
                          const int64_t* sampled, const float* log_ec_sampled,
                          const int64_t* num_tries, const int64_t* labels, int64_t n_labels,
                          int64_t* out_sampled, float* out_log_ec_sampled,
                          float* out_log_ec_labels, int64_t* out_num_tries,
                          int64_t* out_labels, tfs_device_error* err, void* stream);
/* (out_labels: optional copy of labels[0, n_labels) -- the step builds its softmax-row lookup
 * ids y || s in one buffer with out_labels + n_labels == out_sampled.) */

/* ==== Sampled softmax forward + backward (DESIGN §3 O9-O11) ==========
 * "performs a sparse multiplication based on the true class for an example and a set of
 * randomly sampled false classes".  For tokens t < B and candidates j < S (R-7: one candidate
 * set per replica and step, shared by its B tokens):
 *   z_t  = h_t . w_true_t + b_true_t - [Q] log_ec_true_t
 *   Z_tj = h_t . w_s_j    + b_s_j    - [Q] log_ec_s_j,  excluded if [HITS] and s_j == y_t (R-9)
 *   lse_t = log(e^{z_t} + sum_j e^{Z_tj});  loss_t = lse_t - z_t;  loss_sum = c sum_t loss_t
 *   g_t = c (e^{z_t - lse_t} - 1);  G_tj = c e^{Z_tj - lse_t} (0 if excluded);  c = grad_scale
 *   dh_t = g_t w_true_t + sum_j G_tj w_s_j;  dw_true_t = g_t h_t;  db_true_t = g_t
 *   dw_s_j = sum_t G_tj h_t;  db_s_j = sum_t G_tj.
 * Layouts: h, w_true, dh, dw_true [B x dim]; w_s, dw_s [S x dim]; all fp32 row-major; vectors
 * fp32 [B] / [S]; labels, sampled int64.  labels/sampled are only compared for the hit mask.
 * operand_dtype TFS_F32: fp32 products, fp32 accumulation (parity mode, max rel err 1e-5).
 * operand_dtype TFS_BF16: h, w_true, w_s rounded to bf16 (RNE) and G rounded to bf16 before
 * the dh / dw_s / db_s reductions; tensor-core (tcgen05) GEMMs with fp32 accumulation; all
 * other math fp32 (R-18).  The tensor-core path requires dim % 64 == 0, lse != NULL and
 * 16-byte aligned h, w_true, dh, dw_true, dw_s.
 * loss, lse, loss_sum may be NULL; the five gradient outputs are required.
 * vocab > 0 promises labels and sampled lie in [0, vocab) and lets the bf16 path find
 * accidental hits through a candidate map of 8 * vocab bytes at the START of the workspace
 * (tfs_ssm_workspace_bytes includes it): that region must be zero before the first call on a
 * workspace (e.g. zero-filled at allocation) and every call leaves it zero again.  vocab == 0:
 * no map, the hit test compares every (token, candidate) id pair (same result, slower).
 * The 256 bytes after the map (at offset 8 * vocab rounded up to 256; offset 0 when vocab ==
 * 0) hold the tensor-core GEMMs' tile-schedule counters and follow the same rule: zero before
 * the first call, left zero by every call -- a zero-filled workspace satisfies both.  Calls
 * sharing a workspace must not run concurrently. */
/* TFS_BF16_OPERANDS (operand_dtype TFS_BF16 only): h, w_true and w_s point to bf16 arrays
 * (uint16 bits, same shapes) that are already the RNE roundings of the fp32 values -- e.g.
 * produced by tfs_gather with out_dtype TFS_BF16 -- so the call skips its conversion pass;
 * results are identical to passing the fp32 arrays. */
/* TFS_LABEL_IN_CANDIDATES (tfs_ssm_partial_stats / tfs_ssm_backward_from_lse only; excludes
 * TFS_REMOVE_ACCIDENTAL_HITS): the candidates are a slice of the full vocabulary, and a token
 * whose label is among them keeps that logit -- see the sharded full softmax below. */
enum {
  TFS_SUBTRACT_LOG_Q = 1u,
  TFS_REMOVE_ACCIDENTAL_HITS = 2u,
  TFS_BF16_OPERANDS = 4u,
  TFS_LABEL_IN_CANDIDATES = 8u
};
typedef struct {
  int64_t B, S;
  int32_t dim;
  int32_t operand_dtype;
  uint32_t flags;
  float grad_scale;
  const float* h;
  const int64_t* labels;
  const float* w_true;
  const float* b_true;
  const float* log_ec_true;
  const int64_t* sampled;
  const float* w_s;
  const float* b_s;
  const float* log_ec_s;
  float* loss;
  float* lse;
  float* loss_sum;
  float* dh;
  float* dw_true;
  float* db_true;
  float* dw_s;
  float* db_s;
  int64_t vocab;
  /* Optional instrumentation (bf16 path): NULL, or an array of 8 cudaEvent_t (any entry NULL)
   * recorded on the stream at: 0 start, 1 after the prep pass, 2 after the logits GEMM (STATS),
   * 3 after the combine, 4 after the gradient GEMM (GRAD), 5 after the column sums, 6 after
   * the grouped dh / dW_s GEMM, 7 end.  Lets a caller time each GEMM launch live.  When
   * tfs_ssm_grad_from_logits() is 1, 2 is after the logits GEMM that also stores the logits and
   * 4 after the elementwise gradient pass that replaces GRAD.  The fp32 path records 0, 2
   * (after its logits GEMM) and 7 only. */
  void* const* timing_events;
  /* SMs the persistent tensor-core GEMMs of the call leave free (0: use every SM), so work on
   * other streams (e.g. the training step's side streams) progresses while they run. */
  int32_t sm_reserve;
  /* Optional cudaEvent_t (NULL: none), recorded on the stream as soon as dw_true, db_true,
   * dw_s and db_s are final -- before the call's last pass (the dh split-K reduction) -- so a
   * caller can start the softmax-row update on another stream while dh is finished. */
  void* rows_ready_event;
} tfs_ssm_args;
size_t tfs_ssm_workspace_bytes(int64_t B, int64_t S, int32_t dim, int32_t operand_dtype,
                               int64_t vocab);
int32_t tfs_sampled_softmax_fwd_bwd(const tfs_ssm_args* a, void* ws, size_t ws_bytes,
                                    void* stream);
/* 1 if this build's bf16 path keeps the logits from the logits GEMM (fp32, B x S in the
 * workspace) and forms G from them in an elementwise pass, 0 if it recomputes them on the
 * tensor cores (the GRAD GEMM).  Results are identical; only the schedule differs. */
int32_t tfs_ssm_grad_from_logits(void);

/* ==== Vocabulary-sharded full softmax: the two local halves =========
 * "the weights are sharded across several tasks, and the multiplication and gradient
 * calculation are colocated with the shards".  Shard r of R holds the classes
 * v = j R + r (j < S) as candidates w_s / b_s / sampled; the B rows of h are the tokens of ALL
 * replicas (an all-gather).  Per shard, over its candidates only (no true-class term):
 *   tfs_ssm_partial_stats:  row_stats[t] = (m_t, s_t) with m_t = max_j Z_tj log2(e) and
 *     s_t = sum_j 2^(Z_tj log2(e) - m_t)  (log2 domain; float pairs [B x 2], 8-byte aligned;
 *     m = -inf, s = 0 when every logit is excluded).  The caller combines the R shards' pairs
 *     into lse_t = ln 2 (M + log2 sum_r s_r 2^(m_r - M)), M = max_r m_r (tfs_lse_combine_peers).
 *   tfs_ssm_backward_from_lse (a->lse = that global lse, input):
 *     G_tj = c (e^{Z_tj - lse_t} - [s_j == y_t]);  dh = G W_s (this shard's PARTIAL of dh,
 *     summed over shards by the caller); dw_s = G^T h;  db_s = column sums of G;
 *     z_label[t] = Z_t,j* (natural units) for the tokens whose label s_j* is a candidate here
 *     (other entries untouched).
 * With TFS_LABEL_IN_CANDIDATES (labels[B], vocab > 0 required) a label among the candidates
 * is part of the softmax (the full-softmax gradient p - onehot); without it, no label is used.
 * Both calls take the same args and workspace (tfs_ssm_workspace_bytes(B, S, dim, TFS_BF16,
 * vocab), candidate map zero before partial_stats) and must be paired in stream order: the
 * backward reads the operand copies and the map the stats call left in the workspace and
 * leaves the map zero.  Tensor-core path only: operand_dtype TFS_BF16, dim % 64 == 0, B, S >= 1;
 * loss and loss_sum must be NULL; w_true / b_true / dw_true / db_true are not used. */
int32_t tfs_ssm_partial_stats(const tfs_ssm_args* a, float* row_stats, void* ws,
                              size_t ws_bytes, void* stream);
int32_t tfs_ssm_backward_from_lse(const tfs_ssm_args* a, float* z_label, void* ws,
                                  size_t ws_bytes, void* stream);
/* Cross-shard pieces of the sharded full softmax, over peer memory (P2P loads of every
 * shard's buffer -- pointers from a symmetric allocation; R >= 1; deterministic: shards are
 * combined in rank order 0..R-1).
 * tfs_lse_combine_peers: lse[t] = ln 2 (M + log2 sum_r s_r 2^(m_r - M)) over
 *   stats_tab[r][t] = (m_r, s_r) float pairs, t < n.
 * tfs_reduce_peers: out[i] = sum_r src_tab[r][offset + i], i < n (the reduce-scatter of dh:
 *   each rank pulls its own tokens' partials).  16-byte aligned when n % 4 == 0 for speed.
 * tfs_label_loss_sum: out[0] = c sum over t < n with labels[t] mod R == shard of
 *   (lse[t] - z_label[t]), in increasing t (one block). */
int32_t tfs_lse_combine_peers(const float* const* stats_tab, int32_t R, int64_t n, float* lse,
                              void* stream);
int32_t tfs_reduce_peers(const float* const* src_tab, int32_t R, int64_t offset, int64_t n,
                         float* out, void* stream);
int32_t tfs_label_loss_sum(const float* lse, const float* z_label, const int64_t* labels,
                           int64_t n, int32_t R, int32_t shard, float c, float* out,
                           void* stream);
/* Dense SGD with a bf16 shadow: table[i] -= lr * grad[i] (fp32, i < n) and, if shadow is not
 * NULL, shadow[i] = bf16(table[i]) (RNE) -- the updated rows' operand copy for the next
 * step's tensor-core GEMMs.  16-byte aligned table / grad, 8-byte aligned shadow. */
int32_t tfs_dense_sgd(float* table, const float* grad, int64_t n, float lr, void* shadow,
                      void* stream);

/* ==== Sort-reduce of a sparse gradient (R-16) =======================================
 * The gradient of Gather is a sparse (ids, rows) pair; before it is routed to the owner
 * shards the rows of equal ids are summed.  Output: U unique ids in ascending (owner, local)
 * order (owner = id mod num_shards, local = id div num_shards), out_local[u] = local id,
 * out_rows[u, :] = sum of rows[i, :] over i with ids[i] == id, summed in increasing i (a fixed
 * order), optional second value stream rows2/out_rows2 (width 1, e.g. the bias gradient)
 * reduced with the same segments; out_counts[s] = unique ids owned by shard s;
 * *out_num_unique (device int64) = U.  Outputs are sized for U <= n.  ids in [0, vocab). */
size_t tfs_sort_reduce_workspace_bytes(int64_t n, int32_t dim);
int32_t tfs_sort_reduce(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                        const float* rows, int32_t dim, const float* rows2, int64_t* out_local,
                        float* out_rows, float* out_rows2, int64_t* out_counts,
                        int64_t* out_num_unique, void* ws, size_t ws_bytes,
                        tfs_device_error* err, void* stream);

/* ==== ScatterAdd + SGD ===========================
 * "SGD ... the update rule is W' <- W - alpha x dL/dW.  A parameter server can implement SGD by
 * using -= as the write operation"; the update acts "on just the values that were originally
 * gathered".  For every distinct id r among ids[0..n): g = sum over i with ids[i] == r of
 * grad_rows[i, :], accumulated in fp32 in a FIXED order (stable sort by id, i.e. increasing i,
 * R-16), then table[r, :] -= lr * g.  Untouched rows are not written.  Optional companion
 * table2/grad2 (width 1, e.g. the bias b with db) is updated with the same segments.
 * ids outside [0, rows) -> TFS_ERR_OUT_OF_RANGE at the smallest i (those i are skipped).
 * n == 0 is a no-op. */
size_t tfs_scatter_add_sgd_workspace_bytes(int64_t n, int32_t dim);
int32_t tfs_scatter_add_sgd(float* table, int64_t rows, int32_t dim, const int64_t* ids,
                            const float* grad_rows, int64_t n, float lr, float* table2,
                            const float* grad2, void* ws, size_t ws_bytes,
                            tfs_device_error* err, void* stream);

/* ==== Planned ScatterAdd + SGD ==================================================================
 * tfs_scatter_add_sgd split in two.  The PLAN -- ids stably sorted, their segments found -- is a
 * function of the ids alone, so a training step can build it as soon as the ids are known
 * (before the gradient exists, overlapping the dense work); the APPLY step then sums each
 * segment's gradient rows in the same fixed order and updates the table exactly as
 * tfs_scatter_add_sgd does (identical results).
 * tfs_scatter_plan: plan (device, caller-owned, tfs_scatter_plan_bytes(n) bytes) for ids[0..n)
 * against a table of `rows` rows; ids outside [0, rows) -> TFS_ERR_OUT_OF_RANGE in err at the
 * smallest such i (they are skipped by the apply); id -1 is padding: skipped, no error (also
 * in tfs_scatter_add_sgd and tfs_sort_reduce).
 * tfs_scatter_add_sgd_planned: apply with a plan built for the same ids, n and rows (not
 * checked); grad_rows / grad2 indexed like those ids; ws of
 * tfs_scatter_apply_workspace_bytes(n, dim) bytes.  The plan is not modified. */
size_t tfs_scatter_plan_bytes(int64_t n);
int32_t tfs_scatter_plan(const int64_t* ids, int64_t n, int64_t rows, void* plan,
                         size_t plan_bytes, tfs_device_error* err, void* stream);
size_t tfs_scatter_apply_workspace_bytes(int64_t n, int32_t dim);
int32_t tfs_scatter_add_sgd_planned(float* table, int64_t rows, int32_t dim, const void* plan,
                                    size_t plan_bytes, int64_t n, const float* grad_rows,
                                    float lr, float* table2, const float* grad2, void* ws,
                                    size_t ws_bytes, void* stream);

/* ==== Sparse Momentum / Adagrad on the planned ScatterAdd path =====
 * The paper's optimizers "as user-level code" on the same sparse update: per distinct id r,
 * with g the sum of its gradient rows in the plan's fixed order (fp64), elementwise:
 *   kind 0 SGD:      T = fl32(T - lr g)                         (= tfs_scatter_add_sgd_planned)
 *   kind 1 Momentum: m = fl32(mu m + g);   T = fl32(T - lr m)
 *   kind 2 Adagrad:  a = fl32(a + g g);    T = fl32(T - lr g / sqrt(a))
 * slot: the fp32 m / a table, same shape as table (required for kinds 1, 2); slot2 likewise for
 * the width-1 companion table2 (e.g. the bias).  Duplicates are summed before the single step
 * (reading R-29: the synchronous step applies the combined sparse gradient once). */
typedef struct {
  int32_t kind;
  float lr;
  float mu;
  float* slot;
  float* slot2;
  /* Optional bf16 mirror of the table (same shape, NULL: none): every updated row is also
   * written there, rounded to nearest even -- the copy peers read (tfs_gather_peers2_bf16). */
  uint16_t* mirror;
} tfs_sparse_opt;
int32_t tfs_scatter_opt_planned(float* table, int64_t rows, int32_t dim, const void* plan,
                                size_t plan_bytes, int64_t n, const float* grad_rows,
                                float* table2, const float* grad2, const tfs_sparse_opt* opt,
                                void* ws, size_t ws_bytes, void* stream);

/* ==== Fixed-capacity routing between R shards (R > 1; DESIGN.md §2 O3-O12) ======================
 * The requester-side halves of Part / route / Stitch and of sort-reduce / route, in a SLOT
 * layout that needs no host-visible counts (so a whole multi-GPU step can be a CUDA graph):
 * the payload for owner o occupies slots [0, cap) of region o of a send buffer, region o at
 * element offset o * stride; unused slots carry id -1.  Only DISTINCT ids travel (forward
 * dedup): slot s of region o holds the s-th distinct id owned by o in ascending local order.
 * tfs_route_plan: stable composite-key (owner = id mod R, local = id div R) sort plan of
 * ids[0..n) (caller-owned, tfs_route_plan_bytes(n, R) bytes), the send ids (local ids, int64)
 * and, if out_counts != NULL, the distinct ids per owner (device int64 [R]).  More than cap
 * distinct ids for one owner -> TFS_ERR_CAPACITY in err (index = owner; the excess is dropped);
 * ids outside [0, vocab) -> TFS_ERR_OUT_OF_RANGE.
 * tfs_route_unpack: out[t, :] = slot row of ids[t] in the received rows (`slots`, region
 * stride `slots_stride` floats, rows of dim floats): the Stitch of the routed Gather.
 * tfs_route_reduce: the gradient rows of equal ids summed in increasing t (fixed order, fp64
 * accumulation) and written to the slot of that id (rows2 / out_slots2: optional width-1
 * companion, e.g. the bias gradient).  Plans are not modified. */
size_t tfs_route_plan_bytes(int64_t n, int32_t num_shards);
int32_t tfs_route_plan(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                       int64_t cap, void* plan, size_t plan_bytes, int64_t* out_send_local,
                       int64_t send_stride, int64_t* out_counts, tfs_device_error* err,
                       void* stream);
int32_t tfs_route_unpack(const void* plan, size_t plan_bytes, int64_t n, int64_t vocab,
                         int32_t num_shards, int64_t cap, const float* slots,
                         int64_t slots_stride, int32_t dim, float* out, void* stream);
size_t tfs_route_reduce_workspace_bytes(int64_t n, int32_t dim);
int32_t tfs_route_reduce(const void* plan, size_t plan_bytes, int64_t n, int64_t vocab,
                         int32_t num_shards, int64_t cap, const float* rows, int32_t dim,
                         const float* rows2, float* out_slots, int64_t out_stride,
                         float* out_slots2, int64_t out2_stride, void* ws, size_t ws_bytes,
                         void* stream);
/* One-sided NVLink variants (R > 1 with peer-mapped memory, e.g. symmetric allocations): the
 * payload goes straight into the owner's memory instead of a local send buffer.
 * tfs_route_plan_push: as tfs_route_plan, but the send ids of owner o are stored at
 * dst_tab[o] + dst_off (dst_tab: device array of R peer pointers to the owners' inboxes).
 * tfs_route_reduce_push: as tfs_route_reduce, rows of owner o to out_tab[o] + out_off + s * dim
 * (out_off % 4 == 0 when dim % 4 == 0), companions to out2_tab[o] + out2_off + s.
 * tfs_gather_peers: out[t, :] = row (id div R) of shard (id mod R) read through shards[id mod R]
 * (device array of R peer pointers to equally shaped shards of shard_rows rows): Part, both
 * routes, the owner Gather and Stitch in one kernel (pull); out_dtype TFS_F32 copies, TFS_BF16
 * rounds to nearest even (as tfs_gather).  ids outside [0, vocab) ->
 * TFS_ERR_OUT_OF_RANGE (-1: padding, row unwritten).  The caller orders these with device
 * barriers across the GPUs (tables stable during pulls, inboxes complete before use). */
int32_t tfs_route_plan_push(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                            int64_t cap, void* plan, size_t plan_bytes, int64_t* const* dst_tab,
                            int64_t dst_off, int64_t* out_counts, tfs_device_error* err,
                            void* stream);
int32_t tfs_route_reduce_push(const void* plan, size_t plan_bytes, int64_t n, int64_t vocab,
                              int32_t num_shards, int64_t cap, const float* rows, int32_t dim,
                              const float* rows2, float* const* out_tab, int64_t out_off,
                              float* const* out2_tab, int64_t out2_off, void* ws,
                              size_t ws_bytes, void* stream);
int32_t tfs_gather_peers(const float* const* shards, int64_t shard_rows, int32_t dim,
                         const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                         void* out, int32_t out_dtype, tfs_device_error* err, void* stream);
/* tfs_gather_peers2: tfs_gather_peers plus a width-1 companion table sharded the same way
 * (shards2[o] = owner o's [shard_rows] fp32 array): out2[t] = shards2[id % R][id / R]. */
int32_t tfs_gather_peers2(const float* const* shards, int64_t shard_rows, int32_t dim,
                          const float* const* shards2, const int64_t* ids, int64_t n,
                          int64_t vocab, int32_t num_shards, void* out, int32_t out_dtype,
                          float* out2, tfs_device_error* err, void* stream);
/* tfs_gather_peers2_bf16: the same with the rows read from the owners' bf16 MIRRORS of the
 * table (bf16 [shard_rows x dim] each, kept equal to bf16-RNE(table) by the owners' updates:
 * tfs_sparse_opt.mirror) and written as bf16 -- identical output to tfs_gather_peers2 with
 * out_dtype = TFS_BF16, at half the bytes over NVLink.  dim % 8 == 0, out 16-byte aligned. */
int32_t tfs_gather_peers2_bf16(const uint16_t* const* shards, int64_t shard_rows, int32_t dim,
                               const float* const* shards2, const int64_t* ids, int64_t n,
                               int64_t vocab, int32_t num_shards, uint16_t* out, float* out2,
                               tfs_device_error* err, void* stream);
/* Owner side.  tfs_gather_slots: for each slot (o, s) of num_slots regions x cap, the row of id
 * ids[o * ids_stride + s] of the local shard to out + o * out_stride + s * dim (fp32; -1 ids
 * are padding, rows left unwritten).  tfs_scatter_plan_slots / tfs_scatter_add_sgd_planned_slots:
 * the planned ScatterAdd-SGD over the R x cap received slots (entry i = slot (i / cap, i % cap),
 * so equal ids from different requesters are summed in requester order), gradient rows at
 * grad + o * grad_stride + s * dim (grad2 + o * grad2_stride + s).  sorted_runs != 0 promises
 * that every region holds strictly ascending ids followed by -1 padding (what tfs_route_plan
 * sends): the plan is then a merge of the R runs instead of a radix sort; a violated promise is
 * reported as TFS_ERR_INVALID_ARGUMENT in err. */
int32_t tfs_gather_slots(const float* table, int64_t rows, int32_t dim, const int64_t* ids,
                         int64_t ids_stride, int32_t num_slots, int64_t cap, float* out,
                         int64_t out_stride, tfs_device_error* err, void* stream);
int32_t tfs_scatter_plan_slots(const int64_t* ids, int64_t ids_stride, int32_t num_slots,
                               int64_t cap, int64_t rows, int32_t sorted_runs, void* plan,
                               size_t plan_bytes, tfs_device_error* err, void* stream);
int32_t tfs_scatter_add_sgd_planned_slots(float* table, int64_t rows, int32_t dim,
                                          const void* plan, size_t plan_bytes,
                                          int32_t num_slots, int64_t cap, const float* grad,
                                          int64_t grad_stride, float lr, float* table2,
                                          const float* grad2, int64_t grad2_stride, void* ws,
                                          size_t ws_bytes, void* stream);

/* tfs_scatter_opt_planned_slots: tfs_scatter_add_sgd_planned_slots with the sparse optimizer of
 * tfs_scatter_opt_planned (slot / slot2 shaped like this owner's table / table2). */
int32_t tfs_scatter_opt_planned_slots(float* table, int64_t rows, int32_t dim, const void* plan,
                                      size_t plan_bytes, int32_t num_slots, int64_t cap,
                                      const float* grad, int64_t grad_stride, float* table2,
                                      const float* grad2, int64_t grad2_stride,
                                      const tfs_sparse_opt* opt, void* ws, size_t ws_bytes,
                                      void* stream);

/* ==== Communicator: symmetric device heap + device barriers ===========
 * The paper's workers reach the PS tasks through Send/Recv and note RDMA / NCCL as
 * the next transport.  Here every GPU r is worker r and vocabulary shard r (R-26),
 * and the three exchanges of the step are one-sided NVLink loads / stores into a SYMMETRIC
 * heap: every rank allocates the same number of bytes and carves it in the same order, so a
 * buffer has the same offset on every rank and a peer's copy lives at peer_base[r] + offset.
 *
 * Two modes, one code path above them:
 *  - one process per GPU (nlocal = 1): tfs_comm_create allocates this rank's heap
 *    (cudaMalloc on `device`); tfs_comm_export writes its CUDA IPC handle (host, 64 bytes);
 *    the caller all-gathers the R handles (e.g. through torch.distributed -- plumbing) and
 *    passes them to tfs_comm_connect, which maps the peers' heaps (P2P over NVLink/NVSwitch).
 *    Barriers are a one-block kernel per rank: it stores an epoch into slot (channel, rank) of
 *    every peer's flag area (st.release.sys) and waits until its own R slots reach the epoch
 *    (ld.acquire.sys); a wait longer than timeout_ms (0: 10 s) writes TFS_ERR_COMM_TIMEOUT and
 *    the peer index into the comm's device error slot and returns (no hang, no trap).
 *  - all ranks in one process on one GPU (nlocal = nranks, first_rank = 0; test and
 *    development mode): nranks heaps on `device`, no IPC; a barrier is stream ordering
 *    (every local rank records an event, every local rank's stream waits for all of them) --
 *    no kernel ever spins on another kernel.  tfs_comm_connect must not be called.
 * heap_bytes is per rank (tfs_step_heap_bytes gives what a step needs); the first 64 KB of each
 * heap hold the barrier flags.  One comm serves one stepper at a time.
 * tfs_comm_heap: device base of local rank `local`'s heap; tfs_comm_peer_bases: device array
 * int64[nranks] of the heap bases as seen from local rank `local` (for peer pointer tables).
 * tfs_comm_error: device tfs_device_error of local rank `local` (zeroed at create). */
typedef struct tfs_comm tfs_comm;
int32_t tfs_comm_create(int32_t nranks, int32_t first_rank, int32_t nlocal, int32_t device,
                        size_t heap_bytes, uint32_t timeout_ms, tfs_comm** out);
int32_t tfs_comm_export(tfs_comm* comm, void* handle_out /* host, 64 bytes */);
int32_t tfs_comm_connect(tfs_comm* comm, const void* handles /* host, nranks x 64 bytes */);
int32_t tfs_comm_barrier(tfs_comm* comm, int32_t channel, void* stream);  /* nlocal == 1 only */
void* tfs_comm_heap(tfs_comm* comm, int32_t local);
const int64_t* tfs_comm_peer_bases(tfs_comm* comm, int32_t local);
tfs_device_error* tfs_comm_error(tfs_comm* comm, int32_t local);
int32_t tfs_comm_destroy(tfs_comm* comm);

/* ==== The training step ===================================
 * One synchronous step (R-15) of the paper's large-vocabulary LM output path on every
 * local rank: sample -> Part -> route ids -> Gather on the
 * owner -> route rows back -> Stitch -> sampled softmax forward +
 * backward -> per-id gradient sums -> route gradients -> ScatterAdd-SGD
 * `-=` on the owner.  With R = 1 the routes are identities; with R > 1 they are the
 * one-sided NVLink exchanges of the comm (pull of rows, push of distinct ids and gradient sums
 * into the owners' inboxes, three device barriers).  num_sampled == 0 selects the FULL softmax
 * (config F): R = 1 scores every class (true class separate, hit excluded, R-9); R > 1 is the
 * vocabulary-sharded full softmax of P:706-714 (W, b never move; each shard scores all R*B
 * tokens against its V/R classes, R-30).
 * The stepper owns every buffer: tables (shards of E, W, b; in the comm heap when R > 1), the
 * per-step buffers, workspaces, plans, its streams and events; nothing is allocated after
 * tfs_step_create.  The step has no host synchronisation, so tfs_step_capture records it (all
 * local ranks) into one CUDA graph that tfs_step_run replays.
 * Config: tokens = B per replica; lr > 0 SGD step; optimizer 0 SGD / 1 Momentum (momentum) /
 * 2 Adagrad (accumulators start at adagrad_init), slot tables sharded like the tables (R-29);
 * cap_e / cap_w: route slots per owner for the E / W lookups (0: the worst case, B and B + S,
 * so no batch can overflow; smaller values save memory and an overflow is reported as
 * TFS_ERR_CAPACITY in the step's error slot); seed: sampler key; flags as tfs_ssm_args
 * (TFS_SUBTRACT_LOG_Q | TFS_REMOVE_ACCIDENTAL_HITS for the sampled step).
 * loss_sum (buffer TFS_BUF_LOSS_SUM) is this rank's share of the global mean loss: c times the
 * sum of the per-token losses formed on this rank (its own tokens; full-sharded: the tokens
 * whose label it owns); the global loss is the sum over ranks.  c = 1 / (R B) (R-13). */
typedef struct {
  int64_t vocab;
  int32_t dim;
  int32_t num_shards;     /* R */
  int64_t tokens;         /* B per replica */
  int64_t num_sampled;    /* S per replica; 0 = full softmax */
  int32_t operand_dtype;  /* TFS_BF16 (tensor cores) or TFS_F32 (parity mode; R = 1 only) */
  uint32_t flags;
  float lr;
  int32_t unique;         /* sampler: first S distinct draws (1) or S draws (0) */
  uint64_t seed;
  int32_t optimizer;      /* 0 SGD, 1 Momentum, 2 Adagrad */
  float momentum;
  float adagrad_init;
  int64_t cap_e, cap_w;   /* 0 = worst case */
} tfs_step_config;
typedef struct tfs_stepper tfs_stepper;
/* Bytes of symmetric heap per rank that a step with this config needs (host arithmetic). */
size_t tfs_step_heap_bytes(const tfs_step_config* cfg);
/* comm: NULL for R = 1 (one local rank); else a comm of cfg->num_shards ranks with heaps of at
 * least tfs_step_heap_bytes(cfg) bytes (connected, in the one-process-per-GPU mode).  The
 * tables are zero after create: fill them through tfs_step_buffer, then tfs_step_sync. */
int32_t tfs_step_create(const tfs_step_config* cfg, tfs_comm* comm, tfs_stepper** out);
int32_t tfs_step_destroy(tfs_stepper* st);
/* Named buffers of local rank `local` (device pointer, element count, element type 0 f32 /
 * 1 bf16 / 2 int64 / 3 int32): tables and slots (this rank's shard rows), the step's inputs x, y
 * and the lookup ids y||s, the sampler outputs, gathered rows, softmax outputs and gradients,
 * the error slot (2 x int64: code, smallest offending position), the step counter, and the
 * distinct ids per owner of the last step ([2 x R]: E, W). */
enum {
  TFS_BUF_E = 0, TFS_BUF_W, TFS_BUF_B, TFS_BUF_SLOT_E, TFS_BUF_SLOT_W, TFS_BUF_SLOT_B,
  TFS_BUF_X, TFS_BUF_Y, TFS_BUF_QW, TFS_BUF_LOG_EC_S, TFS_BUF_LOG_EC_Y, TFS_BUF_NUM_TRIES,
  TFS_BUF_H, TFS_BUF_W_ROWS, TFS_BUF_B_ROWS, TFS_BUF_LOSS, TFS_BUF_LSE, TFS_BUF_LOSS_SUM,
  TFS_BUF_DH, TFS_BUF_DW, TFS_BUF_DB, TFS_BUF_ERR, TFS_BUF_STEP, TFS_BUF_COUNTS,
  TFS_BUF_COUNT_
};
int32_t tfs_step_buffer(tfs_stepper* st, int32_t local, int32_t which, void** ptr,
                        int64_t* numel, int32_t* elem_type);
/* After the caller wrote tables / slots: refresh derived copies (the bf16 operand shadow of W
 * in the sharded full softmax) and zero the error slots; synchronises the device. */
int32_t tfs_step_sync(tfs_stepper* st);
/* Set every local rank's step counter (the sampler's step, R-17) and re-draw the sample the
 * next step commits (each step draws the following step's candidates ahead of time).  The
 * counter buffer TFS_BUF_STEP is read-only for callers: write it only through this call.
 * Synchronises the device. */
int32_t tfs_step_set_counter(tfs_stepper* st, int64_t value);
/* One step of every local rank on `stream`.  io->host == 0: x / y are DEVICE pointers to
 * [nlocal x B] int64 (rank-major); == 1: HOST pointers (pinned for asynchrony) copied to the
 * step's input buffers on `stream` inside the call, and each local rank's loss_sum is copied
 * back to io->loss_host[nlocal] (host) on `stream` -- the caller synchronises before reading.
 * With one local rank and y == x + B (x || y adjacent in one buffer) the inputs move in ONE
 * copy.
 * The step counter (sampler; TFS_BUF_STEP) advances by one on the device.
 * io->timing_events (one local rank, eager only; NULL normally): 21 cudaEvent_t.  R = 1: the
 * step runs its phases SERIALLY on one stream and records 0 start, 1 sample committed (and the
 * next step's drawn), 2 E rows gathered, 3 W rows + b gathered, 4 softmax done, 5 E plan built,
 * 6 W plan built, 7 E updated, 8 W + b updated; 9..16 the softmax call's 8 events
 * (tfs_ssm_args.timing_events).  R > 1 (phases overlapped as usual; events on the main
 * stream): the sampled step records 0 start, 1 B0 passed, 2 sample committed, 3 W rows
 * pulled, 4 W gradients pushed, 5 B2 passed, 6 W updated, 7 E updated (side joined), and
 * 9..16 as above for the softmax; on the side stream 17 ids pushed (before B1), 18 B1 passed,
 * 19 owner plans built, 20 E gradients pushed; the sharded full softmax records 9 / 10 around its
 * partial-stats call and 11 / 12 around its backward call.  Entries may be NULL. */
typedef struct {
  const int64_t* x;
  const int64_t* y;
  int32_t host;
  float* loss_host;
  void* const* timing_events;
} tfs_step_io;
int32_t tfs_step_run(tfs_stepper* st, const tfs_step_io* io, void* stream);
/* Record one step of every local rank (inputs read from TFS_BUF_X / TFS_BUF_Y, step counter
 * advanced on the device) into a CUDA graph; later tfs_step_run calls replay it.  The capture
 * itself launches nothing (stream capture); tfs_step_uncapture drops the graph. */
int32_t tfs_step_capture(tfs_stepper* st);
int32_t tfs_step_uncapture(tfs_stepper* st);
/* Kernel nodes of the captured graph (0 if none). */
int64_t tfs_step_graph_kernels(tfs_stepper* st);

/* ==== Diagnostics ===============================================================================
 * C[M x N] (fp32, row-major) = sum_k A(m, k) B(n, k) on the tcgen05 path with bf16 operands,
 * K split `ksplit` ways and the splits reduced by a finalize pass in split order
 * (deterministic).  a_mn == 0: A is K-major, A(m, k) = A[m * lda + k]; a_mn != 0: MN-major,
 * A(m, k) = A[k * lda + m]; same for B with ldb.  lda / ldb in elements, multiples of 8; N a
 * multiple of 4 (else TFS_ERR_INVALID_ARGUMENT); bases 16-byte aligned.  Workspace: tfs_debug_gemm_workspace_bytes.  Used by the GEMM unit tests. */
size_t tfs_debug_gemm_workspace_bytes(int32_t M, int32_t N, int32_t K, int32_t ksplit);
int32_t tfs_debug_gemm_bf16(const void* A, int64_t lda, int32_t a_mn, const void* B, int64_t ldb,
                            int32_t b_mn, int32_t M, int32_t N, int32_t K, int32_t ksplit,
                            float* C, void* ws, size_t ws_bytes, void* stream);
/* Total number of CUDA kernels this process has launched through libtfs (host counter,
 * incremented at every launch site; graph replays are not counted).  Used by bench.py to
 * report gpu_launches. */
int64_t tfs_debug_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TFS_H */
