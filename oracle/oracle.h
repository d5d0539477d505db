/*
 * oracle.h -- CPU ORACLE for the sharded-embedding + sampled-softmax training step of
 * Abadi et al., "TensorFlow: A system for large-scale machine learning" (arXiv 1605.08695).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or constant generator with the CUDA path (paper_1605_08695_b200/csrc); neither includes
 * the other.  It is plain, slow and single-threaded on purpose: every function is the
 * definition (or the algorithm step by step) that the paper and DESIGN.md's readings state,
 * accumulated in fp64.
 *
 * Citation keys: "P:n" = /root/reference/PAPER.md line n; "R-k" = reading k in DESIGN.md §3
 * (the survey's C-k table, restated there).
 *
 * Status codes returned by every function: 0 ok, 1 invalid argument, 2 id out of range,
 * 3 bad stitch positions, 8 sampler ran out of draws.  On 2/3 the smallest offending input
 * position is written to *bad (if bad != NULL).
 */
#ifndef TFS_ORACLE_H
#define TFS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Part: stable grouping of ids by owner shard ------------------------------
 * owner = id mod R, local = id div R (R-1); or, when assignments != NULL, owner = assignments[i]
 * and local = ids[i] (SPEC explicit mode).  Output is shard-major, original order inside a
 * shard (R-2).  out_positions[j] = original index of the element placed at slot j. */
int orc_partition(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                  const int32_t* assignments, int64_t* out_local, int64_t* out_positions,
                  int64_t* out_counts, int64_t* bad);

/* ---- Gather: out[j,:] = table[ids[j],:].  out_bf16 != 0 rounds each value to
 * bfloat16 with round-to-nearest-even and stores the 16-bit pattern (uint16 out). */
int orc_gather(const float* table, int64_t rows, int32_t dim, const int64_t* ids, int64_t n,
               int32_t out_bf16, void* out, int64_t* bad);

/* ---- Stitch ("dynamic stitch", R-3): out[positions[j],:] = rows[j,:];
 * positions must be a permutation of 0..n-1 (R-4).  Rows are opaque bytes. */
int orc_stitch(const int64_t* positions, const void* rows, int64_t n, int64_t row_bytes,
               void* out, int64_t* bad);

/* ---- bfloat16 round-to-nearest-even of one fp32 value (R-18), returned as fp32. */
float orc_bf16_round(float x);
void orc_bf16_round_array(const float* x, int64_t n, float* out);

/* ---- Philox4x32-10 (Salmon et al. 2011), counter ctr[4], key key[2] -> out[4] (R-17). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- Log-uniform sampler (R-6..R-10, R-17, R-24). -----------------
 * Thr[k] = floor(2^53 * ln(k+2) / ln(V+1)) (long double), Thr[V-1] = 2^53. */
void orc_log_uniform_thresholds(int64_t vocab, uint64_t* thr);
/* p_k = (ln(k+2) - ln(k+1)) / ln(V+1) */
double orc_log_uniform_prob(int64_t vocab, int64_t k);
/* Draw i of replica r at step tau: Philox(ctr=(i, tau_hi, tau_lo, r), key=(seed_lo, seed_hi))
 * (tau_hi / tau_lo = high / low 32 bits of the 64-bit step) -> m =
 * ((w0<<32)|w1)>>11 -> k = min{k : m < Thr[k]}.  unique: first S distinct in draw order and
 * T = draws consumed; else s_j = k_j, T = S.  log expected counts in fp64 for s and labels:
 * ec = -expm1(T*log1p(-p)) (unique) or S*p.  max_draws bounds the unique loop (status 8). */
int orc_log_uniform_sample(int64_t vocab, int32_t num_sampled, int32_t unique, uint64_t seed,
                           uint64_t step, uint32_t replica, const int64_t* labels,
                           int64_t n_labels, int64_t max_draws, int64_t* out_sampled,
                           double* out_log_ec_sampled, double* out_log_ec_labels,
                           int64_t* out_num_tries);

/* ---- Sampled softmax forward + backward (O8-O11 of DESIGN §3). ----
 * flags: 1 = subtract log expected count (R-10), 2 = remove accidental hits (R-9), 4 = label in
 * candidates (R-30: the sharded full softmax; no true-class term, the label's column carries
 * G = c (p - 1); w_true / b_true / log_ec_true unused; excludes flag 2).
 * bf16 != 0 emulates the bf16-operand mode: h, w_true, w_s rounded RNE to bf16 before use, and
 * the gradient-of-logits G rounded to bf16 before the dh / dW_s / db_s reductions (R-18).
 * Everything else is fp64.  The full log-sum-exp is always computed for every token; the
 * per-token outputs (loss, lse, dh, dw_true, db_true) are written only for the n_tok tokens
 * listed in tok_idx (tok_idx == NULL: all B, in order), and the per-class outputs (dw_s, db_s)
 * only for the n_col classes listed in col_idx (col_idx == NULL: all S).  Output row k of a
 * per-token array belongs to token tok_idx[k]. */
typedef struct {
  int64_t B, S; int32_t dim; int32_t bf16; uint32_t flags; double grad_scale;
  const float* h; const int64_t* labels; const float* w_true; const float* b_true;
  const double* log_ec_true; const int64_t* sampled; const float* w_s; const float* b_s;
  const double* log_ec_s;
  int64_t n_tok; const int64_t* tok_idx; int64_t n_col; const int64_t* col_idx;
  double* loss; double* lse; double* z_true; double* dh; double* dw_true; double* db_true;
  double* dw_s; double* db_s;
  /* optional (NULL = skip): sums of the absolute values of the terms forming loss, dh, dw_s,
   * db_s (|lse| + |z|; |g||W_true| + sum_j |G||W_s|; sum_t |G||h|; sum_t |G|) -- the scale of
   * any evaluation order's rounding error, used by the element-wise parity bound. */
  double* abs_loss; double* abs_dh; double* abs_dw_s; double* abs_db_s;
  /* optional, bf16 mode: 2^-8 x the sum of |terms| whose G rounding is a tie within 2^-14
   * relative (either bf16 neighbour is a correct rounding, reading R-34); 0 elsewhere. */
  double* amb_dh; double* amb_dw_s; double* amb_db_s;
} orc_ssm_io;
int orc_sampled_softmax(const orc_ssm_io* io);

/* ---- Sparse accumulation + SGD. -------------
 * For every touched row r: G[r] = sum over i with ids[i]==r of grad[i,:] (fp64), then
 * table[r] = fl32(table[r] - lr * G[r]).  Duplicates accumulate; untouched rows unchanged. */
int orc_scatter_add_sgd(float* table, int64_t rows, int32_t dim, const int64_t* ids,
                        const double* grad, int64_t n, double lr, int64_t* bad);
/* Sparse Momentum (kind 1) / Adagrad (kind 2) on the same distinct-id sums (reading R-29):
 * momentum m = fl32(mu m + g), T = fl32(T - lr m); adagrad a = fl32(a + g^2),
 * T = fl32(T - lr g / sqrt(a)).  slot: the fp32 m or a table, same shape as table. */
int orc_scatter_opt(int kind, float* table, float* slot, int64_t rows, int32_t dim,
                    const int64_t* ids, const double* grad, int64_t n, double lr, double mu,
                    int64_t* bad);

/* ---- Sort-reduce of a sparse gradient before routing (R-16): unique ids in
 * ascending (owner, local) order, owner = id mod R, local = id div R, fp64 sums. */
int orc_sort_reduce(const int64_t* ids, int64_t n, int32_t num_shards, const double* rows,
                    int32_t dim, int64_t* out_local, double* out_rows, int64_t* out_counts,
                    int64_t* out_num_unique);

#ifdef __cplusplus
}
#endif
#endif
