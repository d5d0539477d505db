// oracle.cpp -- plain, slow, single-threaded CPU ORACLE (test infrastructure, see oracle.h).
//
// Every function below is written from the paper's statement of the operation (cited P:n,
// PAPER.md line n) or, where the paper is silent, from the reading DESIGN.md §3 records (R-k).
// Floating point is accumulated in fp64.  No blocking, fusion or reordering beyond what the
// definitions state.  Shares no code with the CUDA path.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <utility>
#include <vector>

namespace {

constexpr int kOk = 0, kInvalid = 1, kOutOfRange = 2, kBadPositions = 3, kExhausted = 8;

}  // namespace

extern "C" {

// ---------------------------------------------------------------------------------------------
// Part.  P:691-693: "The dynamic partition (Part) operation divides the incoming indices into
// variable-sized tensors that contain the indices destined for each shard".  Shard function
// owner = id mod R, local row = id div R (R-1); stable within a shard (R-2).
int orc_partition(const int64_t* ids, int64_t n, int64_t vocab, int32_t num_shards,
                  const int32_t* assignments, int64_t* out_local, int64_t* out_positions,
                  int64_t* out_counts, int64_t* bad) {
  if (n < 0 || num_shards < 1) return kInvalid;
  // Validate first: the smallest offending position.
  for (int64_t i = 0; i < n; ++i) {
    bool ok = assignments ? (assignments[i] >= 0 && assignments[i] < num_shards)
                          : (ids[i] >= 0 && ids[i] < vocab);
    if (!ok) {
      if (bad) *bad = i;
      return kOutOfRange;
    }
  }
  // One list per shard, appended in input order.
  std::vector<std::vector<std::pair<int64_t, int64_t>>> lists(num_shards);
  for (int64_t i = 0; i < n; ++i) {
    int64_t owner = assignments ? assignments[i] : ids[i] % num_shards;
    int64_t local = assignments ? ids[i] : ids[i] / num_shards;
    lists[owner].push_back({local, i});
  }
  // Concatenate the lists in shard order.
  int64_t j = 0;
  for (int32_t o = 0; o < num_shards; ++o) {
    out_counts[o] = (int64_t)lists[o].size();
    for (auto& e : lists[o]) {
      out_local[j] = e.first;
      out_positions[j] = e.second;
      ++j;
    }
  }
  return kOk;
}

// ---------------------------------------------------------------------------------------------
// bfloat16 round-to-nearest-even (R-18): keep the top 16 bits of the fp32 pattern, rounding
// the discarded 16 bits to nearest, ties to the even kept pattern.  NaN stays NaN.
float orc_bf16_round(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) {
    u |= 0x00400000u;  // quiet NaN
    u &= 0xffff0000u;
  } else {
    uint32_t discarded = u & 0xffffu;
    uint32_t kept = u >> 16;
    if (discarded > 0x8000u || (discarded == 0x8000u && (kept & 1u))) kept += 1;
    u = kept << 16;
  }
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

void orc_bf16_round_array(const float* x, int64_t n, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16_round(x[i]);
}

static uint16_t bf16_bits(float x) {
  float r = orc_bf16_round(x);
  uint32_t u;
  std::memcpy(&u, &r, 4);
  return (uint16_t)(u >> 16);
}

// ---------------------------------------------------------------------------------------------
// Gather.  P:688-691: "Gather, which extracts a sparse set of rows from a tensor".
int orc_gather(const float* table, int64_t rows, int32_t dim, const int64_t* ids, int64_t n,
               int32_t out_bf16, void* out, int64_t* bad) {
  if (n < 0 || dim < 1 || rows < 0) return kInvalid;
  for (int64_t j = 0; j < n; ++j) {
    if (ids[j] < 0 || ids[j] >= rows) {
      if (bad) *bad = j;
      return kOutOfRange;
    }
  }
  for (int64_t j = 0; j < n; ++j) {
    const float* src = table + ids[j] * (int64_t)dim;
    for (int32_t k = 0; k < dim; ++k) {
      if (out_bf16)
        ((uint16_t*)out)[j * dim + k] = bf16_bits(src[k]);
      else
        ((float*)out)[j * dim + k] = src[k];
    }
  }
  return kOk;
}

// ---------------------------------------------------------------------------------------------
// Stitch.  P:693-695: the "dynamic static" [stitch, R-3] operation "reassembles the partial
// results from each shard into a single result tensor".  A position outside 0..n-1, or one
// already claimed by an earlier j, is an error at j (R-4).
int orc_stitch(const int64_t* positions, const void* rows, int64_t n, int64_t row_bytes,
               void* out, int64_t* bad) {
  if (n < 0 || row_bytes < 1) return kInvalid;
  std::vector<char> seen((size_t)n, 0);
  for (int64_t j = 0; j < n; ++j) {
    int64_t p = positions[j];
    if (p < 0 || p >= n || seen[(size_t)p]) {
      if (bad) *bad = j;
      return kBadPositions;
    }
    seen[(size_t)p] = 1;
  }
  for (int64_t j = 0; j < n; ++j)
    std::memcpy((char*)out + positions[j] * row_bytes, (const char*)rows + j * row_bytes,
                (size_t)row_bytes);
  return kOk;
}

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), R-17.  Ten rounds; the key is bumped by
// the Weyl constants before every round after the first.
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = (uint64_t)M0 * c0;
    uint64_t p1 = (uint64_t)M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// ---------------------------------------------------------------------------------------------
// Log-uniform (Zipfian) candidate distribution over frequency-ranked ids (R-6):
// P(k) = ln((k+2)/(k+1)) / ln(V+1).  Integer inverse-CDF thresholds (R-17).
void orc_log_uniform_thresholds(int64_t vocab, uint64_t* thr) {
  const long double denom = logl((long double)vocab + 1.0L);
  for (int64_t k = 0; k < vocab; ++k) {
    long double frac = logl((long double)k + 2.0L) / denom;
    thr[k] = (uint64_t)floorl(ldexpl(frac, 53));
  }
  if (vocab > 0) thr[vocab - 1] = (uint64_t)1 << 53;
}

double orc_log_uniform_prob(int64_t vocab, int64_t k) {
  return (std::log((double)k + 2.0) - std::log((double)k + 1.0)) / std::log((double)vocab + 1.0);
}

int orc_log_uniform_sample(int64_t vocab, int32_t num_sampled, int32_t unique, uint64_t seed,
                           uint64_t step, uint32_t replica, const int64_t* labels,
                           int64_t n_labels, int64_t max_draws, int64_t* out_sampled,
                           double* out_log_ec_sampled, double* out_log_ec_labels,
                           int64_t* out_num_tries) {
  if (vocab < 1 || num_sampled < 0 || (unique && num_sampled > vocab) || n_labels < 0)
    return kInvalid;
  std::vector<uint64_t> thr((size_t)vocab);
  orc_log_uniform_thresholds(vocab, thr.data());
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  auto draw = [&](int64_t i) -> int64_t {
    const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(step >> 32), (uint32_t)step, replica};
    uint32_t w[4];
    orc_philox4x32_10(ctr, key, w);
    uint64_t m = ((((uint64_t)w[0]) << 32) | w[1]) >> 11;  // 53-bit integer
    // k = min{ k : m < Thr[k] }  (first threshold strictly above m)
    return (int64_t)(std::upper_bound(thr.begin(), thr.end(), m) - thr.begin());
  };
  int64_t T = 0;
  if (unique) {
    // First S distinct draws, in order of first occurrence; T = draws consumed (R-8).
    std::set<int64_t> seen;
    int64_t kept = 0, i = 0;
    while (kept < num_sampled) {
      if (i >= max_draws) return kExhausted;
      int64_t k = draw(i);
      ++i;
      if (seen.insert(k).second) out_sampled[kept++] = k;
    }
    T = i;
  } else {
    for (int64_t j = 0; j < num_sampled; ++j) out_sampled[j] = draw(j);
    T = num_sampled;
  }
  *out_num_tries = T;
  // Expected counts (R-10, R-24): ec(k) = 1 - (1 - p_k)^T (unique) or S * p_k.
  auto log_ec = [&](int64_t k) -> double {
    double p = orc_log_uniform_prob(vocab, k);
    double ec = unique ? -std::expm1((double)T * std::log1p(-p)) : (double)num_sampled * p;
    return std::log(ec);
  };
  for (int64_t j = 0; j < num_sampled; ++j) out_log_ec_sampled[j] = log_ec(out_sampled[j]);
  for (int64_t t = 0; t < n_labels; ++t) {
    if (labels[t] < 0 || labels[t] >= vocab) return kOutOfRange;
    out_log_ec_labels[t] = log_ec(labels[t]);
  }
  return kOk;
}

// ---------------------------------------------------------------------------------------------
// Sampled softmax.  P:715-717: "a sampled softmax, which performs a sparse multiplication
// based on the true class for an example and a set of randomly sampled false classes";
// "multiplies the output by a random sparse matrix containing weights for the
// true class and a random sample of false classes".  Logits, loss and gradients are the
// definitions O9-O11 of DESIGN.md §3 (Jean et al., cited P:715).
//
// flag 4 (label in candidates, reading R-30): the vocabulary-sharded FULL softmax of
// P:706-714, where the candidates are classes of the vocabulary and a token's label is one of
// them (no separate true-class term): lse_t = ln sum_j e^{Z_tj}; z_t = Z_{t,j*} with j* the
// first column whose id is y_t (one must exist); G_tj = c (e^{Z_tj - lse_t} - [s_j == y_t]),
// rounded to bf16 as a whole in bf16 mode (the GPU's rounding point); dh = sum_j G_tj W_s,j.
//
// Alongside every gradient the oracle can return the sum of the ABSOLUTE values of the terms
// that form it (abs_* outputs): abs_dh_t = |g_t| |W_true,t| + sum_j |G_tj| |W_s,j|,
// abs_dw_s,j = sum_t |G_tj| |h_t|, abs_db_s,j = sum_t |G_tj|, abs_loss_t = |lse_t| + |z_t|.
// They are the scale of the rounding error any evaluation order commits (the parity tests
// bound |gpu - oracle| by tol x abs_*, element by element).
int orc_sampled_softmax(const orc_ssm_io* io) {
  const int64_t B = io->B, S = io->S;
  const int32_t d = io->dim;
  if (B < 0 || S < 0 || d < 1) return kInvalid;
  const bool sub_q = io->flags & 1u, rm_hits = io->flags & 2u, label_in = io->flags & 4u;
  if (rm_hits && label_in) return kInvalid;
  const double c = io->grad_scale;
  auto op = [&](float v) -> double { return io->bf16 ? (double)orc_bf16_round(v) : (double)v; };
  auto grad_round = [&](double g) -> double {
    return io->bf16 ? (double)orc_bf16_round((float)g) : g;
  };
  // Operands (rounded in bf16 mode), as fp64.  Label-in mode has no true-class operand.
  std::vector<double> h((size_t)(B * d)), wt(label_in ? 0 : (size_t)(B * d)), ws((size_t)(S * d));
  for (int64_t i = 0; i < B * d; ++i) h[i] = op(io->h[i]);
  if (!label_in)
    for (int64_t i = 0; i < B * d; ++i) wt[i] = op(io->w_true[i]);
  for (int64_t i = 0; i < S * d; ++i) ws[i] = op(io->w_s[i]);

  // O9: sampled logits Z_tj and the true logit z_t.
  auto z_samp = [&](int64_t t, int64_t j) -> double {
    double acc = 0.0;
    for (int32_t k = 0; k < d; ++k) acc += h[t * d + k] * ws[j * d + k];
    acc += io->b_s[j];
    if (sub_q) acc -= io->log_ec_s[j];
    return acc;
  };
  auto label_col = [&](int64_t t) -> int64_t {  // label-in: first column holding y_t
    for (int64_t j = 0; j < S; ++j)
      if (io->sampled[j] == io->labels[t]) return j;
    return -1;
  };
  auto z_true = [&](int64_t t) -> double {
    if (label_in) return z_samp(t, label_col(t));
    double acc = 0.0;
    for (int32_t k = 0; k < d; ++k) acc += h[t * d + k] * wt[t * d + k];
    acc += io->b_true[t];
    if (sub_q) acc -= io->log_ec_true[t];
    return acc;
  };
  // Excluded (treated as -inf): an accidental hit of the label among the sampled classes (R-9).
  auto excluded = [&](int64_t t, int64_t j) -> bool {
    return rm_hits && io->sampled[j] == io->labels[t];
  };
  auto is_label = [&](int64_t t, int64_t j) -> bool {
    return label_in && io->sampled[j] == io->labels[t];
  };

  // O10: lse_t = mu + ln(e^{z-mu} + sum_j e^{Z_tj - mu}) (label-in: the label is one of the
  // Z_tj, so there is no separate e^{z-mu} term) for every token an output needs: all tokens
  // when any dW_s / db_s column is asked for (they sum over t), else only the requested ones.
  std::vector<double> lse((size_t)B), zt((size_t)B);
  std::vector<double> Zrow((size_t)S);
  std::vector<char> need((size_t)B, 0);
  const bool all_tokens = !io->tok_idx || !io->col_idx || io->n_col > 0;
  if (!all_tokens)
    for (int64_t r = 0; r < io->n_tok; ++r)
      if (io->tok_idx[r] >= 0 && io->tok_idx[r] < B) need[io->tok_idx[r]] = 1;
  for (int64_t t = 0; t < B; ++t) {
    if (!all_tokens && !need[t]) continue;
    if (label_in && label_col(t) < 0) return kInvalid;
    zt[t] = z_true(t);
    double mu = label_in ? -INFINITY : zt[t];
    for (int64_t j = 0; j < S; ++j) {
      Zrow[j] = z_samp(t, j);
      if (!excluded(t, j)) mu = std::max(mu, Zrow[j]);
    }
    double sum = label_in ? 0.0 : std::exp(zt[t] - mu);
    for (int64_t j = 0; j < S; ++j)
      if (!excluded(t, j)) sum += std::exp(Zrow[j] - mu);
    lse[t] = mu + std::log(sum);
  }
  // O11: G_tj = c e^{Z_tj - lse_t} (label-in: minus c at the label), bf16-rounded in bf16 mode.
  auto G_pre = [&](int64_t t, int64_t j) -> double {
    return c * (std::exp(z_samp(t, j) - lse[t]) - (is_label(t, j) ? 1.0 : 0.0));
  };
  // bf16 mode: is the rounding of this G a tie within evaluation error?  Any implementation
  // forms G from logits that carry rounding error (the GPU: fp32 accumulation, fp32 exp2); when
  // the exact value lies within kAmbiguity (relative) of the midpoint between two bf16 values,
  // either neighbour is a correct rounding (reading R-34), and the element-wise bound admits
  // one bf16 unit (2^-8 relative) of that term: the amb_* outputs.
  constexpr double kAmbiguity = 1.0 / 16384.0;  // 2^-14
  auto ambiguous = [&](double g) -> bool {
    if (!io->bf16 || g == 0.0) return false;
    const float f = (float)g;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    const uint32_t lo_b = u & 0xffff0000u, hi_b = lo_b + 0x10000u;
    float lo, hi;
    std::memcpy(&lo, &lo_b, 4);
    std::memcpy(&hi, &hi_b, 4);
    const double mid = 0.5 * ((double)lo + (double)hi);
    return std::fabs(g - mid) <= kAmbiguity * std::fabs(g);
  };
  constexpr double kBf16Unit = 1.0 / 256.0;  // 2^-8: one bf16 unit, relative
  auto G_at = [&](int64_t t, int64_t j) -> double { return grad_round(G_pre(t, j)); };

  // O10/O11 per token.
  const int64_t n_tok = io->tok_idx ? io->n_tok : B;
  for (int64_t r = 0; r < n_tok; ++r) {
    const int64_t t = io->tok_idx ? io->tok_idx[r] : r;
    if (t < 0 || t >= B) return kInvalid;
    // d loss / d z_t of the separate true-class term (label-in: carried by G, so 0 here)
    const double g = label_in ? 0.0 : c * (std::exp(zt[t] - lse[t]) - 1.0);
    if (io->loss) io->loss[r] = lse[t] - zt[t];
    if (io->abs_loss) io->abs_loss[r] = std::fabs(lse[t]) + std::fabs(zt[t]);
    if (io->lse) io->lse[r] = lse[t];
    if (io->z_true) io->z_true[r] = zt[t];
    if (io->db_true) io->db_true[r] = g;
    if (io->dw_true)
      for (int32_t k = 0; k < d; ++k) io->dw_true[r * d + k] = g * h[t * d + k];
    if (io->dh || io->abs_dh) {
      std::vector<double> dh((size_t)d, 0.0), ad((size_t)d, 0.0);
      if (!label_in)
        for (int32_t k = 0; k < d; ++k) {
          dh[k] = g * wt[t * d + k];
          ad[k] = std::fabs(g * wt[t * d + k]);
        }
      std::vector<double> am((size_t)d, 0.0);
      for (int64_t j = 0; j < S; ++j) {
        if (excluded(t, j)) continue;
        const double Gp = G_pre(t, j), G = grad_round(Gp);
        const bool amb = ambiguous(Gp);
        for (int32_t k = 0; k < d; ++k) {
          dh[k] += G * ws[j * d + k];
          ad[k] += std::fabs(G * ws[j * d + k]);
          if (amb) am[k] += kBf16Unit * std::fabs(G * ws[j * d + k]);
        }
      }
      for (int32_t k = 0; k < d; ++k) {
        if (io->dh) io->dh[r * d + k] = dh[k];
        if (io->abs_dh) io->abs_dh[r * d + k] = ad[k];
        if (io->amb_dh) io->amb_dh[r * d + k] = am[k];
      }
    }
  }

  // O11 per sampled class: dW_s,j = sum_t G_tj h_t ; db_s,j = sum_t G_tj.
  const int64_t n_col = io->col_idx ? io->n_col : S;
  for (int64_t r = 0; r < n_col; ++r) {
    const int64_t j = io->col_idx ? io->col_idx[r] : r;
    if (j < 0 || j >= S) return kInvalid;
    double db = 0.0, adb = 0.0, amb_b = 0.0;
    std::vector<double> dw((size_t)d, 0.0), aw((size_t)d, 0.0), am((size_t)d, 0.0);
    for (int64_t t = 0; t < B; ++t) {
      if (excluded(t, j)) continue;
      const double Gp = G_pre(t, j), G = grad_round(Gp);
      const bool amb = ambiguous(Gp);
      db += G;
      adb += std::fabs(G);
      if (amb) amb_b += kBf16Unit * std::fabs(G);
      for (int32_t k = 0; k < d; ++k) {
        dw[k] += G * h[t * d + k];
        aw[k] += std::fabs(G * h[t * d + k]);
        if (amb) am[k] += kBf16Unit * std::fabs(G * h[t * d + k]);
      }
    }
    for (int32_t k = 0; k < d; ++k) {
      if (io->dw_s) io->dw_s[r * d + k] = dw[k];
      if (io->abs_dw_s) io->abs_dw_s[r * d + k] = aw[k];
      if (io->amb_dw_s) io->amb_dw_s[r * d + k] = am[k];
    }
    if (io->db_s) io->db_s[r] = db;
    if (io->abs_db_s) io->abs_db_s[r] = adb;
    if (io->amb_db_s) io->amb_db_s[r] = amb_b;
  }
  return kOk;
}

// ---------------------------------------------------------------------------------------------
// Sparse update.  P:697-699: "a set of sparse update operations that act on just the values
// that were originally gathered from each of the shards"; W' <- W - alpha*dL/dW
// applied as "-="; the combiner is associative and commutative, so duplicates are
// summed (fp64 here) before the single write.
int orc_scatter_add_sgd(float* table, int64_t rows, int32_t dim, const int64_t* ids,
                        const double* grad, int64_t n, double lr, int64_t* bad) {
  if (n < 0 || dim < 1) return kInvalid;
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= rows) {
      if (bad) *bad = i;
      return kOutOfRange;
    }
  }
  std::map<int64_t, std::vector<double>> acc;
  for (int64_t i = 0; i < n; ++i) {
    auto& g = acc[ids[i]];
    if (g.empty()) g.assign((size_t)dim, 0.0);
    for (int32_t k = 0; k < dim; ++k) g[k] += grad[i * dim + k];
  }
  for (auto& kv : acc) {
    float* row = table + kv.first * (int64_t)dim;
    for (int32_t k = 0; k < dim; ++k) row[k] = (float)((double)row[k] - lr * kv.second[k]);
  }
  return kOk;
}

// Sparse Momentum / Adagrad ("Momentum, Adagrad, ... as user-level code" on the same
// sparse update path; reading R-29).  Per distinct id r, with g the fp64 sum of
// its gradient rows in increasing i (as orc_scatter_add_sgd):
//   momentum: m_r = fl32(mu * m_r + g);        T_r = fl32(T_r - lr * m_r)
//   adagrad:  a_r = fl32(a_r + g * g);         T_r = fl32(T_r - lr * g / sqrt(a_r))
// (elementwise; the slot tables m / a are fp32 like T; the rounded slot value is the one used).
int orc_scatter_opt(int kind, float* table, float* slot, int64_t rows, int32_t dim,
                    const int64_t* ids, const double* grad, int64_t n, double lr, double mu,
                    int64_t* bad) {
  if (n < 0 || dim < 1 || (kind != 1 && kind != 2)) return kInvalid;
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= rows) {
      if (bad) *bad = i;
      return kOutOfRange;
    }
  }
  std::map<int64_t, std::vector<double>> acc;
  for (int64_t i = 0; i < n; ++i) {
    auto& g = acc[ids[i]];
    if (g.empty()) g.assign((size_t)dim, 0.0);
    for (int32_t k = 0; k < dim; ++k) g[k] += grad[i * dim + k];
  }
  for (auto& kv : acc) {
    float* row = table + kv.first * (int64_t)dim;
    float* sl = slot + kv.first * (int64_t)dim;
    for (int32_t k = 0; k < dim; ++k) {
      const double g = kv.second[k];
      if (kind == 1) {
        sl[k] = (float)(mu * (double)sl[k] + g);
        row[k] = (float)((double)row[k] - lr * (double)sl[k]);
      } else {
        sl[k] = (float)((double)sl[k] + g * g);
        row[k] = (float)((double)row[k] - lr * g / std::sqrt((double)sl[k]));
      }
    }
  }
  return kOk;
}

int orc_sort_reduce(const int64_t* ids, int64_t n, int32_t num_shards, const double* rows,
                    int32_t dim, int64_t* out_local, double* out_rows, int64_t* out_counts,
                    int64_t* out_num_unique) {
  if (n < 0 || num_shards < 1 || dim < 1) return kInvalid;
  std::map<std::pair<int64_t, int64_t>, std::vector<double>> acc;  // (owner, local) -> sum
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0) return kOutOfRange;
    auto& g = acc[{ids[i] % num_shards, ids[i] / num_shards}];
    if (g.empty()) g.assign((size_t)dim, 0.0);
    for (int32_t k = 0; k < dim; ++k) g[k] += rows[i * dim + k];
  }
  for (int32_t o = 0; o < num_shards; ++o) out_counts[o] = 0;
  int64_t u = 0;
  for (auto& kv : acc) {
    out_counts[kv.first.first] += 1;
    out_local[u] = kv.first.second;
    for (int32_t k = 0; k < dim; ++k) out_rows[u * dim + k] = kv.second[k];
    ++u;
  }
  *out_num_unique = u;
  return kOk;
}

}  // extern "C"
