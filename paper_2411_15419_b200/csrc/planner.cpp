// Sequence-migration placement: Alg. 1 of the paper with the Eq. (1) cost model.
//
// Runs on the host of every rank with identical inputs (the all-gathered rows_at table), so every
// rank derives the same plan without a controller or RPC (the paper's controller, is
// replaced by a replicated deterministic computation overlapped with the expert GEMMs).
// Exact int64 arithmetic; P (GPU speed) := 1 because it cancels on a homogeneous B200 box (R16).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "luffy.h"
#include "luffy_internal.h"

extern "C" int64_t luffy_attention_cost(int64_t B, int64_t L, int64_t d) {
  // Eq. (1): 3 B L d^2 (Q, K, V projections) + 2 B L^2 d (QK^T and AV).
  return 3 * B * L * d * d + 2 * B * L * L * d;
}

namespace {

struct Key {  // lexicographic (s, f, rank)
  int64_t s, f;
  int32_t j;
  bool operator<(const Key& o) const {
    if (s != o.s) return s < o.s;
    if (f != o.f) return f < o.f;
    return j < o.j;
  }
};

}  // namespace

extern "C" luffy_status luffy_plan_migration(const luffy_migration_problem* prob, int32_t* seq_dest,
                                             int64_t* combine_bytes) {
  using luffy::fail;
  if (!prob || !seq_dest) return fail(LUFFY_E_INVALID, "plan_migration: null argument");
  const int S = prob->num_seqs, P = prob->num_ranks;
  if (S < 0 || P <= 0) return fail(LUFFY_E_INVALID, "plan_migration: num_seqs >= 0 and num_ranks > 0 required");
  if (prob->q < 1) return fail(LUFFY_E_INVALID, "plan_migration: q >= 1 required");
  if (S > 0 && (!prob->seq_len || !prob->rows_at)) return fail(LUFFY_E_INVALID, "plan_migration: null seq_len/rows_at");
  if (prob->row_bytes < 0 || prob->d_model <= 0) return fail(LUFFY_E_INVALID, "plan_migration: bad row_bytes/d_model");
  if (prob->objective != 0 && prob->objective != 1) return fail(LUFFY_E_INVALID, "plan_migration: objective must be 0 or 1");
  int64_t total = 0, longest = 0;
  for (int i = 0; i < S; ++i) {
    if (prob->seq_len[i] < 0) return fail(LUFFY_E_INVALID, "plan_migration: negative sequence length");
    total += prob->seq_len[i];
    longest = std::max<int64_t>(longest, prob->seq_len[i]);
  }
  int64_t cap = prob->capacity_tokens;
  if (cap <= 0) cap = std::max<int64_t>((3 * total + 2 * P - 1) / (2 * P), longest);  // ceil(1.5*sum/P)
  const int64_t d = prob->d_model;

  // Alg. 1 line 1: traffic f_ij of pulling sequence i's rows to GPU j.
  std::vector<int64_t> f((size_t)S * P);
  for (int i = 0; i < S; ++i) {
    const int64_t* r = prob->rows_at + (size_t)i * P;
    int64_t rows = 0;
    for (int j = 0; j < P; ++j) {
      if (r[j] < 0) return fail(LUFFY_E_INVALID, "plan_migration: negative rows_at");
      rows += r[j];
    }
    for (int j = 0; j < P; ++j) f[(size_t)i * P + j] = prob->row_bytes * (rows - r[j]);
  }
  // Alg. 1 line 2: candidate set H_i = q GPUs of least traffic, ties -> lower id.
  const int q = std::min(prob->q, P);
  std::vector<int32_t> H((size_t)S * q);
  std::vector<int32_t> ord(P);
  for (int i = 0; i < S; ++i) {
    std::iota(ord.begin(), ord.end(), 0);
    const int64_t* fi = &f[(size_t)i * P];
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fi[a] < fi[b]; });
    std::copy(ord.begin(), ord.begin() + q, H.begin() + (size_t)i * q);
  }
  // Processing order: longest first, ties by id (R16).
  std::vector<int32_t> seqs(S);
  std::iota(seqs.begin(), seqs.end(), 0);
  std::stable_sort(seqs.begin(), seqs.end(),
                   [&](int a, int b) { return prob->seq_len[a] > prob->seq_len[b]; });
  std::vector<int64_t> B(P, 0), L(P, 0), resident(P, 0);
  const int64_t sign = prob->objective == 0 ? 1 : -1;
  for (int i : seqs) {
    const int64_t li = prob->seq_len[i];
    auto key = [&](int j) {
      // Alg. 1 line 5: s_ij = T_att(B_j + 1, max(L_j, l_i)) - T_att(B_j, L_j).
      int64_t s = luffy_attention_cost(B[j] + 1, std::max(L[j], li), d) - luffy_attention_cost(B[j], L[j], d);
      return Key{sign * s, f[(size_t)i * P + j], j};
    };
    int best = -1;
    Key bk{0, 0, 0};
    for (int c = 0; c < q; ++c) {  // Alg. 1 line 6: best candidate with sufficient capacity
      int j = H[(size_t)i * q + c];
      if (resident[j] + li > cap) continue;
      Key k = key(j);
      if (best < 0 || k < bk) { best = j; bk = k; }
    }
    if (best < 0) {  // widen to every feasible GPU (R16)
      for (int j = 0; j < P; ++j) {
        if (resident[j] + li > cap) continue;
        Key k = key(j);
        if (best < 0 || k < bk) { best = j; bk = k; }
      }
    }
    if (best < 0) return fail(LUFFY_E_CAPACITY, "plan_migration: a sequence fits on no rank (capacity exceeded)");
    seq_dest[i] = best;
    B[best] += 1;
    L[best] = std::max(L[best], li);
    resident[best] += li;
  }
  if (combine_bytes) {
    std::fill(combine_bytes, combine_bytes + (size_t)P * P, 0);
    for (int i = 0; i < S; ++i)
      for (int r = 0; r < P; ++r)
        if (r != seq_dest[i]) combine_bytes[(size_t)r * P + seq_dest[i]] += prob->rows_at[(size_t)i * P + r] * prob->row_bytes;
  }
  return LUFFY_OK;
}

extern "C" luffy_status luffy_adaptive_threshold(double l_ini, double l_prev, int32_t scale2, float* h_out) {
  if (!h_out) return luffy::fail(LUFFY_E_INVALID, "adaptive_threshold: h_out is NULL");
  if (!(l_ini > 0.0) || !std::isfinite(l_ini) || !std::isfinite(l_prev))
    return luffy::fail(LUFFY_E_INVALID, "adaptive_threshold: l_ini must be > 0 and both losses finite");
  const double l_norm = std::max(0.0, (l_ini - l_prev) / l_ini);
  *h_out = (float)((scale2 ? 2.0 : 1.0) / (1.0 + std::exp(l_norm)));
  return LUFFY_OK;
}
