// Host planner: Algorithm 1, the hybrid cost model of Eq. 9
// evaluated from an exported random forest + AIC polynomial,
// and the exact memory plan behind Eq. 6.
//
// Readings: R-17 inner-loop reset, R-18 early return of [P0] x L,
// R-19 gamma-smoothing against the previous plan, R-20 Pareto prune + sort by
// (t, m, id), R-23 strict "<", R-24 ties: first candidate in generation order.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "internal.hpp"
#include "kernels/kernels.hpp"

namespace pds {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

// ------------------------------------------------------------------ Algorithm 1
// Eq. 6 with reading R-22: sum_l m[pi_l] + max_l w[pi_l] < cap (w = NULL: all zero)
bool plan_feasible(const uint8_t* plan, int L, const double* m, const double* w, double cap, Alg1Counters* c) {
  double acc = 0.0, ws = 0.0;
  for (int l = 0; l < L; ++l) {
    acc += m[plan[l]];
    if (w) ws = std::max(ws, w[plan[l]]);
    if (c) c->layer_checks++;
    if (acc + ws >= cap) return false;  // OOM short-circuit
  }
  return acc + ws < cap;
}

double plan_time(const uint8_t* plan, int L, const double* t) {
  double acc = 0.0;
  for (int l = 0; l < L; ++l) acc += t[plan[l]];
  return acc;
}

// pop_useless (line 1): Pareto prune on (t, m, w), sort ascending by (t, m, id)
static std::vector<int> prune_sort(int n, const double* t, const double* m, const double* w, const uint8_t* en) {
  auto W = [&](int a) { return w ? w[a] : 0.0; };
  std::vector<int> keep;
  for (int a = 0; a < n; ++a) {
    if (!en[a]) continue;
    bool dominated = false;
    for (int b = 0; b < n && !dominated; ++b) {
      if (b == a || !en[b]) continue;
      if (t[b] <= t[a] && m[b] <= m[a] && W(b) <= W(a) && (t[b] < t[a] || m[b] < m[a] || W(b) < W(a)))
        dominated = true;
    }
    if (!dominated) keep.push_back(a);
  }
  std::sort(keep.begin(), keep.end(), [&](int a, int b) {
    if (t[a] != t[b]) return t[a] < t[b];
    if (m[a] != m[b]) return m[a] < m[b];
    return a < b;
  });
  return keep;
}

void alg1(int L, int n, const double* t, const double* m, const double* w, const uint8_t* enabled, double cap,
          std::vector<uint8_t>& out, bool* infeasible, bool* early, Alg1Counters* c) {
  std::vector<int> P = prune_sort(n, t, m, w, enabled);
  *infeasible = false;
  *early = false;
  out.assign(L, 0);
  std::vector<uint8_t> s(L), best;
  double best_t = 0.0;
  bool have = false;
  for (size_t i = 0; i < P.size(); ++i) {
    std::fill(s.begin(), s.end(), (uint8_t)P[i]);          // line 7
    if (c) c->plans++;
    const bool ok = plan_feasible(s.data(), L, m, w, cap, c);
    if (i == 0 && ok) {                                     // lines 8-10 (R-18)
      out = s;
      *early = true;
      return;
    }
    if (ok) {                                               // line 12
      const double tp = plan_time(s.data(), L, t);
      if (!have || tp < best_t) { best = s; best_t = tp; have = true; }
    } else {
      for (size_t k = i + 1; k < P.size(); ++k) {           // lines 14-20
        std::fill(s.begin(), s.end(), (uint8_t)P[i]);       // R-17 reset
        for (int l = 0; l < L; ++l) {
          // pop the first element, append P[k] (a left shift of the window)
          std::memmove(s.data(), s.data() + 1, (size_t)(L - 1));
          s[L - 1] = (uint8_t)P[k];
          if (c) c->plans++;
          if (plan_feasible(s.data(), L, m, w, cap, c)) {
            const double tp = plan_time(s.data(), L, t);
            if (!have || tp < best_t) { best = s; best_t = tp; have = true; }
          }
        }
      }
    }
  }
  if (have) {                                               // line 25
    out = best;
  } else {                                                  // line 27
    int least = P[0];
    for (int a : P)
      if (m[a] < m[least] || (m[a] == m[least] && a < least)) least = a;
    std::fill(out.begin(), out.end(), (uint8_t)least);
    *infeasible = true;
  }
}

// ------------------------------------------------------------------ cost bundle (Eq. 9)
pds_status load_bundle(const char* path, Bundle* b) {
  std::ifstream f(path);
  if (!f) PDS_FAIL(PDS_EINVAL, std::string("pds_load_costs: cannot open ") + path);
  std::string tok;
  auto expect = [&](const char* w) -> bool {
    if (!(f >> tok) || tok != w) {
      set_error(std::string("pds_load_costs: expected '") + w + "', got '" + tok + "'");
      return false;
    }
    return true;
  };
  Bundle nb;
  int ver = 0;
  if (!expect("pds_bundle") || !(f >> ver) || ver != 1) PDS_FAIL(PDS_EINVAL, "pds_load_costs: bad header");
  if (!expect("P") || !(f >> nb.P) || !expect("h") || !(f >> nb.h) || !expect("n") || !(f >> nb.n) ||
      !expect("ffn") || !(f >> nb.ffn) || !expect("L") || !(f >> nb.L) || !expect("capacity") ||
      !(f >> nb.capacity) || !expect("reserve") || !(f >> nb.reserve))
    return PDS_EINVAL;
  // optional (Llama variant, R-GQA / R-SWIGLU): "kv <n_kv> act <0|1>"; absent = MHA + GELU
  if (!(f >> tok)) PDS_FAIL(PDS_EINVAL, "pds_load_costs: truncated header");
  if (tok == "kv") {
    if (!(f >> nb.n_kv) || !expect("act") || !(f >> nb.act)) PDS_FAIL(PDS_EINVAL, "pds_load_costs: bad kv / act");
    if (!(f >> tok)) PDS_FAIL(PDS_EINVAL, "pds_load_costs: truncated header");
  }
  if (tok != "norm") PDS_FAIL(PDS_EINVAL, "pds_load_costs: expected 'norm', got '" + tok + "'");
  for (int i = 0; i < 4; ++i) f >> nb.norm[i][0] >> nb.norm[i][1];
  int ns = 0;
  if (!expect("n_strat") || !(f >> ns)) return PDS_EINVAL;
  for (int i = 0; i < ns; ++i) {
    int sid = -1;
    if (!expect("strategy") || !(f >> sid) || sid < 0 || sid >= PDS_N_STRATEGIES)
      PDS_FAIL(PDS_EINVAL, "pds_load_costs: bad strategy id");
    StratCost& sc = nb.strat[sid];
    sc.present = true;
    if (!expect("s_profile_max") || !(f >> sc.s_profile_max)) return PDS_EINVAL;
    if (!expect("poly") || !(f >> sc.poly_deg >> sc.poly_scale)) return PDS_EINVAL;
    sc.poly_coef.resize(sc.poly_deg + 1);
    for (auto& v : sc.poly_coef) f >> v;
    int nt = 0;
    if (!expect("trees") || !(f >> nt)) return PDS_EINVAL;
    sc.trees.resize(nt);
    for (auto& tr : sc.trees) {
      int nn = 0;
      if (!expect("tree") || !(f >> nn)) return PDS_EINVAL;
      tr.feature.resize(nn); tr.left.resize(nn); tr.right.resize(nn);
      tr.threshold.resize(nn); tr.value.resize(nn);
      for (int k = 0; k < nn; ++k)
        f >> tr.feature[k] >> tr.threshold[k] >> tr.left[k] >> tr.right[k] >> tr.value[k];
    }
  }
  if (!expect("end")) return PDS_EINVAL;
  if (f.fail()) PDS_FAIL(PDS_EINVAL, "pds_load_costs: parse error");
  nb.loaded = true;
  *b = nb;
  return PDS_OK;
}

// feature vector: one-hot over the strategies present (reading R-25) + normalised h, n, L, s
static double feat(const Bundle& b, int strategy, int64_t s, int idx) {
  int nen = 0, pos = -1;
  for (int i = 0; i < PDS_N_STRATEGIES; ++i) {
    if (!b.strat[i].present) continue;
    if (i == strategy) pos = nen;
    ++nen;
  }
  if (idx < nen) return idx == pos ? 1.0 : 0.0;
  const double raw[4] = {(double)b.h, (double)b.n, (double)b.L, (double)s};
  const int j = idx - nen;
  const double lo = b.norm[j][0], hi = b.norm[j][1];
  return hi == lo ? 0.0 : (raw[j] - lo) / (hi - lo);
}

double bundle_time(const Bundle& b, int strategy, int64_t s, int* branch) {
  const StratCost& sc = b.strat[strategy];
  if ((double)s <= sc.s_profile_max) {       // RF: interpolation
    if (branch) *branch = 0;
    double acc = 0.0;
    for (const Tree& tr : sc.trees) {
      int node = 0;
      while (tr.left[node] >= 0) {
        node = feat(b, strategy, s, tr.feature[node]) <= tr.threshold[node] ? tr.left[node] : tr.right[node];
      }
      acc += tr.value[node];
    }
    return acc / (double)sc.trees.size();
  }
  if (branch) *branch = 1;                    // PR: extrapolation
  const double x = (double)s / sc.poly_scale;
  double acc = 0.0;
  for (double c : sc.poly_coef) acc = acc * x + c;
  return acc;
}

// ------------------------------------------------------------------ memory plan
int64_t BufPlan::off(const std::vector<Region>& v, const char* n) const {
  for (const auto& r : v)
    if (std::strcmp(r.name, n) == 0) return r.off;
  return -1;
}

static void push(std::vector<Region>& v, int64_t& tot, const char* n, int64_t bytes) {
  v.push_back(Region{n, bytes, tot});
  tot += al(bytes);
}

int64_t persistent_bytes(const pds_model& m, int P) {
  const int64_t h = m.h, F = m.ffn;
  const int64_t nk = m.n_kv_heads > 0 ? m.n_kv_heads : m.n_heads;
  const int64_t qkv = (m.n_heads + 2 * nk) * (h / m.n_heads) * h;     // 3h^2 for MHA
  const int64_t fc = (m.ffn_act == 1 ? 3 : 2) * h * F;                 // SwiGLU: gate, up, down
  return (qkv + h * h + fc) / P * (2 + 4) + 2 * h * (2 + 4);
}

pds_status make_plan(const pds_model& m, int P, int strategy, int64_t s, BufPlan* out) {
  if (P < 1) PDS_FAIL(PDS_EINVAL, "P must be >= 1");
  if (m.h <= 0 || m.n_heads <= 0 || m.ffn <= 0) PDS_FAIL(PDS_EINVAL, "model dims must be positive");
  if (m.batch < 1) PDS_FAIL(PDS_EINVAL, "batch must be >= 1");
  if (m.h % m.n_heads) PDS_FAIL(PDS_EDIVISIBILITY, "h not divisible by n_heads");
  const int64_t d = m.h / m.n_heads;
  if (d != 64 && d != 128) PDS_FAIL(PDS_ENOTIMPL, "head dim must be 64 or 128");
  if (m.h % 256) PDS_FAIL(PDS_ENOTIMPL, "h must be a multiple of 256");
  if (s <= 0 || s % P) PDS_FAIL(PDS_EDIVISIBILITY, "seq_len=" + std::to_string(s) + " not divisible by P=" + std::to_string(P));
  if (m.n_heads % P) PDS_FAIL(PDS_EDIVISIBILITY, "n_heads=" + std::to_string(m.n_heads) + " not divisible by P=" + std::to_string(P));
  if (m.ffn % P || (m.ffn / P) % 64) PDS_FAIL(PDS_EDIVISIBILITY, "ffn/P must be a multiple of 64");
  // Llama variant (R-GQA / R-SWIGLU)
  const int64_t nk = m.n_kv_heads > 0 ? m.n_kv_heads : m.n_heads;
  if (m.n_kv_heads < 0 || m.n_heads % nk) PDS_FAIL(PDS_EINVAL, "n_kv_heads must divide n_heads");
  if (nk % P) PDS_FAIL(PDS_EDIVISIBILITY, "n_kv_heads=" + std::to_string(nk) + " not divisible by P=" + std::to_string(P));
  if (m.ffn_act != 0 && m.ffn_act != 1) PDS_FAIL(PDS_EINVAL, "ffn_act must be 0 (GELU) or 1 (SwiGLU)");

  const int64_t sl = s / P;
  if (sl % 128) PDS_FAIL(PDS_EDIVISIBILITY, "s/P=" + std::to_string(sl) + " must be a multiple of 128 (caller pads, R-15)");
  const int64_t h = m.h, F = m.ffn, nl = m.n_heads / P, hl = h / P, Fl = F / P;
  // Q|K|V widths (local qw = 3 hl for MHA, full qwf = 3 h) and FC1 widths (f1w / f1wf =
  // Fl / F, doubled by SwiGLU's [gate | up])
  const int64_t qw = (nl + 2 * (nk / P)) * (h / m.n_heads), qwf = qw * P;
  const int64_t f1w = (m.ffn_act == 1 ? 2 : 1) * Fl, f1wf = f1w * P;
  const int64_t hkf = nk * (h / m.n_heads);          // all K (V) heads' width (MegatronCZ / ColossalZ)
  // token buffers hold rows = positions x b (layout [s, b, h], reading Q-35); the
  // divisibility checks above are on positions
  const int64_t S = s * m.batch, SL = sl * m.batch;
  const int64_t u = SL * h * 2, lam = nl * S * 4, ell = SL * 4;
  BufPlan p;
  int64_t ts = 0, tw = 0;
  const int64_t dgp = (int64_t)rmsnorm_bwd_grid(SL) * h * 4;
  // fused attention backward: turn counters per (local head, 128-query block) + ticket
  // (its fp32 dQ accumulator borrows a region that is free during the attention
  // backward: ta for TS / UZ, ul + vl for METP)
  const int64_t actr = (nl * (s / 128) + 1) * 4;
  // the attention backward's dS buffer (dS through HBM): measured slower than
  // the split kernels on B200, so the layer plans never reserve it (kDsMaxPos = 0); the
  // path stays selectable for the kernel-level entry point (pds_set_attn_bwd(2))
  const int64_t dsb = s <= kDsMaxPos ? attn_ds_bytes(s, (int)nl, (int)(nk / P), (int)(h / m.n_heads), m.causal,
                                                     kDsBudget) : 0;
  switch (strategy) {
    case PDS_MEGATRON_TS:
      push(p.saved, ts, "rstd1", ell);
      push(p.saved, ts, "qkv", S * qw * 2);
      push(p.saved, ts, "a", S * hl * 2);
      push(p.saved, ts, "lse", lam);
      push(p.saved, ts, "x1", u);
      push(p.saved, ts, "rstd2", ell);
      push(p.saved, ts, "h", S * f1w * 2);
      push(p.ws, tw, "gather", S * h * 2);
      push(p.ws, tw, "partial", S * h * 2);
      push(p.ws, tw, "f0", S * std::max(f1w, qw) * 2);       // G, dH^T, dQKV
      push(p.ws, tw, "f1", S * f1w * 2);                     // dH, dA
      push(p.ws, tw, "dd", lam);
      push(p.ws, tw, "dgp", dgp);
      push(p.ws, tw, "dgl", 2 * h * 4);
      push(p.ws, tw, "ta", std::max(Fl, qw) * S * 2);       // transposed operands (all GEMMs TN)
      push(p.ws, tw, "tb", h * S * 2);
      push(p.ws, tw, "wt", h * std::max(f1w, qw) * 2);
      push(p.ws, tw, "actr", actr);
      if (dsb) push(p.ws, tw, "dsb", dsb);                  // dS through HBM (attention bwd; never at kDsMaxPos = 0)
      if (P > 1) push(p.ws, tw, "gather2", S * h * 2);      // bwd re-gathers prefetched on the side stream
      break;
    case PDS_ULYSSES_Z: {
      const int64_t uq = SL * qwf * 2;            // a [s/P, Q|K|V of all heads] buffer (3u for MHA)
      push(p.saved, ts, "rstd1", ell);
      push(p.saved, ts, "qkv", S * qw * 2);
      push(p.saved, ts, "a", S * hl * 2);
      push(p.saved, ts, "lse", lam);
      push(p.saved, ts, "afull", u);
      push(p.saved, ts, "x1", u);
      push(p.saved, ts, "rstd2", ell);
      push(p.saved, ts, "h", SL * f1wf * 2);
      push(p.ws, tw, "wqkv", qwf * h * 2);
      push(p.ws, tw, "wproj", h * h * 2);
      push(p.ws, tw, "win", f1wf * h * 2);
      push(p.ws, tw, "wout", F * h * 2);
      push(p.ws, tw, "dw", std::max(qwf, f1wf) * h * 4);
      push(p.ws, tw, "u1", u);
      push(p.ws, tw, "s1", std::max(uq, u));
      push(p.ws, tw, "r1", std::max(uq, u));
      push(p.ws, tw, "f0", SL * f1wf * 2);
      push(p.ws, tw, "f1", SL * f1wf * 2);
      push(p.ws, tw, "x3", uq);
      push(p.ws, tw, "x4", uq);
      push(p.ws, tw, "v2", u);
      push(p.ws, tw, "dd", lam);
      push(p.ws, tw, "dgp", dgp);
      push(p.ws, tw, "dgl", 2 * h * 4);
      push(p.ws, tw, "ta", std::max(F, qwf) * SL * 2);
      push(p.ws, tw, "tb", h * SL * 2);
      push(p.ws, tw, "wt", h * std::max(f1wf, qwf) * 2);
      push(p.ws, tw, "actr", actr);
      if (dsb) push(p.ws, tw, "dsb", dsb);                  // dS through HBM (attention bwd; never at kDsMaxPos = 0)
      break;
    }
    case PDS_METP:
    case PDS_METP_FULL: {
      const int64_t c = m.metp_chunks > 0 ? m.metp_chunks : P;
      if (sl % c) PDS_FAIL(PDS_EDIVISIBILITY, "s/P not divisible by metp_chunks");
      const int64_t w = sl / c;
      if (w % 128) PDS_FAIL(PDS_EDIVISIBILITY, "s/(P*metp_chunks)=" + std::to_string(w) + " must be a multiple of 128");
      if (m.metp_recompute != 0 && m.metp_recompute != 1)
        PDS_FAIL(PDS_EINVAL, "metp_recompute must be 0 (ffn) or 1 (full)");
      // QKV recomputed in bwd, not saved
      const bool full = strategy == PDS_METP_FULL || m.metp_recompute == 1;
      const int64_t W = w * m.batch;               // rows of one wave per rank
      const int64_t uw = W * h * 2;
      push(p.saved, ts, "rstd1", ell);
      if (!full) push(p.saved, ts, "qkv", S * qw * 2);
      push(p.saved, ts, "a", S * hl * 2);
      push(p.saved, ts, "lse", lam);
      push(p.saved, ts, "x1", u);
      push(p.saved, ts, "rstd2", ell);
      push(p.ws, tw, "ul", u);
      push(p.ws, tw, "vl", u);
      push(p.ws, tw, "wg", P * uw);
      push(p.ws, tw, "wg2", P * uw);
      push(p.ws, tw, "pw", P * uw);
      push(p.ws, tw, "hw", P * W * f1w * 2);
      push(p.ws, tw, "gw", P * W * f1w * 2);              // G, dH^T
      push(p.ws, tw, "dhw", P * W * f1w * 2);
      push(p.ws, tw, "da", S * hl * 2);
      push(p.ws, tw, "dqkv", S * qw * 2);
      push(p.ws, tw, "dd", lam);
      push(p.ws, tw, "dgp", (int64_t)rmsnorm_bwd_grid(W) * h * 4);
      push(p.ws, tw, "dgl", 2 * h * 4);
      push(p.ws, tw, "ta", std::max(Fl, qw) * P * W * 2);
      push(p.ws, tw, "tb", h * P * W * 2);
      push(p.ws, tw, "wt", h * std::max(f1w, qw) * 2);
      push(p.ws, tw, "actr", actr);
      if (dsb) push(p.ws, tw, "dsb", dsb);                  // dS through HBM (attention bwd; never at kDsMaxPos = 0)
      if (full) push(p.ws, tw, "qkv", S * qw * 2);
      break;
    }
    case PDS_MEGATRON_CZ: {
      if ((sl / 2) % 128 || sl % 2)
        PDS_FAIL(PDS_EDIVISIBILITY, "MegatronCZ: s/(2P)=" + std::to_string(sl / 2) +
                                        " must be a multiple of 128 (zigzag half-chunks, R-CZ; caller pads)");
      // saved: the local rows of TS's tensors (Q/K/V of all heads, A, LSE, H); Q/K/V and
      // LSE on the zigzag rows
      push(p.saved, ts, "rstd1", ell);
      push(p.saved, ts, "qkv", SL * qwf * 2);
      push(p.saved, ts, "a", u);
      push(p.saved, ts, "lse", lam);
      push(p.saved, ts, "x1", u);
      push(p.saved, ts, "rstd2", ell);
      push(p.saved, ts, "h", SL * f1wf * 2);
      push(p.ws, tw, "wqkv", qwf * h * 2);      // [Q all; K all; V all] rows
      push(p.ws, tw, "wproj", h * h * 2);
      push(p.ws, tw, "win", f1wf * h * 2);
      push(p.ws, tw, "wout", F * h * 2);
      push(p.ws, tw, "dw", std::max(qwf, f1wf) * h * 4);
      push(p.ws, tw, "u1", u);
      // ring attention on the zigzag rows (R-CZ): O(u) per rank whatever P
      push(p.ws, tw, "qkvb", SL * qwf * 2);       // QKV of the boundary rows (bwd: dQKV)
      push(p.ws, tw, "kv0", SL * 2 * hkf * 2);    // the K/V block in hand / the next one
      push(p.ws, tw, "kv1", SL * 2 * hkf * 2);
      push(p.ws, tw, "acc", 2 * u);               // fp32 O accumulator (bwd: dQ)
      push(p.ws, tw, "dkv0", SL * 2 * hkf * 4);   // fp32 dK/dV travelling with their block
      push(p.ws, tw, "dkv1", SL * 2 * hkf * 4);
      push(p.ws, tw, "op", u);                    // a pair's partial O (bwd: zigzag dO)
      push(p.ws, tw, "oz", u);                    // zigzag O
      push(p.ws, tw, "lp", lam);                  // a pair's partial LSE
      push(p.ws, tw, "dqkvz", SL * qwf * 2);      // zigzag dQKV
      push(p.ws, tw, "f0", SL * f1wf * 2);
      push(p.ws, tw, "f1", SL * f1wf * 2);
      push(p.ws, tw, "v2", u);
      push(p.ws, tw, "da", u);
      push(p.ws, tw, "dd", lam);
      push(p.ws, tw, "dgp", dgp);
      push(p.ws, tw, "dgl", 2 * h * 4);
      push(p.ws, tw, "ta", std::max(qwf, F) * SL * 2);
      push(p.ws, tw, "tb", h * SL * 2);
      push(p.ws, tw, "wt", h * std::max(qwf, f1wf) * 2);
      break;
    }
    case PDS_COLOSSAL_Z: {
      // saved: TS's local-row tensors without LSE, plus the softmax probabilities of the
      // own rows against every key, [b][n][s/P][s] bf16 (Ring Self-Attention, R-COL)
      const int64_t n = m.n_heads;
      const int64_t quad = n * sl * s * m.batch;       // elements of [b][n][s/P][s]
      push(p.saved, ts, "rstd1", ell);
      push(p.saved, ts, "qkv", SL * qwf * 2);
      push(p.saved, ts, "a", u);
      push(p.saved, ts, "probs", quad * 2);
      push(p.saved, ts, "x1", u);
      push(p.saved, ts, "rstd2", ell);
      push(p.saved, ts, "h", SL * f1wf * 2);
      push(p.ws, tw, "wqkv", qwf * h * 2);
      push(p.ws, tw, "wproj", h * h * 2);
      push(p.ws, tw, "win", f1wf * h * 2);
      push(p.ws, tw, "wout", F * h * 2);
      push(p.ws, tw, "dw", std::max(qwf, f1wf) * h * 4);
      push(p.ws, tw, "u1", u);
      push(p.ws, tw, "scores", quad * 4);          // fp32 scores (bwd: dP)
      push(p.ws, tw, "ds", quad * 2);              // bf16 dS (bwd)
      push(p.ws, tw, "kr0", SL * hkf * 2);         // the K (or V) block in hand / the next one
      push(p.ws, tw, "kr1", SL * hkf * 2);
      push(p.ws, tw, "acc", 2 * u);                // fp32 O (bwd: dQ)
      push(p.ws, tw, "dacc0", SL * hkf * 4);       // fp32 dV / dK travelling with their block
      push(p.ws, tw, "dacc1", SL * hkf * 4);
      push(p.ws, tw, "dqkv", SL * qwf * 2);
      push(p.ws, tw, "f0", SL * f1wf * 2);
      push(p.ws, tw, "f1", SL * f1wf * 2);
      push(p.ws, tw, "v2", u);
      push(p.ws, tw, "da", u);
      push(p.ws, tw, "dd", lam);
      push(p.ws, tw, "dgp", dgp);
      push(p.ws, tw, "dgl", 2 * h * 4);
      push(p.ws, tw, "ta", std::max(qwf, F) * SL * 2);
      push(p.ws, tw, "tb", h * SL * 2);
      push(p.ws, tw, "wt", h * std::max(qwf, f1wf) * 2);
      break;
    }
    default:
      PDS_FAIL(PDS_ESTRATEGY, "unknown strategy id " + std::to_string(strategy));
  }
  p.saved_bytes = ts;
  p.ws_bytes = tw;
  *out = p;
  return PDS_OK;
}

}  // namespace pds

// ------------------------------------------------------------------ C ABI (host only)
using namespace pds;

extern "C" const char* pds_last_error(void) { return g_err.c_str(); }
extern "C" const char* pds_version(void) { return "paradyse-b200 0.1 (sm_100a)"; }

extern "C" pds_status pds_plan_ex(int32_t L, int32_t n_strat, const double* t_layer,
                                  const double* m_layer, const double* w_layer, const uint8_t* enabled, double capacity,
                                  double gamma, const uint8_t* prev_plan, uint8_t* strategy_out,
                                  uint32_t* flags_out, int64_t* counters_out) {
  if (L <= 0) PDS_FAIL(PDS_EINVAL, "L must be >= 1 (SPEC.md:394)");
  if (n_strat <= 0 || n_strat > 255) PDS_FAIL(PDS_EINVAL, "n_strat out of range");
  if (!t_layer || !m_layer || !enabled || !strategy_out) PDS_FAIL(PDS_EINVAL, "NULL argument");
  bool any = false;
  for (int i = 0; i < n_strat; ++i) any |= enabled[i] != 0;
  if (!any) PDS_FAIL(PDS_ESTRATEGY, "no enabled strategy");
  Alg1Counters c;
  std::vector<uint8_t> out;
  bool inf = false, early = false;
  alg1(L, n_strat, t_layer, m_layer, w_layer, enabled, capacity, out, &inf, &early, &c);
  uint32_t flags = (inf ? PDS_PLAN_INFEASIBLE : 0u) | (early ? PDS_PLAN_EARLY : 0u);
  if (prev_plan) {
    bool valid = true, same = true;
    for (int l = 0; l < L; ++l) {
      if (prev_plan[l] >= n_strat || !enabled[prev_plan[l]]) valid = false;
      else if (prev_plan[l] != out[l]) same = false;
    }
    if (valid && !same && plan_feasible(prev_plan, L, m_layer, w_layer, capacity, nullptr) &&
        plan_time(prev_plan, L, t_layer) <= (1.0 + gamma) * plan_time(out.data(), L, t_layer)) {
      std::memcpy(out.data(), prev_plan, (size_t)L);
      flags |= PDS_PLAN_SMOOTHED;
      flags &= ~PDS_PLAN_INFEASIBLE;
    }
  }
  std::memcpy(strategy_out, out.data(), (size_t)L);
  if (flags_out) *flags_out = flags;
  if (counters_out) {
    counters_out[0] = c.layer_checks;
    counters_out[1] = c.plans;
    counters_out[2] = c.cache_hits;
  }
  return PDS_OK;
}

extern "C" pds_status pds_mem_bytes(const pds_model* model, int32_t P, uint8_t strategy,
                                    int64_t seq_len, int64_t* saved_per_layer,
                                    int64_t* transient_peak, int64_t* persistent_per_layer) {
  if (!model) PDS_FAIL(PDS_EINVAL, "NULL model");
  BufPlan p;
  PDS_TRY(make_plan(*model, P, strategy, seq_len, &p));
  // saved per layer = ctx-owned saved arena + the retained layer input x (caller-owned)
  const int64_t x_bytes = seq_len / P * model->batch * model->h * 2;
  if (saved_per_layer) *saved_per_layer = p.saved_bytes + x_bytes;
  if (transient_peak) *transient_peak = p.ws_bytes;
  if (persistent_per_layer) *persistent_per_layer = persistent_bytes(*model, P);
  return PDS_OK;
}
