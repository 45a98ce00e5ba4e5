// Internal declarations of the ParaDySe C-ABI library (not part of the ABI).
#pragma once
#include <cstring>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/paradyse.h"

namespace pds {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
#define PDS_FAIL(code, msg)          \
  do {                               \
    ::pds::set_error(msg);           \
    return (code);                   \
  } while (0)
#define PDS_CUDA(expr)                                                              \
  do {                                                                              \
    cudaError_t e__ = (cudaError_t)(expr);                                          \
    if (e__ != cudaSuccess) {                                                       \
      cudaGetLastError(); /* a failed call must not resurface in a later check */  \
      ::pds::set_error(std::string(#expr) + ": " + cudaGetErrorString(e__));        \
      return e__ == cudaErrorMemoryAllocation ? PDS_ENOMEM : PDS_ECUDA;             \
    }                                                                               \
  } while (0)
#define PDS_TRY(expr)                 \
  do {                                \
    pds_status s__ = (expr);          \
    if (s__ != PDS_OK) return s__;    \
  } while (0)

// ------------------------------------------------------------------ memory plan
// The exact per-rank byte plan of the CUDA path.  The
// allocator and pds_mem_bytes both read it, so the model is exact by construction.
constexpr int64_t kAlign = 256;
// attention backward with dS through HBM: at most this many bytes of dS
// workspace (kernel-level entry, pds_set_attn_bwd(2)); the layer plans use it up to
// kDsMaxPos positions — 0: never (measured slower than the split kernels)
constexpr int64_t kDsBudget = (int64_t)8 << 30;
constexpr int64_t kDsMaxPos = 0;
inline int64_t al(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Region {
  const char* name;
  int64_t bytes;
  int64_t off;
};

struct BufPlan {
  std::vector<Region> saved;  // ctx saved arena (per layer)
  std::vector<Region> ws;     // workspace (per call)
  int64_t saved_bytes = 0;    // aligned sum (ctx-owned)
  int64_t ws_bytes = 0;
  int64_t off(const std::vector<Region>& v, const char* n) const;
  int64_t saved_off(const char* n) const { return off(saved, n); }
  int64_t ws_off(const char* n) const { return off(ws, n); }
  bool has_ws(const char* n) const {
    for (const Region& r : ws)
      if (std::strcmp(r.name, n) == 0) return true;
    return false;
  }
  int64_t ws_size(const char* n) const {
    for (const Region& r : ws)
      if (std::strcmp(r.name, n) == 0) return r.bytes;
    return 0;
  }
};

int rmsnorm_bwd_grid(int64_t rows);

// returns PDS_OK or PDS_EDIVISIBILITY / PDS_ESTRATEGY / PDS_EINVAL with message
pds_status make_plan(const pds_model& m, int P, int strategy, int64_t s, BufPlan* out);
int64_t persistent_bytes(const pds_model& m, int P);

// ------------------------------------------------------------------ planner core
struct Alg1Counters {
  int64_t layer_checks = 0, plans = 0, cache_hits = 0;
};
// Algorithm 1 on explicit costs; returns infeasible flag via *infeasible
// w: per-strategy workspace bytes (one workspace per plan: max over its strategies,
// reading R-22); NULL = none
void alg1(int L, int n, const double* t, const double* m, const double* w, const uint8_t* enabled, double cap,
          std::vector<uint8_t>& out, bool* infeasible, bool* early, Alg1Counters* c);
bool plan_feasible(const uint8_t* plan, int L, const double* m, const double* w, double cap, Alg1Counters* c);
double plan_time(const uint8_t* plan, int L, const double* t);

// ------------------------------------------------------------------ cost bundle
struct Tree {
  std::vector<int32_t> feature, left, right;
  std::vector<double> threshold, value;
};
struct StratCost {
  bool present = false;
  double s_profile_max = 0;
  int poly_deg = 0;
  double poly_scale = 1;
  std::vector<double> poly_coef;
  std::vector<Tree> trees;
};
struct Bundle {
  bool loaded = false;
  int P = 0, h = 0, n = 0, ffn = 0, L = 0;
  int n_kv = 0, act = 0;          // Llama variant (0 = n heads, GELU)
  double capacity = 0, reserve = 0;
  double norm[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  StratCost strat[PDS_N_STRATEGIES];
};
pds_status load_bundle(const char* path, Bundle* b);
double bundle_time(const Bundle& b, int strategy, int64_t s, int* branch);

}  // namespace pds
