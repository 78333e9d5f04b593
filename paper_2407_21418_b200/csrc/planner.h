// planner.h — C++17 tuner core, bit-exact with mktune 0.1.0 (L1-L5):
// enumeration (ukernel.py), analytic metrics (metrics.py), the filter chain
// and relaxation ladder (filtering.py), composition (combine.py) and SIA
// ranking (scoring.py). Integer metrics are exact int64; the float64
// quantities follow numpy's operation order (compile with -ffp-contract=off).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/ftb.h"

namespace ftb {
namespace plan {

struct Frac {
  int64_t n = 0, d = 1;
  static Frac make(int64_t n, int64_t d);
  bool operator==(const Frac& o) const { return n == o.n && d == o.d; }
  bool operator<(const Frac& o) const;
};
Frac operator-(const Frac& a, const Frac& b);
Frac operator*(int64_t k, const Frac& a);

struct Sweep {
  Frac eps_min, eps_max, lam_min, lam_max, eps_step, lam_step;
  int64_t num_steps() const;            // filtering.py:98-103
  Sweep widened(int64_t strides) const; // filtering.py:112-118
  bool operator==(const Sweep& o) const;
};

struct Instance {
  int ns = 0, nr = 0;
  int major = 0;
  std::vector<std::vector<int>> inputs;  // axis indices per input access
  int64_t elem = 4, fpp = 2;
  int64_t ext[FTB_MAX_AXES] = {};
  bool dynamic[FTB_MAX_AXES] = {};
  std::string name[FTB_MAX_AXES];
  int na() const { return ns + nr; }
  int64_t flops() const;
  static Instance from_c(const ftb_instance& c);
};

struct Hw {
  int64_t cores, regs, smem, bw_g, bw_s, peak, zeta, active, align;
  int legality;       // 0 parity, 1 tcgen05 legality (B200 mode)
  int relax_tau = -1; // B200 fallback: space axis whose tile is relaxed
  int relax_level = 2; // 1: tau tile may be any wide MMA N (multiple of 2 * n_step in [n_max / 2, n_max]); 2: any size <= n_max
  // tcgen05 legality parameters (ftb_hw; the sm_100a values by default)
  int64_t tmem_cols = 512, m_max = 128, n_step = 16, n_max = 256, swizzle = 128;
  static Hw from_c(const ftb_hw& h);
};

struct Params {
  Sweep sweep;
  double psi = 1.0;
  int64_t rest_regs = 24;
  int64_t cap = int64_t(1) << 21;
  static Params from_c(const ftb_params& p);
};

// Columnar candidate table + cached metric columns.
struct Cands {
  Instance inst;
  int ns = 0, na = 0;
  std::vector<int64_t> reg, smem;  // n*ns, n*na
  // integer metric columns (metrics.py:155-191) and filter state
  std::vector<int64_t> pad_num, pad_den, blocks, occ_den, regs_in_block, retained;
  std::vector<uint8_t> saturated;
  std::vector<double> cmr, kmem;
  // cached part metrics used by ranking (UKernel fields, ukernel.py:55-57)
  std::vector<double> m_pad, m_occ, m_cmr;
  bool has_metrics = false;
  size_t size() const { return ns ? reg.size() / ns : 0; }
  const int64_t* reg_row(size_t i) const { return &reg[i * ns]; }
  const int64_t* smem_row(size_t i) const { return &smem[i * na]; }
};

struct Report {
  int64_t n_align = 0, n_cross = 0, n_filter = 0, n_final = 0;
  int relaxation = FTB_RELAX_NONE;
  int widen = 0;
  bool truncated = false;
  int tau = 0;
  int stage = 0;
  Sweep used;
};

// Pool entry: nparts, rows and counts (rows index the candidate table).
struct PlanRow {
  int32_t nparts;
  int64_t ra, na_, rb, nb;
};

Cands enumerate(const Instance& in, const Hw& hw, int64_t cap, bool* truncated);
// enumerate + (B200 mode) the tcgen05 legality filter
Cands enumerate_legal(const Instance& in, const Hw& hw, int64_t cap, bool* truncated);
// stage selects the returned set: 0 final (reference), 1 filter, 2 cross, 3 align
// (1-3 are the B200-mode fallback rungs used when the final set cannot cover tau).
Cands compile_shape(const Instance& in, const Hw& hw, const Params& p, Report* rep, int stage = 0);
int select_main_axis(const Instance& in);
int64_t pool_count(const Cands& c, int tau);
std::vector<PlanRow> pool_export(const Cands& c, int tau);
// Top-k with scores; normalize = per-pool min-max (scoring.py:98-112).
std::vector<std::pair<PlanRow, double>> rank_topk(const Cands& c, int tau, const ftb_coeffs& co,
                                                  int k, bool normalize);
// B200 legality predicate (extension; parity mode never calls it).
bool tcgen05_legal(const Instance& in, const Hw& hw, const int64_t* smem, int relax_tau = -1, int relax_level = 2);

}  // namespace plan
}  // namespace ftb
