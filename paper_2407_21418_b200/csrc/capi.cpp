// capi.cpp — extern "C" surface of the planner (include/ftb.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "planner.h"
#include "status.h"

using namespace ftb;
using namespace ftb::plan;

struct ftb_cands {
  Cands c;
};

static void fill_report(const Report& r, double secs, ftb_compile_report* out) {
  if (!out) return;
  out->n_align = r.n_align;
  out->n_cross = r.n_cross;
  out->n_filter = r.n_filter;
  out->n_final = r.n_final;
  out->relaxation = r.relaxation;
  out->widen = r.widen;
  out->truncated = r.truncated;
  out->tau = r.tau;
  const Frac f[6] = {r.used.eps_min, r.used.eps_max, r.used.lam_min,
                     r.used.lam_max, r.used.eps_step, r.used.lam_step};
  for (int i = 0; i < 6; ++i) out->sweep_used[i] = {f[i].n, f[i].d};
  out->stage = r.stage;
  out->seconds = secs;
}

static void fill_program(const Cands& c, int tau, const PlanRow& row, double sia, ftb_program* g) {
  std::memset(g, 0, sizeof(*g));
  g->n_space = c.ns;
  g->n_reduce = c.na - c.ns;
  g->tau = tau;
  g->n_parts = row.nparts;
  const int64_t rows[2] = {row.ra, row.rb};
  const int64_t cnt[2] = {row.na_, row.nb};
  for (int p = 0; p < row.nparts; ++p) {
    for (int s = 0; s < c.ns; ++s) g->reg[p][s] = c.reg_row(rows[p])[s];
    for (int a = 0; a < c.na; ++a) g->smem[p][a] = c.smem_row(rows[p])[a];
    g->count[p] = cnt[p];
  }
  g->sia = sia;
}

static inline double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" {

ftb_status ftb_enumerate(const ftb_hw* hw, const ftb_instance* inst, int64_t cap, ftb_cands** out,
                         int32_t* truncated) {
  return guarded([&] {
    if (!hw || !inst || !out) throw input_error("null argument");
    Instance in = Instance::from_c(*inst);
    Hw h = Hw::from_c(*hw);
    bool tr = false;
    auto* r = new ftb_cands{enumerate_legal(in, h, cap, &tr)};
    if (truncated) *truncated = tr;
    *out = r;
  });
}

ftb_status ftb_compile_shape(const ftb_hw* hw, const ftb_instance* inst, const ftb_params* p,
                             ftb_cands** out, ftb_compile_report* rep) {
  return guarded([&] {
    if (!hw || !inst || !p || !out) throw input_error("null argument");
    auto t0 = std::chrono::steady_clock::now();
    Instance in = Instance::from_c(*inst);
    Hw h = Hw::from_c(*hw);
    Params q = Params::from_c(*p);
    Report r;
    auto* res = new ftb_cands{compile_shape(in, h, q, &r)};
    fill_report(r, secs_since(t0), rep);
    *out = res;
  });
}

ftb_status ftb_cands_from_arrays(const ftb_instance* inst, int64_t n, const int64_t* reg,
                                 const int64_t* smem, const double* pad, const double* occ,
                                 const double* cmr, ftb_cands** out) {
  return guarded([&] {
    if (!inst || !out || (n > 0 && (!reg || !smem))) throw input_error("null argument");
    Instance in = Instance::from_c(*inst);
    auto* r = new ftb_cands();
    Cands& c = r->c;
    c.inst = in;
    c.ns = in.ns;
    c.na = in.na();
    c.reg.assign(reg, reg + n * c.ns);
    c.smem.assign(smem, smem + n * c.na);
    c.m_pad.assign(n, NAN);
    c.m_occ.assign(n, NAN);
    c.m_cmr.assign(n, NAN);
    for (int64_t i = 0; i < n; ++i) {
      if (pad) c.m_pad[i] = pad[i];
      if (occ) c.m_occ[i] = occ[i];
      if (cmr) c.m_cmr[i] = cmr[i];
    }
    c.has_metrics = true;  // per-row NaN marks missing metrics
    *out = r;
  });
}

int64_t ftb_cands_size(const ftb_cands* c) { return c ? static_cast<int64_t>(c->c.size()) : 0; }

ftb_status ftb_cands_export(const ftb_cands* cs, int64_t* reg, int64_t* smem, int64_t* icol,
                            double* fcol) {
  return guarded([&] {
    if (!cs) throw input_error("null argument");
    const Cands& c = cs->c;
    const size_t n = c.size();
    if (reg) std::copy(c.reg.begin(), c.reg.end(), reg);
    if (smem) std::copy(c.smem.begin(), c.smem.end(), smem);
    if (icol) {
      if (c.pad_num.size() != n) throw FtbError(FTB_MISSING_METRICS, "metric columns have not been computed");
      for (size_t i = 0; i < n; ++i) {
        int64_t* o = icol + 7 * i;
        o[0] = c.pad_num[i]; o[1] = c.pad_den[i]; o[2] = c.blocks[i]; o[3] = c.occ_den[i];
        o[4] = c.regs_in_block[i]; o[5] = c.saturated[i]; o[6] = c.retained.empty() ? 0 : c.retained[i];
      }
    }
    if (fcol) {
      if (c.cmr.size() != n) throw FtbError(FTB_MISSING_METRICS, "metric columns have not been computed");
      for (size_t i = 0; i < n; ++i) {
        fcol[2 * i] = c.cmr[i];
        fcol[2 * i + 1] = c.kmem[i];
      }
    }
  });
}

void ftb_cands_destroy(ftb_cands* c) { delete c; }

ftb_status ftb_select_main_axis(const ftb_instance* inst, int32_t* tau) {
  return guarded([&] {
    if (!inst || !tau) throw input_error("null argument");
    *tau = select_main_axis(Instance::from_c(*inst));
  });
}

ftb_status ftb_pool_count(const ftb_cands* c, int32_t tau, int64_t* n) {
  return guarded([&] {
    if (!c || !n) throw input_error("null argument");
    if (tau < 0 || tau >= c->c.ns) throw input_error("tau is not a space axis", "tau");
    *n = pool_count(c->c, tau);
  });
}

ftb_status ftb_pool_export(const ftb_cands* c, int32_t tau, int64_t cap, int64_t* rows, int64_t* n) {
  return guarded([&] {
    if (!c || !n) throw input_error("null argument");
    if (tau < 0 || tau >= c->c.ns) throw input_error("tau is not a space axis", "tau");
    if (c->c.size() == 0)
      throw FtbError(FTB_EMPTY_RESULT, "candidate set is empty", "candidate set");
    auto pool = pool_export(c->c, tau);
    *n = static_cast<int64_t>(pool.size());
    if (rows)
      for (int64_t i = 0; i < std::min<int64_t>(cap, *n); ++i) {
        int64_t* o = rows + 5 * i;
        o[0] = pool[i].nparts; o[1] = pool[i].ra; o[2] = pool[i].na_; o[3] = pool[i].rb; o[4] = pool[i].nb;
      }
  });
}

ftb_status ftb_rank_topk(const ftb_cands* c, int32_t tau, const ftb_coeffs* coeffs, int32_t k,
                         int32_t normalize, int64_t* rows, double* scores, int32_t* n_out) {
  return guarded([&] {
    if (!c || !coeffs || !n_out) throw input_error("null argument");
    if (tau < 0 || tau >= c->c.ns) throw input_error("tau is not a space axis", "tau");
    if (c->c.size() == 0)
      throw FtbError(FTB_EMPTY_RESULT, "candidate set is empty", "candidate set");
    auto top = rank_topk(c->c, tau, *coeffs, k, normalize != 0);
    *n_out = static_cast<int32_t>(top.size());
    for (size_t i = 0; i < top.size(); ++i) {
      if (rows) {
        int64_t* o = rows + 5 * i;
        const PlanRow& p = top[i].first;
        o[0] = p.nparts; o[1] = p.ra; o[2] = p.na_; o[3] = p.rb; o[4] = p.nb;
      }
      if (scores) scores[i] = top[i].second;
    }
  });
}

ftb_status ftb_plan_batch(const ftb_hw* hw, const ftb_instance* insts, int32_t n, const ftb_params* p,
                          const ftb_coeffs* coeffs, int32_t threads, ftb_program* out,
                          ftb_compile_report* reps, ftb_status* statuses) {
  return guarded([&] {
    if (!hw || !insts || !p || !coeffs || !out || n < 0) throw input_error("null argument");
    const Hw h = Hw::from_c(*hw);
    const Params q = Params::from_c(*p);
    int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    nt = std::max(1, std::min(nt, n));
    std::vector<ftb_status> st(n, FTB_OK);
    std::vector<std::string> msgs(n);
    auto work = [&](int tid) {
      for (int i = tid; i < n; i += nt) {
        auto t0 = std::chrono::steady_clock::now();
        try {
          Instance in = Instance::from_c(insts[i]);
          Report r;
          // Parity mode ranks the final set only (an empty pool raises, as
          // combine.py:183-188 does). B200 mode walks a documented fallback
          // ladder when no combination covers tau: ranked set final -> filter
          // -> cross -> align; for a Dense, then the same with the other output
          // axis as the composition axis (its extent may be a multiple of the
          // strict 256-column tile when the main axis is not); then with the
          // main-axis tile relaxed, first to any wide MMA N (multiple of 32 in
          // [128, 256]), then to any size <= 256 (padded inside the MMA tile);
          // then parity mode. Reported stage = set index + 4 * rung.
          struct Rung { int legality, relax, level, tau; };
          std::vector<Rung> rungs;
          if (h.legality) {
            const int tau = select_main_axis(in);
            rungs = {{1, -1, 0, -1}};
            if (in.ns == 2) rungs.push_back({1, -1, 0, 1 - tau});
            rungs.insert(rungs.end(), {{1, tau, 1, -1}, {1, tau, 2, -1}, {0, -1, 0, -1}});
          } else {
            rungs = {{0, -1, 0, -1}};
          }
          bool done = false;
          for (size_t ri = 0; ri < rungs.size() && !done; ++ri) {
            Hw hq = h;
            hq.legality = rungs[ri].legality;
            hq.relax_tau = rungs[ri].relax;
            hq.relax_level = rungs[ri].level;
            const int last = h.legality ? 3 : 0;
            for (int stage = 0; stage <= last && !done; ++stage) {
              try {
                Cands c = compile_shape(in, hq, q, &r, stage);
                if (rungs[ri].tau >= 0) r.tau = rungs[ri].tau;
                auto top = rank_topk(c, r.tau, *coeffs, 1, false);
                if (top.empty()) throw FtbError(FTB_EMPTY_RESULT, "empty program pool", "program pool");
                fill_program(c, r.tau, top[0].first, top[0].second, &out[i]);
                r.stage = stage + 4 * static_cast<int>(ri);
                done = true;
              } catch (const FtbError& e) {
                const bool last_try = (ri + 1 == rungs.size()) && stage == last;
                if (e.code != FTB_EMPTY_RESULT || last_try) throw;
              }
            }
          }
          fill_report(r, secs_since(t0), reps ? &reps[i] : nullptr);
        } catch (const FtbError& e) {
          st[i] = e.code;
          msgs[i] = e.what();
        } catch (const std::exception& e) {
          st[i] = FTB_INTERNAL_ERROR;
          msgs[i] = e.what();
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    ftb_status first = FTB_OK;
    std::string first_msg;
    for (int i = 0; i < n; ++i) {
      if (statuses) statuses[i] = st[i];
      if (st[i] != FTB_OK && first == FTB_OK) first = st[i], first_msg = msgs[i];
    }
    if (first != FTB_OK && !statuses) throw FtbError(first, "shape failed: " + first_msg);
  });
}

}  // extern "C"
