// planner.cpp — bit-exact C++ port of the mktune tuner core with a streaming
// Top-K ranker. See planner.h. Citations are to /root/reference/pkg/src/mktune.
#include "planner.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <thread>
#include <unordered_map>

#include "status.h"

namespace ftb {
namespace plan {

// ------------------------------------------------------------------ helpers

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }  // a,b > 0
// Python floor division / ceil division for signed numerators, positive den.
static inline int64_t py_floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
static inline int64_t py_ceildiv(int64_t a, int64_t b) { return -py_floordiv(-a, b); }
static constexpr int64_t _MAX_WIDEN = 2000;  // filtering.py:267

Frac Frac::make(int64_t n, int64_t d) {
  if (d == 0) throw input_error("zero denominator in sweep parameter");
  if (d < 0) { n = -n; d = -d; }
  int64_t g = std::gcd(n < 0 ? -n : n, d);
  if (g == 0) g = 1;
  Frac f;
  f.n = n / g;
  f.d = d / g;
  return f;
}
bool Frac::operator<(const Frac& o) const {
  return static_cast<__int128>(n) * o.d < static_cast<__int128>(o.n) * d;
}
Frac operator-(const Frac& a, const Frac& b) { return Frac::make(a.n * b.d - b.n * a.d, a.d * b.d); }
Frac operator*(int64_t k, const Frac& a) { return Frac::make(k * a.n, a.d); }
static int64_t frac_trunc_div(const Frac& a, const Frac& b) {  // int(a / b), toward zero
  __int128 num = static_cast<__int128>(a.n) * b.d, den = static_cast<__int128>(a.d) * b.n;
  return static_cast<int64_t>(num / den);
}

int64_t Sweep::num_steps() const {
  return 1 + std::min(frac_trunc_div(eps_max - eps_min, eps_step),
                      frac_trunc_div(lam_max - lam_min, lam_step));
}
Sweep Sweep::widened(int64_t k) const {
  Sweep s = *this;
  const Frac zero = Frac::make(0, 1);
  Frac e = eps_min - k * eps_step, l = lam_min - k * lam_step;
  s.eps_min = e < zero ? zero : e;
  s.lam_min = l < zero ? zero : l;
  return s;
}
bool Sweep::operator==(const Sweep& o) const {
  return eps_min == o.eps_min && eps_max == o.eps_max && lam_min == o.lam_min &&
         lam_max == o.lam_max && eps_step == o.eps_step && lam_step == o.lam_step;
}

int64_t Instance::flops() const {  // workload.py:280-285
  int64_t f = fpp;
  for (int a = 0; a < na(); ++a) f *= ext[a];
  return f;
}

Instance Instance::from_c(const ftb_instance& c) {
  Instance in;
  if (c.n_space < 1 || c.n_reduce < 1 || c.n_space + c.n_reduce > FTB_MAX_AXES)
    throw input_error("operator needs at least one space and one reduce axis", "axes");
  in.ns = c.n_space;
  in.nr = c.n_reduce;
  if (c.major < 0 || c.major >= c.n_space) throw input_error("major axis is not a space axis", "major_axis");
  in.major = c.major;
  if (c.n_inputs < 1 || c.n_inputs > FTB_MAX_INPUTS) throw input_error("bad input access count", "accesses");
  for (int i = 0; i < c.n_inputs; ++i) {
    std::vector<int> axes;
    for (int a = 0; a < c.input_naxes[i]; ++a) {
      int ax = c.input_axes[i][a];
      if (ax < 0 || ax >= in.na()) throw input_error("access references an unknown axis", "axes");
      axes.push_back(ax);
    }
    in.inputs.push_back(axes);
  }
  if (c.elem_bytes < 1) throw input_error("elem_bytes must be >= 1", "elem_bytes");
  if (c.flops_per_point < 1) throw input_error("flops_per_point must be >= 1", "flops_per_point");
  in.elem = c.elem_bytes;
  in.fpp = c.flops_per_point;
  for (int a = 0; a < in.na(); ++a) {
    if (c.extent[a] < 1) throw input_error("axis extent must be >= 1", "extent");
    in.ext[a] = c.extent[a];
    in.dynamic[a] = c.dynamic[a] != 0;
    char buf[17];
    std::memcpy(buf, c.axis_name[a], 16);
    buf[16] = '\0';
    in.name[a] = buf;
  }
  return in;
}

Hw Hw::from_c(const ftb_hw& h) {
  Hw w{h.num_cores, h.regs_per_core, h.smem_per_core_bytes, h.global_bw_bytes_per_s,
       h.shared_bw_bytes_per_s, h.peak_flops, h.default_active_blocks, h.active_blocks_per_core,
       h.align_elems, h.legality};
  const int64_t v[9] = {w.cores, w.regs, w.smem, w.bw_g, w.bw_s, w.peak, w.zeta, w.active, w.align};
  static const char* names[9] = {"num_cores", "regs_per_core", "smem_per_core_bytes",
                                 "global_bw_bytes_per_s", "shared_bw_bytes_per_s", "peak_flops",
                                 "default_active_blocks", "active_blocks_per_core", "align_elems"};
  for (int i = 0; i < 9; ++i)  // hardware.py:50-61
    if (v[i] <= 0) throw input_error(std::string("descriptor field '") + names[i] + "' must be strictly positive", names[i]);
  if (w.align & (w.align - 1)) throw input_error("descriptor field 'align_elems' must be a power of two", "align_elems");
  if (w.legality) {
    auto pick = [](int64_t v, int64_t dflt) { return v > 0 ? v : dflt; };
    w.tmem_cols = pick(h.tmem_columns, 512);
    w.m_max = pick(h.mma_m_max, 128);
    w.n_step = pick(h.mma_n_step, 16);
    w.n_max = pick(h.mma_n_max, 256);
    w.swizzle = pick(h.tma_swizzle_bytes, 128);
    if (w.m_max != 64 && w.m_max != 128) throw input_error("mma_m_atoms: the largest M must be 64 or 128", "mma_m_atoms");
    if (w.n_step != 8 && w.n_step != 16) throw input_error("mma_n_step must be 8 or 16", "mma_n_step");
    if (w.n_max < 2 * w.n_step || w.n_max > 256 || w.n_max % w.n_step)
      throw input_error("mma_n_max must be a multiple of mma_n_step in [2 * step, 256]", "mma_n_max");
    if (w.tmem_cols & (w.tmem_cols - 1) || w.tmem_cols < 2 * w.n_max || w.tmem_cols > 512)
      throw input_error("tmem_columns must be a power of two in [2 * mma_n_max, 512]", "tmem_columns");
    if (w.swizzle != 32 && w.swizzle != 64 && w.swizzle != 128)
      throw input_error("tma_swizzle_bytes must be 32, 64 or 128", "tma_swizzle_bytes");
  }
  return w;
}

Params Params::from_c(const ftb_params& p) {
  Params q;
  q.sweep.eps_min = Frac::make(p.eps_min.num, p.eps_min.den);
  q.sweep.eps_max = Frac::make(p.eps_max.num, p.eps_max.den);
  q.sweep.lam_min = Frac::make(p.lam_min.num, p.lam_min.den);
  q.sweep.lam_max = Frac::make(p.lam_max.num, p.lam_max.den);
  q.sweep.eps_step = Frac::make(p.eps_step.num, p.eps_step.den);
  q.sweep.lam_step = Frac::make(p.lam_step.num, p.lam_step.den);
  q.psi = p.psi;
  q.rest_regs = p.rest_regs;
  q.cap = p.candidate_cap;
  return q;
}

// ------------------------------------------------------------------ enumeration (ukernel.py)

static std::vector<int64_t> divisors(int64_t n) {  // ukernel.py:67-79
  std::vector<int64_t> lo, hi;
  for (int64_t d = 1; d * d <= n; ++d)
    if (n % d == 0) {
      lo.push_back(d);
      if (d != n / d) hi.push_back(n / d);
    }
  lo.insert(lo.end(), hi.rbegin(), hi.rend());
  return lo;
}
static bool is_prime(int64_t n) {  // ukernel.py:82-90
  if (n < 2) return false;
  for (int64_t d = 2; d * d <= n; ++d)
    if (n % d == 0) return false;
  return true;
}
static std::vector<int64_t> reg_tile_candidates(int64_t e, int64_t align) {  // ukernel.py:98-110
  std::vector<int64_t> v = divisors(e);
  if (e > align && is_prime(e)) {
    auto a = divisors(e - 1), b = divisors(e + 1);
    v.insert(v.end(), a.begin(), a.end());
    v.insert(v.end(), b.begin(), b.end());
  }
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}
static std::vector<int64_t> space_options(int64_t e, int64_t r, int64_t align, bool major) {
  const int64_t step = major ? std::lcm(r, align) : r;  // ukernel.py:113-121
  std::vector<int64_t> v;
  const int64_t cnt = cdiv(e, step);
  v.reserve(cnt);
  for (int64_t m = 1; m <= cnt; ++m) v.push_back(step * m);
  return v;
}
static std::vector<int64_t> reduce_options(int64_t e, int64_t align) {  // ukernel.py:124-133
  if (e < align) return {align};
  std::vector<int64_t> v;
  for (int64_t t = align; t <= (e / align) * align; t += align) v.push_back(t);
  return v;
}

bool tcgen05_legal(const Instance& in, const Hw& hw, const int64_t* smem, int relax_tau, int relax_level) {
  // B200 extension: the uKernel's output tile must map onto efficient
  // tcgen05 tiles in one of the two orientations — everything below derives
  // from the descriptor's tcgen05 fields (sm_100a: M atoms up to 128 TMEM
  // lanes, N up to 256 columns, 512 TMEM columns, 128-B TMA swizzle):
  //   lanes  : whole MMA M slabs (m_max, or two of them), or a tile spanning
  //            a short axis (<= m_max);
  //   columns: the widest MMA N (n_max) — measured on B200
  //            (scripts/micro/mma_bench.cu), an M=128 K=16 kind::f16 MMA costs
  //            ~100 clk whatever N <= 128 is (N=256: 128 clk), so narrower
  //            column tiles lose 25-70 % of the tensor pipe — or a whole short
  //            axis; a column tile must also fit a double-buffered TMEM
  //            accumulator (2 x tile <= tmem_columns);
  //   reduce : whole TMA swizzle atoms (swizzle bytes / element bytes).
  // Batch tiles are free (one work item per batch entry).
  if (in.ns < 2) return false;
  const int ai = in.ns - 2, aj = in.ns - 1;
  const int64_t ti = smem[ai], tj = smem[aj], Ei = in.ext[ai], Ej = in.ext[aj];
  const int64_t M = hw.m_max, N = std::min(hw.n_max, hw.tmem_cols / 2);
  const int64_t k_atom = std::max<int64_t>(1, hw.swizzle / in.elem);
  auto lane_ok = [M](int64_t t, int64_t E) { return (t % M == 0 && t <= 2 * M) || (t >= E && t <= M); };
  auto col_ok = [N](int64_t t, int64_t E) { return t == N || (t >= E && t <= N); };
  for (int r = in.ns; r < in.na(); ++r)
    if (smem[r] % k_atom) return false;
  if (relax_tau == ai || relax_tau == aj) {
    const int64_t t_tau = relax_tau == ai ? ti : tj, t_o = relax_tau == ai ? tj : ti;
    const int64_t E_tau = relax_tau == ai ? Ei : Ej, E_o = relax_tau == ai ? Ej : Ei;
    if (relax_level == 1) {
      // first fallback rung: the main-axis tile may be any wide MMA N
      // (multiple of 2 * n_step in [N / 2, N]) so that two parts can cover
      // tau exactly; the other output axis stays strict in the matching role
      const int64_t wstep = 2 * hw.n_step;
      auto col_wide = [N, wstep](int64_t t, int64_t E) {
        return (t % wstep == 0 && t >= N / 2 && t <= N) || (t >= E && t <= N);
      };
      return (col_wide(t_tau, E_tau) && lane_ok(t_o, E_o)) || (lane_ok(t_tau, E_tau) && col_ok(t_o, E_o));
    }
    // last fallback rung: the main-axis tile may take any size <= N (it is
    // padded inside the MMA tile); the other output axis stays strict
    return t_tau <= N && (lane_ok(t_o, E_o) || col_ok(t_o, E_o));
  }
  return (lane_ok(ti, Ei) && col_ok(tj, Ej)) || (lane_ok(tj, Ej) && col_ok(ti, Ei));
}

Cands enumerate(const Instance& in, const Hw& hw, int64_t cap, bool* truncated_out) {
  const int S = in.ns, A = in.na();
  std::vector<std::vector<int64_t>> reg_opts(S);
  for (int s = 0; s < S; ++s) reg_opts[s] = reg_tile_candidates(in.ext[s], hw.align);
  std::vector<std::vector<int64_t>> red_opts(in.nr);
  for (int r = 0; r < in.nr; ++r) red_opts[r] = reduce_options(in.ext[S + r], hw.align);

  Cands c;
  c.inst = in;
  c.ns = S;
  c.na = A;
  bool truncated = false;
  int64_t total = 0;
  std::vector<size_t> ridx(S, 0);
  std::vector<std::vector<int64_t>> opts(A);
  for (int r = 0; r < in.nr; ++r) opts[S + r] = red_opts[r];
  std::vector<int64_t> combo(S), tile(A), minima(A);
  const int64_t limit = hw.smem;
  // footprint of `t` in bytes (ukernel.py:136-144)
  auto footprint = [&](const int64_t* t) {
    int64_t tot = 0;
    for (const auto& acc : in.inputs) {
      int64_t p = 1;
      for (int ax : acc) p *= t[ax];
      tot += p;
    }
    return tot * in.elem;
  };
  bool stop = false;
  while (!stop) {
    for (int s = 0; s < S; ++s) {
      combo[s] = reg_opts[s][ridx[s]];
      opts[s] = space_options(in.ext[s], combo[s], hw.align, s == in.major);
    }
    for (int a = 0; a < A; ++a) minima[a] = opts[a][0];
    // depth-first walk in lexicographic order; a value whose minimal
    // completion overflows ends its level (footprint is monotone per axis).
    std::vector<int64_t> probe(minima);
    std::vector<size_t> pos(A, 0);
    int depth = 0;
    while (depth >= 0 && !stop) {
      if (pos[depth] >= opts[depth].size()) {
        pos[depth] = 0;
        probe[depth] = minima[depth];
        --depth;
        if (depth >= 0) ++pos[depth];
        continue;
      }
      probe[depth] = opts[depth][pos[depth]];
      if (footprint(probe.data()) > limit) {  // this and all larger values overflow
        pos[depth] = opts[depth].size();
        continue;
      }
      if (depth == A - 1) {
        if (cap >= 0 && total >= cap) {
          truncated = true;
          stop = true;
          break;
        }
        c.reg.insert(c.reg.end(), combo.begin(), combo.end());
        c.smem.insert(c.smem.end(), probe.begin(), probe.end());
        ++total;
        ++pos[depth];
      } else {
        ++depth;
        pos[depth] = 0;
      }
    }
    // next register combination (itertools.product order: last axis fastest)
    int s = S - 1;
    for (; s >= 0; --s) {
      if (++ridx[s] < reg_opts[s].size()) break;
      ridx[s] = 0;
    }
    if (s < 0) break;
  }
  if (total == 0)
    throw capacity_error("no tile configuration fits shared memory (" + std::to_string(hw.smem) + " B)");
  if (truncated_out) *truncated_out = truncated;
  return c;
}

// ------------------------------------------------------------------ metrics (metrics.py)

static void subset_inplace(Cands& c, const std::vector<int64_t>& keep);

Cands enumerate_legal(const Instance& in, const Hw& hw, int64_t cap, bool* truncated) {
  Cands all = enumerate(in, hw, cap, truncated);
  if (hw.legality) {  // B200 extension, applied right after enumeration + cap truncation
    std::vector<int64_t> keep;
    for (size_t i = 0; i < all.size(); ++i)
      if (tcgen05_legal(in, hw, all.smem_row(i), hw.relax_tau, hw.relax_level)) keep.push_back(static_cast<int64_t>(i));
    subset_inplace(all, keep);
  }
  return all;
}

static void subset_inplace(Cands& c, const std::vector<int64_t>& keep) {
  Cands out;
  out.inst = c.inst;
  out.ns = c.ns;
  out.na = c.na;
  out.reg.reserve(keep.size() * c.ns);
  out.smem.reserve(keep.size() * c.na);
  for (int64_t i : keep) {
    out.reg.insert(out.reg.end(), c.reg_row(i), c.reg_row(i) + c.ns);
    out.smem.insert(out.smem.end(), c.smem_row(i), c.smem_row(i) + c.na);
  }
  auto pick_i = [&](const std::vector<int64_t>& v) {
    std::vector<int64_t> r;
    if (v.empty()) return r;
    r.reserve(keep.size());
    for (int64_t i : keep) r.push_back(v[i]);
    return r;
  };
  auto pick_d = [&](const std::vector<double>& v) {
    std::vector<double> r;
    if (v.empty()) return r;
    r.reserve(keep.size());
    for (int64_t i : keep) r.push_back(v[i]);
    return r;
  };
  out.pad_num = pick_i(c.pad_num);
  out.pad_den = pick_i(c.pad_den);
  out.blocks = pick_i(c.blocks);
  out.occ_den = pick_i(c.occ_den);
  out.regs_in_block = pick_i(c.regs_in_block);
  out.retained = pick_i(c.retained);
  if (!c.saturated.empty())
    for (int64_t i : keep) out.saturated.push_back(c.saturated[i]);
  out.cmr = pick_d(c.cmr);
  out.kmem = pick_d(c.kmem);
  out.m_pad = pick_d(c.m_pad);
  out.m_occ = pick_d(c.m_occ);
  out.m_cmr = pick_d(c.m_cmr);
  out.has_metrics = c.has_metrics;
  c = std::move(out);
}

// Geometry, registers and intensity columns for every row.
static void annotate(Cands& c, const Hw& hw, int64_t rest_regs) {
  const Instance& in = c.inst;
  const size_t n = c.size();
  int64_t true_elems = 1;
  for (int s = 0; s < in.ns; ++s) true_elems *= in.ext[s];
  c.pad_num.assign(n, true_elems * in.elem);
  c.pad_den.resize(n);
  c.blocks.resize(n);
  c.occ_den.resize(n);
  c.regs_in_block.resize(n);
  c.saturated.resize(n);
  c.cmr.resize(n);
  c.kmem.resize(n);
  const double out_bytes = static_cast<double>(true_elems * in.elem);
  const double compute_time = static_cast<double>(in.flops()) / static_cast<double>(hw.peak);
  const double bw_g = static_cast<double>(hw.bw_g), bw_s = static_cast<double>(hw.bw_s);
  const double elem_d = static_cast<double>(in.elem);
  std::vector<std::vector<uint8_t>> in_acc(in.inputs.size(), std::vector<uint8_t>(in.na(), 0));
  for (size_t q = 0; q < in.inputs.size(); ++q)
    for (int ax : in.inputs[q]) in_acc[q][ax] = 1;
  for (size_t i = 0; i < n; ++i) {
    const int64_t* r = c.reg_row(i);
    const int64_t* t = c.smem_row(i);
    // metrics.py:155-177
    int64_t blocks = 1, covered = 1;
    for (int s = 0; s < in.ns; ++s) {
      const int64_t b = cdiv(in.ext[s], t[s]);
      blocks *= b;
      covered *= b * t[s];
    }
    c.pad_den[i] = covered * in.elem;
    c.blocks[i] = blocks;
    c.occ_den[i] = cdiv(blocks, hw.cores) * hw.cores;
    // metrics.py:180-191 (sum of register tiles, not the product)
    int64_t reg_sum = 0, threads = 1;
    for (int s = 0; s < in.ns; ++s) {
      reg_sum += r[s];
      threads *= t[s] / r[s];
    }
    c.regs_in_block[i] = (reg_sum + rest_regs) * threads;
    // metrics.py:194-241
    int64_t read = 0, tread = 0;
    for (size_t q = 0; q < in.inputs.size(); ++q) {
      int64_t staged = 1, strip = 1, passes = 1;
      for (int s = 0; s < in.ns; ++s) {
        if (in_acc[q][s]) {
          staged *= t[s];
          strip *= t[s];
        } else {
          strip *= t[s] / r[s];
        }
      }
      for (int rr = in.ns; rr < in.na(); ++rr)
        if (in_acc[q][rr]) {
          passes *= cdiv(in.ext[rr], t[rr]);
          staged *= t[rr];
        }
      read += staged * passes;
      tread += strip * passes;
    }
    const double data_r = static_cast<double>(read) * static_cast<double>(blocks) * elem_d;
    const double data_tr = static_cast<double>(tread) * static_cast<double>(blocks) * elem_d;
    const double g = (data_r + out_bytes) / bw_g;
    const double sh = (data_r + data_tr) / bw_s;
    c.kmem[i] = (std::isnan(g) || std::isnan(sh)) ? NAN : (g >= sh ? g : sh);  // np.maximum
    c.cmr[i] = compute_time / c.kmem[i];
    c.saturated[i] = blocks >= hw.cores * hw.active;
  }
}

static void attach_part_metrics(Cands& c) {  // filtering.py:326-329
  const size_t n = c.size();
  c.m_pad.resize(n);
  c.m_occ.resize(n);
  c.m_cmr.resize(n);
  for (size_t i = 0; i < n; ++i) {
    c.m_pad[i] = static_cast<double>(c.pad_num[i]) / static_cast<double>(c.pad_den[i]);
    c.m_occ[i] = static_cast<double>(c.blocks[i]) / static_cast<double>(c.occ_den[i]);
    c.m_cmr[i] = c.cmr[i];
  }
  c.has_metrics = true;
}

// filtering.py:131-162 — closed-form first retaining step (0 = never).
static void retention(const Cands& c, const Sweep& sw, std::vector<int64_t>& steps) {
  const size_t n = c.size();
  steps.resize(n);
  const int64_t en = sw.eps_min.n, ed = sw.eps_min.d, sn = sw.eps_step.n, sd = sw.eps_step.d;
  const int64_t ln = sw.lam_max.n, ld = sw.lam_max.d, tn = sw.lam_step.n, td = sw.lam_step.d;
  const int64_t last = sw.num_steps();
  for (size_t i = 0; i < n; ++i) {
    const int64_t pn = c.pad_num[i], pd = c.pad_den[i], on = c.blocks[i], od = c.occ_den[i];
    const int64_t t_pad = 1 + py_floordiv((pn * ed - en * pd) * sd, pd * ed * sn);
    const int64_t t_occ = std::max<int64_t>(1 + py_ceildiv((ln * od - on * ld) * td, od * ld * tn), 1);
    steps[i] = (t_occ <= std::min(t_pad, last)) ? t_occ : 0;
  }
}

Cands compile_shape(const Instance& in, const Hw& hw, const Params& p, Report* rep, int stage) {
  bool truncated = false;
  Cands all = enumerate_legal(in, hw, p.cap, &truncated);
  annotate(all, hw, p.rest_regs);
  const size_t n = all.size();
  std::vector<uint8_t> reg_ok(n);
  for (size_t i = 0; i < n; ++i) {
    // filtering.py:198-214: bound = min(ceil(blocks/cores), zeta)
    const int64_t bound = std::min(cdiv(all.blocks[i], hw.cores), hw.zeta);
    reg_ok[i] = all.regs_in_block[i] * bound <= hw.regs;
  }
  // staged footprint always fits for enumerated rows (cross_pick :179-189)
  Sweep used = p.sweep;
  int relax = FTB_RELAX_NONE, widen = 0;
  std::vector<int64_t> steps, cross, filt, fin;
  auto run_cross = [&](const Sweep& sw) {
    retention(all, sw, steps);
    cross.clear();
    for (size_t i = 0; i < n; ++i)
      if (steps[i] > 0) cross.push_back(static_cast<int64_t>(i));
    filt.clear();
    for (int64_t i : cross)
      if (reg_ok[i]) filt.push_back(i);
  };
  run_cross(used);
  std::vector<int64_t> retained_all = steps;
  fin.clear();
  for (int64_t i : filt)
    if (all.saturated[i] && all.cmr[i] >= p.psi) fin.push_back(i);
  int64_t n_cross = static_cast<int64_t>(cross.size());
  if (fin.empty() && !filt.empty()) {  // filtering.py:286-291
    relax = FTB_RELAX_DROP_INTENSITY;
    for (int64_t i : filt)
      if (all.saturated[i]) fin.push_back(i);
    if (fin.empty()) {
      relax = FTB_RELAX_DROP_SATURATION;
      fin = filt;
    }
  } else if (filt.empty()) {  // filtering.py:292-318
    // The reference re-runs the sweep for w = 1, 2, ... until the register-
    // bounded set is non-empty. Retention is monotone in w (eps_min and
    // lam_min only decrease, so the padding bound and the step count only
    // grow), so the first successful w is min over register-feasible rows of
    // each row's first retaining w, found by bisection. The loop stops early
    // (drop-sweep) at the first w whose floored bounds equal the previous
    // ones, or past 2000 widenings — computed here without iterating.
    int64_t w_end = 0;  // last w the reference would actually try
    for (int64_t w = 1; w <= _MAX_WIDEN; ++w) {
      if (p.sweep.widened(w) == p.sweep.widened(w - 1)) break;
      w_end = w;
    }
    struct Pt { int64_t en, ed, last; };
    std::vector<Pt> pts(w_end + 1);
    for (int64_t w = 1; w <= w_end; ++w) {
      Sweep sw = p.sweep.widened(w);
      pts[w] = {sw.eps_min.n, sw.eps_min.d, sw.num_steps()};
    }
    const int64_t sn = p.sweep.eps_step.n, sd = p.sweep.eps_step.d;
    const int64_t ln = p.sweep.lam_max.n, ld = p.sweep.lam_max.d;
    const int64_t tn = p.sweep.lam_step.n, td = p.sweep.lam_step.d;
    auto kept_at = [&](size_t i, int64_t w) {
      const int64_t pn = all.pad_num[i], pd = all.pad_den[i], on = all.blocks[i], od = all.occ_den[i];
      const int64_t t_pad = 1 + py_floordiv((pn * pts[w].ed - pts[w].en * pd) * sd, pd * pts[w].ed * sn);
      const int64_t t_occ = std::max<int64_t>(1 + py_ceildiv((ln * od - on * ld) * td, od * ld * tn), 1);
      return t_occ <= std::min(t_pad, pts[w].last);
    };
    int64_t w_star = w_end + 1;
    for (size_t i = 0; i < n && w_end > 0; ++i) {
      if (!reg_ok[i]) continue;
      const int64_t hi0 = std::min(w_star - 1, w_end);
      if (hi0 < 1 || !kept_at(i, hi0)) continue;
      int64_t lo = 1, hi = hi0;  // first w in [1, hi0] with kept_at true
      while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (kept_at(i, mid)) hi = mid; else lo = mid + 1;
      }
      w_star = lo;
    }
    if (w_star <= w_end) {
      used = p.sweep.widened(w_star);
      run_cross(used);
      n_cross = static_cast<int64_t>(cross.size());
      retained_all = steps;
      relax = FTB_RELAX_WIDEN;
      widen = static_cast<int>(w_star);
      if (filt.empty()) throw internal_error("widening bisection disagrees with the sweep");
    } else {
      if (w_end > 0) used = p.sweep.widened(w_end);
      relax = FTB_RELAX_DROP_SWEEP;
      cross.resize(n);
      std::iota(cross.begin(), cross.end(), 0);
      n_cross = static_cast<int64_t>(n);
      retained_all.assign(n, 0);
      filt.clear();
      for (int64_t i : cross)
        if (reg_ok[i]) filt.push_back(i);
      if (filt.empty())
        throw FtbError(FTB_EMPTY_RESULT, "no candidate passes the register budget", "register budget");
    }
    fin = filt;
  }
  all.retained = retained_all;
  const int64_t n_align = static_cast<int64_t>(n), n_filter = static_cast<int64_t>(filt.size());
  const int64_t n_final = static_cast<int64_t>(fin.size());
  if (stage == 0) {
    subset_inplace(all, fin);
  } else if (stage == 1) {
    subset_inplace(all, filt);
  } else if (stage == 2) {
    subset_inplace(all, cross);
  }  // stage 3: the whole (legal) align set
  attach_part_metrics(all);
  if (rep) {
    rep->n_align = n_align;
    rep->n_cross = n_cross;
    rep->n_filter = n_filter;
    rep->n_final = n_final;
    rep->stage = stage;
    rep->relaxation = relax;
    rep->widen = widen;
    rep->truncated = truncated;
    rep->used = used;
    rep->tau = select_main_axis(in);
  }
  return all;
}

// ------------------------------------------------------------------ compose (combine.py)

int select_main_axis(const Instance& in) {  // combine.py:58-68
  int64_t best = 0;
  for (int s = 0; s < in.ns; ++s) best = std::max(best, in.ext[s]);
  int pick = -1;
  bool pick_dyn = false;
  for (int s = 0; s < in.ns; ++s) {
    if (in.ext[s] != best) continue;
    const bool dyn = in.dynamic[s];
    if (pick < 0 || (dyn && !pick_dyn) || (dyn == pick_dyn && in.name[s] < in.name[pick])) {
      pick = s;
      pick_dyn = dyn;
    }
  }
  return pick;
}

static int64_t modinv(int64_t b, int64_t m) {  // b^-1 mod m, gcd(b,m)=1
  int64_t old_r = b % m, r = m, old_s = 1, s = 0;
  if (old_r < 0) old_r += m;
  while (r != 0) {
    int64_t q = old_r / r;
    int64_t t = old_r - q * r; old_r = r; r = t;
    t = old_s - q * s; old_s = s; s = t;
  }
  old_s %= m;
  if (old_s < 0) old_s += m;
  return old_s;
}

// combine.py:71-89: first n2 of the residue class and the class step, or
// n2_first = 0 when no solution exists.
struct PairSol {
  int64_t h, a_, b_, n2_first;  // solutions: n2 = n2_first + t*a_, while n2*b_ <= h - a_
  int64_t count() const {
    if (n2_first == 0 || n2_first * b_ > h - a_) return 0;
    return (h - a_ - n2_first * b_) / (a_ * b_) + 1;
  }
  // n1 for the solution with the t-th smallest n1 (t = 0 .. count-1)
  void nth_smallest_n1(int64_t t, int64_t* n1, int64_t* n2) const {
    const int64_t idx = count() - 1 - t;  // solutions are generated with n2 ascending
    *n2 = n2_first + idx * a_;
    *n1 = (h - *n2 * b_) / a_;
  }
};
static PairSol pair_solutions(int64_t a, int64_t b, int64_t H) {
  PairSol ps{0, 1, 1, 0};
  const int64_t g = std::gcd(a, b);
  if (H % g) return ps;
  ps.a_ = a / g;
  ps.b_ = b / g;
  ps.h = H / g;
  if (ps.a_ == 1) {
    ps.n2_first = 1;
  } else {
    int64_t n2 = static_cast<int64_t>((static_cast<__int128>(ps.h % ps.a_) * modinv(ps.b_, ps.a_)) % ps.a_);
    ps.n2_first = n2 == 0 ? ps.a_ : n2;
  }
  return ps;
}

// Lexicographic tile key comparison (ukernel.py:59-64): reg vector, then smem vector.
static inline int cmp_key(const Cands& c, int64_t x, int64_t y) {
  const int64_t *rx = c.reg_row(x), *ry = c.reg_row(y);
  for (int s = 0; s < c.ns; ++s)
    if (rx[s] != ry[s]) return rx[s] < ry[s] ? -1 : 1;
  const int64_t *sx = c.smem_row(x), *sy = c.smem_row(y);
  for (int a = 0; a < c.na; ++a)
    if (sx[a] != sy[a]) return sx[a] < sy[a] ? -1 : 1;
  return 0;
}

namespace {
struct Layout {
  std::vector<int64_t> uniq;                 // deduplicated rows sorted by tile key
  std::vector<std::vector<int64_t>> groups;  // same non-tau signature, members sorted by key
  int64_t H = 0;
};

Layout make_layout(const Cands& c, int tau) {
  Layout L;
  L.H = c.inst.ext[tau];
  std::vector<int64_t> idx(c.size());
  std::iota(idx.begin(), idx.end(), 0);
  // stable sort keeps the first occurrence first among equal keys (combine.py:150-153)
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return cmp_key(c, a, b) < 0; });
  for (size_t i = 0; i < idx.size(); ++i)
    if (i == 0 || cmp_key(c, idx[i - 1], idx[i]) != 0) L.uniq.push_back(idx[i]);
  // group by signature (combine.py:118-123): reg and smem tiles except tau
  std::map<std::vector<int64_t>, size_t> gid;
  std::vector<int64_t> sig;
  for (int64_t r : L.uniq) {
    sig.clear();
    for (int s = 0; s < c.ns; ++s)
      if (s != tau) sig.push_back(c.reg_row(r)[s]);
    sig.push_back(-1);
    for (int a = 0; a < c.na; ++a)
      if (a != tau) sig.push_back(c.smem_row(r)[a]);
    auto it = gid.find(sig);
    if (it == gid.end()) {
      gid.emplace(sig, L.groups.size());
      L.groups.push_back({r});
    } else {
      L.groups[it->second].push_back(r);  // uniq is key-sorted, so members stay sorted
    }
  }
  return L;
}
}  // namespace

int64_t pool_count(const Cands& c, int tau) {
  Layout L = make_layout(c, tau);
  int64_t n = 0;
  for (int64_t r : L.uniq)
    if (L.H % c.smem_row(r)[tau] == 0) ++n;
  for (const auto& g : L.groups)
    for (size_t x = 0; x < g.size(); ++x)
      for (size_t y = x + 1; y < g.size(); ++y) {
        const int64_t a = c.smem_row(g[x])[tau], b = c.smem_row(g[y])[tau];
        if (a == b) continue;
        n += pair_solutions(std::min(a, b), std::max(a, b), L.H).count();
      }
  return n;
}

static inline int cmp_plan_tiles(const Cands& c, const PlanRow& p, const PlanRow& q) {
  // tuple((tile_key, n) for parts) with Python tuple semantics
  int k = cmp_key(c, p.ra, q.ra);
  if (k) return k;
  if (p.na_ != q.na_) return p.na_ < q.na_ ? -1 : 1;
  if (p.nparts == 1 || q.nparts == 1) return (p.nparts > q.nparts) - (p.nparts < q.nparts);
  k = cmp_key(c, p.rb, q.rb);
  if (k) return k;
  if (p.nb != q.nb) return p.nb < q.nb ? -1 : 1;
  return 0;
}

std::vector<PlanRow> pool_export(const Cands& c, int tau) {
  Layout L = make_layout(c, tau);
  std::vector<PlanRow> singles, pairs;
  for (int64_t r : L.uniq) {
    const int64_t t = c.smem_row(r)[tau];
    if (L.H % t == 0) singles.push_back({1, r, L.H / t, -1, 0});
  }
  for (const auto& g : L.groups)
    for (size_t x = 0; x < g.size(); ++x)
      for (size_t y = x + 1; y < g.size(); ++y) {
        const int64_t a = c.smem_row(g[x])[tau], b = c.smem_row(g[y])[tau];
        if (a == b) continue;
        const bool xlo = a < b;
        const int64_t lo_r = xlo ? g[x] : g[y], hi_r = xlo ? g[y] : g[x];
        PairSol ps = pair_solutions(std::min(a, b), std::max(a, b), L.H);
        const int64_t cnt = ps.count();
        for (int64_t t = 0; t < cnt; ++t) {
          int64_t n1, n2;
          ps.nth_smallest_n1(t, &n1, &n2);
          pairs.push_back({2, lo_r, n1, hi_r, n2});
        }
      }
  std::sort(pairs.begin(), pairs.end(),
            [&](const PlanRow& p, const PlanRow& q) { return cmp_plan_tiles(c, p, q) < 0; });
  if (singles.empty() && pairs.empty())
    throw FtbError(FTB_EMPTY_RESULT, "no uKernel combination covers axis '" + c.inst.name[tau] +
                                         "' (extent " + std::to_string(L.H) + ")",
                   "main-axis coverage");
  singles.insert(singles.end(), pairs.begin(), pairs.end());
  return singles;
}

// ------------------------------------------------------------------ rank (scoring.py)

namespace {
struct Cand {
  PlanRow row;
  double score, mpad;
};
struct Ranker {
  const Cands& c;
  int k;
  // "a ranks before b" under (-score, nparts, -mean_pad, tile_order) (scoring.py:120-123)
  bool before(const Cand& a, const Cand& b) const {
    if (a.score != b.score) return a.score > b.score;
    if (a.row.nparts != b.row.nparts) return a.row.nparts < b.row.nparts;
    if (a.mpad != b.mpad) return a.mpad > b.mpad;
    return cmp_plan_tiles(c, a.row, b.row) < 0;
  }
  struct Cmp {
    const Ranker* r;
    bool operator()(const Cand& a, const Cand& b) const { return r->before(a, b); }
  };
  std::priority_queue<Cand, std::vector<Cand>, Cmp> heap;  // top() = worst kept
  explicit Ranker(const Cands& cc, int kk) : c(cc), k(kk), heap(Cmp{this}) {}
  bool full() const { return static_cast<int>(heap.size()) >= k; }
  // true if `x` would be kept
  bool offer(const Cand& x) {
    if (k <= 0) return false;
    if (!full()) {
      heap.push(x);
      return true;
    }
    if (before(x, heap.top())) {
      heap.pop();
      heap.push(x);
      return true;
    }
    return false;
  }
};
}  // namespace

std::vector<std::pair<PlanRow, double>> rank_topk(const Cands& c, int tau, const ftb_coeffs& co,
                                                  int k, bool normalize) {
  if (co.c0 < 0 || co.c1 < 0 || co.c2 < 0)
    throw input_error("score coefficients must be nonnegative", "coeffs");
  if (co.c0 == 0 && co.c1 == 0 && co.c2 == 0)
    throw input_error("at least one score coefficient must be positive", "coeffs");
  Layout L = make_layout(c, tau);
  const int64_t H = L.H;
  // participation: kernels that appear in at least one plan of the pool
  std::vector<uint8_t> part(c.size(), 0);
  bool any = false;
  for (int64_t r : L.uniq)
    if (H % c.smem_row(r)[tau] == 0) part[r] = 1, any = true;
  for (const auto& g : L.groups) {
    std::vector<int64_t> tv;
    for (int64_t r : g) tv.push_back(c.smem_row(r)[tau]);
    std::vector<int64_t> d(tv);
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    std::vector<uint8_t> ok(d.size(), 0);
    for (size_t x = 0; x < d.size(); ++x)
      for (size_t y = x + 1; y < d.size(); ++y)
        if (pair_solutions(d[x], d[y], H).count() > 0) ok[x] = ok[y] = 1;
    for (size_t m = 0; m < g.size(); ++m) {
      const size_t di = std::lower_bound(d.begin(), d.end(), tv[m]) - d.begin();
      if (ok[di]) part[g[m]] = 1, any = true;
    }
  }
  if (!any)
    throw FtbError(FTB_EMPTY_RESULT, "no uKernel combination covers axis '" + c.inst.name[tau] +
                                         "' (extent " + std::to_string(H) + ")",
                   "main-axis coverage");
  if (!c.has_metrics) throw FtbError(FTB_MISSING_METRICS, "uKernel has no cached metrics; run the compile-stage pipeline first");
  for (size_t r = 0; r < c.size(); ++r)
    if (part[r] && (std::isnan(c.m_pad[r]) || std::isnan(c.m_occ[r]) || std::isnan(c.m_cmr[r])))
      throw FtbError(FTB_MISSING_METRICS, "uKernel has no cached metrics; run the compile-stage pipeline first");
  // per-part scores (scoring.py:49-51), optionally min-max normalised over the pool's parts
  std::vector<double> sc(c.size(), 0.0);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  if (normalize)
    for (size_t r = 0; r < c.size(); ++r)
      if (part[r]) {
        const double m[3] = {c.m_cmr[r], c.m_pad[r], c.m_occ[r]};
        for (int q = 0; q < 3; ++q) lo[q] = std::min(lo[q], m[q]), hi[q] = std::max(hi[q], m[q]);
      }
  for (size_t r = 0; r < c.size(); ++r) {
    double m[3] = {c.m_cmr[r], c.m_pad[r], c.m_occ[r]};
    if (normalize)
      for (int q = 0; q < 3; ++q) m[q] = hi[q] > lo[q] ? (m[q] - lo[q]) / (hi[q] - lo[q]) : 1.0;
    sc[r] = co.c0 * m[0] + co.c1 * m[1] + co.c2 * m[2];
  }
  Ranker R(c, k);
  for (int64_t r : L.uniq) {
    const int64_t t = c.smem_row(r)[tau];
    if (H % t == 0) R.offer({{1, r, H / t, -1, 0}, sc[r], c.m_pad[r]});
  }
  for (const auto& g : L.groups) {
    if (g.size() < 2) continue;
    std::vector<int64_t> m;
    for (int64_t r : g)
      if (part[r]) m.push_back(r);
    std::stable_sort(m.begin(), m.end(), [&](int64_t a, int64_t b) { return sc[a] > sc[b]; });
    for (size_t x = 0; x + 1 < m.size(); ++x) {
      if (R.full() && (sc[m[x]] + sc[m[x + 1]]) / 2.0 < R.heap.top().score) break;
      for (size_t y = x + 1; y < m.size(); ++y) {
        const double s = (sc[m[x]] + sc[m[y]]) / 2.0;  // sum([s1, s2]) / 2 (scoring.py:54-58)
        if (R.full() && s < R.heap.top().score) break;
        const int64_t a = c.smem_row(m[x])[tau], b = c.smem_row(m[y])[tau];
        if (a == b) continue;
        const bool xlo = a < b;
        const int64_t lo_r = xlo ? m[x] : m[y], hi_r = xlo ? m[y] : m[x];
        PairSol ps = pair_solutions(std::min(a, b), std::max(a, b), H);
        const int64_t cnt = ps.count();
        const double mp = (c.m_pad[lo_r] + c.m_pad[hi_r]) / 2.0;
        for (int64_t t = 0; t < cnt; ++t) {
          int64_t n1, n2;
          ps.nth_smallest_n1(t, &n1, &n2);
          if (!R.offer({{2, lo_r, n1, hi_r, n2}, s, mp})) break;  // larger n1 ranks later
        }
      }
    }
  }
  std::vector<Cand> out;
  while (!R.heap.empty()) {
    out.push_back(R.heap.top());
    R.heap.pop();
  }
  std::reverse(out.begin(), out.end());
  std::vector<std::pair<PlanRow, double>> res;
  for (auto& x : out) res.push_back({x.row, x.score});
  return res;
}

}  // namespace plan
}  // namespace ftb
