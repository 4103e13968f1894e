// lp.cpp — bounded primal revised simplex for swarmplan::lp (host side).
//
// Replaces the reference solver (/root/reference/proj/src/lp.cpp:95-822,
// KLU sparse LU + Eigen) with a dependency-free design sized for the
// strategy programs (<= ~1.3k rows at 24 peers):
//
//  * Basis representation. Slack columns are unit vectors, so a basis with
//    S basic slacks reduces to a k x k "kernel" M (k = m - S): the rows not
//    covered by a basic slack times the basic structural columns. M gets a
//    sparse Markowitz LU with threshold pivoting (strategy kernels have ~4
//    nonzeros per column and little fill); the covered rows are recovered by
//    one sparse sweep. Between refactorizations, basis changes are applied
//    as product-form eta columns. ftran/btran cost O(nnz(L+U) + etas*m).
//  * Pricing: devex reference weights (symmetric fleets make whole column
//    families tie; largest-coefficient pricing stalls on them), lowest index
//    on ties, Bland's rule after a run of degenerate pivots. The pivot row
//    and the priced reduced costs are formed row-wise over the nonzeros of
//    rho and y (table1_c: 1.3k instead of 7.6k multiply-adds per pivot row,
//    3.0k instead of 8.1k per pricing pass; daynight 240 instead of 7.6k),
//    and phase 2 updates the reduced costs from the pivot row instead of a
//    second btran per iteration.
//  * Ratio test: exact minimum ratio; near-ties go to the largest pivot,
//    then to the lowest variable index. If roundoff pushes a basic variable
//    out of bounds during phase 2, the solve returns to phase 1 to repair.
//  * Degeneracy: every finite bound is shifted outward by a deterministic
//    1e-6 * [1,2) amount for the main solve, then the exact program is
//    finished from that basis (a standard bound-shifting scheme; the
//    reference applies the same idea, lp.cpp:672-721).
//  * Phase 1 minimizes the sum of bound violations of basic variables
//    (composite objective), phase 2 the real objective. Rows are scaled by
//    their largest |coefficient| on entry.
// Everything is deterministic: fixed loop orders, index tie-breaks, no RNG.

#include "swarmplan/lp.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <set>
#include <sstream>

#include "swarmplan/log.hpp"

namespace swarmplan::lp {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr int kEtaLimit = 48;     // basis changes between refactorizations
constexpr int kStallLimit = 60;   // degenerate pivots before Bland's rule
constexpr double kShift = 1e-6;   // bound perturbation scale
constexpr double kSingular = 1e-11;

std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// deterministic value in [1, 2) keyed by (variable, side)
double shift_unit(std::uint64_t var, std::uint64_t side) {
  return 1.0 + static_cast<double>(mix64(var * 2 + side + 0x5851f42d4c957f2dULL) >> 11) *
                   0x1.0p-53;
}

}  // namespace

LinearProgram::LinearProgram(int nvars)
    : num_vars(nvars),
      objective(Eigen::VectorXd::Zero(nvars)),
      lower(Eigen::VectorXd::Zero(nvars)),
      upper(Eigen::VectorXd::Constant(nvars, kInf)) {}

int LinearProgram::add_row(std::vector<std::pair<int, double>> coeffs, Relation rel,
                           double rhs) {
  Row r;
  r.coeffs = std::move(coeffs);
  r.rel = rel;
  r.rhs = rhs;
  rows.push_back(std::move(r));
  return static_cast<int>(rows.size()) - 1;
}

double check_feasible(const LinearProgram& prog, const Eigen::VectorXd& x) {
  double worst = -kInf;
  for (const auto& row : prog.rows) {
    double lhs = 0.0, scale = 0.0;
    for (const auto& [j, a] : row.coeffs) {
      lhs += a * x(j);
      scale = std::max(scale, std::fabs(a));
    }
    const double gap = (lhs - row.rhs) / (scale > 0.0 ? scale : 1.0);
    worst = std::max(worst, row.rel == Relation::Eq ? std::fabs(gap) : gap);
  }
  for (int j = 0; j < prog.num_vars; ++j) {
    worst = std::max(worst, prog.lower(j) - x(j));
    worst = std::max(worst, x(j) - prog.upper(j));
  }
  return worst;
}

std::string dump(const LinearProgram& prog) {
  std::ostringstream os;
  os << "max";
  for (int j = 0; j < prog.num_vars; ++j)
    if (prog.objective(j) != 0.0)
      os << (prog.objective(j) < 0 ? " " : " +") << prog.objective(j) << " x" << j;
  os << "\n";
  for (std::size_t r = 0; r < prog.rows.size(); ++r) {
    os << "r" << r << ":";
    for (const auto& [j, a] : prog.rows[r].coeffs) os << (a < 0 ? " " : " +") << a << " x" << j;
    os << (prog.rows[r].rel == Relation::Eq ? " = " : " <= ") << prog.rows[r].rhs << "\n";
  }
  for (int j = 0; j < prog.num_vars; ++j)
    os << "x" << j << " in [" << prog.lower(j) << ", " << prog.upper(j) << "]\n";
  return os.str();
}

struct SimplexSolver::Impl {
  enum class St : std::uint8_t { Basic, Lower, Upper, Free };

  struct Var {
    double lo = 0.0, up = kInf, cost = 0.0;
    int slack_row = -1;                       // >= 0 for the slack of that row
    std::vector<std::pair<int, double>> col;  // (row, scaled coefficient)
  };

  struct Eta {
    int p = 0;
    double piv = 1.0;
    std::vector<int> idx;
    std::vector<double> val;
  };

  SimplexOptions opt;
  std::vector<Var> v;
  std::vector<int> structural;  // public index -> internal variable
  std::vector<double> rhs;      // scaled right-hand sides
  std::vector<int> slack_of_row;
  int m = 0;

  std::vector<int> basis;  // position -> variable
  std::vector<int> pos;    // variable -> position, -1 if nonbasic
  std::vector<St> st;
  std::vector<double> x;
  long iters = 0;
  bool factored = false;
  bool basics_stale = false;

  // kernel factorization
  int k = 0;
  std::vector<int> kpos, kvar, krow, row_k, slack_pos;  // snapshot of B0 at factor time
  // sparse LU of the kernel: step t pivots on (kernel row prow[t], kernel
  // column pcol[t]); L column t holds the multipliers of the rows it
  // eliminated, U row t the remaining entries of the pivot row
  std::vector<int> prow, pcol;
  std::vector<double> piv;
  std::vector<int> lbeg, lidx, ubeg, uidx;
  std::vector<double> lval, uval;
  std::vector<Eta> etas;
  std::vector<double> tk1, tk2;

  std::vector<double> saved_lo, saved_up;

  int nv() const { return static_cast<int>(v.size()); }

  static St initial_state(double lo, double up) {
    if (std::isfinite(lo)) return St::Lower;
    if (std::isfinite(up)) return St::Upper;
    return St::Free;
  }
  static double initial_value(double lo, double up) {
    if (std::isfinite(lo)) return lo;
    if (std::isfinite(up)) return up;
    return 0.0;
  }

  Impl(const LinearProgram& prog, SimplexOptions o) : opt(o) {
    if (prog.num_vars < 0 || prog.objective.size() != prog.num_vars ||
        prog.lower.size() != prog.num_vars || prog.upper.size() != prog.num_vars)
      throw MalformedProgram("objective/bounds must have num_vars entries");
    for (int j = 0; j < prog.num_vars; ++j)
      add_structural(prog.lower(j), prog.upper(j), prog.objective(j));
    for (const auto& row : prog.rows) {
      std::vector<std::pair<int, double>> c;
      c.reserve(row.coeffs.size());
      for (const auto& [j, a] : row.coeffs) {
        if (j < 0 || j >= prog.num_vars) throw MalformedProgram("row references unknown variable");
        c.emplace_back(structural[j], a);
      }
      append_row(c, row.rel, row.rhs);
    }
    reset_basis();
  }

  void add_structural(double lo, double up, double cost) {
    if (std::isnan(lo) || std::isnan(up) || std::isnan(cost) || lo > up ||
        lo == kInf || up == -kInf)
      throw MalformedProgram("invalid variable bounds or objective coefficient");
    Var var;
    var.lo = lo;
    var.up = up;
    var.cost = cost;
    v.push_back(std::move(var));
    structural.push_back(nv() - 1);
    pos.push_back(-1);
    st.push_back(initial_state(lo, up));
    x.push_back(initial_value(lo, up));
  }

  // appends row sum a_j x_j (rel) rhs with internal variable ids; returns the
  // slack variable id
  int append_row(const std::vector<std::pair<int, double>>& coeffs, Relation rel, double b) {
    if (!std::isfinite(b)) throw MalformedProgram("row right-hand side must be finite");
    double big = 0.0;
    for (const auto& [j, a] : coeffs) {
      if (j < 0 || j >= nv() || v[j].slack_row >= 0)
        throw MalformedProgram("row references unknown variable");
      if (!std::isfinite(a)) throw MalformedProgram("row coefficient must be finite");
      big = std::max(big, std::fabs(a));
    }
    const double s = big > 0.0 ? 1.0 / big : 1.0;
    const int r = m++;
    rhs.push_back(b * s);
    for (const auto& [j, a] : coeffs) {
      if (a == 0.0) continue;
      auto& col = v[j].col;
      bool merged = false;
      for (auto& e : col)
        if (e.first == r) {
          e.second += a * s;
          merged = true;
        }
      if (!merged) col.emplace_back(r, a * s);
    }
    Var sl;
    sl.lo = 0.0;
    sl.up = rel == Relation::Eq ? 0.0 : kInf;
    sl.slack_row = r;
    sl.col.emplace_back(r, 1.0);
    v.push_back(std::move(sl));
    slack_of_row.push_back(nv() - 1);
    pos.push_back(-1);
    st.push_back(St::Lower);
    x.push_back(0.0);
    return nv() - 1;
  }

  void reset_basis() {
    basis.assign(m, -1);
    std::fill(pos.begin(), pos.end(), -1);
    for (int j = 0; j < nv(); ++j) {
      if (v[j].slack_row >= 0) {
        basis[v[j].slack_row] = j;
        pos[j] = v[j].slack_row;
        st[j] = St::Basic;
      } else {
        st[j] = initial_state(v[j].lo, v[j].up);
        x[j] = initial_value(v[j].lo, v[j].up);
      }
    }
    factored = false;
    recompute_basics();
  }

  // ------------------------------------------------------- factorization
  int fail_col = -1, fail_row = -1;  // set when factor_kernel hits a zero pivot

  bool factor_kernel() {
    fail_col = fail_row = -1;
    slack_pos.assign(m, -1);
    kpos.clear();
    for (int p = 0; p < m; ++p) {
      const int j = basis[p];
      if (v[j].slack_row >= 0)
        slack_pos[v[j].slack_row] = p;
      else
        kpos.push_back(p);
    }
    krow.clear();
    row_k.assign(m, -1);
    for (int r = 0; r < m; ++r)
      if (slack_pos[r] < 0) {
        row_k[r] = static_cast<int>(krow.size());
        krow.push_back(r);
      }
    k = static_cast<int>(kpos.size());
    if (static_cast<int>(krow.size()) != k) return false;
    kvar.resize(k);
    for (int c = 0; c < k; ++c) kvar[c] = basis[kpos[c]];
    return sparse_lu();
  }

  // Markowitz-style sparse LU with threshold pivoting: at each step the
  // active column with the fewest entries, and in it the row with the fewest
  // entries among those within 0.1 of the column's largest magnitude.
  // Strategy-LP kernels have ~4 nonzeros per column and little fill.
  bool sparse_lu() {
    std::vector<std::vector<std::pair<int, double>>> col(k);  // active entries
    std::vector<std::vector<int>> row(k);                     // active pattern
    for (int c = 0; c < k; ++c)
      for (const auto& [r, a] : v[kvar[c]].col)
        if (row_k[r] >= 0 && a != 0.0) {
          col[c].emplace_back(row_k[r], a);
          row[row_k[r]].push_back(c);
        }
    std::vector<char> rdone(k, 0), cdone(k, 0);
    // active columns bucketed by entry count, each bucket ordered by index:
    // the pivot column is the lowest-index one with <= 1 entries, else the
    // lowest-index one of the smallest count (O(log k) instead of a scan)
    std::vector<std::set<int>> bucket(k + 1);
    for (int c = 0; c < k; ++c) bucket[col[c].size()].insert(c);
    std::size_t min_count = 0;
    auto resize_col = [&](int c, std::size_t from) {
      bucket[from].erase(c);
      const std::size_t to = col[c].size();
      if (to >= bucket.size()) bucket.resize(to + 1);
      bucket[to].insert(c);
      min_count = std::min(min_count, to);
    };
    prow.assign(k, -1);
    pcol.assign(k, -1);
    piv.assign(k, 0.0);
    lbeg.assign(1, 0);
    ubeg.assign(1, 0);
    lidx.clear();
    lval.clear();
    uidx.clear();
    uval.clear();
    std::vector<double> urowv;
    std::vector<int> urowc;
    for (int t = 0; t < k; ++t) {
      int q = -1;
      if (!bucket[0].empty() || (bucket.size() > 1 && !bucket[1].empty())) {
        const int c0 = bucket[0].empty() ? k : *bucket[0].begin();
        const int c1 = bucket.size() > 1 && !bucket[1].empty() ? *bucket[1].begin() : k;
        q = std::min(c0, c1);
      } else {
        while (bucket[min_count].empty()) ++min_count;
        q = *bucket[min_count].begin();
      }
      bucket[col[q].size()].erase(q);
      double cmax = 0.0;
      for (const auto& e : col[q]) cmax = std::max(cmax, std::fabs(e.second));
      if (cmax < kSingular) {
        fail_col = q;
        for (int r = 0; r < k; ++r)
          if (!rdone[r]) {
            fail_row = r;
            break;
          }
        return false;
      }
      int p = -1;
      double pv = 0.0;
      std::size_t rbest = SIZE_MAX;
      for (const auto& [r, a] : col[q]) {
        if (std::fabs(a) < 0.1 * cmax) continue;
        if (row[r].size() < rbest || (row[r].size() == rbest && std::fabs(a) > std::fabs(pv))) {
          rbest = row[r].size();
          p = r;
          pv = a;
        }
      }
      prow[t] = p;
      pcol[t] = q;
      piv[t] = pv;
      // U row: the pivot row's other active entries
      urowc.clear();
      urowv.clear();
      for (int c : row[p]) {
        if (c == q || cdone[c]) continue;
        for (const auto& e : col[c])
          if (e.first == p) {
            urowc.push_back(c);
            urowv.push_back(e.second);
            break;
          }
      }
      for (std::size_t u = 0; u < urowc.size(); ++u) {
        uidx.push_back(urowc[u]);
        uval.push_back(urowv[u]);
      }
      ubeg.push_back(static_cast<int>(uidx.size()));
      // eliminate column q from every other active row
      for (const auto& [r, a] : col[q]) {
        if (r == p) continue;
        const double mult = a / pv;
        lidx.push_back(r);
        lval.push_back(mult);
        for (std::size_t u = 0; u < urowc.size(); ++u) {
          auto& cc = col[urowc[u]];
          bool found = false;
          for (auto& e : cc)
            if (e.first == r) {
              e.second -= mult * urowv[u];
              found = true;
              break;
            }
          if (!found) {  // fill-in
            cc.emplace_back(r, -mult * urowv[u]);
            row[r].push_back(urowc[u]);
            resize_col(urowc[u], cc.size() - 1);
          }
        }
      }
      lbeg.push_back(static_cast<int>(lidx.size()));
      // retire row p and column q
      rdone[p] = 1;
      cdone[q] = 1;
      for (int c : row[p]) {
        if (cdone[c]) continue;
        auto& cc = col[c];
        for (std::size_t e = 0; e < cc.size(); ++e)
          if (cc[e].first == p) {
            cc[e] = cc.back();
            cc.pop_back();
            resize_col(c, cc.size() + 1);
            break;
          }
      }
      for (const auto& [r, a] : col[q]) {
        (void)a;
        if (r == p) continue;
        auto& rr = row[r];
        for (std::size_t e = 0; e < rr.size(); ++e)
          if (rr[e] == q) {
            rr[e] = rr.back();
            rr.pop_back();
            break;
          }
      }
      col[q].clear();
      row[p].clear();
    }
    tk1.resize(k);
    tk2.resize(k);
    return true;
  }

  // kernel solve M z = b: b by kernel row (consumed), z by kernel column
  void lu_solve(std::vector<double>& b, std::vector<double>& z) {
    for (int t = 0; t < k; ++t) {
      const double bt = b[prow[t]];
      if (bt == 0.0) continue;
      for (int e = lbeg[t]; e < lbeg[t + 1]; ++e) b[lidx[e]] -= lval[e] * bt;
    }
    for (int t = k - 1; t >= 0; --t) {
      double s = b[prow[t]];
      for (int e = ubeg[t]; e < ubeg[t + 1]; ++e) s -= uval[e] * z[uidx[e]];
      z[pcol[t]] = s / piv[t];
    }
  }

  // kernel solve M' y = c: c by kernel column (consumed), y by kernel row
  void lu_solve_t(std::vector<double>& c, std::vector<double>& y) {
    for (int t = 0; t < k; ++t) {
      const double h = c[pcol[t]] / piv[t];
      y[prow[t]] = h;  // provisional: h_t, finished by the L' pass below
      if (h == 0.0) continue;
      for (int e = ubeg[t]; e < ubeg[t + 1]; ++e) c[uidx[e]] -= uval[e] * h;
    }
    for (int t = k - 1; t >= 0; --t) {
      double s = y[prow[t]];
      for (int e = lbeg[t]; e < lbeg[t + 1]; ++e) s -= lval[e] * y[lidx[e]];
      y[prow[t]] = s;
    }
  }

  void refactor() {
    etas.clear();
    // Basis repair: a numerically dependent structural column is replaced by
    // the slack of a row the factorization could not pivot on, keeping the
    // rest of the warm basis. Only if that fails is the slack basis used.
    for (int attempt = 0; attempt <= m; ++attempt) {
      if (factor_kernel()) {
        factored = true;
        return;
      }
      if (fail_col < 0) break;
      const int out = kvar[fail_col], p = kpos[fail_col], r = krow[fail_row];
      const int sl = slack_of_row[r];
      log_debug("simplex: singular basis, swapping a dependent column for a slack");
      basis[p] = sl;
      pos[sl] = p;
      st[sl] = St::Basic;
      pos[out] = -1;
      st[out] = initial_state(v[out].lo, v[out].up);
      if (std::isfinite(v[out].up) && std::isfinite(v[out].lo) &&
          std::fabs(x[out] - v[out].up) < std::fabs(x[out] - v[out].lo))
        st[out] = St::Upper;
      x[out] = st[out] == St::Upper ? v[out].up : initial_value(v[out].lo, v[out].up);
    }
    log_debug("simplex: basis repair failed, falling back to the slack basis");
    for (int j = 0; j < nv(); ++j) {
      if (st[j] == St::Basic && v[j].slack_row < 0) {
        st[j] = initial_state(v[j].lo, v[j].up);
        x[j] = initial_value(v[j].lo, v[j].up);
        pos[j] = -1;
      }
    }
    for (int j = 0; j < nv(); ++j)
      if (v[j].slack_row >= 0) {
        basis[v[j].slack_row] = j;
        pos[j] = v[j].slack_row;
        st[j] = St::Basic;
      }
    if (!factor_kernel()) throw std::runtime_error("simplex: basis factorization failed");
    factored = true;
  }

  // B w = a  (a by rows, w by basis positions)
  void ftran(const std::vector<double>& a, std::vector<double>& w) {
    w.assign(m, 0.0);
    if (k > 0) {
      for (int i = 0; i < k; ++i) tk2[i] = a[krow[i]];
      lu_solve(tk2, tk1);  // tk1: kernel column order
      for (int i = 0; i < k; ++i) w[kpos[i]] = tk1[i];
    }
    for (int r = 0; r < m; ++r)
      if (slack_pos[r] >= 0) w[slack_pos[r]] = a[r];
    for (int i = 0; i < k; ++i) {
      const double z = tk1[i];
      if (z == 0.0) continue;
      for (const auto& [r, c] : v[kvar[i]].col)
        if (slack_pos[r] >= 0) w[slack_pos[r]] -= c * z;
    }
    for (const Eta& e : etas) {
      const double t = w[e.p] / e.piv;
      if (t != 0.0)
        for (std::size_t q = 0; q < e.idx.size(); ++q) w[e.idx[q]] -= t * e.val[q];
      w[e.p] = t;
    }
  }

  // B' y = c  (c by basis positions, consumed; y by rows)
  void btran(std::vector<double>& c, std::vector<double>& y) {
    for (auto it = etas.rbegin(); it != etas.rend(); ++it) {
      double s = c[it->p];
      for (std::size_t q = 0; q < it->idx.size(); ++q) s -= it->val[q] * c[it->idx[q]];
      c[it->p] = s / it->piv;
    }
    y.assign(m, 0.0);
    for (int r = 0; r < m; ++r)
      if (slack_pos[r] >= 0) y[r] = c[slack_pos[r]];
    if (k == 0) return;
    for (int i = 0; i < k; ++i) {
      double s = c[kpos[i]];
      for (const auto& [r, a] : v[kvar[i]].col)
        if (slack_pos[r] >= 0) s -= a * y[r];
      tk1[i] = s;
    }
    lu_solve_t(tk1, tk2);  // tk1 by kernel column -> tk2 by kernel row
    for (int i = 0; i < k; ++i) y[krow[i]] = tk2[i];
  }

  void recompute_basics() {
    if (!factored) refactor();
    std::vector<double> a(rhs);
    for (int j = 0; j < nv(); ++j) {
      if (st[j] == St::Basic || x[j] == 0.0) continue;
      for (const auto& [r, c] : v[j].col) a[r] -= c * x[j];
    }
    std::vector<double> w;
    ftran(a, w);
    for (int p = 0; p < m; ++p) x[basis[p]] = w[p];
    basics_stale = false;
  }

  double max_violation() const {
    double worst = 0.0;
    for (int p = 0; p < m; ++p) {
      const int j = basis[p];
      worst = std::max(worst, v[j].lo - x[j]);
      worst = std::max(worst, x[j] - v[j].up);
    }
    return worst;
  }

  // ------------------------------------------------------------- phases
  LpStatus run_phase(bool phase1) {
    const double ftol = opt.feas_tol;
    double cmax = 1.0;
    if (!phase1)
      for (const auto& var : v) cmax = std::max(cmax, std::fabs(var.cost));
    const double dtol = phase1 ? opt.opt_tol : opt.opt_tol * cmax;
    std::vector<double> cb(m), y, w, rc(m), rho, aq(m, 0.0);
    std::vector<double> ref(nv(), 1.0);
    // Phase 2 keeps the reduced costs d_j = c_j - y'A_j across iterations and
    // updates them from the pivot row the devex step already computes
    // (d_j -= (d_q / alpha_q) alpha_j), which saves one btran and one pass
    // over the columns per iteration. They are recomputed from a fresh btran
    // after every refactorization, after a Bland pivot, and before optimality
    // is declared.
    std::vector<double> d(nv(), 0.0);
    bool d_valid = false;
    // Row-wise copy of the constraint matrix, so the devex pivot row
    // alpha_j = rho'A_j visits only the rows where rho is nonzero (rho is
    // usually sparse). Columns are stored in ascending row order, so each
    // alpha_j accumulates its terms in ascending row order, as a
    // column-wise dot product would.
    std::vector<int> rbeg(m + 1, 0), rvar;
    std::vector<double> rval, alpha(nv(), 0.0);
    for (int j = 0; j < nv(); ++j)
      for (const auto& rc_ : v[j].col) ++rbeg[rc_.first + 1];
    for (int r = 0; r < m; ++r) rbeg[r + 1] += rbeg[r];
    rvar.resize(rbeg[m]);
    rval.resize(rbeg[m]);
    {
      std::vector<int> fill(rbeg.begin(), rbeg.end() - 1);
      for (int j = 0; j < nv(); ++j)
        for (const auto& [r, c] : v[j].col) {
          rvar[fill[r]] = j;
          rval[fill[r]++] = c;
        }
    }
    struct Cand {
      int p;
      double t, mag;
      bool up;
    };
    std::vector<Cand> cand;
    cand.reserve(m);
    int stall = 0;
    bool bland = false;
    for (;;) {
      if (++iters > opt.max_iters) throw std::runtime_error("simplex: iteration limit exceeded");
      if (log_level() >= LogLevel::Debug && iters % 2000 == 0)
        log_debug("simplex iter " + std::to_string(iters) + (phase1 ? " phase1" : " phase2") +
                  " obj " + std::to_string(objective_value()) + " stall " + std::to_string(stall) +
                  (bland ? " bland" : "") + " violation " + std::to_string(max_violation()));
      bool infeasible = false;
      for (int p = 0; p < m; ++p) {
        const int j = basis[p];
        double c;
        if (phase1) {
          c = x[j] < v[j].lo - ftol ? 1.0 : (x[j] > v[j].up + ftol ? -1.0 : 0.0);
          infeasible = infeasible || c != 0.0;
        } else {
          c = v[j].cost;
        }
        cb[p] = c;
      }
      if (phase1 && !infeasible) return LpStatus::Optimal;
      if (!phase1 && max_violation() > ftol) {
        lost_feasibility = true;  // roundoff pushed a basic out of bounds: repair in phase 1
        return LpStatus::Optimal;
      }
      const bool incremental = !phase1 && d_valid;
      if (!incremental) {
        btran(cb, y);
        // y'A_j for every column, row-wise over the nonzeros of y (same
        // per-column summation order as a column-wise dot product)
        std::fill(alpha.begin(), alpha.end(), 0.0);
        for (int r = 0; r < m; ++r) {
          const double yr = y[r];
          if (yr == 0.0) continue;
          for (int t = rbeg[r]; t < rbeg[r + 1]; ++t) alpha[rvar[t]] += rval[t] * yr;
        }
      }

      int q = -1, dir = 0;
      double best = 0.0;
      for (int j = 0; j < nv(); ++j) {
        const St s = st[j];
        if (s == St::Basic || v[j].lo == v[j].up) continue;
        double dj;
        if (incremental) {
          dj = d[j];
        } else {
          dj = (phase1 ? 0.0 : v[j].cost) - alpha[j];
          d[j] = dj;
        }
        int cd = 0;
        if ((s == St::Lower || s == St::Free) && dj > dtol)
          cd = 1;
        else if ((s == St::Upper || s == St::Free) && dj < -dtol)
          cd = -1;
        if (cd == 0) continue;
        if (bland) {
          q = j;
          dir = cd;
          break;
        }
        const double score = dj * dj / ref[j];
        if (score > best) {
          best = score;
          q = j;
          dir = cd;
        }
      }
      if (q < 0 && incremental) {  // confirm optimality on fresh reduced costs
        d_valid = false;
        --iters;
        continue;
      }
      if (q < 0) return phase1 ? LpStatus::Infeasible : LpStatus::Optimal;
      if (!phase1 && !bland) d_valid = true;

      std::fill(aq.begin(), aq.end(), 0.0);
      for (const auto& [r, c] : v[q].col) aq[r] = c;
      ftran(aq, w);

      // Harris two-pass ratio test. Pass 1 bounds the step with every bound
      // relaxed by the feasibility tolerance; pass 2 takes, among the rows
      // blocking within that step, the one with the largest pivot (then the
      // lowest variable index; Bland: lowest index only). The leaving
      // variable's bound is shifted onto its value if it ends slightly
      // outside (no snapping residual); shifts are undone in optimize().
      const double flip = (std::isfinite(v[q].lo) && std::isfinite(v[q].up)) ? v[q].up - v[q].lo
                                                                               : kInf;
      cand.clear();
      double tmax = flip, wmax = 0.0;
      for (int p = 0; p < m; ++p) wmax = std::max(wmax, std::fabs(w[p]));
      const double ptol = std::max(opt.pivot_tol, 1e-11 * wmax);
      for (int p = 0; p < m; ++p) {
        if (std::fabs(w[p]) <= ptol) continue;
        const int j = basis[p];
        const double rate = -dir * w[p];
        double t = kInf, trel = kInf;
        bool up = false;
        if (rate > 0.0) {
          if (phase1 && x[j] < v[j].lo - ftol) {
            t = trel = (v[j].lo - x[j]) / rate;  // becomes feasible at its lower bound
          } else if (std::isfinite(v[j].up)) {
            t = (v[j].up - x[j]) / rate;
            trel = (v[j].up + ftol - x[j]) / rate;
            up = true;
          }
        } else {
          if (phase1 && x[j] > v[j].up + ftol) {
            t = trel = (x[j] - v[j].up) / -rate;
            up = true;
          } else if (std::isfinite(v[j].lo)) {
            t = (x[j] - v[j].lo) / -rate;
            trel = (x[j] - v[j].lo + ftol) / -rate;
          }
        }
        if (t == kInf) continue;
        cand.push_back(Cand{p, t, std::fabs(w[p]), up});
        tmax = std::min(tmax, trel);
      }
      int leave = -1;
      bool leave_up = false;
      double theta = flip;
      if (!(flip < kInf && flip <= tmax)) {
        double bmag = -1.0;
        for (const Cand& c : cand) {
          if (c.t > tmax) continue;
          const int j = basis[c.p];
          bool take;
          if (leave < 0) take = true;
          else if (bland) take = j < basis[leave];
          else take = c.mag > bmag * (1.0 + 1e-12) ||
                      (c.mag >= bmag * (1.0 - 1e-12) && j < basis[leave]);
          if (take) {
            leave = c.p;
            leave_up = c.up;
            theta = std::max(c.t, 0.0);
            bmag = c.mag;
          }
        }
      }
      if (theta == kInf) {
        if (phase1) throw std::runtime_error("simplex: unbounded phase-1 direction");
        return LpStatus::Unbounded;
      }

      // devex reference-weight update from the pivot row
      if (leave >= 0 && !bland) {
        const double ap = w[leave];
        std::fill(rc.begin(), rc.end(), 0.0);
        rc[leave] = 1.0;
        btran(rc, rho);
        const double wq = ref[q];
        const double td = d[q] / ap;  // dual step (phase 2 reduced-cost update)
        double rmax = 0.0;
        std::fill(alpha.begin(), alpha.end(), 0.0);
        for (int r = 0; r < m; ++r) {
          const double rr = rho[r];
          if (rr == 0.0) continue;
          for (int t = rbeg[r]; t < rbeg[r + 1]; ++t) alpha[rvar[t]] += rval[t] * rr;
        }
        for (int j = 0; j < nv(); ++j) {
          if (st[j] == St::Basic || j == q || v[j].lo == v[j].up) continue;
          const double al = alpha[j];
          if (al == 0.0) continue;
          d[j] -= td * al;
          const double cand = (al / ap) * (al / ap) * wq;
          if (cand > ref[j]) ref[j] = cand;
          rmax = std::max(rmax, ref[j]);
        }
        ref[basis[leave]] = std::max(wq / (ap * ap), 1.0);
        d[basis[leave]] = -td;
        d[q] = 0.0;
        if (rmax > 1e7) std::fill(ref.begin(), ref.end(), 1.0);
      }

      if (leave >= 0 && bland) d_valid = false;

      // move
      if (theta != 0.0) {
        for (int p = 0; p < m; ++p)
          if (w[p] != 0.0) x[basis[p]] -= dir * theta * w[p];
        x[q] += dir * theta;
      }
      if (leave < 0) {
        st[q] = dir > 0 ? St::Upper : St::Lower;
        x[q] = dir > 0 ? v[q].up : v[q].lo;
      } else {
        const int out = basis[leave];
        st[out] = leave_up ? St::Upper : St::Lower;
        if (leave_up) {
          if (x[out] > v[out].up) v[out].up = x[out];  // shift (<= ftol)
          else x[out] = v[out].up;
        } else {
          if (x[out] < v[out].lo) v[out].lo = x[out];
          else x[out] = v[out].lo;
        }
        pos[out] = -1;
        basis[leave] = q;
        pos[q] = leave;
        st[q] = St::Basic;
        Eta e;
        e.p = leave;
        e.piv = w[leave];
        for (int p = 0; p < m; ++p)
          if (p != leave && w[p] != 0.0) {
            e.idx.push_back(p);
            e.val.push_back(w[p]);
          }
        etas.push_back(std::move(e));
        if (static_cast<int>(etas.size()) >= kEtaLimit || std::fabs(w[leave]) < 1e-8) {
          refactor();
          recompute_basics();
          d_valid = false;
        }
      }
      if (theta <= 1e-12) {
        if (++stall > kStallLimit) bland = true;
      } else {
        stall = 0;
        if (bland) {
          bland = false;
          std::fill(ref.begin(), ref.end(), 1.0);
        }
      }
    }
  }

  bool lost_feasibility = false;

  LpStatus solve_rounds() {
    for (int round = 0; round < 40; ++round) {
      LpStatus s = LpStatus::Optimal;
      if (max_violation() > opt.feas_tol) s = run_phase(true);
      if (s != LpStatus::Optimal) return s;
      const long before = iters;
      lost_feasibility = false;
      s = run_phase(false);
      const double drift = max_violation();
      refactor();
      recompute_basics();
      if (log_level() >= LogLevel::Debug)
        log_debug("simplex round " + std::to_string(round) + ": " + std::to_string(iters - before) +
                  " phase-2 iters, violation " + std::to_string(drift) + " -> " +
                  std::to_string(max_violation()) + ", k=" + std::to_string(k) + ", m=" + std::to_string(m));
      if (s != LpStatus::Optimal) return s;
      if (!lost_feasibility && max_violation() <= opt.feas_tol) return s;
    }
    throw std::runtime_error("simplex: no feasible optimum after repeated repair");
  }

  void snap(int j) {
    if (st[j] == St::Lower) x[j] = v[j].lo;
    else if (st[j] == St::Upper) x[j] = v[j].up;
  }

  void save_bounds() {
    saved_lo.resize(nv());
    saved_up.resize(nv());
    for (int j = 0; j < nv(); ++j) {
      saved_lo[j] = v[j].lo;
      saved_up[j] = v[j].up;
    }
  }

  void perturb() {
    save_bounds();
    for (int j = 0; j < nv(); ++j) {
      if (v[j].lo == v[j].up) continue;
      if (std::isfinite(v[j].lo)) v[j].lo -= kShift * shift_unit(j, 0);
      if (std::isfinite(v[j].up)) v[j].up += kShift * shift_unit(j, 1);
      snap(j);
    }
  }

  void restore() {
    for (int j = 0; j < nv(); ++j) {
      v[j].lo = saved_lo[j];
      v[j].up = saved_up[j];
      snap(j);
    }
  }

  LpStatus optimize() {
    if (!factored) refactor();
    // pass 1: perturbed bounds (degeneracy), pass 2: exact bounds; Harris
    // shifts made in either pass are dropped by restore()
    perturb();
    recompute_basics();
    LpStatus s = solve_rounds();
    restore();
    recompute_basics();
    if (s != LpStatus::Optimal) return s;
    for (int attempt = 0; attempt < 4; ++attempt) {
      save_bounds();
      s = solve_rounds();
      restore();
      recompute_basics();
      if (s != LpStatus::Optimal) return s;
      if (max_violation() <= opt.feas_tol) return s;
    }
    if (max_violation() <= 10 * opt.feas_tol) return s;
    throw std::runtime_error("simplex: could not remove bound shifts");
  }

  double objective_value() const {
    double s = 0.0;
    for (int j : structural) s += v[j].cost * x[j];
    return s;
  }
};

SimplexSolver::SimplexSolver(const LinearProgram& prog, SimplexOptions opts)
    : impl_(new Impl(prog, opts)) {}

SimplexSolver::~SimplexSolver() { delete impl_; }

LpStatus SimplexSolver::optimize() { return impl_->optimize(); }

void SimplexSolver::reset() { impl_->reset_basis(); }

void SimplexSolver::set_objective(const Eigen::VectorXd& c) {
  if (c.size() != static_cast<Eigen::Index>(impl_->structural.size()))
    throw MalformedProgram("set_objective: size must equal num_vars()");
  for (std::size_t i = 0; i < impl_->structural.size(); ++i) {
    if (std::isnan(c(static_cast<Eigen::Index>(i))))
      throw MalformedProgram("set_objective: NaN coefficient");
    impl_->v[impl_->structural[i]].cost = c(static_cast<Eigen::Index>(i));
  }
}

void SimplexSolver::set_bounds(int var, double lo, double hi) {
  if (var < 0 || var >= static_cast<int>(impl_->structural.size()))
    throw MalformedProgram("set_bounds: unknown variable");
  if (std::isnan(lo) || std::isnan(hi) || lo > hi) throw MalformedProgram("set_bounds: lo > hi");
  const int j = impl_->structural[var];
  impl_->v[j].lo = lo;
  impl_->v[j].up = hi;
  if (impl_->st[j] == Impl::St::Basic) return;
  impl_->st[j] = Impl::initial_state(lo, hi);
  const double nx = Impl::initial_value(lo, hi);
  if (nx != impl_->x[j]) {
    impl_->x[j] = nx;
    impl_->basics_stale = true;
  }
}

int SimplexSolver::add_var(double lo, double hi, double obj_coeff) {
  impl_->add_structural(lo, hi, obj_coeff);
  return static_cast<int>(impl_->structural.size()) - 1;
}

int SimplexSolver::add_row(const std::vector<std::pair<int, double>>& coeffs, Relation rel,
                           double rhs) {
  std::vector<std::pair<int, double>> c;
  c.reserve(coeffs.size());
  for (const auto& [j, a] : coeffs) {
    if (j < 0 || j >= static_cast<int>(impl_->structural.size()))
      throw MalformedProgram("add_row: unknown variable");
    c.emplace_back(impl_->structural[j], a);
  }
  const int slack = impl_->append_row(c, rel, rhs);
  impl_->basis.push_back(slack);
  impl_->pos[slack] = impl_->m - 1;
  impl_->st[slack] = Impl::St::Basic;
  impl_->factored = false;
  impl_->basics_stale = true;
  return impl_->m - 1;
}

int SimplexSolver::num_vars() const { return static_cast<int>(impl_->structural.size()); }

double SimplexSolver::objective_value() const {
  if (impl_->basics_stale) impl_->recompute_basics();
  return impl_->objective_value();
}

Eigen::VectorXd SimplexSolver::solution() const {
  if (impl_->basics_stale) impl_->recompute_basics();
  Eigen::VectorXd out(static_cast<Eigen::Index>(impl_->structural.size()));
  for (std::size_t i = 0; i < impl_->structural.size(); ++i)
    out(static_cast<Eigen::Index>(i)) = impl_->x[impl_->structural[i]];
  return out;
}

long SimplexSolver::iterations() const { return impl_->iters; }

LpSolution solve(const LinearProgram& prog, const SimplexOptions& opts) {
  SimplexSolver s(prog, opts);
  LpSolution out;
  out.status = s.optimize();
  out.x = s.solution();
  out.iterations = s.iterations();
  if (out.status == LpStatus::Optimal) out.objective = s.objective_value();
  return out;
}

}  // namespace swarmplan::lp
