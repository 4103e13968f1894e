// strategy.cpp — the DeDLOC load balancer (Eq. 1 -> Eq. 5,
// Appendix B) that decides which share of the flattened gradient vector each
// peer aggregates. Semantics restated from the reference
// (/root/reference/proj/src/strategy.cpp):
//   classify            :35-59   computing / recipient sets and unit scales
//   build_lp            :76-177  full program (O(n^3) service rows)
//   build_compact       :193-295 per-reducer M_i compaction + presolve
//   solve_strategy      :299-500 stage A (relaxed xi), 0/1 duty-cycle
//                                restriction, B (max compute), C (max service
//                                floor), D (min flow), fractions
//   round models        :502-532
// Only the linear algebra underneath (swarmplan::lp) is new.

#include "swarmplan/strategy.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <functional>
#include <sstream>

#include "swarmplan/log.hpp"

namespace swarmplan::strategy {

namespace {

constexpr double kBig = 1024.0;  // stands in for an unbounded scaled flow
constexpr double kXiCap = 4.0;   // xi is scaled so the compute bound is 1

struct PeerSets {
  std::vector<int> computing, recipients;
  std::vector<bool> is_computing, is_recipient;
  double flow_scale = 1.0;  // U: bit/s per flow unit (largest peer capacity)
  double xi_scale = 1.0;    // steps/s per xi unit
};

PeerSets classify(const CollaborationSpec& spec, bool communication_only) {
  PeerSets s;
  const int n = spec.size();
  s.is_computing.assign(n, false);
  s.is_recipient.assign(n, false);
  double rate = 0.0, cap = 0.0;
  for (int i = 0; i < n; ++i) {
    const PeerSpec& p = spec.peers[i];
    if (p.can_compute && p.samples_per_sec > 0) {
      s.computing.push_back(i);
      s.is_computing[i] = true;
      rate += p.samples_per_sec;
    }
    if (p.can_compute && !p.client_mode) {
      s.recipients.push_back(i);
      s.is_recipient[i] = true;
    }
    cap = std::max({cap, p.download_bps, p.upload_bps});
  }
  s.flow_scale = cap > 0 ? cap : 1.0;
  s.xi_scale = communication_only ? s.flow_scale / spec.payload_bits() : rate / spec.batch_size;
  return s;
}

void require_valid(const CollaborationSpec& spec) {
  const auto bad = validate(spec);
  if (bad.empty()) return;
  std::ostringstream os;
  os << "invalid collaboration spec:";
  for (const Violation& v : bad) {
    os << " [";
    if (v.peer >= 0) os << spec.peers[v.peer].id << ".";
    os << v.field << ": " << v.message << "]";
  }
  throw std::invalid_argument(os.str());
}

using Terms = std::vector<std::pair<int, double>>;

// Per-peer wire capacity rows shared by both program forms: inbound (a + g
// from every other peer) <= d_i, outbound <= u_i, and per-link limits.
template <class AddRow, class IdxA, class IdxG>
void add_capacity_rows(const CollaborationSpec& spec, double U, IdxA a, IdxG g, AddRow add,
                       int* n_down, int* n_up, int* n_link) {
  const int n = spec.size();
  for (int i = 0; i < n; ++i) {
    Terms t;
    for (int j = 0; j < n; ++j)
      if (j != i) {
        t.emplace_back(a(j, i), 1.0);
        t.emplace_back(g(j, i), 1.0);
      }
    add(std::move(t), spec.peers[i].download_bps / U);
    if (n_down) ++*n_down;
  }
  for (int i = 0; i < n; ++i) {
    Terms t;
    for (int j = 0; j < n; ++j)
      if (j != i) {
        t.emplace_back(a(i, j), 1.0);
        t.emplace_back(g(i, j), 1.0);
      }
    add(std::move(t), spec.peers[i].upload_bps / U);
    if (n_up) ++*n_up;
  }
  for (const LinkLimit& l : spec.links) {
    if (!std::isfinite(l.bps)) continue;
    add(Terms{{a(l.from, l.to), 1.0}, {g(l.from, l.to), 1.0}}, l.bps / U);
    if (n_link) ++*n_link;
  }
}

struct Compact {
  lp::LinearProgram prog;
  int n = 0;
  PeerSets sets;
  int a(int i, int j) const { return i * n + j; }
  int g(int i, int j) const { return n * n + i * n + j; }
  int c(int i) const { return 2 * n * n + i; }
  int xi() const { return 2 * n * n + n; }
  int M(int i) const { return 2 * n * n + n + 1 + i; }
};

Compact build_compact(const CollaborationSpec& spec, bool communication_only) {
  Compact cp;
  const int n = cp.n = spec.size();
  cp.sets = classify(spec, communication_only);
  const PeerSets& s = cp.sets;
  const double U = s.flow_scale, Xi = s.xi_scale, P = spec.payload_bits();
  lp::LinearProgram& prog = cp.prog = lp::LinearProgram(2 * n * n + 2 * n + 1);

  for (int q = 0; q < 2 * n * n; ++q) prog.upper(q) = kBig;
  for (int i = 0; i < n; ++i) {
    if (communication_only || !s.is_computing[i]) {
      const double pin = communication_only && s.is_computing[i] ? 1.0 : 0.0;
      prog.lower(cp.c(i)) = pin;
      prog.upper(cp.c(i)) = pin;
    } else {
      prog.upper(cp.c(i)) = 1.0;
    }
    prog.upper(cp.M(i)) = kBig;
  }
  prog.upper(cp.xi()) = kXiCap;
  prog.objective(cp.xi()) = 1.0;

  // presolve: clients take no inbound flow, non-computing peers send no
  // gradients, non-recipients receive no averaged parts
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (j != i && spec.peers[j].client_mode) {
        prog.upper(cp.a(i, j)) = 0.0;
        prog.upper(cp.g(i, j)) = 0.0;
      }
      if (!s.is_computing[i]) prog.upper(cp.a(i, j)) = 0.0;
      if (!s.is_recipient[j]) prog.upper(cp.g(i, j)) = 0.0;
    }

  auto add = [&](Terms t, double rhs) { prog.add_row(std::move(t), lp::Relation::LessEq, rhs); };
  if (!communication_only) {  // xi <= sum_k s_k c_k / B
    Terms t{{cp.xi(), 1.0}};
    for (int k : s.computing) t.emplace_back(cp.c(k), -spec.peers[k].samples_per_sec / (spec.batch_size * Xi));
    add(std::move(t), 0.0);
  }
  for (int i : s.recipients) {  // every recipient receives a full model per step
    Terms t{{cp.xi(), 1.0}};
    for (int j = 0; j < n; ++j) t.emplace_back(cp.g(j, i), -U / (P * Xi));
    add(std::move(t), 0.0);
  }
  if (!s.recipients.empty()) {
    for (int i = 0; i < n; ++i) {
      for (int j : s.recipients) add(Terms{{cp.g(i, j), 1.0}, {cp.M(i), -1.0}}, 0.0);
      const double di = spec.peers[i].download_bps / U;
      for (int k : s.computing)
        add(Terms{{cp.M(i), 1.0}, {cp.a(k, i), -1.0}, {cp.c(k), di}}, di);
    }
  }
  add_capacity_rows(
      spec, U, [&](int i, int j) { return cp.a(i, j); }, [&](int i, int j) { return cp.g(i, j); },
      add, nullptr, nullptr, nullptr);
  return cp;
}

}  // namespace

StrategyProblem build_lp(const CollaborationSpec& spec) {
  require_valid(spec);
  const int n = spec.size();
  const PeerSets s = classify(spec, false);
  const double U = s.flow_scale, Xi = s.xi_scale, P = spec.payload_bits();
  StrategyProblem sp;
  sp.n = n;
  sp.a_base = 0;
  sp.g_base = n * n;
  sp.c_base = 2 * n * n;
  sp.xi_var = 2 * n * n + n;
  sp.flow_scale = U;
  sp.xi_scale = Xi;
  lp::LinearProgram prog(2 * n * n + n + 1);
  for (int q = 0; q < 2 * n * n; ++q) prog.upper(q) = kBig;
  for (int i = 0; i < n; ++i) prog.upper(sp.c(i)) = spec.peers[i].can_compute ? 1.0 : 0.0;
  prog.upper(sp.xi_var) = kXiCap;
  prog.objective(sp.xi_var) = 1.0;
  for (int i = 0; i < n; ++i) {
    if (!spec.peers[i].client_mode) continue;
    for (int j = 0; j < n; ++j)
      if (j != i) {
        prog.upper(sp.a(j, i)) = 0.0;
        prog.upper(sp.g(j, i)) = 0.0;
      }
  }
  auto add = [&](Terms t, double rhs) { prog.add_row(std::move(t), lp::Relation::LessEq, rhs); };
  {
    Terms t{{sp.xi_var, 1.0}};
    for (int i = 0; i < n; ++i)
      if (spec.peers[i].can_compute)
        t.emplace_back(sp.c(i), -spec.peers[i].samples_per_sec / (spec.batch_size * Xi));
    add(std::move(t), 0.0);
    sp.rows_compute = 1;
  }
  for (int i : s.recipients) {
    Terms t{{sp.xi_var, 1.0}};
    for (int j = 0; j < n; ++j) t.emplace_back(sp.g(j, i), -U / (P * Xi));
    add(std::move(t), 0.0);
    ++sp.rows_aggregate;
  }
  // service: reducer i forwards no faster than its slowest gradient arrival
  // (an idle share of peer k is fetched at d_i instead)
  for (int i = 0; i < n; ++i) {
    const double di = spec.peers[i].download_bps / U;
    for (int j = 0; j < n; ++j)
      for (int k : s.computing) {
        add(Terms{{sp.g(i, j), 1.0}, {sp.a(k, i), -1.0}, {sp.c(k), di}}, di);
        ++sp.rows_service;
      }
  }
  add_capacity_rows(
      spec, U, [&](int i, int j) { return sp.a(i, j); }, [&](int i, int j) { return sp.g(i, j); },
      add, &sp.rows_download, &sp.rows_upload, &sp.rows_link);
  sp.prog = std::move(prog);
  return sp;
}

// Canonical tie-break among optimal strategies. Peers with identical specs
// (and the same duty cycle in the solution) are interchangeable: permuting
// them maps the program of every stage onto itself, so averaging the
// solution over those permutations stays feasible and keeps every stage's
// objective (linear ones exactly, stage C's concave sum of minima cannot
// drop below its optimum). The vertex the simplex stops at is arbitrary when
// the optimum is not unique -- two identical peers can come back as
// fractions [1, 0] ("multiple optimal strategies with equal
// training throughputs") -- while the averaged point is the symmetric one
// (an interior-point solver's answer). Peers named in a
// per-link limit keep their own class.
static void symmetrize(const CollaborationSpec& spec, StrategyAssignment& out) {
  const int n = spec.size();
  std::vector<int> cls(n, -1);
  std::vector<std::vector<int>> members;
  std::vector<bool> linked(n, false);
  for (const LinkLimit& l : spec.links) {
    if (l.from >= 0 && l.from < n) linked[l.from] = true;
    if (l.to >= 0 && l.to < n) linked[l.to] = true;
  }
  for (int i = 0; i < n; ++i) {
    const PeerSpec& p = spec.peers[i];
    for (std::size_t k = 0; k < members.size() && cls[i] < 0; ++k) {
      const int j = members[k][0];
      const PeerSpec& q = spec.peers[j];
      if (!linked[i] && !linked[j] && p.samples_per_sec == q.samples_per_sec &&
          p.download_bps == q.download_bps && p.upload_bps == q.upload_bps &&
          p.can_compute == q.can_compute && p.client_mode == q.client_mode &&
          out.compute[i] == out.compute[j] && std::fabs(out.c_raw[i] - out.c_raw[j]) <= 1e-9)
        cls[i] = static_cast<int>(k);
    }
    if (cls[i] < 0) {
      cls[i] = static_cast<int>(members.size());
      members.push_back({});
    }
    members[cls[i]].push_back(i);
  }
  if (static_cast<int>(members.size()) == n) return;  // no two peers interchangeable
  for (Eigen::MatrixXd* mat : {&out.a, &out.g}) {
    Eigen::MatrixXd& m = *mat;
    const Eigen::MatrixXd src = m;
    for (const auto& A : members)
      for (const auto& B : members) {
        double off = 0.0, diag = 0.0;
        int noff = 0, ndiag = 0;
        for (int i : A)
          for (int j : B) {
            if (i == j) {
              diag += src(i, j);
              ++ndiag;
            } else {
              off += src(i, j);
              ++noff;
            }
          }
        for (int i : A)
          for (int j : B) m(i, j) = i == j ? diag / ndiag : off / noff;
      }
  }
  for (const auto& A : members) {
    double c = 0.0;
    for (int i : A) c += out.c_raw[i];
    for (int i : A) out.c_raw[i] = c / A.size();
  }
}

StrategyAssignment solve_strategy(const CollaborationSpec& spec, const SolveOptions& opts) {
  require_valid(spec);
  const int n = spec.size();
  Compact cp = build_compact(spec, opts.communication_only);
  const PeerSets& s = cp.sets;
  const double U = s.flow_scale;
  lp::SimplexSolver solver(cp.prog, opts.simplex);

  const auto t0 = std::chrono::steady_clock::now();
  long last_iters = 0;
  auto stage = [&](const char* what) {
    if (log_level() < LogLevel::Debug) return;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    log_debug(std::string("solve_strategy ") + what + ": +" +
              std::to_string(solver.iterations() - last_iters) + " iters, " + std::to_string(ms) +
              " ms");
    last_iters = solver.iterations();
  };
  auto must = [&](lp::LpStatus st, const char* msg) {
    if (st != lp::LpStatus::Optimal) throw std::runtime_error(msg);
  };

  // stage A: continuous duty-cycle relaxation
  must(solver.optimize(), "strategy solve did not reach an optimum");
  stage("stage A");
  double xi_star = solver.solution()(cp.xi());

  // Deployable duty cycles are 0/1: if stage A left any c_k strictly inside
  // (0,1), re-solve with the 0/1 masks induced by thresholding the relaxed
  // c at each of its distinct levels (plus "all capable peers on") and keep
  // the best (ties: more computing peers).
  if (!opts.communication_only && !s.computing.empty()) {
    const Eigen::VectorXd x0 = solver.solution();
    bool fractional = false;
    for (int k : s.computing) {
      const double ck = x0(cp.c(k));
      fractional = fractional || (ck > 1e-7 && ck < 1.0 - 1e-7);
    }
    if (fractional) {
      std::vector<double> levels;
      for (int k : s.computing)
        if (x0(cp.c(k)) > 1e-7) levels.push_back(std::min(x0(cp.c(k)), 1.0));
      std::sort(levels.begin(), levels.end(), std::greater<double>());
      levels.erase(std::unique(levels.begin(), levels.end(),
                               [](double hi, double lo) { return hi - lo < 1e-9; }),
                   levels.end());
      levels.push_back(0.0);
      auto pin_mask = [&](const std::vector<bool>& mask) {
        solver.set_bounds(cp.xi(), 0.0, kXiCap);
        for (int k : s.computing) {
          const double pin = mask[k] ? 1.0 : 0.0;
          solver.set_bounds(cp.c(k), pin, pin);
        }
        // the relaxed vertex is far from feasible once c is pinned; the
        // slack basis (all flows zero) is feasible
        solver.reset();
        must(solver.optimize(), "strategy duty-cycle restriction failed");
      };
      double best_xi = -1.0;
      int best_on = -1, prev_on = -1;
      std::vector<bool> best_mask, applied;
      // Candidate masks. The threshold masks depend on which optimal vertex
      // stage A returned (the relaxed optimum is rarely unique), so for small
      // fleets (<= 3 computing peers, the range the reference's own
      // best-mask test covers, test_strategy.cpp:240-259) every nonempty
      // mask is tried instead; the result is then vertex-independent.
      std::vector<std::vector<bool>> masks;
      const int nc = static_cast<int>(s.computing.size());
      if (nc <= 3) {
        for (unsigned bits = (1u << nc) - 1; bits >= 1; --bits) {  // most peers first
          std::vector<bool> mask(n, false);
          for (int b = 0; b < nc; ++b) mask[s.computing[b]] = (bits >> b) & 1u;
          masks.push_back(std::move(mask));
        }
      } else {
        for (double level : levels) {
          std::vector<bool> mask(n, false);
          int on = 0;
          for (int k : s.computing)
            if (x0(cp.c(k)) >= level - 1e-12) {
              mask[k] = true;
              ++on;
            }
          if (on == 0 || on == prev_on) continue;
          prev_on = on;
          masks.push_back(std::move(mask));
        }
      }
      for (const std::vector<bool>& mask : masks) {
        int on = 0;
        for (int k : s.computing) on += mask[k] ? 1 : 0;
        pin_mask(mask);
        stage("duty restriction");
        applied = mask;
        const double xi = solver.solution()(cp.xi());
        const double tol = 1e-9 * std::max(1.0, std::fabs(best_xi));
        if (xi > best_xi + tol || (xi > best_xi - tol && on > best_on)) {
          best_xi = xi;
          best_on = on;
          best_mask = mask;
        }
      }
      if (applied != best_mask) {
        pin_mask(best_mask);
        stage("duty final");
      }
      xi_star = solver.solution()(cp.xi());
    }
  }
  solver.set_bounds(cp.xi(), xi_star, xi_star);

  // stage B: among xi-optimal strategies, maximize compute participation
  if (!opts.communication_only && !s.computing.empty()) {
    Eigen::VectorXd obj = Eigen::VectorXd::Zero(solver.num_vars());
    for (int k : s.computing) obj(cp.c(k)) = spec.peers[k].samples_per_sec;
    solver.set_objective(obj);
    must(solver.optimize(), "strategy stage B failed");
    stage("stage B");
    const Eigen::VectorXd xb = solver.solution();
    for (int k : s.computing) solver.set_bounds(cp.c(k), xb(cp.c(k)), xb(cp.c(k)));
  }

  // stage C: maximize sum_i f_i with f_i <= g_ij for every recipient j
  // (spreads aggregation over equivalent peers)
  if (!s.recipients.empty()) {
    std::vector<int> f(n);
    for (int i = 0; i < n; ++i) f[i] = solver.add_var(0.0, kBig, 0.0);
    for (int i = 0; i < n; ++i)
      for (int j : s.recipients)
        solver.add_row({{f[i], 1.0}, {cp.g(i, j), -1.0}}, lp::Relation::LessEq, 0.0);
    Eigen::VectorXd obj = Eigen::VectorXd::Zero(solver.num_vars());
    for (int i = 0; i < n; ++i) obj(f[i]) = 1.0;
    solver.set_objective(obj);
    must(solver.optimize(), "strategy stage C failed");
    stage("stage C");
    const Eigen::VectorXd xc = solver.solution();
    for (int i = 0; i < n; ++i) solver.set_bounds(f[i], xc(f[i]), xc(f[i]));
  }

  // stage D: least total flow achieving all of the above
  {
    Eigen::VectorXd obj = Eigen::VectorXd::Zero(solver.num_vars());
    for (int q = 0; q < 2 * n * n; ++q) obj(q) = -1.0;
    solver.set_objective(obj);
    must(solver.optimize(), "strategy stage D failed");
    stage("stage D");
  }

  const Eigen::VectorXd x = solver.solution();
  StrategyAssignment out;
  out.a = Eigen::MatrixXd::Zero(n, n);
  out.g = Eigen::MatrixXd::Zero(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      out.a(i, j) = std::max(0.0, x(cp.a(i, j)) * U);  // clip bound-level roundoff
      out.g(i, j) = std::max(0.0, x(cp.g(i, j)) * U);
    }
  out.c_raw.resize(n);
  out.compute.resize(n);
  for (int i = 0; i < n; ++i) {
    out.c_raw[i] = std::clamp(x(cp.c(i)), 0.0, 1.0);
    out.compute[i] = out.c_raw[i] >= 1.0 - 1e-6;
  }
  out.xi = x(cp.xi()) * s.xi_scale;
  out.lp_iterations = static_cast<int>(solver.iterations());
  symmetrize(spec, out);

  // fractions_i = min_{j in R} g_ij / sum_k min_{j in R} g_kj;
  // if every reducer misses some recipient, fall back to outbound mass
  out.fractions.assign(n, 0.0);
  if (!s.recipients.empty()) {
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
      double fl = kUnlimited;
      for (int j : s.recipients) fl = std::min(fl, out.g(i, j));
      out.fractions[i] = fl;
      total += fl;
    }
    if (total > 1e-9 * U) {
      for (double& f : out.fractions) f /= total;
    } else {
      total = 0.0;
      for (int i = 0; i < n; ++i) {
        double mass = 0.0;
        for (int j : s.recipients) mass += out.g(i, j);
        out.fractions[i] = mass;
        total += mass;
      }
      if (total > 0)
        for (double& f : out.fractions) f /= total;
    }
  }
  return out;
}

double allreduce_round_seconds(const CollaborationSpec& spec) {
  require_valid(spec);
  const int n = spec.size();
  if (n < 2) return 0.0;
  double w = kUnlimited;
  for (const PeerSpec& p : spec.peers) w = std::min({w, p.download_bps, p.upload_bps});
  for (const LinkLimit& l : spec.links) w = std::min(w, l.bps);
  return 2.0 * (double(n - 1) / n) * spec.payload_bits() / w;
}

double parameter_server_round_seconds(const CollaborationSpec& spec, int server) {
  require_valid(spec);
  const int n = spec.size();
  if (server < 0 || server >= n) throw std::invalid_argument("parameter server index out of range");
  if (n < 2) return 0.0;
  const double duplex = std::min(spec.peers[server].download_bps, spec.peers[server].upload_bps);
  return (n - 1) * spec.payload_bits() / duplex;
}

double adaptive_round_seconds(const CollaborationSpec& spec) {
  SolveOptions o;
  o.communication_only = true;
  const StrategyAssignment s = solve_strategy(spec, o);
  return s.xi > 0 ? 1.0 / s.xi : kUnlimited;
}

}  // namespace swarmplan::strategy
