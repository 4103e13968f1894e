// C++ API of strategy / partition / groups (the declarations callers of the
// reference compile against), exercised directly rather than via Python.
#include "harness.hpp"
#include "swarmplan/groups.hpp"
#include "swarmplan/partition.hpp"
#include "swarmplan/strategy.hpp"

using namespace swarmplan;

namespace {
CollaborationSpec homogeneous(int n, double s, double mbps, double batch, double params) {
  CollaborationSpec spec;
  spec.batch_size = batch;
  spec.param_count = params;
  for (int i = 0; i < n; ++i) {
    PeerSpec p;
    p.id = "peer" + std::to_string(i);
    p.samples_per_sec = s;
    p.download_bps = p.upload_bps = mbps * kMbps;
    spec.peers.push_back(p);
  }
  return spec;
}
}  // namespace

TEST_CASE("homogeneous8 golden through the C++ API") {
  CollaborationSpec spec = homogeneous(8, 1.0, 1000.0, 8.0, 25.6e6);
  StrategyAssignment s = strategy::solve_strategy(spec);
  CHECK(th::approx(s.xi, 0.697544642857, 1e-9));
  for (double f : s.fractions) CHECK(th::approx(f, 0.125, 1e-6));
  CHECK(s.a.rows() == 8 && s.g.cols() == 8);
}

TEST_CASE("reference program layout") {
  CollaborationSpec spec = homogeneous(2, 1.0, 100.0, 2.0, 1e6);
  spec.set_link_limit(0, 1, 20.0 * kMbps);
  spec.set_link_limit(1, 0, 30.0 * kMbps);
  strategy::StrategyProblem sp = strategy::build_lp(spec);
  CHECK(sp.prog.num_vars == 11);
  CHECK(sp.a(1, 0) == sp.a_base + 2);
  CHECK(sp.g(0, 1) == sp.g_base + 1);
  CHECK(sp.c(1) == sp.c_base + 1);
  for (int v = 0; v < sp.prog.num_vars; ++v) CHECK(sp.prog.objective(v) == (v == sp.xi_var ? 1.0 : 0.0));
}

TEST_CASE("fractions to part offsets") {
  CollaborationSpec spec = homogeneous(4, 1.0, 1000.0, 4.0, 1e6);
  StrategyAssignment s = strategy::solve_strategy(spec);
  std::vector<std::int64_t> off = part_offsets(17847474, s.fractions, 8);
  CHECK(off.size() == 5 && off.front() == 0 && off.back() == 17847474);
  for (int k = 1; k < 4; ++k) CHECK(off[k] % 8 == 0 && off[k] > off[k - 1]);
  CHECK_THROWS_AS(part_offsets(10, {0.5, -0.1}, 1), std::invalid_argument);
}

TEST_CASE("run_plan m = n is the weighted mean") {
  groups::GroupPlan plan = groups::build_plan(4, 4);
  Eigen::MatrixXd v(4, 1);
  v(0, 0) = 0.0;
  v(1, 0) = 0.0;
  v(2, 0) = 0.0;
  v(3, 0) = 4.0;
  groups::RunResult r = groups::run_plan(plan, v);
  for (int i = 0; i < 4; ++i) CHECK(r.values(i, 0) == 1.0 && r.complete[i]);
  r = groups::run_plan(plan, v, {1.0, 1.0, 1.0, 5.0});
  CHECK(r.values(0, 0) == 20.0 / 8.0);
}
