// swarmplan::lp::SimplexSolver warm-start API — ports of
// /root/reference/proj/tests/cpp/test_lp.cpp:292-376 (warm re-optimization,
// bound edits, incremental rows/variables, reset) and :241-250 (repeat).
#include <random>

#include "harness.hpp"
#include "swarmplan/lp.hpp"

using namespace swarmplan::lp;

namespace {
LinearProgram random_box_lp(std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  const int nv = 2 + static_cast<int>(rng() % 3);
  const int rows = 1 + static_cast<int>(rng() % 5);
  LinearProgram prog(nv);
  for (int j = 0; j < nv; ++j) {
    prog.upper(j) = 0.5 + 2.5 * unit(rng);
    prog.objective(j) = 2.0 * unit(rng) - 1.0;
  }
  for (int r = 0; r < rows; ++r) {
    std::vector<std::pair<int, double>> c;
    for (int j = 0; j < nv; ++j)
      if (unit(rng) < 0.8) c.push_back({j, 4.0 * unit(rng) - 2.0});
    if (c.empty()) c.push_back({0, 1.0});
    prog.add_row(std::move(c), (r == 0 && seed % 5 == 0) ? Relation::Eq : Relation::LessEq,
                 4.0 * unit(rng));
  }
  return prog;
}
}  // namespace

TEST_CASE("warm re-optimization matches a cold solve after objective edits") {
  int checked = 0;
  for (std::uint64_t seed = 300; seed < 340; ++seed) {
    LinearProgram prog = random_box_lp(seed);
    if (solve(prog).status != LpStatus::Optimal) continue;
    SimplexSolver solver(prog);
    CHECK(solver.optimize() == LpStatus::Optimal);
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    Eigen::VectorXd c2(prog.num_vars);
    for (int j = 0; j < prog.num_vars; ++j) c2(j) = 2.0 * unit(rng) - 1.0;
    solver.set_objective(c2);
    CHECK(solver.optimize() == LpStatus::Optimal);
    LinearProgram cold = prog;
    cold.objective = c2;
    LpSolution fresh = solve(cold);
    CHECK(fresh.status == LpStatus::Optimal);
    CHECK(th::approx(solver.objective_value(), fresh.objective, 1e-8, 1e-9));
    ++checked;
  }
  CHECK(checked > 10);
}

TEST_CASE("bound edits re-optimize correctly") {
  LinearProgram prog(2);
  prog.objective << 1.0, 1.0;
  prog.upper << 4.0, 4.0;
  prog.add_row({{0, 1.0}, {1, 1.0}}, Relation::LessEq, 5.0);
  SimplexSolver s(prog);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 5.0);
  s.set_bounds(0, 0.0, 0.0);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 4.0);
  CHECK(std::fabs(s.solution()(0)) < 1e-12);
  s.set_bounds(0, 0.0, 4.0);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 5.0);
  CHECK_THROWS_AS(s.set_bounds(99, 0.0, 1.0), MalformedProgram);
  CHECK_THROWS_AS(s.set_bounds(0, 2.0, 1.0), MalformedProgram);
}

TEST_CASE("incremental rows and variables extend the program") {
  LinearProgram prog(1);
  prog.objective(0) = 1.0;
  prog.upper(0) = 10.0;
  prog.add_row({{0, 1.0}}, Relation::LessEq, 3.0);
  SimplexSolver s(prog);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 3.0);
  s.add_row({{0, 1.0}}, Relation::LessEq, 2.0);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 2.0);
  const int z = s.add_var(0.0, 1.5, 2.0);
  CHECK(z == 1);
  CHECK(s.num_vars() == 2);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 5.0);
  s.add_row({{0, 1.0}, {z, 1.0}}, Relation::LessEq, 2.5);
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK_APPROX(s.objective_value(), 4.0);
  CHECK_THROWS_AS(s.add_row({{7, 1.0}}, Relation::LessEq, 1.0), MalformedProgram);
}

TEST_CASE("reset drops the warm basis but not the program") {
  LinearProgram prog = random_box_lp(77);
  SimplexSolver s(prog);
  CHECK(s.optimize() == LpStatus::Optimal);
  const double first = s.objective_value();
  const long it = s.iterations();
  s.reset();
  CHECK(s.optimize() == LpStatus::Optimal);
  CHECK(th::approx(s.objective_value(), first, 1e-10));
  CHECK(s.iterations() >= it);
}

TEST_CASE("repeat solves are bit identical") {
  LinearProgram prog = random_box_lp(424242);
  LpSolution a = solve(prog), b = solve(prog);
  CHECK(a.status == b.status);
  CHECK(a.iterations == b.iterations);
  CHECK(a.objective == b.objective);
  for (int j = 0; j < a.x.size(); ++j) CHECK(a.x(j) == b.x(j));
}

TEST_CASE("check_feasible and dump") {
  LinearProgram prog(2);
  prog.upper << 1.0, 1.0;
  prog.add_row({{0, 2.0}, {1, 2.0}}, Relation::LessEq, 2.0);
  Eigen::VectorXd inside(2), edge(2), outside(2);
  inside << 0.25, 0.25;
  edge << 0.5, 0.5;
  outside << 1.0, 1.0;
  CHECK_APPROX(check_feasible(prog, inside), -0.25);
  CHECK(std::fabs(check_feasible(prog, edge)) < 1e-12);
  CHECK_APPROX(check_feasible(prog, outside), 1.0);
  const std::string text = dump(prog);
  CHECK(text.find("max") != std::string::npos && text.find("<=") != std::string::npos);
}
