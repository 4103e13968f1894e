// module.cpp — pybind11 module `_swarmplan`: the reference's Python API
// (/root/reference/proj/bindings/module.cpp:92-146, re-exported by
// proj/python/swarmplan/__init__.py) with the same names, argument meaning
// and errors (SpecParseError -> ValueError subclass), plus the hooks the
// averaging round needs: part_offsets, plan_parts, run_plan and the LP, and
// the GPU round itself: AveragingRound (swarmplan::round::AveragingRound over
// the libsp_round.so C-ABI) and run_averaging_round, which takes torch CUDA
// tensors (duck-typed: only their data pointers cross, no torch headers or
// library are linked). The GIL is released around solves and rounds.

#include <map>

#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "swarmplan/groups.hpp"
#include "swarmplan/lp.hpp"
#include "swarmplan/model.hpp"
#include "swarmplan/netsim.hpp"
#include "swarmplan/partition.hpp"
#include "swarmplan/round.hpp"
#include "swarmplan/scenario.hpp"
#include "swarmplan/strategy.hpp"

namespace py = pybind11;
using namespace swarmplan;

namespace {

std::vector<std::vector<double>> rows_of(const Eigen::MatrixXd& m) {
  std::vector<std::vector<double>> out(static_cast<std::size_t>(m.rows()));
  for (Eigen::Index i = 0; i < m.rows(); ++i) {
    out[i].resize(static_cast<std::size_t>(m.cols()));
    for (Eigen::Index j = 0; j < m.cols(); ++j) out[i][j] = m(i, j);
  }
  return out;
}

StrategyAssignment solve_nogil(const CollaborationSpec& spec, bool comm_only = false) {
  py::gil_scoped_release release;
  strategy::SolveOptions o;
  o.communication_only = comm_only;
  return strategy::solve_strategy(spec, o);
}

py::dict assignment_dict(const StrategyAssignment& s) {
  py::dict d;
  d["steps_per_sec"] = s.xi;
  d["fractions"] = s.fractions;
  std::vector<bool> compute(s.compute.begin(), s.compute.end());
  d["compute"] = compute;
  d["duty_cycle"] = s.c_raw;
  d["gradient_flows"] = rows_of(s.a);
  d["average_flows"] = rows_of(s.g);
  d["lp_iterations"] = s.lp_iterations;
  return d;
}

lp::LinearProgram program_from_py(int num_vars, const std::vector<double>& objective,
                                  const std::vector<double>& lower, const std::vector<double>& upper,
                                  const py::list& rows) {
  lp::LinearProgram prog(num_vars);
  if (static_cast<int>(objective.size()) != num_vars) prog.objective = Eigen::VectorXd::Zero(static_cast<Eigen::Index>(objective.size()));
  for (std::size_t j = 0; j < objective.size() && static_cast<int>(j) < prog.objective.size(); ++j)
    prog.objective(static_cast<Eigen::Index>(j)) = objective[j];
  for (std::size_t j = 0; j < lower.size() && static_cast<int>(j) < num_vars; ++j) prog.lower(static_cast<Eigen::Index>(j)) = lower[j];
  for (std::size_t j = 0; j < upper.size() && static_cast<int>(j) < num_vars; ++j) prog.upper(static_cast<Eigen::Index>(j)) = upper[j];
  for (const auto& r : rows) {
    auto t = r.cast<py::tuple>();  // (coeffs [(var, coef)], "<=" | "=", rhs)
    auto coeffs = t[0].cast<std::vector<std::pair<int, double>>>();
    const std::string rel = t[1].cast<std::string>();
    prog.add_row(coeffs, rel == "=" ? lp::Relation::Eq : lp::Relation::LessEq, t[2].cast<double>());
  }
  return prog;
}

const char* status_name(lp::LpStatus s) {
  switch (s) {
    case lp::LpStatus::Optimal: return "optimal";
    case lp::LpStatus::Infeasible: return "infeasible";
    case lp::LpStatus::Unbounded: return "unbounded";
  }
  return "?";
}

}  // namespace

PYBIND11_MODULE(_swarmplan, m) {
  m.doc() = "B200-native DeDLOC averaging round: planning core (LP load balancer, group plans)";
  m.attr("__version__") = "0.1.0";
  py::register_exception<SpecParseError>(m, "SpecParseError", PyExc_ValueError);
  py::register_exception<lp::MalformedProgram>(m, "MalformedProgram", PyExc_ValueError);

  // ---- reference API (bindings/module.cpp:99-145) ------------------------
  m.def("solve_strategy",
        [](const std::string& spec_json) { return assignment_dict(solve_nogil(spec_from_json(spec_json))); },
        py::arg("spec_json"),
        "Solve the communication strategy for a collaboration spec (JSON text); returns flows, "
        "duty cycles, aggregation fractions and the optimizer step rate.");
  m.def("assignment_json",
        [](const std::string& spec_json) {
          CollaborationSpec spec = spec_from_json(spec_json);
          return assignment_to_json(spec, solve_nogil(spec));
        },
        py::arg("spec_json"));
  m.def("validate_spec",
        [](const std::string& spec_json) {
          py::list out;
          for (const Violation& v : validate(spec_from_json(spec_json))) {
            py::dict d;
            d["peer"] = v.peer;
            d["field"] = v.field;
            d["message"] = v.message;
            out.append(d);
          }
          return out;
        },
        py::arg("spec_json"));
  m.def("simulate_averaging",
        [](const std::string& spec_json, const std::string& algorithm, int server) {
          CollaborationSpec spec = spec_from_json(spec_json);
          netsim::Algorithm alg = netsim::algorithm_from_name(algorithm);
          py::gil_scoped_release release;
          return netsim::simulate_averaging(spec, alg, server);
        },
        py::arg("spec_json"), py::arg("algorithm"), py::arg("server") = -1,
        "Seconds for one averaging round (allreduce, parameter_server or adaptive).");
  m.def("compare_strategies",
        [](const std::string& spec_json, std::map<std::string, double> measured) {
          CollaborationSpec spec = spec_from_json(spec_json);
          netsim::SimConfig cfg;
          for (const auto& [name, sec] : measured)
            cfg.measured_round_s[static_cast<int>(netsim::algorithm_from_name(name))] = sec;
          std::vector<netsim::StrategyComparison> rows;
          {
            py::gil_scoped_release release;
            rows = netsim::compare_strategies(spec, cfg);
          }
          py::list out;
          for (const auto& c : rows) {
            py::dict d;
            d["algorithm"] = netsim::algorithm_name(c.algorithm);
            d["round_s"] = c.round_s;
            d["steps_per_hour"] = c.steps_per_hour;
            out.append(d);
          }
          return out;
        },
        py::arg("spec_json"), py::arg("measured") = std::map<std::string, double>{},
        "Static-fleet round time and steps/hour per algorithm; `measured` maps algorithm "
        "names to executor round times (s) that replace the fluid model's comm time.");
  m.def("build_plan", [](int n, int msize) { return groups::build_plan(n, msize).rounds; },
        py::arg("n"), py::arg("m"));
  m.def("expected_iterations", &groups::expected_iterations, py::arg("n"), py::arg("m"), py::arg("p"));
  m.def("optimal_group_size", &groups::optimal_group_size, py::arg("n"), py::arg("p"));
  m.def("run_training",
        [](const std::string&, double) -> py::dict {
          throw py::type_error(
              "run_training (churn simulation) is outside this framework's scope: it models whole "
              "training runs, not the averaging round (DESIGN.md, out of scope)");
        },
        py::arg("scenario_json"), py::arg("hours") = 0.0);
  m.def("check_bound",
        [](py::args, py::kwargs) -> py::dict {
          throw py::type_error(
              "check_bound (SGD convergence harness) is outside this framework's scope (DESIGN.md)");
        });

  // ---- averaging-round planning ------------------------------------------
  m.def("part_offsets", &part_offsets, py::arg("n"), py::arg("fractions"), py::arg("align"),
        "Contiguous, aligned part boundaries (G+1 offsets) proportional to LP fractions.");
  m.def("plan_parts",
        [](const std::string& spec_json, std::int64_t n, std::int64_t align) {
          StrategyAssignment s = solve_nogil(spec_from_json(spec_json));
          py::dict d = assignment_dict(s);
          d["offsets"] = part_offsets(n, s.fractions, align);
          return d;
        },
        py::arg("spec_json"), py::arg("n"), py::arg("align"),
        "solve_strategy + part_offsets: what each peer aggregates in the GPU round.");
  m.def("spec_roundtrip", [](const std::string& spec_json) { return spec_to_json(spec_from_json(spec_json)); },
        py::arg("spec_json"), "spec_to_json(spec_from_json(text)): the canonical spec JSON.");
  m.def("scenario_spec_json",
        [](const std::string& scenario_text) { return spec_to_json(scenario_from_json(scenario_text).collaboration); },
        py::arg("scenario_json"));
  m.def("run_plan",
        [](int n, int msize, py::array_t<double, py::array::c_style | py::array::forcecast> values,
           std::vector<double> weights, std::vector<std::pair<int, int>> failures, bool exact) {
          if (values.ndim() != 2) throw std::invalid_argument("values must be 2-D (peers x dim)");
          groups::GroupPlan plan = groups::build_plan(n, msize);
          Eigen::MatrixXd v(values.shape(0), values.shape(1));
          auto r = values.unchecked<2>();
          for (py::ssize_t i = 0; i < values.shape(0); ++i)
            for (py::ssize_t j = 0; j < values.shape(1); ++j) v(i, j) = r(i, j);
          std::set<std::pair<int, int>> fs(failures.begin(), failures.end());
          groups::RunResult res;
          {
            py::gil_scoped_release release;
            res = groups::run_plan(plan, v, weights, fs,
                                   exact ? groups::MergeRule::Exact : groups::MergeRule::Reference);
          }
          py::array_t<double> out({static_cast<py::ssize_t>(res.values.rows()),
                                   static_cast<py::ssize_t>(res.values.cols())});
          auto w = out.mutable_unchecked<2>();
          for (py::ssize_t i = 0; i < out.shape(0); ++i)
            for (py::ssize_t j = 0; j < out.shape(1); ++j) w(i, j) = res.values(i, j);
          py::dict d;
          d["values"] = out;
          std::vector<bool> complete(res.complete.begin(), res.complete.end());
          d["complete"] = complete;
          d["coverage"] = res.coverage;
          d["groups_failed"] = res.groups_failed;
          return d;
        },
        py::arg("n"), py::arg("m"), py::arg("values"), py::arg("weights") = std::vector<double>{},
        py::arg("failures") = std::vector<std::pair<int, int>>{}, py::arg("exact") = false,
        "groups::run_plan on the CPU (fp64): values is peers x dim. exact=True merges classes "
        "per SPEC.md:240-241 instead of the reference's groups.cpp:126-151 rule.");
  m.def("run_plan_device",
        [](int n, int msize, std::vector<std::uintptr_t> values, std::int64_t dim,
           std::vector<std::uintptr_t> out, std::vector<double> weights,
           std::vector<std::pair<int, int>> failures, std::uintptr_t stream, bool exact) {
          if (static_cast<int>(values.size()) != n || static_cast<int>(out.size()) != n)
            throw std::invalid_argument("run_plan_device: one device row per peer");
          groups::GroupPlan plan = groups::build_plan(n, msize);
          std::vector<const double*> src(n);
          std::vector<double*> dst(n);
          for (int i = 0; i < n; ++i) {
            src[i] = reinterpret_cast<const double*>(values[i]);
            dst[i] = reinterpret_cast<double*>(out[i]);
          }
          std::set<std::pair<int, int>> fs(failures.begin(), failures.end());
          groups::RunResult res;
          {
            py::gil_scoped_release release;
            res = groups::run_plan_device(plan, src.data(), dim, dst.data(), weights, fs,
                                          reinterpret_cast<void*>(stream),
                                          exact ? groups::MergeRule::Exact : groups::MergeRule::Reference);
          }
          py::dict d;
          std::vector<bool> complete(res.complete.begin(), res.complete.end());
          d["complete"] = complete;
          d["coverage"] = res.coverage;
          d["groups_failed"] = res.groups_failed;
          return d;
        },
        py::arg("n"), py::arg("m"), py::arg("values"), py::arg("dim"), py::arg("out"),
        py::arg("weights") = std::vector<double>{},
        py::arg("failures") = std::vector<std::pair<int, int>>{}, py::arg("stream") = 0,
        py::arg("exact") = false,
        "groups::run_plan on the GPU: values/out are device addresses of n fp64 rows of "
        "length dim; bit-identical to run_plan.");

  // ---- LP hooks (tests and tools) -----------------------------------------
  m.def("lp_solve",
        [](int num_vars, std::vector<double> objective, std::vector<double> lower,
           std::vector<double> upper, py::list rows) {
          lp::LinearProgram prog = program_from_py(num_vars, objective, lower, upper, rows);
          lp::LpSolution sol;
          {
            py::gil_scoped_release release;
            sol = lp::solve(prog);
          }
          py::dict d;
          d["status"] = status_name(sol.status);
          d["objective"] = sol.objective;
          d["iterations"] = sol.iterations;
          std::vector<double> x(static_cast<std::size_t>(sol.x.size()));
          for (std::size_t j = 0; j < x.size(); ++j) x[j] = sol.x(static_cast<Eigen::Index>(j));
          d["x"] = x;
          d["violation"] = lp::check_feasible(prog, sol.x);
          return d;
        },
        py::arg("num_vars"), py::arg("objective"), py::arg("lower"), py::arg("upper"),
        py::arg("rows"));
  m.def("build_lp_shape",
        [](const std::string& spec_json) {
          strategy::StrategyProblem sp = strategy::build_lp(spec_from_json(spec_json));
          py::dict d;
          d["num_vars"] = sp.prog.num_vars;
          d["rows"] = static_cast<int>(sp.prog.rows.size());
          d["rows_compute"] = sp.rows_compute;
          d["rows_aggregate"] = sp.rows_aggregate;
          d["rows_service"] = sp.rows_service;
          d["rows_download"] = sp.rows_download;
          d["rows_upload"] = sp.rows_upload;
          d["rows_link"] = sp.rows_link;
          d["xi_var"] = sp.xi_var;
          d["xi_scale"] = sp.xi_scale;
          d["flow_scale"] = sp.flow_scale;
          return d;
        },
        py::arg("spec_json"));
  m.def("reference_program_xi",
        [](const std::string& spec_json, std::vector<int> pinned_compute) {
          // xi of the full reference-form program, optionally with duty
          // cycles pinned (the test-only oracle of test_strategy.cpp:88-108)
          strategy::StrategyProblem sp = strategy::build_lp(spec_from_json(spec_json));
          for (std::size_t i = 0; i < pinned_compute.size(); ++i) {
            if (pinned_compute[i] < 0) continue;
            sp.prog.lower(sp.c(static_cast<int>(i))) = pinned_compute[i];
            sp.prog.upper(sp.c(static_cast<int>(i))) = pinned_compute[i];
          }
          lp::LpSolution sol;
          {
            py::gil_scoped_release release;
            sol = lp::solve(sp.prog);
          }
          return py::make_tuple(status_name(sol.status),
                                sol.status == lp::LpStatus::Optimal ? sol.x(sp.xi_var) * sp.xi_scale : 0.0);
        },
        py::arg("spec_json"), py::arg("pinned_compute") = std::vector<int>{});

  // ---- the GPU round (run_averaging_round) -------------------
  py::class_<round::AveragingRound>(m, "AveragingRound",
                                    "One rank's B200 averaging round (swarmplan/round.hpp).")
      .def(py::init([](std::int64_t n, std::vector<std::int64_t> tensor_sizes, const std::string& wire,
                       int q8_block, int peers_per_rank, int rank, int world, int device, float lr,
                       float beta1, float beta2, float eps, float weight_decay, bool bias_correction,
                       double barrier_timeout_s, bool shard_lamb) {
             round::RoundConfig c;
             c.n = n;
             c.tensor_sizes = std::move(tensor_sizes);
             c.wire = wire;
             c.q8_block = q8_block;
             c.peers_per_rank = peers_per_rank;
             c.rank = rank;
             c.world = world;
             c.device = device;
             c.lr = lr;
             c.beta1 = beta1;
             c.beta2 = beta2;
             c.eps = eps;
             c.weight_decay = weight_decay;
             c.bias_correction = bias_correction;
             c.barrier_timeout_s = barrier_timeout_s;
             c.shard_lamb = shard_lamb;
             return std::make_unique<round::AveragingRound>(c);
           }),
           py::arg("n"), py::arg("tensor_sizes") = std::vector<std::int64_t>{}, py::arg("wire") = "fp16",
           py::arg("q8_block") = 4096, py::arg("peers_per_rank") = 1, py::arg("rank") = 0,
           py::arg("world") = 1, py::arg("device") = 0, py::arg("lr") = 1.76e-3f, py::arg("beta1") = 0.9f,
           py::arg("beta2") = 0.999f, py::arg("eps") = 1e-6f, py::arg("weight_decay") = 0.01f,
           py::arg("bias_correction") = true, py::arg("barrier_timeout_s") = 20.0,
           py::arg("shard_lamb") = false)
      .def_property_readonly("align", &round::AveragingRound::align)
      .def_property_readonly("peers", &round::AveragingRound::peers)
      .def_property_readonly("offsets", &round::AveragingRound::offsets)
      .def("assign", &round::AveragingRound::assign, py::arg("fractions"), py::arg("weights"),
           "LP fractions -> part offsets (partition.hpp) + per-peer sample counts.")
      .def("set_assignment", &round::AveragingRound::set_assignment, py::arg("offsets"), py::arg("weights"))
      .def("export_handle",
           [](const round::AveragingRound& r) {
             const std::vector<std::uint8_t> b = r.export_handle();
             return py::bytes(reinterpret_cast<const char*>(b.data()), b.size());
           })
      .def("connect",
           [](round::AveragingRound& r, const py::bytes& all) {
             const std::string s = all;
             r.connect(std::vector<std::uint8_t>(s.begin(), s.end()));
           },
           py::arg("all_handles"));
  m.def("run_averaging_round",
        [](round::AveragingRound& r, const py::list& grads, const py::object& p, const py::object& mom,
           const py::object& var, int step, const py::object& stream) {
          const std::int64_t n = r.offsets().empty() ? 0 : r.offsets().back();
          if (n <= 0) throw std::invalid_argument("run_averaging_round: assign() first");
          // a contiguous CUDA float32 tensor of at least n elements -> its data pointer
          auto ptr = [n](const py::handle& t) -> std::uintptr_t {
            if (!py::hasattr(t, "data_ptr") || !t.attr("is_cuda").cast<bool>())
              throw std::invalid_argument("run_averaging_round: expected CUDA tensors");
            if (py::str(t.attr("dtype")).cast<std::string>() != "torch.float32")
              throw std::invalid_argument("run_averaging_round: tensors must be float32");
            if (!t.attr("is_contiguous")().cast<bool>() || t.attr("numel")().cast<std::int64_t>() < n)
              throw std::invalid_argument("run_averaging_round: tensors must be contiguous with >= n elements");
            return t.attr("data_ptr")().cast<std::uintptr_t>();
          };
          std::vector<const float*> g;
          for (const py::handle& t : grads)
            g.push_back(t.is_none() ? nullptr : reinterpret_cast<const float*>(ptr(t)));
          if (static_cast<int>(g.size()) != r.local_peers())
            throw std::invalid_argument("run_averaging_round: need one gradient per local peer");
          float* pp = reinterpret_cast<float*>(ptr(p));
          float* mp = reinterpret_cast<float*>(ptr(mom));
          float* vp = reinterpret_cast<float*>(ptr(var));
          // default: torch's current stream on the tensors' device (the
          // round is ordered after the caller's backward pass)
          std::uintptr_t st = 0;
          if (stream.is_none()) {
            py::object torch = py::module_::import("torch");
            st = torch.attr("cuda").attr("current_stream")(p.attr("device")).attr("cuda_stream").cast<std::uintptr_t>();
          } else if (py::hasattr(stream, "cuda_stream")) {
            st = stream.attr("cuda_stream").cast<std::uintptr_t>();
          } else {
            st = stream.cast<std::uintptr_t>();
          }
          py::gil_scoped_release release;
          r.run(g.data(), pp, mp, vp, step, reinterpret_cast<void*>(st));
        },
        py::arg("round"), py::arg("grads"), py::arg("p"), py::arg("m"), py::arg("v"), py::arg("step"),
        py::arg("stream") = py::none(),
        "One averaging round + LAMB step on torch CUDA tensors (grads: one per local peer, None "
        "for a weight-0 peer; p/m/v updated in place), ordered on `stream` (default: torch's "
        "current stream). The C++ route to sp_round_run.");
}
