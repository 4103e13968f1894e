// ref_wrap.cpp — C entry points over the reference's OWN compiled code
// (/root/reference/proj/src/groups.cpp and model.cpp, built unmodified by
// oracle/build_ref.py into oracle/_ref/libswarmplan_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ and bench.py's reference arm to
// pin this framework's host code and averaged vectors to the reference
// itself. Plain C types only, so it loads with ctypes beside the product's
// own swarmplan symbols (everything else in the .so is hidden).
#include <cstdint>
#include <cstring>
#include <exception>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "swarmplan/groups.hpp"
#include "swarmplan/model.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

int put(const std::string& s, char* out, int cap) {
  if (!out || cap <= 0) return -3;
  if ((int)s.size() + 1 > cap) return -3;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return (int)s.size();
}

}  // namespace

REF_API const char* ref_last_error(void) { return g_err.c_str(); }

// groups::build_plan (groups.cpp:43-100), serialized as
// [R, then per round: ngroups, then per group: size, members...].
// Returns the number of ints written, -1 on std::invalid_argument, -3 if
// `cap` is too small.
REF_API int ref_build_plan(int n, int m, int* out, int cap) {
  try {
    swarmplan::groups::GroupPlan p = swarmplan::groups::build_plan(n, m);
    std::vector<int> v;
    v.push_back((int)p.rounds.size());
    for (const auto& r : p.rounds) {
      v.push_back((int)r.size());
      for (const auto& g : r) {
        v.push_back((int)g.size());
        v.insert(v.end(), g.begin(), g.end());
      }
    }
    if ((int)v.size() > cap) return -3;
    std::memcpy(out, v.data(), v.size() * sizeof(int));
    return (int)v.size();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  }
}

// groups::run_plan (groups.cpp:102-163) on build_plan(n, m): values and
// out_values are n x dim row-major fp64; weights may be NULL (all 1);
// failures are nfail (round, group) pairs. Returns 0, -1 on
// std::invalid_argument, -2 on any other exception.
REF_API int ref_run_plan(int n, int m, const double* values, int64_t dim, const double* weights,
                         int nweights, const int* failures, int nfail, double* out_values,
                         int* complete, int* coverage, int* groups_failed) {
  try {
    swarmplan::groups::GroupPlan p = swarmplan::groups::build_plan(n, m);
    Eigen::MatrixXd v(n, dim);
    for (int i = 0; i < n; ++i)
      for (int64_t d = 0; d < dim; ++d) v(i, d) = values[(size_t)i * dim + d];
    std::vector<double> w;
    if (weights) w.assign(weights, weights + nweights);
    std::set<std::pair<int, int>> f;
    for (int k = 0; k < nfail; ++k) f.insert({failures[2 * k], failures[2 * k + 1]});
    swarmplan::groups::RunResult r = swarmplan::groups::run_plan(p, v, w, f);
    for (int i = 0; i < n; ++i) {
      for (int64_t d = 0; d < dim; ++d) out_values[(size_t)i * dim + d] = r.values(i, d);
      complete[i] = r.complete[i] ? 1 : 0;
      coverage[i] = r.coverage[i];
    }
    *groups_failed = r.groups_failed;
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// spec_from_json (model.cpp:100-146) then validate (model.cpp:38-83):
// violations as "peer\tfield\tmessage\n" lines. Returns the number of
// violations, -1 on SpecParseError (message in ref_last_error), -3 if `cap`
// is too small.
REF_API int ref_validate(const char* json, char* out, int cap) {
  try {
    swarmplan::CollaborationSpec s = swarmplan::spec_from_json(json);
    std::string txt;
    const auto vs = swarmplan::validate(s);
    for (const auto& x : vs) txt += std::to_string(x.peer) + "\t" + x.field + "\t" + x.message + "\n";
    const int rc = put(txt, out, cap);
    return rc < 0 ? rc : (int)vs.size();
  } catch (const swarmplan::SpecParseError& e) {
    g_err = e.what();
    return -1;
  }
}

// spec_to_json(spec_from_json(json)) (model.cpp:148-176). Returns the text
// length, -1 on SpecParseError, -3 if `cap` is too small.
REF_API int ref_spec_roundtrip(const char* json, char* out, int cap) {
  try {
    return put(swarmplan::spec_to_json(swarmplan::spec_from_json(json)), out, cap);
  } catch (const swarmplan::SpecParseError& e) {
    g_err = e.what();
    return -1;
  }
}

// assignment_to_json (model.cpp:178-205) of an assignment given as arrays
// (a, g: n x n row-major bit/s; compute: 0/1). Returns the text length.
REF_API int ref_assignment_json(const char* spec_json, int n, const double* a, const double* g,
                                const double* c_raw, const int* compute, const double* fractions,
                                double xi, int lp_iterations, char* out, int cap) {
  try {
    swarmplan::CollaborationSpec s = swarmplan::spec_from_json(spec_json);
    swarmplan::StrategyAssignment as;
    as.a.resize(n, n);
    as.g.resize(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        as.a(i, j) = a[i * n + j];
        as.g(i, j) = g[i * n + j];
      }
    as.c_raw.assign(c_raw, c_raw + n);
    for (int i = 0; i < n; ++i) as.compute.push_back(compute[i] != 0);
    as.fractions.assign(fractions, fractions + n);
    as.xi = xi;
    as.lp_iterations = lp_iterations;
    return put(swarmplan::assignment_to_json(s, as), out, cap);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// Weighted mean of G fp32 rows in run_plan's arithmetic at m = n (one
// round, one group: class sums w_i * v_i, merged 0 + s_0 + s_1 + ... in peer
// order, divided by the summed weight; groups.cpp:117-161), computed with
// the reference's own run_plan over column blocks of `block` elements so a
// full-size vector does not need one G x N fp64 matrix. rows[g] may be NULL
// for a peer that contributes nothing (weight 0). out: N fp64 values.
REF_API int ref_weighted_mean(int G, const float* const* rows, const double* weights, int64_t N,
                              int64_t block, double* out) {
  try {
    swarmplan::groups::GroupPlan p = swarmplan::groups::build_plan(G, G > 1 ? G : 2);
    std::vector<double> w(weights, weights + G);
    for (int64_t lo = 0; lo < N; lo += block) {
      const int64_t len = std::min(block, N - lo);
      Eigen::MatrixXd v(G, len);
      for (int g = 0; g < G; ++g)
        for (int64_t d = 0; d < len; ++d) v(g, d) = rows[g] ? (double)rows[g][lo + d] : 0.0;
      swarmplan::groups::RunResult r = swarmplan::groups::run_plan(p, v, w);
      for (int64_t d = 0; d < len; ++d) out[lo + d] = r.values(0, d);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// The same weighted mean over peers' WIRE buffers (the reference arm of
// bench.py): wire 0 fp32, 1 fp16 (IEEE binary16 bits), 2 blockwise 8-bit
// codes with one fp32 scale per `qblock` elements (value = code * scale).
// Each of `threads` threads runs the reference's run_plan over its own
// column blocks (run_plan is a pure function), so the result
// does not depend on the thread count.
REF_API int ref_weighted_mean_wire(int wire, int G, const void* const* rows, const float* const* scales,
                                   int qblock, const double* weights, int64_t N, int64_t block,
                                   int threads, double* out) {
  try {
    const swarmplan::groups::GroupPlan p = swarmplan::groups::build_plan(G, G > 1 ? G : 2);
    const std::vector<double> w(weights, weights + G);
    auto value = [&](int g, int64_t i) -> double {
      if (!rows[g]) return 0.0;
      if (wire == 0) return static_cast<const float*>(rows[g])[i];
      if (wire == 1) return (double)(float)static_cast<const _Float16*>(rows[g])[i];
      return (double)((float)static_cast<const int8_t*>(rows[g])[i] * scales[g][i / qblock]);
    };
    const int64_t nblk = (N + block - 1) / block;
    std::vector<std::string> errs((size_t)std::max(threads, 1));
    auto work = [&](int t) {
      try {
        for (int64_t b = t; b < nblk; b += std::max(threads, 1)) {
          const int64_t lo = b * block, len = std::min(block, N - lo);
          Eigen::MatrixXd v(G, len);
          for (int g = 0; g < G; ++g)
            for (int64_t d = 0; d < len; ++d) v(g, d) = value(g, lo + d);
          swarmplan::groups::RunResult r = swarmplan::groups::run_plan(p, v, w);
          for (int64_t d = 0; d < len; ++d) out[lo + d] = r.values(0, d);
        }
      } catch (const std::exception& e) {
        errs[(size_t)t] = e.what();
      }
    };
    if (threads <= 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
      for (auto& th : pool) th.join();
    }
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}
