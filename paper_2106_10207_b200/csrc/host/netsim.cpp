// netsim.cpp — per-round strategy models (reference:
// /root/reference/proj/src/netsim.cpp:21-36 names, :78-90 best duplex peer,
// :117-134 simulate_averaging, :146-201 static-fleet timing, :360-382
// compare_strategies). The event-driven churn simulator is out of scope.

#include "swarmplan/netsim.hpp"

#include <algorithm>
#include <cmath>

#include <nlohmann/json.hpp>

#include "swarmplan/strategy.hpp"

namespace swarmplan::netsim {

std::string algorithm_name(Algorithm a) {
  switch (a) {
    case Algorithm::AllReduce: return "allreduce";
    case Algorithm::ParameterServer: return "parameter_server";
    case Algorithm::Adaptive: return "adaptive";
  }
  return "?";
}

Algorithm algorithm_from_name(const std::string& name) {
  if (name == "allreduce") return Algorithm::AllReduce;
  if (name == "parameter_server" || name == "ps") return Algorithm::ParameterServer;
  if (name == "adaptive") return Algorithm::Adaptive;
  throw SpecParseError("unknown algorithm: " + name);
}

ChurnTrace trace_from_json(const std::string& text) {
  using ojson = nlohmann::ordered_json;
  ojson j;
  try {
    j = ojson::parse(text);
  } catch (const ojson::exception& e) {
    throw SpecParseError(std::string("invalid trace JSON: ") + e.what());
  }
  try {
    ChurnTrace tr;
    tr.horizon_s = j.value("horizon_s", 3600.0);
    if (j.contains("events"))
      for (const ojson& ej : j["events"]) {
        ChurnEvent ev;
        ev.t = ej.at("t").get<double>();
        ev.peer_id = ej.at("peer").get<std::string>();
        const std::string kind = ej.at("kind").get<std::string>();
        if (kind == "join") ev.kind = ChurnEvent::Kind::Join;
        else if (kind == "leave") ev.kind = ChurnEvent::Kind::Leave;
        else if (kind == "fail") ev.kind = ChurnEvent::Kind::Fail;
        else throw SpecParseError("unknown churn event kind: " + kind);
        if (ev.t < 0) throw SpecParseError("churn event before t=0");
        tr.events.push_back(std::move(ev));
      }
    std::stable_sort(tr.events.begin(), tr.events.end(),
                     [](const ChurnEvent& a, const ChurnEvent& b) { return a.t < b.t; });
    return tr;
  } catch (const ojson::exception& e) {
    throw SpecParseError(std::string("bad trace: ") + e.what());
  }
}

namespace {

int best_duplex_peer(const CollaborationSpec& spec) {
  int best = -1;
  double bw = -1.0;
  for (int i = 0; i < spec.size(); ++i) {
    const double d = std::min(spec.peers[i].download_bps, spec.peers[i].upload_bps);
    if (d > bw) {
      bw = d;
      best = i;
    }
  }
  return best;
}

struct Timing {
  double compute_s = 0.0, comm_s = 0.0;
};

double measured(const SimConfig& cfg, Algorithm alg) {
  const double m = cfg.measured_round_s[static_cast<int>(alg)];
  if (m < 0.0 || !std::isfinite(m)) throw std::invalid_argument("measured round time must be finite and >= 0");
  return m;
}

Timing static_timing(const CollaborationSpec& spec, const SimConfig& cfg) {
  Timing t;
  double rate = 0.0;
  for (const PeerSpec& p : spec.peers)
    if (p.can_compute) rate += p.samples_per_sec;
  if (!(rate > 0)) return t;
  if (cfg.algorithm == Algorithm::Adaptive) {
    const StrategyAssignment s = strategy::solve_strategy(spec);
    double duty = 0.0;
    for (int i = 0; i < spec.size(); ++i) duty += spec.peers[i].samples_per_sec * s.c_raw[i];
    t.compute_s = spec.batch_size / duty;
    double worst = kUnlimited;  // slowest recipient's inbound averaged-part rate
    for (int i = 0; i < spec.size(); ++i) {
      if (!spec.peers[i].can_compute || spec.peers[i].client_mode) continue;
      double in = 0.0;
      for (int j = 0; j < spec.size(); ++j) in += s.g(j, i);
      worst = std::min(worst, in);
    }
    t.comm_s = std::isfinite(worst) && worst > 0 ? spec.payload_bits() / worst : 0.0;
  } else {
    t.compute_s = spec.batch_size / rate;
    if (spec.size() > 1) {
      if (cfg.algorithm == Algorithm::AllReduce) {
        t.comm_s = strategy::allreduce_round_seconds(spec);
      } else {
        const int server = (cfg.ps_server >= 0 && cfg.ps_server < spec.size())
                               ? cfg.ps_server
                               : best_duplex_peer(spec);
        t.comm_s = strategy::parameter_server_round_seconds(spec, server);
      }
    }
  }
  if (const double m = measured(cfg, cfg.algorithm); m > 0.0) t.comm_s = m;
  return t;
}

}  // namespace

double simulate_averaging(const CollaborationSpec& spec, Algorithm alg, int server) {
  switch (alg) {
    case Algorithm::AllReduce: return strategy::allreduce_round_seconds(spec);
    case Algorithm::ParameterServer:
      return strategy::parameter_server_round_seconds(spec, server < 0 ? best_duplex_peer(spec) : server);
    case Algorithm::Adaptive: return strategy::adaptive_round_seconds(spec);
  }
  throw std::invalid_argument("unknown algorithm");
}

std::vector<StrategyComparison> compare_strategies(const CollaborationSpec& spec,
                                                   const SimConfig& config) {
  std::vector<StrategyComparison> out;
  for (Algorithm alg : {Algorithm::AllReduce, Algorithm::ParameterServer, Algorithm::Adaptive}) {
    SimConfig cfg = config;
    cfg.algorithm = alg;
    const Timing tm = static_timing(spec, cfg);
    StrategyComparison c;
    c.algorithm = alg;
    const double m = measured(config, alg);
    c.round_s = m > 0.0 ? m : simulate_averaging(spec, alg, config.ps_server);
    const double step = config.delay_parameter_updates ? std::max(tm.compute_s, tm.comm_s)
                                                       : tm.compute_s + tm.comm_s;
    c.steps_per_hour = step > 0 ? 3600.0 / step : 0.0;
    out.push_back(c);
  }
  return out;
}

}  // namespace swarmplan::netsim
