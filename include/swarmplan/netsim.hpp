// swarmplan/netsim.hpp — round-time comparator of the averaging strategies
// (reference: /root/reference/proj/include/swarmplan/netsim.hpp:12-90).
// Only the per-round models are provided; the churn simulator
// (simulate_training) is outside this framework's scope.
#pragma once

#include <string>
#include <vector>

#include "swarmplan/model.hpp"

namespace swarmplan::netsim {

enum class Algorithm { AllReduce, ParameterServer, Adaptive };

std::string algorithm_name(Algorithm a);
Algorithm algorithm_from_name(const std::string& name);  // SpecParseError if unknown

struct ChurnEvent {
  enum class Kind { Join, Leave, Fail };
  double t = 0.0;
  std::string peer_id;
  Kind kind = Kind::Join;
};

struct ChurnTrace {
  double horizon_s = 3600.0;
  std::vector<ChurnEvent> events;
};

ChurnTrace trace_from_json(const std::string& text);

struct SimConfig {
  Algorithm algorithm = Algorithm::Adaptive;
  bool delay_parameter_updates = true;
  double refresh_s = 30.0;
  double catchup_s = 60.0;
  double stall_timeout_s = 600.0;
  int group_size = 0;
  int ps_server = -1;
  unsigned long seed = 1;
  // Measured executor round times in seconds, indexed by Algorithm
  // (AllReduce, ParameterServer, Adaptive); 0 keeps the fluid model. When
  // set, the measured time replaces the model's comm_s (reference
  // netsim.cpp:146-201) and round_s in compare_strategies,
  // e.g. times from paper_2106_10207_b200.measure.measure_round_times().
  double measured_round_s[3] = {0.0, 0.0, 0.0};
};

// Seconds for one averaging round over the whole fleet; `server` applies to
// ParameterServer only (-1: best duplex peer).
double simulate_averaging(const CollaborationSpec& spec, Algorithm alg, int server = -1);

struct StrategyComparison {
  Algorithm algorithm;
  double round_s = 0.0;
  double steps_per_hour = 0.0;
};

// Static fleet (no churn): round time and steps/hour per algorithm.
std::vector<StrategyComparison> compare_strategies(const CollaborationSpec& spec,
                                                   const SimConfig& config = {});

}  // namespace swarmplan::netsim
