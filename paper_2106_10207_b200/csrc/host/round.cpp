// round.cpp — C++ orchestrator over the libsp_round.so C-ABI
// (include/sp_round.h): LP fractions -> part offsets -> GPU round.

#include "swarmplan/round.hpp"

#include <stdexcept>

#include "swarmplan/partition.hpp"
#include "swarmplan/strategy.hpp"

namespace swarmplan::round {

void check_status(int rc) {
  if (rc == SP_OK) return;
  const std::string msg = sp_last_error();
  if (rc == SP_ERR_ARG || rc == SP_ERR_SHAPE) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

AveragingRound::AveragingRound(const RoundConfig& cfg) : cfg_(cfg) {
  if (cfg_.tensor_sizes.empty()) cfg_.tensor_sizes = {cfg_.n};
  sp_round_cfg c{};
  c.device = cfg_.device;
  c.rank = cfg_.rank;
  c.world = cfg_.world;
  c.peers_per_rank = cfg_.peers_per_rank;
  c.n = cfg_.n;
  if (cfg_.wire == "fp32") c.wire = SP_WIRE_FP32;
  else if (cfg_.wire == "fp16") c.wire = SP_WIRE_FP16;
  else if (cfg_.wire == "q8") c.wire = SP_WIRE_Q8;
  else throw std::invalid_argument("wire must be fp32, fp16 or q8");
  c.q8_block = cfg_.q8_block;
  c.num_tensors = static_cast<int>(cfg_.tensor_sizes.size());
  c.tensor_sizes = cfg_.tensor_sizes.data();
  c.lr = cfg_.lr;
  c.beta1 = cfg_.beta1;
  c.beta2 = cfg_.beta2;
  c.eps = cfg_.eps;
  c.weight_decay = cfg_.weight_decay;
  c.bias_correction = cfg_.bias_correction ? 1 : 0;
  c.barrier_timeout_s = cfg_.barrier_timeout_s;
  c.shard_lamb = cfg_.shard_lamb ? 1 : 0;
  check_status(sp_round_create(&c, &h_));
}

AveragingRound::~AveragingRound() { sp_round_destroy(h_); }

std::vector<std::uint8_t> AveragingRound::export_handle() const {
  std::vector<std::uint8_t> b(sp_round_handle_bytes());
  check_status(sp_round_export(h_, b.data()));
  return b;
}

void AveragingRound::connect(const std::vector<std::uint8_t>& all) {
  if (all.size() != sp_round_handle_bytes() * static_cast<std::size_t>(cfg_.world))
    throw std::invalid_argument("connect: need world * handle_bytes bytes");
  check_status(sp_round_connect(h_, all.data()));
}

int AveragingRound::align() const { return sp_round_align(h_); }

void AveragingRound::set_assignment(const std::vector<std::int64_t>& offsets,
                                    const std::vector<double>& weights) {
  if (static_cast<int>(offsets.size()) != peers() + 1 || static_cast<int>(weights.size()) != peers())
    throw std::invalid_argument("set_assignment: need G+1 offsets and G weights");
  check_status(sp_round_set_assignment(h_, offsets.data(), weights.data()));
  offsets_ = offsets;
}

std::vector<std::int64_t> AveragingRound::assign(const std::vector<double>& fractions,
                                                 const std::vector<double>& weights) {
  if (static_cast<int>(fractions.size()) != peers())
    throw std::invalid_argument("assign: one fraction per peer");
  std::vector<std::int64_t> off = part_offsets(cfg_.n, fractions, align());
  set_assignment(off, weights);
  return off;
}

StrategyAssignment AveragingRound::plan(const CollaborationSpec& spec, const std::vector<double>& weights) {
  if (spec.size() != peers()) throw std::invalid_argument("plan: spec must list one peer per round peer");
  StrategyAssignment s = strategy::solve_strategy(spec);
  assign(s.fractions, weights);
  return s;
}

void AveragingRound::run(const float* const* grads, float* p, float* m, float* v, int step, void* stream) {
  check_status(sp_round_run(h_, grads, p, m, v, step, stream));
}

void AveragingRound::run_host(const float* const* host_grads, float* p, float* m, float* v, int step,
                              void* stream, float* host_p_out) {
  check_status(sp_round_run_host_params(h_, host_grads, p, m, v, step, host_p_out, stream));
}

float* AveragingRound::param_buffer() const {
  float* p = sp_round_param_ptr(h_);
  if (!p) throw std::invalid_argument("param_buffer: the round was created without shard_lamb");
  return p;
}

sp_phase_times AveragingRound::run_phased(const float* const* grads, float* p, float* m, float* v,
                                          int step, void* stream) {
  sp_phase_times t{};
  check_status(sp_round_run_phased(h_, grads, p, m, v, step, stream, &t));
  return t;
}

void AveragingRound::accumulate(int buf, int local_peer, const float* grad, double samples,
                                void* stream) {
  check_status(sp_round_accumulate(h_, buf, local_peer, grad, samples, stream));
}

float* AveragingRound::accumulator(int buf, int local_peer) {
  float* p = sp_round_accumulator_ptr(h_, buf, local_peer);
  if (!p) throw std::invalid_argument("accumulator: bad buffer or peer");
  return p;
}

double AveragingRound::samples(int buf, int local_peer) const {
  return sp_round_samples(h_, buf, local_peer);
}

void AveragingRound::run_accumulated(int buf, float* p, float* m, float* v, int step, void* stream) {
  check_status(sp_round_run_accumulated(h_, buf, p, m, v, step, stream));
}

}  // namespace swarmplan::round
