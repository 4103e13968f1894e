// swarmplan/round.hpp — host orchestrator of the B200 averaging round for C++
// callers (new; the reference stops at the assignment and the CPU
// run_plan). One AveragingRound per rank/GPU:
//
//   StrategyAssignment s = strategy::solve_strategy(spec);      // LP (host)
//   round::AveragingRound r(cfg);                                // C-ABI sp_round_create
//   r.assign(s.fractions, sample_counts);                        // part_offsets + weights
//   r.run(grads, p, m, v, step, stream);                         // GPU round + LAMB
//
// Errors from libsp_round.so map onto the reference's exception classes:
// invalid arguments -> std::invalid_argument, CUDA / peer failures ->
// std::runtime_error.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sp_round.h"
#include "swarmplan/model.hpp"

namespace swarmplan::round {

struct RoundConfig {
  int device = 0;
  int rank = 0;
  int world = 1;
  int peers_per_rank = 1;
  std::int64_t n = 0;
  std::string wire = "fp16";  // fp32 | fp16 | q8
  int q8_block = 4096;
  std::vector<std::int64_t> tensor_sizes;  // empty: one tensor of n
  float lr = 1.76e-3f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-6f, weight_decay = 0.01f;
  bool bias_correction = true;
  double barrier_timeout_s = 20.0;
  bool shard_lamb = false;  // sp_round_cfg::shard_lamb (p must be param_buffer())
};

class AveragingRound {
 public:
  explicit AveragingRound(const RoundConfig& cfg);
  ~AveragingRound();
  AveragingRound(const AveragingRound&) = delete;
  AveragingRound& operator=(const AveragingRound&) = delete;

  // world > 1: exchange these blobs in rank order, then connect().
  std::vector<std::uint8_t> export_handle() const;
  void connect(const std::vector<std::uint8_t>& all_handles);

  int align() const;
  // fractions: StrategyAssignment::fractions (one per peer, G = world*L);
  // weights: accumulated sample counts per peer (0 for aggregation-only).
  std::vector<std::int64_t> assign(const std::vector<double>& fractions,
                                   const std::vector<double>& weights);
  void set_assignment(const std::vector<std::int64_t>& offsets, const std::vector<double>& weights);
  // Solves the strategy for `spec` (one spec peer per round peer) and assigns.
  StrategyAssignment plan(const CollaborationSpec& spec, const std::vector<double>& weights);

  void run(const float* const* grads, float* p, float* m, float* v, int step, void* stream = nullptr);
  // Same round from pinned HOST gradients (sp_round_run_host): the copy of
  // step k overlaps round k-1 through double-buffered device staging.
  // host_p_out != nullptr also copies the updated parameters back to the
  // host after the round (sp_round_run_host_params).
  void run_host(const float* const* host_grads, float* p, float* m, float* v, int step,
                void* stream = nullptr, float* host_p_out = nullptr);
  // shard_lamb: the flat parameter vector the round updates (device fp32[n]).
  float* param_buffer() const;
  sp_phase_times run_phased(const float* const* grads, float* p, float* m, float* v, int step,
                            void* stream = nullptr);

  // Round step 1 on the device: accumulate micro-batch gradients (two
  // buffers for delayed parameter updates) and run the round weighted by the
  // accumulated sample counts (see include/sp_round.h).
  void accumulate(int buf, int local_peer, const float* grad, double samples, void* stream = nullptr);
  float* accumulator(int buf, int local_peer);
  double samples(int buf, int local_peer) const;
  void run_accumulated(int buf, float* p, float* m, float* v, int step, void* stream = nullptr);

  const std::vector<std::int64_t>& offsets() const { return offsets_; }
  sp_round* handle() const { return h_; }
  int peers() const { return cfg_.peers_per_rank * cfg_.world; }
  int local_peers() const { return cfg_.peers_per_rank; }

 private:
  RoundConfig cfg_;
  sp_round* h_ = nullptr;
  std::vector<std::int64_t> offsets_;
};

// Throws the exception class matching an SP_* status (no-op for SP_OK).
void check_status(int rc);

}  // namespace swarmplan::round
