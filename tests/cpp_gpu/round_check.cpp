// GPU check of the C++ orchestrator (include/swarmplan/round.hpp): the LP
// plan for a 4-peer heterogeneous fleet feeds a 4-virtual-peer round on one
// B200; the averaged vector and the LAMB state must equal the CPU oracle
// (oracle/sp_oracle.h) bit for bit (p given the device trust ratios).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../oracle/sp_oracle.h"
#include "swarmplan/round.hpp"
#include "swarmplan/strategy.hpp"

using namespace swarmplan;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("CUDA %s: %s\n", #x, cudaGetErrorString(e_));                \
      return 2;                                                                \
    }                                                                          \
  } while (0)

int main() {
  CollaborationSpec spec;
  spec.batch_size = 4;
  spec.param_count = 11813810;
  for (int i = 0; i < 4; ++i) {
    PeerSpec p;
    p.id = "gpu" + std::to_string(i);
    p.samples_per_sec = 1.0;
    p.download_bps = p.upload_bps = (i == 3 ? 500.0 : 200.0) * kMbps;
    spec.peers.push_back(p);
  }
  const std::vector<int64_t> sizes = {3, 1000, 70001, 2, 4096, 131075, 5};
  int64_t n = 0;
  for (int64_t s : sizes) n += s;
  round::RoundConfig cfg;
  cfg.peers_per_rank = 4;
  cfg.n = n;
  cfg.wire = "fp16";
  cfg.tensor_sizes = sizes;
  round::AveragingRound rnd(cfg);
  const std::vector<double> weights = {3.0, 1.0, 2.0, 7.0};
  StrategyAssignment s = rnd.plan(spec, weights);
  std::printf("xi=%.12f fractions=%.6f %.6f %.6f %.6f\n", s.xi, s.fractions[0], s.fractions[1],
              s.fractions[2], s.fractions[3]);

  std::vector<std::vector<float>> gh(4, std::vector<float>((size_t)n));
  std::vector<float*> gd(4);
  for (int g = 0; g < 4; ++g) {
    sp_oracle_fill_synthetic(gh[g].data(), n, 7, g, 1.7e-3f, 997, 100.0f);
    CK(cudaMalloc(&gd[g], (size_t)n * 4));
    CK(cudaMemcpy(gd[g], gh[g].data(), (size_t)n * 4, cudaMemcpyHostToDevice));
  }
  std::vector<float> ph((size_t)n), mh((size_t)n, 0.0f), vh((size_t)n, 0.0f);
  sp_oracle_fill_synthetic(ph.data(), n, 8, 0, 0.02f, 0, 1.0f);
  float *pd, *md, *vd;
  CK(cudaMalloc(&pd, (size_t)n * 4));
  CK(cudaMalloc(&md, (size_t)n * 4));
  CK(cudaMalloc(&vd, (size_t)n * 4));
  CK(cudaMemcpy(pd, ph.data(), (size_t)n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(md, 0, (size_t)n * 4));
  CK(cudaMemset(vd, 0, (size_t)n * 4));

  // oracle: pack each peer, reduce, then LAMB per step
  std::vector<std::vector<uint16_t>> wire(4, std::vector<uint16_t>((size_t)n));
  for (int g = 0; g < 4; ++g) sp_oracle_pack_fp16(gh[g].data(), wire[g].data(), n);
  const void* wp[4] = {wire[0].data(), wire[1].data(), wire[2].data(), wire[3].data()};
  std::vector<uint16_t> avg((size_t)n);
  sp_oracle_reduce(SPO_FP16, wp, nullptr, weights.data(), 4, 0, n, 4096, avg.data(), nullptr);
  sp_oracle_lamb_hp hp{cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, 1};

  int bad = 0;
  // steps 1-2: device gradients; steps 3-4: the same gradients from host
  // memory through run_host (double-buffered staging, both buffers used)
  std::vector<const float*> hp_ptrs = {gh[0].data(), gh[1].data(), gh[2].data(), gh[3].data()};
  for (int step = 1; step <= 4; ++step) {
    if (step <= 2) rnd.run(gd.data(), pd, md, vd, step);
    else rnd.run_host(hp_ptrs.data(), pd, md, vd, step);
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> got((size_t)n);
    if (sp_round_read(rnd.handle(), SP_BUF_AVG, 0, 0, got.data(), (size_t)n * 2)) return 3;
    if (std::memcmp(got.data(), avg.data(), (size_t)n * 2) != 0) {
      std::printf("step %d: averaged vector differs\n", step);
      ++bad;
    }
    std::vector<float> trust(sizes.size());
    if (sp_round_read(rnd.handle(), SP_BUF_TRUST, 0, 0, trust.data(), trust.size() * 4)) return 3;
    sp_oracle_lamb(SPO_FP16, avg.data(), nullptr, 4096, ph.data(), mh.data(), vh.data(), n,
                   sizes.data(), (int)sizes.size(), &hp, step, trust.data(), nullptr);
    std::vector<float> p2((size_t)n), m2((size_t)n), v2((size_t)n);
    CK(cudaMemcpy(p2.data(), pd, (size_t)n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(m2.data(), md, (size_t)n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(v2.data(), vd, (size_t)n * 4, cudaMemcpyDeviceToHost));
    if (std::memcmp(p2.data(), ph.data(), (size_t)n * 4) || std::memcmp(m2.data(), mh.data(), (size_t)n * 4) ||
        std::memcmp(v2.data(), vh.data(), (size_t)n * 4)) {
      std::printf("step %d: LAMB state differs\n", step);
      ++bad;
    }
  }
  std::printf("%s\n", bad ? "FAIL" : "round_check ok");
  return bad ? 1 : 0;
}
