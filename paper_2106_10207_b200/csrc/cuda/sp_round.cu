// sp_round.cu — C-ABI implementation of the averaging-round executor.
//
// Host side of libsp_round.so: buffer layout, CUDA IPC wiring between ranks,
// assignment upload, the LAMB work plan, CUDA-graph capture/replay of the
// round. Kernels live in sp_kernels.cuh (pack, reduce, barrier, ...) and
// sp_lamb.cuh (LAMB). See include/sp_round.h for the contract and the
// reference interfaces each entry point replaces.
//
// The round, per rank (N = world):
//   [publish sample counts]  accumulated rounds only
//   K1 pack + scatter        fp32 grad -> wire, each owner's range into its inbox
//   barrier                  N > 1
//   K2 reduce (+ push)       weighted average of the owned range; replicated
//                            LAMB: pushed into every rank's avg buffer
//   barrier                  N > 1, replicated
//   K3 LAMB                  k_lamb (both passes, one cooperative kernel)
//   barrier                  N > 1, sharded (every owner's p' has landed)
// One rank with one contributing peer skips K2 (the average is the peer's
// wire vector); with an fp32/fp16 wire K1 then runs inside LAMB pass 1.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sp_kernels.cuh"
#include "sp_lamb.cuh"
#include "sp_round.h"

using namespace sp;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define SP_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return fail(SP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

int wire_bits(int wire) { return wire == SP_WIRE_FP32 ? 32 : wire == SP_WIRE_FP16 ? 16 : 8; }

template <class T>
int upload(T*& dst, size_t& cap, const std::vector<T>& src) {
  if (src.size() > cap || !dst) {
    cudaFree(dst);
    dst = nullptr;
    cap = std::max<size_t>(src.size(), 1);
    SP_CUDA(cudaMalloc(&dst, cap * sizeof(T)));
  }
  if (!src.empty()) SP_CUDA(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return SP_OK;
}

}  // namespace

struct sp_round {
  sp_round_cfg cfg{};
  std::vector<int64_t> tsizes;
  int G = 0, L = 0;
  int64_t n = 0, npad = 0;
  int align = 8;
  size_t buf_bytes = 0;   // one wire/avg buffer (codes + q8 scales)
  size_t flags_bytes = 0;  // barrier flags + per-buffer sample-count tables
  // shared (IPC-exported) allocation:
  //   [flags][inbox slot 0 .. G-1][avg] (+ sharded: [param fp32 npad][norm table world x T])
  // slot g of rank k holds peer g's packed gradient for the range k owns
  char* shared = nullptr;
  size_t shared_bytes = 0;
  char* base[SP_MAX_RANKS] = {};  // every rank's shared allocation (mapped)
  bool connected = false;
  unsigned long long* epoch = nullptr;  // cross-rank barrier epoch
  int* h_err = nullptr;                 // host-mapped: 1 barrier timeout, 2 no samples
  int* d_err = nullptr;
  // LAMB plan (sp_lamb.cuh)
  int sm_count = 148;
  int lamb_grid = 148;
  size_t lamb_smem = 0;  // k_lamb dynamic shared memory: stages + stash
  bool coop = true;  // cooperative launch accepted (also inside graph capture)
  Chunk* d_chunks = nullptr;
  size_t cap_chunks = 0;
  int2* d_tchunk = nullptr;
  size_t cap_tchunk = 0;
  unsigned long long* d_partial = nullptr;  // per chunk: two tagged words
  size_t cap_partial = 0;
  int* d_ovf = nullptr;         // per chunk slot: overflow list
  size_t cap_ovf = 0;
  int* d_cnt = nullptr;         // queue / barrier / tensor counters (LambPlan::cnt)
  size_t cap_cnt = 0;
  unsigned long long* d_trace = nullptr;  // SP_LAMB_TRACE builds only
  int nchunks = 0;
  float* d_trust = nullptr;
  float* d_step_scale = nullptr;
  float* d_hp = nullptr;
  // device-side accumulation (two buffers, so a round can consume one while
  // the next step's micro-batches land in the other)
  float* acc[2][SP_MAX_LOCAL] = {};
  double host_count[2][SP_MAX_LOCAL] = {};
  double* d_stage = nullptr;  // [2][L] staged counts
  int acc_buf = -1;           // >= 0 while enqueuing an accumulated round
  // assignment
  std::vector<int64_t> offsets;
  std::vector<double> weights;
  bool assigned = false;
  // graph cache: two entries, so the double-buffered host-input rounds
  // (sp_round_run_host) alternate between two captured graphs
  cudaStream_t own = nullptr;
  cudaGraphExec_t gexec[2] = {};
  std::vector<const void*> gkey[2];
  int gnext = 0;  // slot replaced on the next miss
  // host-input rounds: pinned host gradients -> device staging (double
  // buffered) on a copy stream, overlapped with the previous round
  float* stg[2][SP_MAX_LOCAL] = {};
  cudaStream_t h2d = nullptr;
  cudaEvent_t stg_ready[2] = {}, stg_free[2] = {};
  bool stg_used[2] = {};
  int stg_next = 0;
  cudaEvent_t ev[7] = {};
  // sharded LAMB (cfg.shard_lamb): flat parameter vector + per-rank norm table
  bool shard = false;
  size_t param_off = 0, norms_off = 0;

  float* param(int rank) const { return reinterpret_cast<float*>(base[rank] + param_off); }
  double2* norms(int rank) const { return reinterpret_cast<double2*>(base[rank] + norms_off); }
  char* wire(int rank, int g) const { return base[rank] + flags_bytes + (size_t)g * buf_bytes; }
  char* avg(int rank) const { return base[rank] + flags_bytes + (size_t)G * buf_bytes; }
  double* counts(int rank, int buf) const {
    return reinterpret_cast<double*>(base[rank] + 256) + (size_t)buf * G;
  }
  unsigned long long* flags(int rank) const {
    return reinterpret_cast<unsigned long long*>(base[rank]);
  }
  int64_t own_lo() const { return offsets[(size_t)cfg.rank * L]; }
  int64_t own_hi() const { return offsets[(size_t)(cfg.rank + 1) * L]; }
};

namespace {

int validate_cfg(const sp_round_cfg* c) {
  if (!c) return fail(SP_ERR_ARG, "cfg is null");
  if (c->world < 1 || c->world > SP_MAX_RANKS) return fail(SP_ERR_ARG, "world must be in [1, 8]");
  if (c->rank < 0 || c->rank >= c->world) return fail(SP_ERR_ARG, "rank out of range");
  if (c->peers_per_rank < 1 || c->peers_per_rank > SP_MAX_LOCAL)
    return fail(SP_ERR_ARG, "peers_per_rank must be in [1, 16]");
  if ((int64_t)c->peers_per_rank * c->world > SP_MAX_PEERS)
    return fail(SP_ERR_ARG, "peers_per_rank * world exceeds 64");
  if (c->n <= 0) return fail(SP_ERR_ARG, "n must be positive");
  if (c->wire < SP_WIRE_FP32 || c->wire > SP_WIRE_Q8) return fail(SP_ERR_ARG, "unknown wire format");
  if (c->wire == SP_WIRE_Q8) {
    int b = c->q8_block;
    if (b < 512 || b > 16384 || (b & (b - 1)) != 0)
      return fail(SP_ERR_ARG, "q8_block must be a power of two in [512, 16384]");
  }
  if (c->num_tensors < 1 || !c->tensor_sizes) return fail(SP_ERR_ARG, "empty tensor table");
  int64_t s = 0;
  for (int t = 0; t < c->num_tensors; ++t) {
    if (c->tensor_sizes[t] <= 0) return fail(SP_ERR_ARG, "tensor sizes must be positive");
    s += c->tensor_sizes[t];
  }
  if (s != c->n) return fail(SP_ERR_SHAPE, "tensor sizes do not sum to n");
  if (!(c->beta1 >= 0 && c->beta1 < 1 && c->beta2 >= 0 && c->beta2 < 1))
    return fail(SP_ERR_ARG, "betas must lie in [0, 1)");
  if (!(c->eps > 0)) return fail(SP_ERR_ARG, "eps must be positive");
  return SP_OK;
}

// ------------------------------------------------------------- LAMB plan
// Tables of k_lamb (sp_lamb.cuh):
//   chunks   the elements this rank steps (replicated: all; sharded: its
//            owned range) cut at tensor edges and every multiple of
//            kLambTile; CTAs claim them at run time in this order: tensor
//            by tensor, largest first (a tensor's pass 2 starts when its
//            last chunk is in, so the kernel ends on small tensors), each
//            tensor's chunks in element order;
//   tensors  the chunk range of every tensor (its norm partials).
// The cut points depend only on kLambTile, so every order gives the same
// partials and the same fp64 sums per tensor.
int build_lamb_plan(sp_round* r) {
  const int T = (int)r->tsizes.size();
  std::vector<Chunk> chunks;
  std::vector<int2> tchunk((size_t)T, make_int2(0, 0));
  const int64_t lo = r->shard ? r->own_lo() : 0, hi = r->shard ? r->own_hi() : r->cfg.n;
  std::vector<int64_t> tstart((size_t)T + 1, 0);
  for (int t = 0; t < T; ++t) tstart[(size_t)t + 1] = tstart[(size_t)t] + r->tsizes[(size_t)t];
  std::vector<int> order((size_t)T);
  for (int t = 0; t < T; ++t) order[(size_t)t] = t;
  std::stable_sort(order.begin(), order.end(),
                   [&](int x, int y) { return r->tsizes[(size_t)x] > r->tsizes[(size_t)y]; });
  for (int t : order) {
    const int64_t t0 = tstart[(size_t)t], t1 = tstart[(size_t)t + 1];
    const int64_t a = std::max(t0, lo), b = std::min(t1, hi);
    tchunk[(size_t)t] = make_int2((int)chunks.size(), (int)chunks.size());
    for (int64_t s = a; s < b;) {
      const int64_t e = std::min(b, (s / kLambTile + 1) * kLambTile);
      Chunk ch{};
      ch.start = s;
      ch.len = (int)(e - s);
      ch.tensor = t;
      ch.head = std::min(ch.len, (int)((4 - (s & 3)) & 3));  // split_chunk (sp_kernels.cuh)
      ch.nbody4 = (ch.len - ch.head) >> 2;
      ch.tail = ch.len - ch.head - 4 * ch.nbody4;
      chunks.push_back(ch);
      s = e;
    }
    tchunk[(size_t)t].y = (int)chunks.size();
  }
  for (Chunk& ch : chunks) ch.tchunks = tchunk[(size_t)ch.tensor].y - tchunk[(size_t)ch.tensor].x;
  r->nchunks = (int)chunks.size();
  if (chunks.empty()) chunks.emplace_back();
  const size_t ncnt = lamb_counter_ints(T);
  SP_CUDA(cudaSetDevice(r->cfg.device));
  if (int rc = upload(r->d_chunks, r->cap_chunks, chunks)) return rc;
  if (int rc = upload(r->d_tchunk, r->cap_tchunk, tchunk)) return rc;
  if (int rc = upload(r->d_partial, r->cap_partial, std::vector<unsigned long long>(2 * chunks.size())))
    return rc;
  if (int rc = upload(r->d_ovf, r->cap_ovf, std::vector<int>(chunks.size()))) return rc;
  if (int rc = upload(r->d_cnt, r->cap_cnt, std::vector<int>(ncnt, 0))) return rc;
  return SP_OK;
}

// With one rank and a single contributing peer the average is the identity
// on that peer's wire values: fp32/fp16 because acc = 1.0f * x = x is exactly
// representable in the wire format, q8 by definition (a single contributor's
// codes and scales are forwarded; sp_oracle_reduce). The averaged vector IS
// the peer's inbox slot and the reduce kernel is skipped.
const char* identity_avg(const sp_round* r) {
  const sp_round_cfg& c = r->cfg;
  if (c.world != 1 || !r->assigned || r->acc_buf >= 0) return nullptr;
  int np = 0, who = -1;
  for (int g = 0; g < r->G; ++g)
    if (r->weights[g] != 0.0) {
      ++np;
      who = g;
    }
  return np == 1 ? r->wire(c.rank, who) : nullptr;
}

const char* avg_buffer(const sp_round* r) {
  const char* id = identity_avg(r);
  return id ? id : r->avg(r->cfg.rank);
}

// Rank order of every push to all ranks (averages, parameters, norm pairs):
// the next rank first and this rank last, so that at any moment the ranks
// write to different owners (all-to-all without incast: ~660 vs ~400 GB/s
// per direction on 4x B200, profiles/r01/p2p_bw.txt).
int push_rank(int rank, int world, int k) { return (rank + 1 + k) % world; }

LambArgs make_lamb_args(sp_round* r, float* p, float* m, float* v) {
  const sp_round_cfg& c = r->cfg;
  LambArgs a{};
  a.avg = avg_buffer(r);
  a.avg_scale = c.wire == SP_WIRE_Q8 ? reinterpret_cast<const float*>(avg_buffer(r) + r->npad)
                                     : nullptr;
  a.p = p;
  a.m = m;
  a.v = v;
  a.hp = r->d_hp;
  a.b1 = c.beta1;
  a.b2 = c.beta2;
  a.omb1 = 1.0f - c.beta1;
  a.omb2 = 1.0f - c.beta2;
  a.eps = c.eps;
  a.wd = c.weight_decay;
  a.qshift = __builtin_ctz((unsigned)std::max(c.q8_block, 1));
  return a;
}

BarrierArgs make_barrier(sp_round* r) {
  const sp_round_cfg& c = r->cfg;
  BarrierArgs ba{};
  for (int k = 0; k < c.world; ++k) ba.flags[k] = r->flags(k);
  ba.epoch = r->epoch;
  ba.err = r->d_err;
  ba.rank = c.rank;
  ba.world = c.world;
  const double to = c.barrier_timeout_s > 0 ? c.barrier_timeout_s : 20.0;
  ba.timeout_ns = (unsigned long long)(to * 1e9);
  return ba;
}

template <int W, bool FP>
cudaError_t launch_lamb_w(sp_round* r, const LambArgs& a, const LambPlan& pl, cudaStream_t st) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)r->lamb_grid);
  lc.blockDim = dim3(kLambThreads);
  lc.dynamicSmemBytes = r->lamb_smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = r->coop ? 1 : 0;
  return cudaLaunchKernelEx(&lc, k_lamb<W, FP>, a, pl);
}

int launch_lamb(sp_round* r, const LambArgs& a, const BarrierArgs& ba, cudaStream_t st) {
  const sp_round_cfg& c = r->cfg;
  LambPlan pl{};
  pl.chunks = r->d_chunks;
  pl.nchunks = r->nchunks;
  pl.tchunk = r->d_tchunk;
  pl.partial = r->d_partial;
  pl.ovf = r->d_ovf;
  pl.cnt = r->d_cnt;
  pl.trust = r->d_trust;
  pl.step_scale = r->d_step_scale;
  pl.cap = (int)((r->lamb_smem - (size_t)kLambStages * kLambStageBytes) / 4);
  pl.T = c.num_tensors;
  pl.shard = r->shard ? 1 : 0;
  pl.trace = r->d_trace;
  if (r->shard) {
    pl.push.ndst = c.world;
    for (int k = 0; k < c.world; ++k) {
      const int d = push_rank(c.rank, c.world, k);
      pl.table[k] = r->norms(d);
      pl.push.dst[k] = r->param(d);
    }
    pl.my_table = r->norms(c.rank);
    pl.bar = ba;  // world 1: the in-kernel barrier only waits on its own flag
  }
  cudaError_t e;
  switch (c.wire) {
    case SP_WIRE_FP32:
      e = a.g32 ? launch_lamb_w<SP_WIRE_FP32, true>(r, a, pl, st) : launch_lamb_w<SP_WIRE_FP32, false>(r, a, pl, st);
      break;
    case SP_WIRE_FP16:
      e = a.g32 ? launch_lamb_w<SP_WIRE_FP16, true>(r, a, pl, st) : launch_lamb_w<SP_WIRE_FP16, false>(r, a, pl, st);
      break;
    default: e = launch_lamb_w<SP_WIRE_Q8, false>(r, a, pl, st); break;
  }
  if (e != cudaSuccess) return fail(SP_ERR_CUDA, std::string("k_lamb launch: ") + cudaGetErrorString(e));
  return SP_OK;
}

int grid_for(int64_t work_items, int threads, int sm_count, int per_sm) {
  int64_t g = (work_items + threads - 1) / threads;
  g = std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count * per_sm));
  return (int)g;
}

int barrier(const BarrierArgs& ba, cudaStream_t st) {
  k_barrier<<<1, 32, 0, st>>>(ba);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// The host half of K1: the owner ranges this rank scatters to (visited from
// the next rank on, empty ranges skipped), in wire units (a q8 block or one
// 16-byte vector), and the CTAs given to each range in proportion to its
// length (>= 1 each). Returns the number of CTAs. Host-only (sp_round_describe
// exposes it for tests at any world size).
int pack_plan(const sp_round_cfg& c, int L, const int64_t* offsets, int sm_count, PackArgs& a) {
  const int64_t unit = c.wire == SP_WIRE_Q8 ? c.q8_block : (c.wire == SP_WIRE_FP16 ? 8 : 4);
  a.nr = 0;
  a.pref[0] = 0;
  for (int d = 1; d <= c.world; ++d) {
    const int k = (c.rank + d) % c.world;
    const int64_t lo = offsets[(size_t)k * L], hi = offsets[(size_t)(k + 1) * L];
    if (hi <= lo) continue;
    a.owner[a.nr] = k;
    a.lo[a.nr] = lo / unit;
    a.pref[a.nr + 1] = a.pref[a.nr] + (hi + unit - 1) / unit - lo / unit;
    ++a.nr;
  }
  a.cta0[0] = 0;
  const int64_t units = a.pref[a.nr];
  if (units <= 0) return 0;
  const int64_t per_cta = c.wire == SP_WIRE_Q8 ? 1 : 256;  // units per CTA per pass
  const int want = c.wire == SP_WIRE_Q8 ? (int)std::min<int64_t>(units, (int64_t)sm_count * 16)
                                        : grid_for(units, 256, sm_count, 8);
  int total = 0;
  for (int j = 0; j < a.nr; ++j) {
    const int64_t len = a.pref[j + 1] - a.pref[j];
    int nct = (int)std::max<int64_t>(1, (int64_t)((double)want * (double)len / (double)units + 0.5));
    nct = (int)std::min<int64_t>(nct, (len + per_cta - 1) / per_cta);
    total += std::max(1, nct);
    a.cta0[j + 1] = total;
  }
  return total;
}

// K1: pack every local peer's gradient, scattering each owner's range into
// that owner's inbox (pack_plan).
int enqueue_pack(sp_round* r, const float* const* grads, cudaStream_t st) {
  const sp_round_cfg& c = r->cfg;
  PackArgs a{};
  bool any = false;
  for (int l = 0; l < r->L; ++l) {
    const int g = c.rank * r->L + l;
    a.src[l] = grads[l];
    for (int k = 0; k < c.world; ++k) a.dst[l][k] = r->wire(k, g);
    const bool zero_copy = c.world == 1 && c.wire == SP_WIRE_FP32 &&
                           (const void*)grads[l] == (const void*)r->wire(c.rank, g);
    if (grads[l] && !zero_copy)
      any = true;
    else
      a.src[l] = nullptr;  // nothing to pack (aggregation-only or zero-copy)
  }
  const int total = pack_plan(c, r->L, r->offsets.data(), r->sm_count, a);
  a.n = r->n;
  a.npad = r->npad;
  a.qblock = c.q8_block;
  if (!any || total <= 0) return SP_OK;
  const int threads = c.wire == SP_WIRE_Q8 ? c.q8_block / 16 : 256;
  dim3 grid((unsigned)total, r->L);
  if (c.wire == SP_WIRE_Q8) k_pack_q8<<<grid, threads, 0, st>>>(a);
  else if (c.wire == SP_WIRE_FP16) k_pack_fp16<<<grid, threads, 0, st>>>(a);
  else k_pack_fp32<<<grid, threads, 0, st>>>(a);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// K2: weighted average of this rank's range from its inbox (local HBM);
// replicated LAMB pushes it into every rank's avg buffer (self last),
// sharded LAMB keeps it local (only the owner steps the range).
int enqueue_reduce(sp_round* r, cudaStream_t st) {
  const sp_round_cfg& c = r->cfg;
  ReduceArgs ra{};
  double wsum = 0.0;
  for (double w : r->weights) wsum += w;
  int np = 0;
  for (int g = 0; g < r->G; ++g) {
    if (r->weights[g] == 0.0) continue;
    ra.src[np] = r->wire(c.rank, g);
    ra.w[np] = (float)(r->weights[g] / wsum);
    ++np;
  }
  ra.npeers = np;
  if (r->acc_buf >= 0) {
    ra.dev_w = r->counts(c.rank, r->acc_buf);
    for (int g = 0; g < r->G; ++g) ra.all_src[g] = r->wire(c.rank, g);
    ra.G = r->G;
    ra.err = r->d_err;
  }
  ra.lo = r->own_lo();
  ra.hi = r->own_hi();
  ra.npad = r->npad;
  ra.qblock = c.q8_block;
  if (ra.hi <= ra.lo) return SP_OK;
  const int nd = r->shard ? 1 : c.world;
  ra.ndst = nd;
  for (int k = 0; k < nd; ++k) ra.dst[k] = r->avg(push_rank(c.rank, c.world, k + (c.world - nd)));
  if (c.wire == SP_WIRE_Q8) {
    const int64_t nb = (ra.hi + c.q8_block - 1) / c.q8_block - ra.lo / c.q8_block;
    const int grid = (int)std::min<int64_t>(nb, (int64_t)r->sm_count * 16);
    k_reduce_q8<<<grid, c.q8_block / 16, 0, st>>>(ra);
  } else if (c.wire == SP_WIRE_FP16) {
    k_reduce_fp16<<<grid_for((ra.hi - ra.lo + 7) / 8, 256, r->sm_count, 8), 256, 0, st>>>(ra);
  } else {
    k_reduce_fp32<<<grid_for((ra.hi - ra.lo + 3) / 4, 256, r->sm_count, 8), 256, 0, st>>>(ra);
  }
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// Enqueues the whole round on `st`. ev != nullptr records phase events.
int enqueue_round(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                  cudaStream_t st, cudaEvent_t* ev) {
  const sp_round_cfg& c = r->cfg;
  auto mark = [&](int k) -> int {
    if (ev) SP_CUDA(cudaEventRecord(ev[k], st));
    return SP_OK;
  };
  if (int rc = mark(0)) return rc;
  const BarrierArgs ba = make_barrier(r);
  LambArgs la = make_lamb_args(r, p, m, v);
  // one rank, one contributing peer, fp32/fp16: the average is the peer's
  // rounded gradient, so the pack runs inside LAMB pass 1 (saves the wire
  // re-read and a launch); the wire buffer is still written
  const bool fuse_pack = c.world == 1 && r->L == 1 && c.wire != SP_WIRE_Q8 && r->acc_buf < 0 &&
                         grads[0] && identity_avg(r) &&
                         (const void*)grads[0] != (const void*)r->wire(c.rank, 0);
  if (fuse_pack) {
    la.g32 = grads[0];
    la.wire_out = r->wire(c.rank, 0);
  }
  if (r->acc_buf >= 0) {  // accumulated round: every rank learns every peer's sample count
    PublishArgs pa{};
    pa.staged = r->d_stage + (size_t)r->acc_buf * r->L;
    for (int k = 0; k < c.world; ++k) pa.table[k] = r->counts(k, r->acc_buf);
    pa.world = c.world;
    pa.first = c.rank * r->L;
    pa.L = r->L;
    k_publish_counts<<<1, 128, 0, st>>>(pa);
    SP_CUDA(cudaGetLastError());
  }
  if (!fuse_pack)
    if (int rc = enqueue_pack(r, grads, st)) return rc;
  if (int rc = mark(1)) return rc;
  if (c.world > 1)
    if (int rc = barrier(ba, st)) return rc;
  if (int rc = mark(2)) return rc;
  if (!identity_avg(r))
    if (int rc = enqueue_reduce(r, st)) return rc;
  if (int rc = mark(3)) return rc;
  // replicated: the averages must have landed everywhere before LAMB reads
  // them. Sharded: they stay with their owner; the next round's pack cannot
  // start before this round's last barrier, which every rank enters after
  // its reduce.
  if (c.world > 1 && !r->shard)
    if (int rc = barrier(ba, st)) return rc;
  if (int rc = mark(4)) return rc;
  if (int rc = launch_lamb(r, la, ba, st)) return rc;
  if (int rc = mark(5)) return rc;
  if (r->shard && c.world > 1)  // every owner's parameters have landed everywhere
    if (int rc = barrier(ba, st)) return rc;
  return mark(6);
}

int check_run_args(sp_round* r, const float* const* grads, float* p, float* m, float* v) {
  if (!r) return fail(SP_ERR_ARG, "null round");
  if (!r->assigned) return fail(SP_ERR_STATE, "sp_round_set_assignment was not called");
  if (r->cfg.world > 1 && !r->connected) return fail(SP_ERR_STATE, "sp_round_connect was not called");
  if (!grads || !p || !m || !v) return fail(SP_ERR_ARG, "null buffer");
  auto aligned = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!aligned(p) || !aligned(m) || !aligned(v)) return fail(SP_ERR_SHAPE, "p/m/v must be 16-byte aligned");
  if (r->shard && p != r->param(r->cfg.rank))
    return fail(SP_ERR_ARG, "shard_lamb: p must be sp_round_param_ptr() (owners store into every rank's copy)");
  for (int l = 0; l < r->L; ++l) {
    const int g = r->cfg.rank * r->L + l;
    if (!grads[l] && r->weights[g] != 0.0)
      return fail(SP_ERR_ARG, "null grad for a peer with nonzero weight");
    if (grads[l] && !aligned(grads[l])) return fail(SP_ERR_SHAPE, "grads must be 16-byte aligned");
  }
  const int err = *(volatile int*)r->h_err;
  if (err == 1) return fail(SP_ERR_PEER, "a cross-rank barrier timed out in an earlier round");
  if (err == 2) {
    *(volatile int*)r->h_err = 0;  // reported once; the executor stays usable
    return fail(SP_ERR_STATE, "an earlier accumulated round had no samples on any peer "
                              "(its averaged vector was not updated)");
  }
  return SP_OK;
}

int upload_hparams(sp_round* r, int step, cudaStream_t st) {
  if (step < 1) return fail(SP_ERR_ARG, "step must be >= 1");
  float hp[4];
  hp[0] = r->cfg.lr;
  if (r->cfg.bias_correction) {
    hp[1] = (float)(1.0 / (1.0 - std::pow((double)r->cfg.beta1, step)));
    hp[2] = (float)(1.0 / (1.0 - std::pow((double)r->cfg.beta2, step)));
  } else {
    hp[1] = hp[2] = 1.0f;
  }
  hp[3] = 0.0f;
  SP_CUDA(cudaMemcpyAsync(r->d_hp, hp, sizeof(hp), cudaMemcpyHostToDevice, st));
  return SP_OK;
}

// Captures the round into a CUDA graph the first time a (pointer set, mode)
// is seen, then replays it; per-step scalars go through d_hp.
void drop_graphs(sp_round* r) {
  for (int k = 0; k < 2; ++k) {
    if (r->gexec[k]) cudaGraphExecDestroy(r->gexec[k]);
    r->gexec[k] = nullptr;
    r->gkey[k].clear();
  }
}

int launch_graph(sp_round* r, const std::vector<const void*>& key, const float* const* grads,
                 float* p, float* m, float* v, int step, cudaStream_t st) {
  int slot = -1;
  for (int k = 0; k < 2; ++k)
    if (r->gexec[k] && r->gkey[k] == key) slot = k;
  if (slot < 0) {
    slot = r->gnext;
    r->gnext ^= 1;
    if (r->gexec[slot]) {
      SP_CUDA(cudaStreamSynchronize(st));
      cudaGraphExecDestroy(r->gexec[slot]);
      r->gexec[slot] = nullptr;
    }
    cudaGraph_t graph;
    SP_CUDA(cudaStreamBeginCapture(r->own, cudaStreamCaptureModeThreadLocal));
    int erc = enqueue_round(r, grads, p, m, v, r->own, nullptr);
    cudaError_t e = cudaStreamEndCapture(r->own, &graph);
    if (erc) {
      if (e == cudaSuccess) cudaGraphDestroy(graph);
      return erc;
    }
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&r->gexec[slot], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(SP_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    r->gkey[slot] = key;
  }
  int rc = upload_hparams(r, step, st);
  if (rc) return rc;
  SP_CUDA(cudaGraphLaunch(r->gexec[slot], st));
  return SP_OK;
}

// k_lamb runs kLambCtasPerSm CTAs per SM; each gets an equal share of the
// SM's shared memory (less the per-CTA reservation): its load stages, the
// rest its stash.
template <int W, bool FP>
int lamb_func_setup(sp_round* r, int per_sm_smem, int optin, int reserved) {
  cudaFuncAttributes fa{};
  SP_CUDA(cudaFuncGetAttributes(&fa, k_lamb<W, FP>));
  const size_t share = (size_t)per_sm_smem / kLambCtasPerSm - (size_t)reserved - fa.sharedSizeBytes;
  const size_t dyn = std::min(share, (size_t)optin - fa.sharedSizeBytes) / 64 * 64;
  if (dyn < (size_t)kLambStages * kLambStageBytes + 4 * (size_t)kLambTile)
    return fail(SP_ERR_CUDA, "k_lamb: shared memory too small for its stages and a stash");
  r->lamb_smem = r->lamb_smem ? std::min(r->lamb_smem, dyn) : dyn;
  SP_CUDA(cudaFuncSetAttribute(k_lamb<W, FP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  return SP_OK;
}

template <int W, bool FP>
int lamb_occupancy(sp_round* r, int* per_sm) {
  SP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_lamb<W, FP>, kLambThreads, r->lamb_smem));
  return SP_OK;
}

}  // namespace

extern "C" {

const char* sp_version(void) { return "sp_round 0.2.0 (sm_100a)"; }
const char* sp_last_error(void) { return g_last_error.c_str(); }

size_t sp_round_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int sp_round_align(const sp_round* r) { return r ? r->align : 0; }
int64_t sp_round_padded_n(const sp_round* r) { return r ? r->npad : 0; }

int sp_round_create(const sp_round_cfg* cfg, sp_round** out) {
  if (!out) return fail(SP_ERR_ARG, "out is null");
  *out = nullptr;
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(cfg->device));
  sp_round* r = new sp_round();
  r->cfg = *cfg;
  r->tsizes.assign(cfg->tensor_sizes, cfg->tensor_sizes + cfg->num_tensors);
  r->cfg.tensor_sizes = r->tsizes.data();
  r->L = cfg->peers_per_rank;
  r->G = cfg->peers_per_rank * cfg->world;
  r->n = cfg->n;
  r->npad = round_up(cfg->n, std::max<int64_t>(kPad, cfg->wire == SP_WIRE_Q8 ? cfg->q8_block : 1));
  r->align = cfg->wire == SP_WIRE_Q8 ? cfg->q8_block : 8;
  r->buf_bytes = (size_t)r->npad * wire_bits(cfg->wire) / 8;
  // q8 scales, with slack: k_lamb stages them in 16-byte windows
  if (cfg->wire == SP_WIRE_Q8) r->buf_bytes += round_up(r->npad / cfg->q8_block * 4 + 64, 256);
  r->buf_bytes = round_up(r->buf_bytes, 256);
  r->flags_bytes = 256 + round_up((int64_t)2 * r->G * 8, 256);
  r->shared_bytes = r->flags_bytes + (size_t)(r->G + 1) * r->buf_bytes;
  if (cfg->shard_lamb) {  // [params fp32 npad][norm table world x T double2]
    r->shard = true;
    r->param_off = r->shared_bytes;
    r->norms_off = r->param_off + round_up(r->npad * 4, 256);
    r->shared_bytes = r->norms_off + round_up((int64_t)cfg->world * cfg->num_tensors * 16, 256);
  }
  int dev_sms = 0, optin = 0, per_sm_smem = 0, reserved = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cfg->device);
  cudaDeviceGetAttribute(&per_sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, cfg->device);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, cfg->device);
  if (dev_sms > 0) r->sm_count = dev_sms;

  auto cleanup = [&](int code) {
    sp_round_destroy(r);
    return code;
  };
  if (int rc2 = lamb_func_setup<SP_WIRE_FP32, false>(r, per_sm_smem, optin, reserved)) return cleanup(rc2);
  if (int rc2 = lamb_func_setup<SP_WIRE_FP32, true>(r, per_sm_smem, optin, reserved)) return cleanup(rc2);
  if (int rc2 = lamb_func_setup<SP_WIRE_FP16, false>(r, per_sm_smem, optin, reserved)) return cleanup(rc2);
  if (int rc2 = lamb_func_setup<SP_WIRE_FP16, true>(r, per_sm_smem, optin, reserved)) return cleanup(rc2);
  if (int rc2 = lamb_func_setup<SP_WIRE_Q8, false>(r, per_sm_smem, optin, reserved)) return cleanup(rc2);
  {
    int occ[5] = {};
    if (int rc2 = lamb_occupancy<SP_WIRE_FP32, false>(r, &occ[0])) return cleanup(rc2);
    if (int rc2 = lamb_occupancy<SP_WIRE_FP32, true>(r, &occ[1])) return cleanup(rc2);
    if (int rc2 = lamb_occupancy<SP_WIRE_FP16, false>(r, &occ[2])) return cleanup(rc2);
    if (int rc2 = lamb_occupancy<SP_WIRE_FP16, true>(r, &occ[3])) return cleanup(rc2);
    if (int rc2 = lamb_occupancy<SP_WIRE_Q8, false>(r, &occ[4])) return cleanup(rc2);
    const int per_sm = std::min({occ[0], occ[1], occ[2], occ[3], occ[4], kLambCtasPerSm});
    if (per_sm < 1) return cleanup(fail(SP_ERR_CUDA, "k_lamb does not fit on an SM (registers / shared memory)"));
    r->lamb_grid = per_sm * r->sm_count;  // cooperative: every CTA resident at once
  }
  {
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, cfg->device);
    r->coop = coop != 0;
  }
  cudaError_t e = cudaMalloc(&r->shared, r->shared_bytes);
  if (e != cudaSuccess) return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc shared: ") + cudaGetErrorString(e)));
  if ((e = cudaMemset(r->shared, 0, r->shared_bytes)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  r->base[cfg->rank] = r->shared;

  const size_t ntens = r->tsizes.size();
  if ((e = cudaMalloc(&r->d_trust, ntens * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_step_scale, ntens * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_hp, 4 * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->epoch, sizeof(unsigned long long))) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
  cudaMemset(r->epoch, 0, sizeof(unsigned long long));
  cudaMemset(r->d_trust, 0, ntens * sizeof(float));
  if ((e = cudaHostAlloc(&r->h_err, sizeof(int), cudaHostAllocMapped)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  *r->h_err = 0;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->d_err), r->h_err, 0);
  if ((e = cudaStreamCreateWithFlags(&r->own, cudaStreamNonBlocking)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  for (auto& ev : r->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  if (cfg->world == 1) r->connected = true;
  *out = r;
  return SP_OK;
}

int sp_round_destroy(sp_round* r) {
  if (!r) return SP_OK;
  cudaSetDevice(r->cfg.device);
  cudaDeviceSynchronize();
  drop_graphs(r);
  for (int k = 0; k < SP_MAX_RANKS; ++k)
    if (r->base[k] && k != r->cfg.rank) cudaIpcCloseMemHandle(r->base[k]);
  cudaFree(r->shared);
  cudaFree(r->d_chunks);
  cudaFree(r->d_tchunk);
  cudaFree(r->d_ovf);
  cudaFree(r->d_partial);
  cudaFree(r->d_cnt);
  cudaFree(r->d_trace);
  cudaFree(r->d_trust);
  cudaFree(r->d_step_scale);
  cudaFree(r->d_hp);
  for (int b = 0; b < 2; ++b)
    for (int l = 0; l < SP_MAX_LOCAL; ++l) cudaFree(r->acc[b][l]);
  cudaFree(r->d_stage);
  for (int b = 0; b < 2; ++b) {
    for (int l = 0; l < SP_MAX_LOCAL; ++l) cudaFree(r->stg[b][l]);
    if (r->stg_ready[b]) cudaEventDestroy(r->stg_ready[b]);
    if (r->stg_free[b]) cudaEventDestroy(r->stg_free[b]);
  }
  if (r->h2d) cudaStreamDestroy(r->h2d);
  cudaFree(r->epoch);
  if (r->h_err) cudaFreeHost(r->h_err);
  for (auto& ev : r->ev)
    if (ev) cudaEventDestroy(ev);
  if (r->own) cudaStreamDestroy(r->own);
  delete r;
  return SP_OK;
}

int sp_round_export(sp_round* r, void* out_handle) {
  if (!r || !out_handle) return fail(SP_ERR_ARG, "null argument");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaIpcMemHandle_t h;
  SP_CUDA(cudaIpcGetMemHandle(&h, r->shared));
  std::memcpy(out_handle, &h, sizeof(h));
  return SP_OK;
}

int sp_round_connect(sp_round* r, const void* all_handles) {
  if (!r || !all_handles) return fail(SP_ERR_ARG, "null argument");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  const char* hb = static_cast<const char*>(all_handles);
  for (int k = 0; k < r->cfg.world; ++k) {
    if (k == r->cfg.rank) continue;
    if (r->base[k]) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + (size_t)k * sizeof(h), sizeof(h));
    void* p = nullptr;
    SP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    r->base[k] = static_cast<char*>(p);
  }
  r->connected = true;
  drop_graphs(r);
  return SP_OK;
}

int sp_round_set_assignment(sp_round* r, const int64_t* offsets, const double* weights) {
  if (!r || !offsets || !weights) return fail(SP_ERR_ARG, "null argument");
  const int G = r->G;
  if (offsets[0] != 0 || offsets[G] != r->n)
    return fail(SP_ERR_ARG, "offsets must start at 0 and end at n");
  for (int g = 0; g < G; ++g) {
    if (offsets[g + 1] < offsets[g]) return fail(SP_ERR_ARG, "offsets must be non-decreasing");
    if (g + 1 < G && offsets[g + 1] % r->align != 0)
      return fail(SP_ERR_ARG, "inner offsets must be multiples of sp_round_align()");
  }
  double wsum = 0.0;
  for (int g = 0; g < G; ++g) {
    if (!(weights[g] >= 0.0) || !std::isfinite(weights[g]))
      return fail(SP_ERR_ARG, "weights must be finite and non-negative");
    wsum += weights[g];
  }
  if (!(wsum > 0.0)) return fail(SP_ERR_ARG, "sum of weights must be positive");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  SP_CUDA(cudaDeviceSynchronize());  // the previous round may still read the tables
  r->offsets.assign(offsets, offsets + G + 1);
  r->weights.assign(weights, weights + G);
  if (int rc = build_lamb_plan(r)) return rc;
#ifdef SP_LAMB_TRACE
  if (!r->d_trace)
    SP_CUDA(cudaMalloc(&r->d_trace, (size_t)r->lamb_grid * kLambTraceStride * sizeof(unsigned long long)));
#endif
  r->assigned = true;
  drop_graphs(r);
  return SP_OK;
}

int sp_round_run(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                 int step, void* stream) {
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<const void*> key;
  for (int l = 0; l < r->L; ++l) key.push_back(grads[l]);
  key.push_back(p);
  key.push_back(m);
  key.push_back(v);
  key.push_back(nullptr);  // mode tag: caller-owned gradients, host weights
  return launch_graph(r, key, grads, p, m, v, step, st);
}

int sp_round_run_host(sp_round* r, const float* const* host_grads, float* p, float* m, float* v,
                      int step, void* stream) {
  return sp_round_run_host_params(r, host_grads, p, m, v, step, nullptr, stream);
}

int sp_round_run_host_params(sp_round* r, const float* const* host_grads, float* p, float* m,
                             float* v, int step, float* host_p_out, void* stream) {
  if (!r || !host_grads) return fail(SP_ERR_ARG, "null argument");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!r->h2d) {
    SP_CUDA(cudaStreamCreateWithFlags(&r->h2d, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      SP_CUDA(cudaEventCreateWithFlags(&r->stg_ready[b], cudaEventDisableTiming));
      SP_CUDA(cudaEventCreateWithFlags(&r->stg_free[b], cudaEventDisableTiming));
    }
  }
  const int b = r->stg_next;
  const float* grads[SP_MAX_LOCAL];
  for (int l = 0; l < r->L; ++l) {
    const int g = r->cfg.rank * r->L + l;
    if (!host_grads[l]) {
      if (r->weights.empty() || r->weights[g] != 0.0)
        return fail(SP_ERR_ARG, "null host grad for a peer with nonzero weight");
      grads[l] = nullptr;
      continue;
    }
    if (!r->stg[b][l]) SP_CUDA(cudaMalloc(&r->stg[b][l], (size_t)r->npad * sizeof(float)));
    grads[l] = r->stg[b][l];
  }
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  // the round that last read staging buffer b (two calls ago) must be done
  // before it is overwritten; the copy then overlaps the previous round
  if (r->stg_used[b]) SP_CUDA(cudaStreamWaitEvent(r->h2d, r->stg_free[b], 0));
  for (int l = 0; l < r->L; ++l)
    if (grads[l])
      SP_CUDA(cudaMemcpyAsync(r->stg[b][l], host_grads[l], (size_t)r->n * sizeof(float),
                              cudaMemcpyHostToDevice, r->h2d));
  SP_CUDA(cudaEventRecord(r->stg_ready[b], r->h2d));
  SP_CUDA(cudaStreamWaitEvent(st, r->stg_ready[b], 0));
  std::vector<const void*> key;
  for (int l = 0; l < r->L; ++l) key.push_back(grads[l]);
  key.push_back(p);
  key.push_back(m);
  key.push_back(v);
  key.push_back(nullptr);
  rc = launch_graph(r, key, grads, p, m, v, step, st);
  if (rc) return rc;
  SP_CUDA(cudaEventRecord(r->stg_free[b], st));
  // the step's result back to the host: the updated parameters, on the
  // round's stream (PCIe is full duplex: overlaps the next step's H2D)
  if (host_p_out)
    SP_CUDA(cudaMemcpyAsync(host_p_out, p, (size_t)r->n * sizeof(float), cudaMemcpyDeviceToHost, st));
  r->stg_used[b] = true;
  r->stg_next = b ^ 1;
  return SP_OK;
}

int sp_round_run_phased(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                        int step, void* stream, sp_phase_times* t) {
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = upload_hparams(r, step, st);
  if (rc) return rc;
  rc = enqueue_round(r, grads, p, m, v, st, r->ev);
  if (rc) return rc;
  SP_CUDA(cudaStreamSynchronize(st));
  if (*(volatile int*)r->h_err == 1) return fail(SP_ERR_PEER, "cross-rank barrier timed out");
  if (t) {
    float* f[6] = {&t->pack_ms, &t->barrier_a_ms, &t->reduce_ms, &t->barrier_b_ms, &t->lamb_ms,
                   &t->barrier_c_ms};
    for (int k = 0; k < 6; ++k) SP_CUDA(cudaEventElapsedTime(f[k], r->ev[k], r->ev[k + 1]));
    SP_CUDA(cudaEventElapsedTime(&t->total_ms, r->ev[0], r->ev[6]));
  }
  return SP_OK;
}

int sp_round_lamb_chunks(const sp_round* r, int* tile) {
  if (tile) *tile = kLambTile;
  return r ? r->nchunks : -1;
}

int sp_round_describe(const sp_round_cfg* cfg, const int64_t* offsets, int sm_count, sp_plan_desc* out) {
  if (int rc = validate_cfg(cfg)) return rc;
  if (!offsets || !out || sm_count < 1) return fail(SP_ERR_ARG, "null argument");
  const int L = cfg->peers_per_rank, world = cfg->world, G = L * world;
  if (offsets[0] != 0 || offsets[G] != cfg->n) return fail(SP_ERR_ARG, "offsets must start at 0 and end at n");
  for (int g = 0; g < G; ++g)
    if (offsets[g + 1] < offsets[g]) return fail(SP_ERR_ARG, "offsets must be non-decreasing");
  *out = sp_plan_desc{};
  PackArgs a{};
  out->pack_ctas = pack_plan(*cfg, L, offsets, sm_count, a);
  out->pack_ranges = a.nr;
  out->unit_elems = cfg->wire == SP_WIRE_Q8 ? cfg->q8_block : (cfg->wire == SP_WIRE_FP16 ? 8 : 4);
  for (int j = 0; j < a.nr; ++j) {
    out->pack_owner[j] = a.owner[j];
    out->pack_first_unit[j] = a.lo[j];
    out->pack_units[j] = a.pref[j + 1] - a.pref[j];
    out->pack_cta_begin[j] = a.cta0[j];
  }
  out->pack_cta_begin[a.nr] = a.cta0[a.nr];
  out->own_lo = offsets[(size_t)cfg->rank * L];
  out->own_hi = offsets[(size_t)(cfg->rank + 1) * L];
  for (int k = 0; k < world; ++k) out->push_order[k] = push_rank(cfg->rank, world, k);
  out->avg_push_ranks = cfg->shard_lamb ? 1 : world;
  return SP_OK;
}

#ifdef SP_LAMB_TRACE
// Diagnostic builds: the stamps of the last k_lamb launch ([grid][stride]
// u64, sp_lamb.cuh kLambTraceStride); returns the grid.
int sp_round_lamb_trace(sp_round* r, unsigned long long* host, int cap) {
  if (!r || !r->d_trace) return -1;
  const int n = std::min(cap, r->lamb_grid * kLambTraceStride);
  cudaDeviceSynchronize();
  cudaMemcpy(host, r->d_trace, (size_t)n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return r->lamb_grid;
}
#endif

void* sp_round_wire_ptr(sp_round* r, int local_peer) {
  if (!r || local_peer < 0 || local_peer >= r->L) return nullptr;
  return r->wire(r->cfg.rank, r->cfg.rank * r->L + local_peer);
}

float* sp_round_param_ptr(sp_round* r) { return r && r->shard ? r->param(r->cfg.rank) : nullptr; }

void* sp_round_avg_ptr(sp_round* r) { return r ? const_cast<char*>(avg_buffer(r)) : nullptr; }

const float* sp_round_trust_ptr(sp_round* r) { return r ? r->d_trust : nullptr; }

int sp_round_copy_trust(sp_round* r, float* dst, void* stream) {
  if (!r || !dst) return fail(SP_ERR_ARG, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SP_CUDA(cudaMemcpyAsync(dst, r->d_trust, r->tsizes.size() * sizeof(float), cudaMemcpyDefault, st));
  return SP_OK;
}

int sp_round_read(sp_round* r, int which, int local_peer, size_t offset_bytes, void* host_dst,
                  size_t bytes) {
  if (!r || !host_dst) return fail(SP_ERR_ARG, "null argument");
  const char* src = nullptr;
  size_t cap = 0;
  if (which == SP_BUF_WIRE) {
    if (local_peer < 0 || local_peer >= r->L) return fail(SP_ERR_ARG, "local_peer out of range");
    src = r->wire(r->cfg.rank, r->cfg.rank * r->L + local_peer);
    cap = r->buf_bytes;
  } else if (which == SP_BUF_AVG) {
    src = avg_buffer(r);
    cap = r->buf_bytes;
  } else if (which == SP_BUF_TRUST) {
    src = reinterpret_cast<const char*>(r->d_trust);
    cap = r->tsizes.size() * sizeof(float);
  } else {
    return fail(SP_ERR_ARG, "unknown buffer");
  }
  if (offset_bytes > cap || bytes > cap - offset_bytes) return fail(SP_ERR_ARG, "read out of range");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  SP_CUDA(cudaDeviceSynchronize());
  SP_CUDA(cudaMemcpy(host_dst, src + offset_bytes, bytes, cudaMemcpyDeviceToHost));
  return SP_OK;
}

}  // extern "C"

namespace {

int ensure_accumulators(sp_round* r, int buf) {
  if (r->acc[buf][0]) return SP_OK;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  for (int l = 0; l < r->L; ++l) SP_CUDA(cudaMalloc(&r->acc[buf][l], (size_t)r->n * sizeof(float)));
  if (!r->d_stage) SP_CUDA(cudaMalloc(&r->d_stage, 2 * (size_t)r->L * sizeof(double)));
  return SP_OK;
}

}  // namespace

extern "C" {

int sp_round_accumulate(sp_round* r, int buf, int local_peer, const float* grad, double samples,
                        void* stream) {
  if (!r || !grad) return fail(SP_ERR_ARG, "null argument");
  if (buf < 0 || buf > 1) return fail(SP_ERR_ARG, "buf must be 0 or 1");
  if (local_peer < 0 || local_peer >= r->L) return fail(SP_ERR_ARG, "local_peer out of range");
  if (!(samples >= 0.0) || !std::isfinite(samples)) return fail(SP_ERR_ARG, "samples must be >= 0");
  if ((reinterpret_cast<uintptr_t>(grad) & 15) != 0) return fail(SP_ERR_SHAPE, "grad must be 16-byte aligned");
  if (int rc = ensure_accumulators(r, buf)) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int overwrite = r->host_count[buf][local_peer] == 0.0 ? 1 : 0;
  k_accumulate<<<grid_for(r->n / 4 + 1, 256, r->sm_count, 8), 256, 0, st>>>(
      r->acc[buf][local_peer], grad, r->n, overwrite);
  SP_CUDA(cudaGetLastError());
  r->host_count[buf][local_peer] += samples;
  return SP_OK;
}

float* sp_round_accumulator_ptr(sp_round* r, int buf, int local_peer) {
  if (!r || buf < 0 || buf > 1 || local_peer < 0 || local_peer >= r->L) return nullptr;
  if (ensure_accumulators(r, buf)) return nullptr;
  return r->acc[buf][local_peer];
}

double sp_round_samples(const sp_round* r, int buf, int local_peer) {
  if (!r || buf < 0 || buf > 1 || local_peer < 0 || local_peer >= r->L) return -1.0;
  return r->host_count[buf][local_peer];
}

int sp_round_add_samples(sp_round* r, int buf, int local_peer, double samples) {
  if (!r || buf < 0 || buf > 1 || local_peer < 0 || local_peer >= r->L)
    return fail(SP_ERR_ARG, "bad buffer or peer");
  if (!(samples >= 0.0) || !std::isfinite(samples)) return fail(SP_ERR_ARG, "samples must be >= 0");
  r->host_count[buf][local_peer] += samples;
  return SP_OK;
}

int sp_round_run_accumulated(sp_round* r, int buf, float* p, float* m, float* v, int step,
                             void* stream) {
  if (!r) return fail(SP_ERR_ARG, "null round");
  if (buf < 0 || buf > 1) return fail(SP_ERR_ARG, "buf must be 0 or 1");
  if (int rc = ensure_accumulators(r, buf)) return rc;
  const float* grads[SP_MAX_LOCAL];
  for (int l = 0; l < r->L; ++l) grads[l] = r->acc[buf][l];
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  if (r->cfg.world == 1) {  // every count is local: refuse an empty round up front
    double s = 0.0;
    for (int l = 0; l < r->L; ++l) s += r->host_count[buf][l];
    if (!(s > 0.0)) return fail(SP_ERR_STATE, "no samples accumulated in this buffer");
  }
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SP_CUDA(cudaMemcpyAsync(r->d_stage + (size_t)buf * r->L, r->host_count[buf],
                          (size_t)r->L * sizeof(double), cudaMemcpyHostToDevice, st));
  r->acc_buf = buf;
  std::vector<const void*> key;
  for (int l = 0; l < r->L; ++l) key.push_back(grads[l]);
  key.push_back(p);
  key.push_back(m);
  key.push_back(v);
  key.push_back(reinterpret_cast<const void*>((uintptr_t)(buf + 1)));  // mode tag
  rc = launch_graph(r, key, grads, p, m, v, step, st);
  r->acc_buf = -1;
  if (rc) return rc;
  for (int l = 0; l < r->L; ++l) r->host_count[buf][l] = 0.0;  // next accumulate overwrites
  return SP_OK;
}

int sp_vec_scale(double* dst, const double* src, double w, int64_t n, void* stream) {
  if (!dst || !src || n < 0) return fail(SP_ERR_ARG, "bad vector");
  if (n == 0) return SP_OK;
  k_vec_scale<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0,
                static_cast<cudaStream_t>(stream)>>>(dst, src, w, n);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_vec_sum(double* dst, const double* const* srcs, int k, int64_t n, void* stream) {
  if (!dst || !srcs || k < 1 || k > SP_MAX_PEERS || n < 0) return fail(SP_ERR_ARG, "bad vector list");
  if (n == 0) return SP_OK;
  VecList l{};
  for (int c = 0; c < k; ++c) {
    if (!srcs[c]) return fail(SP_ERR_ARG, "null source vector");
    l.src[c] = srcs[c];
  }
  l.k = k;
  k_vec_sum<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0,
              static_cast<cudaStream_t>(stream)>>>(dst, l, n);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_vec_div(double* dst, const double* src, double d, int64_t n, void* stream) {
  if (!dst || !src || n < 0) return fail(SP_ERR_ARG, "bad vector");
  if (n == 0) return SP_OK;
  k_vec_div<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0,
              static_cast<cudaStream_t>(stream)>>>(dst, src, d, n);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

int sp_fill_synthetic(float* dev, int64_t n, uint64_t seed, int peer, float scale,
                      int64_t outlier_every, float outlier_mult, void* stream) {
  if (!dev || n < 0) return fail(SP_ERR_ARG, "bad buffer");
  if (n == 0) return SP_OK;
  int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  k_fill_synthetic<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dev, n, (unsigned long long)seed, peer, scale, outlier_every, outlier_mult);
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

}  // extern "C"
