// sp_round.cu — C-ABI implementation of the averaging-round executor.
//
// Host side of libsp_round.so: buffer layout, CUDA IPC wiring between ranks,
// assignment upload, CUDA-graph capture/replay of the round. Kernels live in
// sp_kernels.cuh. See include/sp_round.h for the contract and the reference
// interfaces each entry point replaces.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sp_kernels.cuh"
#include "sp_round_fused.cuh"
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

}  // namespace

struct sp_round {
  sp_round_cfg cfg{};
  std::vector<int64_t> tsizes;
  int G = 0, L = 0;
  int64_t n = 0, npad = 0;
  int align = 8;
  size_t buf_bytes = 0;     // one wire/avg buffer (codes + q8 scales)
  size_t flags_bytes = 256;  // barrier flags + per-buffer sample-count tables
  size_t ctr_bytes = 0;     // arrived[ncells] + ready[ncells] (fused round)
  // fused round (one persistent kernel per round)
  bool fused_round = true;
  int cell = 8192;
  int ncells = 0;
  int round_grid = 0;
  int nritems = 0;
  unsigned* d_ritems = nullptr;
  int* d_rq = nullptr;                // [work, exited]
  unsigned* d_repoch = nullptr;
  unsigned char* d_cell_owners = nullptr;
  std::vector<Chunk> h_chunks;
  // shared (IPC-exported) allocation: [flags][inbox: one slot per peer, G][avg]
  // slot g of rank k holds peer g's packed gradient for the range k owns
  char* shared = nullptr;
  size_t shared_bytes = 0;
  char* base[SP_MAX_RANKS] = {};  // every rank's shared allocation (mapped)
  bool connected = false;
  unsigned long long* epoch = nullptr;  // barrier epoch
  int* h_err = nullptr;  // host-mapped
  int* d_err = nullptr;
  // LAMB tables
  int nchunks = 0;
  int nchunks_cap = 0;
  int64_t lamb_chunk = kLambChunk;
  // segmented pipeline (world > 1): exchange of segment s+1 overlaps LAMB
  // pass 1 of segment s on the aux stream
  int segments = 1;
  int seg_lamb_grid = 1 << 30;  // CTA cap of a segment's pass-1 launch
  int xchg_per_sm = 8;          // CTAs per SM of the exchange kernels
  double pack_local_weight = 1.0;  // CTA share of the local range in the pack (vs remote)
  std::vector<int> p1_off;   // K+1 offsets of the per-segment pass-1 item lists
  int p2_off = 0;            // pass-2 items
  cudaStream_t aux = nullptr;
  cudaEvent_t seg_ev[9] = {};
  // device-side accumulation (two buffers, so a round can consume one while
  // the next step's micro-batches land in the other)
  float* acc[2][SP_MAX_LOCAL] = {};
  double host_count[2][SP_MAX_LOCAL] = {};
  double* d_stage = nullptr;  // [2][L] staged counts
  int acc_buf = -1;           // >= 0 while enqueuing an accumulated round
  Chunk* d_chunks = nullptr;
  int2* d_tchunks = nullptr;
  float2* d_partial = nullptr;
  float* d_trust = nullptr;
  float* d_step_scale = nullptr;
  float* d_hp = nullptr;
  // fused LAMB work queue
  bool fused_lamb = true;
  int l2_hints = 0;
  int lamb_grid = 0;
  int nitems = 0;
  int* d_items = nullptr;
  int* d_qstate = nullptr;           // [work, exited, done[T]...]
  unsigned int* d_ready = nullptr;
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
  cudaEvent_t ev[8] = {};
  int sm_count = 148;
  // sharded LAMB (cfg.shard_lamb): flat parameter vector + per-rank norm table
  bool shard = false;
  size_t param_off = 0, norms_off = 0, nflags_off = 0;
  // one-kernel sharded LAMB (k_shard_lamb_fused): its own work list, grid,
  // epoch, and the norm flags in the shared allocation
  bool shard_fused = false;  // opt-in (SP_SHARD_FUSED=1): measured slower than the chain
  int shard_lag = 0;      // pass-2 items of tensor t queued this many items after its pass 1
  int shard_grid = 0;
  int* d_sitems = nullptr;
  int nsitems = 0;
  unsigned long long* d_sepoch = nullptr;
  // hybrid split: tensors [0, shard_t0) (elements [0, shard_cut)) keep the
  // replicated LAMB on a second stream, tensors [shard_t0, T) are sharded
  int shard_t0 = 0;
  int64_t shard_cut = 0;
  int nchunks_rep = 0;    // chunks of the replicated tensors (full range), first in the table
  int hybrid_grid = 0;    // CTA cap of the replicated LAMB running beside the sharded chain

  float* param(int rank) const { return reinterpret_cast<float*>(base[rank] + param_off); }
  double2* norms(int rank) const { return reinterpret_cast<double2*>(base[rank] + norms_off); }
  unsigned long long* nflags(int rank) const {
    return reinterpret_cast<unsigned long long*>(base[rank] + nflags_off);
  }
  char* wire(int rank, int g) const {
    return base[rank] + flags_bytes + ctr_bytes + (size_t)g * buf_bytes;
  }
  char* avg(int rank) const { return base[rank] + flags_bytes + ctr_bytes + (size_t)G * buf_bytes; }
  double* counts(int rank, int buf) const {
    return reinterpret_cast<double*>(base[rank] + 256) + (size_t)buf * G;
  }
  unsigned* arrived(int rank) const { return reinterpret_cast<unsigned*>(base[rank] + flags_bytes); }
  unsigned* ready(int rank) const {
    return reinterpret_cast<unsigned*>(base[rank] + flags_bytes + ctr_bytes / 2);
  }
  unsigned long long* flags(int rank) const {
    return reinterpret_cast<unsigned long long*>(base[rank]);
  }
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

// Element boundaries where LAMB chunks must split so each chunk lies in one
// segment of one owner's range: owner k's range [lo, hi) is cut at
// lo + align_down((hi - lo) * s / K, align), s = 0..K.
int64_t seg_cut(const sp_round* r, int k, int s) {
  const int64_t lo = r->offsets[(size_t)k * r->L], hi = r->offsets[(size_t)(k + 1) * r->L];
  if (s >= r->segments) return hi;
  return lo + (hi - lo) * s / r->segments / r->align * r->align;
}

// Hybrid sharded LAMB (opt-in experiment): tensors [0, t0) keep the
// replicated LAMB (HBM-bound, every rank steps them) on a second stream while
// tensors [t0, T) are sharded (NVLink-bound: owners step their range and push
// fp32 parameters). t0 is the tensor edge closest to SP_SHARD_FRACTION, or
// with SP_SHARD_FRACTION=model the edge minimizing the modelled time
//   (1-a) * avg push + max(replicated LAMB(1-a), sharded pass 1 + push(a)),
// a = sharded share of the elements. Default: a = 1 (everything sharded).
void choose_shard_cut(sp_round* r) {
  const sp_round_cfg& c = r->cfg;
  const int T = (int)r->tsizes.size();
  const double n = (double)r->n;
  const double b = c.wire == SP_WIRE_FP32 ? 4.0 : c.wire == SP_WIRE_FP16 ? 2.0 : 1.0 + 4.0 / c.q8_block;
  // Default: shard everything. Running the replicated half beside the
  // sharded chain was measured slower at N=4 (both halves contend for SMs
  // and HBM: fp16 234 us at a = 0.5 vs 169 us fully sharded), so
  // the model-chosen split is opt-in: SP_SHARD_FRACTION=<a> or =model.
  double want = 1.0;
  if (const char* e = std::getenv("SP_SHARD_FRACTION"))
    want = std::string(e) == "model" ? -1.0 : std::atof(e);
  const double hbm = 6.2e12, nvl = 6.0e11, w = c.world;
  int best = 0;
  double best_cost = 1e300;
  int64_t off = 0;
  for (int t0 = 0; t0 <= T; ++t0) {
    const double a = (n - (double)off) / n;  // sharded share
    double cost;
    if (want >= 0.0) {
      cost = std::fabs(a - want);
    } else {
      const double push_avg = (1.0 - a) * n * b * (w - 1.0) / w / nvl;
      const double rep = (1.0 - a) * n * (36.0 + b) / hbm;
      const double shd = a * n / w * (36.0 + b) / hbm + a * n * 4.0 * (w - 1.0) / w / nvl;
      cost = push_avg + std::max(rep, shd);
    }
    if (cost < best_cost - 1e-15) {
      best_cost = cost;
      best = t0;
    }
    if (t0 < T) off += r->tsizes[(size_t)t0];
  }
  r->shard_t0 = best;
  int64_t cut = 0;
  for (int t = 0; t < best; ++t) cut += r->tsizes[(size_t)t];
  r->shard_cut = cut;
}

// Chunk table (tensor edges, every multiple of lamb_chunk, segment cuts),
// per-tensor chunk ranges and the fused-LAMB work lists:
//   [pass 1 of segment 0] ... [pass 1 of segment K-1] [pass 2 of all chunks].
// With K = 1 one launch walks both lists (pass 1 first: the in-flight window
// of the persistent grid exceeds L2, so a shorter lag only adds trust waits,
// profiles/r01/lamb_sweep.txt).
int build_lamb_tables(sp_round* r, bool with_cuts) {
  std::vector<int64_t> cuts;
  if (with_cuts && r->segments > 1)
    for (int k = 0; k < r->cfg.world; ++k)
      for (int s = 1; s < r->segments; ++s) cuts.push_back(seg_cut(r, k, s));
  std::sort(cuts.begin(), cuts.end());
  std::vector<Chunk> chunks;
  std::vector<int2> tch;
  // sharded LAMB: the sharded tensors only over the range this rank owns
  int64_t own_lo = 0, own_hi = r->n;
  r->shard_t0 = 0;
  r->shard_cut = 0;
  if (r->shard && !r->offsets.empty()) {
    own_lo = r->offsets[(size_t)r->cfg.rank * r->L];
    own_hi = r->offsets[(size_t)(r->cfg.rank + 1) * r->L];
    choose_shard_cut(r);
  }
  r->nchunks_rep = 0;
  int64_t off = 0;
  size_t ci = 0;
  for (size_t t = 0; t < r->tsizes.size(); ++t) {
    const bool sharded = r->shard && (int)t >= r->shard_t0;
    if (r->shard && (int)t == r->shard_t0) r->nchunks_rep = (int)chunks.size();
    const int64_t end = sharded ? std::min(off + r->tsizes[t], own_hi) : off + r->tsizes[t];
    int2 rg;
    rg.x = (int)chunks.size();
    int64_t s = sharded ? std::max(off, own_lo) : off;
    while (s < end) {
      int64_t e = std::min(end, (s / r->lamb_chunk + 1) * r->lamb_chunk);
      while (ci < cuts.size() && cuts[ci] <= s) ++ci;
      if (ci < cuts.size() && cuts[ci] < e) e = cuts[ci];
      chunks.push_back(Chunk{(long long)s, (int)(e - s), (int)t});
      s = e;
    }
    rg.y = (int)chunks.size();
    tch.push_back(rg);
    off += r->tsizes[t];
  }
  if (r->shard && r->shard_t0 >= (int)r->tsizes.size()) r->nchunks_rep = (int)chunks.size();
  if ((int)chunks.size() > r->nchunks_cap) return fail(SP_ERR_STATE, "LAMB chunk table overflow");
  const int K = with_cuts ? r->segments : 1;
  std::vector<std::vector<int>> p1((size_t)K);
  for (size_t c = 0; c < chunks.size(); ++c) {
    int seg = 0;
    if (K > 1) {
      const int64_t st = chunks[c].start;
      int k0 = 0;
      while (k0 + 1 < r->cfg.world && st >= r->offsets[(size_t)(k0 + 1) * r->L]) ++k0;
      while (seg + 1 < K && st >= seg_cut(r, k0, seg + 1)) ++seg;
    }
    p1[(size_t)seg].push_back((int)c);
  }
  std::vector<int> items;
  r->p1_off.assign((size_t)K + 1, 0);
  const char* lag_env = std::getenv("SP_LAMB_LAG");
  if (r->shard) {  // fused queue over the replicated tensors only
    for (int c = 0; c < r->nchunks_rep; ++c) items.push_back(c);
    r->p1_off[1] = r->p2_off = (int)items.size();
    for (int c = 0; c < r->nchunks_rep; ++c) items.push_back(~c);
  } else if (K == 1 && lag_env) {
    // single launch, pass 2 of tensor t queued `lag` items after its last
    // pass-1 chunk (tuning experiment for L2 reuse between the passes)
    const size_t lag = (size_t)std::max(0, std::atoi(lag_env));
    std::vector<std::pair<int, size_t>> pend;
    size_t head = 0;
    auto flush = [&](bool all) {
      while (head < pend.size() && (all || pend[head].second + lag <= items.size())) {
        const int2 rg = tch[(size_t)pend[head].first];
        for (int c = rg.x; c < rg.y; ++c) items.push_back(~c);
        ++head;
      }
    };
    for (size_t c = 0; c < chunks.size(); ++c) {
      items.push_back((int)c);
      if ((int)c == tch[(size_t)chunks[c].tensor].y - 1) pend.push_back({chunks[c].tensor, items.size()});
      flush(false);
    }
    flush(true);
    r->p1_off[1] = r->p2_off = (int)items.size();
  } else {
    for (int q = 0; q < K; ++q) {
      r->p1_off[(size_t)q] = (int)items.size();
      items.insert(items.end(), p1[(size_t)q].begin(), p1[(size_t)q].end());
    }
    r->p1_off[(size_t)K] = (int)items.size();
    r->p2_off = (int)items.size();
    for (size_t c = 0; c < chunks.size(); ++c) items.push_back(~(int)c);
  }
  r->nchunks = (int)chunks.size();
  r->nitems = (int)items.size();
  if (r->shard && r->d_sitems) {
    // one-kernel sharded LAMB (used when nothing is replicated): pass-1
    // items in chunk order, pass 2 of tensor t `shard_lag` items after its
    // last pass-1 chunk
    std::vector<int> si;
    std::vector<std::pair<int, size_t>> pend;
    size_t head = 0;
    const size_t lag = (size_t)std::max(0, r->shard_lag);
    auto flush = [&](bool all) {
      while (head < pend.size() && (all || pend[head].second + lag <= si.size())) {
        const int2 rg = tch[(size_t)pend[head].first];
        for (int c = rg.x; c < rg.y; ++c) si.push_back(~c);
        ++head;
      }
    };
    for (size_t c = 0; c < chunks.size(); ++c) {
      si.push_back((int)c);
      if ((int)c == tch[(size_t)chunks[c].tensor].y - 1) pend.push_back({chunks[c].tensor, si.size()});
      flush(false);
    }
    flush(true);
    r->nsitems = (int)si.size();
    SP_CUDA(cudaSetDevice(r->cfg.device));
    if (!si.empty())
      SP_CUDA(cudaMemcpy(r->d_sitems, si.data(), si.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  r->h_chunks = chunks;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  SP_CUDA(cudaMemcpy(r->d_chunks, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
  SP_CUDA(cudaMemcpy(r->d_tchunks, tch.data(), tch.size() * sizeof(int2), cudaMemcpyHostToDevice));
  SP_CUDA(cudaMemcpy(r->d_items, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice));
  return SP_OK;
}

int grid_for(int64_t work_items, int threads, int sm_count, int per_sm) {
  int64_t g = (work_items + threads - 1) / threads;
  g = std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sm_count * per_sm));
  return (int)g;
}

// Fused-round work list for this rank (see sp_round_fused.cuh): scatter items
// column by column over owners in rotated order, then this rank's reduce
// cells, then LAMB pass-1 chunks in expected arrival order, then pass 2.
int build_round_items(sp_round* r) {
  const sp_round_cfg& c = r->cfg;
  const int W = c.world, me = c.rank;
  std::vector<int64_t> first(W), len(W);
  std::vector<unsigned char> owners((size_t)r->ncells, 0);
  for (int k = 0; k < W; ++k) {
    const int64_t lo = r->offsets[(size_t)k * r->L], hi = r->offsets[(size_t)(k + 1) * r->L];
    first[k] = lo / r->cell;
    len[k] = hi > lo ? (std::min(hi, r->n) + r->cell - 1) / r->cell - first[k] : 0;
    for (int64_t j = first[k]; j < first[k] + len[k]; ++j) owners[(size_t)j]++;
  }
  std::vector<unsigned> items;
  int64_t maxlen = 0;
  for (int k = 0; k < W; ++k) maxlen = std::max(maxlen, len[k]);
  // LAMB pass-1 chunks grouped by the column of their cell (position within
  // the owning rank's range), the order in which owners finish them
  std::vector<std::vector<int>> l1_by_col((size_t)std::max<int64_t>(maxlen, 1));
  for (size_t i = 0; i < r->h_chunks.size(); ++i) {
    const int64_t st = r->h_chunks[i].start;
    int k0 = 0;
    while (k0 + 1 < W && st >= r->offsets[(size_t)(k0 + 1) * r->L]) ++k0;
    l1_by_col[(size_t)(st / r->cell - first[k0])].push_back((int)i);
  }
  // Interleave: column j's reduce is queued `lag` items after column j's last
  // scatter item, and its pass-1 chunks `lag` items after that, so scatter
  // (NVLink), reduce and LAMB pass 1 (HBM) of different columns run at the
  // same time. Every waiting item only depends on items queued before it
  // (here and, column-wise, on every other rank), so the queue stays
  // deadlock-free. lag = 0 would make every column wait for itself.
  const char* lag_env = std::getenv("SP_ROUND_LAG");
  const size_t lag = lag_env ? (size_t)std::atol(lag_env) : (size_t)r->round_grid;
  std::vector<std::pair<size_t, int64_t>> pend_r, pend_l;  // (ready position, column)
  size_t hr = 0, hl = 0;
  auto flush = [&](bool all) {
    bool moved = true;
    while (moved) {
      moved = false;
      while (hr < pend_r.size() && (all || pend_r[hr].first <= items.size())) {
        const int64_t j = pend_r[hr++].second;
        if (j < len[me]) items.push_back(make_item(kStR, 0u, (unsigned)(first[me] + j)));
        pend_l.push_back({items.size() + lag, j});
        moved = true;
      }
      while (hl < pend_l.size() && (all || pend_l[hl].first <= items.size())) {
        for (int i : l1_by_col[(size_t)pend_l[hl].second]) items.push_back(make_item(kStL1, 0u, (unsigned)i));
        ++hl;
        moved = true;
      }
    }
  };
  for (int64_t j = 0; j < maxlen; ++j) {
    for (int d = 1; d <= W; ++d) {
      const int k = (me + d) % W;
      if (j < len[k]) items.push_back(make_item(kStS, (unsigned)k, (unsigned)(first[k] + j)));
    }
    pend_r.push_back({items.size() + lag, j});
    flush(false);
  }
  flush(true);
  for (size_t i = 0; i < r->h_chunks.size(); ++i) items.push_back(make_item(kStL2, 0u, (unsigned)i));
  r->nritems = (int)items.size();
  SP_CUDA(cudaSetDevice(c.device));
  SP_CUDA(cudaMemcpy(r->d_ritems, items.data(), items.size() * sizeof(unsigned), cudaMemcpyHostToDevice));
  SP_CUDA(cudaMemcpy(r->d_cell_owners, owners.data(), owners.size(), cudaMemcpyHostToDevice));
  return SP_OK;
}

// With one rank and a single contributing peer the average is the identity
// on that peer's wire values: fp32/fp16 because acc = 1.0f * x = x is exactly
// representable in the wire format, q8 by definition (a single contributor's
// codes and scales are forwarded; sp_oracle_reduce). The averaged vector IS
// the peer's inbox slot and the reduce kernel is skipped.
const char* identity_avg(const sp_round* r) {
  const sp_round_cfg& c = r->cfg;
  if (c.world != 1 || !r->assigned || r->fused_round || r->acc_buf >= 0)
    return nullptr;
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

LambArgs make_lamb_args(sp_round* r, float* p, float* m, float* v) {
  const sp_round_cfg& c = r->cfg;
  LambArgs a{};
  a.avg = avg_buffer(r);
  a.avg_scale = c.wire == SP_WIRE_Q8 ? reinterpret_cast<const float*>(avg_buffer(r) + r->npad)
                                     : nullptr;
  a.p = p;
  a.m = m;
  a.v = v;
  a.chunks = r->d_chunks;
  a.partial = r->d_partial;
  a.hp = r->d_hp;
  a.step_scale = r->d_step_scale;
  a.b1 = c.beta1;
  a.b2 = c.beta2;
  a.omb1 = 1.0f - c.beta1;
  a.omb2 = 1.0f - c.beta2;
  a.eps = c.eps;
  a.wd = c.weight_decay;
  a.qshift = __builtin_ctz((unsigned)std::max(c.q8_block, 1));
  a.l2_hints = r->l2_hints;
  return a;
}

FusedLamb make_lamb_queue(sp_round* r) {
  FusedLamb q{};
  q.items = r->d_items;
  q.nitems = r->nitems;
  q.work = r->d_qstate;
  q.exited = r->d_qstate + 1;
  q.done = r->d_qstate + 2;
  q.ready = r->d_ready;
  q.tchunks = r->d_tchunks;
  q.trust = r->d_trust;
  q.ntensors = r->cfg.num_tensors;
  return q;
}

int enqueue_fused(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                  cudaStream_t st, cudaEvent_t* ev) {
  const sp_round_cfg& c = r->cfg;
  if (ev)
    for (int k = 1; k <= 4; ++k) SP_CUDA(cudaEventRecord(ev[k], st));
  RoundFused f{};
  f.items = r->d_ritems;
  f.nitems = r->nritems;
  f.work = r->d_rq;
  f.exited = r->d_rq + 1;
  f.epoch = r->d_repoch;
  f.err = r->d_err;
  const double to = c.barrier_timeout_s > 0 ? c.barrier_timeout_s : 20.0;
  f.timeout_ns = (unsigned long long)(to * 1e9);
  f.n = r->n;
  f.npad = r->npad;
  f.cell = r->cell;
  f.world = c.world;
  f.rank = c.rank;
  f.L = r->L;
  for (int k = 0; k <= c.world; ++k) f.rank_lo[k] = r->offsets[(size_t)k * r->L];
  for (int l = 0; l < r->L; ++l) {
    const int g = c.rank * r->L + l;
    const bool zero_copy = c.world == 1 && c.wire == SP_WIRE_FP32 &&
                           (const void*)grads[l] == (const void*)r->wire(c.rank, g);
    f.src[l] = zero_copy ? nullptr : grads[l];
  }
  for (int k = 0; k < c.world; ++k) {
    f.inbox[k] = r->wire(k, 0);
    f.arrived[k] = r->arrived(k);
    const int d = (c.rank + 1 + k) % c.world;  // push order: next rank first, self last
    f.avg[k] = r->avg(d);
    f.ready_of[k] = r->ready(d);
  }
  f.slot_bytes = r->buf_bytes;
  double wsum = 0.0;
  for (double w : r->weights) wsum += w;
  for (int g = 0; g < r->G; ++g) {
    if (r->weights[g] == 0.0) continue;
    f.peer[f.npeers] = g;
    f.w[f.npeers] = (float)(r->weights[g] / wsum);
    ++f.npeers;
  }
  f.my_ready = r->ready(c.rank);
  f.cell_owners = r->d_cell_owners;
  LambArgs a = make_lamb_args(r, p, m, v);
  FusedLamb q = make_lamb_queue(r);
  const int grid = r->round_grid;
  switch (c.wire) {
    case SP_WIRE_FP32: k_round_fused<SP_WIRE_FP32><<<grid, kLambThreads, 0, st>>>(f, a, q); break;
    case SP_WIRE_FP16: k_round_fused<SP_WIRE_FP16><<<grid, kLambThreads, 0, st>>>(f, a, q); break;
    default: k_round_fused<SP_WIRE_Q8><<<grid, kLambThreads, 0, st>>>(f, a, q); break;
  }
  SP_CUDA(cudaGetLastError());
  if (ev)
    for (int k = 5; k <= 7; ++k) SP_CUDA(cudaEventRecord(ev[k], st));
  return SP_OK;
}

// Enqueues the whole round on `st`. ev != nullptr records phase events.
int launch_lamb(sp_round* r, LambArgs a, int first_item, int nitems, bool final_launch,
                cudaStream_t st) {
  const sp_round_cfg& c = r->cfg;
  FusedLamb f = make_lamb_queue(r);
  f.items = r->d_items + first_item;
  f.nitems = nitems;
  f.final_launch = final_launch ? 1 : 0;
  if (nitems <= 0 && !final_launch) return SP_OK;
  // a segment's pass 1 shares the GPU with the next segment's exchange
  const int cap = final_launch ? r->lamb_grid : std::min(r->lamb_grid, r->seg_lamb_grid);
  const int g = std::max(1, std::min(cap, nitems));
  switch (c.wire) {
    case SP_WIRE_FP32: k_lamb_fused<SP_WIRE_FP32><<<g, kLambThreads, 0, st>>>(a, f); break;
    case SP_WIRE_FP16: k_lamb_fused<SP_WIRE_FP16><<<g, kLambThreads, 0, st>>>(a, f); break;
    default: k_lamb_fused<SP_WIRE_Q8><<<g, kLambThreads, 0, st>>>(a, f); break;
  }
  SP_CUDA(cudaGetLastError());
  return SP_OK;
}

// Sharded LAMB (cfg.shard_lamb), hybrid with the replicated one:
//   aux stream: fused replicated LAMB over tensors [0, t0) (full range, every
//               rank), capped at hybrid_grid CTAs so the chain below has SMs;
//   st:         tensors [t0, T): pass 1 over the owned chunks, per-tensor norm
//               partials pushed to every rank + barrier, trust (rank-ordered
//               sum), pass 2 storing p' into every rank's parameter vector +
//               barrier (no rank may read parameters before every owner has
//               stored its range);
// then st joins aux. HBM-bound and NVLink-bound halves run side by side.
int enqueue_shard_lamb(sp_round* r, const LambArgs& la, const BarrierArgs& ba, cudaStream_t st,
                       cudaEvent_t* ev) {
  const sp_round_cfg& c = r->cfg;
  const int T = c.num_tensors, t0 = r->shard_t0;
  const int nR = r->nchunks_rep, nS = r->nchunks - nR;
  if (nR > 0) {
    SP_CUDA(cudaEventRecord(r->seg_ev[8], st));
    SP_CUDA(cudaStreamWaitEvent(r->aux, r->seg_ev[8], 0));
    FusedLamb f = make_lamb_queue(r);
    f.nitems = 2 * nR;
    f.final_launch = 1;
    const int g = std::max(1, std::min(t0 < T ? r->hybrid_grid : r->lamb_grid, nR));
    switch (c.wire) {
      case SP_WIRE_FP32: k_lamb_fused<SP_WIRE_FP32><<<g, kLambThreads, 0, r->aux>>>(la, f); break;
      case SP_WIRE_FP16: k_lamb_fused<SP_WIRE_FP16><<<g, kLambThreads, 0, r->aux>>>(la, f); break;
      default: k_lamb_fused<SP_WIRE_Q8><<<g, kLambThreads, 0, r->aux>>>(la, f); break;
    }
    SP_CUDA(cudaGetLastError());
  }
  LambArgs ls = la;  // the sharded chunks follow the replicated ones in the table
  ls.chunks = r->d_chunks + nR;
  ls.partial = r->d_partial + nR;
  ParamPush pp{};
  pp.ndst = c.world;
  for (int k = 0; k < c.world; ++k) pp.dst[k] = r->param((c.rank + 1 + k) % c.world);
  // (the choice must not depend on this rank's item count: a rank that owns
  // nothing still publishes zero norms through the same protocol)
  if (t0 < T && nR == 0 && r->shard_fused) {
    // the whole sharded step as one persistent kernel (k_shard_lamb_fused)
    ShardFused f{};
    f.items = r->d_sitems;
    f.nitems = r->nsitems;
    f.work = r->d_qstate;
    f.exited = r->d_qstate + 1;
    f.done = r->d_qstate + 2;
    f.tchunks = r->d_tchunks;
    for (int k = 0; k < c.world; ++k) {
      f.table[k] = r->norms((c.rank + 1 + k) % c.world);
      f.flags[k] = r->nflags((c.rank + 1 + k) % c.world);
    }
    f.my_table = r->norms(c.rank);
    f.my_flags = r->nflags(c.rank);
    f.epoch = r->d_sepoch;
    f.trust = r->d_trust;
    f.step_scale = r->d_step_scale;
    f.push = pp;
    f.rank = c.rank;
    f.world = c.world;
    f.T = T;
    f.err = r->d_err;
    f.timeout_ns = (unsigned long long)((c.barrier_timeout_s > 0 ? c.barrier_timeout_s : 20.0) * 1e9);
    const int g = std::max(1, std::min(r->shard_grid, r->nsitems));
    switch (c.wire) {
      case SP_WIRE_FP32: k_shard_lamb_fused<SP_WIRE_FP32><<<g, kLambThreads, 0, st>>>(ls, f); break;
      case SP_WIRE_FP16: k_shard_lamb_fused<SP_WIRE_FP16><<<g, kLambThreads, 0, st>>>(ls, f); break;
      default: k_shard_lamb_fused<SP_WIRE_Q8><<<g, kLambThreads, 0, st>>>(ls, f); break;
    }
    SP_CUDA(cudaGetLastError());
    if (ev) {
      SP_CUDA(cudaEventRecord(ev[5], st));
      SP_CUDA(cudaEventRecord(ev[6], st));
    }
    if (c.world > 1) {  // every owner's parameters have landed everywhere
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    if (ev) SP_CUDA(cudaEventRecord(ev[7], st));
    return SP_OK;
  }
  if (t0 < T && nR == 0) {
    // default chain, every tensor sharded: pass 1 with the norm publication
    // folded in -> barrier -> pass 2 + push with the trust folded in -> barrier
    ShardNormArgs na{};
    na.tchunks = r->d_tchunks;
    na.ndst = c.world;
    for (int k = 0; k < c.world; ++k) na.table[k] = r->norms((c.rank + 1 + k) % c.world);
    na.rank = c.rank;
    na.T = T;
    na.t0 = 0;
    // one resident wave, grid-stride over the chunks (no partial second wave)
    const int g = std::max(1, std::min(nS, r->lamb_grid));
    switch (c.wire) {
      case SP_WIRE_FP32: k_lamb_moments_shard<SP_WIRE_FP32><<<g, kLambThreads, 0, st>>>(ls, na, r->d_qstate + 2, nS); break;
      case SP_WIRE_FP16: k_lamb_moments_shard<SP_WIRE_FP16><<<g, kLambThreads, 0, st>>>(ls, na, r->d_qstate + 2, nS); break;
      default: k_lamb_moments_shard<SP_WIRE_Q8><<<g, kLambThreads, 0, st>>>(ls, na, r->d_qstate + 2, nS); break;
    }
    SP_CUDA(cudaGetLastError());
    if (ev) SP_CUDA(cudaEventRecord(ev[5], st));
    if (c.world > 1) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    if (ev) SP_CUDA(cudaEventRecord(ev[6], st));
    const double2* tab = r->norms(c.rank);
    switch (c.wire) {
      case SP_WIRE_FP32: k_lamb_update_push_trust<SP_WIRE_FP32><<<g, kLambThreads, 0, st>>>(ls, pp, tab, c.world, T, 0, r->d_trust, r->d_step_scale, nS); break;
      case SP_WIRE_FP16: k_lamb_update_push_trust<SP_WIRE_FP16><<<g, kLambThreads, 0, st>>>(ls, pp, tab, c.world, T, 0, r->d_trust, r->d_step_scale, nS); break;
      default: k_lamb_update_push_trust<SP_WIRE_Q8><<<g, kLambThreads, 0, st>>>(ls, pp, tab, c.world, T, 0, r->d_trust, r->d_step_scale, nS); break;
    }
    SP_CUDA(cudaGetLastError());
    if (c.world > 1) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    if (ev) SP_CUDA(cudaEventRecord(ev[7], st));
    return SP_OK;
  }
  if (t0 < T) {
    if (nS > 0) {
      switch (c.wire) {
        case SP_WIRE_FP32: k_lamb_moments<SP_WIRE_FP32><<<nS, kLambThreads, 0, st>>>(ls); break;
        case SP_WIRE_FP16: k_lamb_moments<SP_WIRE_FP16><<<nS, kLambThreads, 0, st>>>(ls); break;
        default: k_lamb_moments<SP_WIRE_Q8><<<nS, kLambThreads, 0, st>>>(ls); break;
      }
      SP_CUDA(cudaGetLastError());
    }
    if (ev) SP_CUDA(cudaEventRecord(ev[5], st));
    ShardNormArgs na{};
    na.partial = r->d_partial;
    na.tchunks = r->d_tchunks;
    na.ndst = c.world;
    for (int k = 0; k < c.world; ++k) na.table[k] = r->norms((c.rank + 1 + k) % c.world);
    na.rank = c.rank;
    na.T = T;
    na.t0 = t0;
    k_shard_norms<<<T - t0, 256, 0, st>>>(na);
    SP_CUDA(cudaGetLastError());
    if (c.world > 1) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    k_shard_trust<<<(T - t0 + 255) / 256, 256, 0, st>>>(r->norms(c.rank), c.world, T, t0, r->d_hp,
                                                        r->d_trust, r->d_step_scale);
    SP_CUDA(cudaGetLastError());
    if (ev) SP_CUDA(cudaEventRecord(ev[6], st));
    if (nS > 0) {
      switch (c.wire) {
        case SP_WIRE_FP32: k_lamb_update_push<SP_WIRE_FP32><<<nS, kLambThreads, 0, st>>>(ls, pp); break;
        case SP_WIRE_FP16: k_lamb_update_push<SP_WIRE_FP16><<<nS, kLambThreads, 0, st>>>(ls, pp); break;
        default: k_lamb_update_push<SP_WIRE_Q8><<<nS, kLambThreads, 0, st>>>(ls, pp); break;
      }
      SP_CUDA(cudaGetLastError());
    }
    if (c.world > 1) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
  } else if (ev) {
    SP_CUDA(cudaEventRecord(ev[5], st));
    SP_CUDA(cudaEventRecord(ev[6], st));
  }
  if (nR > 0) {  // join
    SP_CUDA(cudaEventRecord(r->seg_ev[7], r->aux));
    SP_CUDA(cudaStreamWaitEvent(st, r->seg_ev[7], 0));
  }
  if (ev) SP_CUDA(cudaEventRecord(ev[7], st));
  return SP_OK;
}

// Enqueues the whole round on `st`. ev != nullptr records phase events.
//
// Kernel pipeline per segment s = 0..K-1 (K = 1 with one rank):
//   K1 pack+scatter(s) -> barrier -> K2 reduce+push(s) -> barrier
// and, with K > 1, LAMB pass 1 of segment s on the aux stream as soon as its
// second barrier passed, overlapping the exchange of segment s+1; then
// LAMB pass 2 (all chunks) on `st` after joining the aux stream.
// Phase events (diagnostic): pack / barrier / reduce of segment 0, the
// remaining exchange, then LAMB.
int enqueue_round(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                  cudaStream_t st, cudaEvent_t* ev) {
  const sp_round_cfg& c = r->cfg;
  if (ev) SP_CUDA(cudaEventRecord(ev[0], st));
  if (r->fused_round) return enqueue_fused(r, grads, p, m, v, st, ev);
  const int K = r->segments;
  BarrierArgs ba{};
  if (c.world > 1) {
    for (int k = 0; k < c.world; ++k) ba.flags[k] = r->flags(k);
    ba.epoch = r->epoch;
    ba.err = r->d_err;
    ba.rank = c.rank;
    ba.world = c.world;
    const double to = c.barrier_timeout_s > 0 ? c.barrier_timeout_s : 20.0;
    ba.timeout_ns = (unsigned long long)(to * 1e9);
  }
  LambArgs la = make_lamb_args(r, p, m, v);
  // one rank, one contributing peer, fp32/fp16: the average is the peer's
  // rounded gradient, so the pack runs inside LAMB pass 1 (saves the wire
  // re-read and a launch); the wire buffer is still written
  const bool fuse_pack = c.world == 1 && r->L == 1 && c.wire != SP_WIRE_Q8 && r->fused_lamb &&
                         r->acc_buf < 0 && !r->shard && grads[0] && identity_avg(r) &&
                         (const void*)grads[0] != (const void*)r->wire(c.rank, 0) &&
                         std::getenv("SP_NO_FUSED_PACK") == nullptr;
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
  if (K > 1) {  // fork the aux stream off `st` (graph-capture safe)
    SP_CUDA(cudaEventRecord(r->seg_ev[8], st));
    SP_CUDA(cudaStreamWaitEvent(r->aux, r->seg_ev[8], 0));
  }
  for (int s = 0; s < K; ++s) {
    // K1: pack this segment of every owner's range, next rank's first
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
    const int64_t unit = c.wire == SP_WIRE_Q8 ? c.q8_block : (c.wire == SP_WIRE_FP16 ? 8 : 4);
    a.nr = 0;
    a.pref[0] = 0;
    for (int d = 1; d <= c.world; ++d) {
      const int k = (c.rank + d) % c.world;
      const int64_t lo = seg_cut(r, k, s), hi = seg_cut(r, k, s + 1);
      if (hi <= lo) continue;
      a.owner[a.nr] = k;
      a.lo[a.nr] = lo / unit;
      a.pref[a.nr + 1] = a.pref[a.nr] + (hi + unit - 1) / unit - lo / unit;
      ++a.nr;
    }
    a.n = r->n;
    a.npad = r->npad;
    a.qblock = c.q8_block;
    const int64_t units = a.pref[a.nr];
    if (any && units > 0 && !fuse_pack) {
      const int threads = c.wire == SP_WIRE_Q8 ? c.q8_block / 16 : 256;
      const int64_t per_cta = c.wire == SP_WIRE_Q8 ? 1 : 256;  // units per CTA per pass
      const int want = c.wire == SP_WIRE_Q8
                           ? (int)std::min<int64_t>(units, (int64_t)r->sm_count * 16)
                           : grid_for(units, 256, r->sm_count, r->xchg_per_sm);
      // split the CTAs over the ranges in proportion to their lengths (>= 1
      // each); the local range (HBM stores) weighted by pack_local_weight
      // against the remote ones (NVLink stores, the slower side)
      int total = 0;
      a.cta0[0] = 0;
      double wsum_r = 0.0;
      for (int j = 0; j < a.nr; ++j)
        wsum_r += (double)(a.pref[j + 1] - a.pref[j]) * (a.owner[j] == c.rank ? r->pack_local_weight : 1.0);
      for (int j = 0; j < a.nr; ++j) {
        const int64_t len = a.pref[j + 1] - a.pref[j];
        const double wj = (double)len * (a.owner[j] == c.rank ? r->pack_local_weight : 1.0);
        int nct = (int)std::max<int64_t>(1, (int64_t)((double)want * wj / wsum_r + 0.5));
        nct = (int)std::min<int64_t>(nct, (len + per_cta - 1) / per_cta);
        total += std::max(1, nct);
        a.cta0[j + 1] = total;
      }
      dim3 grid((unsigned)total, r->L);
      if (c.wire == SP_WIRE_Q8) k_pack_q8<<<grid, threads, 0, st>>>(a);
      else if (c.wire == SP_WIRE_FP16) k_pack_fp16<<<grid, threads, 0, st>>>(a);
      else k_pack_fp32<<<grid, threads, 0, st>>>(a);
      SP_CUDA(cudaGetLastError());
    }
    if (ev && s == 0) SP_CUDA(cudaEventRecord(ev[1], st));
    if (c.world > 1) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    if (ev && s == 0) SP_CUDA(cudaEventRecord(ev[2], st));
    // K2: average this rank's segment, push it to every rank (self last)
    {
      ReduceArgs ra{};
      double wsum = 0.0;
      for (double w : r->weights) wsum += w;
      int np = 0;
      for (int g = 0; g < r->G; ++g) {
        if (r->weights[g] == 0.0) continue;
        ra.src[np] = r->wire(c.rank, g);  // this rank's inbox: local HBM only
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
      ra.lo = seg_cut(r, c.rank, s);
      ra.hi = seg_cut(r, c.rank, s + 1);
      ra.npad = r->npad;
      ra.qblock = c.q8_block;
      // [lo, hi) pushed to `nd` ranks (self last); sharded tensors keep their
      // average local (only their owner steps them)
      auto reduce = [&](int64_t lo, int64_t hi, int nd) -> int {
        if (hi <= lo) return SP_OK;
        ReduceArgs q = ra;
        q.lo = lo;
        q.hi = hi;
        q.ndst = nd;
        for (int k = 0; k < nd; ++k) q.dst[k] = r->avg((c.rank + 1 + k + (c.world - nd)) % c.world);
        if (c.wire == SP_WIRE_Q8) {
          const int64_t nb = (hi + c.q8_block - 1) / c.q8_block - lo / c.q8_block;
          const int grid = (int)std::min<int64_t>(nb, (int64_t)r->sm_count * 16);
          k_reduce_q8<<<grid, c.q8_block / 16, 0, st>>>(q);
        } else if (c.wire == SP_WIRE_FP16) {
          k_reduce_fp16<<<grid_for((hi - lo + 7) / 8, 256, r->sm_count, r->xchg_per_sm), 256, 0, st>>>(q);
        } else {
          k_reduce_fp32<<<grid_for((hi - lo + 3) / 4, 256, r->sm_count, r->xchg_per_sm), 256, 0, st>>>(q);
        }
        SP_CUDA(cudaGetLastError());
        return SP_OK;
      };
      if (ra.hi > ra.lo && !identity_avg(r)) {
        if (r->shard) {
          // the replicated prefix (up to the cut, rounded up to a wire unit)
          // goes to every rank
          const int64_t cu = std::min<int64_t>(r->n, round_up(r->shard_cut, r->align));
          if (int rc = reduce(ra.lo, std::min(ra.hi, cu), c.world)) return rc;
          if (int rc = reduce(std::max(ra.lo, cu), ra.hi, 1)) return rc;
        } else if (int rc = reduce(ra.lo, ra.hi, c.world)) {
          return rc;
        }
      }
    }
    if (ev && s == 0) SP_CUDA(cudaEventRecord(ev[3], st));
    // the averages must have landed everywhere before LAMB reads them; with
    // every tensor sharded they stay with their owner, so no barrier (the
    // next round's pack cannot start before the round's last barrier, which
    // every rank enters after its reduce)
    const bool all_local = r->shard && r->nchunks_rep == 0 && K == 1;
    if (c.world > 1 && !all_local) {
      k_barrier<<<1, 32, 0, st>>>(ba);
      SP_CUDA(cudaGetLastError());
    }
    if (K > 1) {  // LAMB pass 1 of this segment overlaps the next exchange
      SP_CUDA(cudaEventRecord(r->seg_ev[s], st));
      SP_CUDA(cudaStreamWaitEvent(r->aux, r->seg_ev[s], 0));
      const int rc = launch_lamb(r, la, r->p1_off[(size_t)s], r->p1_off[(size_t)s + 1] - r->p1_off[(size_t)s],
                                 false, r->aux);
      if (rc) return rc;
    }
  }
  if (ev) SP_CUDA(cudaEventRecord(ev[4], st));
  if (r->shard) return enqueue_shard_lamb(r, la, ba, st, ev);
  // K3/K4 LAMB on this rank's replica
  if (r->fused_lamb) {
    if (K > 1) {
      SP_CUDA(cudaEventRecord(r->seg_ev[8], r->aux));
      SP_CUDA(cudaStreamWaitEvent(st, r->seg_ev[8], 0));  // join
      if (ev) {
        SP_CUDA(cudaEventRecord(ev[5], st));
        SP_CUDA(cudaEventRecord(ev[6], st));
      }
      const int rc = launch_lamb(r, la, r->p2_off, r->nchunks, true, st);
      if (rc) return rc;
    } else {
      const int rc = launch_lamb(r, la, 0, r->nitems, true, st);
      if (rc) return rc;
      if (ev) {
        SP_CUDA(cudaEventRecord(ev[5], st));
        SP_CUDA(cudaEventRecord(ev[6], st));
      }
    }
  } else {
    const int nc = r->nchunks;
    switch (c.wire) {
      case SP_WIRE_FP32: k_lamb_moments<SP_WIRE_FP32><<<nc, kLambThreads, 0, st>>>(la); break;
      case SP_WIRE_FP16: k_lamb_moments<SP_WIRE_FP16><<<nc, kLambThreads, 0, st>>>(la); break;
      default: k_lamb_moments<SP_WIRE_Q8><<<nc, kLambThreads, 0, st>>>(la); break;
    }
    SP_CUDA(cudaGetLastError());
    if (ev) SP_CUDA(cudaEventRecord(ev[5], st));
    k_lamb_trust<<<c.num_tensors, 256, 0, st>>>(r->d_partial, r->d_tchunks, r->d_hp, r->d_trust,
                                                r->d_step_scale);
    SP_CUDA(cudaGetLastError());
    if (ev) SP_CUDA(cudaEventRecord(ev[6], st));
    switch (c.wire) {
      case SP_WIRE_FP32: k_lamb_update<SP_WIRE_FP32><<<nc, kLambThreads, 0, st>>>(la); break;
      case SP_WIRE_FP16: k_lamb_update<SP_WIRE_FP16><<<nc, kLambThreads, 0, st>>>(la); break;
      default: k_lamb_update<SP_WIRE_Q8><<<nc, kLambThreads, 0, st>>>(la); break;
    }
    SP_CUDA(cudaGetLastError());
  }
  if (ev) SP_CUDA(cudaEventRecord(ev[7], st));
  return SP_OK;
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
  if (*r->h_err) return fail(SP_ERR_PEER, "a cross-rank barrier timed out in an earlier round");
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
    if (erc) return erc;
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

}  // namespace

extern "C" {

const char* sp_version(void) { return "sp_round 0.1.0 (sm_100a)"; }
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
  if (cfg->wire == SP_WIRE_Q8) r->buf_bytes += round_up(r->npad / cfg->q8_block * 4, 256);
  r->buf_bytes = round_up(r->buf_bytes, 256);
  {
    const char* legacy = std::getenv("SP_ROUND_LEGACY");
    // one-kernel round (sp_round_fused.cuh) is opt-in: measured equal at N=4
    // and slower at N=1 than the kernel pipeline
    const char* fused = std::getenv("SP_ROUND_FUSED");
    r->fused_round = fused && fused[0] == '1' && !(legacy && legacy[0] == '1') &&
                     (cfg->wire != SP_WIRE_Q8 || cfg->q8_block == 4096);
    r->cell = (int)std::max<int64_t>(kLambChunk, cfg->wire == SP_WIRE_Q8 ? cfg->q8_block : 0);
    if (const char* ce = std::getenv("SP_ROUND_CELL")) {  // tuning knob: multiple of the cell
      const int want = std::atoi(ce);
      if (want > r->cell && want % r->cell == 0) r->cell = want;
    }
    r->ncells = (int)((cfg->n + r->cell - 1) / r->cell);
    r->ctr_bytes = 2 * round_up((int64_t)r->ncells * 4, 256);
  }
  r->flags_bytes = 256 + round_up((int64_t)2 * r->G * 8, 256);
  r->shared_bytes = r->flags_bytes + r->ctr_bytes + (size_t)(r->G + 1) * r->buf_bytes;
  if (cfg->shard_lamb) {  // [params fp32 npad][norm table world x T double2]
    r->shard = true;
    r->fused_round = false;
    r->param_off = r->shared_bytes;
    r->norms_off = r->param_off + round_up(r->npad * 4, 256);
    r->nflags_off = r->norms_off + round_up((int64_t)cfg->world * cfg->num_tensors * 16, 256);
    r->shared_bytes = r->nflags_off + round_up((int64_t)cfg->world * cfg->num_tensors * 8, 256);
  }
  int dev_sms = 0;
  cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  if (dev_sms > 0) r->sm_count = dev_sms;

  auto cleanup = [&](int code) {
    sp_round_destroy(r);
    return code;
  };
  cudaError_t e = cudaMalloc(&r->shared, r->shared_bytes);
  if (e != cudaSuccess) return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc shared: ") + cudaGetErrorString(e)));
  if ((e = cudaMemset(r->shared, 0, r->shared_bytes)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  r->base[cfg->rank] = r->shared;

  const char* chunk_env = std::getenv("SP_LAMB_CHUNK");
  r->lamb_chunk = chunk_env ? std::max(64, std::atoi(chunk_env)) : kLambChunk;
  {
    const char* seg_env = std::getenv("SP_SEGMENTS");
    const char* unf = std::getenv("SP_LAMB_UNFUSED");
    const bool unfused = unf && unf[0] == '1';
    if (const char* g = std::getenv("SP_SEG_LAMB_GRID")) r->seg_lamb_grid = std::max(1, std::atoi(g));
    if (const char* x = std::getenv("SP_XCHG_PER_SM")) r->xchg_per_sm = std::max(1, std::atoi(x));
    if (const char* x = std::getenv("SP_PACK_LOCAL_WEIGHT")) r->pack_local_weight = std::max(0.01, std::atof(x));
    r->segments = (cfg->world > 1 && !unfused && !r->fused_round && !r->shard)
                      ? std::max(1, std::min(8, seg_env ? std::atoi(seg_env) : 1))
                      : 1;
  }
  {
    int64_t base = 0;
    for (int64_t sz : r->tsizes) base += sz / r->lamb_chunk + 2;
    r->nchunks_cap = (int)(base + (int64_t)cfg->world * (r->segments + 1) + 8);
  }
  const size_t ntens = r->tsizes.size();
  if ((e = cudaMalloc(&r->d_chunks, (size_t)r->nchunks_cap * sizeof(Chunk))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_tchunks, ntens * sizeof(int2))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_partial, (size_t)r->nchunks_cap * sizeof(float2))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_trust, ntens * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_step_scale, ntens * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_hp, 4 * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&r->d_items, 2 * (size_t)r->nchunks_cap * sizeof(int))) != cudaSuccess ||
      (e = cudaMalloc(&r->epoch, sizeof(unsigned long long))) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
  if (r->shard) {
    if (const char* e2 = std::getenv("SP_SHARD_FUSED")) r->shard_fused = e2[0] == '1';
    if (const char* e2 = std::getenv("SP_SHARD_LAG")) r->shard_lag = std::max(0, std::atoi(e2));
    int per_sm = 0;
    cudaError_t oe;
    switch (cfg->wire) {
      case SP_WIRE_FP32: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shard_lamb_fused<SP_WIRE_FP32>, kLambThreads, 0); break;
      case SP_WIRE_FP16: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shard_lamb_fused<SP_WIRE_FP16>, kLambThreads, 0); break;
      default: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_shard_lamb_fused<SP_WIRE_Q8>, kLambThreads, 0); break;
    }
    if (oe != cudaSuccess || per_sm < 1) return cleanup(fail(SP_ERR_CUDA, "occupancy query failed for the sharded LAMB kernel"));
    r->shard_grid = per_sm * r->sm_count;
    if ((e = cudaMalloc(&r->d_sitems, 2 * (size_t)r->nchunks_cap * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&r->d_sepoch, sizeof(unsigned long long))) != cudaSuccess)
      return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
    cudaMemset(r->d_sepoch, 0, sizeof(unsigned long long));
  }
  if (int rc2 = build_lamb_tables(r, false)) return cleanup(rc2);
  {
    const char* env = std::getenv("SP_LAMB_UNFUSED");
    r->fused_lamb = !(env && env[0] == '1');
    const char* hint_env = std::getenv("SP_LAMB_L2HINTS");
    r->l2_hints = hint_env ? std::atoi(hint_env) : 1;
    int per_sm = 0;
    cudaError_t oe;
    switch (cfg->wire) {
      case SP_WIRE_FP32: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lamb_fused<SP_WIRE_FP32>, kLambThreads, 0); break;
      case SP_WIRE_FP16: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lamb_fused<SP_WIRE_FP16>, kLambThreads, 0); break;
      default: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lamb_fused<SP_WIRE_Q8>, kLambThreads, 0); break;
    }
    if (oe != cudaSuccess || per_sm < 1) return cleanup(fail(SP_ERR_CUDA, "occupancy query failed for the fused LAMB kernel"));
    // persistent grid (the work queue is safe either way: items are taken in
    // order and only wait on earlier ones)
    r->lamb_grid = std::max(1, per_sm * r->sm_count);
    if (const char* lg = std::getenv("SP_LAMB_GRID")) r->lamb_grid = std::max(1, std::min(r->lamb_grid, std::atoi(lg)));
    // hybrid sharded LAMB: the replicated part leaves one CTA slot per SM to
    // the sharded chain running beside it
    r->hybrid_grid = std::max(1, r->lamb_grid - r->sm_count);
    if (const char* hg = std::getenv("SP_HYBRID_LAMB_GRID")) r->hybrid_grid = std::max(1, std::atoi(hg));
    if ((e = cudaMalloc(&r->d_qstate, (2 + ntens) * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&r->d_ready, ntens * sizeof(unsigned int))) != cudaSuccess)
      return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
    cudaMemset(r->d_qstate, 0, (2 + ntens) * sizeof(int));
    cudaMemset(r->d_ready, 0, ntens * sizeof(unsigned int));
  }
  {
    int per_sm = 0;
    cudaError_t oe;
    switch (cfg->wire) {
      case SP_WIRE_FP32: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_round_fused<SP_WIRE_FP32>, kLambThreads, 0); break;
      case SP_WIRE_FP16: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_round_fused<SP_WIRE_FP16>, kLambThreads, 0); break;
      default: oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_round_fused<SP_WIRE_Q8>, kLambThreads, 0); break;
    }
    if (oe != cudaSuccess || per_sm < 1) return cleanup(fail(SP_ERR_CUDA, "occupancy query failed for the fused round kernel"));
    r->round_grid = per_sm * r->sm_count;
    const size_t cap = 2 * (size_t)r->ncells + SP_MAX_RANKS + 2 * (size_t)r->nchunks_cap + 16;
    if ((e = cudaMalloc(&r->d_ritems, cap * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMalloc(&r->d_rq, 2 * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&r->d_repoch, sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMalloc(&r->d_cell_owners, (size_t)r->ncells)) != cudaSuccess)
      return cleanup(fail(SP_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e)));
    cudaMemset(r->d_rq, 0, 2 * sizeof(int));
    cudaMemset(r->d_repoch, 0, sizeof(unsigned));
  }
  cudaMemset(r->epoch, 0, sizeof(unsigned long long));
  cudaMemset(r->d_trust, 0, ntens * sizeof(float));
  if ((e = cudaHostAlloc(&r->h_err, sizeof(int), cudaHostAllocMapped)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  *r->h_err = 0;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&r->d_err), r->h_err, 0);
  if ((e = cudaStreamCreateWithFlags(&r->own, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&r->aux, cudaStreamNonBlocking)) != cudaSuccess)
    return cleanup(fail(SP_ERR_CUDA, cudaGetErrorString(e)));
  for (auto& ev : r->seg_ev)
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
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
  cudaFree(r->d_tchunks);
  cudaFree(r->d_partial);
  cudaFree(r->d_trust);
  cudaFree(r->d_step_scale);
  cudaFree(r->d_hp);
  cudaFree(r->d_items);
  cudaFree(r->d_sitems);
  cudaFree(r->d_sepoch);
  cudaFree(r->d_qstate);
  for (int b = 0; b < 2; ++b)
    for (int l = 0; l < SP_MAX_LOCAL; ++l) cudaFree(r->acc[b][l]);
  cudaFree(r->d_stage);
  for (int b = 0; b < 2; ++b) {
    for (int l = 0; l < SP_MAX_LOCAL; ++l) cudaFree(r->stg[b][l]);
    if (r->stg_ready[b]) cudaEventDestroy(r->stg_ready[b]);
    if (r->stg_free[b]) cudaEventDestroy(r->stg_free[b]);
  }
  if (r->h2d) cudaStreamDestroy(r->h2d);
  cudaFree(r->d_ritems);
  cudaFree(r->d_rq);
  cudaFree(r->d_repoch);
  cudaFree(r->d_cell_owners);
  cudaFree(r->d_ready);
  cudaFree(r->epoch);
  if (r->h_err) cudaFreeHost(r->h_err);
  for (auto& ev : r->ev)
    if (ev) cudaEventDestroy(ev);
  if (r->own) cudaStreamDestroy(r->own);
  if (r->aux) cudaStreamDestroy(r->aux);
  for (auto& ev : r->seg_ev)
    if (ev) cudaEventDestroy(ev);
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
  r->offsets.assign(offsets, offsets + G + 1);
  r->weights.assign(weights, weights + G);
  SP_CUDA(cudaSetDevice(r->cfg.device));
  SP_CUDA(cudaDeviceSynchronize());  // the previous round may still read the tables
  if (int rc = build_lamb_tables(r, true)) return rc;
  if (r->fused_round) {
    const int rc = build_round_items(r);
    if (rc) return rc;
  }
  r->assigned = true;
  drop_graphs(r);
  return SP_OK;
}

int sp_round_run(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                 int step, void* stream) {
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
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
  if (!r || !host_grads) return fail(SP_ERR_ARG, "null argument");
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
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
  r->stg_used[b] = true;
  r->stg_next = b ^ 1;
  return SP_OK;
}

int sp_round_run_phased(sp_round* r, const float* const* grads, float* p, float* m, float* v,
                        int step, void* stream, sp_phase_times* t) {
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
  rc = upload_hparams(r, step, st);
  if (rc) return rc;
  rc = enqueue_round(r, grads, p, m, v, st, r->ev);
  if (rc) return rc;
  SP_CUDA(cudaStreamSynchronize(st));
  if (*r->h_err) return fail(SP_ERR_PEER, "cross-rank barrier timed out");
  if (t) {
    float* f[7] = {&t->pack_ms, &t->barrier_a_ms, &t->reduce_ms, &t->barrier_b_ms,
                   &t->moments_ms, &t->trust_ms, &t->update_ms};
    for (int k = 0; k < 7; ++k) SP_CUDA(cudaEventElapsedTime(f[k], r->ev[k], r->ev[k + 1]));
    SP_CUDA(cudaEventElapsedTime(&t->total_ms, r->ev[0], r->ev[7]));
  }
  return SP_OK;
}

void* sp_round_wire_ptr(sp_round* r, int local_peer) {
  if (!r || local_peer < 0 || local_peer >= r->L) return nullptr;
  return r->wire(r->cfg.rank, r->cfg.rank * r->L + local_peer);
}

float* sp_round_param_ptr(sp_round* r) { return r && r->shard ? r->param(r->cfg.rank) : nullptr; }

int64_t sp_round_shard_cut(const sp_round* r) { return r && r->shard ? r->shard_cut : -1; }

void* sp_round_avg_ptr(sp_round* r) { return r ? const_cast<char*>(avg_buffer(r)) : nullptr; }

const float* sp_round_trust_ptr(sp_round* r) { return r ? r->d_trust : nullptr; }

int sp_round_copy_trust(sp_round* r, float* dst, void* stream) {
  if (!r || !dst) return fail(SP_ERR_ARG, "null argument");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
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

namespace {

int ensure_accumulators(sp_round* r, int buf) {
  if (r->acc[buf][0]) return SP_OK;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  for (int l = 0; l < r->L; ++l) SP_CUDA(cudaMalloc(&r->acc[buf][l], (size_t)r->n * sizeof(float)));
  if (!r->d_stage) SP_CUDA(cudaMalloc(&r->d_stage, 2 * (size_t)r->L * sizeof(double)));
  return SP_OK;
}

}  // namespace

int sp_round_accumulate(sp_round* r, int buf, int local_peer, const float* grad, double samples,
                        void* stream) {
  if (!r || !grad) return fail(SP_ERR_ARG, "null argument");
  if (buf < 0 || buf > 1) return fail(SP_ERR_ARG, "buf must be 0 or 1");
  if (local_peer < 0 || local_peer >= r->L) return fail(SP_ERR_ARG, "local_peer out of range");
  if (!(samples >= 0.0) || !std::isfinite(samples)) return fail(SP_ERR_ARG, "samples must be >= 0");
  if ((reinterpret_cast<uintptr_t>(grad) & 15) != 0) return fail(SP_ERR_SHAPE, "grad must be 16-byte aligned");
  if (int rc = ensure_accumulators(r, buf)) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
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
  if (r->fused_round) return fail(SP_ERR_STATE, "accumulated rounds use the kernel pipeline");
  if (int rc = ensure_accumulators(r, buf)) return rc;
  const float* grads[SP_MAX_LOCAL];
  for (int l = 0; l < r->L; ++l) grads[l] = r->acc[buf][l];
  int rc = check_run_args(r, grads, p, m, v);
  if (rc) return rc;
  SP_CUDA(cudaSetDevice(r->cfg.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : r->own;
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
