/*
 * sp_round.h — C-ABI of the B200 averaging-round executor (libsp_round.so).
 *
 * This is the drop-in boundary for the one data-parallel hot path of DeDLOC
 * (arXiv 2106.10207): the butterfly averaging round over a flattened gradient
 * vector split into LP-assigned, non-uniform parts, followed by a LAMB step.
 *
 * The reference (`swarmplan`, /root/reference/proj) has no C-ABI and no GPU
 * code; the round exists there only as
 *   - the part assignment:   strategy::solve_strategy -> StrategyAssignment::
 *                            fractions   (proj/src/strategy.cpp:473-498)
 *   - the averaging:         groups::run_plan, weighted mean sum(w_i v_i)/sum(w_i)
 *                            in peer order (proj/src/groups.cpp:102-163,
 *                            declared proj/include/swarmplan/groups.hpp:35-37)
 *   - the round-time model:  strategy::allreduce_round_seconds /
 *                            adaptive_round_seconds (proj/src/strategy.cpp:502-532)
 * Each entry point below cites the reference interface it replaces or feeds.
 * Plain pointers and sizes only; no torch / Eigen / C++ types cross this line.
 *
 * Execution model: one process ("rank") per GPU. A rank hosts
 * `peers_per_rank` consecutive peers (virtual peers when > 1, e.g. all 8
 * peers of a fleet on one GPU for parity tests). Peer g owns the element
 * range [offsets[g], offsets[g+1]). Ranks exchange one CUDA IPC handle each
 * (sp_round_export / sp_round_connect). The pack kernel scatters every
 * peer's packed part straight into the owning rank's inbox over NVLink
 * (reduce-scatter as posted writes); the owner averages its range from local
 * HBM and pushes the result into every rank's buffer (all-gather).
 *
 * Status codes: every function returns SP_OK (0) or an SP_ERR_* code; the
 * message of the last failure on the calling thread is sp_last_error().
 *
 * Streams: every `void* stream` argument is a cudaStream_t and NULL is the
 * CUDA legacy default stream, as everywhere in CUDA. All work of a call is
 * ordered on that stream: it starts after the work the caller enqueued
 * before it (e.g. the backward pass writing the gradients) and the next
 * work on the stream (e.g. the forward reading p) starts after the round.
 * Host-input rounds copy on an internal stream that is joined to `stream`
 * with events.
 */
#ifndef SP_ROUND_H_
#define SP_ROUND_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_OK 0
#define SP_ERR_ARG 1      /* invalid argument (maps to std::invalid_argument) */
#define SP_ERR_CUDA 2     /* CUDA runtime failure (maps to std::runtime_error) */
#define SP_ERR_STATE 3    /* call out of order, e.g. run before set_assignment */
#define SP_ERR_PEER 4     /* cross-rank barrier timed out (a peer is gone) */
#define SP_ERR_SHAPE 5    /* buffer misaligned / sizes disagree */

#define SP_MAX_PEERS 64   /* total peers G = peers_per_rank * world */
#define SP_MAX_RANKS 8    /* GPUs of one NVSwitch box */
#define SP_MAX_LOCAL 16   /* peers hosted by one rank */

/* Wire format of gradient parts and averaged parts. The reference only scales
 * its timing model by bits_per_param (proj/include/swarmplan/model.hpp:39-42);
 * these formats are defined by this framework (SPEC.md:192 lists compression
 * as a non-goal of the reference). */
typedef enum {
  SP_WIRE_FP32 = 0, /* 4 B/param, zero-copy when the grad is the wire buffer */
  SP_WIRE_FP16 = 1, /* 2 B/param, round-to-nearest-even                      */
  SP_WIRE_Q8 = 2    /* 1 B/param + fp32 absmax scale per q8_block elements   */
} sp_wire;

typedef struct sp_round sp_round;

typedef struct {
  int device;          /* CUDA device ordinal this rank drives               */
  int rank;            /* 0..world-1                                          */
  int world;           /* number of ranks (GPUs), <= SP_MAX_RANKS             */
  int peers_per_rank;  /* L, peers hosted per rank; G = L*world <= 64         */
  int64_t n;           /* flattened vector length (param_count)              */
  int wire;            /* sp_wire                                             */
  int q8_block;        /* elements per 8-bit block: 512..16384, power of 2   */
  int num_tensors;     /* LAMB tensor table: trust ratio is per tensor       */
  const int64_t* tensor_sizes; /* num_tensors sizes summing to n (copied)    */
  float lr, beta1, beta2, eps, weight_decay;
  int bias_correction; /* 1: Adam-style bias correction of m and v           */
  double barrier_timeout_s; /* cross-rank spin limit (0 -> 20 s)             */
  int shard_lamb;      /* 1: sharded LAMB (ZeRO-1 style): each
                        * rank steps only the range it owns, per-tensor norm
                        * sums are exchanged over NVLink inside the LAMB
                        * kernel, and the updated parameters (not the averaged
                        * gradient) are pushed to every rank. p must be
                        * sp_round_param_ptr(); m and v stay full-length but
                        * only the owned range is kept. Pays off on uniform
                        * splits; with a dominant owner the replicated mode is
                        * faster (roofline.choose_shard_lamb picks per plan). */
} sp_round_cfg;

/* Per-phase device times of the last sp_round_run_phased call (ms). */
typedef struct {
  float pack_ms;      /* K1: fp32 -> wire + scatter to the owners (0 when fused
                         into LAMB: one rank, one peer, fp32/fp16 wire)      */
  float barrier_a_ms; /* cross-rank barrier after the scatter (0 if N=1)     */
  float reduce_ms;    /* K2: weighted average of the owned range (+ push of the
                         averages to every rank with replicated LAMB)        */
  float barrier_b_ms; /* barrier after the push (replicated LAMB, N>1)       */
  float lamb_ms;      /* K3: k_lamb, both LAMB passes (sharded: + norm
                         exchange and parameter push)                        */
  float barrier_c_ms; /* closing barrier (sharded LAMB, N>1)                 */
  float total_ms;
} sp_phase_times;

/* Creates the executor for one rank: allocates the IPC-shareable wire/avg
 * buffers (padded, zero-filled) and the LAMB chunk table. */
int sp_round_create(const sp_round_cfg* cfg, sp_round** out);
int sp_round_destroy(sp_round* r);

/* Multi-rank wiring (world > 1): every rank exports one opaque handle blob of
 * sp_round_handle_bytes() bytes; the caller all-gathers them in rank order
 * (e.g. torch.distributed) and passes the world*bytes array to connect. */
size_t sp_round_handle_bytes(void);
int sp_round_export(sp_round* r, void* out_handle);
int sp_round_connect(sp_round* r, const void* all_handles);

/* Replaces the reference's fractions -> weighted-mean hand-off:
 * offsets[G+1] come from the host partitioner over
 * StrategyAssignment::fractions (proj/src/strategy.cpp:473-485); weights[G]
 * are per-peer accumulated sample counts, the `weights` argument of
 * groups::run_plan (proj/include/swarmplan/groups.hpp:35-37, applied at
 * proj/src/groups.cpp:119). Offsets must be non-decreasing, start at 0, end
 * at n, and be multiples of sp_round_align() except the last. sum(weights)
 * must be > 0 (the reference divides by it unchecked, groups.cpp:158). */
int sp_round_align(const sp_round* r);
int sp_round_set_assignment(sp_round* r, const int64_t* offsets,
                            const double* weights);

/* One averaging round + LAMB step, stream-ordered on `stream`
 * (cudaStream_t; NULL = legacy default stream). grads[l] is the
 * accumulated gradient of local peer l (device fp32[n]; NULL for an
 * aggregation-only peer whose weight is 0). p/m/v are this rank's replica
 * (device fp32[n]), updated in place. `step` is the 1-based optimizer step
 * (bias correction). The first call with a given pointer set captures the
 * round into a CUDA graph; later calls replay it. Replaces the m = n,
 * no-failure case of groups::run_plan (proj/src/groups.cpp:102-163) plus the
 * optimizer step the reference leaves out of scope. */
int sp_round_run(sp_round* r, const float* const* grads, float* p, float* m,
                 float* v, int step, void* stream);

/* The same round fed from HOST gradients (the drop-in call for a peer whose
 * accumulated gradients live in host memory). host_grads[l] should be
 * pinned (cudaHostAlloc / torch pin_memory) for the copy to be asynchronous.
 * The copy goes to one of two device staging buffers on an internal copy
 * stream, so step k's host->device copy overlaps round k-1 on `stream`;
 * the round itself is sp_round_run on the staged buffer (graph replay; the
 * two staging buffers keep two cached graphs). The host buffers may be
 * reused once `stream` has passed this round. */
int sp_round_run_host(sp_round* r, const float* const* host_grads, float* p,
                      float* m, float* v, int step, void* stream);

/* sp_round_run_host that also returns the step's result: the updated
 * parameters p (n floats) are copied into host_p_out (pinned, or the copy is
 * synchronous) on `stream` after the round (the device->host half of
 * groups::run_plan's by-value result, proj/src/groups.cpp:154-161). PCIe is
 * full duplex, so this copy overlaps the next step's gradient upload.
 * host_p_out == NULL is sp_round_run_host. */
int sp_round_run_host_params(sp_round* r, const float* const* host_grads, float* p,
                             float* m, float* v, int step, float* host_p_out,
                             void* stream);

/* Same round without graph capture, with CUDA events between phases;
 * synchronizes the stream and fills *t. Diagnostic only. */
int sp_round_run_phased(sp_round* r, const float* const* grads, float* p,
                        float* m, float* v, int step, void* stream,
                        sp_phase_times* t);

/* Buffers owned by the executor (device pointers). wire(l) is this rank's
 * inbox slot of local peer l (holding the part of l's packed gradient this
 * rank owns; with world == 1 the whole vector). With world == 1 and
 * SP_WIRE_FP32, grads[l] == wire(l) skips the pack (zero-copy). avg is this
 * rank's all-gathered averaged vector in the wire format; q8 scales follow
 * the codes at avg + padded_n. */
void* sp_round_wire_ptr(sp_round* r, int local_peer);

/* shard_lamb: this rank's flat fp32[n] parameter vector, inside the
 * IPC-shared allocation so that owners can store their updated ranges into
 * every rank's copy (NULL without shard_lamb). */
float* sp_round_param_ptr(sp_round* r);

/* Host-only description of this rank's exchange plan (no device is touched;
 * used to test the pointer tables at any world size, e.g. 8 ranks on a
 * machine without GPUs). */
typedef struct {
  int pack_ranges;                          /* owner ranges K1 scatters to    */
  int pack_owner[SP_MAX_RANKS];             /* in visiting order: next rank first */
  int64_t pack_first_unit[SP_MAX_RANKS];    /* first wire unit of each range  */
  int64_t pack_units[SP_MAX_RANKS];         /* units of each range            */
  int pack_cta_begin[SP_MAX_RANKS + 1];     /* CTAs [begin[j], begin[j+1]) on range j */
  int pack_ctas;                            /* K1 grid (x)                    */
  int unit_elems;                           /* elements per wire unit         */
  int64_t own_lo, own_hi;                   /* range this rank averages (K2)  */
  int push_order[SP_MAX_RANKS];             /* rank order of pushes to all ranks (self last) */
  int avg_push_ranks;                       /* ranks K2 writes the average to */
} sp_plan_desc;
int sp_round_describe(const sp_round_cfg* cfg, const int64_t* offsets, int sm_count,
                      sp_plan_desc* out);

/* Number of chunks of the LAMB plan: the elements this rank steps
 * (replicated: all n; sharded: its owned range) cut at tensor edges and
 * every multiple of the chunk tile; *tile receives the tile (elements) when
 * not null. Valid after sp_round_set_assignment; -1 for a null handle. */
int sp_round_lamb_chunks(const sp_round* r, int* tile);
void* sp_round_avg_ptr(sp_round* r);
int64_t sp_round_padded_n(const sp_round* r);
/* Per-tensor trust ratios of the last step (device float[num_tensors]). */
const float* sp_round_trust_ptr(sp_round* r);

/* Synchronous device->host copy of an executor buffer, for checks and for
 * reading a step's result back: which = SP_BUF_WIRE (local peer's wire
 * buffer), SP_BUF_AVG (averaged vector) or SP_BUF_TRUST (float[num_tensors]).
 * Waits for all work on the executor's device. */
/* Asynchronous copy of the last step's per-tensor trust ratios into dst
 * (pinned host or device memory, float[num_tensors]) on `stream`: the
 * device->host read of a round's result. */
int sp_round_copy_trust(sp_round* r, float* dst, void* stream);

#define SP_BUF_WIRE 0
#define SP_BUF_AVG 1
#define SP_BUF_TRUST 2
int sp_round_read(sp_round* r, int which, int local_peer, size_t offset_bytes,
                  void* host_dst, size_t bytes);

/* Device-side accumulation to the target batch (the round's first step; the
 * reference only models it: samples = rate * time, /root/reference/proj/src/
 * netsim.cpp:338-339, and weights the mean by them, groups.cpp:119). Two
 * accumulator buffers per local peer let a round consume one while the next
 * step's micro-batches land in the other (DPU).
 *  - sp_round_accumulate: acc[buf][l] = grad (first call of the round) or
 *    acc + grad (fp32), and adds `samples` to the peer's count.
 *  - sp_round_accumulator_ptr: the device fp32[n] accumulator, for writing
 *    gradients in place (then report them with sp_round_add_samples).
 *  - sp_round_run_accumulated: the round over acc[buf] weighted by the sample
 *    counts, which every rank publishes to every rank over NVLink; the
 *    `weights` of sp_round_set_assignment are not used. Resets the counts of
 *    `buf` (its next accumulate overwrites). The accumulator may be refilled
 *    only after this call is ordered before the refill (same stream or event).
 */
int sp_round_accumulate(sp_round* r, int buf, int local_peer, const float* grad,
                        double samples, void* stream);
float* sp_round_accumulator_ptr(sp_round* r, int buf, int local_peer);
int sp_round_add_samples(sp_round* r, int buf, int local_peer, double samples);
double sp_round_samples(const sp_round* r, int buf, int local_peer);
int sp_round_run_accumulated(sp_round* r, int buf, float* p, float* m, float* v,
                             int step, void* stream);

/* fp64 vector primitives for group all-reduce plans on device-resident rows
 * (groups::run_plan_device): dst = src * w, dst =
 * ((0 + s_0) + s_1) + ... (k <= 64), dst = src / d — the operations of
 * groups::run_plan (/root/reference/proj/src/groups.cpp:120,141-143,158).
 * Stream-ordered on `stream` (cudaStream_t, NULL = legacy default). */
int sp_vec_scale(double* dst, const double* src, double w, int64_t n, void* stream);
int sp_vec_sum(double* dst, const double* const* srcs, int k, int64_t n, void* stream);
int sp_vec_div(double* dst, const double* src, double d, int64_t n, void* stream);

/* Synthetic accumulated gradient, bit-identical to the CPU oracle's
 * generator (oracle/sp_oracle.c: sp_oracle_fill_synthetic):
 *   u = splitmix64(seed ^ (peer << 40) ^ i) >> 40;
 *   x = ((float)u - 2^23) * 2^-23 * scale;  x *= outlier_mult if i % outlier_every == 0
 * The idea follows the reference's counter-keyed generators
 * (proj/src/sgd.cpp:170-172, proj/src/lp.cpp:33-39). */
int sp_fill_synthetic(float* dev, int64_t n, uint64_t seed, int peer,
                      float scale, int64_t outlier_every, float outlier_mult,
                      void* stream);

/* Library version and last error of the calling thread. */
const char* sp_version(void);
const char* sp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SP_ROUND_H_ */
