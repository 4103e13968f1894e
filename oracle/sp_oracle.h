/*
 * sp_oracle.h — CPU oracle for the averaging round. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library, and only as the checker or
 * the timed CPU reference. The product path (libsp_round.so) never calls it.
 *
 * What it restates, and how it is pinned:
 *  - weighted mean (sp_oracle_weighted_average_f64): groups::run_plan
 *    semantics, /root/reference/proj/src/groups.cpp:117-161 — per-peer
 *    sum = w_i * v_i (:120), merged in peer order (:133-144), divided by the
 *    summed weight at the end (:158). Pinned to SPEC.md's known answers
 *    ([0,0,0,4] -> 1.0, mean of [1..9] = 5.0)
 *    in tests/test_oracle.py. run_plan itself has no tests in the reference
 *    (proj/tests/cpp/test_groups.cpp is an empty stub) and the reference
 *    cannot be compiled here (Eigen/KLU absent), so beyond those known
 *    answers this part is "parity unpinned".
 *  - part offsets (sp_oracle_part_offsets): not in the reference; fractions
 *    are StrategyAssignment::fractions (proj/src/strategy.cpp:473-485).
 *  - fp16 / blockwise-8-bit wire, fp32 fmaf reduction, LAMB: absent from the
 *    reference ("Non-goals: Gradient compression"; SPEC.md:519
 *    "LAMB/LARS optimizers ... out of scope"). Defined here; parity unpinned
 *    against the reference by construction — the GPU must match THIS
 *    definition bit for bit (codes, averaged parts, m, v) or within the
 *    tolerance stated in the tests (p).
 */
#ifndef SP_ORACLE_H_
#define SP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SPO_FP32 = 0, SPO_FP16 = 1, SPO_Q8 = 2 };

uint64_t sp_oracle_splitmix64(uint64_t x);

/* u = splitmix64(seed ^ (peer << 40) ^ i) >> 40 (24 bits);
 * x = ((float)u - 2^23) * 2^-23 * scale; x *= mult when i % every == 0. */
void sp_oracle_fill_synthetic(float* out, int64_t n, uint64_t seed, int peer,
                              float scale, int64_t every, float mult);

/* offsets[0] = 0, offsets[G] = n, offsets[k] = clamp(align *
 * llround(n * sum_{i<k} f_i / align), offsets[k-1], n): contiguous parts in
 * peer order, proportional to the LP fractions, aligned to `align`. */
void sp_oracle_part_offsets(int64_t n, int G, const double* fractions,
                            int64_t align, int64_t* offsets);

uint16_t sp_oracle_f2h(float x);  /* IEEE binary16, round to nearest even */
float sp_oracle_h2f(uint16_t h);

/* Wire pack: fp16 RNE, or blockwise int8: amax = max|x| over the block,
 * inv = 127/amax, q = clamp(rint(x*inv), -127, 127), scale = amax/127;
 * amax == 0 gives codes 0 and scale 0. */
void sp_oracle_pack_fp16(const float* x, uint16_t* out, int64_t n);
void sp_oracle_pack_q8(const float* x, int8_t* codes, float* scales,
                       int64_t n, int block);

/* groups::run_plan for m = n without failures: out = (sum_g w_g v_g) / sum w
 * in fp64, peer order. values[g] points at peer g's n doubles. */
void sp_oracle_weighted_average_f64(const double* const* values,
                                    const double* weights, int G, int64_t n,
                                    double* out);

/* The executor's fp32 reduction of elements [lo, hi): wn_g = (float)(w_g /
 * sum w) (fp64 division); over the peers with w_g != 0 in peer order,
 * acc = wn_first * x_first, then acc = fmaf(wn_g, x_g, acc), x_g the dequantized wire value (q8: (float)q * scale); result
 * re-encoded in the wire format into out_wire (and out_scales for q8, whose
 * blocks are aligned: lo % block == 0). wire[g]/scales[g] are peer g's full
 * buffers. q8 with a single contributor forwards its codes and scales
 * unchanged: the exact average of one peer is that peer's values, and
 * requantizing them reproduces the codes but can move the scale by one ulp
 * (fl(fl(127 s)/127) != s for 0.8% of mantissas). */
void sp_oracle_reduce(int wire, const void* const* wires,
                      const float* const* scales, const double* weights,
                      int G, int64_t lo, int64_t hi, int block,
                      void* out_wire, float* out_scales);

typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int bias_correction;
} sp_oracle_lamb_hp;

/* LAMB on the averaged vector (wire format), per tensor trust ratio
 * ||p||/||u|| in fp64 (1 if either is 0). trust_in (nullable) overrides the
 * computed trust ratios so the update can be checked bit-exactly against a
 * device-computed trust; trust_out (nullable) receives the (float) ratios
 * that were computed. */
void sp_oracle_lamb(int wire, const void* avg, const float* avg_scales,
                    int block, float* p, float* m, float* v, int64_t n,
                    const int64_t* tensor_sizes, int num_tensors,
                    const sp_oracle_lamb_hp* hp, int step,
                    const float* trust_in, float* trust_out);

/* Whole round on the CPU for G peers (the CPU baseline): pack every peer's
 * gradient, reduce all parts, LAMB on the averaged vector. Scratch buffers are
 * allocated internally. threads <= 0 uses every OpenMP thread. Returns 0. */
int sp_oracle_round(int wire, int block, int G, int64_t n,
                    const float* const* grads, const double* weights,
                    float* p, float* m, float* v,
                    const int64_t* tensor_sizes, int num_tensors,
                    const sp_oracle_lamb_hp* hp, int step, int threads,
                    float* trust_out);

int sp_oracle_max_threads(void);
/* OpenMP threads of the calls that follow (<= 0: unchanged). */
void sp_oracle_set_threads(int threads);
/* fp64 -> fp32 -> wire format (fp32 / fp16 RNE / blockwise 8-bit). */
void sp_oracle_wire_from_f64(int wire, const double* x, void* out, float* scales, int64_t n,
                             int block);

#ifdef __cplusplus
}
#endif
#endif /* SP_ORACLE_H_ */
