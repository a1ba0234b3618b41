/*
 * gravac_oracle.h -- CPU restatement of the GraVAC hot path (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It is never linked into, or called by, the product package.
 *
 * Every function restates one reference function; the file:line citations
 * point into /root/reference/pkg/src/gravac/.  Pinning: the restatement is
 * checked against golden vectors produced by the unmodified reference
 * (tests/golden/make_golden.py -> tests/golden/<family>.npz, tests/test_oracle_golden.py)
 * for Top-k, Redsync, multi-level compression, error feedback, gains,
 * decompress/aggregate and the small-n DGC degenerate case.
 *
 * PARITY UNPINNED (by design, see DESIGN.md section "Random positions"): the exact
 * positions chosen by Random-k and by DGC's threshold sample.  The reference
 * draws them with numpy Generator.choice over Philox4x64 (gradcore.py:144-149,
 * compressors.py:118,180), an inherently sequential algorithm; this build
 * replaces it with the counter-based sampler below (Philox4x32-10 hash per
 * position, k smallest hashes, ties to the lower index).  The oracle restates
 * that sampler bit-exactly; agreement with the reference is property-level
 * (support size, determinism, values at indices, DGC >= 95% overlap).
 */
#ifndef GRAVAC_ORACLE_H
#define GRAVAC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_ERR_NAN = -1,   /* a NaN magnitude makes the selection order undefined (reference F8) */
    ORC_ERR_ARG = -2,
    ORC_ERR_NOMEM = -3,
};

enum { ORC_TOPK = 0, ORC_DGC = 1, ORC_REDSYNC = 2, ORC_RANDOMK = 3 };

/* Philox4x32-10 (Salmon et al., SC'11): out = philox(ctr, key). */
/* OpenMP threads of the O(n) passes (default 1: the checker's exact
 * sequential semantics).  bench.py's CPU legs set the host's cores. */
void orc_set_threads(int t);
int orc_get_threads(void);

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Counter-based position hash of the DGC sample:
 * ctr = (lo(i), hi(i), lo(stream), hi(stream)), key = (lo(seed), hi(seed)) -> out[0].
 * Random-k's key of position i: out[i & 3] at ctr = (lo(i >> 2), hi(i >> 2), lo(stream),
 * hi(stream)) -- one Philox evaluation per four consecutive positions. */
uint32_t orc_randomk_hash(uint64_t seed, uint64_t stream, uint64_t i);
void orc_dgc_sample_positions(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                              uint32_t *out);
uint32_t orc_position_hash(uint64_t seed, uint64_t stream, uint64_t i);

/* feedback.py:32-36: out = fl32(g + r). */
void orc_ef_add(const float *g, const float *r, float *out, uint64_t n);

/* gradcore.py:61-70: sum of squares in float64 (sequential order). */
double orc_sq_norm(const float *x, uint64_t n);

/* numpy's float64 pairwise summation (the add.reduce inner loop numpy 2.3
 * uses for a contiguous float64 array); used for Redsync's mean (compressors.py:188). */
double orc_pairwise_sum_f64(const double *a, uint64_t n);

/* compressors.py:86-99 + :185: the k largest |x| (ties to the lower index),
 * written as k ascending positions.  k >= n returns 0..n-1. */
int orc_topk_indices(const float *x, uint64_t n, uint64_t k, uint32_t *out_idx);

/* Generic form of the above over 32-bit keys: the k largest keys, ties to the
 * lower index, ascending positions. */
int orc_select_keys(const uint32_t *keys, uint64_t n, uint64_t k, uint32_t *out_idx);

/* compressors.py:164-190: one compressor selection over values[0..n) keeping k.
 * Writes k ascending positions and the values to send.  pos_base is added to
 * the position counter of the hash (layerwise segments use their global start).
 * seed/stream come from SeededRng(seed, stream) (gradcore.py:129-158). */
int orc_select(int kind, const float *values, uint64_t n, uint64_t k,
               uint64_t seed, uint64_t stream, uint64_t pos_base,
               double dgc_sample_fraction,
               uint32_t *out_idx, float *out_vals);

/* compressors.py:256-271: fp64 worker-ascending sum of N sparse parts, /N, ->fp32.
 * idx/vals hold the parts back to back; part p has counts[p] entries. */
int orc_aggregate(const uint32_t *idx, const float *vals, const uint64_t *counts,
                  int nparts, uint64_t n, float *out);

/* compressors.py:274-285: fp64 mean of N dense parts (row-major [nparts][n]). */
int orc_aggregate_dense(const float *parts, int nparts, uint64_t n, float *out);

/* feedback.py:39-51: r = g_ef; r[idx] -= vals. */
void orc_update_residual(const float *g_ef, const uint32_t *idx, const float *vals,
                         uint64_t k, uint64_t n, float *r_out);

#ifdef __cplusplus
}
#endif
#endif
