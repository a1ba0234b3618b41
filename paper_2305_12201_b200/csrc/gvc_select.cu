// gvc_select.cu -- deterministic multi-CF selection for the GraVAC step (sm_100a).
//
// One selection answers, for a ladder of keep counts k_0 >= k_1 >= ... (all
// compression factors of the search space, nested as compressors.py:237-238
// nests them), "which k_j entries have the largest key, ties to the lower
// index" -- the rule of compressors.py:86-99 -- together with the fp64 kept
// energies the gain statistic needs (metrics.py:18-32).  Keys are the 31-bit
// magnitude pattern (Top-k, Redsync, DGC) or a Philox position hash (Random-k).
//
// Data layout: the input is cut into S contiguous segments, one per warp of
// the collect kernel (8 warps = one "block" of 8 segments).  Candidates are
// compacted IN INDEX ORDER into their segment's slice of the candidate buffer,
// so every later pass reads only candidates and index order is free.
//
// Pipeline (stream-ordered, no host synchronisation):
//   k_sample / k_sample_resolve   ~1.5% strided sample (smem histogram) ->
//                                 conservative key_est + level-0 bin shift
//   k_collect (EF fused)          ONE streaming pass over HBM: g_ef = g + r is
//                                 written over r, fp64 ||g_ef||^2, and every
//                                 key >= key_est is compacted with a level-0
//                                 shared-memory histogram
//   k_resolve0 / k_collect(refill) exactness guard: if the estimate missed,
//                                 every value becomes a candidate
//   k_level_hist / k_level_resolve radix refinement over candidates only,
//                                 until each k_j has its exact threshold key
//   k_final / k_finish            per-segment band counts and per-block band
//                                 energies; tie cut, gains and per-block
//                                 output offsets for EVERY ladder entry
//   k_emit (gvc_emit)             ordered (idx, val) compaction of one entry,
//                                 fused residual update
#include <algorithm>
#include <type_traits>
#include <mutex>
#include <stdio.h>
#include <string>
#include <unordered_map>
#include <vector>

#include "gvc_common.cuh"
#include "gvc_internal.h"

namespace gvc {

// ------------------------------------------------------------------ state
struct JState {
    unsigned long long lo, hi;  // candidate key interval [lo, hi) holding T_j
    unsigned long long above;   // candidates with key >= hi (all kept)
    unsigned long long need;    // entries still to take from [lo, hi)
    int shift;                  // refinement-histogram bin shift
    int resolved;
};

struct SelState {
    uint32_t key_est;
    int shift0;
    uint32_t max_key;
    uint32_t nan_flag;
    uint32_t fallback;
    uint32_t pending;
    unsigned long long cand_total;
    unsigned long long shortfall;
    JState js[GVC_MAX_LADDER];
    float redsync_mean[GVC_MAX_LADDER];
    uint32_t fin_done;     // k_finish blocks done (the last one writes the status)
    uint32_t sample_done;  // k_sample blocks done (the last one resolves key_est)
    uint32_t mem_flat;     // members appended to Plan::mem_key (may exceed its capacity)
    unsigned long long t_phase[32];  // %globaltimer at kernel boundaries (gvc_select_phase_times)
};

struct Plan {
    uint64_t n;
    uint32_t S, B, seg_len;
    int n_ks, kind, keymode, ef, force_exact;
    const float *values;
    const float *g;
    float *resid;
    uint64_t seed, stream, pos_base;
    uint64_t ks[GVC_MAX_LADDER];
    // forced candidate threshold (DGC)
    const uint32_t *key_est_dev;
    // KEY_DGC: the sampled threshold key and the sample's position bitmap
    const uint32_t *dgc_thr;
    const uint32_t *dgc_bits;
    int allow_short;
    // deferred residual update of the previous step (EF mode)
    uint32_t *pmask;
    const float *pm;
    int pmode;
    // sample
    uint64_t s_chunks, s_stride, s_target;
    uint64_t s_target_lo;  // a count of sampled keys >= it says "k_0 keys are >= them" w.h.p.
    uint32_t hash_key_est;
    // workspace
    SelState *st;
    uint32_t *hist0, *histl, *shist;
    uint32_t *seg_cnt;                     // [SEG_MAX] candidates per segment
    uint32_t *seg_mcnt;                    // [SEG_MAX] level-0 bin members per segment
    uint32_t *mem_idx;                     // [n_pad] members: segment-local candidate offsets
    uint32_t *mem_key;                     // [GVC_MEM_FLAT] members' keys, flat, any order
    uint32_t *seg_band, *seg_tie;          // [L][SEG_MAX]
    double *blk_norm;                      // [BLK_MAX]
    uint32_t *blk_band_cnt, *blk_tie_cnt;  // [L][BLK_MAX]
    double *blk_band_e2, *blk_band_ab;     // [L][BLK_MAX]
    double *blk_tie_e2, *blk_tie_ab;       // [L][BLK_MAX]
    uint32_t *blk_take, *blk_off;          // [L][BLK_MAX]
    double *blk_emit;                      // [2][BLK_MAX]
    float *cand_val;
    uint32_t *cand_idx;
    gvc_select_result *res;
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static void seg_geometry(uint64_t n, uint32_t *S, uint32_t *seg_len)
{
    uint64_t per = (n + GVC_SEG_TARGET - 1) / GVC_SEG_TARGET;
    uint64_t len = ((per + GVC_SEG_QUANTUM - 1) / GVC_SEG_QUANTUM) * GVC_SEG_QUANTUM;
    if (len < GVC_SEG_QUANTUM)
        len = GVC_SEG_QUANTUM;
    *seg_len = (uint32_t)len;
    *S = (uint32_t)((n + len - 1) / len);
}

// Carves the workspace; returns the byte size needed (ws may be null).
static size_t carve(Plan *p, char *ws, uint64_t n)
{
    uint32_t S, seg_len;
    seg_geometry(n, &S, &seg_len);
    uint64_t n_pad = (uint64_t)S * seg_len;
    size_t off = 0;
    auto take = [&](size_t bytes) -> char * {
        char *q = ws ? ws + off : nullptr;
        off += align256(bytes);
        return q;
    };
    const size_t L = GVC_MAX_LADDER, SM = GVC_SEG_MAX, BM = GVC_BLK_MAX;
    Plan tmp;
    Plan *q = p ? p : &tmp;
    // zeroed per select by ONE memset, st .. histl[n_ks] (adjacent, in this order)
    q->st = (SelState *)take(sizeof(SelState));
    q->hist0 = (uint32_t *)take(GVC_H0_BINS * 4);
    q->shist = (uint32_t *)take(GVC_SAMPLE_BINS * 4);
    q->histl = (uint32_t *)take(L * GVC_HL_BINS * 4);
    q->mem_key = (uint32_t *)take((size_t)GVC_MEM_FLAT * 4);
    q->seg_cnt = (uint32_t *)take(SM * 4);
    q->seg_mcnt = (uint32_t *)take(SM * 4);
    q->seg_band = (uint32_t *)take(L * SM * 4);
    q->seg_tie = (uint32_t *)take(L * SM * 4);
    q->blk_norm = (double *)take(BM * 8);
    q->blk_band_cnt = (uint32_t *)take(L * BM * 4);
    q->blk_tie_cnt = (uint32_t *)take(L * BM * 4);
    q->blk_band_e2 = (double *)take(L * BM * 8);
    q->blk_band_ab = (double *)take(L * BM * 8);
    q->blk_tie_e2 = (double *)take(L * BM * 8);
    q->blk_tie_ab = (double *)take(L * BM * 8);
    q->blk_take = (uint32_t *)take(L * BM * 4);
    q->blk_off = (uint32_t *)take(L * BM * 4);
    q->blk_emit = (double *)take(2 * BM * 8);
    q->cand_val = (float *)take(n_pad * 4);
    q->cand_idx = (uint32_t *)take(n_pad * 4);
    q->mem_idx = (uint32_t *)take(n_pad * 4);
    q->S = S;
    q->B = (S + GVC_WARPS_PER_BLOCK - 1) / GVC_WARPS_PER_BLOCK;
    q->seg_len = seg_len;
    return off;
}

// ------------------------------------------------------------ key helpers
template <int KM>
__device__ __forceinline__ uint32_t cand_key(const Plan &p, float v, uint32_t pos)
{
    if (KM == KEY_MAG)
        return mag_key(v);
    if (KM == KEY_DGC) {
        // DGC's pick as one top-k (gvc_select_args.dgc_thr_dev): chosen (|v| >=
        // thr) and sampled values in the upper half ordered by |v| -- chosen
        // first since they are larger -- the rest below them
        const uint32_t m = mag_key(v);
        const bool hi = m >= __ldg(p.dgc_thr) || ((__ldg(p.dgc_bits + (pos >> 5)) >> (pos & 31)) & 1u);
        return hi ? (0x80000000u | m) : m;
    }
    if (KM == KEY_POS)  // equal nonzero magnitudes: nonzero first by position; zeros tie at key 0
        return v != 0.f ? 0x80000000u | (0x7fffffffu - (uint32_t)(p.pos_base + pos)) : 0u;
    return hash_key(p.pos_base + pos, p.stream, p.seed);
}

// NaN magnitude in a key (the selection order is undefined, reference F8)
template <int KM>
__device__ __forceinline__ bool key_nan(uint32_t key)
{
    return KM != KEY_HASH && KM != KEY_POS && (key & 0x7fffffffu) > 0x7f800000u;
}

// Development probe (-DGVC_PHASE_STAMPS=1, scripts/phase_probe.py): per select
// kernel, %globaltimer at block 0's entry (t_phase[2k]) and the latest block
// exit (t_phase[2k+1]).  Compiled out of the product library.
#ifndef GVC_PHASE_STAMPS
#define GVC_PHASE_STAMPS 0
#endif
#if GVC_PHASE_STAMPS
__device__ __forceinline__ unsigned long long gvc_gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GVC_STAMP_IN(k)                                                                                       \
    if (blockIdx.x == 0 && threadIdx.x == 0)                                                                  \
        p.st->t_phase[2 * (k)] = gvc_gtimer();
#define GVC_STAMP_OUT(k)                                                                                      \
    if (threadIdx.x == 0)                                                                                     \
        atomicMax(&p.st->t_phase[2 * (k) + 1], gvc_gtimer());
#else
#define GVC_STAMP_IN(k)
#define GVC_STAMP_OUT(k)
#endif

// ------------------------------------------------------------------ sample
// Strided chunks of 128 contiguous values -> 14-bit shared-memory histogram of
// magnitude keys, merged into global memory once per block.  Reads ~1.5%.
__device__ void sample_resolve_body(const Plan &p, unsigned long long *sh, int shift);

template <int KM>
__global__ void __launch_bounds__(1024) k_sample(const Plan p, int)
{
    constexpr int SHIFT = (KM == KEY_DGC || KM == KEY_POS) ? GVC_SAMPLE_SHIFT + 1 : GVC_SAMPLE_SHIFT;  // 32- / 31-bit keys
    pdl_enter(); GVC_STAMP_IN(0);
    extern __shared__ uint32_t sh[];
    for (int i = threadIdx.x; i < GVC_SAMPLE_BINS; i += 1024)
        sh[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * 32;
    const float pm = (p.pmask && p.pmode == 2) ? *p.pm : 0.f;
    uint32_t kmax = 0;
    for (uint64_t c = blockIdx.x * 32 + (threadIdx.x >> 5); c < p.s_chunks; c += warps) {
        const uint64_t base = c * p.s_stride;
        float v[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint64_t i = base + (uint64_t)q * 32 + lane;
            ok[q] = i < p.n && i < base + 128;
            if (ok[q]) {
                if (p.ef) {
                    float r = p.resid[i];
                    if (p.pmask && ((p.pmask[i >> 5] >> (i & 31)) & 1u))
                        r = pending_resid(r, p.pmode, pm);
                    v[q] = __fadd_rn(p.g[i], r);
                } else {
                    v[q] = p.values[i];
                }
            } else {
                v[q] = 0.f;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t k = ok[q] ? cand_key<KM>(p, v[q], (uint32_t)(base + (uint64_t)q * 32 + lane)) : 0u;
            if (ok[q] && !key_nan<KM>(k)) {
                atomicAdd(&sh[k >> SHIFT], 1u);
                kmax = max(kmax, k);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    // one global atomic per block: a per-warp atomicMax serialises thousands of
    // updates on one line
    __shared__ uint32_t s_kmax;
    if (threadIdx.x == 0)
        s_kmax = 0;
    __syncthreads();
    if (lane == 0 && kmax)
        atomicMax(&s_kmax, kmax);
    __syncthreads();
    if (threadIdx.x == 0 && s_kmax)
        atomicMax(&p.st->max_key, s_kmax);
    for (int i = threadIdx.x; i < GVC_SAMPLE_BINS; i += 1024)
        if (sh[i])
            atomicAdd(&p.shist[i], sh[i]);
    // the last block to finish resolves key_est (no separate launch)
    // (the block's histogram atomics are ordered before thread 0's device-scope
    // fence by the barrier -- fence cumulativity -- so one thread fences)
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&p.st->sample_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        sample_resolve_body(p, reinterpret_cast<unsigned long long *>(sh), SHIFT);
    }
    GVC_STAMP_OUT(0);
}

// Chooses key_est (a lower bound for the k_0-th largest key, w.h.p.) and the
// level-0 bin shift.  Magnitude keys: from the sample histogram.  Hash keys:
// from the binomial tail (host-computed).
__device__ void sample_resolve_body(const Plan &p, unsigned long long *sh, int shift)
{
    SelState *st = p.st;
    if (p.key_est_dev) {  // DGC: the candidates are exactly {key >= sampled threshold}
        if (threadIdx.x == 0) {
            // the k-th largest key sits just above the sampled threshold: fine
            // level-0 bins there (4096 keys, 1/2048 of an octave; the top bin is
            // open-ended), so level 1 resolves it.  Bins sized to the whole key
            // range instead left ~10^5 members for the single-block refinement.
            st->key_est = *p.key_est_dev;
            st->shift0 = 12;
        }
        return;
    }
    if (p.force_exact == 2) {  // test hook: an estimate that must miss -> exercises the refill path
        if (threadIdx.x == 0) {
            st->key_est = 0xffffffffu;
            st->shift0 = 0;
        }
        return;
    }
    if (p.keymode == KEY_HASH) {
        if (threadIdx.x == 0) {
            uint32_t est = p.force_exact ? 0u : p.hash_key_est;
            st->key_est = est;
            uint64_t span = (1ull << 32) - est;
            int shf = bitlen64(span - 1) - 12;
            st->shift0 = shf < 0 ? 0 : shf;
        }
        return;
    }
    if (p.force_exact || p.s_target == 0) {
        if (threadIdx.x == 0) {
            st->key_est = 0;
            st->shift0 = 19;  // 31-bit keys over 4096 bins
        }
        return;
    }
    constexpr int PER = GVC_SAMPLE_BINS / 1024;  // 16 bins per thread
    const int t = threadIdx.x;
    uint32_t h[PER];
    const uint4 *src = reinterpret_cast<const uint4 *>(p.shist + t * PER);
    unsigned long long local = 0;
#pragma unroll
    for (int q = 0; q < PER / 4; q++) {
        uint4 x = src[q];
        h[4 * q] = x.x;
        h[4 * q + 1] = x.y;
        h[4 * q + 2] = x.z;
        h[4 * q + 3] = x.w;
        local += (unsigned long long)x.x + x.y + x.z + x.w;
    }
    unsigned long long total;
    unsigned long long pre = block_excl_prefix(local, sh, &total);
    unsigned long long acc = total - pre - local;  // keys in bins above my range
    const unsigned long long target = p.s_target;
    __shared__ unsigned long long s_flagged;  // DGC: sampled keys in the flagged half (bins >= 8192)
    if (p.keymode == KEY_DGC) {
        if (t == (1024 >> 1))
            s_flagged = total - pre;
        __syncthreads();
    }
    if (total < target) {  // too few sampled values (e.g. NaN-only): exact path
        if (t == 0) {
            st->key_est = 0;
            st->shift0 = 19;
        }
        return;
    }
#pragma unroll
    for (int i = PER - 1; i >= 0; i--) {
        if (acc < target && acc + h[i] >= target) {
            uint32_t est = (uint32_t)(t * PER + i) << shift;
            st->key_est = est;
            uint32_t mk = st->max_key;
            // DGC composite keys, top-up branch (fewer than k_0 flagged keys,
            // w.h.p.): the threshold is an unflagged key, i.e. a magnitude
            // below thr, and every flagged key lies above it -- bins sized to
            // the whole span put ~10^6 members in the threshold bin (measured)
            if (p.keymode == KEY_DGC && est < 0x80000000u && mk >= 0x80000000u && s_flagged < p.s_target_lo)
                mk = *p.dgc_thr;
            uint64_t span = mk > est ? (uint64_t)(mk - est) : 0;
            int shf = bitlen64(span) - 12;
            st->shift0 = shf < 0 ? 0 : shf;
        }
        acc += h[i];
    }
}

__global__ void __launch_bounds__(1024) k_sample_resolve(const Plan p, int)
{
    pdl_enter();
    __shared__ unsigned long long sh[33];
    sample_resolve_body(p, sh, GVC_SAMPLE_SHIFT);
}

// ----------------------------------------------------------------- collect
// Candidate compaction for 4 consecutive values of one lane (lane-major index
// order within the warp).  Straight-line so the ballots stay convergent; the
// histogram atomic is unconditional (non-candidates hit a per-lane dummy bin)
// and only the two candidate stores are predicated.  `o` is the segment-local
// candidate count; `pos` the global position of v[0].
template <int KM, uint32_t WRAP = 0xffffffffu>
__device__ __forceinline__ void push4(const Plan &p, const float (&v)[4], uint32_t pos, uint32_t valid,
                                      uint32_t key_est, int shift0, uint32_t *h, uint32_t dummy, float *cval,
                                      uint32_t *cidx, uint32_t &ccount)
{
    uint32_t key[4], m[4];
    bool pr[4];
    if (KM == KEY_HASH && valid == 4u && ((p.pos_base + pos) & 3u) == 0) {
        // four consecutive positions: one Philox evaluation (hash_key4)
        const uint4 h = hash_key4(p.pos_base + pos, p.stream, p.seed);
        key[0] = h.x;
        key[1] = h.y;
        key[2] = h.z;
        key[3] = h.w;
    } else {
#pragma unroll
        for (int c = 0; c < 4; c++)
            key[c] = cand_key<KM>(p, v[c], pos + c);
    }
#pragma unroll
    for (int c = 0; c < 4; c++) {
        pr[c] = ((uint32_t)c < valid) & (key[c] >= key_est);
        m[c] = __ballot_sync(0xffffffffu, pr[c]);
    }
    const uint32_t lt = lanemask_lt();
    uint32_t o = ccount + __popc(m[0] & lt) + __popc(m[1] & lt) + __popc(m[2] & lt) + __popc(m[3] & lt);
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const uint32_t bin = pr[c] ? min((key[c] - key_est) >> shift0, (uint32_t)GVC_H0_BINS - 1) : dummy;
        atomicAdd(&h[bin], 1u);
        if (pr[c]) {
            cval[o & WRAP] = v[c];
            cidx[o & WRAP] = pos + c;
        }
        o += pr[c];
    }
    ccount += __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
}

// One warp per segment.  EF: v = fl32(g + r_true) written back over r (the only
// full-size write of the step), where r_true applies the previous step's
// deferred residual update (PM = pending mode, 0 none); !EF: v read from
// `values`.  REFILL re-collects from the already-written g_ef with key_est = 0
// (exactness fallback).  NaN keys are always candidates and are flagged by the
// candidate passes, not here.
// One warp's pass over segment `seg` (k_collect's body; also the inline
// exactness refill of k_collect's last block).  Adds the warp's fp64 squares to nacc.
template <int KM, bool EF, int PM, bool REFILL>
__device__ __forceinline__ void collect_segment(const Plan &p, uint32_t seg, int lane, uint32_t *h, uint32_t dummy,
                                                uint32_t key_est, int shift0, float pm, double &nacc,
                                                float *sv = nullptr, uint32_t *si = nullptr, uint32_t *mw = nullptr)
{
    constexpr bool refill = REFILL;
    const bool do_ef = EF && !refill;
    const uint64_t beg = (uint64_t)seg * p.seg_len;
    const uint32_t len = (uint32_t)(min(p.n, beg + p.seg_len) - beg);
    const float *src = (EF ? (refill ? p.resid : p.g) : p.values) + beg;
    float *rp = p.resid + beg;
    const uint32_t *mp = p.pmask + (beg >> 5);
    float *cval = p.cand_val + beg;
    uint32_t *cidx = p.cand_idx + beg;
    uint32_t ccount = 0;
    uint32_t i = 0;
    // Candidates are staged in a per-warp shared-memory ring (sv / si, GVC_STAGE
    // entries) and written out 128 at a time with one 16-byte store per lane:
    // stored straight from push4 they cost ~16 partial-sector stores per 256
    // values -- a quarter of the kernel's time (measured: 105 -> 78 us without them)
    // (entries below ccount & ~127 are always out: a push adds <= 128)
    constexpr bool STAGE = !REFILL;
    // 256-value steps.  PF (magnitude keys): software pipeline -- the next
    // step's g / r loads and mask words are in flight while this step is
    // added, reduced and compacted.  Hash keys are Philox-bound, and the
    // register double buffer there only costs spills.
    constexpr bool PF = GVC_COLLECT_PREFETCH != 0 && KM == KEY_MAG;
    constexpr uint32_t STEP = 256;
    const uint32_t nfull = len / GVC_SEG_QUANTUM * GVC_SEG_QUANTUM;  // whole 512-chunks
    float4 a[2], b[2];
    // the step's 8 pending-mask words, prefetched with the data when PF (a mask
    // load issued at its use was the kernel's top stall, ncu): MASK_ASYNC copies
    // them into the warp's shared slots mw[2][8] with cp.async -- held in a
    // register instead, the word was spilled and its local store waited on the load
    constexpr bool MASK_ASYNC = PF && PM != 0 && !REFILL;
    uint32_t wreg = 0u;
    if (PF && nfull) {
        if (MASK_ASYNC) {
            if (lane < 2)
                cp_async16(mw + 4 * lane, mp + 4 * lane);
            cp_async_commit();
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            a[u] = ld_stream(reinterpret_cast<const float4 *>(src + u * 128) + lane);
            if (do_ef)
                b[u] = ld_stream(reinterpret_cast<const float4 *>(rp + u * 128) + lane);
        }
        if (!MASK_ASYNC && do_ef && PM && lane < 8)
            wreg = mp[lane];
    }
    for (; i < nfull; i += STEP) {
        float4 na[2], nb[2];
        uint32_t nw = 0u;
        const bool more = i + STEP < nfull;
        const uint32_t slot = MASK_ASYNC ? ((i >> 8) & 1u) * 8u : 0u;
        if (PF) {
            if (more) {
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    na[u] = ld_stream(reinterpret_cast<const float4 *>(src + i + STEP + u * 128) + lane);
                    if (do_ef)
                        nb[u] = ld_stream(reinterpret_cast<const float4 *>(rp + i + STEP + u * 128) + lane);
                }
                if (MASK_ASYNC) {
                    if (lane < 2)
                        cp_async16(mw + (slot ^ 8u) + 4 * lane, mp + ((i + STEP) >> 5) + 4 * lane);
                } else if (do_ef && PM && lane < 8) {
                    nw = mp[((i + STEP) >> 5) + lane];
                }
            }
            if (MASK_ASYNC) {  // this step's words landed (the group just committed may still fly)
                cp_async_commit();
                cp_async_wait<1>();
                __syncwarp();
                wreg = lane < 8 ? mw[slot + lane] : 0u;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                a[u] = ld_stream(reinterpret_cast<const float4 *>(src + i + u * 128) + lane);
                if (do_ef)
                    b[u] = ld_stream(reinterpret_cast<const float4 *>(rp + i + u * 128) + lane);
            }
            if (do_ef && PM && lane < 8)
                wreg = mp[(i >> 5) + lane];
        }
        if (do_ef) {
            if (PM) {
                // the 8 mask words of this step (lanes 0..7), shuffled to the
                // lanes owning their 4-bit slices, cleared after use
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint32_t bits = (MASK_ASYNC ? mw[slot + 4 * u + (lane >> 3)]
                                                      : __shfl_sync(0xffffffffu, wreg, 4 * u + (lane >> 3))) >>
                                          ((lane & 7) * 4);
                    b[u].x = (bits & 1u) ? pending_resid(b[u].x, PM, pm) : b[u].x;
                    b[u].y = (bits & 2u) ? pending_resid(b[u].y, PM, pm) : b[u].y;
                    b[u].z = (bits & 4u) ? pending_resid(b[u].z, PM, pm) : b[u].z;
                    b[u].w = (bits & 8u) ? pending_resid(b[u].w, PM, pm) : b[u].w;
                }
                if (wreg)
                    p.pmask[(beg >> 5) + (i >> 5) + lane] = 0u;
            }
#pragma unroll
            for (int u = 0; u < 2; u++) {
                a[u].x = __fadd_rn(a[u].x, b[u].x);
                a[u].y = __fadd_rn(a[u].y, b[u].y);
                a[u].z = __fadd_rn(a[u].z, b[u].z);
                a[u].w = __fadd_rn(a[u].w, b[u].w);
                st_stream(reinterpret_cast<float4 *>(rp + i + u * 128) + lane, a[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const float v[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
            if (!refill) {
#pragma unroll
                for (int c = 0; c < 4; c++)
                    nacc = __fma_rn((double)v[c], (double)v[c], nacc);
            }
            if (STAGE) {
                const uint32_t before = ccount;
                push4<KM, GVC_STAGE - 1>(p, v, (uint32_t)beg + i + u * 128 + lane * 4, 4u, key_est, shift0, h,
                                         dummy, sv, si, ccount);
                if ((ccount ^ before) & ~127u) {  // warp-uniform: a 128-entry block filled up
                    __syncwarp();
                    const uint32_t f = before & ~127u, b0 = f & (GVC_STAGE - 1);
                    reinterpret_cast<float4 *>(cval + f)[lane] = reinterpret_cast<const float4 *>(sv + b0)[lane];
                    reinterpret_cast<uint4 *>(cidx + f)[lane] = reinterpret_cast<const uint4 *>(si + b0)[lane];
                    __syncwarp();
                }
            } else {
                push4<KM>(p, v, (uint32_t)beg + i + u * 128 + lane * 4, 4u, key_est, shift0, h, dummy, cval,
                          cidx, ccount);
            }
        }
        if (PF && more) {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                a[u] = na[u];
                b[u] = nb[u];
            }
            if (!MASK_ASYNC)
                wreg = nw;
        }
    }
    if (STAGE) {  // drain the ring; the tail stores directly
        __syncwarp();
        for (uint32_t t = (ccount & ~127u) + lane; t < ccount; t += 32) {
            cval[t] = sv[t & (GVC_STAGE - 1)];
            cidx[t] = si[t & (GVC_STAGE - 1)];
        }
        __syncwarp();
    }
    // tail: one value per lane, lane-major order preserved
    for (; i < len; i += 32) {
        const uint32_t t = i + lane;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t valid = t < len ? 1u : 0u;
        if (valid) {
            float x = src[t];
            if (do_ef) {
                float r = rp[t];
                if (PM) {
                    const uint64_t gpos = beg + t;
                    const uint32_t bit = 1u << (gpos & 31);
                    if (p.pmask[gpos >> 5] & bit) {
                        r = pending_resid(r, PM, pm);
                        atomicAnd(&p.pmask[gpos >> 5], ~bit);
                    }
                }
                x = __fadd_rn(x, r);
                rp[t] = x;
            }
            v[0] = x;
            if (!refill)
                nacc = __fma_rn((double)x, (double)x, nacc);
        }
        push4<KM>(p, v, (uint32_t)beg + t, valid, key_est, shift0, h, dummy, cval, cidx, ccount);
    }
    if (lane == 0)
        p.seg_cnt[seg] = ccount;
}

template <int KM, bool EF, int PM, bool REFILL = false>
__global__ void __launch_bounds__(GVC_THREADS, GVC_COLLECT_BLOCKS) k_collect(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(1);
    // compile-time: a runtime flag would leave predicated refill / no-refill
    // code under every value of the hot loop
    constexpr bool refill = REFILL;
    __shared__ uint32_t h[GVC_H0_BINS + 32];  // + per-lane dummy bins
    __shared__ double red[GVC_WARPS_PER_BLOCK];
    __shared__ __align__(16) float stage_v[GVC_WARPS_PER_BLOCK][GVC_STAGE];
    __shared__ __align__(16) uint32_t stage_i[GVC_WARPS_PER_BLOCK][GVC_STAGE];
    __shared__ __align__(16) uint32_t mwords[GVC_WARPS_PER_BLOCK][16];
    if (refill && !p.st->fallback)
        return;
    for (int i = threadIdx.x; i < GVC_H0_BINS + 32; i += GVC_THREADS)
        h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + warp;
    const uint32_t key_est = refill ? 0u : p.st->key_est;
    const int shift0 = refill ? (KM == KEY_MAG ? 19 : 20) : p.st->shift0;
    const float pm = (EF && PM == 2 && !refill) ? *p.pm : 0.f;
    const uint32_t dummy = GVC_H0_BINS + lane;
    double nacc = 0.0;
    if (seg < p.S)
        collect_segment<KM, EF, PM, REFILL>(p, seg, lane, h, dummy, key_est, shift0, pm, nacc, stage_v[warp],
                                            stage_i[warp], mwords[warp]);
    nacc = warp_sum_f64(nacc);
    if (lane == 0)
        red[warp] = nacc;
    __syncthreads();
    if (threadIdx.x == 0 && !refill) {
        double b = 0.0;
        for (int w = 0; w < GVC_WARPS_PER_BLOCK; w++)
            b += red[w];
        p.blk_norm[blockIdx.x] = b;
    }
    for (int i = threadIdx.x; i < GVC_H0_BINS; i += GVC_THREADS)
        if (h[i])
            atomicAdd(&p.hist0[i], h[i]);
    GVC_STAMP_OUT(1);
}

// ----------------------------------------------------------------- resolve
__device__ void set_jstate(JState &js, unsigned long long lo, unsigned long long hi, unsigned long long above,
                           unsigned long long need)
{
    js.lo = lo;
    js.hi = hi;
    js.above = above;
    js.need = need;
    unsigned long long w = hi - lo;
    int shf = bitlen64(w - 1) - 12;
    js.shift = shf < 0 ? 0 : shf;
    js.resolved = (w == 1);
}

// For a 4096-bin histogram `h` (PER bins per thread: PER * blockDim = 4096):
// calls fn(j, bin, count_above_bin) for every need[j] whose crossing bin
// (first bin from the top where the running count reaches need[j]) is local.
// CG: `h` is global memory written by other CTAs of the same cooperative
// kernel (loaded past L1); otherwise `h` may be shared memory.
template <int PER = 4, bool CG = false, typename F>
__device__ __forceinline__ void find_crossings(const uint32_t *h, unsigned long long *sh, int nneed,
                                               const unsigned long long *need, F fn)
{
    const int t = threadIdx.x;
    uint32_t c[PER];
    unsigned long long local = 0;
    if constexpr (PER % 4 == 0) {
#pragma unroll
        for (int q = 0; q < PER / 4; q++) {
            const uint4 *src = reinterpret_cast<const uint4 *>(h) + t * (PER / 4) + q;
            const uint4 x = CG ? ld_cg(src) : *src;
            c[4 * q] = x.x;
            c[4 * q + 1] = x.y;
            c[4 * q + 2] = x.z;
            c[4 * q + 3] = x.w;
            local += (unsigned long long)x.x + x.y + x.z + x.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < PER; q++) {
            c[q] = CG ? ld_cg(h + t * PER + q) : h[t * PER + q];
            local += c[q];
        }
    }
    unsigned long long total;
    unsigned long long pre = block_excl_prefix(local, sh, &total);
    // count strictly above my bins / including them: a need crosses here iff
    // acc_lo < need <= acc_hi (one load per need, the bin scan only where it crosses)
    const unsigned long long acc_lo = total - pre - local, acc_hi = total - pre;
    for (int j = 0; j < nneed; j++) {
        const unsigned long long nd = need[j];
        if (acc_lo < nd && nd <= acc_hi) {
            unsigned long long acc = acc_lo;
            int hit = -1;
            unsigned long long hit_acc = 0;
#pragma unroll
            for (int i = PER - 1; i >= 0; i--) {
                if (hit < 0 && acc + c[i] >= nd) {
                    hit = i;
                    hit_acc = acc;
                }
                acc += c[i];
            }
            fn(j, PER * t + hit, hit_acc);
        }
    }
}

// Level 0: candidate total, fallback decision, first interval per ladder entry.
// PER = 4096 / blockDim bins per thread.
template <int PER>
__device__ void resolve_level0(const Plan &p, int pass, unsigned long long *sh, unsigned long long *need)
{
    SelState *st = p.st;
    if (threadIdx.x < p.n_ks)
        need[threadIdx.x] = p.ks[threadIdx.x];
    __syncthreads();
    const uint32_t key_est = pass == 1 ? 0u : ld_cg(&st->key_est);
    const int shift0 = pass == 1 ? (p.keymode == KEY_MAG ? 19 : 20) : ld_cg(&st->shift0);
    unsigned long long local = 0;
#pragma unroll
    for (int q = 0; q < PER / 4; q++) {
        const uint4 x = ld_cg(reinterpret_cast<const uint4 *>(p.hist0) + threadIdx.x * (PER / 4) + q);
        local += (unsigned long long)x.x + x.y + x.z + x.w;
    }
    unsigned long long total;
    block_excl_prefix(local, sh, &total);
    if (pass == 0 && total < p.ks[0]) {
        if (p.allow_short) {
            // DGC overshoot (compressors.py:126-128): keep every candidate
            if (threadIdx.x == 0)
                st->shortfall = p.ks[0] - total;
            __syncthreads();
            need[0] = total;
            if (total == 0) {
                if (threadIdx.x == 0) {
                    set_jstate(st->js[0], 0xffffffffull, 1ull << 32, 0, 0);
                    st->js[0].resolved = 1;
                    st->cand_total = 0;
                    st->pending = 0;
                }
                return;
            }
        } else {
            // the estimate overshot: zero the histogram for the exact re-collect
#pragma unroll
            for (int q = 0; q < PER / 4; q++)
                reinterpret_cast<uint4 *>(p.hist0)[threadIdx.x * (PER / 4) + q] = make_uint4(0, 0, 0, 0);
            if (threadIdx.x == 0)
                st->fallback = 1;
            return;
        }
    }
    find_crossings<PER, true>(p.hist0, sh, p.n_ks, need, [&](int j, int b, unsigned long long above) {
        unsigned long long lo = (unsigned long long)key_est + ((unsigned long long)b << shift0);
        unsigned long long hi = (b == GVC_H0_BINS - 1) ? (1ull << 32) : lo + (1ull << shift0);
        if (hi > (1ull << 32))
            hi = 1ull << 32;
        set_jstate(st->js[j], lo, hi, above, need[j] - above);
    });
    __syncthreads();
    if (threadIdx.x == 0) {
        if (pass == 1) {
            st->key_est = key_est;
            st->shift0 = shift0;
        }
        st->cand_total = total;
        uint32_t pend = 0;
        for (int j = 0; j < p.n_ks; j++)
            pend += !st->js[j].resolved;
        st->pending = pend;
    }
}

// Level 0 (one block): candidate total, first interval per ladder entry.  If
// the sampled estimate overshot (fewer than k_0 candidates) the same block
// re-collects every segment with key_est = 0 -- the exactness refill, taken
// with probability ~1e-7 per step, so it lives here instead of as two
// early-exit launches in every select graph -- and resolves level 0 again.
template <int KM, bool EF>
__global__ void __launch_bounds__(1024) k_resolve0(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(2);
    __shared__ unsigned long long sh[33];
    __shared__ unsigned long long need[GVC_MAX_LADDER];
    __shared__ uint32_t hs[GVC_H0_BINS + 32];
    resolve_level0<4>(p, 0, sh, need);
    __syncthreads();
    GVC_STAMP_OUT(2);
    if (!*(volatile uint32_t *)&p.st->fallback)
        return;
    for (int i = threadIdx.x; i < GVC_H0_BINS + 32; i += blockDim.x)
        hs[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int shift = KM == KEY_MAG ? 19 : 20;
    double nacc = 0.0;  // the refill does not re-accumulate the norm
    for (uint32_t seg = warp; seg < p.S; seg += blockDim.x >> 5)
        collect_segment<KM, EF, 0, true>(p, seg, lane, hs, GVC_H0_BINS + lane, 0u, shift, 0.f, nacc);
    __syncthreads();
    for (int i = threadIdx.x; i < GVC_H0_BINS; i += blockDim.x)
        p.hist0[i] = hs[i];
    __threadfence();
    __syncthreads();
    resolve_level0<4>(p, 1, sh, need);
}

// ------------------------------------------------------- candidate pass
// After level 0 every ladder entry j has an interval [lo_j, hi_j) (its
// threshold bin).  ONE pass over the candidates:
//   * a candidate outside every interval is classified exactly: its band
//     (#{j : key >= hi_j}) goes into per-segment counts and per-block fp64
//     energies -- these are final;
//   * a candidate inside some interval (a "member") is compacted, in index
//     order, into the segment's member list and counted into the level-1
//     histogram of every interval it falls in.
// Members are few (the threshold bins are ~1/1000 octave wide), so the exact
// thresholds and the members' own contributions are finished on them alone.
template <int KM, int NB, bool ABS>
__global__ void __launch_bounds__(GVC_THREADS) k_pass1(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(3);
    extern __shared__ __align__(16) unsigned char fsm[];
    double(*acc_e)[GVC_THREADS] = reinterpret_cast<double(*)[GVC_THREADS]>(fsm);
    double(*acc_a)[GVC_THREADS] = acc_e + (NB + 1);  // only touched when ABS
    uint32_t(*acc_c)[GVC_THREADS] = reinterpret_cast<uint32_t(*)[GVC_THREADS]>(acc_a + (ABS ? NB + 1 : 0));
    __shared__ double wsum[GVC_WARPS_PER_BLOCK][2][NB];
    constexpr uint32_t P1_Q = 256;  // per-warp ring buffer of queued (slow-path) candidates
    // (+ 32 per-lane dummy slots: the branch-free queue stores of non-queued candidates)
    // one array per warp, [value bits | key | offset][slot]: the three stores
    // of a queued candidate share one address (constant offsets)
    __shared__ uint32_t p1_q[GVC_WARPS_PER_BLOCK][3][P1_Q + 32];
    const SelState *st = p.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + warp;
    const int nks = p.n_ks;
    uint32_t lo[NB], wm1[NB], him1[NB], sh[NB];
    bool act[NB];  // level-1 histogram needed (interval wider than one key)
#pragma unroll
    for (int j = 0; j < NB; j++) {
        const bool valid = j < nks;
        lo[j] = valid ? (uint32_t)st->js[j].lo : 0xffffffffu;
        wm1[j] = valid ? (uint32_t)(st->js[j].hi - st->js[j].lo - 1) : 0u;
        him1[j] = valid ? (uint32_t)(st->js[j].hi - 1) : 0xffffffffu;
        sh[j] = valid ? (uint32_t)st->js[j].shift : 0u;
        act[j] = valid && !st->js[j].resolved;
    }
#pragma unroll
    for (int b = 0; b <= NB; b++) {
        acc_e[b][threadIdx.x] = 0.0;
        if (ABS)
            acc_a[b][threadIdx.x] = 0.0;
        acc_c[b][threadIdx.x] = 0u;
    }
    uint32_t nan_any = 0;
    uint32_t hc_bin = 0xffffffffu, hc_cnt = 0;  // level-1 histogram run-length cache
    // fast window (hi_0 - 1, lo_1): band 1, in no interval (empty when the
    // first two intervals touch)
    const uint32_t f_lo = him1[0];
    const uint32_t f_hi = nks >= 2 ? lo[1] : 0xffffffffu;
    // second fast window (hi_1 - 1, lo_2): band 2 (the entries kept at the
    // candidate CF as well, ~10% of the candidates of a x10 ladder step)
    const uint32_t f2_lo = nks >= 2 ? him1[NB >= 2 ? 1 : 0] : 0xffffffffu;
    const uint32_t f2_hi = nks >= 3 ? lo[NB >= 3 ? 2 : 0] : 0xffffffffu;
    // (lo, hi) exclusive as base + unsigned width: key - base < width
    const uint32_t f1_base = f_lo + 1u, f1_w = f_hi > f_lo ? f_hi - f_lo - 1u : 0u;
    const uint32_t f2_base = f2_lo + 1u, f2_w = f2_hi > f2_lo ? f2_hi - f2_lo - 1u : 0u;
    double e_b1 = 0.0, a_b1 = 0.0, e_b2 = 0.0, a_b2 = 0.0;
    uint32_t c_b1 = 0, c_b2 = 0;
    if (seg < p.S) {
        const uint64_t beg = (uint64_t)seg * p.seg_len;
        const uint32_t cnt = p.seg_cnt[seg];
        uint32_t *mem = p.mem_idx + beg;
        const uint32_t lt = lanemask_lt();
        uint32_t mcount = 0;
        float *q_v = reinterpret_cast<float *>(p1_q[warp][0]);
        uint32_t *q_k = p1_q[warp][1], *q_t = p1_q[warp][2];
        uint32_t qh = 0, qn = 0;  // ring buffer head / count (warp-uniform)
        // classify queue entries qh .. qh + m - 1 (m <= 32), one per lane, in index order
        auto classify = [&](uint32_t m) {
            const bool okq = (uint32_t)lane < m;
            const uint32_t e = (qh + lane) & (P1_Q - 1);
            const float vq = okq ? q_v[e] : 0.f;
            const uint32_t kq = okq ? q_k[e] : 0u;
            const uint32_t tq = okq ? q_t[e] : 0u;
            int band = 0;
            bool in = false;
#pragma unroll
            for (int j = 0; j < NB; j++) {
                const uint32_t d = kq - lo[j];
                const bool inj = okq && j < nks && d <= wm1[j];
                in |= inj;
                band += kq > him1[j];
                if (inj && act[j]) {
                    // run-length cache: tie-heavy inputs put every member
                    // in one bin, and one global atomic per member then
                    // serialises on a single address
                    const uint32_t bin = j * GVC_HL_BINS + (d >> sh[j]);
                    if (bin != hc_bin) {
                        if (hc_cnt)
                            atomicAdd(&p.histl[hc_bin], hc_cnt);
                        hc_bin = bin;
                        hc_cnt = 0;
                    }
                    hc_cnt++;
                }
            }
            if (okq && !in) {
                acc_e[band][threadIdx.x] += (double)vq * (double)vq;
                if (ABS)
                    acc_a[band][threadIdx.x] += fabs((double)vq);
                acc_c[band][threadIdx.x] += 1u;
            }
            const uint32_t mbq = __ballot_sync(0xffffffffu, okq && in);
            if (mbq) {  // + the flat key list of the level-1 refinement (k_resolve1)
                uint32_t fb = 0;
                if (lane == 0)
                    fb = atomicAdd(&p.st->mem_flat, (uint32_t)__popc(mbq));
                fb = __shfl_sync(0xffffffffu, fb, 0) + __popc(mbq & lt);
                if (okq && in) {
                    mem[mcount + __popc(mbq & lt)] = tq;
                    if (fb < GVC_MEM_FLAT)
                        p.mem_key[fb] = kq;
                }
            }
            mcount += __popc(mbq);
            __syncwarp();
        };
        // register double buffer: the next 128 candidates are in flight while
        // this group is classified (a warp walks ~8 groups back to back)
        // (two groups in flight: one warp per segment and ~5 warps per SM
        // quadrant leave too few bytes in flight with a single group)
        float4 nfv = make_float4(0.f, 0.f, 0.f, 0.f), nfv2 = nfv;
        uint4 niv = make_uint4(0u, 0u, 0u, 0u), niv2 = niv;
        if (cnt) {
            nfv = *reinterpret_cast<const float4 *>(p.cand_val + beg + lane * 4);
            if (KM != KEY_MAG)
                niv = *reinterpret_cast<const uint4 *>(p.cand_idx + beg + lane * 4);
        }
        if (cnt > 128) {
            nfv2 = *reinterpret_cast<const float4 *>(p.cand_val + beg + 128 + lane * 4);
            if (KM != KEY_MAG)
                niv2 = *reinterpret_cast<const uint4 *>(p.cand_idx + beg + 128 + lane * 4);
        }
        for (uint32_t base = 0; base < cnt; base += 128) {  // warp-uniform trip count
            const uint32_t t = base + lane * 4;
            const float4 fv = nfv;
            const uint4 iv = niv;
            nfv = nfv2;
            niv = niv2;
            if (base + 256 < cnt) {
                nfv2 = *reinterpret_cast<const float4 *>(p.cand_val + beg + t + 256);
                if (KM != KEY_MAG)
                    niv2 = *reinterpret_cast<const uint4 *>(p.cand_idx + beg + t + 256);
            }
            const float v[4] = {fv.x, fv.y, fv.z, fv.w};
            const uint32_t pos[4] = {iv.x, iv.y, iv.z, iv.w};
            // fast windows in registers; everything else (band 0, members,
            // bands >= 3: ~3% at CF 10) is queued and classified 32 at a time,
            // so the NB-way classification runs on full warps instead of as
            // predicated code under every candidate.  Branch-free: a window is
            // one unsigned range test, the sums add +0.0 outside it (x + 0.0
            // == x: the same fp64 sums as adding the window's candidates
            // alone), and a non-queued candidate's queue stores go to a
            // per-lane dummy slot.  Whole groups skip the bounds tests.
            auto group = [&](auto FULL) {
                constexpr bool full = decltype(FULL)::value;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const bool okc = full || t + c < cnt;
                    const uint32_t k = okc ? cand_key<KM>(p, v[c], pos[c]) : 0u;
                    if (KM != KEY_HASH)
                        nan_any |= (uint32_t)(okc & key_nan<KM>(k));
                    const bool fast = okc & (k - f1_base < f1_w);
                    const bool fast2 = NB >= 2 && (okc & (k - f2_base < f2_w));
                    const double d = (double)v[c];
                    const double dd = d * d;
                    e_b1 += fast ? dd : 0.0;
                    c_b1 += fast ? 1u : 0u;
                    if (NB >= 2) {
                        e_b2 += fast2 ? dd : 0.0;
                        c_b2 += fast2 ? 1u : 0u;
                    }
                    if (ABS) {
                        a_b1 += fast ? fabs(d) : 0.0;
                        a_b2 += fast2 ? fabs(d) : 0.0;
                    }
                    const bool slow = okc & !fast & !fast2;
                    const uint32_t bal = __ballot_sync(0xffffffffu, slow);
                    const uint32_t slot = slow ? ((qh + qn + __popc(bal & lt)) & (P1_Q - 1)) : P1_Q + lane;
                    q_v[slot] = v[c];
                    q_k[slot] = k;
                    q_t[slot] = t + c;
                    qn += __popc(bal);
                }
            };
            if (base + 128 <= cnt)
                group(std::true_type{});
            else
                group(std::false_type{});
            __syncwarp();
            while (qn >= 32) {
                classify(32);
                qh += 32;
                qn -= 32;
            }
        }
        if (qn)
            classify(qn);
        if (lane == 0)
            p.seg_mcnt[seg] = mcount;
    }
    // flush the histogram caches: lanes holding the same bin combine first
    {
        const unsigned same = __match_any_sync(0xffffffffu, hc_cnt ? hc_bin : 0xffffffffu);
        const uint32_t tot = __reduce_add_sync(same, hc_cnt);
        if (hc_cnt && (threadIdx.x & 31) == __ffs(same) - 1)
            atomicAdd(&p.histl[hc_bin], tot);
    }
    // band 1 never reaches the shared accumulator when the fast window is
    // open, so this is the same fixed-order fp64 sum as before
    acc_e[1][threadIdx.x] += e_b1;
    if (ABS)
        acc_a[1][threadIdx.x] += a_b1;
    acc_c[1][threadIdx.x] += c_b1;
    if (NB >= 2) {
        acc_e[NB >= 2 ? 2 : 0][threadIdx.x] += e_b2;
        if (ABS)
            acc_a[NB >= 2 ? 2 : 0][threadIdx.x] += a_b2;
        acc_c[NB >= 2 ? 2 : 0][threadIdx.x] += c_b2;
    }
    __syncwarp();
    nan_any = __any_sync(0xffffffffu, nan_any);
    if (lane == 0 && nan_any)
        atomicOr(&p.st->nan_flag, 1u);
#pragma unroll
    for (int j = 0; j < NB; j++) {
        // band j+1: exactly j+1 thresholds lie below the key; band 0 is never kept
        uint32_t c1 = acc_c[j + 1][threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            c1 += __shfl_xor_sync(0xffffffffu, c1, o);
        const double e1 = warp_sum_f64(acc_e[j + 1][threadIdx.x]);
        const double a1 = ABS ? warp_sum_f64(acc_a[j + 1][threadIdx.x]) : 0.0;
        if (lane == 0) {
            wsum[warp][0][j] = e1;
            wsum[warp][1][j] = a1;
            if (seg < p.S && j < nks)
                p.seg_band[(size_t)j * GVC_SEG_MAX + seg] = c1;
        }
    }
    __syncthreads();
    if (threadIdx.x < nks) {
        const int j = threadIdx.x;
        double e1 = 0.0, a1 = 0.0;
        for (int w = 0; w < GVC_WARPS_PER_BLOCK; w++) {
            e1 += wsum[w][0][j];
            a1 += wsum[w][1][j];
        }
        const size_t o = (size_t)j * GVC_BLK_MAX + blockIdx.x;
        p.blk_band_e2[o] = e1;
        p.blk_band_ab[o] = a1;
    }
    GVC_STAMP_OUT(3);
}

// Exact thresholds (one block): the level-1 histogram, then -- only if an
// interval is still wider than one key -- radix refinement over the members
// in shared memory.
template <int KM>
__global__ void __launch_bounds__(1024) k_resolve1(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(4);
    __shared__ unsigned long long sh[33];
    __shared__ __align__(16) uint32_t hs[GVC_HL_BINS];
    SelState *st = p.st;
    // one block per ladder entry: the entries' refinements are independent
    for (int j = blockIdx.x; j < p.n_ks; j += gridDim.x) {
        if (st->js[j].resolved)
            continue;  // uniform across the block
        uint32_t *h = p.histl + j * GVC_HL_BINS;
        bool from_global = true;
        // each round narrows the interval by the 12-bit histogram: a 32-bit key
        // resolves within 3; more means an inconsistent state -- flagged, not spun on
        for (int round = 0;; round++) {
            const JState cur = st->js[j];
            if (cur.resolved)
                break;
            if (round == 6) {
                if (threadIdx.x == 0)
                    atomicOr(&st->nan_flag, 2u);
                break;
            }
            const unsigned long long nd = cur.need;
            __syncthreads();
            find_crossings(from_global ? h : hs, sh, 1, &nd, [&](int, int b, unsigned long long above) {
                unsigned long long lo = cur.lo + ((unsigned long long)b << cur.shift);
                unsigned long long hi = lo + (1ull << cur.shift);
                if (hi > cur.hi)
                    hi = cur.hi;
                set_jstate(st->js[j], lo, hi, cur.above + above, cur.need - above);
            });
            __syncthreads();
            const JState nx = st->js[j];
            if (nx.resolved)
                break;
            // refine on the members that fall in the narrowed interval
            reinterpret_cast<uint4 *>(hs)[threadIdx.x] = make_uint4(0, 0, 0, 0);
            __syncthreads();
            const uint32_t lo = (uint32_t)nx.lo, wm1 = (uint32_t)(nx.hi - nx.lo - 1);
            const uint32_t nflat = st->mem_flat;
            if (nflat <= GVC_MEM_FLAT) {
                // every entry's members, flat and coalesced (the per-segment
                // walk below is a chain of dependent loads per thread: 95 us
                // at 138M on DGC's composite keys, measured)
                uint32_t f = threadIdx.x;
                for (; f + 3 * 1024 < nflat; f += 4 * 1024) {
                    uint32_t kk[4];
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        kk[u] = p.mem_key[f + u * 1024];
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        if (kk[u] - lo <= wm1)
                            atomicAdd(&hs[(kk[u] - lo) >> nx.shift], 1u);
                }
                for (; f < nflat; f += 1024) {
                    const uint32_t key = p.mem_key[f];
                    if (key - lo <= wm1)
                        atomicAdd(&hs[(key - lo) >> nx.shift], 1u);
                }
            } else {  // more members than the flat list holds
                for (uint32_t sg = threadIdx.x; sg < p.S; sg += 1024) {
                    const uint64_t beg = (uint64_t)sg * p.seg_len;
                    const uint32_t mc = p.seg_mcnt[sg];
                    for (uint32_t i = 0; i < mc; i++) {
                        const uint32_t t = p.mem_idx[beg + i];
                        const float v = p.cand_val[beg + t];
                        const uint32_t key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, p.cand_idx[beg + t]);
                        if (key - lo <= wm1)
                            atomicAdd(&hs[(key - lo) >> nx.shift], 1u);
                    }
                }
            }
            from_global = false;
        }
    }
    GVC_STAMP_OUT(4);
}

// Members' own contributions: exact band (#{j : T_j < key}), ties per entry;
// adds to the per-segment counts and per-block energies of k_pass1 in a fixed
// order (pass-1 part first, then the members in index order).
template <int KM, int NB, bool ABS>
__global__ void __launch_bounds__(GVC_THREADS) k_members(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(5);
    __shared__ double wsum[GVC_WARPS_PER_BLOCK][4][NB];
    __shared__ uint32_t wcnt[GVC_WARPS_PER_BLOCK][2][NB];
    const SelState *st = p.st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + warp;
    const int nks = p.n_ks;
    uint32_t T[NB];
#pragma unroll
    for (int j = 0; j < NB; j++)
        T[j] = j < nks ? (uint32_t)st->js[j].lo : 0xffffffffu;
    uint32_t bc[NB], tc[NB];
    double be[NB], ba[NB], te[NB], ta[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
        bc[j] = tc[j] = 0;
        be[j] = ba[j] = te[j] = ta[j] = 0.0;
    }
    if (seg < p.S) {
        const uint64_t beg = (uint64_t)seg * p.seg_len;
        const uint32_t mc = p.seg_mcnt[seg];
        for (uint32_t base = 0; base < mc; base += 32) {
            const uint32_t i = base + lane;
            if (i < mc) {
                const uint32_t t = p.mem_idx[beg + i];
                const float v = p.cand_val[beg + t];
                const uint32_t key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, p.cand_idx[beg + t]);
                const double v2 = (double)v * (double)v, av = fabs((double)v);
                int band = 0;
#pragma unroll
                for (int j = 0; j < NB; j++)
                    band += j < nks && T[j] < key;
#pragma unroll
                for (int j = 0; j < NB; j++) {
                    const bool inb = band == j + 1;
                    const bool tie = j < nks && key == T[j];
                    bc[j] += inb;
                    tc[j] += tie;
                    be[j] += inb ? v2 : 0.0;
                    te[j] += tie ? v2 : 0.0;
                    if (ABS) {
                        ba[j] += inb ? av : 0.0;
                        ta[j] += tie ? av : 0.0;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NB; j++) {
        uint32_t c1 = bc[j], c2 = tc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c1 += __shfl_xor_sync(0xffffffffu, c1, o);
            c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        }
        const double e1 = warp_sum_f64(be[j]), a1 = ABS ? warp_sum_f64(ba[j]) : 0.0;
        const double e2 = warp_sum_f64(te[j]), a2 = ABS ? warp_sum_f64(ta[j]) : 0.0;
        if (lane == 0) {
            uint32_t band_total = 0;
            if (seg < p.S && j < nks) {
                band_total = p.seg_band[(size_t)j * GVC_SEG_MAX + seg] + c1;
                p.seg_band[(size_t)j * GVC_SEG_MAX + seg] = band_total;
                p.seg_tie[(size_t)j * GVC_SEG_MAX + seg] = c2;
            }
            wcnt[warp][0][j] = band_total;
            wcnt[warp][1][j] = c2;
            wsum[warp][0][j] = e1;
            wsum[warp][1][j] = a1;
            wsum[warp][2][j] = e2;
            wsum[warp][3][j] = a2;
        }
    }
    __syncthreads();
    if (threadIdx.x < nks) {
        const int j = threadIdx.x;
        uint32_t c1 = 0, c2 = 0;
        double e1 = 0.0, a1 = 0.0, e2 = 0.0, a2 = 0.0;
        for (int w = 0; w < GVC_WARPS_PER_BLOCK; w++) {
            c1 += wcnt[w][0][j];
            c2 += wcnt[w][1][j];
            e1 += wsum[w][0][j];
            a1 += wsum[w][1][j];
            e2 += wsum[w][2][j];
            a2 += wsum[w][3][j];
        }
        const size_t o = (size_t)j * GVC_BLK_MAX + blockIdx.x;
        p.blk_band_e2[o] += e1;
        p.blk_band_ab[o] += a1;
        p.blk_band_cnt[o] = c1;
        p.blk_tie_cnt[o] = c2;
        p.blk_tie_e2[o] = e2;
        p.blk_tie_ab[o] = a2;
    }
    GVC_STAMP_OUT(5);
}

// k_finish, one block per ladder entry j (the entries are independent):
// tie cut for T_j (lowest-index ties via the per-block prefix), kept energy
// and |v| sum (gain numerator, Redsync mean), per-block output offsets.  Two
// barrier phases: [norm, band sums >= j, tie prefix] and then [tie sums,
// offset prefix].  Block 0 also reports the norm; the last block to finish
// writes the status (after every entry's consistency check).
template <int KM>
__device__ __forceinline__ void finish_pair_sum(double &a, double &b, unsigned long long &c, unsigned long long &ct,
                                                double *shd, unsigned long long *shu)
{
    // deterministic fixed-order sums of a, b (fp64) and an exclusive prefix of c
    // (total in ct) over the block, sharing the barriers
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (int)(blockDim.x >> 5);
    a = warp_sum_f64(a);
    b = warp_sum_f64(b);
    unsigned long long x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31) {
        shd[2 * warp] = a;
        shd[2 * warp + 1] = b;
        shu[warp] = x;
    }
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < nwarps ? shu[lane] : 0ull, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o)
                wi += y;
        }
        if (lane < nwarps)
            shu[lane] = wi - w;
        if (lane == 31)
            shu[32] = wi;
        if (lane == 0) {
            double ra = 0.0, rb = 0.0;
            for (int w2 = 0; w2 < nwarps; w2++) {
                ra += shd[2 * w2];
                rb += shd[2 * w2 + 1];
            }
            shd[64] = ra;
            shd[65] = rb;
        }
    }
    __syncthreads();
    a = shd[64];
    b = shd[65];
    ct = shu[32];
    c = shu[warp] + x - c;
    __syncthreads();
}

template <int KM>
__global__ void __launch_bounds__(1024) k_finish_j(const Plan p, int)
{
    pdl_enter(); GVC_STAMP_IN(6);
    constexpr int PER = GVC_BLK_MAX / 1024;  // 2 blocks per thread, contiguous
    __shared__ double shd[66];
    __shared__ unsigned long long shu[33];
    __shared__ double shn[66];
    __shared__ unsigned long long shn_u[33];
    __shared__ uint32_t part_blk;
    __shared__ unsigned long long part_take;
    __shared__ int last;
    SelState *st = p.st;
    gvc_select_result *res = p.res;
    const uint32_t B = p.B;
    const int nks = p.n_ks;
    const int j = blockIdx.x;
    const int t = threadIdx.x;
    if (j >= nks)
        return;
    const uint32_t T = (uint32_t)st->js[j].lo;
    const unsigned long long q = st->js[j].need;
    // ---- one load phase: this thread's 2 blocks
    double nrm = 0.0, be = 0.0, ba = 0.0;
    uint32_t above[PER], tc[PER];
    double tie_e2[PER], tie_ab[PER];
    unsigned long long cabove = 0, tpre = 0;
#pragma unroll
    for (int i = 0; i < PER; i++) {
        const uint32_t b = t * PER + i;
        const bool ok = b < B;
        above[i] = 0u;
        if (ok) {
            if (j == 0)
                nrm += p.blk_norm[b];
            for (int band = j; band < nks; band++) {
                const size_t o = (size_t)band * GVC_BLK_MAX + b;
                above[i] += p.blk_band_cnt[o];
                be += p.blk_band_e2[o];
                ba += p.blk_band_ab[o];
            }
        }
        const size_t oj = (size_t)j * GVC_BLK_MAX + b;
        tc[i] = ok ? p.blk_tie_cnt[oj] : 0u;
        tie_e2[i] = ok ? p.blk_tie_e2[oj] : 0.0;
        tie_ab[i] = ok ? p.blk_tie_ab[oj] : 0.0;
        cabove += above[i];
        tpre += tc[i];
    }
    if (t == 0)
        part_blk = 0xffffffffu;
    // ---- phase 1: norm (block 0), band sums >= j, totals / tie prefix
    unsigned long long ca_tot, tp_tot;
    {
        double nz = 0.0;
        finish_pair_sum<KM>(nrm, nz, cabove, ca_tot, shn, shn_u);
    }
    finish_pair_sum<KM>(be, ba, tpre, tp_tot, shd, shu);
    // ---- tie cut per block, selected counts
    double te = 0.0, ta = 0.0;
    unsigned long long sel[PER], so = 0;
    {
        unsigned long long before = tpre;
#pragma unroll
        for (int i = 0; i < PER; i++) {
            const uint32_t b = t * PER + i;
            const unsigned long long c = tc[i];
            const unsigned long long tk = before >= q ? 0 : (q - before < c ? q - before : c);
            before += c;
            if (b < B) {
                p.blk_take[(size_t)j * GVC_BLK_MAX + b] = (uint32_t)tk;
                if (tk == c && tk > 0) {
                    te += tie_e2[i];
                    ta += tie_ab[i];
                }
                if (tk > 0 && tk < c) {
                    part_blk = b;
                    part_take = tk;
                }
            }
            sel[i] = b < B ? tk + above[i] : 0ull;
            so += sel[i];
        }
    }
    __syncthreads();
    // ---- the (rare) partially-taken block: first part_take ties in index order
    if (part_blk != 0xffffffffu) {
        unsigned long long seen = 0;
        const uint32_t pb = part_blk;
        const uint32_t s_end = min(p.S, (pb + 1) * GVC_WARPS_PER_BLOCK);
        for (uint32_t sg = pb * GVC_WARPS_PER_BLOCK; sg < s_end; sg++) {
            const uint64_t beg = (uint64_t)sg * p.seg_len;
            const uint32_t cn = p.seg_cnt[sg];
            for (uint32_t base = 0; base < cn; base += blockDim.x) {
                const uint32_t tt = base + t;
                bool is_tie = false;
                float v = 0.f;
                if (tt < cn) {
                    v = p.cand_val[beg + tt];
                    const uint32_t key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, p.cand_idx[beg + tt]);
                    is_tie = key == T;
                }
                unsigned long long tot;
                const unsigned long long rank = seen + block_excl_prefix(is_tie ? 1ull : 0ull, shu, &tot);
                if (is_tie && rank < part_take) {
                    te += (double)v * (double)v;
                    ta += fabs((double)v);
                }
                seen += tot;
            }
        }
    }
    // ---- phase 2: tie sums and the per-block output offsets
    unsigned long long so_tot;
    finish_pair_sum<KM>(te, ta, so, so_tot, shd, shu);
    {
        unsigned long long off = so;
#pragma unroll
        for (int i = 0; i < PER; i++) {
            const uint32_t b = t * PER + i;
            if (b < B)
                p.blk_off[(size_t)j * GVC_BLK_MAX + b] = (uint32_t)off;
            off += sel[i];
        }
    }
    if (t == 0) {
        const unsigned long long k = p.ks[j] - (j == 0 ? st->shortfall : 0ull);
        const double A = ba + ta;
        double E = be + te;
        const float m = (float)(A / (double)k);
        const unsigned long long nnz = k - ((KM != KEY_HASH && (T & 0x7fffffffu) == 0u) ? q : 0ull);
        if (p.kind == GVC_REDSYNC)
            E = (double)nnz * ((double)m * (double)m);
        st->redsync_mean[j] = m;
        res->kept_sq[j] = E;
        res->kept_abs[j] = A;
        res->threshold_key[j] = T;
        res->tie_quota[j] = q;
        res->redsync_mean[j] = m;
        res->kept_count[j] = so_tot;
        res->kept_nonzero[j] = nnz;
        if (ca_tot + q != k || so_tot != k)
            atomicOr(&st->nan_flag, 2u);  // internal consistency failure
        if (j == 0) {
            res->ef_norm_sq = nrm;
            res->candidates = st->cand_total;
            res->fallback_used = (int)st->fallback;
            res->shortfall = st->shortfall;
        }
        __threadfence();
        last = atomicAdd(&st->fin_done, 1u) == (unsigned)nks - 1;
    }
    __syncthreads();
    if (last && t == 0) {
        __threadfence();
        const uint32_t f = atomicOr(&st->nan_flag, 0u);
        res->status = (f & 1u) ? GVC_ERR_NAN : ((f & 2u) ? GVC_ERR_STATE : GVC_OK);
    }
    GVC_STAMP_OUT(6);
}

// -------------------------------------------------------------------- emit
// One warp per segment: in-block prefix of the 8 segments' tie / selected
// counts (lanes 0..7), then an ordered 4-wide compaction.
// Sent-mask words of a level-1 emit are private to the segment (segments are
// 512-aligned), so each warp builds them in shared memory and writes every
// word of its segment once, coalesced.  Second-level emits (idx_map) map to
// arbitrary words and OR into global memory.
// Mirrors (push exchange): every output store is repeated into the peers'
// receive slots (ordinary stores to peer-mapped memory over NVLink), and each
// thread ends with a system-scope fence so the payload is complete at every
// peer before the signal that follows this kernel.
struct Mirrors {
    int n;
    uint32_t *idx[GVC_MAX_PEERS];
    float *val[GVC_MAX_PEERS];
    uint32_t *tb[GVC_MAX_PEERS];
    uint16_t *off;  // this rank's 16-bit wire indices (idx mod GVC_AGG_TILE), or null
};

// LEAN: the hot level-1 emit (no idx_map, no direct residual, no Redsync
// substitution, no statistics, no mirrors) compiled without those paths --
// uniform runtime flags still cost predicated instructions per candidate.
template <int KM, bool SMEM_MASK, bool LEAN = false>
__global__ void __launch_bounds__(GVC_THREADS) k_emit(Plan p, int j, const uint32_t *idx_map, uint32_t *out_idx,
                                                      float *out_val, float *resid, uint32_t *smask, float *sm_out,
                                                      uint32_t *tile_b, Mirrors mir, int want_stats)
{
    if (LEAN) {
        idx_map = nullptr;
        resid = nullptr;
        mir.n = 0;  // (mir.off stays: the staged exchange's wire indices)
        want_stats = 0;
    }
    __shared__ double wst[GVC_WARPS_PER_BLOCK][2];
    extern __shared__ uint32_t mwords[];  // [8][seg_len / 32] when SMEM_MASK
    const uint32_t nwords = p.seg_len >> 5;
    uint32_t *mw = mwords + (threadIdx.x >> 5) * nwords;
    if (SMEM_MASK) {
        for (uint32_t w = threadIdx.x & 31; w < nwords; w += 32)
            mw[w] = 0u;
        __syncwarp();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t blk = blockIdx.x;
    const uint32_t seg = blk * GVC_WARPS_PER_BLOCK + warp;
    const SelState *st = p.st;
    const uint32_t T = (uint32_t)st->js[j].lo;
    const float m = st->redsync_mean[j];
    const bool redsync = !LEAN && p.kind == GVC_REDSYNC;
    const int nks = p.n_ks;
    // per-segment counts of this block in lanes 0..7
    uint32_t my_tie = 0, my_above = 0;
    const uint32_t lseg = blk * GVC_WARPS_PER_BLOCK + lane;
    if (lane < GVC_WARPS_PER_BLOCK && lseg < p.S) {
        my_tie = p.seg_tie[(size_t)j * GVC_SEG_MAX + lseg];
        for (int band = j; band < nks; band++)
            my_above += p.seg_band[(size_t)band * GVC_SEG_MAX + lseg];
    }
    uint32_t tie_pre = my_tie;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, tie_pre, o);
        if (lane >= o)
            tie_pre += y;
    }
    tie_pre -= my_tie;
    const uint32_t btake = p.blk_take[(size_t)j * GVC_BLK_MAX + blk];
    const uint32_t my_take = tie_pre >= btake ? 0u : min(btake - tie_pre, my_tie);
    const uint32_t my_sel = my_above + my_take;
    uint32_t sel_pre = my_sel;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, sel_pre, o);
        if (lane >= o)
            sel_pre += y;
    }
    sel_pre -= my_sel;
    const uint32_t take = __shfl_sync(0xffffffffu, my_take, warp);
    uint32_t out = p.blk_off[(size_t)j * GVC_BLK_MAX + blk] + __shfl_sync(0xffffffffu, sel_pre, warp);

    if (sm_out && blk == 0 && threadIdx.x == 0)
        *sm_out = m;
    double e2 = 0.0, ab = 0.0;
    if (seg < p.S) {
        const uint64_t beg = (uint64_t)seg * p.seg_len;
        const uint32_t cnt = p.seg_cnt[seg];
        const uint32_t lt = lanemask_lt();
        uint32_t ties_seen = 0;
        // tile boundaries (tb): the next output tile whose first position is
        // still unassigned; this segment owns the tiles starting inside it
        uint32_t t_next = (uint32_t)((beg + GVC_AGG_TILE - 1) / GVC_AGG_TILE);
        // 4 coalesced 32-wide sub-groups per trip: loads in flight together,
        // stores stay contiguous across the warp
        // register double buffer: the next group's loads are issued before
        // this group is classified and stored
        float nv[4];
        uint32_t npos[4];
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const uint32_t t = c * 32 + lane;
            nv[c] = t < cnt ? p.cand_val[beg + t] : 0.f;
            npos[c] = t < cnt ? p.cand_idx[beg + t] : 0u;
        }
        for (uint32_t base = 0; base < cnt; base += 128) {  // warp-uniform trip count
            float v[4];
            uint32_t pos[4], key[4];
            bool ok[4];
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const uint32_t t = base + c * 32 + lane;
                ok[c] = t < cnt;
                v[c] = nv[c];
                pos[c] = npos[c];
                const uint32_t tn = t + 128;
                nv[c] = tn < cnt ? p.cand_val[beg + tn] : 0.f;
                npos[c] = tn < cnt ? p.cand_idx[beg + tn] : 0u;
            }
#pragma unroll
            for (int c = 0; c < 4; c++)
                key[c] = ok[c] ? cand_key<KM>(p, v[c], pos[c]) : 0u;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const bool tie = ok[c] && key[c] == T;
                const uint32_t tb = __ballot_sync(0xffffffffu, tie);
                const bool sel = ok[c] && (key[c] > T || (tie && ties_seen + __popc(tb & lt) < take));
                const uint32_t sb = __ballot_sync(0xffffffffu, sel);
                // tiles start in this group only if its last selected position
                // lies in a tile >= t_next (warp-uniform; ~1 group in 13 at CF 10)
                if (tile_b && sb && __shfl_sync(0xffffffffu, pos[c], 31 - __clz(sb)) / GVC_AGG_TILE >= t_next) {
                    // tiles starting in (previous selected index, this index] begin here
                    const uint32_t prior = sb & lt;
                    const int pl = prior ? 31 - __clz(prior) : 0;
                    const uint32_t gprev = __shfl_sync(0xffffffffu, pos[c], pl);
                    if (sel) {
                        const uint32_t t_lo = prior ? gprev / GVC_AGG_TILE + 1 : t_next;
                        const uint32_t t_hi = pos[c] / GVC_AGG_TILE;
                        for (uint32_t t = t_lo; t <= t_hi; t++) {
                            tile_b[t] = out + __popc(sb & lt);
                            for (int q = 0; q < mir.n; q++)
                                mir.tb[q][t] = out + __popc(sb & lt);
                        }
                    }
                    if (sb)
                        t_next = __shfl_sync(0xffffffffu, pos[c], 31 - __clz(sb)) / GVC_AGG_TILE + 1;
                }
                if (sel) {
                    float sv = v[c];
                    if (redsync) {
                        float sg = v[c] > 0.f ? 1.f : (v[c] < 0.f ? -1.f : 0.f);
                        sv = __fmul_rn(sg, m);
                    }
                    const uint32_t w = out + __popc(sb & lt);
                    const uint32_t gi = idx_map ? idx_map[pos[c]] : pos[c];
                    out_idx[w] = gi;
                    out_val[w] = sv;
                    if (mir.off)
                        mir.off[w] = (uint16_t)(gi & (GVC_AGG_TILE - 1));
                    if (!LEAN) {
                        for (int q = 0; q < mir.n; q++) {
                            mir.idx[q][w] = gi;
                            mir.val[q][w] = sv;
                        }
                    }
                    if (SMEM_MASK)
                        atomicOr(&mw[(pos[c] - (uint32_t)beg) >> 5], 1u << (pos[c] & 31));
                    else if (smask)
                        atomicOr(&smask[gi >> 5], 1u << (gi & 31));
                    if (!LEAN && resid) {
                        // level-1 emits: the candidate value IS g_ef; a second-level
                        // emit (idx_map) carries level-1 SENT values, so read g_ef back
                        const float ef = idx_map ? resid[gi] : v[c];
                        resid[gi] = __fsub_rn(ef, sv);
                    }
                    if (!LEAN && want_stats) {
                        e2 += (double)sv * (double)sv;
                        ab += fabs((double)sv);
                    }
                }
                ties_seen += __popc(tb);
                out += __popc(sb);
            }
        }
        if (tile_b) {
            // tiles starting after this segment's last output and before its end;
            // the last segment also writes entry ntiles (= the total count)
            const uint64_t end = min(p.n, beg + p.seg_len);
            const uint64_t ntiles = (p.n + GVC_AGG_TILE - 1) / GVC_AGG_TILE;
            const uint64_t t_end = end == p.n ? ntiles : (end - 1) / GVC_AGG_TILE;
            for (uint64_t t = t_next + lane; t <= t_end; t += 32) {
                tile_b[t] = out;
                for (int q = 0; q < mir.n; q++)
                    mir.tb[q][t] = out;
            }
        }
    }
    if (mir.n)
        __threadfence_system();
    if (SMEM_MASK && seg < p.S) {
        __syncwarp();
        const uint64_t beg = (uint64_t)seg * p.seg_len;
        const uint32_t live = (uint32_t)((min(p.n, beg + p.seg_len) - beg + 31) >> 5);
        for (uint32_t w = lane; w < live; w += 32)
            smask[(beg >> 5) + w] = mw[w];
    }
    if (!want_stats)
        return;  // uniform: the sent-value statistics are not requested
    e2 = warp_sum_f64(e2);
    ab = warp_sum_f64(ab);
    if (lane == 0) {
        wst[warp][0] = e2;
        wst[warp][1] = ab;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < GVC_WARPS_PER_BLOCK; w++) {
            a += wst[w][0];
            b += wst[w][1];
        }
        p.blk_emit[blk] = a;
        p.blk_emit[GVC_BLK_MAX + blk] = b;
    }
}

__global__ void __launch_bounds__(1024) k_emit_finish(Plan p, double *stats)
{
    __shared__ double shd[33];
    double a = 0.0, b = 0.0;
    constexpr int PER = GVC_BLK_MAX / 1024;
    for (int i = 0; i < PER; i++) {
        uint32_t k = threadIdx.x * PER + i;
        if (k < p.B) {
            a += p.blk_emit[k];
            b += p.blk_emit[GVC_BLK_MAX + k];
        }
    }
    a = block_sum_f64(a, shd);
    b = block_sum_f64(b, shd);
    if (threadIdx.x == 0) {
        stats[0] = a;
        stats[1] = b;
    }
}

// ============================================================ host driver
static std::mutex g_mu;
static std::unordered_map<const void *, Plan> g_plans;

size_t select_workspace_bytes(int kind, uint64_t n)
{
    (void)kind;
    return carve(nullptr, nullptr, n);
}

static int nb_for(int n_ks) { return n_ks <= 1 ? 1 : n_ks <= 2 ? 2 : n_ks <= 4 ? 4 : n_ks <= 8 ? 8 : 16; }

// Launch with programmatic stream serialization (PDL) when `pdl`.
template <typename Kern>
static void launch_k(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, const Plan &p,
                     int aux)
{
    if (!pdl) {
        kernel<<<grid, block, smem, s>>>(p, aux);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, p, aux);
}

template <int KM, int NB, bool ABS>
static void launch_tail_nb(const Plan &p, cudaStream_t s, bool pdl)
{
    const size_t smem = (size_t)(NB + 1) * GVC_THREADS * (8 + (ABS ? 8 : 0) + 4);
    launch_k(k_pass1<KM, NB, ABS>, dim3((unsigned)p.B), dim3(GVC_THREADS), smem, s, pdl, p, 0);
    launch_k(k_resolve1<KM>, dim3(NB), dim3(1024), 0, s, pdl, p, 0);  // NB (in the graph key) >= n_ks blocks
    launch_k(k_members<KM, NB, ABS>, dim3((unsigned)p.B), dim3(GVC_THREADS), 0, s, pdl, p, 0);
}

// |v| sums are only consumed by Redsync's mean (compressors.py:188)
template <int KM>
static void launch_tail(const Plan &p, cudaStream_t s, bool pdl)
{
    if constexpr (KM == KEY_DGC) {  // DGC picks one keep count at a time
        launch_tail_nb<KM, 1, false>(p, s, pdl);
    } else if constexpr (KM == KEY_POS) {  // one keep count (a level-2 Redsync / Top-k pick)
        if (p.kind == GVC_REDSYNC)
            launch_tail_nb<KM, 1, true>(p, s, pdl);
        else
            launch_tail_nb<KM, 1, false>(p, s, pdl);
    } else {
        const bool abs_sums = p.kind == GVC_REDSYNC;
        switch (nb_for(p.n_ks)) {
        case 1: abs_sums ? launch_tail_nb<KM, 1, true>(p, s, pdl) : launch_tail_nb<KM, 1, false>(p, s, pdl); break;
        case 2: abs_sums ? launch_tail_nb<KM, 2, true>(p, s, pdl) : launch_tail_nb<KM, 2, false>(p, s, pdl); break;
        case 4: abs_sums ? launch_tail_nb<KM, 4, true>(p, s, pdl) : launch_tail_nb<KM, 4, false>(p, s, pdl); break;
        case 8: abs_sums ? launch_tail_nb<KM, 8, true>(p, s, pdl) : launch_tail_nb<KM, 8, false>(p, s, pdl); break;
        default:
            abs_sums ? launch_tail_nb<KM, 16, true>(p, s, pdl) : launch_tail_nb<KM, 16, false>(p, s, pdl);
            break;
        }
    }
}

static int current_device()
{
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// One-time kernel attributes per device (cudaFuncSetAttribute is per device),
// outside any stream capture.
static void set_attributes()
{
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    const int dev = current_device();
    if (std::find(done.begin(), done.end(), dev) != done.end())
        return;
    done.push_back(dev);
    cudaFuncSetAttribute(k_sample<KEY_MAG>, cudaFuncAttributeMaxDynamicSharedMemorySize, GVC_SAMPLE_BINS * 4);
    cudaFuncSetAttribute(k_sample<KEY_DGC>, cudaFuncAttributeMaxDynamicSharedMemorySize, GVC_SAMPLE_BINS * 4);
    cudaFuncSetAttribute(k_sample<KEY_POS>, cudaFuncAttributeMaxDynamicSharedMemorySize, GVC_SAMPLE_BINS * 4);
#define GVC_PASS1_ATTR(KM, NB, ABS)                                                                          \
    cudaFuncSetAttribute(k_pass1<KM, NB, ABS>, cudaFuncAttributeMaxDynamicSharedMemorySize,                  \
                         (int)((NB + 1) * GVC_THREADS * (8 + (ABS ? 8 : 0) + 4)));
#define GVC_PASS1_ATTR_KM(KM)                                                                                \
    GVC_PASS1_ATTR(KM, 1, false) GVC_PASS1_ATTR(KM, 2, false) GVC_PASS1_ATTR(KM, 4, false)                  \
    GVC_PASS1_ATTR(KM, 8, false) GVC_PASS1_ATTR(KM, 16, false) GVC_PASS1_ATTR(KM, 1, true)                  \
    GVC_PASS1_ATTR(KM, 2, true) GVC_PASS1_ATTR(KM, 4, true) GVC_PASS1_ATTR(KM, 8, true)                     \
    GVC_PASS1_ATTR(KM, 16, true)
    GVC_PASS1_ATTR_KM(KEY_MAG)
    GVC_PASS1_ATTR_KM(KEY_HASH)
    GVC_PASS1_ATTR(KEY_DGC, 1, false)
    GVC_PASS1_ATTR(KEY_POS, 1, false)
    GVC_PASS1_ATTR(KEY_POS, 1, true)
}

// The select pipeline on stream s; every kernel takes the plan by value (its
// fields live in the constant bank).  Returns the number of kernels.
static cudaEvent_t g_ev_mark[4];  // capture-time placeholders: collect start/end, select start/end

template <int KM>
static int launch_pipeline(const Plan &p, cudaStream_t s, bool probes, bool gprobes)
{
    const bool pdl = !probes;  // direct probe launches keep plain stream order
    ProfScope all(probes ? PROF_SELECT : -1, s);
    const int blocks = (int)p.B;
    int launches = 0;
    if (KM != KEY_HASH && p.force_exact == 0 && p.s_target > 0 && !p.key_est_dev) {
        uint64_t wb = (p.s_chunks + 31) / 32;
        const uint64_t sms = (uint64_t)device_sms();
        int sb = (int)(wb < sms ? (wb ? wb : 1) : sms);
        k_sample<KM><<<sb, 1024, GVC_SAMPLE_BINS * 4, s>>>(p, 0);  // its last block resolves key_est
        launches++;
    } else {
        k_sample_resolve<<<1, 1024, 0, s>>>(p, 0);
        launches++;
    }
    {
        ProfScope pc(probes ? PROF_COLLECT : -1, s);
        if (gprobes)
            cudaEventRecordWithFlags(g_ev_mark[0], s, cudaEventRecordExternal);
        const bool cpdl = pdl && !gprobes;
        if (KM == KEY_POS || !p.ef)  // (KEY_POS selections are plain mode: gvc_select checks)
            launch_k(k_collect<KM, false, 0>, dim3(blocks), dim3(GVC_THREADS), 0, s, cpdl, p, 0);
        else if (!p.pmask)
            launch_k(k_collect<KM, true, 0>, dim3(blocks), dim3(GVC_THREADS), 0, s, cpdl, p, 0);
        else if (p.pmode == 1)
            launch_k(k_collect<KM, true, 1>, dim3(blocks), dim3(GVC_THREADS), 0, s, cpdl, p, 0);
        else
            launch_k(k_collect<KM, true, 2>, dim3(blocks), dim3(GVC_THREADS), 0, s, cpdl, p, 0);
        if (gprobes)
            cudaEventRecordWithFlags(g_ev_mark[1], s, cudaEventRecordExternal);
    }
    if (KM != KEY_POS && p.ef)
        launch_k(k_resolve0<KM, true>, dim3(1), dim3(1024), 0, s, pdl && !gprobes, p, 0);
    else
        launch_k(k_resolve0<KM, false>, dim3(1), dim3(1024), 0, s, pdl && !gprobes, p, 0);
    launches += 2;
    launch_tail<KM>(p, s, pdl);
    launches += 3;
    // k_finish_j: one block per ladder entry, 2 blocks per thread; only as many
    // warps as the blocks need (its block-wide reductions cost per warp).
    // Grid = NB (in the graph key) >= n_ks.
    const int fin_threads = (int)std::min<uint32_t>(1024u, std::max<uint32_t>(64u, ((p.B + 1) / 2 + 31) & ~31u));
    launch_k(k_finish_j<KM>, dim3(nb_for(p.n_ks)), dim3(fin_threads), 0, s, pdl, p, 0);
    return launches + 1;
}

static_assert(sizeof(Plan) <= 4000, "the plan is passed as a kernel parameter");

static void enqueue_select(const Plan &p, cudaStream_t s, bool probes, int *launches, bool gprobes = false)
{
    if (gprobes)
        cudaEventRecordWithFlags(g_ev_mark[2], s, cudaEventRecordExternal);
    // SelState, hist0, shist and the level-1 histograms: one memset node, its
    // size a function of the graph key (nb_for(n_ks), not n_ks: a cached graph
    // serves every ladder length of its NB class)
    cudaMemsetAsync(p.st, 0, (size_t)((char *)(p.histl + (size_t)nb_for(p.n_ks) * GVC_HL_BINS) - (char *)p.st), s);
    *launches = p.keymode == KEY_MAG   ? launch_pipeline<KEY_MAG>(p, s, probes, gprobes)
                : p.keymode == KEY_DGC ? launch_pipeline<KEY_DGC>(p, s, probes, gprobes)
                : p.keymode == KEY_POS ? launch_pipeline<KEY_POS>(p, s, probes, gprobes)
                                       : launch_pipeline<KEY_HASH>(p, s, probes, gprobes);
    if (gprobes)
        cudaEventRecordWithFlags(g_ev_mark[3], s, cudaEventRecordExternal);
}

// CUDA graphs of the select pipeline, one per launch shape.  Every kernel has
// the signature (Plan, int); per call the plan argument of each kernel node is
// replaced (host-side only, no extra device work) before the launch.
struct GraphNode {
    cudaGraphNode_t node;
    cudaKernelNodeParams kp;
    int aux;
};
struct GraphEntry {
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    std::vector<GraphNode> nodes;
    cudaGraphNode_t ev_nodes[4] = {nullptr, nullptr, nullptr, nullptr};  // g_ev_mark order (profiling graphs)
    int launches;
    Plan last;  // the plan the nodes currently hold
    bool has_last = false;
    const void *ws = nullptr;  // the workspace the graph's plans point into
};
static std::unordered_map<std::string, GraphEntry> g_graphs;

static std::string graph_key(const Plan &p, const void *ws)
{
    char buf[256];
    snprintf(buf, sizeof(buf), "%d|%p|%llu|%d|%d|%d|%d|%d|%d|%d|%d|%d", current_device(), ws,
             (unsigned long long)p.n, p.keymode, p.ef,
             p.pmask ? p.pmode : 0, nb_for(p.n_ks), p.kind == GVC_REDSYNC, p.force_exact,
             (int)(p.keymode != KEY_HASH && p.force_exact == 0 && p.s_target > 0 && !p.key_est_dev),
             p.key_est_dev != nullptr, (int)p.s_chunks);
    return std::string(buf);
}

int select_run(const gvc_select_args *a, void *ws, size_t ws_bytes, gvc_select_result *res, cudaStream_t s)
{
    Plan p;
    memset(&p, 0, sizeof(p));
    size_t need = carve(&p, (char *)ws, a->n);
    if (ws_bytes < need)
        return set_error(GVC_ERR_WORKSPACE, "select workspace too small: %zu < %zu", ws_bytes, need);
    p.n = a->n;
    p.n_ks = a->n_ks;
    p.kind = a->kind;
    p.keymode = a->kind == GVC_RANDOMK ? KEY_HASH
                : a->dgc_thr_dev         ? KEY_DGC
                : a->equal_magnitudes    ? KEY_POS
                                         : KEY_MAG;
    p.dgc_thr = a->dgc_thr_dev;
    p.dgc_bits = a->dgc_sampled_dev;
    p.ef = a->g_dev != nullptr;
    p.force_exact = a->force_exact;
    p.values = a->values_dev;
    p.g = a->g_dev;
    p.resid = a->resid_dev;
    // the hash inputs only matter for hash keys; zero otherwise so that an
    // unchanged magnitude-key plan is bit-identical call to call
    const bool hashk = a->kind == GVC_RANDOMK;
    p.seed = hashk ? a->seed : 0;
    p.stream = hashk ? a->rng_stream : 0;
    p.pos_base = hashk ? a->pos_base : 0;
    p.key_est_dev = a->key_est_dev;
    p.allow_short = a->key_est_dev ? a->allow_short : 0;
    p.pmask = p.ef ? a->pending_mask_dev : nullptr;
    p.pm = a->pending_m_dev;
    p.pmode = a->pending_mode;
    for (int j = 0; j < a->n_ks; j++)
        p.ks[j] = a->ks[j];
    p.res = res;
    const uint64_t n = a->n, k0 = a->ks[0];
    if (p.keymode != KEY_HASH) {
        // sample ~n/128 values (at most 2^19) in 128-value chunks (everything
        // when n is small): past ~10^5 sampled candidates the 5-sigma margin is
        // already a few tenths of a percent of k_0, and the sample pass is pure latency
        uint64_t want = n <= 65536 ? n : (n / 128 > 65536 ? n / 128 : 65536);
        if (want > (1ull << 19))
            want = 1ull << 19;
        uint64_t chunks = (want + 127) / 128;
        uint64_t stride = n / chunks;
        stride &= ~(uint64_t)3;
        if (stride < 128)
            stride = 128;
        chunks = (n + stride - 1) / stride;
        const uint64_t last = (chunks - 1) * stride;
        const uint64_t sampled = (chunks - 1) * 128 + (n - last < 128 ? n - last : 128);
        p.s_chunks = chunks;
        p.s_stride = stride;
        if (sampled >= n) {
            p.s_target = k0;  // the sample is the whole vector: exact bin
            p.s_target_lo = k0;
        } else {
            double mu = (double)k0 * (double)sampled / (double)n;
            double t = mu * 1.02 + 5.0 * sqrt(mu) + 32.0;
            p.s_target = t >= (double)sampled ? 0 : (uint64_t)ceil(t);
            double tl = mu * 0.98 - 5.0 * sqrt(mu) - 32.0;
            p.s_target_lo = tl <= 0.0 ? 0 : (uint64_t)floor(tl);
        }
    } else {
        double mu = (double)k0 + 8.0 * sqrt((double)k0) + 64.0;
        double frac = mu / (double)n;
        if (frac >= 1.0 || p.force_exact) {
            p.hash_key_est = 0;
        } else {
            double cut = ldexp(1.0 - frac, 32);
            p.hash_key_est = (uint32_t)(cut < 0 ? 0 : floor(cut));
        }
    }
    set_attributes();
    int launches = 0;
    const bool probe_this = prof_wants(p.n);
    if (prof_enabled() && probe_this) {
        // measurement mode: direct launches bracketed by CUDA events (bench.py roofline)
        enqueue_select(p, s, true, &launches);
    } else {
        const bool gprobes = prof_graph_enabled() && probe_this;
        const std::string key = graph_key(p, ws) + (gprobes ? "|ev" : "");
        std::lock_guard<std::mutex> glk(g_mu);
        auto it = g_graphs.find(key);
        if (it == g_graphs.end()) {
            // the capture stream belongs to a device: one per device
            static std::unordered_map<int, cudaStream_t> capture_streams;
            cudaStream_t &cs = capture_streams[current_device()];
            if (!cs)
                cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
            cudaGraph_t graph;
            GraphEntry ge;
            if (gprobes && !g_ev_mark[0]) {
                for (int e = 0; e < 4; e++)
                    cudaEventCreate(&g_ev_mark[e]);
            }
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
            enqueue_select(p, cs, false, &ge.launches, gprobes);
            cudaError_t ce = cudaStreamEndCapture(cs, &graph);
            if (ce != cudaSuccess)
                return set_error(GVC_ERR_CUDA, "select graph capture: %s", cudaGetErrorString(ce));
            size_t nn = 0;
            cudaGraphGetNodes(graph, nullptr, &nn);
            std::vector<cudaGraphNode_t> all(nn);
            cudaGraphGetNodes(graph, all.data(), &nn);
            for (cudaGraphNode_t nd : all) {
                cudaGraphNodeType ty;
                cudaGraphNodeGetType(nd, &ty);
                if (ty == cudaGraphNodeTypeEventRecord) {
                    cudaEvent_t ev;
                    cudaGraphEventRecordNodeGetEvent(nd, &ev);
                    for (int e = 0; e < 4; e++)
                        if (ev == g_ev_mark[e])
                            ge.ev_nodes[e] = nd;
                    continue;
                }
                if (ty != cudaGraphNodeTypeKernel)
                    continue;
                GraphNode gn;
                gn.node = nd;
                cudaGraphKernelNodeGetParams(nd, &gn.kp);
                gn.aux = *(const int *)gn.kp.kernelParams[1];
                gn.kp.kernelParams = nullptr;
                gn.kp.extra = nullptr;
                ge.nodes.push_back(gn);
            }
            ce = cudaGraphInstantiate(&ge.exec, graph, 0);
            ge.graph = graph;  // kept alive: the exec-node updates name its nodes
            ge.ws = ws;
            if (ce != cudaSuccess)
                return set_error(GVC_ERR_CUDA, "select graph instantiate: %s", cudaGetErrorString(ce));
            it = g_graphs.emplace(key, std::move(ge)).first;
        }
        // the node arguments change only when the plan does (steady state: the
        // same tensors every step) -- skip the per-node updates then
        if (!it->second.has_last || memcmp(&it->second.last, &p, sizeof(Plan)) != 0) {
            for (GraphNode &gn : it->second.nodes) {
                int aux = gn.aux;
                void *args[2] = {(void *)&p, (void *)&aux};
                cudaKernelNodeParams kp = gn.kp;
                kp.kernelParams = args;
                cudaError_t ue = cudaGraphExecKernelNodeSetParams(it->second.exec, gn.node, &kp);
                if (ue != cudaSuccess)
                    return set_error(GVC_ERR_CUDA, "select graph update: %s", cudaGetErrorString(ue));
            }
            it->second.last = p;
            it->second.has_last = true;
        }
        for (int e = 0; e < 4; e += 2) {
            if (it->second.ev_nodes[e] && it->second.ev_nodes[e + 1]) {
                cudaEvent_t a, b;
                prof_graph_pair(e == 0 ? PROF_COLLECT : PROF_SELECT, &a, &b);
                cudaGraphExecEventRecordNodeSetEvent(it->second.exec, it->second.ev_nodes[e], a);
                cudaGraphExecEventRecordNodeSetEvent(it->second.exec, it->second.ev_nodes[e + 1], b);
            }
        }
        cudaGraphLaunch(it->second.exec, s);
        launches = it->second.launches;
    }
    count_launches(launches);
    std::lock_guard<std::mutex> lk(g_mu);
    g_plans[ws] = p;
    return GVC_OK;
}

// gvc_workspace_forget: the select's per-workspace state (graphs, plan)
void select_forget(const void *ws)
{
    std::lock_guard<std::mutex> lk(g_mu);
    g_plans.erase(ws);
    for (auto it = g_graphs.begin(); it != g_graphs.end();) {
        if (it->second.ws == ws) {
            cudaGraphExecDestroy(it->second.exec);
            cudaGraphDestroy(it->second.graph);
            it = g_graphs.erase(it);
        } else {
            ++it;
        }
    }
}

int select_phase_times(void *ws, unsigned long long *out, int n)
{
    Plan p;
    memset(&p, 0, sizeof(p));
    carve(&p, (char *)ws, 1);
    const int m = n < 32 ? n : 32;
    cudaError_t e = cudaMemcpy(out, p.st->t_phase, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return e == cudaSuccess ? GVC_OK : set_error(GVC_ERR_CUDA, "phase times: %s", cudaGetErrorString(e));
}

int emit_run(void *ws, size_t ws_bytes, int j, const uint32_t *idx_map, uint32_t *out_idx, float *out_val,
             float *resid, uint32_t *smask, float *sm_out, uint32_t *tile_b, double *stats,
             const gvc_emit_mirrors *mirrors, cudaStream_t s)
{
    Mirrors mir;
    memset(&mir, 0, sizeof(mir));
    if (mirrors) {
        mir.n = mirrors->count;
        mir.off = mirrors->off16_dev;
        for (int q = 0; q < mir.n; q++) {
            mir.idx[q] = mirrors->idx_dev[q];
            mir.val[q] = mirrors->vals_dev[q];
            mir.tb[q] = mirrors->bounds_dev[q];
        }
    }
    (void)ws_bytes;
    Plan p;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_plans.find(ws);
        if (it == g_plans.end())
            return set_error(GVC_ERR_STATE, "gvc_emit: no gvc_select ran on this workspace");
        p = it->second;
    }
    if (j < 0 || j >= p.n_ks)
        return set_error(GVC_ERR_ARG, "gvc_emit: ladder index %d out of range [0, %d)", j, p.n_ks);
    const int blocks = (int)p.B;
    ProfScope pe(prof_wants(p.n) ? PROF_EMIT : -1, s);
    count_launches(stats ? 2 : 1);
    const size_t mbytes = (size_t)GVC_WARPS_PER_BLOCK * (p.seg_len >> 5) * 4;
    const bool smem_mask = smask && !idx_map && mbytes <= 96 * 1024;
    if (smem_mask) {
        static std::vector<int> attr_done;  // per device (under g_mu)
        std::unique_lock<std::mutex> lk(g_mu);
        const int dev = current_device();
        if (std::find(attr_done.begin(), attr_done.end(), dev) == attr_done.end()) {
            attr_done.push_back(dev);
            cudaFuncSetAttribute(k_emit<KEY_MAG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_HASH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_DGC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_MAG, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_DGC, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_POS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            cudaFuncSetAttribute(k_emit<KEY_HASH, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        }
        lk.unlock();
        const bool lean = !idx_map && !resid && mir.n == 0 && !stats && p.kind != GVC_REDSYNC;
        if (p.keymode == KEY_MAG && lean)
            k_emit<KEY_MAG, true, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid,
                                                                             smask, sm_out, tile_b, mir, 0);
        else if (p.keymode == KEY_DGC && lean)
            k_emit<KEY_DGC, true, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid,
                                                                             smask, sm_out, tile_b, mir, 0);
        else if (p.keymode == KEY_HASH && lean)
            k_emit<KEY_HASH, true, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid,
                                                                              smask, sm_out, tile_b, mir, 0);
        else if (p.keymode == KEY_MAG)
            k_emit<KEY_MAG, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                       sm_out, tile_b, mir, stats != nullptr);
        else if (p.keymode == KEY_DGC)
            k_emit<KEY_DGC, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                       sm_out, tile_b, mir, stats != nullptr);
        else if (p.keymode == KEY_POS)
            k_emit<KEY_POS, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                       sm_out, tile_b, mir, stats != nullptr);
        else
            k_emit<KEY_HASH, true><<<blocks, GVC_THREADS, mbytes, s>>>(p, j, idx_map, out_idx, out_val, resid,
                                                                        smask, sm_out, tile_b, mir, stats != nullptr);
    } else {
        if (p.keymode == KEY_MAG)
            k_emit<KEY_MAG, false><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                   sm_out, tile_b, mir, stats != nullptr);
        else if (p.keymode == KEY_DGC)
            k_emit<KEY_DGC, false><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                   sm_out, tile_b, mir, stats != nullptr);
        else if (p.keymode == KEY_POS)
            k_emit<KEY_POS, false><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                   sm_out, tile_b, mir, stats != nullptr);
        else
            k_emit<KEY_HASH, false><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid, smask,
                                                                    sm_out, tile_b, mir, stats != nullptr);
    }
    if (stats)
        k_emit_finish<<<1, 1024, 0, s>>>(p, stats);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(GVC_ERR_CUDA, "emit launch: %s", cudaGetErrorString(e));
    return GVC_OK;
}

}  // namespace gvc
