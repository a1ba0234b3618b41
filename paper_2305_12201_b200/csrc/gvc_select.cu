// gvc_select.cu -- deterministic multi-CF selection for the GraVAC step (sm_100a).
//
// One selection answers, for a ladder of keep counts k_0 >= k_1 >= ... (all
// compression factors of the search space, nested as compressors.py:237-238
// nests them), "which k_j entries have the largest key, ties to the lower
// index" -- the rule of compressors.py:86-99 -- together with the fp64 kept
// energies the gain statistic needs (metrics.py:18-32).  Keys are the 31-bit
// magnitude pattern (Top-k, Redsync, DGC) or a Philox position hash (Random-k).
//
// Pipeline (all stream-ordered, no host synchronisation):
//   k_sample / k_sample_resolve   1-2% strided sample -> conservative key_est
//   k_collect (EF fused)          ONE streaming pass over HBM: g_ef = g + r is
//                                 written over r, fp64 ||g_ef||^2, and every
//                                 key >= key_est is compacted, index-ordered,
//                                 into the warp's segment of the candidate
//                                 buffer with a level-0 histogram
//   k_resolve0 / k_collect(refill) exactness guard: if the estimate missed,
//                                 every value becomes a candidate
//   k_level_hist / k_level_resolve radix refinement over candidates only,
//                                 until each k_j has its exact threshold key
//   k_final / k_finish            per-segment band energies, tie counts, tie
//                                 cut and output offsets for EVERY ladder entry
//   k_emit (gvc_emit)             ordered (idx, val) compaction of one entry,
//                                 fused residual update
#include <mutex>
#include <unordered_map>

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
    JState js[GVC_MAX_LADDER];
    float redsync_mean[GVC_MAX_LADDER];
};

struct Plan {
    uint64_t n;
    uint32_t S, seg_len;
    int n_ks, kind, keymode, ef, force_exact;
    const float *values;
    const float *g;
    float *resid;
    uint64_t seed, stream, pos_base;
    uint64_t ks[GVC_MAX_LADDER];
    // sample
    uint64_t s_chunks, s_stride, s_target;
    uint32_t hash_key_est;
    // workspace
    SelState *st;
    uint32_t *hist0, *histl, *shist;
    uint32_t *seg_cnt;
    double *norm_part;
    uint32_t *band_cnt;  // [GVC_MAX_LADDER][SEG_MAX]
    double *band_e2, *band_ab;
    uint32_t *tie_cnt;
    double *tie_e2, *tie_ab;
    uint32_t *seg_take, *seg_off;
    double *seg_emit;  // [2][SEG_MAX]
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
    const size_t L = GVC_MAX_LADDER, SM = GVC_SEG_MAX;
    Plan tmp;
    Plan *q = p ? p : &tmp;
    q->st = (SelState *)take(sizeof(SelState));
    q->hist0 = (uint32_t *)take(GVC_H0_BINS * 4);
    q->histl = (uint32_t *)take(L * GVC_HL_BINS * 4);
    q->shist = (uint32_t *)take(GVC_SAMPLE_BINS * 4);
    q->seg_cnt = (uint32_t *)take(SM * 4);
    q->norm_part = (double *)take(SM * 8);
    q->band_cnt = (uint32_t *)take(L * SM * 4);
    q->band_e2 = (double *)take(L * SM * 8);
    q->band_ab = (double *)take(L * SM * 8);
    q->tie_cnt = (uint32_t *)take(L * SM * 4);
    q->tie_e2 = (double *)take(L * SM * 8);
    q->tie_ab = (double *)take(L * SM * 8);
    q->seg_take = (uint32_t *)take(L * SM * 4);
    q->seg_off = (uint32_t *)take(L * SM * 4);
    q->seg_emit = (double *)take(2 * SM * 8);
    q->cand_val = (float *)take(n_pad * 4);
    q->cand_idx = (uint32_t *)take(n_pad * 4);
    q->S = S;
    q->seg_len = seg_len;
    return off;
}

// ------------------------------------------------------------ key helpers
template <int KM>
__device__ __forceinline__ uint32_t cand_key(const Plan &p, float v, uint32_t pos)
{
    if (KM == KEY_MAG)
        return mag_key(v);
    return hash_key(p.pos_base + pos, p.stream, p.seed);
}

// ------------------------------------------------------------------ sample
// Strided chunks of 128 contiguous values (one warp-load) -> 16-bit histogram
// of magnitude keys in global memory.  Reads ~1.5% of the bytes.
__global__ void __launch_bounds__(GVC_THREADS) k_sample(Plan p)
{
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * GVC_WARPS_PER_BLOCK;
    uint32_t kmax = 0;
    for (uint64_t c = blockIdx.x * GVC_WARPS_PER_BLOCK + (threadIdx.x >> 5); c < p.s_chunks; c += warps) {
        uint64_t base = c * p.s_stride;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint64_t i = base + (uint64_t)q * 32 + lane;
            if (i < p.n && i < base + 128) {
                float v = p.ef ? p.g[i] + p.resid[i] : p.values[i];
                uint32_t k = mag_key(v);
                if (k <= 0x7f800000u) {
                    atomicAdd(&p.shist[k >> GVC_SAMPLE_SHIFT], 1u);
                    kmax = max(kmax, k);
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    if (lane == 0 && kmax)
        atomicMax(&p.st->max_key, kmax);
}

// Block-wide exclusive SUFFIX sums of a histogram: out[b] = sum_{b' > b} h[b'].
// 1024 threads, nb a multiple of 1024; scratch holds 1024 u64.
template <int NB>
__device__ void suffix_counts(const uint32_t *h, unsigned long long *out, unsigned long long *scratch)
{
    constexpr int PER = NB / 1024;
    const int t = threadIdx.x;
    unsigned long long local = 0;
    for (int i = 0; i < PER; i++)
        local += h[t * PER + i];
    scratch[t] = local;
    __syncthreads();
    // inclusive suffix scan over scratch (Hillis-Steele, 10 steps)
    for (int o = 1; o < 1024; o <<= 1) {
        unsigned long long v = (t + o < 1024) ? scratch[t + o] : 0;
        __syncthreads();
        scratch[t] += v;
        __syncthreads();
    }
    unsigned long long acc = (t + 1 < 1024) ? scratch[t + 1] : 0;  // bins beyond my range
    for (int i = PER - 1; i >= 0; i--) {
        out[t * PER + i] = acc;
        acc += h[t * PER + i];
    }
    __syncthreads();
}

// Chooses key_est (a lower bound for the k_0-th largest key, w.h.p.) and the
// level-0 bin shift.  Magnitude keys: from the sample histogram.  Hash keys:
// from the binomial tail (host-computed).
__global__ void __launch_bounds__(1024) k_sample_resolve(Plan p)
{
    __shared__ unsigned long long scratch[1024];
    __shared__ unsigned long long suf_chunk[1024];
    SelState *st = p.st;
    if (p.keymode == KEY_HASH) {
        if (threadIdx.x == 0) {
            uint32_t est = p.force_exact ? 0u : p.hash_key_est;
            st->key_est = est;
            uint64_t span = (1ull << 32) - est;
            int sh = bitlen64(span - 1) - 12;
            st->shift0 = sh < 0 ? 0 : sh;
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
    // per-thread chunk of 64 bins; suffix over chunks
    const int t = threadIdx.x;
    unsigned long long local = 0;
    for (int i = 0; i < 64; i++)
        local += p.shist[t * 64 + i];
    scratch[t] = local;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        unsigned long long v = (t + o < 1024) ? scratch[t + o] : 0;
        __syncthreads();
        scratch[t] += v;
        __syncthreads();
    }
    suf_chunk[t] = (t + 1 < 1024) ? scratch[t + 1] : 0;
    __syncthreads();
    const unsigned long long target = p.s_target;
    const unsigned long long total = scratch[0];
    if (t == 0 && total < target) {  // too few sampled values (e.g. NaN-only): exact path
        st->key_est = 0;
        st->shift0 = 19;
    }
    if (total >= target) {
        unsigned long long acc = suf_chunk[t];
        for (int i = 63; i >= 0; i--) {
            uint32_t c = p.shist[t * 64 + i];
            if (acc < target && acc + c >= target) {
                uint32_t b = (uint32_t)(t * 64 + i);
                uint32_t est = b << GVC_SAMPLE_SHIFT;
                st->key_est = est;
                uint32_t mk = st->max_key;
                uint64_t span = mk > est ? (uint64_t)(mk - est) : 0;
                int sh = bitlen64(span) - 12;
                st->shift0 = sh < 0 ? 0 : sh;
            }
            acc += c;
        }
    }
}

// ----------------------------------------------------------------- collect
// Candidate compaction for 4 values of one lane in lane-major index order.
template <int KM>
__device__ __forceinline__ void push4(const Plan &p, const float (&v)[4], uint32_t pos0, int valid,
                                      uint32_t key_est, int shift0, uint32_t *h, float *cval,
                                      uint32_t *cidx, uint32_t &ccount, uint32_t &nan_any)
{
    uint32_t key[4];
    bool pr[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        key[c] = cand_key<KM>(p, v[c], pos0 + c);
        pr[c] = (c < valid) && key[c] >= key_est;
        if (KM == KEY_MAG && c < valid && key[c] > 0x7f800000u)
            nan_any = 1;
    }
    const uint32_t lt = lanemask_lt();
    uint32_t m0 = __ballot_sync(0xffffffffu, pr[0]);
    uint32_t m1 = __ballot_sync(0xffffffffu, pr[1]);
    uint32_t m2 = __ballot_sync(0xffffffffu, pr[2]);
    uint32_t m3 = __ballot_sync(0xffffffffu, pr[3]);
    uint32_t any = m0 | m1 | m2 | m3;
    if (any == 0)
        return;
    uint32_t o = ccount + __popc(m0 & lt) + __popc(m1 & lt) + __popc(m2 & lt) + __popc(m3 & lt);
#pragma unroll
    for (int c = 0; c < 4; c++) {
        if (pr[c]) {
            cval[o] = v[c];
            cidx[o] = pos0 + c;
            uint32_t bin = (key[c] - key_est) >> shift0;
            atomicAdd(&h[bin < GVC_H0_BINS ? bin : GVC_H0_BINS - 1], 1u);
            o++;
        }
    }
    ccount += __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3);
}

// One warp per segment.  EF: v = fl32(g + r) written back over r (the only
// full-size write of the step); !EF: v read from `src`.  REFILL re-collects
// from the already-written g_ef with key_est = 0 (exactness fallback).
template <int KM, bool EF>
__global__ void __launch_bounds__(GVC_THREADS) k_collect(Plan p, int refill)
{
    __shared__ uint32_t h[GVC_H0_BINS];
    if (refill && !p.st->fallback)
        return;
    for (int i = threadIdx.x; i < GVC_H0_BINS; i += GVC_THREADS)
        h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + (threadIdx.x >> 5);
    const uint32_t key_est = refill ? 0u : p.st->key_est;
    const int shift0 = refill ? (KM == KEY_MAG ? 19 : 20) : p.st->shift0;
    const bool do_ef = EF && !refill;
    const float *src = (EF ? (refill ? p.resid : p.g) : p.values);
    if (seg < p.S) {
        const uint64_t beg = (uint64_t)seg * p.seg_len;
        const uint64_t end = min(p.n, beg + p.seg_len);
        float *cval = p.cand_val + beg;
        uint32_t *cidx = p.cand_idx + beg;
        uint32_t ccount = 0, nan_any = 0;
        double nacc = 0.0;
        uint64_t i = beg;
        for (; i + GVC_SEG_QUANTUM <= end; i += GVC_SEG_QUANTUM) {
            float4 a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
                a[u] = ld_stream(reinterpret_cast<const float4 *>(src + i + u * 128) + lane);
            if (do_ef) {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    b[u] = ld_stream(reinterpret_cast<const float4 *>(p.resid + i + u * 128) + lane);
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    a[u].x = __fadd_rn(a[u].x, b[u].x);
                    a[u].y = __fadd_rn(a[u].y, b[u].y);
                    a[u].z = __fadd_rn(a[u].z, b[u].z);
                    a[u].w = __fadd_rn(a[u].w, b[u].w);
                    st_stream(reinterpret_cast<float4 *>(p.resid + i + u * 128) + lane, a[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                float v[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
                if (!refill) {
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        nacc = __fma_rn((double)v[c], (double)v[c], nacc);
                }
                push4<KM>(p, v, (uint32_t)(i + u * 128 + lane * 4), 4, key_est, shift0, h, cval, cidx,
                          ccount, nan_any);
            }
        }
        // tail: one value per lane, lane-major order preserved
        for (; i < end; i += 32) {
            uint64_t t = i + lane;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            int valid = t < end ? 1 : 0;
            if (valid) {
                float x = src[t];
                if (do_ef) {
                    x = __fadd_rn(x, p.resid[t]);
                    p.resid[t] = x;
                }
                v[0] = x;
                if (!refill)
                    nacc = __fma_rn((double)x, (double)x, nacc);
            }
            push4<KM>(p, v, (uint32_t)t, valid, key_est, shift0, h, cval, cidx, ccount, nan_any);
        }
        nacc = warp_sum_f64(nacc);
        nan_any = __any_sync(0xffffffffu, nan_any);
        if (lane == 0) {
            p.seg_cnt[seg] = ccount;
            if (!refill)
                p.norm_part[seg] = nacc;
            if (nan_any)
                atomicOr(&p.st->nan_flag, 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < GVC_H0_BINS; i += GVC_THREADS)
        if (h[i])
            atomicAdd(&p.hist0[i], h[i]);
}

// ----------------------------------------------------------------- resolve
__device__ void set_jstate(JState &js, unsigned long long lo, unsigned long long hi,
                           unsigned long long above, unsigned long long need)
{
    js.lo = lo;
    js.hi = hi;
    js.above = above;
    js.need = need;
    unsigned long long w = hi - lo;
    int sh = bitlen64(w - 1) - 12;
    js.shift = sh < 0 ? 0 : sh;
    js.resolved = (w == 1);
}

// Level 0: candidate total, fallback decision, first interval per ladder entry.
__global__ void __launch_bounds__(1024) k_resolve0(Plan p, int pass)
{
    __shared__ unsigned long long scratch[1024];
    __shared__ unsigned long long suf[GVC_H0_BINS];
    SelState *st = p.st;
    if (pass == 1 && !st->fallback)
        return;
    suffix_counts<GVC_H0_BINS>(p.hist0, suf, scratch);
    const unsigned long long total = suf[0] + p.hist0[0];
    if (pass == 0 && total < p.ks[0]) {
        // estimate overshot: zero the histogram for the exact re-collect
        for (int i = threadIdx.x; i < GVC_H0_BINS; i += 1024)
            p.hist0[i] = 0;
        if (threadIdx.x == 0)
            st->fallback = 1;
        return;
    }
    const uint32_t key_est = pass == 1 ? 0u : st->key_est;
    const int shift0 = pass == 1 ? (p.keymode == KEY_MAG ? 19 : 20) : st->shift0;
    if (pass == 1 && threadIdx.x == 0) {
        st->key_est = key_est;
        st->shift0 = shift0;
    }
    for (int b = threadIdx.x; b < GVC_H0_BINS; b += 1024) {
        unsigned long long above = suf[b], c = p.hist0[b];
        for (int j = 0; j < p.n_ks; j++) {
            unsigned long long k = p.ks[j];
            if (above < k && above + c >= k) {
                unsigned long long lo = (unsigned long long)key_est + ((unsigned long long)b << shift0);
                unsigned long long hi = (b == GVC_H0_BINS - 1) ? (1ull << 32)
                                                                : lo + (1ull << shift0);
                if (hi > (1ull << 32))
                    hi = 1ull << 32;
                set_jstate(st->js[j], lo, hi, above, k - above);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        st->cand_total = total;
        uint32_t pend = 0;
        for (int j = 0; j < p.n_ks; j++)
            pend += !st->js[j].resolved;
        st->pending = pend;
    }
}

// Refinement histogram: candidates whose key lies in an unresolved interval.
template <int KM>
__global__ void __launch_bounds__(GVC_THREADS) k_level_hist(Plan p)
{
    __shared__ JState js[GVC_MAX_LADDER];
    SelState *st = p.st;
    if (st->pending == 0)
        return;
    if (threadIdx.x < p.n_ks)
        js[threadIdx.x] = st->js[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + (threadIdx.x >> 5);
    if (seg >= p.S)
        return;
    const uint64_t beg = (uint64_t)seg * p.seg_len;
    const uint32_t cnt = p.seg_cnt[seg];
    for (uint32_t t = lane; t < cnt; t += 32) {
        uint32_t key = KM == KEY_MAG ? mag_key(p.cand_val[beg + t]) : cand_key<KM>(p, 0.f, p.cand_idx[beg + t]);
        for (int j = 0; j < p.n_ks; j++) {
            if (!js[j].resolved && key >= js[j].lo && key < js[j].hi)
                atomicAdd(&p.histl[j * GVC_HL_BINS + (uint32_t)((key - js[j].lo) >> js[j].shift)], 1u);
        }
    }
}

__global__ void __launch_bounds__(1024) k_level_resolve(Plan p)
{
    __shared__ unsigned long long scratch[1024];
    __shared__ unsigned long long suf[GVC_HL_BINS];
    SelState *st = p.st;
    if (st->pending == 0)
        return;
    for (int j = 0; j < p.n_ks; j++) {
        if (st->js[j].resolved)
            continue;  // uniform across the block
        uint32_t *h = p.histl + j * GVC_HL_BINS;
        suffix_counts<GVC_HL_BINS>(h, suf, scratch);
        JState cur = st->js[j];
        __syncthreads();
        for (int b = threadIdx.x; b < GVC_HL_BINS; b += 1024) {
            unsigned long long above = suf[b], c = h[b];
            if (above < cur.need && above + c >= cur.need) {
                unsigned long long lo = cur.lo + ((unsigned long long)b << cur.shift);
                unsigned long long hi = lo + (1ull << cur.shift);
                if (hi > cur.hi)
                    hi = cur.hi;
                set_jstate(st->js[j], lo, hi, cur.above + above, cur.need - above);
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < GVC_HL_BINS; b += 1024)
            h[b] = 0;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        uint32_t pend = 0;
        for (int j = 0; j < p.n_ks; j++)
            pend += !st->js[j].resolved;
        st->pending = pend;
    }
}

// ------------------------------------------------------------------- final
// Per segment: band counts / energies (band = #{j : T_j < key}) and, per
// ladder entry, the count and energy of keys equal to T_j.  fp64 sums are
// per-lane sequential then a fixed xor-tree: bit-reproducible.
template <int KM, int NB>
__global__ void __launch_bounds__(GVC_THREADS) k_final(Plan p)
{
    __shared__ uint32_t Ts[GVC_MAX_LADDER];
    SelState *st = p.st;
    if (threadIdx.x < GVC_MAX_LADDER)
        Ts[threadIdx.x] = threadIdx.x < p.n_ks ? (uint32_t)st->js[threadIdx.x].lo : 0xffffffffu;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + (threadIdx.x >> 5);
    if (seg >= p.S)
        return;
    uint32_t T[NB];
#pragma unroll
    for (int j = 0; j < NB; j++)
        T[j] = Ts[j];
    const int nks = p.n_ks;
    uint32_t bc[NB], tc[NB];
    double be[NB], ba[NB], te[NB], ta[NB];
#pragma unroll
    for (int j = 0; j < NB; j++) {
        bc[j] = tc[j] = 0;
        be[j] = ba[j] = te[j] = ta[j] = 0.0;
    }
    const uint64_t beg = (uint64_t)seg * p.seg_len;
    const uint32_t cnt = p.seg_cnt[seg];
    for (uint32_t t = lane; t < cnt; t += 32) {
        float v = p.cand_val[beg + t];
        uint32_t key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, p.cand_idx[beg + t]);
        double v2 = (double)v * (double)v;
        double av = fabs((double)v);
        int band = 0;
#pragma unroll
        for (int j = 0; j < NB; j++)
            band += (j < nks && T[j] < key);
#pragma unroll
        for (int j = 0; j < NB; j++) {
            if (band == j + 1) {
                bc[j]++;
                be[j] += v2;
                ba[j] += av;
            }
            if (j < nks && key == T[j]) {
                tc[j]++;
                te[j] += v2;
                ta[j] += av;
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
        double e1 = warp_sum_f64(be[j]), a1 = warp_sum_f64(ba[j]);
        double e2 = warp_sum_f64(te[j]), a2 = warp_sum_f64(ta[j]);
        if (lane == 0 && j < nks) {
            size_t o = (size_t)j * GVC_SEG_MAX + seg;
            p.band_cnt[o] = c1;
            p.band_e2[o] = e1;
            p.band_ab[o] = a1;
            p.tie_cnt[o] = c2;
            p.tie_e2[o] = e2;
            p.tie_ab[o] = a2;
        }
    }
}

// Block (1024 threads) fixed-order sum of S doubles.
__device__ double block_sum_f64(const double *x, uint32_t S, double *red)
{
    double acc = 0.0;
    for (uint32_t s = threadIdx.x; s < S; s += 1024)
        acc += x[s];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    double r = red[0];
    __syncthreads();
    return r;
}

// Block exclusive scan of S u32 values (per-thread contiguous chunks).
// Writes out[s] = sum_{s' < s} in[s'] and returns the total.
__device__ unsigned long long block_excl_scan(const uint32_t *in, uint32_t *out, uint32_t S,
                                              unsigned long long *scratch)
{
    const uint32_t per = (S + 1023) / 1024;
    const uint32_t b0 = threadIdx.x * per, b1 = min(S, b0 + per);
    unsigned long long local = 0;
    for (uint32_t s = b0; s < b1; s++)
        local += in[s];
    scratch[threadIdx.x] = local;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        unsigned long long v = threadIdx.x >= o ? scratch[threadIdx.x - o] : 0;
        __syncthreads();
        scratch[threadIdx.x] += v;
        __syncthreads();
    }
    unsigned long long acc = scratch[threadIdx.x] - local;
    for (uint32_t s = b0; s < b1; s++) {
        uint32_t v = in[s];
        out[s] = (uint32_t)acc;
        acc += v;
    }
    unsigned long long total = scratch[1023];
    __syncthreads();
    return total;
}

// Gains, tie cut and output offsets for every ladder entry (one block).
template <int KM>
__global__ void __launch_bounds__(1024) k_finish(Plan p)
{
    __shared__ double red[1024];
    __shared__ unsigned long long scratch[1024];
    __shared__ double BE[GVC_MAX_LADDER], BA[GVC_MAX_LADDER];
    __shared__ unsigned long long BC[GVC_MAX_LADDER];
    __shared__ uint32_t part_seg;
    __shared__ unsigned long long part_take;
    SelState *st = p.st;
    gvc_select_result *res = p.res;
    const uint32_t S = p.S;
    const int nks = p.n_ks;

    double norm = block_sum_f64(p.norm_part, S, red);
    for (int b = 0; b < nks; b++) {
        double e = block_sum_f64(p.band_e2 + (size_t)b * GVC_SEG_MAX, S, red);
        double a = block_sum_f64(p.band_ab + (size_t)b * GVC_SEG_MAX, S, red);
        if (threadIdx.x == 0) {
            BE[b] = e;
            BA[b] = a;
        }
    }
    for (int b = 0; b < nks; b++) {
        unsigned long long c = 0;
        for (uint32_t s = threadIdx.x; s < S; s += 1024)
            c += p.band_cnt[(size_t)b * GVC_SEG_MAX + s];
        scratch[threadIdx.x] = c;
        __syncthreads();
        for (int o = 512; o > 0; o >>= 1) {
            if (threadIdx.x < o)
                scratch[threadIdx.x] += scratch[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0)
            BC[b] = scratch[0];
        __syncthreads();
    }

    for (int j = 0; j < nks; j++) {
        const uint32_t T = (uint32_t)st->js[j].lo;
        const unsigned long long q = st->js[j].need;
        // tie cut: exclusive prefix of per-segment tie counts
        uint32_t *ties = p.tie_cnt + (size_t)j * GVC_SEG_MAX;
        uint32_t *take = p.seg_take + (size_t)j * GVC_SEG_MAX;
        block_excl_scan(ties, take, S, scratch);  // take[] temporarily = tie prefix
        if (threadIdx.x == 0)
            part_seg = 0xffffffffu;
        __syncthreads();
        for (uint32_t s = threadIdx.x; s < S; s += 1024) {
            unsigned long long before = take[s], c = ties[s];
            unsigned long long tk = before >= q ? 0 : (q - before < c ? q - before : c);
            take[s] = (uint32_t)tk;
            if (tk > 0 && tk < c) {
                part_seg = s;
                part_take = tk;
            }
        }
        __syncthreads();
        // energy of the fully-taken tie segments (fixed order)
        double te = 0.0, ta = 0.0;
        for (uint32_t s = threadIdx.x; s < S; s += 1024) {
            size_t o = (size_t)j * GVC_SEG_MAX + s;
            if (take[s] == p.tie_cnt[o] && take[s] > 0) {
                te += p.tie_e2[o];
                ta += p.tie_ab[o];
            }
        }
        // the one partially-taken segment: first `part_take` ties in index order
        if (part_seg != 0xffffffffu) {
            const uint32_t s = part_seg;
            const uint64_t beg = (uint64_t)s * p.seg_len;
            const uint32_t cnt = p.seg_cnt[s];
            unsigned long long seen = 0;
            for (uint32_t base = 0; base < cnt; base += 1024) {
                uint32_t t = base + threadIdx.x;
                bool tie = false;
                float v = 0.f;
                if (t < cnt) {
                    v = p.cand_val[beg + t];
                    uint32_t key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, p.cand_idx[beg + t]);
                    tie = key == T;
                }
                // block exclusive rank of ties
                scratch[threadIdx.x] = tie;
                __syncthreads();
                for (int o = 1; o < 1024; o <<= 1) {
                    unsigned long long x = threadIdx.x >= o ? scratch[threadIdx.x - o] : 0;
                    __syncthreads();
                    scratch[threadIdx.x] += x;
                    __syncthreads();
                }
                unsigned long long rank = seen + scratch[threadIdx.x] - tie;
                if (tie && rank < part_take) {
                    te += (double)v * (double)v;
                    ta += fabs((double)v);
                }
                seen += scratch[1023];
                __syncthreads();
            }
        }
        red[threadIdx.x] = te;
        __syncthreads();
        for (int o = 512; o > 0; o >>= 1) {
            if (threadIdx.x < o)
                red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        double tie_e = red[0];
        __syncthreads();
        red[threadIdx.x] = ta;
        __syncthreads();
        for (int o = 512; o > 0; o >>= 1) {
            if (threadIdx.x < o)
                red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        double tie_a = red[0];
        __syncthreads();
        // output offsets: selected per segment = sum_{b >= j} band_cnt + take
        uint32_t *off = p.seg_off + (size_t)j * GVC_SEG_MAX;
        for (uint32_t s = threadIdx.x; s < S; s += 1024) {
            uint32_t sel = take[s];
            for (int b = j; b < nks; b++)
                sel += p.band_cnt[(size_t)b * GVC_SEG_MAX + s];
            off[s] = sel;  // counts, scanned in place below
        }
        __syncthreads();
        unsigned long long total_sel = block_excl_scan(off, off, S, scratch);
        if (threadIdx.x == 0) {
            double e_above = 0.0, a_above = 0.0;
            unsigned long long c_above = 0;
            for (int b = j; b < nks; b++) {
                e_above += BE[b];
                a_above += BA[b];
                c_above += BC[b];
            }
            const unsigned long long k = p.ks[j];
            double A = a_above + tie_a;
            double E = e_above + tie_e;
            float m = (float)(A / (double)k);
            unsigned long long nnz = k - ((KM == KEY_MAG && T == 0u) ? q : 0ull);
            if (p.kind == GVC_REDSYNC)
                E = (double)nnz * ((double)m * (double)m);
            st->redsync_mean[j] = m;
            res->kept_sq[j] = E;
            res->kept_abs[j] = A;
            res->threshold_key[j] = T;
            res->tie_quota[j] = q;
            res->redsync_mean[j] = m;
            res->kept_count[j] = total_sel;
            res->kept_nonzero[j] = nnz;
            if (c_above + q != k || total_sel != k)
                atomicOr(&st->nan_flag, 2u);  // internal consistency failure
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        res->ef_norm_sq = norm;
        res->candidates = st->cand_total;
        res->status = (st->nan_flag & 1u) ? GVC_ERR_NAN : ((st->nan_flag & 2u) ? GVC_ERR_STATE : GVC_OK);
        res->fallback_used = (int)st->fallback;
    }
}

// -------------------------------------------------------------------- emit
template <int KM>
__global__ void __launch_bounds__(GVC_THREADS) k_emit(Plan p, int j, const uint32_t *idx_map,
                                                      uint32_t *out_idx, float *out_val, float *resid)
{
    const int lane = threadIdx.x & 31;
    const uint32_t seg = blockIdx.x * GVC_WARPS_PER_BLOCK + (threadIdx.x >> 5);
    if (seg >= p.S)
        return;
    const SelState *st = p.st;
    const uint32_t T = (uint32_t)st->js[j].lo;
    const float m = st->redsync_mean[j];
    const bool redsync = p.kind == GVC_REDSYNC;
    const size_t o = (size_t)j * GVC_SEG_MAX + seg;
    const uint32_t take = p.seg_take[o];
    uint32_t out = p.seg_off[o];
    const uint64_t beg = (uint64_t)seg * p.seg_len;
    const uint32_t cnt = p.seg_cnt[seg];
    const uint32_t lt = lanemask_lt();
    uint32_t ties_seen = 0;
    double e2 = 0.0, ab = 0.0;
    for (uint32_t base = 0; base < cnt; base += 32) {
        uint32_t t = base + lane;
        bool valid = t < cnt;
        float v = 0.f;
        uint32_t pos = 0, key = 0;
        if (valid) {
            v = p.cand_val[beg + t];
            pos = p.cand_idx[beg + t];
            key = KM == KEY_MAG ? mag_key(v) : cand_key<KM>(p, v, pos);
        }
        bool tie = valid && key == T;
        uint32_t tb = __ballot_sync(0xffffffffu, tie);
        bool sel = valid && (key > T || (tie && ties_seen + __popc(tb & lt) < take));
        uint32_t sb = __ballot_sync(0xffffffffu, sel);
        if (sel) {
            uint32_t w = out + __popc(sb & lt);
            float sv = v;
            if (redsync) {
                float sg = v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f);
                sv = __fmul_rn(sg, m);
            }
            uint32_t gi = idx_map ? idx_map[pos] : pos;
            out_idx[w] = gi;
            out_val[w] = sv;
            if (resid) {
                // level-1 emits: the candidate value IS g_ef; a second-level emit
                // (idx_map) carries level-1 SENT values, so read g_ef back
                float ef = idx_map ? resid[gi] : v;
                resid[gi] = __fsub_rn(ef, sv);
            }
            e2 += (double)sv * (double)sv;
            ab += fabs((double)sv);
        }
        ties_seen += __popc(tb);
        out += __popc(sb);
    }
    e2 = warp_sum_f64(e2);
    ab = warp_sum_f64(ab);
    if (lane == 0) {
        p.seg_emit[seg] = e2;
        p.seg_emit[GVC_SEG_MAX + seg] = ab;
    }
}

__global__ void __launch_bounds__(1024) k_emit_finish(Plan p, double *stats)
{
    __shared__ double red[1024];
    double e = block_sum_f64(p.seg_emit, p.S, red);
    double a = block_sum_f64(p.seg_emit + GVC_SEG_MAX, p.S, red);
    if (threadIdx.x == 0) {
        stats[0] = e;
        stats[1] = a;
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

static int nb_for(int n_ks)
{
    return n_ks <= 1 ? 1 : n_ks <= 2 ? 2 : n_ks <= 4 ? 4 : n_ks <= 8 ? 8 : 16;
}

template <int KM>
static void launch_final(const Plan &p, cudaStream_t s, int blocks)
{
    switch (nb_for(p.n_ks)) {
    case 1: k_final<KM, 1><<<blocks, GVC_THREADS, 0, s>>>(p); break;
    case 2: k_final<KM, 2><<<blocks, GVC_THREADS, 0, s>>>(p); break;
    case 4: k_final<KM, 4><<<blocks, GVC_THREADS, 0, s>>>(p); break;
    case 8: k_final<KM, 8><<<blocks, GVC_THREADS, 0, s>>>(p); break;
    default: k_final<KM, 16><<<blocks, GVC_THREADS, 0, s>>>(p); break;
    }
}

template <int KM>
static void launch_pipeline(Plan &p, cudaStream_t s)
{
    ProfScope all(PROF_SELECT, s);
    const int blocks = (int)((p.S + GVC_WARPS_PER_BLOCK - 1) / GVC_WARPS_PER_BLOCK);
    int launches = 0;
    if (KM == KEY_MAG && !p.force_exact && p.s_target > 0) {
        uint64_t wb = (p.s_chunks + GVC_WARPS_PER_BLOCK - 1) / GVC_WARPS_PER_BLOCK;
        int sb = (int)(wb < 2048 ? (wb ? wb : 1) : 2048);
        k_sample<<<sb, GVC_THREADS, 0, s>>>(p);
        launches++;
    }
    k_sample_resolve<<<1, 1024, 0, s>>>(p);
    {
        ProfScope pc(PROF_COLLECT, s);
        if (p.ef)
            k_collect<KM, true><<<blocks, GVC_THREADS, 0, s>>>(p, 0);
        else
            k_collect<KM, false><<<blocks, GVC_THREADS, 0, s>>>(p, 0);
    }
    k_resolve0<<<1, 1024, 0, s>>>(p, 0);
    if (p.ef)
        k_collect<KM, true><<<blocks, GVC_THREADS, 0, s>>>(p, 1);
    else
        k_collect<KM, false><<<blocks, GVC_THREADS, 0, s>>>(p, 1);
    k_resolve0<<<1, 1024, 0, s>>>(p, 1);
    launches += 5;
    for (int l = 0; l < GVC_MAX_LEVELS; l++) {
        k_level_hist<KM><<<blocks, GVC_THREADS, 0, s>>>(p);
        k_level_resolve<<<1, 1024, 0, s>>>(p);
        launches += 2;
    }
    launch_final<KM>(p, s, blocks);
    k_finish<KM><<<1, 1024, 0, s>>>(p);
    count_launches(launches + 2);
}

int select_run(const gvc_select_args *a, void *ws, size_t ws_bytes, gvc_select_result *res,
               cudaStream_t s)
{
    Plan p;
    memset(&p, 0, sizeof(p));
    size_t need = carve(&p, (char *)ws, a->n);
    if (ws_bytes < need)
        return set_error(GVC_ERR_WORKSPACE, "select workspace too small: %zu < %zu", ws_bytes, need);
    p.n = a->n;
    p.n_ks = a->n_ks;
    p.kind = a->kind;
    p.keymode = a->kind == GVC_RANDOMK ? KEY_HASH : KEY_MAG;
    p.ef = a->g_dev != nullptr;
    p.force_exact = a->force_exact;
    p.values = a->values_dev;
    p.g = a->g_dev;
    p.resid = a->resid_dev;
    p.seed = a->seed;
    p.stream = a->rng_stream;
    p.pos_base = a->pos_base;
    for (int j = 0; j < a->n_ks; j++)
        p.ks[j] = a->ks[j];
    p.res = res;
    const uint64_t n = a->n, k0 = a->ks[0];
    if (p.keymode == KEY_MAG) {
        // sample ~n/64 values in 128-value chunks (everything when n is small)
        uint64_t want = n <= 65536 ? n : (n / 64 > 65536 ? n / 64 : 65536);
        uint64_t chunks = (want + 127) / 128;
        uint64_t stride = n / chunks;
        stride &= ~(uint64_t)3;
        if (stride < 128)
            stride = 128;
        chunks = (n + stride - 1) / stride;
        uint64_t sampled = 0;
        {  // exact sample size: full chunks plus the clipped tail chunk
            uint64_t last = (chunks - 1) * stride;
            sampled = (chunks - 1) * 128 + (n - last < 128 ? n - last : 128);
        }
        p.s_chunks = chunks;
        p.s_stride = stride;
        if (sampled >= n) {
            p.s_target = k0;  // the sample is the whole vector: exact bin
        } else {
            double mu = (double)k0 * (double)sampled / (double)n;
            double t = mu * 1.02 + 5.0 * sqrt(mu) + 32.0;
            p.s_target = t >= (double)sampled ? 0 : (uint64_t)ceil(t);
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
    cudaMemsetAsync(p.st, 0, sizeof(SelState), s);
    cudaMemsetAsync(p.hist0, 0, GVC_H0_BINS * 4, s);
    cudaMemsetAsync(p.histl, 0, GVC_MAX_LADDER * GVC_HL_BINS * 4, s);
    if (p.keymode == KEY_MAG)
        cudaMemsetAsync(p.shist, 0, GVC_SAMPLE_BINS * 4, s);
    if (p.keymode == KEY_MAG)
        launch_pipeline<KEY_MAG>(p, s);
    else
        launch_pipeline<KEY_HASH>(p, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(GVC_ERR_CUDA, "select launch: %s", cudaGetErrorString(e));
    std::lock_guard<std::mutex> lk(g_mu);
    g_plans[ws] = p;
    return GVC_OK;
}

int emit_run(void *ws, size_t ws_bytes, int j, const uint32_t *idx_map, uint32_t *out_idx,
             float *out_val, float *resid, double *stats, cudaStream_t s)
{
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
    const int blocks = (int)((p.S + GVC_WARPS_PER_BLOCK - 1) / GVC_WARPS_PER_BLOCK);
    ProfScope pe(PROF_EMIT, s);
    count_launches(stats ? 2 : 1);
    if (p.keymode == KEY_MAG)
        k_emit<KEY_MAG><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid);
    else
        k_emit<KEY_HASH><<<blocks, GVC_THREADS, 0, s>>>(p, j, idx_map, out_idx, out_val, resid);
    if (stats)
        k_emit_finish<<<1, 1024, 0, s>>>(p, stats);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(GVC_ERR_CUDA, "emit launch: %s", cudaGetErrorString(e));
    return GVC_OK;
}

}  // namespace gvc
