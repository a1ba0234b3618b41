// gvc_segsel.cu -- layerwise compression as ONE segmented selection (sm_100a).
//
// compressors.compress(..., layerwise=True) (compressors.py:204-217) keeps
// k_s = keep_count(len_s, cf) entries of every layer segment s, chosen inside
// the segment by the compressor's rule (ties to the lower index), offsets
// them by the segment start and concatenates the segments in order.  A
// ResNet-101 gradient has ~300 segments; instead of one selection pipeline per
// segment, every segment is resolved at once:
//   * work items = (segment, chunk of <= SS_CHUNK values), one CTA each;
//   * 3 radix passes of 11 / 11 / 10 key bits, most significant first: every CTA
//     histograms the keys of its chunk that match its segment's resolved
//     prefix (2048 shared-memory bins, merged into the segment's global bins);
//     one warp per segment then picks the digit where the count from the top
//     reaches the segment's remaining rank -> after 3 passes each segment has
//     its exact threshold key T_s and tie quota q_s;
//   * counts per item (> T, == T), one CTA scans them into per-item output
//     offsets and tie quotas (the segments' outputs are contiguous and in
//     order, so one exclusive scan over the items gives every offset);
//   * an ordered compaction writes (global index, value) per item.
// Keys: 31-bit |v| (Top-k) or the Philox position hash of the global
// position (Random-k, the counter-based sampler with pos_base = segment start,
// DESIGN.md).  10 launches whatever the number of segments.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "gvc_common.cuh"
#include "gvc_internal.h"

namespace gvc {

#define SS_CHUNK 16384
#define SS_THREADS 256

struct SegState {
    uint32_t prefix;     // resolved key bits (most significant first)
    uint32_t all;        // k >= len: every value is kept
    unsigned long long need;  // rank still to take at/below the resolved prefix
};

struct SegPlan {
    const float *values;
    uint64_t n;
    int nseg, nitems, keymode;
    uint64_t seed, stream;
    const uint64_t *seg_lo;   // [nseg + 1] segment offsets
    const uint64_t *seg_k;    // [nseg]
    const uint32_t *item_seg;  // [nitems]
    const uint64_t *item_lo;   // [nitems] global start of the item
    const uint32_t *item_len;  // [nitems]
    SegState *seg;             // [nseg]
    uint32_t *hist;            // [SS_PASSES][nseg][SS_BINS]
    uint32_t *item_gt, *item_eq;  // [nitems]
    uint32_t *warp_gt, *warp_eq;  // [nitems][SS_THREADS / 32]: the same counts per k_ss_write warp slice
    uint32_t *item_take;          // [nitems] ties this item keeps
    unsigned long long *item_out; // [nitems] output offset
    unsigned long long *item_E;   // [nitems] exclusive scan of the == counts
    const uint32_t *seg_first;    // [nseg] first item of the segment
    uint32_t *status;             // bit 1: NaN
    // KEY_DGC (layerwise DGC): segment q's sampled threshold key is
    // dgc_seg[q].prefix (the sample selection's states); dgc_bits = the
    // samples' global position bitmap
    const SegState *dgc_seg;
    const uint32_t *dgc_bits;
    int thr_only;  // the sample selection: k = len resolves the minimum key too
};

// (the key mode is a template parameter of every pass: a runtime test per
// value cost the compaction pass ~20% of its issue slots)
template <int KM>
__device__ __forceinline__ uint32_t ss_key(const SegPlan &P, float v, uint64_t pos, uint32_t thr)
{
    if (KM == KEY_DGC) {  // the composite key of gvc_select's KEY_DGC, per segment
        const uint32_t m = mag_key(v);
        const bool hi = m >= thr || ((__ldg(P.dgc_bits + (pos >> 5)) >> (pos & 31)) & 1u);
        return hi ? (0x80000000u | m) : m;
    }
    return KM == KEY_HASH ? hash_key(pos, P.stream, P.seed) : mag_key(v);
}

template <int KM>
__device__ __forceinline__ uint32_t ss_thr(const SegPlan &P, uint32_t s)
{
    return KM == KEY_DGC ? P.dgc_seg[s].prefix : 0u;
}

// Radix digits, most significant first: 11 + 11 + 10 bits (3 passes; 8-bit
// digits took 4 passes of ~44 us each over a 44.5M gradient).
#define SS_PASSES 3
#define SS_BINS 2048
__host__ __device__ __forceinline__ int ss_shift(int d) { return d == 0 ? 21 : (d == 1 ? 10 : 0); }
__host__ __device__ __forceinline__ int ss_nbins(int d) { return d == 2 ? 1024 : 2048; }
__host__ __device__ __forceinline__ uint32_t ss_pmask(int d) { return d == 0 ? 0u : (d == 1 ? 0xffe00000u : 0xfffffc00u); }

// Pass d: histogram of digit d of the keys matching the segment's prefix.
// The item is read 16 bytes per load (scalar head and tail to the 16-byte
// boundary), four loads in flight per thread.
template <int KM>
__global__ void __launch_bounds__(SS_THREADS) k_ss_hist(SegPlan P, int d)
{
    __shared__ uint32_t h[SS_BINS];
    const int it = blockIdx.x;
    const uint32_t s = P.item_seg[it];
    const SegState st = P.seg[s];
    const int nb = ss_nbins(d);
    for (int i = threadIdx.x; i < nb; i += SS_THREADS)
        h[i] = 0;
    __syncthreads();
    if (!st.all) {
        const uint64_t lo = P.item_lo[it];
        const uint32_t len = P.item_len[it];
        const int shift = ss_shift(d);
        const uint32_t dmask = (uint32_t)nb - 1u;
        const uint32_t pmask = ss_pmask(d);
        const uint32_t thr = ss_thr<KM>(P, s);
        uint32_t nan = 0;
        auto one = [&](float v, uint64_t pos) {
            const uint32_t key = ss_key<KM>(P, v, pos, thr);
            if (d == 0 && KM != KEY_HASH)
                nan |= (key & 0x7fffffffu) > 0x7f800000u;
            if ((key & pmask) == st.prefix)
                atomicAdd(&h[(key >> shift) & dmask], 1u);
        };
        // 16-byte aligned body [head, head + 4 * nv)
        uint32_t head = (uint32_t)((4 - ((reinterpret_cast<uintptr_t>(P.values + lo) >> 2) & 3)) & 3);
        if (head > len)
            head = len;
        const uint32_t nv = (len - head) >> 2;
        for (uint32_t i = threadIdx.x; i < head; i += SS_THREADS)
            one(P.values[lo + i], lo + i);
        const float4 *v4 = reinterpret_cast<const float4 *>(P.values + lo + head);
        for (uint32_t b = threadIdx.x; b < nv; b += 4 * SS_THREADS) {
            float4 q[4];
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (b + u * SS_THREADS < nv)
                    q[u] = v4[b + u * SS_THREADS];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t e = b + u * SS_THREADS;
                if (e < nv) {
                    const uint64_t pos = lo + head + 4ull * e;
                    one(q[u].x, pos);
                    one(q[u].y, pos + 1);
                    one(q[u].z, pos + 2);
                    one(q[u].w, pos + 3);
                }
            }
        }
        for (uint32_t i = head + 4 * nv + threadIdx.x; i < len; i += SS_THREADS)
            one(P.values[lo + i], lo + i);
        if (d == 0 && __any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0)
            atomicOr(P.status, 1u);
    }
    __syncthreads();
    uint32_t *g = P.hist + ((size_t)d * P.nseg + s) * SS_BINS;
    for (int i = threadIdx.x; i < nb; i += SS_THREADS)
        if (h[i])
            atomicAdd(&g[i], h[i]);
}

// One CTA per segment: the digit where the count from the top reaches `need`
// (thread t holds nb / 256 consecutive descending digits; a block scan).
__global__ void __launch_bounds__(SS_THREADS) k_ss_resolve(SegPlan P, int d)
{
    __shared__ unsigned long long sh[33];
    const int s = blockIdx.x;
    SegState st = P.seg[s];
    if (st.all)
        return;  // (uniform over the block)
    const int nb = ss_nbins(d), per = nb / SS_THREADS;
    const uint32_t *g = P.hist + ((size_t)d * P.nseg + s) * SS_BINS;
    const int top = nb - 1 - per * (int)threadIdx.x;
    uint32_t c[SS_BINS / SS_THREADS];
    unsigned long long local = 0;
#pragma unroll
    for (int i = 0; i < SS_BINS / SS_THREADS; i++) {
        c[i] = i < per ? g[top - i] : 0u;
        local += c[i];
    }
    const unsigned long long before = block_excl_prefix(local, sh);
    const unsigned long long nd = st.need;
    if (before < nd && nd <= before + local) {
        unsigned long long acc = before;
        for (int i = 0; i < per; i++) {
            if (acc + c[i] >= nd) {
                st.prefix |= (uint32_t)(top - i) << ss_shift(d);
                st.need = nd - acc;
                P.seg[s] = st;
                break;
            }
            acc += c[i];
        }
    }
}

// The slice of an item that warp w of k_ss_count / k_ss_write owns (contiguous,
// a multiple of 32 values).
__device__ __forceinline__ void ss_slice(uint32_t len, int warp, uint32_t &wb, uint32_t &we)
{
    constexpr int W = SS_THREADS / 32;
    const uint32_t per = ((len + W - 1) / W + 31) & ~31u;
    wb = min(len, warp * per);
    we = min(len, wb + per);
}

// Segment states from the (cached) tables: nothing to copy per call.
__global__ void k_ss_init(SegPlan P)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= P.nseg)
        return;
    const uint64_t len = P.seg_lo[q + 1] - P.seg_lo[q], k = P.seg_k[q];
    SegState st;
    st.prefix = 0;
    st.all = len == 0 || (!P.thr_only && k >= len);
    st.need = k;
    P.seg[q] = st;
}

// Per item and per warp slice: keys above the threshold and equal to it.
template <int KM>
__global__ void __launch_bounds__(SS_THREADS) k_ss_count(SegPlan P)
{
    constexpr int W = SS_THREADS / 32;
    __shared__ uint32_t s_gt[W], s_eq[W];
    const int it = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const SegState st = P.seg[P.item_seg[it]];
    const uint32_t thr = ss_thr<KM>(P, P.item_seg[it]);
    const uint64_t lo = P.item_lo[it];
    uint32_t wb, we;
    ss_slice(P.item_len[it], warp, wb, we);
    uint32_t gt = 0, eq = 0;
    uint32_t base = st.all ? we : wb;  // (a segment kept whole is not read)
    for (; base + 256 <= we; base += 256) {  // full trips: 8 loads in flight per lane, no bounds checks
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; u++)
            v[u] = P.values[lo + base + u * 32 + lane];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const uint32_t key = ss_key<KM>(P, v[u], lo + base + u * 32 + lane, thr);
            gt += key > st.prefix;
            eq += key == st.prefix;
        }
    }
    for (uint32_t i = base + lane; i < we; i += 32) {
        const uint32_t key = ss_key<KM>(P, P.values[lo + i], lo + i, thr);
        gt += key > st.prefix;
        eq += key == st.prefix;
    }
    if (st.all && lane == 0)  // every value kept, no ties
        gt = we - wb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        gt += __shfl_xor_sync(0xffffffffu, gt, o);
        eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    if (lane == 0) {
        s_gt[warp] = gt;
        s_eq[warp] = eq;
        P.warp_gt[it * W + warp] = gt;
        P.warp_eq[it * W + warp] = eq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0, b = 0;
        for (int w = 0; w < W; w++) {
            a += s_gt[w];
            b += s_eq[w];
        }
        P.item_gt[it] = a;
        P.item_eq[it] = b;
    }
}

// One CTA: per item the ties it keeps (the first q_s ties of its segment in
// index order: E = exclusive scan of the == counts, ties before the item =
// E[item] - E[first item of the segment]) and its output offset (exclusive
// scan of the kept counts: the segments' outputs are contiguous and in order).
__global__ void __launch_bounds__(1024) k_ss_scan(SegPlan P)
{
    __shared__ unsigned long long sh[33];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (int base = 0; base < P.nitems; base += blockDim.x) {
        const int it = base + threadIdx.x;
        const unsigned long long eq = it < P.nitems ? P.item_eq[it] : 0ull;
        const unsigned long long c0 = carry;  // read before thread 0 advances it
        unsigned long long tot;
        const unsigned long long pre = block_excl_prefix(eq, sh, &tot) + c0;
        if (it < P.nitems)
            P.item_E[it] = pre;
        if (threadIdx.x == 0)
            carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        carry = 0;
    __syncthreads();
    for (int base = 0; base < P.nitems; base += blockDim.x) {
        const int it = base + threadIdx.x;
        const bool ok = it < P.nitems;
        unsigned long long kept = 0, tk = 0;
        if (ok) {
            const uint32_t s = P.item_seg[it];
            const SegState st = P.seg[s];
            const unsigned long long before = P.item_E[it] - P.item_E[P.seg_first[s]];
            const unsigned long long eq = P.item_eq[it];
            tk = st.all || before >= st.need ? 0ull : (st.need - before < eq ? st.need - before : eq);
            kept = P.item_gt[it] + tk;
        }
        const unsigned long long c0 = carry;
        unsigned long long tot;
        const unsigned long long out = block_excl_prefix(kept, sh, &tot) + c0;
        if (ok) {
            P.item_take[it] = (uint32_t)tk;
            P.item_out[it] = out;
        }
        if (threadIdx.x == 0)
            carry += tot;
        __syncthreads();
    }
}

// Ordered compaction of one item, warp-cooperative: warp w owns a contiguous
// slice of the item and walks it 32 values at a time (coalesced loads, ballot
// compaction, coalesced stores); kept = key > T, or key == T among the item's
// first `take` ties.  k_ss_count's per-slice counts give each warp its output
// offset and its first tie rank.  (Thread-contiguous slices read and wrote
// with a 256-byte stride across the warp: 368 us at 44.5M, measured; with a
// counting pass of its own, 117 us.)
template <int KM>
__global__ void __launch_bounds__(SS_THREADS) k_ss_write(SegPlan P, uint32_t *out_idx, float *out_val)
{
    constexpr int W = SS_THREADS / 32;
    const int it = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const SegState st = P.seg[P.item_seg[it]];
    const uint32_t thr = ss_thr<KM>(P, P.item_seg[it]);
    const uint32_t lo = (uint32_t)P.item_lo[it];  // n < 2^32 (gvc_segmented_select checks)
    const uint32_t take = P.item_take[it];
    uint32_t wb, we;
    ss_slice(P.item_len[it], warp, wb, we);
    // this warp's first tie rank and output offset within the item
    uint32_t ties = 0;
    uint32_t o = (uint32_t)P.item_out[it];
    for (int w = 0; w < warp; w++) {
        const uint32_t e = P.warp_eq[it * W + w];
        const uint32_t tk = ties >= take ? 0u : min(take - ties, e);
        o += P.warp_gt[it * W + w] + tk;
        ties += e;
    }
    const uint32_t lt = lanemask_lt();
    // kept entries go through a per-warp shared ring and leave 128 at a time
    // in whole 128-byte rows (stored straight from the ballot, every row of 32
    // values cost two partial-sector stores)
    __shared__ uint32_t ring_i[W][256];
    __shared__ float ring_v[W][256];
    uint32_t cnt = 0, flushed = 0;
    // the tie logic only where k_ss_count saw a tie in this warp's slice, the
    // bounds checks only in the last partial trip (the row loop is
    // instruction-bound: ~54 instructions per 32 values with both)
    const bool ties_here = !st.all && P.warp_eq[it * W + warp] != 0;
    auto trip = [&](uint32_t base, auto ties_t, auto full_t) {
        constexpr bool TIES = decltype(ties_t)::value, FULL = decltype(full_t)::value;
        // U rows of 32 loaded before any is compacted
        constexpr int U = 8;
        float v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t i = base + u * 32 + lane;
            v[u] = (FULL || i < we) ? P.values[lo + i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t i = base + u * 32 + lane;
            const bool ok = FULL || i < we;
            const uint32_t key = ss_key<KM>(P, v[u], lo + i, thr);
            bool keep = ok && (st.all || key > st.prefix);
            if (TIES) {
                const bool iseq = ok && !st.all && key == st.prefix;
                const uint32_t em = __ballot_sync(0xffffffffu, iseq);
                if (em) {  // warp-uniform: ties in this row (rare)
                    keep |= iseq && ties + __popc(em & lt) < take;
                    ties += __popc(em);
                }
            }
            const uint32_t km = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t r = (cnt + __popc(km & lt)) & 255u;
                ring_i[warp][r] = (uint32_t)(lo + i);
                ring_v[warp][r] = v[u];
            }
            cnt += __popc(km);
            if (cnt - flushed >= 128) {  // warp-uniform; the ring never holds more than 159
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const uint32_t e = flushed + q * 32 + lane;
                    out_idx[o + e] = ring_i[warp][e & 255u];
                    out_val[o + e] = ring_v[warp][e & 255u];
                }
                flushed += 128;
                __syncwarp();
            }
        }
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    uint32_t base = wb;
    if (ties_here) {
        for (; base + 256 <= we; base += 256)
            trip(base, T_(), T_());
        if (base < we)
            trip(base, T_(), F_());
    } else {
        for (; base + 256 <= we; base += 256)
            trip(base, F_(), T_());
        if (base < we)
            trip(base, F_(), F_());
    }
    __syncwarp();
    for (uint32_t e = flushed + lane; e < cnt; e += 32) {
        out_idx[o + e] = ring_i[warp][e & 255u];
        out_val[o + e] = ring_v[warp][e & 255u];
    }
}

// Layerwise Redsync (compressors.py:140-161, :187-189, per segment): the
// segmented Top-k support is Redsync's support; each segment's
// kept values become sign(v) * fl32(mean_f64 |v|) of that segment.  The kept
// values are cut into 16384-entry items (a segment's items are consecutive);
// pass 1 sums |v| per item (fixed-order block sum), pass 2 adds a segment's
// item sums in item order and substitutes the item's values -- every item in
// parallel, however unequal the segments (VGG16's first fc layer keeps 10.3M
// of the 13.8M).  A segment that keeps all its values passes through
// unchanged (compressors.py:172-173): it has no items.
#define RS_ITEM 16384
static size_t al256x(size_t x) { return (x + 255) & ~(size_t)255; }
struct RsPlan {
    float *vals;
    const uint32_t *item_seg;   // [nitems]
    const uint64_t *item_lo;    // [nitems] output range [lo, hi)
    const uint64_t *item_hi;
    const uint32_t *seg_first;  // [nseg] first item of the segment
    const uint32_t *seg_items;  // [nseg] its item count
    const uint64_t *seg_k;      // [nseg] kept count
    double *partial;            // [nitems]
};

__global__ void __launch_bounds__(256) k_rs_sum(RsPlan P)
{
    __shared__ double sh[33];
    const int it = blockIdx.x;
    double acc = 0.0;
    for (uint64_t i = P.item_lo[it] + threadIdx.x; i < P.item_hi[it]; i += blockDim.x)
        acc += fabs((double)P.vals[i]);
    const double s = block_sum_f64(acc, sh);
    if (threadIdx.x == 0)
        P.partial[it] = s;
}

__global__ void __launch_bounds__(256) k_rs_substitute(RsPlan P)
{
    __shared__ float s_m;
    const int it = blockIdx.x;
    const uint32_t q = P.item_seg[it];
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (uint32_t j = 0; j < P.seg_items[q]; j++)
            sum += P.partial[P.seg_first[q] + j];
        s_m = (float)(sum / (double)P.seg_k[q]);
    }
    __syncthreads();
    const float m = s_m;
    for (uint64_t i = P.item_lo[it] + threadIdx.x; i < P.item_hi[it]; i += blockDim.x) {
        const float v = P.vals[i];
        const float sg = v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f);
        P.vals[i] = __fmul_rn(sg, m);
    }
}

size_t seg_redsync_workspace_bytes(uint64_t total, int nseg)
{
    const uint64_t items = total / RS_ITEM + (uint64_t)nseg + 1;
    return al256x(items * 4) + al256x(items * 8) * 3 + al256x((size_t)nseg * 4) * 2 + al256x((size_t)nseg * 8) + 256;
}

int seg_redsync_run(float *vals, const uint64_t *out_off, const uint64_t *seg_len, int nseg, void *ws,
                    size_t ws_bytes, cudaStream_t s)
{
    std::vector<uint32_t> iseg, sfirst(nseg), sitems(nseg);
    std::vector<uint64_t> ilo, ihi, sk(nseg);
    for (int q = 0; q < nseg; q++) {
        const uint64_t a = out_off[q], b = out_off[q + 1];
        if (b < a)
            return set_error(GVC_ERR_ARG, "segmented redsync: segment %d output range reversed", q);
        sk[q] = b - a;
        sfirst[q] = (uint32_t)iseg.size();
        if (b - a == 0 || b - a >= seg_len[q])
            continue;  // identity pass-through
        for (uint64_t c = a; c < b; c += RS_ITEM) {
            iseg.push_back((uint32_t)q);
            ilo.push_back(c);
            ihi.push_back(c + RS_ITEM < b ? c + RS_ITEM : b);
        }
        sitems[q] = (uint32_t)iseg.size() - sfirst[q];
    }
    const int nitems = (int)iseg.size();
    if (nitems == 0)
        return GVC_OK;
    if (seg_redsync_workspace_bytes(out_off[nseg], nseg) > ws_bytes)
        return set_error(GVC_ERR_WORKSPACE, "segmented redsync workspace too small");
    char *w = (char *)ws;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *q = w + off;
        off += al256x(bytes);
        return q;
    };
    RsPlan P;
    P.vals = vals;
    P.item_seg = (const uint32_t *)take(nitems * 4);
    P.item_lo = (const uint64_t *)take(nitems * 8);
    P.item_hi = (const uint64_t *)take(nitems * 8);
    P.partial = (double *)take(nitems * 8);
    P.seg_first = (const uint32_t *)take(nseg * 4);
    P.seg_items = (const uint32_t *)take(nseg * 4);
    P.seg_k = (const uint64_t *)take(nseg * 8);
    // (pageable host vectors: the copies complete before the calls return)
    cudaMemcpyAsync((void *)P.item_seg, iseg.data(), nitems * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((void *)P.item_lo, ilo.data(), nitems * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((void *)P.item_hi, ihi.data(), nitems * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((void *)P.seg_first, sfirst.data(), nseg * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((void *)P.seg_items, sitems.data(), nseg * 4, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync((void *)P.seg_k, sk.data(), nseg * 8, cudaMemcpyHostToDevice, s);
    count_launches(2);
    k_rs_sum<<<nitems, 256, 0, s>>>(P);
    k_rs_substitute<<<nitems, 256, 0, s>>>(P);
    return GVC_OK;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t segsel_workspace_bytes(uint64_t n, int nseg)
{
    const uint64_t items = n / SS_CHUNK + (uint64_t)nseg + 1;
    return al256(nseg * sizeof(SegState)) + al256((size_t)SS_PASSES * nseg * SS_BINS * 4) + al256((nseg + 1) * 8) * 2 +
           al256(nseg * 4) + al256(items * 4) * 6 + al256(items * 8) * 3 + al256(items * (SS_THREADS / 32) * 4) * 2 +
           256;
}

// The work-item tables of a segment layout, uploaded once per (workspace,
// layout): a steady training loop calls with the same layer offsets and keep
// counts every step, and then only the launches are issued.
struct SegLayout {
    uint64_t n = 0;
    int kind = -1;
    std::vector<uint64_t> off, k;
    int nitems = 0;
};
static std::mutex g_seg_mu;
static std::unordered_map<const void *, SegLayout> g_seg_layouts;
static std::unordered_map<const void *, const void *> g_seg_alias;  // layerwise DGC: its sample selection's tables

void segsel_forget(const void *ws)
{
    std::lock_guard<std::mutex> lk(g_seg_mu);
    g_seg_layouts.erase(ws);
    auto a = g_seg_alias.find(ws);
    if (a != g_seg_alias.end()) {
        g_seg_layouts.erase(a->second);
        g_seg_alias.erase(a);
    }
}

// One segmented selection.  keymode KEY_MAG / KEY_HASH / KEY_DGC (dgc_seg,
// dgc_bits); thr_only: stop after the radix passes (each segment's threshold
// key left in its state; k = len resolves the minimum).
static int segsel_launch(int keymode, int thr_only, const SegState *dgc_seg, const uint32_t *dgc_bits,
                         const float *values, uint64_t n, const uint64_t *seg_off, const uint64_t *seg_k, int nseg,
                         uint64_t seed, uint64_t stream, uint32_t *out_idx, float *out_val, void *ws,
                         size_t ws_bytes, uint32_t *status, cudaStream_t s)
{
    const int kind = keymode * 2 + thr_only;  // (the cached layout's tag)
    for (int q = 0; q < nseg; q++) {
        const uint64_t a = seg_off[q], b = seg_off[q + 1];
        if (b < a || b > n)
            return set_error(GVC_ERR_ARG, "segmented select: segment %d [%llu, %llu) outside [0, %llu)", q,
                             (unsigned long long)a, (unsigned long long)b, (unsigned long long)n);
        if (b - a && seg_k[q] < 1 && !thr_only)
            return set_error(GVC_ERR_ARG, "segmented select: keep count 0 in segment %d", q);
    }
    if (segsel_workspace_bytes(n, nseg) > ws_bytes)
        return set_error(GVC_ERR_WORKSPACE, "segmented select workspace too small");
    std::lock_guard<std::mutex> lk(g_seg_mu);
    SegLayout &L = g_seg_layouts[ws];
    const bool same = L.n == n && L.kind == kind && (int)L.k.size() == nseg &&
                      std::equal(L.off.begin(), L.off.end(), seg_off) && std::equal(L.k.begin(), L.k.end(), seg_k);
    int nitems = L.nitems;
    std::vector<uint32_t> iseg, ilen, sfirst;
    std::vector<uint64_t> ilo;
    if (!same) {
        sfirst.assign(nseg, 0);
        for (int q = 0; q < nseg; q++) {
            sfirst[q] = (uint32_t)iseg.size();
            for (uint64_t c = seg_off[q]; c < seg_off[q + 1]; c += SS_CHUNK) {
                iseg.push_back((uint32_t)q);
                ilo.push_back(c);
                ilen.push_back((uint32_t)(seg_off[q + 1] - c < SS_CHUNK ? seg_off[q + 1] - c : SS_CHUNK));
            }
        }
        nitems = (int)iseg.size();
    }
    if (nitems == 0)
        return GVC_OK;
    char *w = (char *)ws;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *q = w + off;
        off += al256(bytes);
        return q;
    };
    SegPlan P;
    P.values = values;
    P.n = n;
    P.nseg = nseg;
    P.nitems = nitems;
    P.keymode = keymode;
    P.thr_only = thr_only;
    P.dgc_seg = dgc_seg;
    P.dgc_bits = dgc_bits;
    P.seed = seed;
    P.stream = stream;
    P.seg = (SegState *)take(nseg * sizeof(SegState));
    P.hist = (uint32_t *)take((size_t)SS_PASSES * nseg * SS_BINS * 4);
    P.seg_lo = (const uint64_t *)take((nseg + 1) * 8);
    P.seg_k = (const uint64_t *)take((nseg + 1) * 8);
    P.item_seg = (const uint32_t *)take(nitems * 4);
    P.item_len = (const uint32_t *)take(nitems * 4);
    P.item_gt = (uint32_t *)take(nitems * 4);
    P.item_eq = (uint32_t *)take(nitems * 4);
    P.item_take = (uint32_t *)take(nitems * 4);
    P.item_lo = (const uint64_t *)take(nitems * 8);
    P.item_out = (unsigned long long *)take(nitems * 8);
    P.item_E = (unsigned long long *)take(nitems * 8);
    P.seg_first = (const uint32_t *)take(nseg * 4);
    P.warp_gt = (uint32_t *)take((size_t)nitems * (SS_THREADS / 32) * 4);
    P.warp_eq = (uint32_t *)take((size_t)nitems * (SS_THREADS / 32) * 4);
    P.status = status;
    if (!same) {
        // (pageable host vectors: the copies complete before the calls return)
        cudaMemcpyAsync((void *)P.seg_lo, seg_off, (nseg + 1) * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync((void *)P.seg_k, seg_k, nseg * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync((void *)P.item_seg, iseg.data(), nitems * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync((void *)P.item_len, ilen.data(), nitems * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync((void *)P.item_lo, ilo.data(), nitems * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync((void *)P.seg_first, sfirst.data(), nseg * 4, cudaMemcpyHostToDevice, s);
        L.n = n;
        L.kind = kind;
        L.off.assign(seg_off, seg_off + nseg + 1);
        L.k.assign(seg_k, seg_k + nseg);
        L.nitems = nitems;
    }
    cudaMemsetAsync(P.hist, 0, (size_t)SS_PASSES * nseg * SS_BINS * 4, s);
    k_ss_init<<<(nseg + 255) / 256, 256, 0, s>>>(P);
    const int rgrid = nseg;
    for (int d = 0; d < SS_PASSES; d++) {
        if (keymode == KEY_HASH)
            k_ss_hist<KEY_HASH><<<nitems, SS_THREADS, 0, s>>>(P, d);
        else if (keymode == KEY_DGC)
            k_ss_hist<KEY_DGC><<<nitems, SS_THREADS, 0, s>>>(P, d);
        else
            k_ss_hist<KEY_MAG><<<nitems, SS_THREADS, 0, s>>>(P, d);
        k_ss_resolve<<<rgrid, SS_THREADS, 0, s>>>(P, d);
    }
    if (thr_only) {
        count_launches(1 + 2 * SS_PASSES);
        return GVC_OK;
    }
    if (keymode == KEY_HASH)
        k_ss_count<KEY_HASH><<<nitems, SS_THREADS, 0, s>>>(P);
    else if (keymode == KEY_DGC)
        k_ss_count<KEY_DGC><<<nitems, SS_THREADS, 0, s>>>(P);
    else
        k_ss_count<KEY_MAG><<<nitems, SS_THREADS, 0, s>>>(P);
    k_ss_scan<<<1, 1024, 0, s>>>(P);
    if (keymode == KEY_HASH)
        k_ss_write<KEY_HASH><<<nitems, SS_THREADS, 0, s>>>(P, out_idx, out_val);
    else if (keymode == KEY_DGC)
        k_ss_write<KEY_DGC><<<nitems, SS_THREADS, 0, s>>>(P, out_idx, out_val);
    else
        k_ss_write<KEY_MAG><<<nitems, SS_THREADS, 0, s>>>(P, out_idx, out_val);
    count_launches(4 + 2 * SS_PASSES);
    return GVC_OK;
}

int segsel_run(int kind, const float *values, uint64_t n, const uint64_t *seg_off, const uint64_t *seg_k, int nseg,
               uint64_t seed, uint64_t stream, uint32_t *out_idx, float *out_val, void *ws, size_t ws_bytes,
               uint32_t *status, cudaStream_t s)
{
    return segsel_launch(kind == GVC_RANDOMK ? KEY_HASH : KEY_MAG, 0, nullptr, nullptr, values, n, seg_off, seg_k,
                         nseg, seed, stream, out_idx, out_val, ws, ws_bytes, status, s);
}

// ------------------------------------------------------------ layerwise DGC
// compressors.py:204-217 with the DGC rule (:110-137) inside every segment,
// as three steps over all segments at once:
//   1. k_sdgc_sample: segment q draws s_q = min(len, max(256, round(f len)))
//      stratified positions (dgc_position with pos_base = the segment start,
//      as the per-segment selection draws them), gathers their values into
//      the segment's run of the sample vector and marks them in a global
//      position bitmap;
//   2. a threshold-only segmented selection over the samples: segment q's
//      rank_q-th largest sampled |v|, rank_q = min(s_q, max(1, round(k s / len)))
//      (rank_q = s_q: the minimum); segments sampled in full (s_q = len, exact
//      top-k) have no samples and threshold 0, under which every key is in
//      the upper half -- plain top-k;
//   3. the segmented selection over gvc_select's DGC composite key
//      ((|v| >= T_q or sampled) ? 2^31 | |v| : |v|) with segment q's T_q.
__global__ void __launch_bounds__(256) k_sdgc_sample(const float *__restrict__ values, uint64_t seed, uint64_t stream,
                                                     const uint64_t *__restrict__ seg_off,
                                                     const uint64_t *__restrict__ samp_off, int nseg,
                                                     float *__restrict__ vP, uint32_t *bits)
{
    const uint64_t S = samp_off[nseg];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t J = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; J < S; J += stride) {
        int a = 0, b = nseg - 1;  // the segment q with samp_off[q] <= J < samp_off[q + 1]
        while (a < b) {
            const int m = (a + b + 1) >> 1;
            if (__ldg(samp_off + m) <= J)
                a = m;
            else
                b = m - 1;
        }
        const uint64_t s0 = samp_off[a], sq = samp_off[a + 1] - s0;
        const uint64_t base = seg_off[a], len = seg_off[a + 1] - base;
        const uint64_t q = base + dgc_position(J - s0, len, sq, 1.0 / (double)sq, seed, stream, base);
        vP[J] = values[q];
        atomicOr(&bits[q >> 5], 1u << (q & 31));
    }
}

// the per-segment sample sizes and ranks (host; compressors.py:112, :119-121)
static void sdgc_counts(const uint64_t *seg_off, const uint64_t *seg_k, int nseg, double frac,
                        std::vector<uint64_t> &samp_off, std::vector<uint64_t> &rank)
{
    samp_off.assign(nseg + 1, 0);
    rank.assign(nseg, 0);
    for (int q = 0; q < nseg; q++) {
        const uint64_t len = seg_off[q + 1] - seg_off[q], k = seg_k[q];
        uint64_t sq = 0;
        if (len && k < len) {
            const double r = std::nearbyint(frac * (double)len);  // Python round(): ties to even
            sq = std::min<uint64_t>(len, std::max<uint64_t>(256, (uint64_t)r));
            if (sq >= len)
                sq = 0;  // the full sample: exact top-k (:113-115)
            else {
                // k s / len correctly rounded (k s < 2^53 for any n < 2^32 here:
                // s <= ~n / 100 + 256), then round half to even
                const double x = (double)(k * sq) / (double)len;
                rank[q] = std::min<uint64_t>(sq, std::max<uint64_t>(1, (uint64_t)std::nearbyint(x)));
            }
        }
        samp_off[q + 1] = samp_off[q] + sq;
    }
}

static uint64_t sdgc_sample_bound(uint64_t n, int nseg, double frac)
{
    const double b = std::ceil(frac * (double)n) + 258.0 * nseg;
    return std::min<uint64_t>(n, (uint64_t)b);
}

size_t seg_dgc_workspace_bytes(uint64_t n, int nseg, double frac)
{
    const uint64_t S = sdgc_sample_bound(n, nseg, frac);
    return segsel_workspace_bytes(n, nseg) + segsel_workspace_bytes(S, nseg) + al256(S * 4) + al256((n + 31) / 32 * 4) +
           al256((size_t)(nseg + 1) * 8) * 2 + 256;
}

int seg_dgc_run(const float *values, uint64_t n, const uint64_t *seg_off, const uint64_t *seg_k, int nseg, double frac,
                uint64_t seed, uint64_t stream, uint32_t *out_idx, float *out_val, void *ws, size_t ws_bytes,
                uint32_t *status, cudaStream_t s)
{
    if (!(frac > 0.0 && frac <= 1.0))
        return set_error(GVC_ERR_ARG, "segmented DGC: sample fraction %g outside (0, 1]", frac);
    for (int q = 0; q < nseg; q++)
        if (seg_off[q + 1] < seg_off[q] || seg_off[q + 1] > n)
            return set_error(GVC_ERR_ARG, "segmented DGC: segment %d outside [0, %llu)", q, (unsigned long long)n);
    if (seg_dgc_workspace_bytes(n, nseg, frac) > ws_bytes)
        return set_error(GVC_ERR_WORKSPACE, "segmented DGC workspace too small");
    std::vector<uint64_t> samp_off, rank;
    sdgc_counts(seg_off, seg_k, nseg, frac, samp_off, rank);
    const uint64_t S = samp_off[nseg];
    char *w = (char *)ws;
    char *ws_main = w;
    char *ws_samp = ws_main + segsel_workspace_bytes(n, nseg);
    float *vP = (float *)(ws_samp + segsel_workspace_bytes(sdgc_sample_bound(n, nseg, frac), nseg));
    uint32_t *bits = (uint32_t *)((char *)vP + al256(sdgc_sample_bound(n, nseg, frac) * 4));
    uint64_t *d_seg_off = (uint64_t *)((char *)bits + al256((n + 31) / 32 * 4));
    uint64_t *d_samp_off = (uint64_t *)((char *)d_seg_off + al256((size_t)(nseg + 1) * 8));
    // (pageable host arrays: the copies complete before the calls return)
    cudaMemcpyAsync(d_seg_off, seg_off, (nseg + 1) * 8, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_samp_off, samp_off.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(bits, 0, (n + 31) / 32 * 4, s);
    {
        std::lock_guard<std::mutex> lk(g_seg_mu);
        g_seg_alias[ws] = ws_samp;
    }
    if (!S)  // every segment exact or kept whole: thresholds 0 (no sample selection runs)
        cudaMemsetAsync(ws_samp, 0, nseg * sizeof(SegState), s);
    else {
        count_launches(1);
        const int blocks = (int)std::min<uint64_t>((S + 255) / 256, (uint64_t)device_sms() * 8);
        k_sdgc_sample<<<blocks, 256, 0, s>>>(values, seed, stream, d_seg_off, d_samp_off,
                                                                          nseg, vP, bits);
    }
    // the sample selection's states are at the start of its workspace (segsel_launch's carve)
    int rc = segsel_launch(KEY_MAG, 1, nullptr, nullptr, vP, S, samp_off.data(), rank.data(), nseg, seed, stream,
                           nullptr, nullptr, ws_samp, segsel_workspace_bytes(sdgc_sample_bound(n, nseg, frac), nseg),
                           status, s);
    if (rc)
        return rc;
    return segsel_launch(KEY_DGC, 0, (const SegState *)ws_samp, bits, values, n, seg_off, seg_k, nseg, seed, stream,
                         out_idx, out_val, ws_main, segsel_workspace_bytes(n, nseg), status, s);
}

}  // namespace gvc
