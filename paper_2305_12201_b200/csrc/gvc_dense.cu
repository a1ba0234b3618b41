// gvc_dense.cu -- dense-side kernels of the GraVAC step (sm_100a):
// error-feedback add, fp64 norm, residual scatter, decompress and the
// shared-memory-tiled fp64 decompress-average of N sparse parts.

#include "gvc_common.cuh"
#include "gvc_internal.h"

namespace gvc {

// SMs of the current device (cached per device): grid caps are whole waves of
// the part the kernel runs on, not of a hard-coded B200
int device_sms()
{
    static int cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64)
        return 148;
    if (!cache[dev]) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = sms > 0 ? sms : 148;
    }
    return cache[dev];
}

static inline int grid_for(uint64_t work, int per_block, int cap)
{
    uint64_t b = (work + per_block - 1) / per_block;
    if (b < 1)
        b = 1;
    return (int)(b > (uint64_t)cap ? cap : b);
}

static inline bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

// ------------------------------------------------------------- EF add
__global__ void k_ef_add(const float *__restrict__ g, const float *__restrict__ r, float *__restrict__ out,
                         uint64_t n, int vec)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (vec) {
        const uint64_t n4 = n / 4;
        for (uint64_t i = t0; i < n4; i += stride) {
            float4 a = ld_stream(reinterpret_cast<const float4 *>(g) + i);
            float4 b = ld_stream(reinterpret_cast<const float4 *>(r) + i);
            a.x = __fadd_rn(a.x, b.x);
            a.y = __fadd_rn(a.y, b.y);
            a.z = __fadd_rn(a.z, b.z);
            a.w = __fadd_rn(a.w, b.w);
            reinterpret_cast<float4 *>(out)[i] = a;
        }
        for (uint64_t i = n4 * 4 + t0; i < n; i += stride)
            out[i] = __fadd_rn(g[i], r[i]);
    } else {
        for (uint64_t i = t0; i < n; i += stride)
            out[i] = __fadd_rn(g[i], r[i]);
    }
}

int ef_add_run(const float *g, const float *r, float *out, uint64_t n, cudaStream_t s)
{
    int vec = aligned16(g) && aligned16(r) && aligned16(out);
    count_launches(1);
    k_ef_add<<<grid_for(n / 4 + 1, 256, device_sms() * 16), 256, 0, s>>>(g, r, out, n, vec);
    return GVC_OK;
}

// ------------------------------------------------------------- fp64 norm
// Grid size depends on n only, so the reduction order is reproducible.
#define NORM_BLOCKS_MAX 2048
__global__ void k_sq_norm_part(const float *__restrict__ x, uint64_t n, double *part)
{
    __shared__ double red[256];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double v = (double)x[i];
        acc = __fma_rn(v, v, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        part[blockIdx.x] = red[0];
}

__global__ void k_sq_norm_final(const double *part, int nb, double *out)
{
    __shared__ double red[1024];
    double acc = 0.0;
    for (int i = threadIdx.x; i < nb; i += 1024)
        acc += part[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        *out = red[0];
}

size_t sq_norm_workspace_bytes(uint64_t n)
{
    (void)n;
    return NORM_BLOCKS_MAX * sizeof(double);
}

int sq_norm_run(const float *x, uint64_t n, double *out, void *ws, size_t ws_bytes, cudaStream_t s)
{
    if (ws_bytes < sq_norm_workspace_bytes(n))
        return set_error(GVC_ERR_WORKSPACE, "sq_norm workspace too small");
    int nb = grid_for(n, 256 * 16, NORM_BLOCKS_MAX);
    count_launches(1);
    k_sq_norm_part<<<nb, 256, 0, s>>>(x, n, (double *)ws);
    count_launches(1);
    k_sq_norm_final<<<1, 1024, 0, s>>>((const double *)ws, nb, out);
    return GVC_OK;
}

// ---------------------------------------------------- residual scatter
__global__ void k_sub_scatter(const uint32_t *__restrict__ idx, const float *__restrict__ vals, uint64_t k,
                              float *resid)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        uint32_t p = idx[i];
        resid[p] = __fsub_rn(resid[p], vals[i]);
    }
}

int update_residual_run(const float *ef, const uint32_t *idx, const float *vals, uint64_t k, uint64_t n,
                        float *resid, cudaStream_t s)
{
    if (ef != resid)
        cudaMemcpyAsync(resid, ef, n * sizeof(float), cudaMemcpyDeviceToDevice, s);
    if (k)
        count_launches(1);
    k_sub_scatter<<<grid_for(k, 256, device_sms() * 16), 256, 0, s>>>(idx, vals, k, resid);
    return GVC_OK;
}

// ---------------------------------------------- deferred residual masks
__global__ void k_mark_sent(const uint32_t *__restrict__ idx, uint64_t k, uint32_t *mask)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    // grid-stride in whole warps so the per-word OR can use warp collectives
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ull; base < k; base += stride) {
        const uint64_t i = base + lane;
        const bool ok = i < k;
        const uint32_t gi = ok ? idx[i] : 0xffffffffu;
        const uint32_t word = gi >> 5;
        const uint32_t grp = __match_any_sync(0xffffffffu, word);
        const uint32_t bits = __reduce_or_sync(grp, ok ? (1u << (gi & 31)) : 0u);
        if (ok && (__ffs(grp) - 1) == lane)
            atomicOr(&mask[word], bits);
    }
}

int mark_sent_run(const uint32_t *idx, uint64_t k, uint32_t *mask, cudaStream_t s)
{
    if (k) {
        count_launches(1);
        k_mark_sent<<<grid_for(k, 256, device_sms() * 16), 256, 0, s>>>(idx, k, mask);
    }
    return GVC_OK;
}

__global__ void k_apply_pending(float *resid, uint32_t *mask, uint64_t n, int mode, const float *m_ptr)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const float m = (mode == 2 && m_ptr) ? *m_ptr : 0.f;
    const uint64_t nw = (n + 31) / 32;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
        uint32_t bits = mask[w];
        if (!bits)
            continue;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint64_t i = w * 32 + b;
            if (i < n)
                resid[i] = pending_resid(resid[i], mode, m);
        }
        mask[w] = 0u;
    }
}

int apply_pending_run(float *resid, uint32_t *mask, uint64_t n, int mode, const float *m, cudaStream_t s)
{
    count_launches(1);
    k_apply_pending<<<grid_for((n + 31) / 32, 256, device_sms() * 16), 256, 0, s>>>(resid, mask, n, mode, m);
    return GVC_OK;
}

// ------------------------------------------------------------ DGC helpers
// (stratum_lo / dgc_position: gvc_common.cuh, shared with the layerwise DGC)
__global__ void k_dgc_sample(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                             uint32_t *__restrict__ out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const double inv_s = 1.0 / (double)s;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < s; j += stride)
        out[j] = dgc_position(j, n, s, inv_s, seed, stream, pos_base);
}

// gvc_dgc_sample + gvc_gather_ef + the sample's position bitmap in one pass
// (bits zeroed by the caller's memset; strata are wider than 32 positions only
// past s ~ n / 32, so two samples can share a word: atomicOr)
__global__ void k_dgc_sample_gather(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                                    const float *__restrict__ values, const float *__restrict__ g,
                                    const float *__restrict__ resid, const uint32_t *pmask, const float *pm_ptr,
                                    int pmode, float *__restrict__ out, uint32_t *bits)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const double inv_s = 1.0 / (double)s;
    const float pm = (pmask && pmode == 2) ? *pm_ptr : 0.f;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < s; j += stride) {
        const uint32_t q = dgc_position(j, n, s, inv_s, seed, stream, pos_base);
        if (g) {
            float r = resid[q];
            if (pmask && ((pmask[q >> 5] >> (q & 31)) & 1u))
                r = pending_resid(r, pmode, pm);
            out[j] = __fadd_rn(g[q], r);
        } else {
            out[j] = values[q];
        }
        atomicOr(&bits[q >> 5], 1u << (q & 31));
    }
}

int dgc_sample_gather_run(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                          const float *values, const float *g, const float *resid, const uint32_t *pmask,
                          const float *pm, int pmode, float *out, uint32_t *bits, cudaStream_t st)
{
    if (s < 1 || s > n || n > 0xffffffffull)
        return set_error(GVC_ERR_ARG, "dgc_sample_gather: %llu samples of %llu positions", (unsigned long long)s,
                         (unsigned long long)n);
    cudaMemsetAsync(bits, 0, (n + 31) / 32 * 4, st);
    count_launches(1);
    k_dgc_sample_gather<<<grid_for(s, 256, device_sms() * 16), 256, 0, st>>>(n, s, seed, stream, pos_base, values, g, resid,
                                                                    pmask, pm, pmode, out, bits);
    return GVC_OK;
}

int dgc_sample_run(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base, uint32_t *out,
                   cudaStream_t st)
{
    if (s < 1 || s > n || n > 0xffffffffull)
        return set_error(GVC_ERR_ARG, "dgc_sample: %llu samples of %llu positions", (unsigned long long)s,
                         (unsigned long long)n);
    count_launches(1);
    k_dgc_sample<<<grid_for(s, 256, device_sms() * 8), 256, 0, st>>>(n, s, seed, stream, pos_base, out);
    return GVC_OK;
}

__global__ void k_gather_ef(const uint32_t *__restrict__ pos, uint64_t k, const float *__restrict__ values,
                            const float *__restrict__ g, const float *__restrict__ resid, const uint32_t *pmask,
                            const float *pm_ptr, int pmode, float *__restrict__ out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const float pm = (pmask && pmode == 2) ? *pm_ptr : 0.f;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint32_t q = pos[i];
        if (g) {
            float r = resid[q];
            if (pmask && ((pmask[q >> 5] >> (q & 31)) & 1u))
                r = pending_resid(r, pmode, pm);
            out[i] = __fadd_rn(g[q], r);
        } else {
            out[i] = values[q];
        }
    }
}

int gather_ef_run(const uint32_t *pos, uint64_t k, const float *values, const float *g, const float *resid,
                  const uint32_t *pmask, const float *pm, int pmode, float *out, cudaStream_t s)
{
    if (k) {
        count_launches(1);
        k_gather_ef<<<grid_for(k, 256, device_sms() * 16), 256, 0, s>>>(pos, k, values, g, resid, pmask, pm, pmode, out);
    }
    return GVC_OK;
}

__global__ void k_below_keys(const float *__restrict__ v, const uint32_t *__restrict__ pos, uint64_t n,
                             const uint32_t *thr_ptr, const uint32_t *excl, float *__restrict__ out,
                             unsigned long long *count)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t thr = *thr_ptr;
    unsigned long long c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t key = mag_key(v[i]);
        bool ok = key < thr;
        if (ok && excl) {
            const uint32_t q = pos ? pos[i] : (uint32_t)i;
            ok = !((excl[q >> 5] >> (q & 31)) & 1u);
        }
        // key + 1 keeps the order of eligible magnitudes and lifts |v| = 0 above
        // the excluded entries (+0.0); keys < thr < 2^31 so key + 1 is a finite float
        out[i] = __uint_as_float(ok ? key + 1u : 0u);
        c += ok;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c)
        atomicAdd(count, c);
}

int below_keys_run(const float *v, const uint32_t *pos, uint64_t n, const uint32_t *thr, const uint32_t *excl,
                   float *out, unsigned long long *count, cudaStream_t s)
{
    count_launches(1);
    k_below_keys<<<grid_for(n, 256, device_sms() * 16), 256, 0, s>>>(v, pos, n, thr, excl, out, count);
    return GVC_OK;
}

// Ordered compaction of a bit mask: block b owns 1024 words (4 per thread).
#define CMP_WORDS 1024
__global__ void k_compact_count(const uint32_t *__restrict__ mask, uint64_t nw, unsigned long long *blk)
{
    __shared__ unsigned long long sh[33];
    const uint64_t w0 = (uint64_t)blockIdx.x * CMP_WORDS + threadIdx.x * 4;
    unsigned long long c = 0;
    for (int q = 0; q < 4; q++)
        if (w0 + q < nw)
            c += __popc(mask[w0 + q]);
    unsigned long long tot;
    block_excl_prefix(c, sh, &tot);
    if (threadIdx.x == 0)
        blk[blockIdx.x] = tot;
}

__global__ void k_compact_scan(unsigned long long *blk, uint64_t nb, unsigned long long *count)
{
    __shared__ unsigned long long sh[33];
    const uint64_t per = (nb + 1023) / 1024;
    const uint64_t b0 = threadIdx.x * per;
    unsigned long long local = 0;
    for (uint64_t b = b0; b < min(nb, b0 + per); b++)
        local += blk[b];
    unsigned long long tot;
    unsigned long long acc = block_excl_prefix(local, sh, &tot);
    for (uint64_t b = b0; b < min(nb, b0 + per); b++) {
        const unsigned long long v = blk[b];
        blk[b] = acc;
        acc += v;
    }
    if (threadIdx.x == 0)
        *count = tot;
}

__global__ void k_compact_write(const uint32_t *__restrict__ mask, uint64_t nw, const unsigned long long *blk,
                                uint32_t *__restrict__ out)
{
    __shared__ unsigned long long sh[33];
    const uint64_t w0 = (uint64_t)blockIdx.x * CMP_WORDS + threadIdx.x * 4;
    uint32_t w[4];
    unsigned long long c = 0;
    for (int q = 0; q < 4; q++) {
        w[q] = w0 + q < nw ? mask[w0 + q] : 0u;
        c += __popc(w[q]);
    }
    unsigned long long o = blk[blockIdx.x] + block_excl_prefix(c, sh);
    for (int q = 0; q < 4; q++) {
        uint32_t bits = w[q];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            out[o++] = (uint32_t)((w0 + q) * 32 + b);
        }
    }
}

size_t compact_workspace_bytes(uint64_t n)
{
    const uint64_t nw = (n + 31) / 32;
    return (size_t)((nw + CMP_WORDS - 1) / CMP_WORDS + 1) * sizeof(unsigned long long);
}

int compact_mask_run(const uint32_t *mask, uint64_t n, uint32_t *out, unsigned long long *count, void *ws,
                     size_t ws_bytes, cudaStream_t s)
{
    if (ws_bytes < compact_workspace_bytes(n))
        return set_error(GVC_ERR_WORKSPACE, "compact workspace too small");
    const uint64_t nw = (n + 31) / 32;
    const uint64_t nb = (nw + CMP_WORDS - 1) / CMP_WORDS;
    unsigned long long *blk = (unsigned long long *)ws;
    count_launches(3);
    k_compact_count<<<(unsigned)nb, 256, 0, s>>>(mask, nw, blk);
    k_compact_scan<<<1, 1024, 0, s>>>(blk, nb, count);
    k_compact_write<<<(unsigned)nb, 256, 0, s>>>(mask, nw, blk, out);
    return GVC_OK;
}

// ------------------------------------------------- tiled decompress/average
// One CTA owns a TILE-value slice of the dense output.  For every part (in
// worker order) it binary-searches the slice's sub-range of that part's
// ascending index list and accumulates into a shared-memory tile (fp64 for
// the average, fp32 assignment for decompress); parts are separated by a
// barrier so each position sees its adds in worker order, as
// compressors.py:265-271 does.  The tile leaves in coalesced 128-bit stores.
#define AGG_TILE GVC_AGG_TILE
#define AGG_THREADS 256
#define AGG_MAX_PARTS 64

// Every part by its own pointers: the parts of one gathered buffer, or the
// payload slots of the peers' symmetric buffers (read over NVLink).
struct PeerFlags {
    uint32_t *flags[GVC_MAX_PEERS];
};

struct AggParts {
    const uint32_t *idx[AGG_MAX_PARTS];
    const float *vals[AGG_MAX_PARTS];
    const uint32_t *bounds[AGG_MAX_PARTS];
    uint64_t cnt[AGG_MAX_PARTS];
};

// Tile boundaries of every part in one streaming pass over the index lists:
// bounds[p * (ntiles + 1) + b] = first entry of part p with index >= b * TILE.
__global__ void k_tile_bounds(AggParts parts, int nparts, uint64_t ntiles, uint32_t *__restrict__ bounds)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const int p = blockIdx.y;
    if (p >= nparts)
        return;
    const uint32_t *pi = parts.idx[p];
    const uint64_t cnt = parts.cnt[p];
    uint32_t *bp = bounds + (uint64_t)p * (ntiles + 1);
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= cnt; t += stride) {
        int64_t prev = t == 0 ? -1 : (int64_t)(pi[t - 1] / AGG_TILE);
        int64_t cur = t == cnt ? (int64_t)ntiles : (int64_t)(pi[t] / AGG_TILE);
        for (int64_t b = prev + 1; b <= cur; b++)
            bp[b] = (uint32_t)t;
    }
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Staged pull (C1 + K7 overlapped): the first `ncopy` CTAs of the merge grid
// (by block index, or by start order with GVC_STAGED_TICKET) are copiers.  They wait for every peer's payload
// flag, then stream the peers' (idx, vals) chunk by chunk over NVLink into
// local staging slots and publish each chunk with a release store of the
// epoch into ready[chunk].  The remaining CTAs are the usual tiles; a tile
// waits only for the chunks its entries fall in, so the merge trails the
// transfer instead of following it.  Every wait is bounded (wait_epoch).
struct Staged {
    int ncopy;           // copier CTAs (0: direct pull, no staging)
    int self;            // this rank's part (already local)
    uint32_t ch_log2;    // entries per chunk = 1 << ch_log2 (multiple of 4)
    uint32_t nchunks;
    uint32_t nb;         // tile-bound words per part (ntiles + 1)
    uint32_t *ready;     // [b < ncopy]: bound slice b's epoch; [ncopy + c]: chunk c's epoch
    const uint32_t *src_idx[GVC_MAX_PEERS];  // peer p's payload (remote)
    const float *src_val[GVC_MAX_PEERS];
    const uint32_t *src_bounds[GVC_MAX_PEERS];
    // 16-bit wire indices (all parts or none): the copiers move src_off
    // instead of src_idx into off[p], and the tiles read off[p] (own part's
    // included) -- 6 bytes per entry over NVLink instead of 8
    int use_off;
    const uint16_t *src_off[GVC_MAX_PEERS];
    const uint16_t *off[GVC_MAX_PEERS];
    uint32_t *err;  // the flag area's error word (bounded waits)
    uint32_t *ticket;    // dispatch-order CTA ticket (flags word GVC_FLAG_TICKET_WORD, reset by the last CTA)
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Peer waits are bounded.  `err` is a word of this rank's peer-buffer flag
// area (GVC_FLAG_ERR_WORD): a wait that times out (~4 s -- a rank died or
// diverged) sets bit 4 there, and every later wait of the exchange sees it and
// stops waiting, so a dead peer costs seconds instead of a hung GPU.  The
// host (exchange.PeerExchange) reads the word back every few exchanges.
#define GVC_FLAG_ERR_WORD 63
#define GVC_FLAG_TICKET_WORD 62  // staged merge: CTA roles in dispatch order
__device__ __forceinline__ void wait_epoch(const uint32_t *word, uint32_t epoch, bool sys, uint32_t *err)
{
    long long t0 = 0;
    while ((int32_t)((sys ? ld_acquire_sys(word) : ld_acquire_gpu(word)) - epoch) < 0) {
        if (*(volatile uint32_t *)err)
            return;
        if (t0 == 0) {
            t0 = clock64();
        } else if (clock64() - t0 > (1ll << 33)) {
            atomicOr(err, 4u);
            return;
        }
        __nanosleep(64);
    }
}

__device__ __forceinline__ uint32_t *flag_err(const uint32_t *flags)
{
    return const_cast<uint32_t *>(flags) + GVC_FLAG_ERR_WORD;
}

#ifndef GVC_COPIER_TMA
#define GVC_COPIER_TMA 0
#endif
template <bool OFF>
__device__ void staged_copier(const Staged &st, const AggParts &parts, int nparts, const uint32_t *flags,
                              uint32_t epoch, uint32_t vb, void *sbuf = nullptr, uint32_t sbytes = 0)
{
    if (threadIdx.x < nparts && (int)threadIdx.x != st.self)
        wait_epoch(flags + threadIdx.x, epoch, true, st.err);
    __syncthreads();
    // first the tile bounds (every tile needs them before it can look for its
    // chunks): copier b stages slice b of every remote part's bounds
    {
        const uint32_t per = (st.nb + st.ncopy - 1) / st.ncopy;
        const uint32_t b0 = vb * per, b1 = min(st.nb, b0 + per);
        for (int q = 0; q < nparts; q++) {
            if (q == st.self)
                continue;
            uint32_t *dst = const_cast<uint32_t *>(parts.bounds[q]);
            for (uint32_t i = b0 + threadIdx.x; i < b1; i += AGG_THREADS)
                __stcg(dst + i, __ldcg(st.src_bounds[q] + i));
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(st.ready + vb), "r"(epoch) : "memory");
    }
    constexpr int U = 4;
    if (GVC_COPIER_TMA && !OFF && sbuf && nparts == 2 && (4u << st.ch_log2) <= sbytes / 2) {
        // the TMA path (two parts: one remote): thread 0 moves the chunks
        // through the CTA's (unused) tile buffer with bulk copies -- both
        // arrays of a chunk in flight on two mbarriers, the next chunk's loads
        // issued as soon as this chunk's stores have read shared memory, the
        // chunk published once its stores completed
        __shared__ __align__(8) uint64_t mbar[2];
        if (threadIdx.x == 0) {
            const int q = 1 - st.self;
            const uint64_t k = parts.cnt[q];
            const uint32_t half = sbytes / 2;  // one array of a chunk per half
            const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sbuf);
            const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb0 + 8));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            auto range = [&](uint32_t c, uint64_t &a, uint32_t &bytes) {
                const uint64_t lo = (uint64_t)c << st.ch_log2;
                const uint64_t hi = min((unsigned long long)k, (unsigned long long)(lo + (1ull << st.ch_log2)));
                a = lo & ~3ull;
                bytes = lo >= hi ? 0u : (uint32_t)((((hi + 3) & ~3ull) - a) * 4);  // padded slots
            };
            auto load = [&](uint32_t c) {
                uint64_t a;
                uint32_t bytes;
                range(c, a, bytes);
                if (!bytes)
                    return;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0), "r"(bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sb), "l"(st.src_idx[q] + a), "r"(bytes), "r"(mb0) : "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb0 + 8), "r"(bytes)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sb + half), "l"(st.src_val[q] + a), "r"(bytes), "r"(mb0 + 8) : "memory");
            };
            auto wait = [&](uint32_t mb, uint32_t phase) {
                const long long t0 = clock64();
                for (;;) {
                    uint32_t done;
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                                 "selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done)
                                 : "r"(mb), "r"(phase)
                                 : "memory");
                    if (done || clock64() - t0 > (1ll << 33)) {
                        if (!done)
                            atomicOr(st.err, 4u);
                        return;
                    }
                }
            };
            uint32_t phase = 0;
            if (vb < st.nchunks)
                load(vb);
            for (uint32_t c = vb; c < st.nchunks; c += st.ncopy) {
                uint64_t a;
                uint32_t bytes;
                range(c, a, bytes);
                if (bytes) {
                    wait(mb0, phase);
                    wait(mb0 + 8, phase);
                    phase ^= 1u;
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     const_cast<uint32_t *>(parts.idx[q]) + a),
                                 "r"(sb), "r"(bytes)
                                 : "memory");
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     const_cast<float *>(parts.vals[q]) + a),
                                 "r"(sb + half), "r"(bytes)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                }
                if (c + st.ncopy < st.nchunks)
                    load(c + st.ncopy);
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(st.ready + st.ncopy + c), "r"(epoch)
                             : "memory");
            }
        }
        return;
    }
    for (uint32_t c = vb; c < st.nchunks; c += st.ncopy) {
        for (int q = 0; q < nparts; q++) {
            if (q == st.self)
                continue;
            const uint64_t k = parts.cnt[q];
            const uint64_t lo = (uint64_t)c << st.ch_log2;
            const uint64_t hi = min((unsigned long long)k, (unsigned long long)(lo + (1ull << st.ch_log2)));
            if (lo >= hi)
                continue;
            const int4 *sv = reinterpret_cast<const int4 *>(st.src_val[q]);
            int4 *dv = reinterpret_cast<int4 *>(const_cast<float *>(parts.vals[q]));
            if (OFF) {
                // (u16 offset, f32 value): offsets in int4 granules of 8 (the
                // offset area is padded to 8 entries), values in granules of 4
                const uint32_t lo8 = (uint32_t)(lo >> 3), hi8 = (uint32_t)((hi + 7) >> 3);
                const uint32_t lo4 = (uint32_t)(lo >> 2), hi4 = (uint32_t)((hi + 3) >> 2);
                const int4 *so = reinterpret_cast<const int4 *>(st.src_off[q]);
                int4 *dO = reinterpret_cast<int4 *>(const_cast<uint16_t *>(st.off[q]));
                const uint32_t n8 = hi8 - lo8, n4 = hi4 - lo4;  // n8 <= (n4 + 1) / 2
                // value granule i and offset granule i in flight together: a
                // 4096-entry chunk in one round trip over NVLink, as the u32 path
                for (uint32_t i0 = threadIdx.x; i0 < n4; i0 += U * AGG_THREADS) {
                    int4 a[U], b[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const uint32_t i = i0 + u * AGG_THREADS;
                        if (i < n8)
                            a[u] = __ldcg(so + lo8 + i);
                        if (i < n4)
                            b[u] = __ldcg(sv + lo4 + i);
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const uint32_t i = i0 + u * AGG_THREADS;
                        if (i < n8)
                            __stcg(dO + lo8 + i, a[u]);
                        if (i < n4)
                            __stcg(dv + lo4 + i, b[u]);
                    }
                }
                continue;
            }
            // int4 granules; the slots are padded to 4 entries, so rounding up is safe
            const uint32_t lo4 = (uint32_t)(lo >> 2), hi4 = (uint32_t)((hi + 3) >> 2);
            const int4 *si = reinterpret_cast<const int4 *>(st.src_idx[q]);
            int4 *di = reinterpret_cast<int4 *>(const_cast<uint32_t *>(parts.idx[q]));
            for (uint32_t i0 = lo4 + threadIdx.x; i0 < hi4; i0 += U * AGG_THREADS) {
                int4 a[U], b[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t i = i0 + u * AGG_THREADS;
                    if (i < hi4) {
                        a[u] = __ldcg(si + i);
                        b[u] = __ldcg(sv + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t i = i0 + u * AGG_THREADS;
                    if (i < hi4) {
                        __stcg(di + i, a[u]);
                        __stcg(dv + i, b[u]);
                    }
                }
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(st.ready + st.ncopy + c), "r"(epoch) : "memory");
    }
}

// The CTA's role in the staged merge, from a ticket taken when it starts:
// tickets 0 .. ncopy-1 copy, the rest merge tile (ticket - ncopy).  A tile
// that waits for a chunk therefore runs only after every copier has started
// -- block indices carry no such guarantee (CTAs may be dispatched in any
// order, and SMs can be held by other work).  The last ticket resets the
// counter for the next exchange (stream-ordered).
// GVC_STAGED_TICKET=1: roles by the dispatch-order ticket.  Measured at N = 4
// (ResNet101 44.5M, scripts/ab_n4.sh): median step 0.425 ms vs 0.390 with
// block-index roles, and tail steps up to 0.9 ms -- ~11K CTAs take the same
// atomic -- so the default keeps block-index roles: the low-index copiers are
// dispatched first in practice, and every wait is bounded, so an unlucky
// schedule costs a timeout error, not a hung GPU.
#ifndef GVC_STAGED_TICKET
#define GVC_STAGED_TICKET 0
#endif
__device__ __forceinline__ uint32_t staged_ticket(const Staged &st)
{
    if (!GVC_STAGED_TICKET)
        return blockIdx.x;
    __shared__ uint32_t s_vb;
    if (threadIdx.x == 0) {
        const uint32_t t = atomicAdd(st.ticket, 1u);
        if (t == gridDim.x - 1)
            atomicExch(st.ticket, 0u);
        s_vb = t;
    }
    __syncthreads();
    return s_vb;
}

// A tile's wait for the staged bound slices holding entries t and t + 1.
__device__ __forceinline__ void staged_wait_bounds(const Staged &st, int q, uint32_t t, uint32_t epoch)
{
    if (q == st.self)
        return;
    const uint32_t per = (st.nb + st.ncopy - 1) / st.ncopy;
    for (uint32_t b = t / per; b <= (t + 1) / per; b++)
        wait_epoch(st.ready + b, epoch, false, st.err);
}

// A tile's wait for the staged chunks of part q covering entries [a, b).
__device__ __forceinline__ void staged_wait(const Staged &st, int q, uint32_t a, uint32_t b, uint32_t epoch)
{
    if (q == st.self || b <= a)
        return;
    for (uint32_t c = a >> st.ch_log2; c <= (b - 1) >> st.ch_log2; c++)
        wait_epoch(st.ready + st.ncopy + c, epoch, false, st.err);
}

// MODE 0: decompress (fp32 assignment, -0.0 kept); 1: mean of ONE part
// (0.0 + v in fp64 then /1: v, except -0.0 -> +0.0); 2: fp64 mean of N parts.
// Parts are taken in groups of NP: the group's tile bounds are fetched by NP
// threads at once, then (when every part of the group has at most
// U * AGG_THREADS entries in this tile, the common case) ALL their entries
// are loaded into registers before the part-ordered accumulation starts, so
// a tile costs two dependent memory latencies instead of two per part --
// what matters when the parts sit behind NVLink.
// WAIT: the parts live in the peers' memory; before reading part p a thread
// waits until peer p has posted `epoch` into flags[p] (its payload is
// complete), and all part reads bypass L1 (ld.global.cg), so no stale line of
// an earlier exchange through the same slot can be hit.
template <int MODE, bool WAIT, int NP, bool STAGED = false, bool OFF = false>
__global__ void __launch_bounds__(AGG_THREADS) k_tile_merge(AggParts parts, int nparts, uint64_t n,
                                                            float *__restrict__ out, const uint32_t *flags,
                                                            uint32_t epoch, Staged stg)
{
    constexpr int U = NP >= 8 ? 2 : 4;
    __shared__ __align__(16) double acc[MODE == 2 ? AGG_TILE : 2];
    __shared__ __align__(16) float accf[MODE == 2 ? 4 : AGG_TILE];
    __shared__ uint32_t s_a[NP], s_b[NP];
    const uint32_t vb = STAGED ? staged_ticket(stg) : blockIdx.x;
    if (STAGED && (int)vb < stg.ncopy) {
        staged_copier<OFF>(stg, parts, nparts, flags, epoch, vb, MODE == 2 ? (void *)acc : (void *)accf,
                      MODE == 2 ? (uint32_t)sizeof(acc) : (uint32_t)sizeof(accf));
        return;
    }
    const uint32_t tile = STAGED ? vb - stg.ncopy : blockIdx.x;
    constexpr bool use_off = STAGED && OFF;  // 16-bit wire indices: tile offsets directly
    const uint64_t lo = (uint64_t)tile * AGG_TILE;
    const uint32_t width = (uint32_t)min((uint64_t)AGG_TILE, n - lo);
    if (MODE == 2) {
        for (int i = threadIdx.x; i < AGG_TILE / 2; i += AGG_THREADS)
            reinterpret_cast<double2 *>(acc)[i] = make_double2(0.0, 0.0);
    } else {
        for (int i = threadIdx.x; i < AGG_TILE / 4; i += AGG_THREADS)
            reinterpret_cast<float4 *>(accf)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    auto put = [&](uint32_t r, float v) {
        if (MODE == 2)
            acc[r] += (double)v;
        else if (MODE == 1)
            accf[r] = v == 0.0f ? 0.0f : v;
        else
            accf[r] = v;
    };
    for (int p0 = 0; p0 < nparts; p0 += NP) {
        const int np = min(NP, nparts - p0);
        if (threadIdx.x < np) {
            const int p = p0 + threadIdx.x;
            if (WAIT)
                wait_epoch(flags + p, epoch, true, flag_err(flags));
            if (STAGED)
                staged_wait_bounds(stg, p, tile, epoch);
            s_a[threadIdx.x] = __ldcg(parts.bounds[p] + tile);
            s_b[threadIdx.x] = __ldcg(parts.bounds[p] + tile + 1);
            if (STAGED)
                staged_wait(stg, p, s_a[threadIdx.x], s_b[threadIdx.x], epoch);
        }
        __syncthreads();
        uint32_t maxlen = 0;
        for (int q = 0; q < np; q++)
            maxlen = max(maxlen, s_b[q] - s_a[q]);
        if (maxlen <= U * AGG_THREADS) {
            uint32_t r[NP][U];
            float v[NP][U];
            int left[NP];
#pragma unroll
            for (int q = 0; q < NP; q++) {
                left[q] = 0;
                if (q < np) {
                    const uint32_t a = s_a[q] + threadIdx.x;
                    left[q] = (int)s_b[q] - (int)a;
                    const uint32_t *pi = parts.idx[p0 + q] + a;
                    const uint16_t *po = use_off ? stg.off[p0 + q] + a : nullptr;
                    const float *pv = parts.vals[p0 + q] + a;
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        if (u * AGG_THREADS < left[q]) {
                            r[q][u] = use_off ? (uint32_t)__ldcg(po + u * AGG_THREADS)
                                              : __ldcg(pi + u * AGG_THREADS) - (uint32_t)lo;
                            v[q][u] = __ldcg(pv + u * AGG_THREADS);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < NP; q++) {
                if (q < np) {
#pragma unroll
                    for (int u = 0; u < U; u++)
                        if (u * AGG_THREADS < left[q])
                            put(r[q][u], v[q][u]);
                    if (MODE == 2)
                        __syncthreads();  // worker order per position (compressors.py:266-269)
                }
            }
        } else {
            for (int q = 0; q < np; q++) {
                const uint32_t *pi = parts.idx[p0 + q];
                const uint16_t *po = use_off ? stg.off[p0 + q] : nullptr;
                const float *pv = parts.vals[p0 + q];
                const uint32_t b = s_b[q];
                for (uint32_t t0 = s_a[q] + threadIdx.x; t0 < b; t0 += U * AGG_THREADS) {
                    uint32_t r[U];
                    float v[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        if (t0 + u * AGG_THREADS < b) {
                            r[u] = use_off ? (uint32_t)__ldcg(po + t0 + u * AGG_THREADS)
                                           : __ldcg(pi + t0 + u * AGG_THREADS) - (uint32_t)lo;
                            v[u] = __ldcg(pv + t0 + u * AGG_THREADS);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; u++)
                        if (t0 + u * AGG_THREADS < b)
                            put(r[u], v[u]);
                }
                if (MODE == 2)
                    __syncthreads();
            }
        }
        __syncthreads();  // s_a / s_b are rewritten by the next group
    }
    // x / N == x * (1/N) exactly only for power-of-two N; zeros skip the divide
    const double np = (double)nparts;
    const bool pow2 = (nparts & (nparts - 1)) == 0;
    const double inv = (double)(1.0f / (float)nparts);  // exact when it is used (power-of-two N)
    auto mean = [&](double a) -> float {
        if (a == 0.0)
            return 0.0f;
        return (float)(pow2 ? a * inv : a / np);
    };
    if (width == AGG_TILE && (((uintptr_t)(out + lo)) & 15) == 0) {
        for (int i = threadIdx.x; i < AGG_TILE / 4; i += AGG_THREADS) {
            float4 v;
            if (MODE == 2) {
                const double2 d0 = reinterpret_cast<const double2 *>(acc)[2 * i];
                const double2 d1 = reinterpret_cast<const double2 *>(acc)[2 * i + 1];
                v = make_float4(mean(d0.x), mean(d0.y), mean(d1.x), mean(d1.y));
            } else {
                v = reinterpret_cast<const float4 *>(accf)[i];
            }
            st_stream(reinterpret_cast<float4 *>(out + lo) + i, v);
        }
    } else {
        for (uint32_t i = threadIdx.x; i < width; i += AGG_THREADS)
            out[lo + i] = MODE == 2 ? mean(acc[i]) : accf[i];
    }
}

// The same tile merge for nparts <= NP <= 4 without the fp64 read-modify-
// write: every part scatters its values into its OWN fp32 shared tile (no
// ordering between parts needed, one barrier), and each output is then
// formed in registers as ((0.0 + v_0) + v_1 + ...) in fp64, part order --
// exactly aggregate()'s sum, because a part without an entry at a position
// contributes +0.0, which leaves any fp64 sum starting from +0.0 unchanged
// (it can never be -0.0).  MODE 0: decompress (one part, fp32 copy, -0.0
// kept); MODE 1: average.  Dynamic shared memory: NP * AGG_TILE floats.
template <int MODE, bool WAIT, int NP, bool STAGED = false, bool OFF = false>
__global__ void __launch_bounds__(AGG_THREADS) k_tile_part(AggParts parts, int nparts, uint64_t n,
                                                           float *__restrict__ out, const uint32_t *flags,
                                                           uint32_t epoch, Staged stg)
{
    constexpr int U = NP >= 4 ? 2 : 4;
    extern __shared__ __align__(16) float tiles[];
    __shared__ uint32_t s_a[NP], s_b[NP];
    const uint32_t vb = STAGED ? staged_ticket(stg) : blockIdx.x;
    if (STAGED && (int)vb < stg.ncopy) {
        staged_copier<OFF>(stg, parts, nparts, flags, epoch, vb, tiles, (uint32_t)(nparts * AGG_TILE * 4));
        return;
    }
    const uint32_t tile = STAGED ? vb - stg.ncopy : blockIdx.x;
    constexpr bool use_off = STAGED && OFF;  // 16-bit wire indices: tile offsets directly
    const uint64_t lo = (uint64_t)tile * AGG_TILE;
    const uint32_t width = (uint32_t)min((uint64_t)AGG_TILE, n - lo);
    if (threadIdx.x < nparts) {
        const int p = threadIdx.x;
        if (WAIT)
            wait_epoch(flags + p, epoch, true, flag_err(flags));
        if (STAGED)
            staged_wait_bounds(stg, p, tile, epoch);
        s_a[p] = __ldcg(parts.bounds[p] + tile);
        s_b[p] = __ldcg(parts.bounds[p] + tile + 1);
        if (STAGED)
            staged_wait(stg, p, s_a[p], s_b[p], epoch);
    }
    for (int i = threadIdx.x; i < nparts * (AGG_TILE / 4); i += AGG_THREADS)
        reinterpret_cast<float4 *>(tiles)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    uint32_t maxlen = 0;
#pragma unroll
    for (int q = 0; q < NP; q++)
        if (q < nparts)
            maxlen = max(maxlen, s_b[q] - s_a[q]);
    if (maxlen <= U * AGG_THREADS) {
        // every entry of every part in flight before the first store
        uint32_t r[NP][U];
        float v[NP][U];
        // per part: this thread's first entry and how many it may take
        // (pointers formed once; the U loads use immediate offsets)
        int left[NP];
#pragma unroll
        for (int q = 0; q < NP; q++) {
            left[q] = 0;
            if (q < nparts) {
                const uint32_t a = s_a[q] + threadIdx.x;
                left[q] = (int)s_b[q] - (int)a;
                const uint32_t *pi = parts.idx[q] + a;
                const uint16_t *po = use_off ? stg.off[q] + a : nullptr;
                const float *pv = parts.vals[q] + a;
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (u * AGG_THREADS < left[q]) {
                        r[q][u] = use_off ? (uint32_t)__ldcg(po + u * AGG_THREADS)
                                          : __ldcg(pi + u * AGG_THREADS) - (uint32_t)lo;
                        v[q][u] = __ldcg(pv + u * AGG_THREADS);
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NP; q++) {
            float *tq = tiles + q * AGG_TILE;
#pragma unroll
            for (int u = 0; u < U; u++)
                if (u * AGG_THREADS < left[q])
                    tq[r[q][u]] = v[q][u];
        }
    } else {
        for (int q = 0; q < nparts; q++) {
            const uint32_t *pi = parts.idx[q];
            const uint16_t *po = use_off ? stg.off[q] : nullptr;
            const float *pv = parts.vals[q];
            const uint32_t b = s_b[q];
            for (uint32_t t0 = s_a[q] + threadIdx.x; t0 < b; t0 += U * AGG_THREADS) {
                uint32_t r[U];
                float v[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    if (t0 + u * AGG_THREADS < b) {
                        r[u] = use_off ? (uint32_t)__ldcg(po + t0 + u * AGG_THREADS)
                                       : __ldcg(pi + t0 + u * AGG_THREADS) - (uint32_t)lo;
                        v[u] = __ldcg(pv + t0 + u * AGG_THREADS);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (t0 + u * AGG_THREADS < b)
                        tiles[q * AGG_TILE + r[u]] = v[u];
            }
        }
    }
    __syncthreads();
    // Output = fl32(((0.0 + v_0) + v_1 + ...) / N) in fp64, part order.  For a
    // power-of-two N with at most two non-zero terms the fp32 evaluation
    // ((0.0f + v_0) + v_1 + ...) * (1/N) is bit-identical: adding zeros is
    // exact, one fp32 add of two fp32 values rounds exactly like the fp64 add
    // followed by the fp32 rounding (the fp64 sum of two fp32 values is exact
    // unless their exponents differ by > 29, and then both round to the larger
    // term), and the 1/N scaling is exact above the subnormal range.  Every
    // other output (>= 3 non-zero terms, a tiny sum, non-power-of-two N) takes
    // the fp64 path, as does an fp32 sum that overflowed.  This keeps the fp64 convert/add units -- a fraction of
    // the fp32 rate -- off the common path.
    const bool pow2 = (nparts & (nparts - 1)) == 0;
    const float invf = 1.0f / (float)nparts;  // exact for the power-of-two N the fast path needs
    auto combine = [&](const float (&t)[NP]) -> float {
        if (MODE == 0)
            return t[0];
        float s = 0.0f;
        int nz = 0;
#pragma unroll
        for (int q = 0; q < NP; q++) {
            if (q < nparts) {
                s += t[q];
                nz += t[q] != 0.0f;
            }
        }
        if (NP == 1)
            return s;  // 0.0f + v: -0.0 -> +0.0, exact otherwise
        // fp32 fast path unless the sum is tiny (scaling could round) or
        // overflowed in fp32 (the fp64 sum may still be finite)
        if (pow2 && nz <= 2 && (s == 0.0f || (fabsf(s) >= 0x1p-100f && fabsf(s) <= 3.4028234663852886e38f)))
            return s * invf;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < NP; q++)
            if (q < nparts)
                acc += (double)t[q];
        if (acc == 0.0)
            return 0.0f;
        const double np = (double)nparts;
        return (float)(pow2 ? acc * (1.0 / np) : acc / np);
    };
    // |s| == 0 or 2^-100 <= |s| <= FLT_MAX, on the bits
    auto range_ok = [](float x) -> bool {
        const uint32_t u = __float_as_uint(x) & 0x7fffffffu;
        return u == 0u || (u - 0x0d800000u) < (0x7f800000u - 0x0d800000u);
    };
    if (width == AGG_TILE && (((uintptr_t)(out + lo)) & 15) == 0) {
        for (int i = threadIdx.x; i < AGG_TILE / 4; i += AGG_THREADS) {
            float4 t4[NP];
#pragma unroll
            for (int q = 0; q < NP; q++)
                t4[q] = q < nparts ? reinterpret_cast<const float4 *>(tiles + q * AGG_TILE)[i]
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            float4 o;
            if (MODE == 0) {
                o = t4[0];
            } else {
                // fp32 sums from +0.0 in part order (parts past nparts add +0.0)
                float4 s4 = make_float4(0.0f + t4[0].x, 0.0f + t4[0].y, 0.0f + t4[0].z, 0.0f + t4[0].w);
#pragma unroll
                for (int q = 1; q < NP; q++) {
                    s4.x += t4[q].x;
                    s4.y += t4[q].y;
                    s4.z += t4[q].z;
                    s4.w += t4[q].w;
                }
                bool ok = true;
                if (NP > 1) {
                    ok = pow2 && range_ok(s4.x) && range_ok(s4.y) && range_ok(s4.z) && range_ok(s4.w);
                    if (NP > 2) {  // at most two non-zero terms per output
                        int mx = 0;
                        auto nzc = [&](int c) {
                            int z = 0;
#pragma unroll
                            for (int q = 0; q < NP; q++) {
                                const float v = c == 0 ? t4[q].x : c == 1 ? t4[q].y : c == 2 ? t4[q].z : t4[q].w;
                                z += (__float_as_uint(v) << 1) != 0u;
                            }
                            return z;
                        };
                        mx = max(max(nzc(0), nzc(1)), max(nzc(2), nzc(3)));
                        ok = ok && mx <= 2;
                    }
                }
                if (ok) {
                    o = NP == 1 ? s4 : make_float4(s4.x * invf, s4.y * invf, s4.z * invf, s4.w * invf);
                } else {
                    float tx[NP], ty[NP], tz[NP], tw[NP];
#pragma unroll
                    for (int q = 0; q < NP; q++) {
                        tx[q] = t4[q].x;
                        ty[q] = t4[q].y;
                        tz[q] = t4[q].z;
                        tw[q] = t4[q].w;
                    }
                    o = make_float4(combine(tx), combine(ty), combine(tz), combine(tw));
                }
            }
            st_stream(reinterpret_cast<float4 *>(out + lo) + i, o);
        }
    } else {
        for (uint32_t i = threadIdx.x; i < width; i += AGG_THREADS) {
            float t[NP];
#pragma unroll
            for (int q = 0; q < NP; q++)
                t[q] = q < nparts ? tiles[q * AGG_TILE + i] : 0.0f;
            out[lo + i] = combine(t);
        }
    }
}

size_t aggregate_workspace_bytes(int nparts, uint64_t n)
{
    uint64_t ntiles = (n + AGG_TILE - 1) / AGG_TILE;
    return (size_t)(nparts < 1 ? 1 : nparts) * (ntiles + 1) * sizeof(uint32_t);
}

// Parts without tile bounds get them from k_tile_bounds into ws first.
static int tile_merge_run(bool avg, AggParts &P, int nparts, uint64_t n, float *out, void *ws, size_t ws_bytes,
                          const uint32_t *flags, uint32_t epoch, cudaStream_t s, const Staged *staged = nullptr)
{
    const uint64_t ntiles = (n + AGG_TILE - 1) / AGG_TILE;
    ProfScope pa(PROF_AGGREGATE, s);
    if (!P.bounds[0]) {
        if (ws_bytes < aggregate_workspace_bytes(nparts, n))
            return set_error(GVC_ERR_WORKSPACE, "aggregate workspace too small: %zu < %zu", ws_bytes,
                             aggregate_workspace_bytes(nparts, n));
        uint64_t maxcnt = 1;
        for (int p = 0; p < nparts; p++)
            maxcnt = P.cnt[p] + 1 > maxcnt ? P.cnt[p] + 1 : maxcnt;
        dim3 bg((unsigned)grid_for(maxcnt, 256, 1024), (unsigned)nparts);
        count_launches(1);
        k_tile_bounds<<<bg, 256, 0, s>>>(P, nparts, ntiles, (uint32_t *)ws);
        for (int p = 0; p < nparts; p++)
            P.bounds[p] = (const uint32_t *)ws + (uint64_t)p * (ntiles + 1);
    }
    count_launches(1);
    const unsigned g = (unsigned)ntiles;
    const size_t sm1 = AGG_TILE * 4, sm2 = 2 * sm1;
    // measured (scripts/merge_bench.py): per-part fp32 tiles win for 1-2 parts,
    // the single fp64 tile (less shared memory, higher occupancy) above
    Staged none;
    memset(&none, 0, sizeof(none));
    const Staged &st = staged ? *staged : none;
    const unsigned gs = g + (unsigned)st.ncopy;
    if (staged && st.use_off) {  // 16-bit wire indices
        if (nparts <= 2)
            k_tile_part<1, true, 2, true, true><<<gs, AGG_THREADS, nparts * sm1, s>>>(P, nparts, n, out, flags, epoch,
                                                                                     st);
        else if (nparts <= 4)
            k_tile_merge<2, true, 4, true, true><<<gs, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
        else
            k_tile_merge<2, true, 8, true, true><<<gs, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
    } else if (staged) {
        if (nparts <= 2)
            k_tile_part<1, true, 2, true><<<gs, AGG_THREADS, nparts * sm1, s>>>(P, nparts, n, out, flags, epoch, st);
        else if (nparts <= 4)
            k_tile_merge<2, true, 4, true><<<gs, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
        else
            k_tile_merge<2, true, 8, true><<<gs, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
    } else if (flags) {
        if (nparts <= 2)
            k_tile_part<1, true, 2><<<g, AGG_THREADS, nparts * sm1, s>>>(P, nparts, n, out, flags, epoch, st);
        else if (nparts <= 4)
            k_tile_merge<2, true, 4><<<g, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
        else
            k_tile_merge<2, true, 8><<<g, AGG_THREADS, 0, s>>>(P, nparts, n, out, flags, epoch, st);
    } else if (!avg) {
        k_tile_part<0, false, 1><<<g, AGG_THREADS, sm1, s>>>(P, nparts, n, out, nullptr, 0, st);
    } else if (nparts == 1) {
        k_tile_part<1, false, 1><<<g, AGG_THREADS, sm1, s>>>(P, nparts, n, out, nullptr, 0, st);
    } else if (nparts == 2) {
        k_tile_part<1, false, 2><<<g, AGG_THREADS, sm2, s>>>(P, nparts, n, out, nullptr, 0, st);
    } else if (nparts <= 4) {
        k_tile_merge<2, false, 4><<<g, AGG_THREADS, 0, s>>>(P, nparts, n, out, nullptr, 0, st);
    } else {
        k_tile_merge<2, false, 8><<<g, AGG_THREADS, 0, s>>>(P, nparts, n, out, nullptr, 0, st);
    }
    return GVC_OK;
}

int aggregate_run(const uint32_t *idx, const float *vals, const uint64_t *offs, const uint64_t *counts,
                  int nparts, uint64_t n, float *out, void *ws, size_t ws_bytes, const uint32_t *bounds,
                  uint64_t bounds_stride, cudaStream_t s)
{
    if (nparts < 1 || nparts > AGG_MAX_PARTS)
        return set_error(GVC_ERR_ARG, "aggregate: nparts %d outside [1, %d]", nparts, AGG_MAX_PARTS);
    AggParts P;
    for (int p = 0; p < nparts; p++) {
        P.idx[p] = idx + offs[p];
        P.vals[p] = vals + offs[p];
        P.bounds[p] = bounds ? bounds + (uint64_t)p * bounds_stride : nullptr;
        P.cnt[p] = counts[p];
    }
    return tile_merge_run(true, P, nparts, n, out, ws, ws_bytes, nullptr, 0, s);
}

int decompress_run(const uint32_t *idx, const float *vals, uint64_t k, uint64_t n, float *out, void *ws,
                   size_t ws_bytes, cudaStream_t s)
{
    AggParts P;
    P.idx[0] = idx;
    P.vals[0] = vals;
    P.bounds[0] = nullptr;
    P.cnt[0] = k;
    return tile_merge_run(false, P, 1, n, out, ws, ws_bytes, nullptr, 0, s);
}

// ------------------------------------------------ peer-memory exchange (C1+K7)
// Rank `rank` posts `epoch` into slot [rank] of every rank's flag array (its
// own included) once its payload is complete.  The payload was written by
// earlier kernels of this stream, so it sits in this GPU's L2 -- the point
// of coherence for the peers' NVLink reads -- and the system-scope fence +
// release store order the flag after it.
__global__ void k_peer_signal(PeerFlags f, int nranks, int rank, uint32_t epoch)
{
    const int q = threadIdx.x;
    if (q < nranks) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.flags[q] + rank), "r"(epoch) : "memory");
    }
}

int peer_signal_run(uint32_t *const *peer_flags, int nranks, int rank, uint32_t epoch, cudaStream_t s)
{
    if (nranks < 1 || nranks > GVC_MAX_PEERS || rank < 0 || rank >= nranks)
        return set_error(GVC_ERR_ARG, "peer_signal: rank %d of %d (at most %d ranks)", rank, nranks, GVC_MAX_PEERS);
    PeerFlags f;
    for (int q = 0; q < nranks; q++) {
        if (!peer_flags[q])
            return set_error(GVC_ERR_ARG, "peer_signal: null flag pointer of rank %d", q);
        f.flags[q] = peer_flags[q];
    }
    count_launches(1);
    k_peer_signal<<<1, 32, 0, s>>>(f, nranks, rank, epoch);
    return GVC_OK;
}

int aggregate_peers_run(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                        const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                        float *out, cudaStream_t s)
{
    if (nparts < 1 || nparts > GVC_MAX_PEERS)
        return set_error(GVC_ERR_ARG, "aggregate_peers: nparts %d outside [1, %d]", nparts, GVC_MAX_PEERS);
    if (!flags)
        return set_error(GVC_ERR_ARG, "aggregate_peers: null flags");
    AggParts P;
    for (int p = 0; p < nparts; p++) {
        if (!idx[p] || !vals[p] || !bounds[p])
            return set_error(GVC_ERR_ARG, "aggregate_peers: part %d has a null pointer", p);
        P.idx[p] = idx[p];
        P.vals[p] = vals[p];
        P.bounds[p] = bounds[p];
        P.cnt[p] = counts[p];
    }
    return tile_merge_run(true, P, nparts, n, out, nullptr, 0, flags, epoch, s);
}

int aggregate_peers_staged_run(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                               const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                               const gvc_peer_staging *sg, float *out, cudaStream_t s)
{
    if (nparts < 1 || nparts > GVC_MAX_PEERS)
        return set_error(GVC_ERR_ARG, "aggregate_peers_staged: nparts %d outside [1, %d]", nparts, GVC_MAX_PEERS);
    if (!flags || !sg || !sg->ready_dev || sg->self < 0 || sg->self >= nparts || sg->copy_blocks < 1)
        return set_error(GVC_ERR_ARG, "aggregate_peers_staged: bad flags / staging");
    const uint32_t ce = sg->chunk_entries;
    if (ce < 4 || (ce & (ce - 1)))
        return set_error(GVC_ERR_ARG, "aggregate_peers_staged: chunk_entries %u is not a power of two >= 4", ce);
    AggParts P;
    Staged st;
    memset(&st, 0, sizeof(st));
    st.ncopy = sg->copy_blocks;
    st.self = sg->self;
    st.ch_log2 = (uint32_t)__builtin_ctz(ce);
    st.ready = sg->ready_dev;
    st.err = const_cast<uint32_t *>(flags) + GVC_FLAG_ERR_WORD;
    st.ticket = const_cast<uint32_t *>(flags) + GVC_FLAG_TICKET_WORD;
    uint64_t kmax = 0;
    for (int p = 0; p < nparts; p++) {
        if (!idx[p] || !vals[p] || !bounds[p] || (p != sg->self && (!sg->src_idx_dev[p] || !sg->src_vals_dev[p])))
            return set_error(GVC_ERR_ARG, "aggregate_peers_staged: part %d has a null pointer", p);
        P.idx[p] = idx[p];
        P.vals[p] = vals[p];
        P.bounds[p] = bounds[p];
        P.cnt[p] = counts[p];
        st.src_idx[p] = sg->src_idx_dev[p];
        st.src_val[p] = sg->src_vals_dev[p];
        st.src_bounds[p] = sg->src_bounds_dev[p];
        st.src_off[p] = sg->src_off16_dev[p];
        st.off[p] = sg->off16_dev[p];
        if (p != sg->self && !sg->src_bounds_dev[p])
            return set_error(GVC_ERR_ARG, "aggregate_peers_staged: part %d has no source bounds", p);
        kmax = counts[p] > kmax ? counts[p] : kmax;
    }
    // 16-bit wire indices only when every part has them (local and remote)
    st.use_off = 1;
    for (int p = 0; p < nparts; p++)
        if (!st.off[p] || (p != sg->self && !st.src_off[p]))
            st.use_off = 0;
    st.nchunks = (uint32_t)((kmax + ce - 1) / ce);
    st.nb = (uint32_t)((n + AGG_TILE - 1) / AGG_TILE + 1);
    return tile_merge_run(true, P, nparts, n, out, nullptr, 0, flags, epoch, s, &st);
}

int tile_bounds_run(const uint32_t *idx, uint64_t k, uint64_t n, uint32_t *bounds, cudaStream_t s)
{
    AggParts P;
    P.idx[0] = idx;
    P.cnt[0] = k;
    const uint64_t ntiles = (n + AGG_TILE - 1) / AGG_TILE;
    count_launches(1);
    k_tile_bounds<<<dim3((unsigned)grid_for(k + 1, 256, 1024), 1), 256, 0, s>>>(P, 1, ntiles, bounds);
    return GVC_OK;
}

// --------------------------------------------------------- dense average
__global__ void k_aggregate_dense(const float *__restrict__ parts, int nparts, uint64_t n, float *__restrict__ out)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        double acc = 0.0;
        for (int p = 0; p < nparts; p++)
            acc += (double)parts[(uint64_t)p * n + i];
        out[i] = (float)(acc / (double)nparts);
    }
}

int aggregate_dense_run(const float *parts, int nparts, uint64_t n, float *out, cudaStream_t s)
{
    if (nparts < 1)
        return set_error(GVC_ERR_ARG, "aggregate_dense of zero parts");
    count_launches(1);
    k_aggregate_dense<<<grid_for(n, 256, device_sms() * 16), 256, 0, s>>>(parts, nparts, n, out);
    return GVC_OK;
}

// ------------------------------------------------ C3 over peer memory
// The dense fallback's exchange + mean (controller.py:259-264 -> aggregate_dense,
// compressors.py:274-285) as a reduce-scatter + all-gather fused over NVLink:
// every rank's dense input sits in its peer-mapped buffer; rank `rank` owns
// the float4 range [lo4, hi4), sums the W inputs there in fp64 in rank order,
// divides by W and rounds to fp32 -- aggregate_dense's arithmetic -- and
// writes the result range into EVERY rank's buffer, over the inputs (only the
// owner reads that range).  Each rank moves 2 (W-1)/W of the vector over
// NVLink instead of receiving W-1 whole vectors.
struct DensePeers {
    float *buf[GVC_MAX_PEERS];
};

// Bounded wait for flags[q] >= epoch (q < W); bit 4 of *err on timeout.
__device__ __forceinline__ void wait_peer_flags(const uint32_t *flags, int W, uint32_t epoch, uint32_t *err)
{
    if (threadIdx.x < W) {
        const long long t0 = clock64();
        while ((int32_t)(ld_acquire_sys(flags + threadIdx.x) - epoch) < 0) {
            __nanosleep(64);
            if (clock64() - t0 > (1ll << 33)) {  // ~4 s: a rank died or diverged
                atomicOr(err, 4u);
                break;
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_dense_mean_peers(DensePeers P, int W, uint64_t lo4, uint64_t hi4,
                                                          const uint32_t *flags, uint32_t epoch, uint32_t *err)
{
    wait_peer_flags(flags, W, epoch, err);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const double inv = 1.0 / (double)W;
    (void)inv;
    for (uint64_t i = lo4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi4; i += stride) {
        float4 x[GVC_MAX_PEERS];
#pragma unroll
        for (int q = 0; q < GVC_MAX_PEERS; q++)
            if (q < W)
                x[q] = __ldcg(reinterpret_cast<const float4 *>(P.buf[q]) + i);
        double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
#pragma unroll
        for (int q = 0; q < GVC_MAX_PEERS; q++) {
            if (q < W) {
                a += (double)x[q].x;
                b += (double)x[q].y;
                c += (double)x[q].z;
                d += (double)x[q].w;
            }
        }
        const float4 o = make_float4((float)(a / (double)W), (float)(b / (double)W), (float)(c / (double)W),
                                     (float)(d / (double)W));
#pragma unroll
        for (int q = 0; q < GVC_MAX_PEERS; q++)
            if (q < W)
                __stcg(reinterpret_cast<float4 *>(P.buf[q]) + i, o);
    }
    __threadfence_system();  // the result ranges are visible at every peer before this rank signals
}

// Wait until every rank wrote its result range into this buffer, then copy the
// mean out of the peer-mapped buffer.
__global__ void __launch_bounds__(256) k_dense_collect(const float *own, float *out, uint64_t n, const uint32_t *flags,
                                                       int W, uint32_t epoch, uint32_t *err)
{
    wait_peer_flags(flags, W, epoch, err);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n4 = n / 4;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
        __stcs(reinterpret_cast<float4 *>(out) + i, __ldcg(reinterpret_cast<const float4 *>(own) + i));
    for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = __ldcg(own + i);
}

int dense_mean_peers_run(float *const *bufs, int nranks, int rank, uint64_t n, const uint32_t *flags,
                         uint32_t epoch, uint32_t *err, cudaStream_t s)
{
    if (nranks < 1 || nranks > GVC_MAX_PEERS || rank < 0 || rank >= nranks || !flags || !err)
        return set_error(GVC_ERR_ARG, "dense_mean_peers: rank %d of %d", rank, nranks);
    DensePeers P;
    for (int q = 0; q < nranks; q++) {
        if (!bufs[q] || ((uintptr_t)bufs[q] & 15))
            return set_error(GVC_ERR_ARG, "dense_mean_peers: buffer of rank %d null or not 16-byte aligned", q);
        P.buf[q] = bufs[q];
    }
    const uint64_t n4 = (n + 3) / 4;  // the buffers hold n rounded up to 4 floats
    const uint64_t lo4 = n4 * rank / nranks, hi4 = n4 * (rank + 1) / nranks;
    const int sms = device_sms();
    count_launches(1);
    k_dense_mean_peers<<<grid_for(hi4 - lo4, 256, sms * 8), 256, 0, s>>>(P, nranks, lo4, hi4, flags, epoch, err);
    return GVC_OK;
}

int dense_collect_run(const float *own, float *out, uint64_t n, const uint32_t *flags, int nranks, uint32_t epoch,
                      uint32_t *err, cudaStream_t s)
{
    if (!own || !out || !flags || !err || nranks < 1 || nranks > GVC_MAX_PEERS)
        return set_error(GVC_ERR_ARG, "dense_collect: bad arguments");
    const int sms = device_sms();
    count_launches(1);
    k_dense_collect<<<grid_for(n / 4 + 1, 256, sms * 8), 256, 0, s>>>(own, out, n, flags, nranks, epoch, err);
    return GVC_OK;
}

// Layerwise per-segment path: segment-local output positions -> global
// indices (idx[j] += start of the segment whose outputs hold j), one launch
// for every segment; the segment of j by binary search over the output
// offsets staged in shared memory.
__global__ void k_add_seg_offsets(uint32_t *idx, uint64_t total, const uint64_t *out_off, const uint64_t *starts,
                                  int nseg)
{
    extern __shared__ uint64_t so[];  // [nseg + 1] offsets, then [nseg] starts
    for (int q = threadIdx.x; q <= nseg; q += blockDim.x)
        so[q] = out_off[q];
    for (int q = threadIdx.x; q < nseg; q += blockDim.x)
        so[nseg + 1 + q] = starts[q];
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += stride) {
        int lo = 0, hi = nseg - 1;  // last q with so[q] <= j
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (so[mid] <= j)
                lo = mid;
            else
                hi = mid - 1;
        }
        idx[j] += (uint32_t)so[nseg + 1 + lo];
    }
}

int add_seg_offsets_run(uint32_t *idx, uint64_t total, const uint64_t *out_off, const uint64_t *starts, int nseg,
                        cudaStream_t s)
{
    if (nseg < 1 || nseg > 3000 || !idx || !out_off || !starts)  // (<= 48 KB of shared memory)
        return set_error(GVC_ERR_ARG, "add_seg_offsets: %d segments", nseg);
    if (!total)
        return GVC_OK;
    const size_t smem = (size_t)(2 * nseg + 1) * 8;
    count_launches(1);
    k_add_seg_offsets<<<grid_for(total, 256, device_sms() * 8), 256, smem, s>>>(idx, total, out_off, starts, nseg);
    return GVC_OK;
}

__global__ void k_iota(uint32_t *out, uint64_t n)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (uint32_t)i;
}

int iota_run(uint32_t *out, uint64_t n, cudaStream_t s)
{
    count_launches(1);
    k_iota<<<grid_for(n, 256, device_sms() * 16), 256, 0, s>>>(out, n);
    return GVC_OK;
}

}  // namespace gvc
