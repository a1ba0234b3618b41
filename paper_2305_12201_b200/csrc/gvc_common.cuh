// gvc_common.cuh -- shared device helpers for the GraVAC sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gravac_b200.h"

#define GVC_WARPS_PER_BLOCK 8
#define GVC_THREADS (GVC_WARPS_PER_BLOCK * 32)
// Segments: the input is cut into S contiguous ranges, one per warp of the
// collect kernel.  S depends only on n (never on the device), so every
// reduction order is a function of the input size alone.
#ifndef GVC_COLLECT_PREFETCH
#define GVC_COLLECT_PREFETCH 1
#endif
#if GVC_COLLECT_PREFETCH
#define GVC_COLLECT_BLOCKS 4  // register double buffer: 64 regs
#else
#define GVC_COLLECT_BLOCKS 5  // no register buffer: 48 regs, latency hidden by warps
#endif
// 148 SMs x resident collect blocks x 8 warps: the collect grid is one full wave
#define GVC_SEG_TARGET (148 * GVC_COLLECT_BLOCKS * 8)
#define GVC_SEG_MAX 16384
#define GVC_MEM_FLAT (1u << 22)  // flat member-key list of the level-1 refinement (16 MB)
#define GVC_STAGE 256        // per-warp candidate staging ring in k_collect (entries)
#define GVC_SEG_QUANTUM 512  // elements per warp iteration: 32 lanes x 4 float4
#define GVC_H0_BINS 4096     // level-0 histogram (shared memory, 16 KB)
#define GVC_HL_BINS 4096     // refinement histogram per ladder entry (global)
#define GVC_BLK_MAX (GVC_SEG_MAX / GVC_WARPS_PER_BLOCK)
#define GVC_SAMPLE_BINS 16384  // shared-memory sample histogram (64 KB)
#define GVC_SAMPLE_SHIFT 17    // 31-bit magnitude key >> 17 -> 14-bit bin (1/64 octave)
#define GVC_MAX_LEVELS 3

namespace gvc {

// KEY_MAG: 31-bit |v|; KEY_HASH: Philox position hash (Random-k); KEY_DGC:
// DGC's composite key (gvc_select_args.dgc_thr_dev), 32-bit.
// KEY_POS: equal nonzero magnitudes (a Redsync level-1 output): nonzero first,
// then lower position -- the magnitude order with its ties already broken
enum KeyMode { KEY_MAG = 0, KEY_HASH = 1, KEY_DGC = 2, KEY_POS = 3 };

// |x| as an order-preserving integer: clear the sign bit (-0 -> 0).  Monotone
// for every non-NaN float; NaN keys are > 0x7f800000.
// Programmatic dependent launch: a select kernel lets its successor launch
// as soon as all its CTAs are running, and waits for its predecessor's
// completion (and memory) before touching its outputs.  Both are no-ops when
// the kernel was launched without the attribute.
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7fffffffu; }

// Philox4x32-10 (Salmon et al. SC'11), output word 0.  Counter-based position
// hash replacing numpy Generator.choice (gradcore.py:144-149): counter =
// (lo i, hi i, lo stream, hi stream), key = (lo seed, hi seed).
__device__ __forceinline__ uint32_t philox_x0(uint64_t i, uint64_t stream, uint64_t seed)
{
    uint32_t c0 = (uint32_t)i, c1 = (uint32_t)(i >> 32), c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return c0;
}

// DGC's threshold sample: one position per stratum [j n / s, (j + 1) n / s),
// offset = Philox word 0 at counter (pos_base + lo_j, stream) scaled to the
// stratum width (the C-ABI header states the definition).
// floor(j n / s) without a 64-bit integer division: with n < 2^32 and
// j <= s <= n, j n fits 64 bits and the fp64 quotient is within 2^-20 of the
// true one, so one correction step makes the floor exact
__device__ __forceinline__ uint64_t stratum_lo(uint64_t j, uint64_t n, uint64_t s, double inv_s)
{
    const uint64_t a = j * n;
    uint64_t q = (uint64_t)((double)a * inv_s);
    if (q * s > a)
        q--;
    else if ((q + 1) * s <= a)
        q++;
    return q;
}

__device__ __forceinline__ uint32_t dgc_position(uint64_t j, uint64_t n, uint64_t s, double inv_s, uint64_t seed,
                                                 uint64_t stream, uint64_t pos_base)
{
    const uint64_t lo = stratum_lo(j, n, s, inv_s), hi = stratum_lo(j + 1, n, s, inv_s);
    const uint32_t h = philox_x0(pos_base + lo, stream, seed);
    return (uint32_t)(lo + (((uint64_t)h * (hi - lo)) >> 32));
}

// All four output words of Philox4x32-10 at counter (lo i, hi i, lo stream,
// hi stream).
__device__ __forceinline__ uint4 philox4(uint64_t i, uint64_t stream, uint64_t seed)
{
    uint32_t c0 = (uint32_t)i, c1 = (uint32_t)(i >> 32), c2 = (uint32_t)stream, c3 = (uint32_t)(stream >> 32);
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// Random-k selection key of position pos: word (pos & 3) of Philox4x32-10 at
// counter (pos >> 2, stream) -- one Philox evaluation serves four consecutive
// positions.  The k SMALLEST hashes win, so the key (larger wins) is the
// bitwise complement.
__device__ __forceinline__ uint32_t hash_key(uint64_t pos, uint64_t stream, uint64_t seed)
{
    const uint4 h = philox4(pos >> 2, stream, seed);
    const uint32_t w = (uint32_t)pos & 3u;
    return ~(w == 0 ? h.x : w == 1 ? h.y : w == 2 ? h.z : h.w);
}

// The keys of positions 4q .. 4q + 3 from one evaluation.
__device__ __forceinline__ uint4 hash_key4(uint64_t pos4, uint64_t stream, uint64_t seed)
{
    const uint4 h = philox4(pos4 >> 2, stream, seed);
    return make_uint4(~h.x, ~h.y, ~h.z, ~h.w);
}

__device__ __forceinline__ double warp_sum_f64(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t lanemask_lt()
{
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int bitlen64(uint64_t x) { return x ? 64 - __clzll((long long)x) : 0; }

// Exclusive prefix sum across a block of up to 1024 threads (warp shuffles, 2 barriers).
// `sh` must hold 33 u64; *total (optional) receives the block total.
__device__ __forceinline__ unsigned long long block_excl_prefix(unsigned long long v, unsigned long long *sh,
                                                                unsigned long long *total = nullptr)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nwarps = (int)(blockDim.x >> 5);
        unsigned long long w = lane < nwarps ? sh[lane] : 0ull, wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o)
                wi += y;
        }
        sh[lane] = wi - w;
        if (lane == 31)
            sh[32] = wi;
    }
    __syncthreads();
    unsigned long long r = sh[warp] + x - v;
    if (total)
        *total = sh[32];
    __syncthreads();
    return r;
}

// Deterministic fp64 sum across a block (<= 1024 threads): fixed xor tree per warp,
// then warps added in index order.  `sh` must hold 33 doubles.
__device__ __forceinline__ double block_sum_f64(double v, double *sh)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum_f64(v);
    if (lane == 0)
        sh[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        const int nwarps = (int)(blockDim.x >> 5);
        for (int w = 0; w < nwarps; w++)
            r += sh[w];
        sh[32] = r;
    }
    __syncthreads();
    double r = sh[32];
    __syncthreads();
    return r;
}

// Deferred residual (gvc_select_args.pending_*): the true residual of a sent
// position whose buffer still holds g_ef.
__device__ __forceinline__ float pending_resid(float r, int mode, float m)
{
    if (mode == 2) {
        const float sg = r > 0.f ? 1.f : (r < 0.f ? -1.f : 0.f);
        return __fsub_rn(r, __fmul_rn(sg, m));
    }
    return __fsub_rn(r, r);
}

// ------------------------------------------------------- grid barriers
// For cooperative launches only (every CTA is resident, so a CTA spinning here
// cannot starve one that has not started).  The counters live in the select
// state, which is zeroed before every launch, so each barrier instance is
// used once.  Spins are bounded: after ~4 s the barrier gives up and sets
// bit 4 of *err (reported as GVC_ERR_STATE) instead of hanging the GPU.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

#define GVC_SPIN_LIMIT (1ll << 33)  // clock64 ticks (~4 s at 1.9 GHz)

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// All CTAs arrive; the CTA that arrives last runs `last_fn()` (whole block)
// before the others are released, so its global writes are visible to every
// CTA after the barrier.  Release/acquire at gpu scope by one thread per CTA
// (bar.sync orders the rest of the block); read what other CTAs wrote with
// ld_cg, ideally once per CTA (a line every thread of the grid polls is an L2
// hot spot).
template <typename F>
__device__ __forceinline__ void grid_sync_last(uint32_t *bar, uint32_t nblocks, uint32_t *err, F last_fn)
{
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        s_last = atomicAdd(&bar[0], 1u) == nblocks - 1;
        if (s_last)
            fence_acq_rel_gpu();
    }
    __syncthreads();
    if (s_last) {
        last_fn();
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_acq_rel_gpu();
            st_release_u32(&bar[1], 1u);
        }
    } else if (threadIdx.x == 0) {
        const long long t0 = clock64();
        while (ld_acquire_u32(&bar[1]) == 0u) {
            __nanosleep(32);
            if (clock64() - t0 > GVC_SPIN_LIMIT) {
                atomicOr(err, 4u);
                break;
            }
        }
    }
    __syncthreads();
}

template <typename T>
__device__ __forceinline__ T ld_cg(const T *p)
{
    return __ldcg(p);
}

// One L2 read per CTA of a value another CTA wrote, broadcast through shared
// memory (contains a __syncthreads).
template <typename T>
__device__ __forceinline__ T bcast_cg(const T *p)
{
    __shared__ T v;
    __syncthreads();
    if (threadIdx.x == 0)
        v = __ldcg(p);
    __syncthreads();
    return v;
}

// Streaming loads / stores: the gradient and residual are touched once per
// step, so they should not displace the candidate buffer in L2.
__device__ __forceinline__ float4 ld_stream(const float4 *p) { return __ldcs(p); }
// 16-byte global -> shared copy that holds no register (L2 only), and its groups
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait()
{
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) { __stcs(p, v); }

}  // namespace gvc
