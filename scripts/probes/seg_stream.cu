// Does per-warp contiguous-segment streaming (the k_collect access pattern)
// reach the same HBM bandwidth as a grid-stride stream?  r = g + r over 44.5M
// floats, 12 B/value.  Development probe: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gridstride(const float4 *g, float4 *r, size_t n4)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        float4 a = __ldcs(g + i), b = __ldcs(r + i);
        a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        __stcs(r + i, a);
    }
}

// one warp per contiguous segment, 256 values (2 float4 per lane) per step,
// the next step's loads issued before this step's add (k_collect's pipeline)
template <int U>
__global__ void __launch_bounds__(256) segstream(const float *g, float *r, size_t n, size_t seg_len, int nseg)
{
    const int lane = threadIdx.x & 31;
    const int seg = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (seg >= nseg)
        return;
    const size_t beg = (size_t)seg * seg_len;
    const size_t len = min(seg_len, n - beg);
    const float4 *gs = reinterpret_cast<const float4 *>(g + beg);
    float4 *rs = reinterpret_cast<float4 *>(r + beg);
    const size_t steps = len / (128 * U);
    float4 a[U], b[U];
    for (int u = 0; u < U; u++) {
        a[u] = __ldcs(gs + u * 32 + lane);
        b[u] = __ldcs(rs + u * 32 + lane);
    }
    for (size_t s = 0; s < steps; s++) {
        float4 na[U], nb[U];
        const bool more = s + 1 < steps;
        if (more)
            for (int u = 0; u < U; u++) {
                na[u] = __ldcs(gs + (s + 1) * 32 * U + u * 32 + lane);
                nb[u] = __ldcs(rs + (s + 1) * 32 * U + u * 32 + lane);
            }
        for (int u = 0; u < U; u++) {
            float4 x = a[u];
            x.x += b[u].x; x.y += b[u].y; x.z += b[u].z; x.w += b[u].w;
            __stcs(rs + s * 32 * U + u * 32 + lane, x);
        }
        if (more)
            for (int u = 0; u < U; u++) {
                a[u] = na[u];
                b[u] = nb[u];
            }
    }
}

int main()
{
    const size_t n = 44500000, n4 = n / 4;
    float *g, *r, *flush;
    cudaMalloc(&g, n * 4);
    cudaMalloc(&r, n * 4);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(g, 0, n * 4);
    cudaMemset(r, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        float best = 1e9f;
        for (int it = 0; it < 20; it++) {
            cudaMemset(flush, it, 256 << 20);
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 2 && ms < best)
                best = ms;
        }
        printf("%-40s %8.1f us  %6.0f GB/s\n", name, best * 1e3, 12.0 * n / (best * 1e-3) / 1e9);
    };
    for (int blocks : {148 * 4, 148 * 8, 148 * 16})
        run(blocks == 592 ? "gridstride 592x256" : blocks == 1184 ? "gridstride 1184x256" : "gridstride 2368x256",
            [&] { gridstride<<<blocks, 256>>>((const float4 *)g, (float4 *)r, n4); });
    for (int wpsm : {32, 48, 64}) {
        const int nseg = 148 * wpsm;
        size_t seg_len = ((n + nseg - 1) / nseg + 511) / 512 * 512;
        int nsegs = (int)((n + seg_len - 1) / seg_len);
        char name[64];
        snprintf(name, sizeof name, "segstream U=2, %d warps/SM", wpsm);
        run(name, [&] { segstream<2><<<(nsegs + 7) / 8, 256>>>(g, r, n, seg_len, nsegs); });
        snprintf(name, sizeof name, "segstream U=4, %d warps/SM", wpsm);
        run(name, [&] { segstream<4><<<(nsegs + 7) / 8, 256>>>(g, r, n, seg_len, nsegs); });
    }
    return 0;
}
