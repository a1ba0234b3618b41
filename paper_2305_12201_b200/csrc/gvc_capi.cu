// gvc_capi.cu -- extern "C" entry points of libgravac_b200.so (include/gravac_b200.h).
// Argument validation mirrors the reference's ValueError checks; the kernels
// live in gvc_select.cu / gvc_dense.cu.
#include <atomic>
#include <mutex>
#include <stdarg.h>
#include <vector>
#include <stdio.h>
#include <string.h>

#include "gvc_internal.h"

namespace gvc {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

// ---------------------------------------------------------------- profiler
static std::mutex g_prof_mu;
static bool g_prof_on = false;     // mode 1: direct launches bracketed by events
static bool g_prof_graph = false;  // mode 2: event-record nodes around k_collect inside the select graph
static uint64_t g_prof_min_n = 0;  // only selects / emits of at least this many values are probed
static std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> g_prof_pending;
static std::vector<cudaEvent_t> g_prof_free;
static double g_prof_ms[PROF_NCAT];
static unsigned long long g_prof_cnt[PROF_NCAT];
static std::atomic<unsigned long long> g_launches{0};

static cudaEvent_t prof_event()
{
    if (!g_prof_free.empty()) {
        cudaEvent_t e = g_prof_free.back();
        g_prof_free.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(int cat, cudaStream_t st) : slot(-1), s(st)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    // mode 2 (graph probes) still brackets the directly launched emit / average
    const bool on = g_prof_on || (g_prof_graph && (cat == PROF_EMIT || cat == PROF_AGGREGATE));
    if (!on || cat < 0)
        return;
    cudaEvent_t a = prof_event(), b = prof_event();
    cudaEventRecord(a, s);
    g_prof_pending.push_back({cat, {a, b}});
    slot = (int)g_prof_pending.size() - 1;
}

ProfScope::~ProfScope()
{
    if (slot < 0)
        return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_prof_pending[slot].second.second, s);
}

void count_launches(int n) { g_launches += (unsigned long long)n; }

bool prof_enabled()
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    return g_prof_on;
}

bool prof_wants(uint64_t n)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    return n >= g_prof_min_n;
}

bool prof_graph_enabled()
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    return g_prof_graph && !g_prof_on;
}

void prof_graph_pair(int cat, cudaEvent_t *a, cudaEvent_t *b)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    *a = prof_event();
    *b = prof_event();
    g_prof_pending.push_back({cat, {*a, *b}});
}

static int check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_error(GVC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return GVC_OK;
}

}  // namespace gvc

using namespace gvc;

#define STREAM(s) ((cudaStream_t)(s))

extern "C" {

const char *gvc_last_error(void) { return g_err; }

int gvc_abi_version(void) { return GVC_ABI_VERSION; }

void gvc_prof_min_n(uint64_t n)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_min_n = n;
}

void gvc_prof_enable(int on)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on == 1;
    g_prof_graph = on == 2;
    // pre-create events so the timed region never pays cudaEventCreate
    while ((g_prof_on || g_prof_graph) && g_prof_free.size() < 4096) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess)
            break;
        g_prof_free.push_back(e);
    }
}

int gvc_prof_read(double *ms, unsigned long long *counts, int ncat)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &pe : g_prof_pending) {
        float t = 0.f;
        cudaEventSynchronize(pe.second.second);
        if (cudaEventElapsedTime(&t, pe.second.first, pe.second.second) == cudaSuccess) {
            g_prof_ms[pe.first] += t;
            g_prof_cnt[pe.first] += 1;
        }
        g_prof_free.push_back(pe.second.first);
        g_prof_free.push_back(pe.second.second);
    }
    g_prof_pending.clear();
    for (int c = 0; c < ncat && c < PROF_NCAT; c++) {
        ms[c] = g_prof_ms[c];
        counts[c] = g_prof_cnt[c];
        g_prof_ms[c] = 0.0;
        g_prof_cnt[c] = 0;
    }
    return PROF_NCAT;
}

unsigned long long gvc_launch_count(void) { return g_launches.load(); }

int gvc_select_phase_times(void *ws, unsigned long long *out, int n)
{
    if (!ws || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_select_phase_times: bad arguments");
    return select_phase_times(ws, out, n);
}

size_t gvc_select_workspace_bytes(int kind, uint64_t n) { return select_workspace_bytes(kind, n); }

int gvc_select(const gvc_select_args *a, void *ws, size_t ws_bytes, gvc_select_result *res, void *stream)
{
    if (!a || !ws || !res)
        return set_error(GVC_ERR_ARG, "gvc_select: null argument");
    if (a->kind < GVC_TOPK || a->kind > GVC_RANDOMK)
        return set_error(GVC_ERR_ARG, "unknown compressor kind %d", a->kind);
    if (a->kind == GVC_DGC && !a->dgc_thr_dev)
        return set_error(GVC_ERR_ARG, "dgc selects need dgc_thr_dev and dgc_sampled_dev (gvc_dgc_sample + gvc_select "
                                      "over the sample give the threshold)");
    if (a->dgc_thr_dev && (!a->dgc_sampled_dev || a->n_ks != 1 || a->key_est_dev || a->force_exact ||
                           a->kind == GVC_RANDOMK || a->kind == GVC_REDSYNC))
        return set_error(GVC_ERR_ARG, "dgc_thr_dev needs dgc_sampled_dev, one ladder entry and no forced threshold");
    if (a->equal_magnitudes &&
        (a->n_ks != 1 || !a->values_dev || a->g_dev || a->dgc_thr_dev || a->key_est_dev || a->pending_mask_dev ||
         (a->kind != GVC_TOPK && a->kind != GVC_REDSYNC) || a->n + a->pos_base >= (1ull << 31) - 1))
        return set_error(GVC_ERR_ARG, "equal_magnitudes needs plain mode, one ladder entry, Top-k or Redsync and "
                                      "n + pos_base < 2^31 - 1");
    if (a->allow_short && (!a->key_est_dev || a->n_ks != 1 || a->kind != GVC_TOPK))
        return set_error(GVC_ERR_ARG, "allow_short needs key_est_dev, one ladder entry and magnitude keys");
    if (a->n < 1 || a->n >= (1ull << 32))
        return set_error(GVC_ERR_ARG, "gradient length %llu outside [1, 2^32)", (unsigned long long)a->n);
    if (a->n_ks < 1 || a->n_ks > GVC_MAX_LADDER)
        return set_error(GVC_ERR_ARG, "ladder length %d outside [1, %d]", a->n_ks, GVC_MAX_LADDER);
    for (int j = 0; j < a->n_ks; j++) {
        if (a->ks[j] < 1 || a->ks[j] >= a->n)
            return set_error(GVC_ERR_ARG, "keep count %llu outside [1, n)", (unsigned long long)a->ks[j]);
        if (j && a->ks[j] > a->ks[j - 1])
            return set_error(GVC_ERR_ARG, "keep counts must be non-increasing");
    }
    const bool ef = a->g_dev != nullptr;
    if (a->pending_mask_dev && (!ef || a->pending_mode < 1 || a->pending_mode > 2 ||
                                (a->pending_mode == 2 && !a->pending_m_dev)))
        return set_error(GVC_ERR_ARG, "gvc_select: pending mask needs EF mode and mode 1 or 2 (+m)");
    if (ef ? (a->resid_dev == nullptr) : (a->values_dev == nullptr))
        return set_error(GVC_ERR_ARG, "gvc_select: need values_dev, or g_dev and resid_dev");
    const void *src = ef ? (const void *)a->g_dev : (const void *)a->values_dev;
    if (((uintptr_t)src & 15) || (ef && ((uintptr_t)a->resid_dev & 15)))
        return set_error(GVC_ERR_ARG, "gvc_select: inputs must be 16-byte aligned");
    return select_run(a, ws, ws_bytes, res, STREAM(stream));
}

int gvc_emit_mirrored(void *ws, size_t ws_bytes, int j, const uint32_t *idx_map, uint32_t *out_idx, float *out_val,
                      float *resid, uint32_t *sent_mask, float *sent_m, uint32_t *tile_bounds, double *stats,
                      const gvc_emit_mirrors *mirrors, void *stream)
{
    if (!ws || !out_idx || !out_val)
        return set_error(GVC_ERR_ARG, "gvc_emit: null argument");
    if (resid && sent_mask)
        return set_error(GVC_ERR_ARG, "gvc_emit: pass resid_dev or sent_mask_dev, not both");
    if (tile_bounds && idx_map)
        return set_error(GVC_ERR_ARG, "gvc_emit: tile bounds need output indices in selection order (no idx_map)");
    if (mirrors) {
        if (mirrors->count < 0 || mirrors->count >= GVC_MAX_PEERS)
            return set_error(GVC_ERR_ARG, "gvc_emit: %d mirrors (at most %d)", mirrors->count, GVC_MAX_PEERS - 1);
        for (int m = 0; m < mirrors->count; m++)
            if (!mirrors->idx_dev[m] || !mirrors->vals_dev[m] || (tile_bounds && !mirrors->bounds_dev[m]))
                return set_error(GVC_ERR_ARG, "gvc_emit: mirror %d has a null pointer", m);
    }
    return emit_run(ws, ws_bytes, j, idx_map, out_idx, out_val, resid, sent_mask, sent_m, tile_bounds, stats,
                    mirrors, STREAM(stream));
}

int gvc_emit(void *ws, size_t ws_bytes, int j, const uint32_t *idx_map, uint32_t *out_idx, float *out_val,
             float *resid, uint32_t *sent_mask, float *sent_m, uint32_t *tile_bounds, double *stats, void *stream)
{
    return gvc_emit_mirrored(ws, ws_bytes, j, idx_map, out_idx, out_val, resid, sent_mask, sent_m, tile_bounds,
                             stats, nullptr, stream);
}

int gvc_mark_sent(const uint32_t *idx, uint64_t k, uint32_t *mask, void *stream)
{
    if ((k && !idx) || !mask)
        return set_error(GVC_ERR_ARG, "gvc_mark_sent: bad arguments");
    int rc = mark_sent_run(idx, k, mask, STREAM(stream));
    return rc ? rc : check_launch("mark_sent");
}

int gvc_apply_pending(float *resid, uint32_t *mask, uint64_t n, int mode, const float *m, void *stream)
{
    if (!resid || !mask || n < 1 || mode < 1 || mode > 2 || (mode == 2 && !m))
        return set_error(GVC_ERR_ARG, "gvc_apply_pending: bad arguments");
    int rc = apply_pending_run(resid, mask, n, mode, m, STREAM(stream));
    return rc ? rc : check_launch("apply_pending");
}

int gvc_ef_add(const float *g, const float *r, float *out, uint64_t n, void *stream)
{
    if (!g || !r || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_ef_add: bad arguments");
    int rc = ef_add_run(g, r, out, n, STREAM(stream));
    return rc ? rc : check_launch("ef_add");
}

size_t gvc_sq_norm_workspace_bytes(uint64_t n) { return sq_norm_workspace_bytes(n); }

int gvc_sq_norm(const float *x, uint64_t n, double *out, void *ws, size_t ws_bytes, void *stream)
{
    if (!x || !out || n < 1)
        return set_error(GVC_ERR_ARG, "squared_l2_norm of empty vector");
    int rc = sq_norm_run(x, n, out, ws, ws_bytes, STREAM(stream));
    return rc ? rc : check_launch("sq_norm");
}

int gvc_update_residual(const float *ef, const uint32_t *idx, const float *vals, uint64_t k, uint64_t n,
                        float *resid, void *stream)
{
    if (!ef || !resid || n < 1 || (k && (!idx || !vals)))
        return set_error(GVC_ERR_ARG, "gvc_update_residual: bad arguments");
    int rc = update_residual_run(ef, idx, vals, k, n, resid, STREAM(stream));
    return rc ? rc : check_launch("update_residual");
}

int gvc_decompress(const uint32_t *idx, const float *vals, uint64_t k, uint64_t n, float *out, void *ws,
                   size_t ws_bytes, void *stream)
{
    if (!idx || !vals || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_decompress: bad arguments");
    int rc = decompress_run(idx, vals, k, n, out, ws, ws_bytes, STREAM(stream));
    return rc ? rc : check_launch("decompress");
}

size_t gvc_aggregate_workspace_bytes(int nparts, uint64_t n) { return aggregate_workspace_bytes(nparts, n); }

int gvc_aggregate(const uint32_t *idx, const float *vals, const uint64_t *offs, const uint64_t *counts,
                  int nparts, uint64_t n, float *out, void *ws, size_t ws_bytes, const uint32_t *bounds,
                  uint64_t bounds_stride, void *stream)
{
    if (nparts < 1)
        return set_error(GVC_ERR_ARG, "aggregate of zero parts");
    if (!idx || !vals || !offs || !counts || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_aggregate: bad arguments");
    int rc = aggregate_run(idx, vals, offs, counts, nparts, n, out, ws, ws_bytes, bounds, bounds_stride,
                           STREAM(stream));
    return rc ? rc : check_launch("aggregate");
}

int gvc_peer_signal(uint32_t *const *peer_flags, int nranks, int rank, uint32_t epoch, void *stream)
{
    if (!peer_flags)
        return set_error(GVC_ERR_ARG, "gvc_peer_signal: null flag array");
    int rc = peer_signal_run(peer_flags, nranks, rank, epoch, STREAM(stream));
    return rc ? rc : check_launch("peer_signal");
}

int gvc_aggregate_peers(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                        const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                        float *out, void *stream)
{
    if (!idx || !vals || !bounds || !counts || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_aggregate_peers: bad arguments");
    int rc = aggregate_peers_run(idx, vals, bounds, counts, nparts, n, flags, epoch, out, STREAM(stream));
    return rc ? rc : check_launch("aggregate_peers");
}

int gvc_aggregate_peers_staged(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                               const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                               const gvc_peer_staging *staging, float *out, void *stream)
{
    if (!idx || !vals || !bounds || !counts || !out || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_aggregate_peers_staged: bad arguments");
    int rc = aggregate_peers_staged_run(idx, vals, bounds, counts, nparts, n, flags, epoch, staging, out,
                                        STREAM(stream));
    return rc ? rc : check_launch("aggregate_peers_staged");
}

int gvc_dgc_sample(uint64_t n, uint64_t s, uint64_t seed, uint64_t rng_stream, uint64_t pos_base, uint32_t *out,
                   void *stream)
{
    if (!out)
        return set_error(GVC_ERR_ARG, "gvc_dgc_sample: null output");
    int rc = dgc_sample_run(n, s, seed, rng_stream, pos_base, out, STREAM(stream));
    return rc ? rc : check_launch("dgc_sample");
}

int gvc_dgc_sample_gather(uint64_t n, uint64_t s, uint64_t seed, uint64_t rng_stream, uint64_t pos_base,
                          const float *values, const float *g, const float *resid, const uint32_t *pending_mask,
                          const float *pending_m, int pending_mode, float *out, uint32_t *bits, void *stream)
{
    if (!out || !bits || (!values && (!g || !resid)) || (pending_mask && !g) || (pending_mode == 2 && !pending_m))
        return set_error(GVC_ERR_ARG, "gvc_dgc_sample_gather: bad arguments");
    int rc = dgc_sample_gather_run(n, s, seed, rng_stream, pos_base, values, g, resid, pending_mask, pending_m,
                                   pending_mode, out, bits, STREAM(stream));
    return rc ? rc : check_launch("dgc_sample_gather");
}

int gvc_tile_bounds(const uint32_t *idx, uint64_t k, uint64_t n, uint32_t *bounds, void *stream)
{
    if (!idx || !bounds || n < 1 || k > n)
        return set_error(GVC_ERR_ARG, "gvc_tile_bounds: bad arguments");
    int rc = tile_bounds_run(idx, k, n, bounds, STREAM(stream));
    return rc ? rc : check_launch("tile_bounds");
}

int gvc_aggregate_dense(const float *parts, int nparts, uint64_t n, float *out, void *stream)
{
    if (nparts < 1)
        return set_error(GVC_ERR_ARG, "aggregate of zero parts");
    int rc = aggregate_dense_run(parts, nparts, n, out, STREAM(stream));
    return rc ? rc : check_launch("aggregate_dense");
}

size_t gvc_segmented_select_workspace_bytes(uint64_t n, int nseg) { return segsel_workspace_bytes(n, nseg); }

int gvc_read_async(void *host_dst, const void *dev_src, size_t bytes, void *stream, void *side_stream,
                   void **events)
{
    if (!host_dst || !dev_src || !events)  // (a NULL stream is the legacy default stream)
        return set_error(GVC_ERR_ARG, "gvc_read_async: bad arguments");
    for (int e = 0; e < 2; e++)
        if (!events[e] && cudaEventCreateWithFlags((cudaEvent_t *)&events[e], cudaEventDisableTiming) != cudaSuccess)
            return set_error(GVC_ERR_CUDA, "gvc_read_async: event create");
    cudaEventRecord((cudaEvent_t)events[0], STREAM(stream));
    cudaStreamWaitEvent(STREAM(side_stream), (cudaEvent_t)events[0], 0);
    cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, STREAM(side_stream));
    cudaEventRecord((cudaEvent_t)events[1], STREAM(side_stream));
    return check_launch("read_async");
}

int gvc_event_record(void **event, void *stream)
{
    if (!event)
        return set_error(GVC_ERR_ARG, "gvc_event_record: null slot");
    if (!*event && cudaEventCreateWithFlags((cudaEvent_t *)event, cudaEventDisableTiming) != cudaSuccess)
        return set_error(GVC_ERR_CUDA, "gvc_event_record: event create");
    cudaEventRecord((cudaEvent_t)*event, STREAM(stream));
    return check_launch("event_record");
}

int gvc_copy_async(void *dst, const void *src, size_t bytes, void *stream)
{
    if (!dst || !src)
        return set_error(GVC_ERR_ARG, "gvc_copy_async: null pointer");
    cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, STREAM(stream));
    return check_launch("copy_async");
}

int gvc_stream_wait_event(void *stream, void *event)
{
    if (!event)
        return set_error(GVC_ERR_ARG, "gvc_stream_wait_event: null event");
    cudaStreamWaitEvent(STREAM(stream), (cudaEvent_t)event, 0);
    return check_launch("stream_wait_event");
}

int gvc_event_done(void *event)
{
    const cudaError_t e = cudaEventQuery((cudaEvent_t)event);
    if (e == cudaSuccess)
        return 1;
    if (e == cudaErrorNotReady)
        return 0;
    return set_error(GVC_ERR_CUDA, "gvc_event_done: %s", cudaGetErrorString(e));
}

size_t gvc_segmented_redsync_workspace_bytes(uint64_t total, int nseg)
{
    return seg_redsync_workspace_bytes(total, nseg);
}

int gvc_segmented_redsync_values(float *vals_dev, const uint64_t *out_off, const uint64_t *seg_len, int nseg,
                                 void *ws_dev, size_t ws_bytes, void *stream)
{
    if (!vals_dev || !out_off || !seg_len || nseg < 1 || !ws_dev)
        return set_error(GVC_ERR_ARG, "gvc_segmented_redsync_values: bad arguments");
    int rc = seg_redsync_run(vals_dev, out_off, seg_len, nseg, ws_dev, ws_bytes, STREAM(stream));
    return rc ? rc : check_launch("segmented_redsync_values");
}

int gvc_add_segment_offsets(uint32_t *idx_dev, uint64_t total, const uint64_t *out_off_dev,
                            const uint64_t *starts_dev, int nseg, void *stream)
{
    int rc = add_seg_offsets_run(idx_dev, total, out_off_dev, starts_dev, nseg, STREAM(stream));
    return rc ? rc : check_launch("add_segment_offsets");
}

int gvc_workspace_forget(void *ws)
{
    if (!ws)
        return set_error(GVC_ERR_ARG, "gvc_workspace_forget: null workspace");
    select_forget(ws);
    segsel_forget(ws);
    return GVC_OK;
}

size_t gvc_segmented_dgc_workspace_bytes(uint64_t n, int nseg, double sample_fraction)
{
    return seg_dgc_workspace_bytes(n, nseg, sample_fraction);
}

int gvc_segmented_dgc_select(const float *values_dev, uint64_t n, const uint64_t *seg_offsets, const uint64_t *seg_k,
                             int nseg, double sample_fraction, uint64_t seed, uint64_t rng_stream, uint32_t *out_idx_dev,
                             float *out_val_dev, void *ws_dev, size_t ws_bytes, uint32_t *status_dev, void *stream)
{
    if (!values_dev || !seg_offsets || !seg_k || nseg < 1 || !out_idx_dev || !out_val_dev || !ws_dev || !status_dev)
        return set_error(GVC_ERR_ARG, "segmented DGC: null argument or no segment");
    if (n >= (1ull << 32))
        return set_error(GVC_ERR_ARG, "segmented DGC: length %llu >= 2^32", (unsigned long long)n);
    int rc = seg_dgc_run(values_dev, n, seg_offsets, seg_k, nseg, sample_fraction, seed, rng_stream, out_idx_dev,
                         out_val_dev, ws_dev, ws_bytes, status_dev, STREAM(stream));
    return rc ? rc : check_launch("segmented_dgc_select");
}

int gvc_segmented_select(int kind, const float *values_dev, uint64_t n, const uint64_t *seg_offsets,
                         const uint64_t *seg_k, int nseg, uint64_t seed, uint64_t rng_stream, uint32_t *out_idx_dev,
                         float *out_val_dev, void *ws_dev, size_t ws_bytes, uint32_t *status_dev, void *stream)
{
    if (kind != GVC_TOPK && kind != GVC_RANDOMK)
        return set_error(GVC_ERR_ARG, "segmented select: Top-k and Random-k (DGC / Redsync go per segment)");
    if (!values_dev || !seg_offsets || !seg_k || nseg < 1 || !out_idx_dev || !out_val_dev || !ws_dev || !status_dev)
        return set_error(GVC_ERR_ARG, "segmented select: null argument or no segment");
    if (n >= (1ull << 32))
        return set_error(GVC_ERR_ARG, "segmented select: length %llu >= 2^32", (unsigned long long)n);
    int rc = segsel_run(kind, values_dev, n, seg_offsets, seg_k, nseg, seed, rng_stream, out_idx_dev, out_val_dev,
                        ws_dev, ws_bytes, status_dev, STREAM(stream));
    return rc ? rc : check_launch("segmented_select");
}

int gvc_dense_mean_peers(float *const *peer_bufs, int nranks, int rank, uint64_t n, const uint32_t *flags,
                         uint32_t epoch, uint32_t *err_dev, void *stream)
{
    if (!peer_bufs)
        return set_error(GVC_ERR_ARG, "gvc_dense_mean_peers: null buffer table");
    int rc = dense_mean_peers_run(peer_bufs, nranks, rank, n, flags, epoch, err_dev, STREAM(stream));
    return rc ? rc : check_launch("dense_mean_peers");
}

int gvc_dense_collect(const float *own_dev, float *out_dev, uint64_t n, const uint32_t *flags, int nranks,
                      uint32_t epoch, uint32_t *err_dev, void *stream)
{
    int rc = dense_collect_run(own_dev, out_dev, n, flags, nranks, epoch, err_dev, STREAM(stream));
    return rc ? rc : check_launch("dense_collect");
}

int gvc_gather_ef(const uint32_t *pos, uint64_t k, const float *values, const float *g, const float *resid,
                  const uint32_t *pmask, const float *pm, int pmode, float *out, void *stream)
{
    if ((k && !pos) || !out || (g ? !resid : !values) || (pmask && (!g || pmode < 1 || pmode > 2)))
        return set_error(GVC_ERR_ARG, "gvc_gather_ef: bad arguments");
    int rc = gather_ef_run(pos, k, values, g, resid, pmask, pm, pmode, out, STREAM(stream));
    return rc ? rc : check_launch("gather_ef");
}

int gvc_below_keys(const float *v, const uint32_t *pos, uint64_t n, const uint32_t *thr, const uint32_t *excl,
                   float *out, unsigned long long *count, void *stream)
{
    if (!v || !thr || !out || !count || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_below_keys: bad arguments");
    int rc = below_keys_run(v, pos, n, thr, excl, out, count, STREAM(stream));
    return rc ? rc : check_launch("below_keys");
}

size_t gvc_compact_workspace_bytes(uint64_t n) { return compact_workspace_bytes(n); }

int gvc_compact_mask(const uint32_t *mask, uint64_t n, uint32_t *out, unsigned long long *count, void *ws,
                     size_t ws_bytes, void *stream)
{
    if (!mask || !out || !count || n < 1)
        return set_error(GVC_ERR_ARG, "gvc_compact_mask: bad arguments");
    int rc = compact_mask_run(mask, n, out, count, ws, ws_bytes, STREAM(stream));
    return rc ? rc : check_launch("compact_mask");
}

int gvc_iota(uint32_t *out, uint64_t n, void *stream)
{
    int rc = iota_run(out, n, STREAM(stream));
    return rc ? rc : check_launch("iota");
}

}  // extern "C"
