// gvc_internal.h -- declarations shared by the translation units of libgravac_b200.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/gravac_b200.h"

namespace gvc {

// Records the message for gvc_last_error() and returns `code`.
int set_error(int code, const char *fmt, ...);

// Live kernel timing for bench.py (CUDA events on the launching stream).
enum ProfCat { PROF_COLLECT = 0, PROF_SELECT = 1, PROF_EMIT = 2, PROF_AGGREGATE = 3, PROF_NCAT = 4 };
struct ProfScope {
    int slot;
    cudaStream_t s;
    ProfScope(int cat, cudaStream_t s);
    ~ProfScope();
};
void count_launches(int n);
bool prof_enabled();
bool prof_graph_enabled();
bool prof_wants(uint64_t n);  // the select / emit of an n-value vector is probed (gvc_prof_min_n)
void prof_graph_pair(int cat, cudaEvent_t *a, cudaEvent_t *b);

size_t select_workspace_bytes(int kind, uint64_t n);
int select_run(const gvc_select_args *a, void *ws, size_t ws_bytes, gvc_select_result *res,
               cudaStream_t s);
int select_phase_times(void *ws, unsigned long long *out, int n);
int emit_run(void *ws, size_t ws_bytes, int j, const uint32_t *idx_map, uint32_t *out_idx, float *out_val,
             float *resid, uint32_t *smask, float *sm_out, uint32_t *tile_b, double *stats,
             const gvc_emit_mirrors *mirrors, cudaStream_t s);
int mark_sent_run(const uint32_t *idx, uint64_t k, uint32_t *mask, cudaStream_t s);
int apply_pending_run(float *resid, uint32_t *mask, uint64_t n, int mode, const float *m, cudaStream_t s);

size_t sq_norm_workspace_bytes(uint64_t n);
int sq_norm_run(const float *x, uint64_t n, double *out, void *ws, size_t ws_bytes, cudaStream_t s);
int ef_add_run(const float *g, const float *r, float *out, uint64_t n, cudaStream_t s);
int update_residual_run(const float *ef, const uint32_t *idx, const float *vals, uint64_t k,
                        uint64_t n, float *resid, cudaStream_t s);
int decompress_run(const uint32_t *idx, const float *vals, uint64_t k, uint64_t n, float *out, void *ws,
                   size_t ws_bytes, cudaStream_t s);
size_t aggregate_workspace_bytes(int nparts, uint64_t n);
int peer_signal_run(uint32_t *const *peer_flags, int nranks, int rank, uint32_t epoch, cudaStream_t s);
int aggregate_peers_run(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                        const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                        float *out, cudaStream_t s);
int aggregate_peers_staged_run(const uint32_t *const *idx, const float *const *vals, const uint32_t *const *bounds,
                               const uint64_t *counts, int nparts, uint64_t n, const uint32_t *flags, uint32_t epoch,
                               const gvc_peer_staging *sg, float *out, cudaStream_t s);
int device_sms();
int add_seg_offsets_run(uint32_t *idx, uint64_t total, const uint64_t *out_off, const uint64_t *starts, int nseg,
                        cudaStream_t s);  // SM count of the current device (cached)
int dgc_sample_run(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base, uint32_t *out,
                   cudaStream_t st);
int dgc_sample_gather_run(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                          const float *values, const float *g, const float *resid, const uint32_t *pmask,
                          const float *pm, int pmode, float *out, uint32_t *bits, cudaStream_t st);
int tile_bounds_run(const uint32_t *idx, uint64_t k, uint64_t n, uint32_t *bounds, cudaStream_t s);
int aggregate_run(const uint32_t *idx, const float *vals, const uint64_t *offs, const uint64_t *counts,
                  int nparts, uint64_t n, float *out, void *ws, size_t ws_bytes, const uint32_t *bounds,
                  uint64_t bounds_stride, cudaStream_t s);
int aggregate_dense_run(const float *parts, int nparts, uint64_t n, float *out, cudaStream_t s);
int dense_mean_peers_run(float *const *bufs, int nranks, int rank, uint64_t n, const uint32_t *flags,
                         uint32_t epoch, uint32_t *err, cudaStream_t s);
int dense_collect_run(const float *own, float *out, uint64_t n, const uint32_t *flags, int nranks, uint32_t epoch,
                      uint32_t *err, cudaStream_t s);
int iota_run(uint32_t *out, uint64_t n, cudaStream_t s);
size_t segsel_workspace_bytes(uint64_t n, int nseg);
void select_forget(const void *ws);
void segsel_forget(const void *ws);
size_t seg_redsync_workspace_bytes(uint64_t total, int nseg);
int seg_redsync_run(float *vals, const uint64_t *out_off, const uint64_t *seg_len, int nseg, void *ws,
                    size_t ws_bytes, cudaStream_t s);
size_t seg_dgc_workspace_bytes(uint64_t n, int nseg, double frac);
int seg_dgc_run(const float *values, uint64_t n, const uint64_t *seg_off, const uint64_t *seg_k, int nseg, double frac,
                uint64_t seed, uint64_t stream, uint32_t *out_idx, float *out_val, void *ws, size_t ws_bytes,
                uint32_t *status, cudaStream_t s);
int segsel_run(int kind, const float *values, uint64_t n, const uint64_t *seg_off, const uint64_t *seg_k, int nseg,
               uint64_t seed, uint64_t stream, uint32_t *out_idx, float *out_val, void *ws, size_t ws_bytes,
               uint32_t *status, cudaStream_t s);
int gather_ef_run(const uint32_t *pos, uint64_t k, const float *values, const float *g, const float *resid,
                  const uint32_t *pmask, const float *pm, int pmode, float *out, cudaStream_t s);
int below_keys_run(const float *v, const uint32_t *pos, uint64_t n, const uint32_t *thr, const uint32_t *excl,
                   float *out, unsigned long long *count, cudaStream_t s);
size_t compact_workspace_bytes(uint64_t n);
int compact_mask_run(const uint32_t *mask, uint64_t n, uint32_t *out, unsigned long long *count, void *ws,
                     size_t ws_bytes, cudaStream_t s);

}  // namespace gvc
