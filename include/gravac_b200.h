/*
 * gravac_b200.h -- C-ABI of the B200-native GraVAC gradient-compression step.
 *
 * The reference (arxiv 2305.12201, /root/reference/pkg/src/gravac) has no
 * FFI: its boundary is the Python API re-exported by gravac/__init__.py:3-17.
 * This header is the native layer UNDER those Python names; the package
 * paper_2305_12201_b200 binds it with ctypes and keeps the reference's
 * function names, argument meaning and ValueError behaviour.  Each entry point
 * cites the reference function(s) it replaces.
 *
 * Conventions
 *   - every pointer named *_dev is a device pointer (cudaMalloc / torch CUDA
 *     storage); everything else is host memory;
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *     allocation-free (the caller passes a workspace sized by
 *     gvc_select_workspace_bytes) and deterministic: identical inputs give
 *     bit-identical outputs, including fp64 reductions (fixed-order trees);
 *   - every call returns an int status (GVC_OK or a negative gvc_status);
 *     gvc_last_error() returns the message of the last failure on this thread.
 *   - no call synchronises the stream.
 */
#ifndef GRAVAC_B200_H
#define GRAVAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GVC_API __attribute__((visibility("default")))
#else
#define GVC_API
#endif

#define GVC_ABI_VERSION 2
#define GVC_MAX_LADDER 16
#define GVC_AGG_TILE 4096 /* outputs per CTA of the decompress-average */

typedef enum {
    GVC_OK = 0,
    GVC_ERR_ARG = -1,       /* invalid argument (ValueError in the reference)          */
    GVC_ERR_NAN = -2,       /* NaN in the gradient: selection order undefined           */
    GVC_ERR_WORKSPACE = -3, /* workspace too small                                      */
    GVC_ERR_CUDA = -4,      /* CUDA launch / runtime failure                            */
    GVC_ERR_STATE = -5      /* call order violated (emit before select, ...)            */
} gvc_status;

/* Compressor kinds, compressors.py:21-25 */
typedef enum { GVC_TOPK = 0, GVC_DGC = 1, GVC_REDSYNC = 2, GVC_RANDOMK = 3 } gvc_kind;

/* Device-resident result of one gvc_select (read back by the host controller). */
typedef struct {
    double ef_norm_sq;                      /* ||values||^2 in fp64 (gradcore.py:61-70)        */
    double kept_sq[GVC_MAX_LADDER];         /* ||C_j(values)||^2 of the values to SEND, fp64   */
    double kept_abs[GVC_MAX_LADDER];        /* sum |v| over the kept support, fp64             */
    uint32_t threshold_key[GVC_MAX_LADDER]; /* k_j-th largest selection key                    */
    uint32_t pad0[GVC_MAX_LADDER];
    uint64_t tie_quota[GVC_MAX_LADDER];     /* how many keys == threshold are kept             */
    float redsync_mean[GVC_MAX_LADDER];     /* fl32(mean_f64 |v|) (compressors.py:188)         */
    uint64_t candidates;                    /* size of the candidate superset                  */
    int32_t status;                         /* GVC_OK or GVC_ERR_NAN                           */
    int32_t fallback_used;                  /* 1 when the threshold estimate missed (exact re-scan ran) */
    uint64_t kept_count[GVC_MAX_LADDER];    /* == ks[j] (sanity)                               */
    uint64_t kept_nonzero[GVC_MAX_LADDER];  /* kept entries with |v| > 0                       */
    uint64_t shortfall;                     /* allow_short: ks[0] - candidates (else 0)        */
} gvc_select_result;

/* Arguments of one selection over n values.  Two input modes:
 *   EF mode   (g_dev != NULL, resid_dev != NULL): values = fl32(g + resid) is
 *             computed on the fly (feedback.py:32-36) and written over
 *             resid_dev, which then holds g_ef;
 *   plain mode (values_dev != NULL): the values are read as given.            */
typedef struct {
    int32_t kind;                 /* gvc_kind                                               */
    int32_t n_ks;                 /* ladder length, 1..GVC_MAX_LADDER                       */
    uint64_t n;                   /* number of values (>= 1)                                */
    const float *values_dev;      /* plain mode input                                       */
    const float *g_dev;           /* EF mode raw gradient                                   */
    float *resid_dev;             /* EF mode residual in, g_ef out                          */
    uint64_t ks[GVC_MAX_LADDER];  /* keep counts, non-increasing, each in [1, n)            */
    uint64_t seed;                /* SeededRng.seed   (gradcore.py:139-142)                 */
    uint64_t rng_stream;          /* SeededRng.stream (after split).  Random-k keeps the k
                                     positions i with the smallest hash h(i) = word (i & 3)
                                     of Philox4x32-10 at counter (i >> 2, rng_stream), key
                                     seed (i = pos_base + position), ties to the lower index */
    uint64_t pos_base;            /* hash counter offset (layerwise segments)               */
    double dgc_sample_fraction;   /* CompressorKind.dgc_sample_fraction (compressors.py:36) */
    int32_t force_exact;          /* 1: skip the threshold estimate (every value is a candidate);
                                     2: test hook, an estimate that misses (exercises the exact re-scan) */
    int32_t pending_mode;         /* deferred residual update of the previous step, see below   */
    uint32_t *pending_mask_dev;   /* EF mode: bit i set = resid[i] still holds g_ef of a SENT   */
    const float *pending_m_dev;   /*   position; the true residual is fl32(r - f(r)) with
                                     f(r) = r (pending_mode 1: Top-k / Random-k / DGC) or
                                     f(r) = sign(r) * m (mode 2, Redsync, m = *pending_m_dev).
                                     The collect pass applies it while streaming r and clears
                                     the consumed mask words (feedback.py:39-51, deferred). */
    const uint32_t *key_est_dev;  /* optional: force the candidate threshold to this device key
                                     (DGC's sampled threshold, compressors.py:121-123): the
                                     candidates are then exactly {key >= *key_est_dev}        */
    int32_t allow_short;          /* with key_est_dev: if fewer than ks[0] candidates exist, keep
                                     them ALL (DGC overshoot, compressors.py:126-128) and report
                                     the shortfall in gvc_select_result.shortfall              */
    /* 1: every nonzero |value| is the same (a Redsync level-1 output, ±m or
     * 0: compressors.py:226-246 then orders by position alone) -- the order is
     * "nonzero first, then the lower index", one pass without the tie path.
     * Plain mode, one ladder entry, Top-k or Redsync, n + pos_base < 2^31. */
    int32_t equal_magnitudes;
    /* DGC in one selection, both branches of compressors.py:123-137 (no host
     * decision): with dgc_thr_dev (the sampled threshold key, device u32) and
     * dgc_sampled_dev (bit i set = position i is in the threshold sample,
     * u32[ceil(n/32)]) every value gets the composite key
     *     (|v| >= thr || sampled(i)) ? 0x80000000 | |v| : |v|
     * whose top-k IS the DGC pick: if k entries reach thr, the k largest of
     * them; otherwise all of them, then the largest sampled values below thr,
     * then the largest of the rest (global top-up), ties to the lower index. */
    const uint32_t *dgc_thr_dev;
    const uint32_t *dgc_sampled_dev;
} gvc_select_args;

GVC_API const char *gvc_last_error(void);
GVC_API int gvc_abi_version(void);

/* Workspace bytes for selections over up to n values of the given kind. */
GVC_API size_t gvc_select_workspace_bytes(int kind, uint64_t n);

/* Thresholds, tie quotas and kept energies for every ladder entry in one pass
 * over HBM.  Replaces: feedback.apply_feedback (feedback.py:32-36),
 * gradcore.squared_l2_norm (gradcore.py:61-70), compressors._select /
 * _exact_topk / _redsync_pick / _dgc_pick / RandomK choice
 * (compressors.py:86-190), compressors.compress_further for nested Top-k
 * (compressors.py:226-246, every ladder entry at once) and
 * metrics.compression_gain_raw numerators (metrics.py:18-32).
 * Writes *result_dev (device memory). */
GVC_API int gvc_select(const gvc_select_args *args, void *ws_dev, size_t ws_bytes,
               gvc_select_result *result_dev, void *stream);

/* Materialise ladder entry j of the last gvc_select on this workspace as an
 * index-ascending (u32 index, f32 value) list of exactly ks[j] entries.
 *   idx_map_dev: optional; output index = idx_map_dev[position] (second-level
 *                compression maps local positions back, compressors.py:242-244);
 *   resid_dev:   optional; resid[index] = fl32(value - sent_value) at every sent
 *                position, i.e. update_residual (feedback.py:39-51) given that
 *                resid_dev holds g_ef;
 *   sent_mask_dev: optional (instead of resid_dev); sets bit `index` for every sent
 *                position -- the deferred form the next gvc_select applies;
 *   sent_m_dev:  optional; receives the Redsync mean m of this entry (device float);
 *   tile_bounds_dev: optional (level-1 emits only), u32[ceil(n / GVC_AGG_TILE) + 1]: entry t =
 *                first output position whose index is >= t * GVC_AGG_TILE -- the tile
 *                boundaries gvc_aggregate needs, produced while the list is written;
 *   sent_stats_dev: optional double[2] = {sum sent^2, sum |sent|} (fp64, fixed order).
 * Replaces compressors._select's sort+gather (compressors.py:185-190). */
GVC_API int gvc_emit(void *ws_dev, size_t ws_bytes, int j, const uint32_t *idx_map_dev,
             uint32_t *out_idx_dev, float *out_val_dev, float *resid_dev,
             uint32_t *sent_mask_dev, float *sent_m_dev, uint32_t *tile_bounds_dev,
             double *sent_stats_dev, void *stream);

/* Mark k sent positions in a deferred-residual mask (bit idx[i] of mask). */
GVC_API int gvc_mark_sent(const uint32_t *idx_dev, uint64_t k, uint32_t *mask_dev, void *stream);

/* Materialise a deferred residual update in place: resid[i] = fl32(r - f(r))
 * wherever the mask bit is set (mode/m as in gvc_select_args), then clear the mask. */
GVC_API int gvc_apply_pending(float *resid_dev, uint32_t *mask_dev, uint64_t n, int mode,
                              const float *m_dev, void *stream);

/* out = fl32(g + r) (feedback.py:32-36, non-mutating form). */
GVC_API int gvc_ef_add(const float *g_dev, const float *r_dev, float *out_dev, uint64_t n, void *stream);

/* *out_dev = sum x^2 in fp64, fixed-order (gradcore.py:61-70).
 * Workspace: gvc_sq_norm_workspace_bytes(n). */
GVC_API size_t gvc_sq_norm_workspace_bytes(uint64_t n);
GVC_API int gvc_sq_norm(const float *x_dev, uint64_t n, double *out_dev, void *ws_dev, size_t ws_bytes,
                void *stream);

/* resid[idx[i]] = fl32(ef[idx[i]] - vals[i]) after resid = ef (feedback.py:39-51).
 * ef_dev may equal resid_dev (in-place). */
GVC_API int gvc_update_residual(const float *ef_dev, const uint32_t *idx_dev, const float *vals_dev,
                        uint64_t k, uint64_t n, float *resid_dev, void *stream);

/* Dense vector from one sparse part: zeros + scatter, -0.0 preserved
 * (compressors.py:249-253).  Workspace: gvc_aggregate_workspace_bytes(1, n). */
GVC_API int gvc_decompress(const uint32_t *idx_dev, const float *vals_dev, uint64_t k, uint64_t n,
                   float *out_dev, void *ws_dev, size_t ws_bytes, void *stream);

/* Mean of nparts index-ascending sparse parts, fp64 accumulation in part
 * order, /nparts, -> fp32 (compressors.py:256-271).  Part p is
 * (idx_dev + offs[p], vals_dev + offs[p]) with counts[p] entries; offs/counts are
 * HOST arrays.  Shared-memory tiles of the dense output, one coalesced
 * 128-bit store per 4 outputs.  bounds_dev (optional): part p's tile boundaries
 * (gvc_emit tile_bounds_dev) at bounds_dev + p * bounds_stride; otherwise they are
 * computed in a first pass.  This is the decompress-average half of the
 * sparse allgather. */
GVC_API int gvc_aggregate(const uint32_t *idx_dev, const float *vals_dev, const uint64_t *offs,
                  const uint64_t *counts, int nparts, uint64_t n, float *out_dev,
                  void *ws_dev, size_t ws_bytes, const uint32_t *bounds_dev, uint64_t bounds_stride,
                  void *stream);
GVC_API size_t gvc_aggregate_workspace_bytes(int nparts, uint64_t n);

/* ---- fused sparse allgather + decompress-average over peer memory (C1 + K7) ----
 * The reference simulates the workers in one process and calls
 * aggregate(parts) (compressors.py:256-271; simworkers.py:242-245).  On one
 * NVLink/NVSwitch node every rank's payload lives in a peer-mapped
 * (symmetric) buffer, and K7 reads the peers' (idx, vals, tile bounds)
 * directly -- the all-gather never materialises a gathered copy.
 *
 * gvc_peer_signal: once this rank's payload is complete (stream order), post
 *   `epoch` into peer_flags[q][rank] for every rank q (own included).
 *   peer_flags: HOST array of nranks device pointers (each rank's u32 flag
 *   array of >= nranks words, peer-mapped).
 * gvc_aggregate_peers: every CTA first waits until flags_dev[p] >= epoch
 *   (wrap-around compare) for p < nparts, then averages the parts exactly as
 *   gvc_aggregate (fp64, part order, /nparts).  idx/vals/bounds: HOST arrays
 *   of nparts device pointers (peer-mapped), bounds as gvc_emit's
 *   tile_bounds_dev; counts: HOST array.
 * Reuse rule (the caller's): with a payload double buffer and one epoch per
 *   exchange, slot e % 2 is rewritten only after every rank has posted epoch
 *   e + 1, i.e. after every rank's merge of epoch e has completed. */
#define GVC_MAX_PEERS 8

/* Push form of the exchange: the emit also writes its (idx, vals, tile
 * bounds) into up to GVC_MAX_PEERS - 1 further destinations -- the peers'
 * receive slots in their symmetric buffers -- with ordinary stores over
 * NVLink while it runs, then every thread issues a system-scope fence.  The
 * NVLink transfer overlaps the emit itself, and the merge reads only local
 * memory.  Fields: count (0..GVC_MAX_PEERS-1) and per destination the device
 * pointers (bounds_dev only used when the emit writes tile bounds). */
typedef struct gvc_emit_mirrors {
    int32_t count;
    int32_t reserved;
    uint32_t *idx_dev[GVC_MAX_PEERS];
    float *vals_dev[GVC_MAX_PEERS];
    uint32_t *bounds_dev[GVC_MAX_PEERS];
    /* the staged exchange's 16-bit wire index (idx mod GVC_AGG_TILE; the
     * tile bounds say which tile an entry lies in), written beside out_idx
     * into this rank's own slot; NULL = none.  count may be 0 for this alone. */
    uint16_t *off16_dev;
} gvc_emit_mirrors;
/* gvc_emit plus mirrors (NULL mirrors == gvc_emit). */
GVC_API int gvc_emit_mirrored(void *ws_dev, size_t ws_bytes, int j, const uint32_t *idx_map_dev,
             uint32_t *out_idx_dev, float *out_val_dev, float *resid_dev,
             uint32_t *sent_mask_dev, float *sent_m_dev, uint32_t *tile_bounds_dev,
             double *sent_stats_dev, const gvc_emit_mirrors *mirrors, void *stream);
GVC_API int gvc_peer_signal(uint32_t *const *peer_flags, int nranks, int rank, uint32_t epoch, void *stream);

/* ---- layerwise compression (compressors.py:204-217) as one segmented selection ----
 * Segment q = [seg_offsets[q], seg_offsets[q + 1]) keeps seg_k[q] entries
 * (keep_count of its length) by the compressor's key -- |v| for Top-k, the
 * Philox position hash h(i) of the global position for Random-k (as in
 * gvc_select_args.rng_stream) -- ties to the
 * lower index; out = the segments' (global index, value) lists concatenated
 * in segment order (sum seg_k entries; a segment with seg_k >= its length
 * keeps everything).  seg_offsets / seg_k are HOST arrays.  Every segment is
 * resolved by the same 10 launches (a state init, 3 radix passes of 11 / 11
 * / 10 key bits over all segments at once -- a histogram and a resolve each --,
 * per-slice counts, one scan, an ordered compaction) however many segments
 * there are.  *status_dev |= 1 on a NaN
 * magnitude.  The layout's work-item tables live in the workspace and are
 * uploaded only when (n, kind, seg_offsets, seg_k) differ from the previous
 * call on the same workspace address -- as with gvc_select's cached graphs,
 * a workspace is identified by its address: a new buffer must not reuse a
 * freed workspace's address while the library holds state for it (or call
 * gvc_workspace_forget first). */
GVC_API size_t gvc_segmented_select_workspace_bytes(uint64_t n, int nseg);
/* Layerwise Redsync: after gvc_segmented_select in Top-k mode (the support),
 * replace segment q's kept values vals_dev[out_off[q] .. out_off[q+1]) by
 * sign(v) * fl32(mean_f64 |v|) of that segment (compressors.py:140-161,
 * :187-189); a segment whose count reaches its length (seg_len[q]) is an
 * identity pass-through (:172-173).  out_off: u64[nseg + 1] and seg_len:
 * u64[nseg] are HOST arrays; the work is cut into 16384-entry items, two
 * launches however unequal the segments. */
GVC_API size_t gvc_segmented_redsync_workspace_bytes(uint64_t total_kept, int nseg);
GVC_API int gvc_segmented_redsync_values(float *vals_dev, const uint64_t *out_off, const uint64_t *seg_len, int nseg,
                                         void *ws_dev, size_t ws_bytes, void *stream);
/* Layerwise (compressors.py:211-213): idx_dev[j] += starts_dev[q] for the
 * segment q whose outputs out_off_dev[q] <= j < out_off_dev[q + 1] hold j --
 * segment-local positions to global indices in one launch.  Device arrays;
 * 1 <= nseg <= 3000. */
GVC_API int gvc_add_segment_offsets(uint32_t *idx_dev, uint64_t total, const uint64_t *out_off_dev,
                                    const uint64_t *starts_dev, int nseg, void *stream);
/* Drop every per-workspace cache entry (select graphs and plans, segment
 * tables) for `ws` before its memory is freed or reused. */
GVC_API int gvc_workspace_forget(void *ws);

/* The controller's one read-back per step, started without host stream
 * bookkeeping: once `stream` reaches this point, copy `bytes` from dev_src to
 * (pinned) host_dst on side_stream.  events[2] (ready, done) are created on
 * first use and reused; gvc_event_done(events[1]) polls completion (1 done,
 * 0 not yet, < 0 error). */
GVC_API int gvc_read_async(void *host_dst, const void *dev_src, size_t bytes, void *stream, void *side_stream,
                           void **events);
GVC_API int gvc_event_done(void *event);
/* Stream ordering without host-side stream objects: record *event (created on
 * first use) on `stream`; make `stream` wait for `event`. */
GVC_API int gvc_event_record(void **event, void *stream);
GVC_API int gvc_stream_wait_event(void *stream, void *event);
/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream): a caller's
 * host->device gradient upload without host-side stream objects. */
GVC_API int gvc_copy_async(void *dst, const void *src, size_t bytes, void *stream);
/* Layerwise DGC (compressors.py:204-217 with the DGC rule of :110-137 in every
 * segment; replaces the per-segment gvc_dgc_sample_gather + threshold select
 * + composite-key gvc_select sequence): segment q draws
 * s_q = min(len, max(256, round(sample_fraction * len))) stratified positions
 * (the gvc_dgc_sample definition with pos_base = the segment start), its
 * threshold is the rank_q-th largest sampled |v| (rank_q = min(s_q, max(1,
 * round(seg_k[q] s_q / len)))), and it keeps the top seg_k[q] of the DGC
 * composite key -- the same picks as the per-segment sequence, for every
 * segment at once (one sample launch + 9 + 12 segmented-selection launches).
 * A segment with s_q = len takes the exact top-k.  Host seg_offsets /
 * seg_k as in gvc_segmented_select; *status_dev |= 1 on a NaN. */
GVC_API size_t gvc_segmented_dgc_workspace_bytes(uint64_t n, int nseg, double sample_fraction);
GVC_API int gvc_segmented_dgc_select(const float *values_dev, uint64_t n, const uint64_t *seg_offsets,
                                     const uint64_t *seg_k, int nseg, double sample_fraction, uint64_t seed,
                                     uint64_t rng_stream, uint32_t *out_idx_dev, float *out_val_dev, void *ws_dev,
                                     size_t ws_bytes, uint32_t *status_dev, void *stream);
GVC_API int gvc_segmented_select(int kind, const float *values_dev, uint64_t n, const uint64_t *seg_offsets,
                                 const uint64_t *seg_k, int nseg, uint64_t seed, uint64_t rng_stream,
                                 uint32_t *out_idx_dev, float *out_val_dev, void *ws_dev, size_t ws_bytes,
                                 uint32_t *status_dev, void *stream);

/* ---- dense fallback over peer memory (C3) ----
 * The dense message of a step whose decision is DENSE (controller.py:217-230,
 * 259-264) and its mean, aggregate_dense (compressors.py:274-285), as one
 * fused reduce-scatter + all-gather over NVLink.  peer_bufs[q]: rank q's
 * peer-mapped buffer holding its dense input (n floats, 16-byte aligned,
 * room for n rounded up to 4).  After every rank posted `epoch` into flags
 * (gvc_peer_signal), gvc_dense_mean_peers makes rank `rank` sum its range
 * [n4*rank/W, n4*(rank+1)/W) of float4s (n4 = ceil(n/4)) over the W inputs in
 * fp64 in rank order, divide by W, round to fp32, and write the result range
 * into every rank's buffer.  Once every rank has posted a second epoch
 * (signal after gvc_dense_mean_peers), gvc_dense_collect copies the full mean
 * from this rank's buffer to out_dev.  Waits are bounded (~4 s): a timeout
 * sets bit 4 of *err_dev instead of hanging. */
GVC_API int gvc_dense_mean_peers(float *const *peer_bufs, int nranks, int rank, uint64_t n, const uint32_t *flags,
                                 uint32_t epoch, uint32_t *err_dev, void *stream);
GVC_API int gvc_dense_collect(const float *own_dev, float *out_dev, uint64_t n, const uint32_t *flags, int nranks,
                              uint32_t epoch, uint32_t *err_dev, void *stream);
GVC_API int gvc_aggregate_peers(const uint32_t *const *idx_dev, const float *const *vals_dev,
                        const uint32_t *const *bounds_dev, const uint64_t *counts, int nparts, uint64_t n,
                        const uint32_t *flags_dev, uint32_t epoch, float *out_dev, void *stream);
/* Staged pull: the same merge, but the first copy_blocks CTAs of its grid
 * stream the peers' tile bounds, then their (idx, vals) chunk by chunk
 * (chunk_entries, a power of two), over NVLink into LOCAL staging slots --
 * idx_dev / vals_dev / bounds_dev[p] for p != self.  ready_dev (local, zeroed
 * once, copy_blocks + ceil(k / chunk_entries) words of monotonic epochs):
 * word b < copy_blocks tags bound slice b, word copy_blocks + c chunk c.  Each
 * tile waits only for its own chunks, so the transfer and the merge overlap.
 * src_*_dev[p]: peer p's payload (peer-mapped). */
typedef struct gvc_peer_staging {
    int32_t self;
    int32_t copy_blocks;
    uint32_t chunk_entries;
    uint32_t reserved;
    uint32_t *ready_dev;
    const uint32_t *src_idx_dev[GVC_MAX_PEERS];
    const float *src_vals_dev[GVC_MAX_PEERS];
    const uint32_t *src_bounds_dev[GVC_MAX_PEERS];
    /* 16-bit wire indices (gvc_emit_mirrors.off16_dev): when every part has
     * them, the copiers move (u16 offset, f32 value) -- 6 bytes per entry over
     * NVLink instead of 8 -- and the tiles read offsets, not idx: src_off16_dev[p]
     * peer p's (remote), off16_dev[p] the local slot (p == self: this rank's own). */
    const uint16_t *src_off16_dev[GVC_MAX_PEERS];
    uint16_t *off16_dev[GVC_MAX_PEERS];
} gvc_peer_staging;
GVC_API int gvc_aggregate_peers_staged(const uint32_t *const *idx_dev, const float *const *vals_dev,
                        const uint32_t *const *bounds_dev, const uint64_t *counts, int nparts, uint64_t n,
                        const uint32_t *flags_dev, uint32_t epoch, const gvc_peer_staging *staging,
                        float *out_dev, void *stream);
/* Tile boundaries (gvc_emit's tile_bounds_dev layout) of one index-ascending
 * list of k entries over [0, n): u32[ceil(n / GVC_AGG_TILE) + 1]. */
GVC_API int gvc_tile_bounds(const uint32_t *idx_dev, uint64_t k, uint64_t n, uint32_t *bounds_dev, void *stream);

/* fp64 mean of nparts dense vectors laid out [nparts][n] (compressors.py:274-285). */
GVC_API int gvc_aggregate_dense(const float *parts_dev, int nparts, uint64_t n, float *out_dev,
                        void *stream);

/* Measurement hooks (bench.py).  on = 1: the selection runs as direct
 * launches and CUDA events bracket the collect kernel, the whole selection,
 * the emit and the decompress-average on the launching stream.  on = 2: the
 * selection keeps running as its CUDA graph, with event-record nodes around
 * the collect kernel only (its duration inside the timed loop itself).
 * gvc_prof_read synchronises on the events, returns per-category
 * milliseconds and launch counts (categories: 0 collect, 1 select, 2 emit,
 * 3 aggregate) and resets.  gvc_launch_count is a running count of every
 * kernel this library launched. */
GVC_API void gvc_prof_enable(int on);
/* Probe only the selects / emits of vectors of at least n values (default 0:
 * all) -- a step with several selects (DGC's sample, the level-2 select) then
 * reports the full-size one alone. */
GVC_API void gvc_prof_min_n(uint64_t n);
GVC_API int gvc_prof_read(double *ms, unsigned long long *counts, int ncat);
GVC_API unsigned long long gvc_launch_count(void);

/* Diagnostic: the %globaltimer stamps (ns) the last gvc_select on `ws`
 * recorded at its phase boundaries (collect start, sample barriers, pass end,
 * level-0 resolve, ...); synchronous.  Development aid for the roofline work. */
GVC_API int gvc_select_phase_times(void *ws, unsigned long long *out, int n);

/* DGC's threshold sample (compressors.py:118; parity-unpinned):
 * s ascending positions of [0, n), one per stratum [j n / s, (j + 1) n / s),
 * at lo_j + floor(h_j * width_j / 2^32), h_j = Philox4x32-10 word 0 at
 * counter (pos_base + lo_j, stream), key seed. */
GVC_API int gvc_dgc_sample(uint64_t n, uint64_t s, uint64_t seed, uint64_t rng_stream, uint64_t pos_base,
                           uint32_t *out_pos_dev, void *stream);
/* The same sample, fused with its use (compressors.py:118-121): out[j] = the
 * value at the j-th sampled position (as gvc_gather_ef: fl32(g + r_true) in EF
 * mode, else values_dev), and bits_dev (u32[ceil(n/32)], overwritten) = the
 * bitmap of the sampled positions, as gvc_select_args.dgc_sampled_dev wants it. */
GVC_API int gvc_dgc_sample_gather(uint64_t n, uint64_t s, uint64_t seed, uint64_t rng_stream, uint64_t pos_base,
                                  const float *values_dev, const float *g_dev, const float *resid_dev,
                                  const uint32_t *pending_mask_dev, const float *pending_m_dev, int pending_mode,
                                  float *out, uint32_t *bits_dev, void *stream);
/* DGC helpers (compressors.py:110-137).
 * gvc_gather_ef: out[i] = values at pos[i]: fl32(g + r_true) in EF mode (g_dev and
 *   resid_dev, with the deferred mask of gvc_select_args applied), else values_dev[pos[i]].
 * gvc_below_keys: out[i] = a non-negative float whose magnitude key is key(v[i]) + 1
 *   when key(v[i]) < *thr_dev and (excl_mask_dev == NULL or bit pos[i] clear), else +0.0;
 *   a Top-k over `out` ranks exactly "the largest below the threshold, ties to the
 *   lower index" (:129-131, :102-107); *count_dev += number of eligible entries.
 * gvc_compact_mask: the set bits of mask[0..ceil(n/32)) as ascending positions;
 *   *count_dev = their number.  Workspace: gvc_compact_workspace_bytes(n). */
GVC_API int gvc_gather_ef(const uint32_t *pos_dev, uint64_t k, const float *values_dev, const float *g_dev,
                          const float *resid_dev, const uint32_t *pending_mask_dev, const float *pending_m_dev,
                          int pending_mode, float *out_dev, void *stream);
GVC_API int gvc_below_keys(const float *v_dev, const uint32_t *pos_dev, uint64_t n, const uint32_t *thr_dev,
                           const uint32_t *excl_mask_dev, float *out_dev, unsigned long long *count_dev,
                           void *stream);
GVC_API size_t gvc_compact_workspace_bytes(uint64_t n);
GVC_API int gvc_compact_mask(const uint32_t *mask_dev, uint64_t n, uint32_t *out_dev,
                             unsigned long long *count_dev, void *ws_dev, size_t ws_bytes, void *stream);

/* Fill out[i] = i (identity support for k >= n, compressors.py:172-173). */
GVC_API int gvc_iota(uint32_t *out_dev, uint64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif
