/*
 * gravac_oracle.c -- CPU restatement of the GraVAC hot path (TEST INFRASTRUCTURE).
 * See gravac_oracle.h for scope, pinning and the "parity unpinned" note.
 *
 * Plain C99, deliberately simple: two-level radix counting
 * for the exact k-th key, then one ordered scan that keeps everything above
 * the threshold and the lowest-index ties.  That is the selection rule of
 * compressors.py:86-99 (np.partition kth, flatnonzero(mag > kth), first
 * `need` of flatnonzero(mag == kth)) without the partition.
 *
 * Threads: one by default -- the checker.  orc_set_threads(T > 1) (bench.py's
 * CPU legs only) splits the O(n) passes over T OpenMP threads in index-ordered
 * chunks: EF add, keys, counting, the ordered compaction (per-chunk counts,
 * prefix, parallel write), residual update and aggregation give the same
 * outputs; only the fp64 norm is then summed per chunk (a different rounding).
 */
#include "gravac_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 1;

void orc_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int orc_get_threads(void) { return g_threads; }

/* [lo, hi) of chunk c of C over n */
static inline uint64_t chunk_lo(uint64_t n, int c, int C) { return n * (uint64_t)c / (uint64_t)C; }

/* |x| as an order-preserving integer key: clear the sign bit (-0 -> 0).
 * Monotone for every non-NaN float (compressors.py:174 np.abs + compare). */
static inline uint32_t mag_key(float v)
{
    uint32_t b;
    memcpy(&b, &v, 4);
    return b & 0x7fffffffu;
}

static inline int key_is_nan(uint32_t k) { return k > 0x7f800000u; }

/* ------------------------------------------------------------------ Philox */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint32_t orc_randomk_hash(uint64_t seed, uint64_t stream, uint64_t i)
{
    uint64_t q = i >> 2;
    uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[i & 3];
}

uint32_t orc_position_hash(uint64_t seed, uint64_t stream, uint64_t i)
{
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[0];
}

/* ------------------------------------------------------------ dense pieces */
void orc_ef_add(const float *g, const float *r, float *out, uint64_t n)
{
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
    for (uint64_t i = 0; i < n; i++) {
        volatile float s = g[i] + r[i]; /* one IEEE fp32 rounding, no contraction */
        out[i] = s;
    }
}

double orc_sq_norm(const float *x, uint64_t n)
{
    if (g_threads > 1 && n >= (1u << 20)) {
        const int C = g_threads;
        double part[256];
#pragma omp parallel for num_threads(C) schedule(static, 1)
        for (int c = 0; c < C; c++) {
            double acc = 0.0;
            for (uint64_t i = chunk_lo(n, c, C); i < chunk_lo(n, c + 1, C); i++) {
                double v = (double)x[i];
                acc += v * v;
            }
            part[c] = acc;
        }
        double acc = 0.0;
        for (int c = 0; c < C; c++)
            acc += part[c];
        return acc;
    }
    double acc = 0.0;
    for (uint64_t i = 0; i < n; i++) {
        double v = (double)x[i];
        acc += v * v;
    }
    return acc;
}

/* numpy/_core/src/umath/loops_utils.h.src pairwise_sum for doubles:
 * blocks of <= 128 use 8 interleaved accumulators, larger ranges split in
 * halves rounded down to a multiple of 8. */
static double pairwise_rec(const double *a, uint64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (uint64_t i = 0; i < n; i++)
            res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++)
            r[j] = a[j];
        uint64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++)
                r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++)
            res += a[i];
        return res;
    }
    uint64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_rec(a, n2) + pairwise_rec(a + n2, n - n2);
}

double orc_pairwise_sum_f64(const double *a, uint64_t n)
{
    /* add.reduce over a contiguous float64 array: the identity 0.0 is the
     * initial value and the whole array goes through one pairwise call */
    return 0.0 + pairwise_rec(a, n);
}

/* ------------------------------------------------------- exact key select */
/* Find the k-th largest key T and the tie quota q = k - #(key > T).
 * Two counting passes: top 16 bits, then low 16 bits inside the bin. */
/* cnt[b] += #{i : keys[i] >> 16 == b} (hi) or #{i : keys[i] >> 16 == bin, keys[i] & 0xffff == b} */
static void count_keys(const uint32_t *keys, uint64_t n, int hi, uint32_t bin, uint64_t *cnt)
{
    const int C = (g_threads > 1 && n >= (1u << 20)) ? g_threads : 1;
    if (C == 1) {
        for (uint64_t i = 0; i < n; i++) {
            if (hi)
                cnt[keys[i] >> 16]++;
            else if ((keys[i] >> 16) == bin)
                cnt[keys[i] & 0xffffu]++;
        }
        return;
    }
    uint32_t *loc = (uint32_t *)calloc((size_t)C * 65536, sizeof(uint32_t));
#pragma omp parallel for num_threads(C) schedule(static, 1)
    for (int c = 0; c < C; c++) {
        uint32_t *h = loc + (size_t)c * 65536;
        for (uint64_t i = chunk_lo(n, c, C); i < chunk_lo(n, c + 1, C); i++) {
            if (hi)
                h[keys[i] >> 16]++;
            else if ((keys[i] >> 16) == bin)
                h[keys[i] & 0xffffu]++;
        }
    }
#pragma omp parallel for num_threads(C) schedule(static)
    for (int b = 0; b < 65536; b++)
        for (int c = 0; c < C; c++)
            cnt[b] += loc[(size_t)c * 65536 + b];
    free(loc);
}

static void kth_key(const uint32_t *keys, uint64_t n, uint64_t k, uint32_t *T, uint64_t *q)
{
    uint64_t *cnt = (uint64_t *)calloc(65536, sizeof(uint64_t));
    count_keys(keys, n, 1, 0, cnt);
    uint64_t above = 0;
    int b = 65535;
    for (; b >= 0; b--) {
        if (above + cnt[b] >= k)
            break;
        above += cnt[b];
    }
    uint64_t need = k - above;
    memset(cnt, 0, 65536 * sizeof(uint64_t));
    count_keys(keys, n, 0, (uint32_t)b, cnt);
    uint64_t above2 = 0;
    int t = 65535;
    for (; t >= 0; t--) {
        if (above2 + cnt[t] >= need)
            break;
        above2 += cnt[t];
    }
    *T = ((uint32_t)b << 16) | (uint32_t)t;
    *q = need - above2;
    free(cnt);
}

int orc_select_keys(const uint32_t *keys, uint64_t n, uint64_t k, uint32_t *out_idx)
{
    if (n == 0 || k == 0)
        return ORC_ERR_ARG;
    if (k >= n) {
        for (uint64_t i = 0; i < n; i++)
            out_idx[i] = (uint32_t)i;
        return ORC_OK;
    }
    uint32_t T;
    uint64_t q;
    kth_key(keys, n, k, &T, &q);
    const int C = (g_threads > 1 && n >= (1u << 20)) ? g_threads : 1;
    if (C > 1 && C <= 256) {
        /* per-chunk (above, tie) counts, prefix, then every chunk writes its
         * slice: the same ascending list as the scan below */
        uint64_t ab[257], ti[257];
#pragma omp parallel for num_threads(C) schedule(static, 1)
        for (int c = 0; c < C; c++) {
            uint64_t a = 0, t = 0;
            for (uint64_t i = chunk_lo(n, c, C); i < chunk_lo(n, c + 1, C); i++) {
                a += keys[i] > T;
                t += keys[i] == T;
            }
            ab[c] = a;
            ti[c] = t;
        }
        uint64_t o0[257], t0[257], oa = 0, ta = 0;
        for (int c = 0; c < C; c++) {
            o0[c] = oa;
            t0[c] = ta;
            const uint64_t take = ta >= q ? 0 : (q - ta < ti[c] ? q - ta : ti[c]);
            oa += ab[c] + take;
            ta += ti[c];
        }
        if (oa != k)
            return ORC_ERR_ARG;
#pragma omp parallel for num_threads(C) schedule(static, 1)
        for (int c = 0; c < C; c++) {
            uint64_t o = o0[c], ties = t0[c];
            for (uint64_t i = chunk_lo(n, c, C); i < chunk_lo(n, c + 1, C); i++) {
                uint32_t key = keys[i];
                if (key > T || (key == T && ties++ < q))
                    out_idx[o++] = (uint32_t)i;
            }
        }
        return ORC_OK;
    }
    uint64_t o = 0, ties = 0;
    for (uint64_t i = 0; i < n; i++) {
        uint32_t key = keys[i];
        if (key > T || (key == T && ties++ < q))
            out_idx[o++] = (uint32_t)i;
    }
    return o == k ? ORC_OK : ORC_ERR_ARG;
}

static uint32_t *mag_keys(const float *x, uint64_t n, int *nan_seen)
{
    uint32_t *keys = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
    if (!keys)
        return NULL;
    int nan = 0;
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static) reduction(|: nan)
    for (uint64_t i = 0; i < n; i++) {
        keys[i] = mag_key(x[i]);
        if (key_is_nan(keys[i]))
            nan = 1;
    }
    *nan_seen = nan;
    return keys;
}

int orc_topk_indices(const float *x, uint64_t n, uint64_t k, uint32_t *out_idx)
{
    int nan_seen;
    uint32_t *keys = mag_keys(x, n, &nan_seen);
    if (!keys)
        return ORC_ERR_NOMEM;
    int rc = nan_seen ? ORC_ERR_NAN : orc_select_keys(keys, n, k, out_idx);
    free(keys);
    return rc;
}

static int cmp_u32(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/* (key desc, position asc) -- np.argsort(-mag, kind="stable") over ascending positions */
typedef struct { uint32_t key; uint32_t pos; } keypos;
static int cmp_keypos(const void *a, const void *b)
{
    const keypos *x = (const keypos *)a, *y = (const keypos *)b;
    if (x->key != y->key)
        return x->key > y->key ? -1 : 1;
    return (x->pos > y->pos) - (x->pos < y->pos);
}

static int cmp_desc_u32(const void *a, const void *b) { return -cmp_u32(a, b); }

/* DGC's threshold sample (compressors.py:118 draws s positions without
 * replacement with numpy's Generator.choice; parity-unpinned):
 * [0, n) is cut into s strata [floor(j n / s), floor((j + 1) n / s)) and
 * stratum j contributes the position lo_j + floor(h_j * width_j / 2^32),
 * h_j = Philox4x32-10 word 0 at counter (pos_base + lo_j, stream), key seed.
 * Exactly s distinct, ascending positions; a stratified sample of the same
 * size as the reference's simple random sample. */
void orc_dgc_sample_positions(uint64_t n, uint64_t s, uint64_t seed, uint64_t stream, uint64_t pos_base,
                              uint32_t *out)
{
    for (uint64_t j = 0; j < s; j++) {
        const uint64_t lo = j * n / s, hi = (j + 1) * n / s;
        const uint32_t h = orc_position_hash(seed, stream, pos_base + lo);
        out[j] = (uint32_t)(lo + (((uint64_t)h * (hi - lo)) >> 32));
    }
}

/* compressors.py:110-137 with the counter-based sample (see header). */
static int dgc_pick(const float *v, const uint32_t *mk, uint64_t n, uint64_t k, uint64_t seed,
                    uint64_t stream, uint64_t pos_base, double frac, uint32_t *out_idx)
{
    double want = nearbyint(frac * (double)n); /* Python round(): half to even */
    uint64_t s = (uint64_t)(want < 256.0 ? 256.0 : want);
    if (s > n)
        s = n;
    if (s >= n)
        return orc_select_keys(mk, n, k, out_idx);
    /* sample = one position per stratum (orc_dgc_sample_positions) */
    uint32_t *hk = (uint32_t *)malloc(1 * sizeof(uint32_t));
    uint32_t *samp = (uint32_t *)malloc(s * sizeof(uint32_t));
    uint32_t *sk = (uint32_t *)malloc(s * sizeof(uint32_t));
    uint8_t *picked = (uint8_t *)calloc(n, 1);
    if (!hk || !samp || !sk || !picked)
        return ORC_ERR_NOMEM;
    orc_dgc_sample_positions(n, s, seed, stream, pos_base, samp);
    for (uint64_t j = 0; j < s; j++)
        sk[j] = mk[samp[j]];
    qsort(sk, s, sizeof(uint32_t), cmp_desc_u32); /* np.sort(...)[::-1] */
    double rr = nearbyint((double)(k * s) / (double)n);
    uint64_t rank = rr < 1.0 ? 1 : (uint64_t)rr;
    if (rank > s)
        rank = s;
    uint32_t thr = sk[rank - 1];

    uint64_t chosen = 0;
    for (uint64_t i = 0; i < n; i++)
        if (mk[i] >= thr) {
            picked[i] = 1;
            chosen++;
        }
    int rc = ORC_OK;
    if (chosen >= k) {
        /* chosen[_exact_topk(mag[chosen], k)] */
        uint32_t *cpos = (uint32_t *)malloc(chosen * sizeof(uint32_t));
        uint32_t *ckey = (uint32_t *)malloc(chosen * sizeof(uint32_t));
        uint32_t *sel = (uint32_t *)malloc(k * sizeof(uint32_t));
        uint64_t c = 0;
        for (uint64_t i = 0; i < n; i++)
            if (picked[i]) {
                cpos[c] = (uint32_t)i;
                ckey[c] = mk[i];
                c++;
            }
        rc = orc_select_keys(ckey, chosen, k, sel);
        for (uint64_t j = 0; j < k; j++)
            out_idx[j] = cpos[sel[j]];
        free(cpos); free(ckey); free(sel);
    } else {
        uint64_t shortfall = k - chosen;
        /* pad from the sampled pool below the threshold, largest first */
        keypos *below = (keypos *)malloc(s * sizeof(keypos));
        uint64_t nb = 0;
        for (uint64_t j = 0; j < s; j++)
            if (mk[samp[j]] < thr) {
                below[nb].key = mk[samp[j]];
                below[nb].pos = samp[j];
                nb++;
            }
        qsort(below, nb, sizeof(keypos), cmp_keypos);
        uint64_t take = nb < shortfall ? nb : shortfall;
        for (uint64_t j = 0; j < take; j++)
            picked[below[j].pos] = 1;
        shortfall -= take;
        free(below);
        if (shortfall > 0) {
            /* _global_topup: largest outside the chosen set, ties -> lower index */
            uint64_t nrest = 0;
            for (uint64_t i = 0; i < n; i++)
                nrest += !picked[i];
            uint32_t *rpos = (uint32_t *)malloc(nrest * sizeof(uint32_t));
            uint32_t *rkey = (uint32_t *)malloc(nrest * sizeof(uint32_t));
            uint32_t *sel = (uint32_t *)malloc(shortfall * sizeof(uint32_t));
            uint64_t c = 0;
            for (uint64_t i = 0; i < n; i++)
                if (!picked[i]) {
                    rpos[c] = (uint32_t)i;
                    rkey[c] = mk[i];
                    c++;
                }
            rc = orc_select_keys(rkey, nrest, shortfall, sel);
            for (uint64_t j = 0; j < shortfall; j++)
                picked[rpos[sel[j]]] = 1;
            free(rpos); free(rkey); free(sel);
        }
        uint64_t o = 0;
        for (uint64_t i = 0; i < n; i++)
            if (picked[i])
                out_idx[o++] = (uint32_t)i;
        if (o != k)
            rc = ORC_ERR_ARG;
    }
    free(hk); free(samp); free(sk); free(picked);
    return rc;
}

int orc_select(int kind, const float *values, uint64_t n, uint64_t k,
               uint64_t seed, uint64_t stream, uint64_t pos_base,
               double dgc_sample_fraction, uint32_t *out_idx, float *out_vals)
{
    if (n == 0 || k == 0)
        return ORC_ERR_ARG;
    if (k >= n) { /* compressors.py:172-173 identity passthrough for every kind */
        for (uint64_t i = 0; i < n; i++) {
            out_idx[i] = (uint32_t)i;
            out_vals[i] = values[i];
        }
        return ORC_OK;
    }
    int rc = ORC_OK;
    if (kind == ORC_RANDOMK) {
        uint32_t *hk = (uint32_t *)malloc(n * sizeof(uint32_t));
        if (!hk)
            return ORC_ERR_NOMEM;
        for (uint64_t i = 0; i < n; i++)
            hk[i] = ~orc_randomk_hash(seed, stream, pos_base + i);
        rc = orc_select_keys(hk, n, k, out_idx);
        free(hk);
    } else {
        int nan_seen;
        uint32_t *mk = mag_keys(values, n, &nan_seen);
        if (!mk)
            return ORC_ERR_NOMEM;
        if (nan_seen)
            rc = ORC_ERR_NAN;
        else if (kind == ORC_DGC)
            rc = dgc_pick(values, mk, n, k, seed, stream, pos_base, dgc_sample_fraction, out_idx);
        else /* TOPK and REDSYNC share the support (compressors.py:157-161 -> exact top-k) */
            rc = orc_select_keys(mk, n, k, out_idx);
        free(mk);
    }
    if (rc != ORC_OK)
        return rc;
    for (uint64_t j = 0; j < k; j++)
        out_vals[j] = values[out_idx[j]];
    if (kind == ORC_REDSYNC) {
        /* compressors.py:187-189: vals = sign(v) * fl32(mean_f64(|v|)) */
        double *a = (double *)malloc(k * sizeof(double));
        if (!a)
            return ORC_ERR_NOMEM;
        for (uint64_t j = 0; j < k; j++)
            a[j] = fabs((double)out_vals[j]);
        double mean = orc_pairwise_sum_f64(a, k) / (double)k;
        free(a);
        float m = (float)mean;
        for (uint64_t j = 0; j < k; j++) {
            float v = out_vals[j];
            float sg = v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : 0.0f);
            volatile float p = sg * m;
            out_vals[j] = p;
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------- aggregation */
int orc_aggregate(const uint32_t *idx, const float *vals, const uint64_t *counts,
                  int nparts, uint64_t n, float *out)
{
    if (nparts < 1)
        return ORC_ERR_ARG;
    double *acc = (double *)calloc(n, sizeof(double));
    if (!acc)
        return ORC_ERR_NOMEM;
    uint64_t off = 0;
    for (int p = 0; p < nparts; p++) {
        for (uint64_t j = 0; j < counts[p]; j++)
            if (idx[off + j] >= n) {
                free(acc);
                return ORC_ERR_ARG;
            }
        /* a part's indices are distinct: its scatter splits over threads
         * (parts in order, so every sum keeps the part order) */
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
        for (uint64_t j = 0; j < counts[p]; j++)
            acc[idx[off + j]] += (double)vals[off + j];
        off += counts[p];
    }
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
    for (uint64_t i = 0; i < n; i++)
        out[i] = (float)(acc[i] / (double)nparts);
    free(acc);
    return ORC_OK;
}

int orc_aggregate_dense(const float *parts, int nparts, uint64_t n, float *out)
{
    if (nparts < 1)
        return ORC_ERR_ARG;
    for (uint64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int p = 0; p < nparts; p++)
            acc += (double)parts[(uint64_t)p * n + i];
        out[i] = (float)(acc / (double)nparts);
    }
    return ORC_OK;
}

void orc_update_residual(const float *g_ef, const uint32_t *idx, const float *vals,
                         uint64_t k, uint64_t n, float *r_out)
{
    if (r_out != g_ef) {
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
        for (uint64_t i = 0; i < n; i++)
            r_out[i] = g_ef[i];
    }
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
    for (uint64_t j = 0; j < k; j++) {
        volatile float d = r_out[idx[j]] - vals[j];
        r_out[idx[j]] = d;
    }
}
