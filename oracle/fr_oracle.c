/*
 * fr_oracle.c -- CPU restatement of the fluidrank reference path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * product in paper_1202_6158_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links, imports or falls back to it.
 *
 * Every routine cites the reference file:line it restates
 * (reference = /root/reference/pkg/src/fluidrank/...).  The sequential solver
 * and power iteration reproduce the reference's floating-point operation
 * order exactly (including numpy's pairwise summation), so on the same graph
 * they return bit-identical vectors and counters; tests/test_oracle_golden.py
 * pins that against vectors produced by the reference itself.
 *
 * The synthetic graph generator (fro_gen_*) restates the BASELINE.json config
 * generators (config 1 "uniform", configs 2-5 "web"); it is the specification
 * the CUDA generator must match bit for bit.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off: no FMA contraction,
 * so float results equal the reference's numpy/scipy arithmetic).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* numpy pairwise summation (np.sum of a contiguous float64 array).          */
/* Used wherever the reference calls .sum(): engine.py:146 exact_residual,   */
/* engine.py:159 init residual, engine.py:236 _normalized, baseline.py:45.  */
/* ------------------------------------------------------------------------ */
static double pw_sum(const double *a, int64_t n, int absval)
{
    if (n < 8) {
        double res = 0.;
        for (int64_t i = 0; i < n; i++) res += absval ? fabs(a[i]) : a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = absval ? fabs(a[j]) : a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += absval ? fabs(a[i + j]) : a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += absval ? fabs(a[i]) : a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2, absval) + pw_sum(a + n2, n - n2, absval);
    }
}

double fro_pairwise_sum(const double *a, int64_t n, int absval) { return pw_sum(a, n, absval); }

/* ------------------------------------------------------------------------ */
/* Synthetic generator specification (BASELINE.json configs).               */
/* Counter-based hashing: every value is a pure function of (seed, node,     */
/* slot), so a GPU thread can compute any edge independently.               */
/* ------------------------------------------------------------------------ */
#define GOLD 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t z)
{
    z += GOLD;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) { return mix64(seed + stream * GOLD); }
static inline uint64_t frand(uint64_t key, uint64_t a, uint64_t b) { return mix64(mix64(key ^ a) + b); }
static inline double u53(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

enum { FRO_STREAM_DEG = 1, FRO_STREAM_EDGE = 3, FRO_STREAM_ZIPF = 4, FRO_STREAM_FEISTEL = 5 };

typedef struct {
    int32_t kind;          /* 0 = uniform (config 1), 1 = web (configs 2-5) */
    int32_t max_out;       /* uniform: out-degree uniform in {0..max_out}    */
    double mean_degree;    /* web: target mean out-degree (before dedup)     */
    double alpha;          /* web: power-law exponent of out-degree          */
    int32_t max_degree;    /* web: power-law truncation                      */
    int32_t window;        /* web: local targets within +-window             */
    double dangling_frac;  /* web: fraction of nodes forced to out-degree 0  */
    double local_frac;     /* web: fraction of targets that are local        */
    double zipf_s;         /* web: Zipf exponent of the non-local targets    */
} fro_gen_config;

static uint32_t frac_to_u32(double f)
{
    double x = floor(f * 4294967296.0);
    if (x < 0) x = 0;
    if (x > 4294967295.0) x = 4294967295.0;
    return (uint32_t)x;
}

/* first index i with cdf[i] > x  (numpy searchsorted side='right') */
static inline int64_t search_right(const double *cdf, int64_t len, double x)
{
    int64_t lo = 0, hi = len - 1;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (cdf[mid] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* Power-law out-degree table and the Q32 scale that rescales its mean. */
int fro_gen_powerlaw_table(const fro_gen_config *c, double *cdf /* max_degree */, uint64_t *scale_q32)
{
    int64_t kmax = c->max_degree;
    if (kmax < 1) return -1;
    double cum = 0.0, wsum = 0.0, kwsum = 0.0;
    for (int64_t k = 1; k <= kmax; k++) {
        double w = pow((double)k, -c->alpha);
        cum += w;
        cdf[k - 1] = cum;
    }
    for (int64_t k = 1; k <= kmax; k++) {
        double w = pow((double)k, -c->alpha);
        wsum += w;
        kwsum += (double)k * w;
    }
    for (int64_t k = 0; k < kmax; k++) cdf[k] = cdf[k] / cum;
    cdf[kmax - 1] = 1.0;
    double p_live = 1.0 - (double)frac_to_u32(c->dangling_frac) / 4294967296.0;
    double mean_k = kwsum / wsum;
    double scale = c->mean_degree / (p_live * mean_k);
    *scale_q32 = (uint64_t)llround(scale * 4294967296.0);
    return 0;
}

/* Zipf(s) CDF over ranks 0..n-1 (weight of rank k is (k+1)^-s). */
void fro_gen_zipf_table(int64_t n, double s, double *cdf)
{
    double cum = 0.0;
    for (int64_t k = 0; k < n; k++) {
        double w = (s == 1.0) ? 1.0 / (double)(k + 1) : pow((double)(k + 1), -s);
        cum += w;
        cdf[k] = cum;
    }
    for (int64_t k = 0; k < n; k++) cdf[k] = cdf[k] / cum;
    cdf[n - 1] = 1.0;
}

/* The Zipf table of the last (n, s) asked for, kept across fill rounds. */
static double *zipf_cache;
static int64_t zipf_cache_n = -1;
static double zipf_cache_s;
static const double *zipf_cached(int64_t n, double s)
{
    if (zipf_cache && zipf_cache_n == n && zipf_cache_s == s) return zipf_cache;
    free(zipf_cache);
    zipf_cache = (double *)malloc(sizeof(double) * (size_t)n);
    zipf_cache_n = zipf_cache ? n : -1;
    zipf_cache_s = s;
    if (zipf_cache) fro_gen_zipf_table(n, s, zipf_cache);
    return zipf_cache;
}

/* Keyed Feistel bijection on [0, n) with cycle walking: the "random
 * permutation of node IDs" the Zipf targets are drawn over. */
static uint64_t feistel(uint64_t x, uint64_t n, const uint64_t keys[4], int half)
{
    uint64_t mask = (1ull << half) - 1;
    do {
        uint64_t L = x >> half, R = x & mask;
        for (int r = 0; r < 4; r++) {
            uint64_t t = R;
            R = L ^ (mix64(R ^ keys[r]) & mask);
            L = t;
        }
        x = (L << half) | R;
    } while (x >= n);
    return x;
}
static int feistel_half(uint64_t n)
{
    int bits = 2;
    while ((1ull << bits) < n) bits++;
    if (bits & 1) bits++;
    return bits / 2;
}
uint64_t fro_gen_feistel(uint64_t x, uint64_t n, uint64_t seed)
{
    uint64_t keys[4];
    for (int r = 0; r < 4; r++) keys[r] = stream_key(seed, FRO_STREAM_FEISTEL + r);
    return feistel(x, n, keys, feistel_half(n));
}

/* Out-degree of every node (pre-dedup slot count). Returns total slots. */
int64_t fro_gen_degrees(const fro_gen_config *c, int64_t n, uint64_t seed, uint32_t *deg)
{
    uint64_t kd = stream_key(seed, FRO_STREAM_DEG);
    int64_t total = 0;
    if (c->kind == 0) {
#pragma omp parallel for reduction(+ : total) schedule(static)
        for (int64_t u = 0; u < n; u++) {
            uint64_t g = frand(kd, (uint64_t)u, 0) % (uint64_t)(c->max_out + 1);
            if (n < 2) g = 0;
            else if (g > (uint64_t)(n - 1)) g = (uint64_t)(n - 1);
            deg[u] = (uint32_t)g;
            total += (int64_t)g;
        }
        return total;
    }
    double *cdf = (double *)malloc(sizeof(double) * (size_t)c->max_degree);
    uint64_t scale_q32;
    if (!cdf || fro_gen_powerlaw_table(c, cdf, &scale_q32)) { free(cdf); return -1; }
    uint32_t dthr = frac_to_u32(c->dangling_frac);
#pragma omp parallel for reduction(+ : total) schedule(static)
    for (int64_t u = 0; u < n; u++) {
        uint64_t g = 0;
        if (n >= 2 && (uint32_t)(frand(kd, (uint64_t)u, 0) >> 32) >= dthr) {
            uint64_t k = (uint64_t)search_right(cdf, c->max_degree, u53(frand(kd, (uint64_t)u, 1))) + 1;
            g = (k * scale_q32 + (frand(kd, (uint64_t)u, 2) & 0xffffffffull)) >> 32;
            if (g < 1) g = 1;
            if (g > (uint64_t)(n - 1)) g = (uint64_t)(n - 1);
        }
        deg[u] = (uint32_t)g;
        total += (int64_t)g;
    }
    free(cdf);
    return total;
}

/* Target of slot j of source u (web kind needs the zipf table).  zipf_only:
 * the node's local window already holds every id (a fill round), so the
 * local class is skipped. */
static inline uint32_t gen_target(const fro_gen_config *c, int64_t n, uint64_t ke, uint64_t kz,
                                  const double *zcdf, const uint64_t fk[4], int half,
                                  uint32_t lthr, int64_t u, int64_t j, int zipf_only)
{
    uint64_t r = frand(ke, (uint64_t)u, (uint64_t)j);
    if (c->kind == 0) {
        uint64_t t = r % (uint64_t)(n - 1);
        if (t >= (uint64_t)u) t++;
        return (uint32_t)t;
    }
    if (!zipf_only && (uint32_t)(r >> 32) < lthr) {
        uint32_t w2 = 2u * (uint32_t)c->window;
        int64_t o = (int64_t)((uint32_t)r % w2);
        int64_t off = o < c->window ? o - c->window : o - c->window + 1;
        int64_t v = (u + off) % n;
        if (v < 0) v += n;
        return (uint32_t)v;
    }
    int64_t rank = search_right(zcdf, n, u53(frand(kz, (uint64_t)u, (uint64_t)j)));
    return (uint32_t)feistel((uint64_t)rank, (uint64_t)n, fk, half);
}

/* Draw-stream keys of fill round r (fro_gen_edges_round): round 0 is the base
 * draw; round r > 0 redraws the slots that cleaning dropped (duplicates,
 * self-loops) from fresh edge / Zipf streams.  The Feistel permutation is a
 * property of the graph and stays the same in every round. */
#define FILL_GOLD 0xD1B54A32D192ED03ull
static void round_keys(uint64_t seed, uint32_t round, uint64_t *ke, uint64_t *kz)
{
    *ke = stream_key(seed, FRO_STREAM_EDGE);
    *kz = stream_key(seed, FRO_STREAM_ZIPF);
    if (round) {
        *ke = mix64(*ke ^ ((uint64_t)round * FILL_GOLD));
        *kz = mix64(*kz ^ ((uint64_t)round * FILL_GOLD));
    }
}

/* first position in t[lo, hi) holding a value >= x */
static int64_t lower_u32(const uint32_t *t, int64_t lo, int64_t hi, uint64_t x)
{
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if ((uint64_t)t[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Ids of node u's local window (u +- window, wrapped, u excluded) present in
 * its sorted row tgt[lo, hi). */
static int64_t window_count(const uint32_t *tgt, int64_t lo, int64_t hi, int64_t u, int64_t w, int64_t n)
{
    /* count of row entries in [a, b] (inclusive, 0 <= a <= b < n) */
#define ROW_RANGE(a, b) (lower_u32(tgt, lo, hi, (uint32_t)(b) + 1ull) - lower_u32(tgt, lo, hi, (uint32_t)(a)))
    if (2 * w + 1 >= n) return hi - lo;  /* the window is every other node */
    int64_t a = u - w, b = u + w;
    if (a >= 0 && b < n) return ROW_RANGE(a, b);
    if (a < 0) return ROW_RANGE(0, b) + ROW_RANGE(a + n, n - 1);
    return ROW_RANGE(a, n - 1) + ROW_RANGE(0, b - n);
#undef ROW_RANGE
}

/* Edge list in source-major slot order: edges of u occupy
 * [eoff[u], eoff[u] + deg[u]).  src/dst have length sum(deg).  round 0 is the
 * base draw (fro_gen_edges); deg is then the per-node deficit of a fill round
 * and (off, tgt) the clean graph so far: a node whose local window is already
 * complete in it draws its fill slots from the Zipf class only. */
int fro_gen_edges_round(const fro_gen_config *c, int64_t n, uint64_t seed, uint32_t round, const uint32_t *deg,
                        const int64_t *off, const uint32_t *tgt, uint32_t *src, uint32_t *dst)
{
    uint64_t ke, kz;
    round_keys(seed, round, &ke, &kz);
    uint64_t fk[4];
    for (int r = 0; r < 4; r++) fk[r] = stream_key(seed, FRO_STREAM_FEISTEL + r);
    int half = feistel_half((uint64_t)n);
    const double *zcdf = NULL;
    if (c->kind == 1 && !(zcdf = zipf_cached(n, c->zipf_s))) return -1;
    uint32_t lthr = frac_to_u32(c->local_frac);
    int64_t *eoff = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!eoff) return -1;
    eoff[0] = 0;
    for (int64_t u = 0; u < n; u++) eoff[u + 1] = eoff[u] + deg[u];
    const int64_t wfull = 2 * (int64_t)c->window < n - 1 ? 2 * (int64_t)c->window : n - 1;
    /* every slot is a pure function of (seed, round, u, j): the order of the
     * per-node work does not change the output */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t u = 0; u < n; u++) {
        if (!deg[u]) continue;
        const int zonly = c->kind == 1 && off && window_count(tgt, off[u], off[u + 1], u, c->window, n) >= wfull;
        int64_t e = eoff[u];
        for (int64_t j = 0; j < (int64_t)deg[u]; j++, e++) {
            src[e] = (uint32_t)u;
            dst[e] = gen_target(c, n, ke, kz, zcdf, fk, half, lthr, u, j, zonly);
        }
    }
    free(eoff);
    return 0;
}

int fro_gen_edges(const fro_gen_config *c, int64_t n, uint64_t seed, const uint32_t *deg,
                  uint32_t *src, uint32_t *dst)
{
    return fro_gen_edges_round(c, n, seed, 0, deg, NULL, NULL, src, dst);
}

/* ------------------------------------------------------------------------ */
/* CSR construction.                                                        */
/* strict (clean=0): graph.py:74-97 SparseGraph.from_edges -- range check,   */
/*   self-loop check, lexsort by (src, dst), duplicate check, cumsum of the  */
/*   out-degree bincount.                                                   */
/* clean (clean=1): graph.py:183-200 build_clean_edges then from_edges --    */
/*   self-loops dropped, duplicates collapsed, counts reported.             */
/* Returns 0 ok, 1 endpoint out of range, 2 self-loop, 3 duplicate edge.    */
/* ------------------------------------------------------------------------ */
static int cmp_u32(const void *a, const void *b)
{
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

int fro_csr_build(int64_t n, int64_t m, const uint32_t *src, const uint32_t *dst, int clean,
                  int64_t *off /* n+1 */, uint32_t *tgt /* m */, int64_t *stats /* 3 */)
{
    int64_t loops = 0, dups = 0;
    for (int64_t e = 0; e < m; e++)
        if ((int64_t)src[e] >= n || (int64_t)dst[e] >= n) return 1;
    for (int64_t e = 0; e < m; e++) {
        if (src[e] == dst[e]) {
            if (!clean) return 2;
            loops++;
        }
    }
    memset(off, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t e = 0; e < m; e++)
        if (src[e] != dst[e]) off[src[e] + 1]++;
    for (int64_t i = 0; i < n; i++) off[i + 1] += off[i];
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!cur) return -1;
    memcpy(cur, off, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m; e++)
        if (src[e] != dst[e]) tgt[cur[src[e]]++] = dst[e];
    free(cur);
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++)
        qsort(tgt + off[i], (size_t)(off[i + 1] - off[i]), sizeof(uint32_t), cmp_u32);
    int64_t w = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t b = off[i], e = off[i + 1];
        off[i] = w;
        for (int64_t k = b; k < e; k++) {
            if (k > b && tgt[k] == tgt[k - 1]) {
                if (!clean) return 3;
                dups++;
                continue;
            }
            tgt[w++] = tgt[k];
        }
    }
    off[n] = w;
    if (stats) { stats[0] = w; stats[1] = dups; stats[2] = loops; }
    return 0;
}

/* Clean union of a clean CSR (rows sorted, unique, no self-loops) with extra
 * edges (src2, dst2): build_clean_edges (graph.py:183-200) of the concatenated
 * edge list, computed row by row as a merge.  stats = {L, duplicates dropped,
 * self-loops dropped} of the extra edges. */
int fro_csr_merge(int64_t n, const int64_t *off, const uint32_t *tgt, int64_t m2, const uint32_t *src2,
                  const uint32_t *dst2, int64_t *off_out /* n+1 */, uint32_t *tgt_out /* off[n]+m2 */,
                  int64_t *stats /* 3 */)
{
    int64_t *o2 = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    uint32_t *t2 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(m2 > 0 ? m2 : 1));
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    if (!o2 || !t2 || !cur) { free(o2); free(t2); free(cur); return -1; }
    int64_t loops = 0, dups = 0;
    for (int64_t e = 0; e < m2; e++) {
        if ((int64_t)src2[e] >= n || (int64_t)dst2[e] >= n) { free(o2); free(t2); free(cur); return 1; }
        if (src2[e] == dst2[e]) loops++;
        else o2[src2[e] + 1]++;
    }
    for (int64_t i = 0; i < n; i++) o2[i + 1] += o2[i];
    memcpy(cur, o2, sizeof(int64_t) * (size_t)n);
    for (int64_t e = 0; e < m2; e++)
        if (src2[e] != dst2[e]) t2[cur[src2[e]]++] = dst2[e];
    /* pass 1 (rows in parallel): sort the extra edges, size of each row's union */
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        int64_t b2 = o2[i], e2 = o2[i + 1];
        if (e2 == b2) { cur[i] = off[i + 1] - off[i]; continue; }
        qsort(t2 + b2, (size_t)(e2 - b2), sizeof(uint32_t), cmp_u32);
        int64_t a = off[i], ae = off[i + 1], k = b2, cnt = 0;
        uint32_t last = 0;
        while (a < ae || k < e2) {
            const uint32_t v = (k >= e2 || (a < ae && tgt[a] <= t2[k])) ? tgt[a++] : t2[k++];
            if (cnt && last == v) continue;
            last = v;
            cnt++;
        }
        cur[i] = cnt;
    }
    int64_t w = 0;
    for (int64_t i = 0; i < n; i++) {
        off_out[i] = w;
        w += cur[i];
    }
    off_out[n] = w;
    dups = (off[n] + (m2 - loops)) - w;  /* the existing rows are unique: every repeat is an extra edge */
    /* pass 2 (rows in parallel): write the unions */
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        int64_t a = off[i], ae = off[i + 1], k = o2[i], e2 = o2[i + 1], o = off_out[i], row0 = o;
        while (a < ae || k < e2) {
            const uint32_t v = (k >= e2 || (a < ae && tgt[a] <= t2[k])) ? tgt[a++] : t2[k++];
            if (o > row0 && tgt_out[o - 1] == v) continue;
            tgt_out[o++] = v;
        }
    }
    free(o2); free(t2); free(cur);
    if (stats) { stats[0] = w; stats[1] = dups; stats[2] = loops; }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Sequential diffusion run: engine.py:240-341 (run) with the schedulers of  */
/* sched.py (sweep 69-113, max 16-25, per 52-66, op/op2 116-144) and the     */
/* diffusion step of engine.py:175-199 / 315-329.                            */
/* ------------------------------------------------------------------------ */
enum { FRO_SWEEP = 0, FRO_MAX = 1, FRO_PER = 2, FRO_OP = 3, FRO_OP2 = 4 };

typedef struct {
    int64_t elementary_steps;
    int64_t diffusions;
    double residual;
    double bound; /* NaN when undefined (damping >= 1) */
} fro_trace_row;

typedef struct {
    int64_t diffusions;
    int64_t elementary_steps;
    double residual;
    int64_t trace_len;
    int64_t sweeps;      /* parallel-sweep runs only */
    int32_t status;      /* 0 ok, 3 starvation */
} fro_run_result;

static int64_t trace_last_diff;
static void trace_push(fro_trace_row *tr, int64_t cap, int64_t *len, int64_t steps, int64_t diff,
                       double residual, double d)
{
    trace_last_diff = diff;
    if (*len < cap) {
        tr[*len].elementary_steps = steps;
        tr[*len].diffusions = diff;
        tr[*len].residual = residual;
        tr[*len].bound = d >= 1.0 ? NAN : residual / (1.0 - d);
    }
    (*len)++;
}

static int64_t argmax_scaled(const double *f, const double *w, int64_t n, int signed_)
{
    /* np.argmax: first index of the maximum */
    int64_t best = 0;
    double bv = 0.0;
    for (int64_t i = 0; i < n; i++) {
        double v = signed_ ? fabs(f[i]) : f[i];
        if (w) v = v * w[i];
        if (i == 0 || v > bv) { bv = v; best = i; }
    }
    return best;
}

/* fluid/history are the in/out state (engine.DiffusionState).  in_deg is
 * only read for kind op.  rank_out receives _normalized(history). */
int fro_run_seq(int64_t n, const int64_t *off, const uint32_t *tgt, const int64_t *in_deg,
                double d, double target_error, int kind, double decay, int64_t max_diffusions,
                int64_t trace_every, int signed_, double *fluid, double *history,
                double residual0, int64_t diffusions0, int64_t steps0,
                fro_trace_row *trace, int64_t trace_cap, double *rank_out, fro_run_result *res)
{
    double threshold = target_error * (1.0 - d);
    int64_t diffusions = diffusions0, steps = steps0;
    double residual = residual0;
    int64_t tlen = 0;
    if (trace_every <= 0) trace_every = n;
    int64_t next_trace = diffusions + trace_every;
    int64_t next_refresh = diffusions + n;
    int status = 0;

    double *w = NULL;
    if (kind == FRO_OP || kind == FRO_OP2) {
        w = (double *)malloc(sizeof(double) * (size_t)n);
        for (int64_t i = 0; i < n; i++) {
            double wt = (double)(off[i + 1] - off[i] + 1);
            if (kind == FRO_OP) wt *= (double)(in_deg[i] + 1);
            w[i] = 1.0 / wt;
        }
    }
    /* sweep scheduler state (sched.py:79-85) */
    int have_thr = 0;
    double sw_thr = 0.0;
    int64_t cursor = 0, hits_in_pass = 0;
    int64_t per_count = 0;
    /* starvation bookkeeping (engine.py:283-287) */
    int64_t *stamp = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int64_t epoch = 1, distinct_empty = 0, empty_streak = 0, streak_cap = 64 * n;

    trace_push(trace, trace_cap, &tlen, steps, diffusions, residual, d);
    for (;;) {
        if (residual <= threshold) {
            residual = pw_sum(fluid, n, signed_);
            if (residual <= threshold) break;
        }
        if (max_diffusions >= 0 && diffusions >= max_diffusions) break;

        int64_t i = 0;
        switch (kind) {
        case FRO_MAX: i = argmax_scaled(fluid, NULL, n, signed_); break;
        case FRO_OP:
        case FRO_OP2: i = argmax_scaled(fluid, w, n, signed_); break;
        case FRO_PER: i = per_count % n; per_count++; break;
        default: { /* FRO_SWEEP, sched.py:87-110 */
            if (!have_thr) {
                double mx = -INFINITY;
                for (int64_t k = 0; k < n; k++) { double v = signed_ ? fabs(fluid[k]) : fluid[k]; if (v > mx) mx = v; }
                sw_thr = mx;
                have_thr = 1;
            }
            for (;;) {
                int64_t k;
                for (k = cursor; k < n; k++) {
                    double v = signed_ ? fabs(fluid[k]) : fluid[k];
                    if (v >= sw_thr) break;
                }
                if (k < n) { i = k; cursor = k + 1; hits_in_pass++; break; }
                if (hits_in_pass == 0) {
                    double peak = -INFINITY;
                    for (int64_t q = 0; q < n; q++) { double v = signed_ ? fabs(fluid[q]) : fluid[q]; if (v > peak) peak = v; }
                    if (peak <= 0.0) { cursor = 1 % n; i = 0; goto picked; }
                    sw_thr *= decay;
                }
                cursor = 0;
                hits_in_pass = 0;
            }
        }
        }
    picked:;
        double sent = fluid[i];
        if (sent == 0.0) {
            empty_streak++;
            if (stamp[i] != epoch) { stamp[i] = epoch; distinct_empty++; }
            if (distinct_empty >= n || empty_streak >= streak_cap) {
                residual = pw_sum(fluid, n, signed_);
                if (residual <= threshold) break;
                status = 3;
                break;
            }
            continue;
        }
        fluid[i] = 0.0;
        history[i] += sent;
        int64_t lo = off[i], hi = off[i + 1], deg = hi - lo;
        if (deg) {
            double push = sent * (d / (double)deg);
            for (int64_t k = lo; k < hi; k++) fluid[tgt[k]] += push;
            residual -= fabs(sent) * (1.0 - d);
            steps += deg;
        } else {
            residual -= fabs(sent);
        }
        diffusions++;
        empty_streak = 0;
        distinct_empty = 0;
        epoch++;
        if (diffusions >= next_refresh) {
            residual = pw_sum(fluid, n, signed_);
            next_refresh = diffusions + n;
        }
        if (diffusions >= next_trace) {
            trace_push(trace, trace_cap, &tlen, steps, diffusions, residual, d);
            next_trace = diffusions + trace_every;
        }
    }
    if (status == 0) {
        residual = pw_sum(fluid, n, signed_);
        if (tlen == 0 || trace_last_diff != diffusions)
            trace_push(trace, trace_cap, &tlen, steps, diffusions, residual, d);
        if (rank_out) {
            double total = pw_sum(history, n, 1);
            for (int64_t k = 0; k < n; k++) rank_out[k] = total > 0.0 ? history[k] / total : history[k];
        }
    }
    free(stamp);
    free(w);
    res->diffusions = diffusions;
    res->elementary_steps = steps;
    res->residual = residual;
    res->trace_len = tlen;
    res->sweeps = 0;
    res->status = status;
    return status;
}

/* ------------------------------------------------------------------------ */
/* Data-parallel threshold sweep (the B200 product's schedule), restated     */
/* sequentially.  One sweep = select every node with |f| >= theta, move its  */
/* fluid to history, then push d*f/deg to its children (pushes land after    */
/* the selection, i.e. Jacobi within a sweep).  theta policy:                */
/*   0 exhaust   : theta *= decay only after a sweep that selected nothing   */
/*                 (the reference sweep scheduler's rule, sched.py:101-108)  */
/*   1 geometric : theta *= decay after every sweep (sec. 4.2,      */
/*                 "scaling down the threshold progressively")               */
/*   2 adaptive  : theta *= clamp(decay * sqrt(E / (edge_frac * m)),         */
/*                 0.25, 1.5), E = edges pushed by the sweep (product rule,  */
/*                 fr_diffuse.cu k_finalize)                                 */
/* Used to check the GPU's sweep counters and as the schedule model.        */
/* ------------------------------------------------------------------------ */
int fro_run_psweep(int64_t n, const int64_t *off, const uint32_t *tgt, double d, double target_error,
                   int policy, double decay, int64_t max_sweeps, int signed_, double *fluid,
                   double *history, fro_trace_row *trace, int64_t trace_cap, double *rank_out,
                   fro_run_result *res, const double *weight /* score multiplier (op/op2) or NULL */,
                   double edge_frac /* policy 2 target; <= 0: 0.2 */)
{
    const double edge_target = (edge_frac > 0.0 ? edge_frac : 0.2) * (double)(off[n] - off[0]);
    double threshold = target_error * (1.0 - d);
    int64_t diffusions = 0, steps = 0, sweeps = 0, tlen = 0;
    int64_t *sel = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double *sent = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double theta = 0.0, residual = pw_sum(fluid, n, signed_);
    for (int64_t i = 0; i < n; i++) { double v = fabs(fluid[i]) * (weight ? weight[i] : 1.0); if (v > theta) theta = v; }
    trace_push(trace, trace_cap, &tlen, steps, diffusions, residual, d);
    while (residual > threshold && (max_sweeps < 0 || sweeps < max_sweeps)) {
        int64_t ns = 0, steps0 = steps;
        double mass = 0.0, absorbed = 0.0, mx = 0.0;
        for (int64_t i = 0; i < n; i++) {
            double f = fluid[i], a = fabs(f);
            double sc = weight ? a * weight[i] : a;
            mass += a;
            if (sc > mx) mx = sc;
            if (f != 0.0 && sc >= theta) {
                fluid[i] = 0.0;
                history[i] += f;
                sel[ns] = i;
                sent[ns++] = f;
                absorbed += (off[i + 1] > off[i]) ? a * (1.0 - d) : a;
            }
        }
        for (int64_t s = 0; s < ns; s++) {
            int64_t i = sel[s], lo = off[i], hi = off[i + 1], deg = hi - lo;
            if (!deg) continue;
            double push = sent[s] * (d / (double)deg);
            for (int64_t k = lo; k < hi; k++) fluid[tgt[k]] += push;
            steps += deg;
        }
        diffusions += ns;
        sweeps++;
        residual = mass - absorbed;
        if (policy == 1) theta *= decay;
        if (policy == 2) {
            double ratio = edge_target > 0.0 ? (double)(steps - steps0) / edge_target : 1.0;
            double q = decay * sqrt(ratio > 1e-6 ? ratio : 1e-6);
            theta *= q < 0.25 ? 0.25 : (q > 1.5 ? 1.5 : q);
        }
        if (ns == 0 && mx > 0.0)
            while (theta > mx) theta *= decay;
        trace_push(trace, trace_cap, &tlen, steps, diffusions, residual, d);
    }
    residual = pw_sum(fluid, n, signed_);
    if (rank_out) {
        double total = pw_sum(history, n, 1);
        for (int64_t k = 0; k < n; k++) rank_out[k] = total > 0.0 ? history[k] / total : history[k];
    }
    free(sel);
    free(sent);
    res->diffusions = diffusions;
    res->elementary_steps = steps;
    res->residual = residual;
    res->trace_len = tlen;
    res->sweeps = sweeps;
    res->status = 0;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Power iteration: baseline.py:20-56.  in_off/in_src is the transposed    */
/* CSR (rows = targets, sources ascending), i.e. graph.to_matrix()'s scipy   */
/* CSR (graph.py:158-165); the row loop is scipy's csr_matvec.              */
/* teleport NULL = uniform 1/n.  Returns iterations, or -1 (no convergence). */
/* ------------------------------------------------------------------------ */
int64_t fro_power_iterate(int64_t n, const int64_t *in_off, const uint32_t *in_src,
                          const int64_t *out_deg, int64_t edge_count, double d,
                          const double *teleport, double target_error, int64_t max_iterations,
                          int64_t trace_every, double *x_out, fro_trace_row *trace,
                          int64_t trace_cap, int64_t *trace_len, double *diff_out)
{
    double *v = (double *)malloc(sizeof(double) * (size_t)n);
    double *inv = (double *)malloc(sizeof(double) * (size_t)n);
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        v[i] = teleport ? teleport[i] : 1.0 / (double)n;
        inv[i] = out_deg[i] ? 1.0 / (double)out_deg[i] : 0.0;
        x_out[i] = v[i];
    }
    double scale = d / (1.0 - d);
    int64_t steps = 0, tlen = 0, it;
    double diff = 0.0;
    if (trace_every <= 0) trace_every = 1;
    for (it = 1; it <= max_iterations; it++) {
        for (int64_t i = 0; i < n; i++) {
            double s = 0.0;
            for (int64_t k = in_off[i]; k < in_off[i + 1]; k++) s += inv[in_src[k]] * x_out[in_src[k]];
            y[i] = d * s + (1.0 - d) * v[i];
        }
        double c = 1.0 - pw_sum(y, n, 0);
        for (int64_t i = 0; i < n; i++) y[i] += c * v[i];
        for (int64_t i = 0; i < n; i++) tmp[i] = y[i] - x_out[i];
        diff = pw_sum(tmp, n, 1);
        memcpy(x_out, y, sizeof(double) * (size_t)n);
        steps += edge_count;
        if (it % trace_every == 0 || diff * scale <= target_error) {
            if (tlen < trace_cap) {
                trace[tlen].elementary_steps = steps;
                trace[tlen].diffusions = it;
                trace[tlen].residual = diff;
                trace[tlen].bound = diff * scale;
            }
            tlen++;
        }
        if (diff * scale <= target_error) break;
    }
    free(v); free(inv); free(y); free(tmp);
    if (trace_len) *trace_len = tlen;
    if (diff_out) *diff_out = diff;
    return it > max_iterations ? -1 : it;
}
