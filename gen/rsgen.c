/*
 * rsgen — seeded synthetic community graphs for the RSI hot path.
 *
 * INPUT GENERATOR ONLY. This module holds none of the method's arithmetic
 * (no histogram, entropy, weight, triad or ranking code). It is the one
 * module both sides (oracle/ and the CUDA path) may consume, as the task's
 * parity rules require; neither side imports the other.
 *
 * Model (SURVEY.md §8(d) "Synthetic inputs"): a degree-corrected stochastic
 * block model (Chung–Lu inside and across blocks) with
 *   - Zipf(s) community sizes over n_comm blocks,
 *   - Pareto(gamma) expected degrees clipped at dmax, rescaled to 2m/n,
 *   - mixing mu: an edge's second endpoint is drawn from the first
 *     endpoint's own block with probability 1-mu, else from the whole graph,
 *   - triadic closure tau: that fraction of edges closes a random wedge
 *     a-b-c of the base graph (creates the triangles Type-I triads need),
 *   - random vertex and community relabeling (no locality gift).
 * The result is canonical (SURVEY C-17): simple, undirected, stored
 * symmetric, every row strictly ascending, no self-loops.
 *
 * Randomness is counter-based: every draw is mix(seed, stream, index), so
 * the output is bit-identical for any OpenMP thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n;
    int64_t m_target;   /* undirected edges wanted (before dedup losses) */
    double gamma;       /* power-law exponent of expected degrees        */
    double dmax;        /* expected-degree clip                          */
    int32_t n_comm;     /* number of planted communities                 */
    double zipf_s;      /* community size exponent                       */
    double mu;          /* probability an edge leaves its block          */
    double tau;         /* fraction of edges made by triadic closure     */
    double oversample;  /* edge draws multiplier (dedup compensation)    */
    uint64_t seed;
} rsgen_params;

typedef struct {
    int64_t n, nnz;
    int64_t *rowptr;   /* n+1 */
    int32_t *col;      /* nnz */
    int32_t *comm;     /* n   */
} rsgen_graph;

/* ---------------- counter-based RNG ---------------- */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t rng(uint64_t seed, uint64_t stream, uint64_t i) {
    uint64_t k = mix64(seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1)));
    return mix64(k ^ mix64(i * 0xD1B54A32D192ED03ULL + 0x8CB92BA72F3D8DD7ULL));
}
static inline double u01(uint64_t x) { return (double)(x >> 11) * (1.0 / 9007199254740992.0); }

/* ---------------- alias tables (Vose) ---------------- */
typedef struct { double *prob; int64_t *alias; } alias_t;

static void alias_build(const double *w, int64_t len, double *prob, int64_t *alias) {
    double sum = 0; for (int64_t i = 0; i < len; i++) sum += w[i];
    int64_t *small = malloc(sizeof(int64_t) * len), *large = malloc(sizeof(int64_t) * len);
    int64_t ns = 0, nl = 0;
    for (int64_t i = 0; i < len; i++) {
        prob[i] = w[i] * (double)len / sum;
        alias[i] = i;
        if (prob[i] < 1.0) small[ns++] = i; else large[nl++] = i;
    }
    while (ns && nl) {
        int64_t s = small[--ns], l = large[--nl];
        alias[s] = l;
        prob[l] = (prob[l] + prob[s]) - 1.0;
        if (prob[l] < 1.0) small[ns++] = l; else large[nl++] = l;
    }
    while (nl) prob[large[--nl]] = 1.0;
    while (ns) prob[small[--ns]] = 1.0;
    free(small); free(large);
}
/* draw from table slice [base, base+len) with one 64-bit random word */
static inline int64_t alias_draw(const double *prob, const int64_t *alias, int64_t base, int64_t len, uint64_t r) {
    int64_t b = (int64_t)(((r >> 32) * (uint64_t)len) >> 32);
    double coin = (double)(r & 0xffffffffULL) * (1.0 / 4294967296.0);
    return coin < prob[base + b] ? base + b : alias[base + b];
}

/* ---------------- CSR build from an edge list ---------------- */
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b; return (x > y) - (x < y);
}

/* edges: pairs (src[i], dst[i]) with src!=dst or src<0 (dropped). Builds
 * symmetric, sorted, deduplicated CSR. */
static int build_csr(int64_t n, int64_t ne, const int32_t *src, const int32_t *dst,
                     int64_t **rowptr_out, int32_t **col_out, int64_t *nnz_out) {
    int64_t *deg = calloc(n + 1, sizeof(int64_t));
    if (!deg) return -1;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; i++) {
        if (src[i] < 0) continue;
        __atomic_fetch_add(&deg[src[i]], 1, __ATOMIC_RELAXED);
        __atomic_fetch_add(&deg[dst[i]], 1, __ATOMIC_RELAXED);
    }
    int64_t *off = malloc(sizeof(int64_t) * (n + 1));
    off[0] = 0;
    for (int64_t v = 0; v < n; v++) off[v + 1] = off[v] + deg[v];
    int64_t tot = off[n];
    int32_t *tmp = malloc(sizeof(int32_t) * (tot ? tot : 1));
    int64_t *pos = deg; /* reuse as cursor */
    memcpy(pos, off, sizeof(int64_t) * n);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ne; i++) {
        if (src[i] < 0) continue;
        int64_t p = __atomic_fetch_add(&pos[src[i]], 1, __ATOMIC_RELAXED); tmp[p] = dst[i];
        int64_t q = __atomic_fetch_add(&pos[dst[i]], 1, __ATOMIC_RELAXED); tmp[q] = src[i];
    }
    int64_t *nd = malloc(sizeof(int64_t) * (n + 1));
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++) {
        int32_t *r = tmp + off[v]; int64_t d = off[v + 1] - off[v];
        if (d > 1) qsort(r, (size_t)d, sizeof(int32_t), cmp_i32);
        int64_t w = 0;
        for (int64_t j = 0; j < d; j++) if (j == 0 || r[j] != r[j - 1]) r[w++] = r[j];
        nd[v] = w;
    }
    int64_t *rp = malloc(sizeof(int64_t) * (n + 1));
    rp[0] = 0;
    for (int64_t v = 0; v < n; v++) rp[v + 1] = rp[v] + nd[v];
    int32_t *col = malloc(sizeof(int32_t) * (rp[n] ? rp[n] : 1));
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t v = 0; v < n; v++) memcpy(col + rp[v], tmp + off[v], sizeof(int32_t) * nd[v]);
    free(deg); free(off); free(tmp); free(nd);
    *rowptr_out = rp; *col_out = col; *nnz_out = rp[n];
    return 0;
}

/* ---------------- generator ---------------- */
enum { ST_PERM = 1, ST_CPERM = 2, ST_THETA = 3, ST_BASE = 4, ST_CLOSE = 5 };

typedef struct { uint64_t key; int64_t idx; } keyidx;
static int cmp_keyidx(const void *a, const void *b) {
    const keyidx *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->idx > y->idx) - (x->idx < y->idx);
}

int rsgen_generate(const rsgen_params *p, rsgen_graph *g) {
    memset(g, 0, sizeof(*g));
    const int64_t n = p->n;
    const int32_t nc = p->n_comm;
    if (n < 2 || n > 2147483647LL || nc < 1 || nc > n || p->m_target < 0) return -1;

    /* 1. Zipf community sizes (blocks of the pre-relabel id space) */
    int64_t *cstart = malloc(sizeof(int64_t) * (nc + 1));
    {
        double z = 0; for (int c = 0; c < nc; c++) z += pow(c + 1.0, -p->zipf_s);
        int64_t acc = 0;
        for (int c = 0; c < nc; c++) {
            int64_t s = (int64_t)llround((double)n * pow(c + 1.0, -p->zipf_s) / z);
            if (s < 2) s = 2;
            cstart[c] = acc; acc += s;
        }
        /* absorb the rounding difference in the largest block */
        int64_t diff = n - acc;
        for (int c = 1; c < nc; c++) cstart[c] += diff;
        cstart[nc] = n;
        if (cstart[1] - cstart[0] < 2) { free(cstart); return -2; }
    }
    int32_t *block = malloc(sizeof(int32_t) * n);
    for (int c = 0; c < nc; c++) for (int64_t v = cstart[c]; v < cstart[c + 1]; v++) block[v] = c;

    /* 2. random relabeling: vertex permutation pi and community permutation */
    int32_t *pi = malloc(sizeof(int32_t) * n);
    {
        keyidx *ki = malloc(sizeof(keyidx) * n);
        #pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < n; v++) { ki[v].key = rng(p->seed, ST_PERM, (uint64_t)v); ki[v].idx = v; }
        qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
        for (int64_t r = 0; r < n; r++) pi[ki[r].idx] = (int32_t)r;   /* old id ki[r].idx -> new id r */
        free(ki);
    }
    int32_t *cperm = malloc(sizeof(int32_t) * nc);
    {
        keyidx *ki = malloc(sizeof(keyidx) * nc);
        for (int c = 0; c < nc; c++) { ki[c].key = rng(p->seed, ST_CPERM, (uint64_t)c); ki[c].idx = c; }
        qsort(ki, (size_t)nc, sizeof(keyidx), cmp_keyidx);
        for (int r = 0; r < nc; r++) cperm[ki[r].idx] = r;
        free(ki);
    }

    /* 3. expected degrees: Pareto(gamma-1) tail, rescaled to mean 2m/n, clipped at dmax */
    double *theta = malloc(sizeof(double) * n);
    {
        const double a = 1.0 / (p->gamma - 1.0);
        #pragma omp parallel for schedule(static)
        for (int64_t v = 0; v < n; v++) theta[v] = pow(1.0 - u01(rng(p->seed, ST_THETA, (uint64_t)v)), -a);
        const double want = 2.0 * (double)p->m_target;
        for (int it = 0; it < 8; it++) {
            double s = 0; for (int64_t v = 0; v < n; v++) s += theta[v];
            double f = want / s;
            for (int64_t v = 0; v < n; v++) { theta[v] *= f; if (p->dmax > 0 && theta[v] > p->dmax) theta[v] = p->dmax; }
        }
    }
    double *gprob = malloc(sizeof(double) * n);  int64_t *galias = malloc(sizeof(int64_t) * n);
    double *cprob = malloc(sizeof(double) * n);  int64_t *calias = malloc(sizeof(int64_t) * n);
    alias_build(theta, n, gprob, galias);
    for (int c = 0; c < nc; c++) {
        int64_t b = cstart[c], len = cstart[c + 1] - b;
        alias_build(theta + b, len, cprob + b, calias + b);
        for (int64_t i = b; i < b + len; i++) calias[i] += b;  /* slice-local -> global */
    }
    free(theta);

    /* 4. base DC-SBM edges (new ids) */
    const int64_t m_base = (int64_t)llround((double)p->m_target * (1.0 - p->tau) * p->oversample);
    const int64_t m_close = (int64_t)llround((double)p->m_target * p->tau * p->oversample);
    int32_t *src = malloc(sizeof(int32_t) * (m_base + m_close + 1));
    int32_t *dst = malloc(sizeof(int32_t) * (m_base + m_close + 1));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m_base; i++) {
        uint64_t r0 = rng(p->seed, ST_BASE, 3 * (uint64_t)i);
        uint64_t r1 = rng(p->seed, ST_BASE, 3 * (uint64_t)i + 1);
        uint64_t r2 = rng(p->seed, ST_BASE, 3 * (uint64_t)i + 2);
        int64_t a = alias_draw(gprob, galias, 0, n, r0), b;
        if (u01(r1) >= p->mu) {
            int c = block[a]; b = alias_draw(cprob, calias, cstart[c], cstart[c + 1] - cstart[c], r2);
        } else {
            b = alias_draw(gprob, galias, 0, n, r2);
        }
        if (a == b) { src[i] = -1; dst[i] = -1; }
        else { src[i] = pi[a]; dst[i] = pi[b]; }
    }
    free(gprob); free(galias); free(cprob); free(calias);

    /* 5. triadic closure over the base graph */
    int64_t *brp; int32_t *bcol; int64_t bnnz;
    if (build_csr(n, m_base, src, dst, &brp, &bcol, &bnnz)) return -3;
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < m_close; j++) {
        int64_t i = m_base + j;
        src[i] = -1; dst[i] = -1;
        if (bnnz == 0) continue;
        uint64_t r0 = rng(p->seed, ST_CLOSE, 2 * (uint64_t)j);
        uint64_t r1 = rng(p->seed, ST_CLOSE, 2 * (uint64_t)j + 1);
        int64_t e = (int64_t)(((r0 >> 11) % (uint64_t)bnnz));
        /* row of entry e: largest a with brp[a] <= e */
        int64_t lo = 0, hi = n;
        while (hi - lo > 1) { int64_t mid = (lo + hi) >> 1; if (brp[mid] <= e) lo = mid; else hi = mid; }
        int32_t a = (int32_t)lo, b = bcol[e];
        int64_t db = brp[b + 1] - brp[b];
        int32_t c = bcol[brp[b] + (int64_t)((r1 >> 11) % (uint64_t)db)];
        if (c != a) { src[i] = a; dst[i] = c; }
    }
    free(brp); free(bcol);

    /* 6. final canonical CSR */
    if (build_csr(n, m_base + m_close, src, dst, &g->rowptr, &g->col, &g->nnz)) return -4;
    free(src); free(dst);
    g->n = n;
    g->comm = malloc(sizeof(int32_t) * n);
    for (int64_t v = 0; v < n; v++) g->comm[pi[v]] = cperm[block[v]];
    free(pi); free(block); free(cstart); free(cperm);
    return 0;
}

/* ---------------- handle API for the Python wrapper ---------------- */
void *rsgen_create(const rsgen_params *p, int *status) {
    rsgen_graph *g = malloc(sizeof(rsgen_graph));
    int s = rsgen_generate(p, g);
    if (status) *status = s;
    if (s) { free(g); return NULL; }
    return g;
}
int64_t rsgen_n(const void *h) { return ((const rsgen_graph *)h)->n; }
int64_t rsgen_nnz(const void *h) { return ((const rsgen_graph *)h)->nnz; }
void rsgen_fill(const void *h, int64_t *rowptr, int32_t *col, int32_t *comm) {
    const rsgen_graph *g = h;
    memcpy(rowptr, g->rowptr, sizeof(int64_t) * (g->n + 1));
    memcpy(col, g->col, sizeof(int32_t) * g->nnz);
    memcpy(comm, g->comm, sizeof(int32_t) * g->n);
}
void rsgen_destroy(void *h) {
    rsgen_graph *g = h; if (!g) return;
    free(g->rowptr); free(g->col); free(g->comm); free(g);
}
