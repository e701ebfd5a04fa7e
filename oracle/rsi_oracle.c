/*
 * RSI ORACLE — plain, slow, single-threaded CPU definition of the method of
 * arXiv 2508.01485 ("A Parallel Algorithm for Finding Robust Spanners in
 * Large Social Networks"), written from PAPER.md.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library. The product path (paper_2508_01485_b200/, librs.so) never links,
 * imports or executes it, and shares no code, header, helper or table with
 * it. Citations "P:n" are PAPER.md line numbers; "C-n" are the readings
 * listed in SURVEY.md §8(c) and DESIGN.md §3.
 *
 * Precision: IEEE fp64 everywhere (the paper states none; C-19), base-2
 * logarithms (C-2, forced by the worked example's H = 1 at P:491), and the
 * per-head triad sum taken exactly in 128-bit fixed point with quantum 2^-80
 * so the sum is independent of enumeration order (C-12): each fp64 term is
 * rounded once to the 2^-80 grid, summed exactly, and converted back with one
 * rounding.
 *
 * Every function below is pinned by tests/test_oracle_*.py against values the
 * paper prints, closed forms, special cases and an independent brute-force
 * O(n^3) triple enumeration (tests/bruteforce.py). None is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---- O0. Target communities ("sort ... by size in descending
 * order and select the top k"; C-15 ties -> ascending community id). ---- */
typedef struct { int32_t id; int64_t size; } comm_size;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
static int cmp_size_desc_id_asc(const void *a, const void *b) {
    const comm_size *x = a, *y = b;
    if (x->size != y->size) return x->size > y->size ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* returns the number of distinct communities, or -1 if k is out of range */
int64_t oracle_select_targets(int64_t n, const int32_t *C, int32_t k, int32_t *targets_out) {
    int32_t *s = malloc(sizeof(int32_t) * (n ? n : 1));
    memcpy(s, C, sizeof(int32_t) * n);
    qsort(s, (size_t)n, sizeof(int32_t), cmp_i32);
    comm_size *cs = malloc(sizeof(comm_size) * (n ? n : 1));
    int64_t nc = 0;
    for (int64_t i = 0; i < n; i++) {
        if (i == 0 || s[i] != s[i - 1]) { cs[nc].id = s[i]; cs[nc].size = 0; nc++; }
        cs[nc - 1].size++;
    }
    qsort(cs, (size_t)nc, sizeof(comm_size), cmp_size_desc_id_asc);
    int64_t ret = nc;
    if (k < 1 || k > nc) ret = -1;
    else for (int32_t i = 0; i < k; i++) targets_out[i] = cs[i].id;
    free(s); free(cs);
    return ret;
}

/* column of community c among the k targets, or -1 (the symbol ⊥) */
static int32_t column_of(int32_t c, int32_t k, const int32_t *targets) {
    for (int32_t i = 0; i < k; i++) if (targets[i] == c) return i;
    return -1;
}

/* ---- O1. Border vertices ("u is called a community border vertex if
 * there exists at least one neighbor v in N(u) such that C(u) != C(v)";
 * Algorithm 1 Step 1). Over ALL communities. ---- */
int64_t oracle_border(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C,
                      uint8_t *border_out) {
    int64_t nb = 0;
    for (int64_t u = 0; u < n; u++) {
        uint8_t b = 0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++)
            if (C[col[e]] != C[u]) { b = 1; break; }
        border_out[u] = b;
        nb += b;
    }
    return nb;
}

/* ---- O2. Neighbour-community histogram (P:452-453 count_neighbor_community:
 * "counting the number of neighbors belonging to each community"
 * T = sum of the k considered communities; C-5: only the k targets count).
 * f_out is n*k row-major, T_out is n. ---- */
void oracle_counts(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C,
                   int32_t k, const int32_t *targets, int32_t *f_out, int32_t *T_out) {
    for (int64_t u = 0; u < n; u++) {
        int32_t *f = f_out + u * k;
        for (int32_t i = 0; i < k; i++) f[i] = 0;
        int32_t T = 0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
            int32_t j = column_of(C[col[e]], k, targets);
            if (j >= 0) { f[j]++; T++; }
        }
        T_out[u] = T;
    }
}

/* ---- O3. Weights. Eq.3 entropy of L(u,v) with
 * p(f_j) = f_j / sum_{l != i} f_l, summed directly over j != i with
 * f_j > 0 in ascending j; Eq.5 omega = H * |L| with Algorithm 2's
 * |L| = L_all - 1 (reading C-3); rows with L_all <= 1 are zero
 * (C-4, C-6; this also makes Y = T - f_i > 0 for every remaining column).
 * omega_out is n*k row-major, column i = omega_v(C_i) (Lemma 1). ---- */
void oracle_weights(int64_t n, int32_t k, const int32_t *f_all, double *omega_out) {
    for (int64_t v = 0; v < n; v++) {
        const int32_t *f = f_all + v * k;
        double *w = omega_out + v * k;
        int64_t T = 0; int32_t L_all = 0;
        for (int32_t j = 0; j < k; j++) { T += f[j]; if (f[j] > 0) L_all++; }
        for (int32_t i = 0; i < k; i++) {
            if (L_all <= 1) { w[i] = 0.0; continue; }
            double Y = (double)(T - f[i]);
            double H = 0.0;
            for (int32_t j = 0; j < k; j++) {
                if (j == i || f[j] == 0) continue;
                double p = (double)f[j] / Y;
                H -= p * log2(p);
            }
            w[i] = H * (double)(L_all - 1);
        }
    }
}

/* Algorithm 2 / Eq. H_optimal closed form, kept only so the
 * tests can check it against the direct form. C-18: X sums
 * f_i log f_i over the row; T is the row total. */
void oracle_weights_closed_form(int64_t n, int32_t k, const int32_t *f_all, double *omega_out) {
    for (int64_t v = 0; v < n; v++) {
        const int32_t *f = f_all + v * k;
        double *w = omega_out + v * k;
        double X = 0.0; int64_t T = 0; int32_t L_all = 0;
        for (int32_t i = 0; i < k; i++) {
            T += f[i];
            if (f[i] > 0) { X += (double)f[i] * log2((double)f[i]); L_all++; }
        }
        for (int32_t i = 0; i < k; i++) {
            if (L_all <= 1) { w[i] = 0.0; continue; }
            double Y = (double)(T - f[i]);
            double last = f[i] > 0 ? (double)f[i] * log2((double)f[i] / Y) : 0.0;
            double H = -(1.0 / Y) * (X - (double)T * log2(Y) - last);
            w[i] = H * (double)(L_all - 1);
        }
    }
}

/* ---- O4. omega_max (Algorithm 1 line "Find max edge weight", P:279;
 * normalize_weights divides every element by the maximum, P:485-486;
 * reading C-7: max over all cells). ---- */
double oracle_omega_max(int64_t n, int32_t k, const double *omega) {
    double m = 0.0;
    for (int64_t i = 0; i < n * (int64_t)k; i++) if (omega[i] > m) m = omega[i];
    return m;
}

/* ---- NEXT-3: the paper's literal variants. ----
 * flags & 1: |L(u,v)| as Eq. 2 defines L: the communities of N(v)
 *            other than C(u) = C_i, i.e. L_all - [f_i > 0] (not Algorithm 2's
 *            L_all - 1 for every column);
 * flags & 2: Algorithm 1's gate: omega_v(C_i) = 0 unless |L| > 1.
 * Entropy exactly as oracle_weights (Eq. 3, direct sum). */
void oracle_weights_variant(int64_t n, int32_t k, const int32_t *f_all, int32_t flags, double *omega_out) {
    for (int64_t v = 0; v < n; v++) {
        const int32_t *f = f_all + v * k;
        double *w = omega_out + v * k;
        int64_t T = 0; int32_t L_all = 0;
        for (int32_t j = 0; j < k; j++) { T += f[j]; if (f[j] > 0) L_all++; }
        for (int32_t i = 0; i < k; i++) {
            const int32_t L = (flags & 1) ? L_all - (f[i] > 0) : L_all - 1;
            double H = 0.0;
            const double Y = (double)(T - f[i]);
            if (Y > 0.0)
                for (int32_t j = 0; j < k; j++) {
                    if (j == i || f[j] == 0) continue;
                    double p = (double)f[j] / Y;
                    H -= p * log2(p);
                }
            w[i] = ((flags & 2) && L <= 1) || L <= 0 ? 0.0 : H * (double)L;
            if (w[i] == 0.0) w[i] = 0.0;   /* canonical +0 */
        }
    }
}

/* omega_max over Algorithm 1's E_b only ("max edge weight in E_b"):
 * the pairs (u, v) of border vertices with C(u) = C(v) or v in N(u)
 * whose |L(u,v)| > 1 (|L| per flags & 1 as above) give the edge
 * (v -> u) of weight omega_v(C(u)). For v in V_b and target column i
 * such a u exists iff C_i = C(v) (u = v; the loop includes it) or v has a
 * neighbour in C_i (that neighbour is a border vertex). */
double oracle_omega_max_eb(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C, int32_t k,
                           const int32_t *targets, const int32_t *f_all, int32_t flags, const double *omega) {
    double m = 0.0;
    for (int64_t v = 0; v < n; v++) {
        int border = 0;
        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) if (C[col[e]] != C[v]) { border = 1; break; }
        if (!border) continue;
        const int32_t *f = f_all + v * k;
        int32_t L_all = 0;
        for (int32_t j = 0; j < k; j++) if (f[j] > 0) L_all++;
        for (int32_t i = 0; i < k; i++) {
            const int32_t L = (flags & 1) ? L_all - (f[i] > 0) : L_all - 1;
            if (L <= 1) continue;
            if (targets[i] != C[v] && f[i] == 0) continue;
            if (omega[v * k + i] > m) m = omega[v * k + i];
        }
    }
    return m;
}

/* ---- O5a. G' predecessor lists ((v->u) in E_b iff (u,v) in E, both
 * border and C(u) != C(v); adjacency + different communities already makes
 * both endpoints border vertices). pred_off is n+1; pred_out receives the
 * lists (ascending) when non-NULL. Returns the number of entries. ---- */
int64_t oracle_pred(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C,
                    int64_t *pred_off, int32_t *pred_out) {
    int64_t cnt = 0;
    for (int64_t u = 0; u < n; u++) {
        pred_off[u] = cnt;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++)
            if (C[col[e]] != C[u]) { if (pred_out) pred_out[cnt] = col[e]; cnt++; }
    }
    pred_off[n] = cnt;
    return cnt;
}

/* ---- exact fixed-point helpers (C-12) ---- */
typedef __int128 i128;

/* round-half-even(t * 2^80) for finite t >= 0, from the fp64 bits. */
static i128 quantize80(double t) {
    if (t == 0.0) return 0;
    int ex;
    double mant = frexp(t, &ex);                  /* t = mant * 2^ex, mant in [0.5,1) */
    int64_t m = (int64_t)ldexp(mant, 53);         /* exact 53-bit integer             */
    int shift = ex - 53 + 80;                     /* t * 2^80 = m * 2^shift           */
    if (shift >= 0) return (i128)m << shift;
    int s = -shift;
    if (s >= 64) return 0;                        /* m < 2^53 <= half ulp of 2^s    */
    int64_t q = m >> s;
    int64_t rem = m & (((int64_t)1 << s) - 1);
    int64_t half = (int64_t)1 << (s - 1);
    if (rem > half || (rem == half && (q & 1))) q++;
    return q;
}
static double from_fixed80(i128 s) { return ldexp((double)s, -80); }

/* ---- O5-O7. RSI (Eq.4) over valid triads (Eq.6, P:163-171;
 * Type-I / Type-II), one head at a time.
 *
 * For head u with col(u) != ⊥ and d(u) >= 2 (C-9, C-22), enumerate ordered
 * (w, v): w in N(u), C(w) != C(u); v in N(w), v != u, C(v) != C(w); and
 *   Type-II  if C(v) == C(u)                                (C-10, C-21)
 *   Type-I   else if v in N(u) and col(v) != ⊥               (C-9)
 * Each valid triad adds t = ( omega_v(C(u))/wmax * omega_w(C(v))/wmax *
 * omega_w(C(u))/wmax )^(1/3) (Eq.4 and Algorithm 1 line P:286; factor order
 * pinned by the worked example P:506). Terms with a zero factor
 * are 0 but the triad is still counted. R(u) = sum / (d(u)(d(u)-1)) with d the
 * degree in G (C-16). If wmax <= 0 every score is +0.0.
 *
 * heads: list of nh vertex ids to score (all vertices for a full run);
 * R_out / nI_out / nII_out are indexed like heads. ---- */
void oracle_rsi(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C,
                int32_t k, const int32_t *targets, const double *omega, double wmax,
                int64_t nh, const int64_t *heads, double *R_out, int64_t *nI_out, int64_t *nII_out) {
    int32_t *cols = malloc(sizeof(int32_t) * (n ? n : 1));
    for (int64_t x = 0; x < n; x++) cols[x] = column_of(C[x], k, targets);
    int64_t *mark = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t x = 0; x < n; x++) mark[x] = -1;

    for (int64_t h = 0; h < nh; h++) {
        int64_t u = heads[h];
        int64_t d = rowptr[u + 1] - rowptr[u];
        int32_t cu = cols[u];
        R_out[h] = 0.0; nI_out[h] = 0; nII_out[h] = 0;
        if (cu < 0 || d < 2) continue;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) mark[col[e]] = u;
        i128 S = 0;
        int64_t nI = 0, nII = 0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
            int32_t w = col[e];
            if (C[w] == C[u]) continue;
            for (int64_t e2 = rowptr[w]; e2 < rowptr[w + 1]; e2++) {
                int32_t v = col[e2];
                if (v == u || C[v] == C[w]) continue;
                int32_t cv;
                if (C[v] == C[u]) { cv = cu; nII++; }
                else if (mark[v] == u && cols[v] >= 0) { cv = cols[v]; nI++; }
                else continue;
                double f1 = omega[(int64_t)v * k + cu];   /* omega_v(u) = omega_v(C(u)) */
                double f2 = omega[(int64_t)w * k + cv];   /* omega_w(v) = omega_w(C(v)) */
                double f3 = omega[(int64_t)w * k + cu];   /* omega_w(u) = omega_w(C(u)) */
                if (wmax <= 0.0 || f1 == 0.0 || f2 == 0.0 || f3 == 0.0) continue;
                double t = cbrt((f1 / wmax) * (f2 / wmax) * (f3 / wmax));
                S += quantize80(t);
            }
        }
        nI_out[h] = nI; nII_out[h] = nII;
        R_out[h] = wmax > 0.0 ? from_fixed80(S) / ((double)d * (double)(d - 1)) : 0.0;
    }
    free(cols); free(mark);
}

/* ---- NEXT-2: every community a target (DESIGN reading C-32).
 * Exactly O2-O4 and O5-O7 above with targets = all k distinct communities
 * (column i = targets[i], oracle_select_targets order), except that each row of
 * the n*k histogram is kept as its nonzero columns only -- a dense table is
 * O(n * #communities). A column with f = 0 is still a cell: Eq.3 with Y = T
 * (the whole row's entropy) times (L_all - 1), the same for every absent
 * column of the row (omega_abs_out[u]); omega_max runs over all n*k cells
 * (C-7), i.e. the present cells and, when L_all < k, the absent one. The
 * present weights sum j ascending over the nonzero columns, the same order as
 * oracle_weights, so both give identical bits.
 * Outputs (caller-allocated, nnz = rowptr[n] entries suffice): off_out[n+1],
 * cols_out / cnt_out / omega_out per (vertex, nonzero column), ascending
 * columns. Returns the number of entries. ---- */
int64_t oracle_tables_all(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C, int32_t k,
                          const int32_t *targets, int64_t *off_out, int32_t *cols_out, int32_t *cnt_out,
                          double *omega_out, double *omega_abs_out, double *wmax_out) {
    int32_t cmax = 0;
    for (int32_t i = 0; i < k; i++) if (targets[i] > cmax) cmax = targets[i];
    int32_t *colmap = malloc(sizeof(int32_t) * ((size_t)cmax + 1));
    for (int32_t i = 0; i < k; i++) colmap[targets[i]] = i;
    int64_t dmax = 0;
    for (int64_t u = 0; u < n; u++) if (rowptr[u + 1] - rowptr[u] > dmax) dmax = rowptr[u + 1] - rowptr[u];
    int32_t *tmp = malloc(sizeof(int32_t) * (dmax ? dmax : 1));
    double wmax = 0.0;
    int64_t at = 0;
    for (int64_t u = 0; u < n; u++) {
        const int64_t d = rowptr[u + 1] - rowptr[u];
        off_out[u] = at;
        for (int64_t e = 0; e < d; e++) tmp[e] = colmap[C[col[rowptr[u] + e]]];
        qsort(tmp, (size_t)d, sizeof(int32_t), cmp_i32);
        const int64_t b = at;
        for (int64_t e = 0; e < d; e++) {                 /* nonzero columns, ascending */
            if (e == 0 || tmp[e] != tmp[e - 1]) { cols_out[at] = tmp[e]; cnt_out[at] = 0; at++; }
            cnt_out[at - 1]++;
        }
        const int32_t L_all = (int32_t)(at - b);
        const double T = (double)d;                        /* every neighbour is in a target */
        for (int64_t i = b; i < at; i++) {                 /* Eq.3 / Eq.5 for a present column */
            if (L_all <= 1) { omega_out[i] = 0.0; continue; }
            const double Y = T - (double)cnt_out[i];
            double H = 0.0;
            for (int64_t j = b; j < at; j++) {
                if (j == i) continue;
                const double p = (double)cnt_out[j] / Y;
                H -= p * log2(p);
            }
            omega_out[i] = H * (double)(L_all - 1);
            if (omega_out[i] > wmax) wmax = omega_out[i];
        }
        double wabs = 0.0;                                 /* every absent column: Y = T */
        if (L_all > 1) {
            double H = 0.0;
            for (int64_t j = b; j < at; j++) {
                const double p = (double)cnt_out[j] / T;
                H -= p * log2(p);
            }
            wabs = H * (double)(L_all - 1);
        }
        omega_abs_out[u] = wabs;
        if (L_all < k && wabs > wmax) wmax = wabs;
    }
    off_out[n] = at;
    *wmax_out = wmax;
    free(tmp);
    free(colmap);
    return at;
}

/* omega_v(c) from the row tables of oracle_tables_all */
static double omega_all(const int64_t *off, const int32_t *cols, const double *omega, const double *omega_abs,
                        int64_t v, int32_t c) {
    int64_t lo = off[v], hi = off[v + 1];
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (cols[mid] < c) lo = mid + 1; else hi = mid;
    }
    return (lo < off[v + 1] && cols[lo] == c) ? omega[lo] : omega_abs[v];
}

/* O5-O7 with targets = all (every col(x) defined), weights from the row tables:
 * the same enumeration, factors and exact sum as oracle_rsi. */
void oracle_rsi_all(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C, int32_t k,
                    const int32_t *targets, const int64_t *off, const int32_t *cols, const double *omega,
                    const double *omega_abs, double wmax, int64_t nh, const int64_t *heads, double *R_out,
                    int64_t *nI_out, int64_t *nII_out) {
    int32_t cmax = 0;
    for (int32_t i = 0; i < k; i++) if (targets[i] > cmax) cmax = targets[i];
    int32_t *colmap = malloc(sizeof(int32_t) * ((size_t)cmax + 1));
    for (int32_t i = 0; i < k; i++) colmap[targets[i]] = i;
    int64_t *mark = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t x = 0; x < n; x++) mark[x] = -1;
    for (int64_t h = 0; h < nh; h++) {
        const int64_t u = heads[h];
        const int64_t d = rowptr[u + 1] - rowptr[u];
        const int32_t cu = colmap[C[u]];
        R_out[h] = 0.0; nI_out[h] = 0; nII_out[h] = 0;
        if (d < 2) continue;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) mark[col[e]] = u;
        i128 S = 0;
        int64_t nI = 0, nII = 0;
        for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
            const int32_t w = col[e];
            if (C[w] == C[u]) continue;
            for (int64_t e2 = rowptr[w]; e2 < rowptr[w + 1]; e2++) {
                const int32_t v = col[e2];
                if (v == u || C[v] == C[w]) continue;
                int32_t cv;
                if (C[v] == C[u]) { cv = cu; nII++; }
                else if (mark[v] == u) { cv = colmap[C[v]]; nI++; }
                else continue;
                const double f1 = omega_all(off, cols, omega, omega_abs, v, cu);
                const double f2 = omega_all(off, cols, omega, omega_abs, w, cv);
                const double f3 = omega_all(off, cols, omega, omega_abs, w, cu);
                if (wmax <= 0.0 || f1 == 0.0 || f2 == 0.0 || f3 == 0.0) continue;
                const double t = cbrt((f1 / wmax) * (f2 / wmax) * (f3 / wmax));
                S += quantize80(t);
            }
        }
        nI_out[h] = nI; nII_out[h] = nII;
        R_out[h] = wmax > 0.0 ? from_fixed80(S) / ((double)d * (double)(d - 1)) : 0.0;
    }
    free(colmap);
    free(mark);
}

/* ---- O8. Top-K (Algorithm 1 optional Step 4): the K highest R,
 * ties by ascending vertex id (C-14: zeros eligible, K clamped to n). ---- */
typedef struct { double r; int32_t id; } scored;
static int cmp_scored(const void *a, const void *b) {
    const scored *x = a, *y = b;
    if (x->r != y->r) return x->r > y->r ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}
int64_t oracle_topk(int64_t n, const double *R, int64_t K, int32_t *ids_out, double *scores_out) {
    scored *s = malloc(sizeof(scored) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) { s[i].r = R[i]; s[i].id = (int32_t)i; }
    qsort(s, (size_t)n, sizeof(scored), cmp_scored);
    int64_t cnt = K < n ? K : n;
    for (int64_t i = 0; i < cnt; i++) { ids_out[i] = s[i].id; scores_out[i] = s[i].r; }
    free(s);
    return cnt;
}

/* ---- NEXT-1: absolute AWCC under cumulative random removal (PAPER §VII.B,
 * P:667-676; SPEC awcc / absolute_awcc / simulate_removal).
 *
 * AWCC(S) = (1/|S|) sum_{v in S} |zeta(v)| / d(v), zeta(v) = the community ids
 * of v's neighbours. The absolute variant recomputes zeta over the
 * surviving edges/vertices while d(v) stays the original degree; a
 * removed v in S contributes 0, as does d(v) = 0.
 *
 * Removal (DESIGN readings C-28/C-29): "random removal of 5% of the
 * edges/nodes at each iteration ... until up to 75%" is cumulative
 * within a trial: every item (undirected edge {u, v} with id
 * min(u,v) << 32 | max(u,v), or vertex v) of trial t gets the key
 * mix64(s_t ^ id), mix64 = the splitmix64 finaliser (a bijection on 64-bit
 * words, so keys are distinct), s_t = mix64(seed + (2t + mode) * 0x9E3779B97F4A7C15)
 * for mode 0 = edges, 1 = nodes; step j removes the r_j = floor(j * step% * M / 100)
 * items of smallest key (M = |E| or |V|), i.e. those with key < T_j, T_j the key
 * of rank r_j (all items when r_j = M). Ids are the caller's (original) ids.
 * Here: all keys, one qsort, then zeta by scanning each v's row; the j-th
 * per-trial value sums |zeta|/d(v) in S order and divides by |S|, the mean sums
 * the trial values in trial order and divides by the trial count. ---- */
uint64_t oracle_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* returns J + 1 (steps 0..J), or -1 on bad arguments */
int64_t oracle_awcc_removal(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C,
                            const int32_t *S, int64_t nS, int32_t mode, int32_t step_pct, int32_t max_pct,
                            int32_t trials, uint64_t seed, int32_t *zeta_out, double *mean_out) {
    if (nS < 1 || step_pct < 1 || max_pct < 0 || max_pct > 100 || trials < 1 || (mode != 0 && mode != 1)) return -1;
    const int64_t J = max_pct / step_pct;
    const int64_t m = rowptr[n] / 2;
    const int64_t M = mode == 0 ? m : n;
    uint64_t *keys = malloc(sizeof(uint64_t) * (M ? M : 1));
    uint64_t *T = malloc(sizeof(uint64_t) * (J + 1));
    int *all = malloc(sizeof(int) * (J + 1));
    int64_t dmax = 1;
    for (int64_t s = 0; s < nS; s++) {
        const int64_t d = rowptr[S[s] + 1] - rowptr[S[s]];
        if (d > dmax) dmax = d;
    }
    int32_t *cbuf = malloc(sizeof(int32_t) * dmax);
    for (int64_t j = 0; j <= J; j++) mean_out[j] = 0.0;
    for (int32_t t = 0; t < trials; t++) {
        const uint64_t st = oracle_mix64(seed + (uint64_t)(2 * (int64_t)t + mode) * 0x9E3779B97F4A7C15ull);
        /* keys of every item */
        int64_t q = 0;
        if (mode == 0) {
            for (int64_t u = 0; u < n; u++)
                for (int64_t e = rowptr[u]; e < rowptr[u + 1]; e++)
                    if ((int64_t)col[e] > u) keys[q++] = oracle_mix64(st ^ (((uint64_t)u << 32) | (uint64_t)col[e]));
        } else {
            for (int64_t v = 0; v < n; v++) keys[q++] = oracle_mix64(st ^ (uint64_t)v);
        }
        qsort(keys, (size_t)M, sizeof(uint64_t), cmp_u64);
        for (int64_t j = 0; j <= J; j++) {
            const int64_t r = (j * step_pct * M) / 100;
            all[j] = r >= M;
            T[j] = r >= M ? 0 : keys[r];
        }
        for (int64_t j = 0; j <= J; j++) {
            double acc = 0.0;
            for (int64_t s = 0; s < nS; s++) {
                const int64_t v = S[s];
                const int64_t d = rowptr[v + 1] - rowptr[v];
                int64_t z = 0;
                int v_removed = 0;
                if (mode == 1) v_removed = all[j] || oracle_mix64(st ^ (uint64_t)v) < T[j];
                if (!v_removed) {
                    int64_t nb = 0;   /* communities of the surviving neighbours, then distinct count */
                    for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) {
                        const int64_t x = col[e];
                        int removed;
                        if (mode == 0) {
                            const uint64_t id = ((uint64_t)(v < x ? v : x) << 32) | (uint64_t)(v < x ? x : v);
                            removed = all[j] || oracle_mix64(st ^ id) < T[j];
                        } else {
                            removed = all[j] || oracle_mix64(st ^ (uint64_t)x) < T[j];
                        }
                        if (removed) continue;
                        cbuf[nb++] = C[x];
                    }
                    qsort(cbuf, (size_t)nb, sizeof(int32_t), cmp_i32);
                    for (int64_t i = 0; i < nb; i++) z += (i == 0 || cbuf[i] != cbuf[i - 1]);
                }
                zeta_out[((int64_t)t * (J + 1) + j) * nS + s] = (int32_t)z;
                if (d > 0) acc += (double)z / (double)d;
            }
            mean_out[j] += acc / (double)nS;
        }
    }
    for (int64_t j = 0; j <= J; j++) mean_out[j] /= (double)trials;
    free(keys); free(T); free(all); free(cbuf);
    return J + 1;
}

/* ---- NEXT-4: structural hole influence index (PAPER §VII.A, P:602-605;
 * SPEC diffuse / shii; DESIGN reading C-31).
 * SHII(u_s) = (influenced outside C(u_s)) / (influenced), averaged over runs.
 * Run r of model m (0 = IC, 1 = LT) draws from s_r = mix64(seed + (2r + m + 1)
 * * 0xD1B54A32D192ED03):
 *  IC (independent cascade with probability p): each newly active a gets one
 *     chance per inactive neighbour b, succeeding iff mix64(s_r ^ (a << 32 | b))
 *     < thr, thr = floor(p * 2^64) (every edge when p >= 1). The outcome is the
 *     set reachable from the seed over those "live" directed edges (the coin of
 *     a -> b is drawn once, whenever a is active), computed here by a queue.
 *  LT (linear threshold): theta_v = mix64(s_r ^ v) / 2^64; an inactive v
 *     activates once (active neighbours) / d(v) >= theta_v with at least one
 *     active neighbour; iterated over all vertices to the fixpoint.
 * The seed is always influenced. Per seed: out[(s * runs + r) * 2 + {0, 1}] =
 * {influenced, influenced outside C(seed)}; shii_out[s] = the mean over runs of
 * their ratio (summed in run order); returns the mean of shii_out over S. ---- */
static int lt_ready(uint64_t key, int64_t d, int64_t act) {
    /* act / d >= key / 2^64  <=>  act * 2^64 >= key * d, exactly (act >= 1) */
    if (act < 1) return 0;
    const unsigned __int128 lhs = (unsigned __int128)(uint64_t)act << 64;
    const unsigned __int128 rhs = (unsigned __int128)key * (uint64_t)d;
    return lhs >= rhs;
}

double oracle_shii(int64_t n, const int64_t *rowptr, const int32_t *col, const int32_t *C, const int32_t *S,
                   int64_t nS, int32_t model, double p, int32_t runs, uint64_t seed, int64_t *out,
                   double *shii_out) {
    unsigned char *act = malloc(n ? n : 1);
    int32_t *queue = malloc(sizeof(int32_t) * (n ? n : 1));
    const int all_live = p >= 1.0;
    const uint64_t thr = all_live ? 0 : (uint64_t)ldexp(p, 64);
    double setmean = 0.0;
    for (int64_t s = 0; s < nS; s++) {
        const int32_t u0 = S[s];
        double acc = 0.0;
        for (int32_t r = 0; r < runs; r++) {
            const uint64_t sr = oracle_mix64(seed + (uint64_t)(2 * (int64_t)r + model + 1) * 0xD1B54A32D192ED03ull);
            memset(act, 0, n);
            act[u0] = 1;
            if (model == 0) {
                int64_t qh = 0, qt = 0;
                queue[qt++] = u0;
                while (qh < qt) {
                    const int64_t a = queue[qh++];
                    for (int64_t e = rowptr[a]; e < rowptr[a + 1]; e++) {
                        const int64_t b = col[e];
                        if (act[b]) continue;
                        const uint64_t key = oracle_mix64(sr ^ (((uint64_t)a << 32) | (uint64_t)b));
                        if (all_live || key < thr) { act[b] = 1; queue[qt++] = (int32_t)b; }
                    }
                }
            } else {
                int changed = 1;
                while (changed) {
                    changed = 0;
                    for (int64_t v = 0; v < n; v++) {
                        if (act[v]) continue;
                        int64_t a = 0;
                        for (int64_t e = rowptr[v]; e < rowptr[v + 1]; e++) a += act[col[e]];
                        if (lt_ready(oracle_mix64(sr ^ (uint64_t)v), rowptr[v + 1] - rowptr[v], a)) {
                            act[v] = 1;
                            changed = 1;
                        }
                    }
                }
            }
            int64_t inf = 0, outc = 0;
            for (int64_t v = 0; v < n; v++)
                if (act[v]) { inf++; if (C[v] != C[u0]) outc++; }
            out[(s * runs + r) * 2] = inf;
            out[(s * runs + r) * 2 + 1] = outc;
            acc += (double)outc / (double)inf;
        }
        shii_out[s] = acc / (double)runs;
        setmean += shii_out[s];
    }
    free(act); free(queue);
    return setmean / (double)nS;
}
