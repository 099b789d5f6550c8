/*
 * hs_oracle.c -- CPU restatement of the hetsched hot path (parity oracle).
 *
 * TEST INFRASTRUCTURE ONLY (see hs_oracle.h).  Every function names the
 * reference lines it restates; paths are relative to
 * /root/reference/pkg/src/hetsched/.
 *
 * Float-order contracts (pinned in tests/test_oracle_golden.py):
 *   - contiguous numpy reductions (`x.sum()`, `m.sum(axis=1)` of an np.ix_
 *     gather, `np.mean(list)`) use numpy's pairwise sum (pw_sum below);
 *   - `w[:, grp].mean(axis=1)` (scheduler.py:283,363) reduces an
 *     F-contiguous fancy-index result and therefore sums SEQUENTIALLY
 *     (seq_sum), then divides by the count;
 *   - `np.cumsum` is sequential.
 * Build with -ffp-contract=off; no fast-math.
 */
#include "hs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define MAX_EXACT_TSP 16

struct orc_inst {
    int n, k, m;
    double *dp, *pp, *sw;
};

/* ------------------------------------------------------------------ */
/* numpy float-order contracts                                          */

/* numpy pairwise_sum (loops_utils.h.src); used by every contiguous reduce */
static double pw_sum(const double *a, long n) {
    if (n < 8) {
        double r = 0.0;
        for (long i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

static double seq_sum(const double *a, long n) {
    double r = 0.0;
    for (long i = 0; i < n; i++) r += a[i];
    return r;
}

/* ------------------------------------------------------------------ */
/* instance tables: costmodel.py:134-141, scheduler.py:84-88            */

orc_inst *orc_create(int n, const double *lat, const double *bw, int d_pp, int d_dp,
                     double dp_num, double pp_num, double sw_num) {
    orc_inst *in = (orc_inst *)calloc(1, sizeof(orc_inst));
    in->n = n;
    in->k = d_pp;
    in->m = d_dp;
    size_t nn = (size_t)n * n;
    in->dp = (double *)malloc(nn * sizeof(double));
    in->pp = (double *)malloc(nn * sizeof(double));
    in->sw = (double *)malloc(nn * sizeof(double));
    double ddp = (double)d_dp;
    for (int i = 0; i < n; i++) {
        for (int j = 0; j < n; j++) {
            size_t x = (size_t)i * n + j;
            double l = lat[x], b = bw[x];
            /* dp_pair_seconds: 2.0 * (lat + (8.0*c_dp) / (d_dp*bw)); diagonal
             * zeroed by np.fill_diagonal in datap_cost_group (:167) */
            in->dp[x] = (i == j) ? 0.0 : 2.0 * (l + dp_num / (ddp * b));
            /* pp_edge_seconds: 2.0 * (lat + (8.0*c_pp) / bw) */
            in->pp[x] = 2.0 * (l + pp_num / b);
            /* SurrogateWeights.from_instance: lat + 8.0*(c_pp+c_dp)/bw, 0 diag */
            in->sw[x] = (i == j) ? 0.0 : l + sw_num / b;
        }
    }
    return in;
}

void orc_destroy(orc_inst *in) {
    if (!in) return;
    free(in->dp);
    free(in->pp);
    free(in->sw);
    free(in);
}

void orc_tables(const orc_inst *in, double *dp, double *pp, double *sw) {
    size_t nn = (size_t)in->n * in->n * sizeof(double);
    if (dp) memcpy(dp, in->dp, nn);
    if (pp) memcpy(pp, in->pp, nn);
    if (sw) memcpy(sw, in->sw, nn);
}

/* ------------------------------------------------------------------ */
/* data-parallel level: costmodel.py:154-175                             */

double orc_datap_group(const orc_inst *in, const int32_t *mem, int cnt) {
    if (cnt == 1) return 0.0;
    double row[1024];
    double worst = -INFINITY;
    for (int r = 0; r < cnt; r++) {
        const double *dr = in->dp + (size_t)mem[r] * in->n;
        for (int c = 0; c < cnt; c++) row[c] = (r == c) ? 0.0 : dr[mem[c]];
        double s = pw_sum(row, cnt); /* m.sum(axis=1) of the ix_ gather */
        if (s > worst || r == 0) worst = s;
    }
    return worst;
}

/* ------------------------------------------------------------------ */
/* bottleneck matching: combinatorics.py:86-131,147-189                   */

typedef struct {
    int m;
    int adj[64][64];
    int deg[64];
} adjlist;

static void build_adj(adjlist *A, const double *w, int m, double thr) {
    A->m = m;
    for (int r = 0; r < m; r++) {
        A->deg[r] = 0;
        for (int c = 0; c < m; c++)
            if (w[r * m + c] <= thr) A->adj[r][A->deg[r]++] = c;
    }
}

/* _augment (:86-94) */
static int augment(int row, const adjlist *A, int *match_col, int *seen) {
    for (int t = 0; t < A->deg[row]; t++) {
        int col = A->adj[row][t];
        if (!seen[col]) {
            seen[col] = 1;
            if (match_col[col] < 0 || augment(match_col[col], A, match_col, seen)) {
                match_col[col] = row;
                return 1;
            }
        }
    }
    return 0;
}

/* _perfect_matching (:97-103) */
static int perfect_matching(const adjlist *A, int *match_col) {
    int m = A->m;
    for (int c = 0; c < m; c++) match_col[c] = -1;
    for (int row = 0; row < m; row++) {
        int seen[64] = {0};
        if (!augment(row, A, match_col, seen)) return 0;
    }
    return 1;
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* _optimal_threshold (:106-125): binary search over np.unique(w) */
static double optimal_threshold(const double *w, int m) {
    int mm = m * m;
    double vals[4096];
    memcpy(vals, w, (size_t)mm * sizeof(double));
    qsort(vals, mm, sizeof(double), cmp_double);
    int u = 0;
    for (int i = 0; i < mm; i++)
        if (u == 0 || vals[i] != vals[u - 1]) vals[u++] = vals[i];
    int lo = 0, hi = u - 1;
    adjlist *A = (adjlist *)malloc(sizeof(adjlist));
    int match_col[64];
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        build_adj(A, w, m, vals[mid]);
        if (perfect_matching(A, match_col))
            hi = mid;
        else
            lo = mid + 1;
    }
    free(A);
    return vals[lo];
}

double orc_bottleneck_value(const double *w, int m) { return optimal_threshold(w, m); }

/* bottleneck_perfect_matching (:134-144) + _lex_smallest_pairing (:147-189) */
int orc_bottleneck_matching(const double *w, int m, int32_t *pairs, double *value) {
    double b = optimal_threshold(w, m);
    adjlist *A = (adjlist *)malloc(sizeof(adjlist));
    build_adj(A, w, m, b);
    int match_col[64], match_row[64], fixed[64] = {0};
    if (!perfect_matching(A, match_col)) {
        free(A);
        return -1;
    }
    for (int c = 0; c < m; c++) match_row[match_col[c]] = c;
    for (int row = 0; row < m; row++) {
        int chosen = -1;
        for (int t = 0; t < A->deg[row]; t++) {
            int col = A->adj[row][t];
            if (fixed[col]) continue;
            if (match_row[row] == col) {
                chosen = col;
                break;
            }
            int displaced = match_col[col];
            int old_col = match_row[row];
            match_col[col] = row;
            match_col[old_col] = -1;
            int seen[64] = {0};
            seen[col] = 1;
            for (int fc = 0; fc < m; fc++)
                if (fixed[fc]) seen[fc] = 1;
            if (augment(displaced, A, match_col, seen)) {
                chosen = col;
                for (int r2 = 0; r2 < m; r2++) match_row[r2] = -1;
                for (int c2 = 0; c2 < m; c2++)
                    if (match_col[c2] >= 0) match_row[match_col[c2]] = c2;
                break;
            }
            match_col[old_col] = row;
            match_col[col] = displaced;
        }
        if (chosen < 0) {
            free(A);
            return -1;
        }
        pairs[row] = chosen;
        fixed[chosen] = 1;
    }
    free(A);
    *value = b;
    return 0;
}

/* ------------------------------------------------------------------ */
/* open-loop TSP: combinatorics.py:68-79,232-342                         */

double orc_path_cost(const double *w, int k, const int32_t *order, int len) {
    double total = 0.0;
    for (int i = len - 2; i >= 0; i--) total = w[order[i] * k + order[i + 1]] + total;
    return total;
}

/* _held_karp (:253-296).  h[s][u] = cheapest path starting at u covering s */
int orc_open_loop_tsp(const double *w, int k, double *total_out, int32_t *order) {
    if (k == 1) {
        *total_out = 0.0;
        if (order) order[0] = 0;
        return 0;
    }
    if (k > MAX_EXACT_TSP) return -1;
    int full = (1 << k) - 1;
    double *h = (double *)malloc(sizeof(double) * (size_t)(full + 1) * k);
    for (long i = 0; i < (long)(full + 1) * k; i++) h[i] = INFINITY;
    for (int u = 0; u < k; u++) h[(size_t)(1 << u) * k + u] = 0.0;
    for (int s = 3; s <= full; s++) {
        if ((s & (s - 1)) == 0) continue;
        for (int u = 0; u < k; u++) {
            if (!(s >> u & 1)) continue;
            int r = s ^ (1 << u);
            double best = INFINITY;
            for (int v = 0; v < k; v++) {
                if (!(r >> v & 1)) continue;
                double c = w[u * k + v] + h[(size_t)r * k + v];
                if (c < best) best = c;
            }
            h[(size_t)s * k + u] = best;
        }
    }
    const double *hf = h + (size_t)full * k;
    double total = hf[0];
    for (int u = 1; u < k; u++)
        if (hf[u] < total) total = hf[u];
    int start = 0;
    while (hf[start] != total) start++;
    if (order) {
        int n = 0, cur = start, s = full ^ (1 << start);
        double target = total;
        order[n++] = start;
        while (s) {
            int found = 0;
            for (int u = 0; u < k; u++) {
                if (!(s >> u & 1)) continue;
                if (w[cur * k + u] + h[(size_t)s * k + u] == target) {
                    order[n++] = u;
                    target = h[(size_t)s * k + u];
                    cur = u;
                    s ^= 1 << u;
                    found = 1;
                    break;
                }
            }
            if (!found) {
                free(h);
                return -2;
            }
        }
    }
    free(h);
    *total_out = total;
    return 0;
}

/* _nn_two_opt (:299-319) and _two_opt (:322-342) */
static void two_opt(const double *w, int k, int32_t *o) {
    int improved = 1;
    while (improved) {
        improved = 0;
        for (int i = 0; i < k - 1; i++) {
            for (int j = i + 1; j < k; j++) {
                double before = 0.0, after = 0.0;
                if (i > 0) {
                    before += w[o[i - 1] * k + o[i]];
                    after += w[o[i - 1] * k + o[j]];
                }
                if (j < k - 1) {
                    before += w[o[j] * k + o[j + 1]];
                    after += w[o[i] * k + o[j + 1]];
                }
                if (after < before) {
                    for (int a = i, b = j; a < b; a++, b--) {
                        int32_t t = o[a];
                        o[a] = o[b];
                        o[b] = t;
                    }
                    improved = 1;
                }
            }
        }
    }
}

int orc_open_loop_tsp_heuristic(const double *w, int k, double *total_out, int32_t *order) {
    if (k == 1) {
        *total_out = 0.0;
        order[0] = 0;
        return 0;
    }
    if (k <= MAX_EXACT_TSP) return orc_open_loop_tsp(w, k, total_out, order);
    int32_t *o = (int32_t *)malloc(sizeof(int32_t) * k);
    int32_t *best = (int32_t *)malloc(sizeof(int32_t) * k);
    char *left = (char *)malloc(k);
    double best_total = INFINITY;
    int have = 0;
    for (int start = 0; start < k; start++) {
        memset(left, 1, k);
        left[start] = 0;
        o[0] = start;
        for (int t = 1; t < k; t++) {
            int cur = o[t - 1], nxt = -1;
            for (int v = 0; v < k; v++) {
                if (!left[v]) continue;
                if (nxt < 0 || w[cur * k + v] < w[cur * k + nxt]) nxt = v;
            }
            o[t] = nxt;
            left[nxt] = 0;
        }
        two_opt(w, k, o);
        double tot = orc_path_cost(w, k, o, k);
        if (tot < best_total) {
            best_total = tot;
            memcpy(best, o, sizeof(int32_t) * k);
            have = 1;
        }
    }
    (void)have;
    if (best[0] > best[k - 1])
        for (int a = 0, b = k - 1; a < b; a++, b--) {
            int32_t t = best[a];
            best[a] = best[b];
            best[b] = t;
        }
    memcpy(order, best, sizeof(int32_t) * k);
    *total_out = orc_path_cost(w, k, best, k);
    free(o);
    free(best);
    free(left);
    return 0;
}

/* ------------------------------------------------------------------ */
/* comm_cost: costmodel.py:200-229                                       */

static void coarse_edges(const orc_inst *in, const int32_t *groups, double *E) {
    int k = in->k, m = in->m, n = in->n;
    double sub[4096];
    for (int j = 0; j < k; j++) E[j * k + j] = 0.0;
    for (int j = 0; j < k; j++) {
        for (int j2 = j + 1; j2 < k; j2++) {
            const int32_t *a = groups + j * m, *b = groups + j2 * m;
            for (int r = 0; r < m; r++)
                for (int c = 0; c < m; c++) sub[r * m + c] = in->pp[(size_t)a[r] * n + b[c]];
            double v = optimal_threshold(sub, m);
            E[j * k + j2] = E[j2 * k + j] = v;
        }
    }
}

int orc_comm_cost(const orc_inst *in, const int32_t *groups, double *out3, double *per_group,
                  int32_t *order) {
    int k = in->k, m = in->m;
    double pg[256];
    double datap = 0.0;
    for (int j = 0; j < k; j++) {
        pg[j] = orc_datap_group(in, groups + j * m, m);
        if (j == 0 || pg[j] > datap) datap = pg[j]; /* max(per_group) */
    }
    double *E = (double *)malloc(sizeof(double) * k * k);
    coarse_edges(in, groups, E);
    double pipe;
    int32_t ord[256];
    int rc = orc_open_loop_tsp(E, k, &pipe, ord);
    free(E);
    if (rc) return rc;
    out3[0] = datap + pipe;
    out3[1] = datap;
    out3[2] = pipe;
    if (per_group) memcpy(per_group, pg, sizeof(double) * k);
    if (order) memcpy(order, ord, sizeof(int32_t) * k);
    return 0;
}

/* comm_cost(..., heuristic=True) (costmodel.py:217-229): exact Held-Karp up
 * to 16 stages, nearest neighbour + 2-opt beyond (combinatorics.py:243-249) */
int orc_comm_cost_heuristic(const orc_inst *in, const int32_t *groups, double *out3, int32_t *order) {
    int k = in->k, m = in->m;
    if (k <= MAX_EXACT_TSP) return orc_comm_cost(in, groups, out3, NULL, order);
    double datap = 0.0;
    for (int j = 0; j < k; j++) {
        double v = orc_datap_group(in, groups + j * m, m);
        if (j == 0 || v > datap) datap = v;
    }
    double *E = (double *)malloc(sizeof(double) * k * k);
    coarse_edges(in, groups, E);
    double pipe;
    int32_t ord[256];
    orc_open_loop_tsp_heuristic(E, k, &pipe, ord);
    free(E);
    out3[0] = datap + pipe;
    out3[1] = datap;
    out3[2] = pipe;
    if (order) memcpy(order, ord, sizeof(int32_t) * k);
    return 0;
}

typedef struct {
    const orc_inst *in;
    const int16_t *groups;
    int64_t lo, hi;
    double *total, *datap, *pipe;
    int rc;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *jb = (batch_job *)arg;
    int km = jb->in->k * jb->in->m;
    int32_t g[4096];
    double o3[3];
    for (int64_t p = jb->lo; p < jb->hi; p++) {
        for (int t = 0; t < km; t++) g[t] = jb->groups[p * km + t];
        int rc = orc_comm_cost(jb->in, g, o3, NULL, NULL);
        if (rc) {
            jb->rc = rc;
            return NULL;
        }
        jb->total[p] = o3[0];
        if (jb->datap) jb->datap[p] = o3[1];
        if (jb->pipe) jb->pipe[p] = o3[2];
    }
    return NULL;
}

int orc_comm_cost_batch(const orc_inst *in, const int16_t *groups, int64_t P, double *total,
                        double *datap, double *pipelinep, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 1024) nthreads = 1024;
    pthread_t th[1024];
    batch_job jobs[1024];
    int64_t per = (P + nthreads - 1) / nthreads;
    int used = 0;
    for (int t = 0; t < nthreads; t++) {
        int64_t lo = t * per, hi = lo + per < P ? lo + per : P;
        if (lo >= hi) break;
        jobs[t] = (batch_job){in, groups, lo, hi, total, datap, pipelinep, 0};
        if (nthreads == 1)
            batch_worker(&jobs[t]);
        else
            pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
        used++;
    }
    int rc = 0;
    for (int t = 0; t < used; t++) {
        if (nthreads > 1) pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    return rc;
}

/* ------------------------------------------------------------------ */
/* numpy Generator / PCG64 (numpy/random/src/pcg64, distributions.c,      */
/* _generator.pyx).  Call sites: scheduler.py:118,157-170,411,549-550.    */

static const unsigned __int128 PCG_MULT =
    ((unsigned __int128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;

uint64_t orc_next64(orc_pcg64 *g) {
    unsigned __int128 st = ((unsigned __int128)g->state_hi << 64) | g->state_lo;
    unsigned __int128 inc = ((unsigned __int128)g->inc_hi << 64) | g->inc_lo;
    st = st * PCG_MULT + inc;
    g->state_hi = (uint64_t)(st >> 64);
    g->state_lo = (uint64_t)st;
    uint64_t x = g->state_hi ^ g->state_lo;
    unsigned rot = (unsigned)(g->state_hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

uint32_t orc_next32(orc_pcg64 *g) {
    if (g->has_uint32) {
        g->has_uint32 = 0;
        return g->uinteger;
    }
    uint64_t v = orc_next64(g);
    g->has_uint32 = 1;
    g->uinteger = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

/* random_bounded_uint64 with use_masked=0: Lemire on 32-bit draws */
static uint64_t bounded(orc_pcg64 *g, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFULL) return orc_next32(g);
    uint32_t ex = (uint32_t)rng + 1u;
    uint64_t mprod = (uint64_t)orc_next32(g) * ex;
    uint32_t left = (uint32_t)mprod;
    if (left < ex) {
        uint32_t thr = (uint32_t)(0xFFFFFFFFu - (uint32_t)rng) % ex;
        while (left < thr) {
            mprod = (uint64_t)orc_next32(g) * ex;
            left = (uint32_t)mprod;
        }
    }
    return mprod >> 32;
}

/* random_interval: masked rejection, used by shuffle/permutation */
static uint64_t interval(orc_pcg64 *g, uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    while ((v = (orc_next32(g) & mask)) > mx) {
    }
    return v;
}

int64_t orc_integers(orc_pcg64 *g, int64_t low, int64_t high) {
    return low + (int64_t)bounded(g, (uint64_t)(high - low - 1));
}

void orc_permutation(orc_pcg64 *g, int n, int32_t *out) {
    for (int i = 0; i < n; i++) out[i] = i;
    for (int i = n - 1; i >= 1; i--) {
        int j = (int)interval(g, (uint64_t)i);
        int32_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Generator.choice(pop, size, replace=False): Floyd + Fisher-Yates draws;
 * the caller sorts the result (scheduler.py:161), so only the set and the
 * number of draws matter. */
void orc_choice_noreplace_sorted(orc_pcg64 *g, int pop, int size, int32_t *out) {
    int cnt = 0;
    for (int j = pop - size; j < pop; j++) {
        int32_t v = (int32_t)bounded(g, (uint64_t)j);
        int dup = 0;
        for (int t = 0; t < cnt; t++)
            if (out[t] == v) dup = 1;
        out[cnt++] = dup ? j : v;
    }
    for (int i = size - 1; i >= 1; i--) (void)bounded(g, (uint64_t)i);
    qsort(out, size, sizeof(int32_t), cmp_i32);
}

double orc_uniform(orc_pcg64 *g, double lo, double hi) {
    double u = (double)(orc_next64(g) >> 11) * (1.0 / 9007199254740992.0);
    return lo + (hi - lo) * u;
}

/* random_partition (scheduler.py:114-121) */
void orc_random_partition(orc_pcg64 *g, int n, int k, int m, int32_t *groups) {
    orc_permutation(g, n, groups);
    for (int j = 0; j < k; j++) qsort(groups + j * m, m, sizeof(int32_t), cmp_i32);
}

/* ------------------------------------------------------------------ */
/* variable-size group lists (chains unbalance groups: scheduler.py:299)  */

typedef struct {
    int k, cap;
    int *sz;
    int32_t *mem; /* k * cap */
} glist;

static glist gl_new(int k, int cap) {
    glist G;
    G.k = k;
    G.cap = cap;
    G.sz = (int *)calloc(k, sizeof(int));
    G.mem = (int32_t *)calloc((size_t)k * cap, sizeof(int32_t));
    return G;
}
static void gl_free(glist *G) {
    free(G->sz);
    free(G->mem);
}
static void gl_load(glist *G, const int32_t *groups, int m) {
    for (int j = 0; j < G->k; j++) {
        G->sz[j] = m;
        memcpy(G->mem + (size_t)j * G->cap, groups + j * m, sizeof(int32_t) * m);
    }
}
static void gl_store(const glist *G, int32_t *groups, int m) {
    for (int j = 0; j < G->k; j++) memcpy(groups + j * m, G->mem + (size_t)j * G->cap, sizeof(int32_t) * m);
}
static int32_t *gl_row(const glist *G, int j) { return G->mem + (size_t)j * G->cap; }
static void gl_remove(glist *G, int j, int32_t d) {
    int32_t *r = gl_row(G, j);
    int s = G->sz[j], i = 0;
    while (i < s && r[i] != d) i++;
    for (; i + 1 < s; i++) r[i] = r[i + 1];
    G->sz[j] = s - 1;
}
static void gl_insort(glist *G, int j, int32_t d) { /* bisect.insort (right) */
    int32_t *r = gl_row(G, j);
    int s = G->sz[j], i = s;
    while (i > 0 && r[i - 1] > d) {
        r[i] = r[i - 1];
        i--;
    }
    r[i] = d;
    G->sz[j] = s + 1;
}

/* crossover (scheduler.py:139-174) */
void orc_crossover(const int32_t *p1, const int32_t *p2, int k, int m, orc_pcg64 *g,
                   int32_t *out) {
    int n = k * m;
    int *in1 = (int *)malloc(sizeof(int) * n); /* group of each device in p1 */
    for (int j = 0; j < k; j++)
        for (int i = 0; i < m; i++) in1[p1[j * m + i]] = j;
    int32_t *diffs = (int32_t *)malloc(sizeof(int32_t) * n);
    int *dcnt = (int *)calloc(k, sizeof(int));
    int slots[4096], ns = 0;
    for (int j = 0; j < k; j++) {
        /* sorted(set(p2[j]) - set(p1[j])): p2[j] is ascending already */
        for (int i = 0; i < m; i++) {
            int32_t d = p2[j * m + i];
            if (in1[d] != j) diffs[j * m + dcnt[j]++] = d;
        }
        if (dcnt[j]) slots[ns++] = j;
    }
    if (ns == 0) {
        memcpy(out, p1, sizeof(int32_t) * n);
        free(in1);
        free(diffs);
        free(dcnt);
        return;
    }
    int j = slots[orc_integers(g, 0, ns)];
    int nd = dcnt[j];
    int mi = (int)orc_integers(g, 1, nd + 1);
    int32_t picked[4096];
    orc_choice_noreplace_sorted(g, nd, mi, picked);
    glist G = gl_new(k, m + 1);
    gl_load(&G, p1, m);
    int *home = in1; /* reuse */
    int32_t pool[4096];
    int npool = m;
    memcpy(pool, p1 + j * m, sizeof(int32_t) * m);
    for (int t = 0; t < mi; t++) {
        int32_t d = diffs[j * m + picked[t]];
        int src = home[d];
        gl_remove(&G, src, d);
        gl_insort(&G, j, d);
        home[d] = j;
        int vi = (int)orc_integers(g, 0, npool);
        int32_t victim = pool[vi];
        for (int q = vi; q + 1 < npool; q++) pool[q] = pool[q + 1];
        npool--;
        gl_remove(&G, j, victim);
        gl_insort(&G, src, victim);
        home[victim] = src;
    }
    gl_store(&G, out, m);
    gl_free(&G);
    free(in1);
    free(diffs);
    free(dcnt);
}

/* ------------------------------------------------------------------ */
/* surrogate gains and local search (scheduler.py:181-449)              */

static double row_pw_sum(const double *w, int n, int32_t u, const int32_t *grp, int cnt) {
    double buf[1024];
    if (cnt <= 0) return 0.0; /* numpy: the sum of an empty selection */
    for (int i = 0; i < cnt; i++) buf[i] = w[(size_t)u * n + grp[i]];
    return pw_sum(buf, cnt);
}

static double row_seq_mean(const double *w, int n, int32_t u, const int32_t *grp, int cnt) {
    double buf[1024];
    for (int i = 0; i < cnt; i++) buf[i] = w[(size_t)u * n + grp[i]];
    return seq_sum(buf, cnt) / (double)cnt;
}

/* _gain_ours (:206-209) */
static double gain_ours_raw(const double *w, int n, const int32_t *gj, int cj,
                            const int32_t *gj2, int cj2, int d1, int d2, int d1p, int d2p) {
    double t1 = row_pw_sum(w, n, d1, gj2, cj2) / (double)cj2 - w[(size_t)d1 * n + d2];
    double t2 = row_pw_sum(w, n, d1p, gj, cj) / (double)cj - w[(size_t)d1p * n + d2p];
    return t1 + t2;
}

double orc_gain_ours(const orc_inst *in, const int32_t *groups, int j, int j2, int d1, int d2,
                     int d1p, int d2p) {
    int m = in->m;
    return gain_ours_raw(in->sw, in->n, groups + j * m, m, groups + j2 * m, m, d1, d2, d1p, d2p);
}

/* gain_kl (:212-230) */
double orc_gain_kl(const orc_inst *in, const int32_t *groups, int d, int d2) {
    int k = in->k, m = in->m, n = in->n, jd = -1, jd2 = -1;
    for (int j = 0; j < k; j++)
        for (int i = 0; i < m; i++) {
            if (groups[j * m + i] == d) jd = j;
            if (groups[j * m + i] == d2) jd2 = j;
        }
    if (jd < 0 || jd2 < 0 || jd == jd2) return NAN;
    const int32_t *gj = groups + jd * m, *gj2 = groups + jd2 * m;
    int32_t ex[1024];
    int c;
    double t1 = row_pw_sum(in->sw, n, d, gj2, m);
    c = 0;
    for (int i = 0; i < m; i++)
        if (gj[i] != d) ex[c++] = gj[i];
    double t2 = row_pw_sum(in->sw, n, d, ex, c);
    double t3 = row_pw_sum(in->sw, n, d2, gj, m);
    c = 0;
    for (int i = 0; i < m; i++)
        if (gj2[i] != d2) ex[c++] = gj2[i];
    double t4 = row_pw_sum(in->sw, n, d2, ex, c);
    return t1 - t2 + t3 - t4 - 2.0 * in->sw[(size_t)d * n + d2];
}

/* _fast_edge (:237-249) */
static void fast_edge(const double *w, int n, const int32_t *grp, int cnt, int *a, int *b) {
    double best_v = INFINITY;
    *a = grp[0];
    *b = grp[1];
    for (int i = 0; i < cnt; i++)
        for (int l = i + 1; l < cnt; l++) {
            double v = w[(size_t)grp[i] * n + grp[l]];
            if (v < best_v) {
                best_v = v;
                *a = grp[i];
                *b = grp[l];
            }
        }
}

void orc_fast_edge(const orc_inst *in, const int32_t *grp, int cnt, int32_t *out2) {
    int a, b;
    fast_edge(in->sw, in->n, grp, cnt, &a, &b);
    out2[0] = a;
    out2[1] = b;
}

/* _best_candidate (:260-276) */
static double best_candidate(const double *w, int n, const glist *G, int j, int j2, int *oa,
                             int *ob) {
    int d1, d2, d1p, d2p;
    const int32_t *gj = gl_row(G, j), *gj2 = gl_row(G, j2);
    int cj = G->sz[j], cj2 = G->sz[j2];
    fast_edge(w, n, gj, cj, &d1, &d2);
    fast_edge(w, n, gj2, cj2, &d1p, &d2p);
    int cand[4][4] = {{d1, d2, d1p, d2p}, {d1, d2, d2p, d1p}, {d2, d1, d1p, d2p}, {d2, d1, d2p, d1p}};
    double best = -INFINITY;
    *oa = d1;
    *ob = d1p;
    for (int c = 0; c < 4; c++) {
        double gn = gain_ours_raw(w, n, gj, cj, gj2, cj2, cand[c][0], cand[c][1], cand[c][2], cand[c][3]);
        if (gn > best) {
            best = gn;
            *oa = cand[c][0];
            *ob = cand[c][2];
        }
    }
    return best;
}

static void do_swap(glist *G, int j, int j2, int a, int b) { /* _swap (:252-257) */
    gl_remove(G, j, a);
    gl_remove(G, j2, b);
    gl_insort(G, j2, a);
    gl_insort(G, j, b);
}

static void do_move(glist *G, int v, int src, int dst) { /* _move (:294-296) */
    gl_remove(G, src, v);
    gl_insort(G, dst, v);
}

/* _home_costs (:287-291) restricted to one member; fastest_free (:318-328) */
static int fastest_free(const double *w, int n, const glist *G, int i, const char *locked,
                        double *home_out) {
    const int32_t *grp = gl_row(G, i);
    int cnt = G->sz[i];
    if (cnt < 2) return -1;
    int best = -1;
    double bh = 0.0;
    for (int a = 0; a < cnt; a++) {
        int d = grp[a];
        if (locked[d]) continue;
        double h = INFINITY;
        for (int b = 0; b < cnt; b++) {
            if (b == a) continue;
            double v = w[(size_t)d * n + grp[b]];
            if (v < h) h = v;
        }
        /* min by (home, id): members ascend, so strict < keeps first */
        if (best < 0 || h < bh) {
            best = d;
            bh = h;
        }
    }
    if (best >= 0) *home_out = bh;
    return best;
}

/* _chain_round (:299-391) */
static int chain_round(const double *w, int n, glist *G, char *locked, int *nlocked,
                       double *mean /* n*k */) {
    int k = G->k;
    for (int i = 0; i < k; i++)
        for (int u = 0; u < n; u++) mean[(size_t)u * k + i] = row_seq_mean(w, n, u, gl_row(G, i), G->sz[i]);
    double best_start = -INFINITY;
    int start = -1;
    for (int i = 0; i < k; i++) {
        double home;
        int v = fastest_free(w, n, G, i, locked, &home);
        if (v < 0) continue;
        double mx = -INFINITY;
        int first = 1;
        for (int j = 0; j < k; j++) {
            if (j == i) continue;
            double x = mean[(size_t)v * k + j];
            if (first || x > mx) mx = x;
            first = 0;
        }
        double gain = mx - home;
        if (gain > best_start) {
            best_start = gain;
            start = i;
        }
    }
    if (start < 0) return 0;
    int mv_v[256], mv_src[256], mv_dst[256], nm = 0;
    double steps[256], closers[256];
    int cur = start, natural = 0;
    for (int it = 0; it < k; it++) {
        double home;
        int v = fastest_free(w, n, G, cur, locked, &home);
        if (v < 0) break;
        int dst = -1;
        double sc = -INFINITY;
        for (int j = 0; j < k; j++) {
            if (j == cur) continue;
            double x = mean[(size_t)v * k + j];
            if (dst < 0 || x > sc) {
                sc = x;
                dst = j;
            }
        }
        closers[nm] = (cur != start) ? mean[(size_t)v * k + start] - home : -INFINITY;
        steps[nm] = sc - home;
        do_move(G, v, cur, dst);
        locked[v] = 1;
        (*nlocked)++;
        mv_v[nm] = v;
        mv_src[nm] = cur;
        mv_dst[nm] = dst;
        nm++;
        int cols[2] = {cur, dst};
        for (int t = 0; t < 2; t++) {
            int col = cols[t];
            for (int u = 0; u < n; u++)
                mean[(size_t)u * k + col] = row_seq_mean(w, n, u, gl_row(G, col), G->sz[col]);
        }
        cur = dst;
        if (cur == start) {
            natural = 1;
            break;
        }
    }
    if (nm == 0) return 0;
    double prefix[257];
    prefix[0] = 0.0;
    for (int t = 0; t < nm; t++) prefix[t + 1] = prefix[t] + steps[t]; /* np.cumsum */
    double best_v = -INFINITY;
    int best_l = -1;
    for (int l = 0; l < nm; l++) {
        double value = prefix[l] + closers[l];
        if (value > best_v) {
            best_v = value;
            best_l = l;
        }
    }
    if (natural && prefix[nm] > best_v) {
        best_v = prefix[nm];
        best_l = nm;
    }
    if (best_v <= 0.0) {
        for (int t = nm - 1; t >= 0; t--) do_move(G, mv_v[t], mv_dst[t], mv_src[t]);
        return 0;
    }
    for (int t = nm - 1; t >= best_l; t--) do_move(G, mv_v[t], mv_dst[t], mv_src[t]);
    if (best_l < nm) do_move(G, mv_v[best_l], mv_src[best_l], start);
    return 1;
}

/* _pass_ours (:394-428) */
static int pass_ours(const double *w, int n, glist *G, orc_pcg64 *g, int phase, double *mean) {
    int k = G->k, d_dp = G->sz[0], changed = 0;
    if (d_dp < 2) return 0;
    if (phase % 2 == 0) {
        int np = k * (k - 1) / 2;
        int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (np > 0 ? np : 1));
        int *pj = (int *)malloc(sizeof(int) * (np > 0 ? np : 1)), *pj2 = (int *)malloc(sizeof(int) * (np > 0 ? np : 1));
        int t = 0;
        for (int j = 0; j < k; j++)
            for (int j2 = j + 1; j2 < k; j2++) {
                pj[t] = j;
                pj2[t] = j2;
                t++;
            }
        orc_permutation(g, np, perm);
        for (int q = 0; q < np; q++) {
            int j = pj[perm[q]], j2 = pj2[perm[q]];
            for (int it = 0; it < d_dp; it++) {
                int a, b;
                double gain = best_candidate(w, n, G, j, j2, &a, &b);
                if (gain <= 0.0) break;
                do_swap(G, j, j2, a, b);
                changed = 1;
            }
        }
        free(perm);
        free(pj);
        free(pj2);
        return changed;
    }
    char *locked = (char *)calloc(n, 1);
    int nlocked = 0;
    while (nlocked < n) {
        int before = nlocked;
        if (chain_round(w, n, G, locked, &nlocked, mean)) changed = 1;
        if (nlocked == before) break;
    }
    free(locked);
    return changed;
}

/* _pass_kl (:431-449) */
static int pass_kl(const double *w, int n, glist *G) {
    int k = G->k, changed = 0;
    for (int j = 0; j < k; j++) {
        for (int j2 = j + 1; j2 < k; j2++) {
            const int32_t *a1 = gl_row(G, j), *a2 = gl_row(G, j2);
            int c1 = G->sz[j], c2 = G->sz[j2];
            double s11[1024], s12[1024], s22[1024], s21[1024];
            for (int i = 0; i < c1; i++) {
                s11[i] = row_pw_sum(w, n, a1[i], a1, c1);
                s12[i] = row_pw_sum(w, n, a1[i], a2, c2);
            }
            for (int l = 0; l < c2; l++) {
                s22[l] = row_pw_sum(w, n, a2[l], a2, c2);
                s21[l] = row_pw_sum(w, n, a2[l], a1, c1);
            }
            double best = 0.0;
            int bi = -1, bl = -1;
            for (int i = 0; i < c1; i++)
                for (int l = 0; l < c2; l++) {
                    double gn = ((s12[i] - s11[i]) + (s21[l] - s22[l])) - 2.0 * w[(size_t)a1[i] * n + a2[l]];
                    if (bi < 0 || gn > best) { /* np.argmax: first maximum */
                        best = gn;
                        bi = i;
                        bl = l;
                    }
                }
            if (best > 0.0) {
                do_swap(G, j, j2, a1[bi], a2[bl]);
                changed = 1;
            }
        }
    }
    return changed;
}

int orc_pass(const orc_inst *in, int32_t *groups, int kind, orc_pcg64 *g, int phase) {
    glist G = gl_new(in->k, in->m + 1);
    gl_load(&G, groups, in->m);
    double *mean = (double *)malloc(sizeof(double) * (size_t)in->n * in->k);
    int ch = kind == 0 ? pass_ours(in->sw, in->n, &G, g, phase, mean) : pass_kl(in->sw, in->n, &G);
    gl_store(&G, groups, in->m);
    gl_free(&G);
    free(mean);
    return ch;
}

/* _refine (:455-487).  Writes the refined partition into best_groups and
 * its cost; returns the number of true-cost evaluations. */
static int refine(const orc_inst *in, const int32_t *p, int kind, orc_pcg64 *g, int max_passes,
                  int32_t *best_groups, double *best3) {
    int k = in->k, m = in->m, n = in->n, evals = 0;
    memcpy(best_groups, p, sizeof(int32_t) * k * m);
    orc_comm_cost(in, p, best3, NULL, NULL);
    evals++;
    glist G = gl_new(k, m + 1);
    gl_load(&G, p, m);
    double *mean = (double *)malloc(sizeof(double) * (size_t)n * k);
    int32_t *cand = (int32_t *)malloc(sizeof(int32_t) * k * m);
    int stop_after = kind == 0 ? 2 : 1, stale = 0;
    for (int t = 0; t < max_passes; t++) {
        int changed = kind == 0 ? pass_ours(in->sw, n, &G, g, t, mean) : pass_kl(in->sw, n, &G);
        if (!changed) {
            stale++;
            if (stale >= stop_after) break;
            continue;
        }
        stale = 0;
        gl_store(&G, cand, m);
        double c3[3];
        orc_comm_cost(in, cand, c3, NULL, NULL);
        evals++;
        if (c3[0] < best3[0]) {
            memcpy(best_groups, cand, sizeof(int32_t) * k * m);
            memcpy(best3, c3, sizeof(c3));
        }
    }
    gl_free(&G);
    free(mean);
    free(cand);
    return evals;
}

int orc_local_search(const orc_inst *in, int32_t *groups, int kind, orc_pcg64 *g, int max_passes) {
    int32_t *best = (int32_t *)malloc(sizeof(int32_t) * in->k * in->m);
    double b3[3];
    int ev = refine(in, groups, kind, g, max_passes, best, b3);
    memcpy(groups, best, sizeof(int32_t) * in->k * in->m);
    free(best);
    return ev;
}

/* Partition.canonical() (costmodel.py:86-88): groups sorted as tuples;
 * groups are disjoint, so the first member decides. */
static void canonicalize(int32_t *groups, int k, int m) {
    int32_t tmp[1024];
    for (int a = 1; a < k; a++) {
        memcpy(tmp, groups + a * m, sizeof(int32_t) * m);
        int b = a - 1;
        while (b >= 0 && groups[b * m] > tmp[0]) {
            memcpy(groups + (b + 1) * m, groups + b * m, sizeof(int32_t) * m);
            b--;
        }
        memcpy(groups + (b + 1) * m, tmp, sizeof(int32_t) * m);
    }
}

/* evolve (:515-574) */
int orc_evolve(const orc_inst *in, const orc_ga_cfg *cfg, orc_pcg64 *g, int32_t *best_groups,
               double *best3, double *best_per_group, int32_t *best_order, double *trace_best,
               double *trace_mean, int64_t *evaluations) {
    int k = in->k, m = in->m, n = in->n, P = cfg->pop_size, km = k * m;
    if (cfg->kind == 0 && k == 1) return -3; /* reference raises in _chain_round */
    int32_t *pop = (int32_t *)malloc(sizeof(int32_t) * (size_t)P * km);
    double *tot = (double *)malloc(sizeof(double) * P);
    double *tmp = (double *)malloc(sizeof(double) * P);
    int64_t evals = 0;
    double c3[3];
    for (int i = 0; i < P; i++) orc_random_partition(g, n, k, m, pop + (size_t)i * km);
    for (int i = 0; i < P; i++) {
        orc_comm_cost(in, pop + (size_t)i * km, c3, NULL, NULL);
        tot[i] = c3[0];
        evals++;
    }
    int best_i = 0;
    for (int i = 1; i < P; i++)
        if (tot[i] < tot[best_i]) best_i = i;
    int32_t *bestp = (int32_t *)malloc(sizeof(int32_t) * km);
    int32_t *off = (int32_t *)malloc(sizeof(int32_t) * km);
    int32_t *ref = (int32_t *)malloc(sizeof(int32_t) * km);
    memcpy(bestp, pop + (size_t)best_i * km, sizeof(int32_t) * km);
    double best_total = tot[best_i];
    int since = 0, rows = 0;
    for (int gen = 0; gen < cfg->generations; gen++) {
        int i = (int)orc_integers(g, 0, P);
        int i2 = (int)orc_integers(g, 0, P - 1);
        if (i2 >= i) i2++;
        orc_crossover(pop + (size_t)i * km, pop + (size_t)i2 * km, k, m, g, off);
        double cb;
        if (cfg->kind == 2) {
            memcpy(ref, off, sizeof(int32_t) * km);
            orc_comm_cost(in, off, c3, NULL, NULL);
            evals++;
            cb = c3[0];
        } else {
            double r3[3];
            evals += refine(in, off, cfg->kind, g, cfg->max_passes, ref, r3);
            cb = r3[0];
        }
        int worst = 0;
        for (int t = 1; t < P; t++)
            if (tot[t] > tot[worst]) worst = t;
        if (cb < tot[worst]) {
            memcpy(pop + (size_t)worst * km, ref, sizeof(int32_t) * km);
            tot[worst] = cb;
        }
        if (cb < best_total) {
            memcpy(bestp, ref, sizeof(int32_t) * km);
            best_total = cb;
            since = 0;
        } else {
            since++;
        }
        memcpy(tmp, tot, sizeof(double) * P);
        trace_best[rows] = best_total;
        trace_mean[rows] = pw_sum(tmp, P) / (double)P;
        rows++;
        if (cfg->patience > 0 && since >= cfg->patience) break;
    }
    canonicalize(bestp, k, m);
    memcpy(best_groups, bestp, sizeof(int32_t) * km);
    orc_comm_cost(in, bestp, best3, best_per_group, best_order);
    evals++;
    *evaluations = evals;
    free(pop);
    free(tot);
    free(tmp);
    free(bestp);
    free(off);
    free(ref);
    return rows;
}

/* ------------------------------------------------------------------ */
/* fixed layouts: evaluation.py:162-243                                  */

int orc_random_assignment(orc_pcg64 *g, int n, int k, int m, int32_t *grid, int32_t *order) {
    int32_t *p = (int32_t *)malloc(sizeof(int32_t) * n);
    orc_random_partition(g, n, k, m, p);
    orc_permutation(g, k, order);
    for (int b = 0; b < k; b++)
        for (int i = 0; i < m; i++) grid[i * k + b] = p[order[b] * m + i];
    free(p);
    return 0;
}

int orc_evaluate_assignment(const orc_inst *in, const int32_t *grid, double *out3, double *per_col) {
    int k = in->k, m = in->m, n = in->n;
    int32_t col[1024];
    double datap = 0.0;
    for (int b = 0; b < k; b++) {
        for (int i = 0; i < m; i++) col[i] = grid[i * k + b];
        qsort(col, m, sizeof(int32_t), cmp_i32);
        double v = orc_datap_group(in, col, m);
        if (per_col) per_col[b] = v;
        if (b == 0 || v > datap) datap = v;
    }
    double pipe = 0.0;
    double bnd[1024];
    for (int b = 0; b < k - 1; b++) {
        double worst = 0.0;
        for (int i = 0; i < m; i++) {
            double c = in->pp[(size_t)grid[i * k + b] * n + grid[i * k + b + 1]];
            if (c > worst) worst = c;
        }
        bnd[b] = worst;
    }
    for (int b = k - 2; b >= 0; b--) pipe = bnd[b] + pipe;
    out3[0] = datap + pipe;
    out3[1] = datap;
    out3[2] = pipe;
    return 0;
}

int orc_materialize(const orc_inst *in, const int32_t *groups, int32_t *grid, int32_t *order) {
    int k = in->k, m = in->m, n = in->n;
    double *E = (double *)malloc(sizeof(double) * k * k);
    int32_t *pairs = (int32_t *)malloc(sizeof(int32_t) * k * k * m);
    double sub[4096];
    for (int j = 0; j < k; j++) E[j * k + j] = 0.0;
    for (int j = 0; j < k; j++)
        for (int j2 = j + 1; j2 < k; j2++) {
            for (int r = 0; r < m; r++)
                for (int c = 0; c < m; c++) sub[r * m + c] = in->pp[(size_t)groups[j * m + r] * n + groups[j2 * m + c]];
            double v;
            if (orc_bottleneck_matching(sub, m, pairs + (size_t)(j * k + j2) * m, &v)) {
                free(E);
                free(pairs);
                return -1;
            }
            E[j * k + j2] = E[j2 * k + j] = v;
        }
    double tot;
    int rc = orc_open_loop_tsp(E, k, &tot, order);
    if (rc) {
        free(E);
        free(pairs);
        return rc;
    }
    int32_t cols[1024];
    for (int i = 0; i < m; i++) cols[i] = groups[order[0] * m + i];
    for (int i = 0; i < m; i++) grid[i * k + 0] = cols[i];
    for (int b = 1; b < k; b++) {
        int prev = order[b - 1], cur = order[b];
        int lo = prev < cur ? prev : cur, hi = prev < cur ? cur : prev;
        const int32_t *pr = pairs + (size_t)(lo * k + hi) * m;
        const int32_t *lo_devs = groups + lo * m, *hi_devs = groups + hi * m;
        for (int i = 0; i < m; i++) {
            int32_t d = cols[i], nx = -1;
            if (prev == lo) {
                for (int r = 0; r < m; r++)
                    if (lo_devs[r] == d) nx = hi_devs[pr[r]];
            } else {
                for (int r = 0; r < m; r++)
                    if (hi_devs[pr[r]] == d) nx = lo_devs[r];
            }
            cols[i] = nx;
            grid[i * k + b] = nx;
        }
    }
    free(E);
    free(pairs);
    return 0;
}
