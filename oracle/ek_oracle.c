/*
 * ek_oracle.c -- CPU restatement of the reference elastic-distance engines.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path and the "port" CPU baseline in bench.py.  Nothing in the product
 * package (paper_2102_05221_b200/) links or calls it.
 *
 * It restates, in plain C, the arithmetic of the reference package `elastik`:
 *   - move costs      : pkg/src/elastik/kernels.py:70-77, 95-105, 181-242
 *                       (compiled twin: pkg/src/elastik/_speedups.pyx:33-94)
 *   - borders         : pkg/src/elastik/kernels.py:244-262, 280-289
 *   - engine "base"   : pkg/src/elastik/_speedups.pyx:105-126 (_pyloops.py:20-44)
 *   - engine "ea"     : pkg/src/elastik/_speedups.pyx:129-162 (_pyloops.py:47-89)
 *   - engine "eapruned": pkg/src/elastik/_speedups.pyx:165-271 (_pyloops.py:92-241)
 *   - diagonal UB     : pkg/src/elastik/engines.py:87-103
 *   - variant facade  : pkg/src/elastik/engines.py:106-147
 *   - nn_search scan  : pkg/src/elastik/search.py:81-125 (lb="none")
 * Every floating-point operation is performed in the same order as the
 * reference; build with -ffp-contract=off (as pkg/setup.py:20 does) so no
 * FMA contraction changes a rounding.  Cell counts follow the reference's
 * counting exactly, so EngineResult equality can be asserted.
 *
 * Parity pin: tests/test_oracle_pins.py checks this file against the golden
 * fixtures generated from the live reference (tests/golden/make_golden.py)
 * and against the reference's own known-answer values.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EKO_INF (INFINITY)

enum { K_DTW = 0, K_CDTW = 1, K_WDTW = 2, K_ERP = 3, K_MSM = 4, K_TWE = 5 };
enum { E_BASE = 0, E_EA = 1, E_EAPRUNED = 2 };
enum { V_BASE = 0, V_EA = 1, V_EAPRUNED = 2, V_PRUNED_ONLY = 3 };

typedef struct {
    int kind;
    int mode;          /* 0 squared, 1 absolute */
    double gap, msm_c, nu, lam;
    const double *wt;  /* wdtw weight table indexed by |i-j| (len >= max(nl,nc)+1) */
    const double *vb;  /* erp left border, index 0..nl  (NULL => +inf)          */
    const double *hb;  /* erp top border,  index 0..nc  (NULL => +inf)          */
} eko_rec;

/* ---- point and move costs (kernels.py:70-77, 95-105; _speedups.pyx:33-94) ---- */

static inline double pcost(double a, double b, int mode) {
    if (mode == 0) {
        double d = a - b;
        return d * d;
    }
    return fabs(a - b);
}

static inline double msm_sm(double np_, double x, double y, double c) {
    if ((x <= np_ && np_ <= y) || (x >= np_ && np_ >= y)) return c;
    double d1 = fabs(np_ - x), d2 = fabs(np_ - y);
    return c + (d1 < d2 ? d1 : d2);
}

/* 1-based i (row / lines), j (col / cols) */
static inline double mv_canon(const double *l, const double *c, long i, long j, const eko_rec *r) {
    long dd = i >= j ? i - j : j - i;
    switch (r->kind) {
    case K_WDTW: return pcost(l[i - 1], c[j - 1], r->mode) * r->wt[dd];
    case K_MSM: return fabs(l[i - 1] - c[j - 1]);
    case K_TWE: {
        double sp = i >= 2 ? l[i - 2] : 0.0, tp = j >= 2 ? c[j - 2] : 0.0;
        double dij = (double)dd;
        return (pcost(l[i - 1], c[j - 1], r->mode) + pcost(sp, tp, r->mode)) + r->nu * (dij + dij);
    }
    default: return pcost(l[i - 1], c[j - 1], r->mode); /* dtw, cdtw, erp */
    }
}

static inline double mv_row(const double *l, const double *c, long i, long j, const eko_rec *r) {
    switch (r->kind) {
    case K_ERP: return pcost(l[i - 1], r->gap, r->mode);
    case K_MSM: return msm_sm(l[i - 1], i >= 2 ? l[i - 2] : l[i - 1], c[j - 1], r->msm_c);
    case K_TWE: return (pcost(l[i - 1], i >= 2 ? l[i - 2] : 0.0, r->mode) + r->nu) + r->lam;
    default: return mv_canon(l, c, i, j, r);
    }
}

static inline double mv_col(const double *l, const double *c, long i, long j, const eko_rec *r) {
    switch (r->kind) {
    case K_ERP: return pcost(r->gap, c[j - 1], r->mode);
    case K_MSM: return msm_sm(c[j - 1], l[i - 1], j >= 2 ? c[j - 2] : c[j - 1], r->msm_c);
    case K_TWE: return (pcost(c[j - 1], j >= 2 ? c[j - 2] : 0.0, r->mode) + r->nu) + r->lam;
    default: return mv_canon(l, c, i, j, r);
    }
}

static inline double vbord(long i, const eko_rec *r) { return r->vb ? r->vb[i] : EKO_INF; }
static inline double hbord(long j, const eko_rec *r) { return r->hb ? r->hb[j] : EKO_INF; }

/* the three-dependency cell in the reference's comparison order */
static inline double cell3(double d, double t, double lft, const double *l, const double *c,
                           long i, long j, const eko_rec *r) {
    double v = d + mv_canon(l, c, i, j, r);
    double a = t + mv_row(l, c, i, j, r);
    if (a < v) v = a;
    a = lft + mv_col(l, c, i, j, r);
    if (a < v) v = a;
    return v;
}

/* ---- engines ---- */

static double eng_base(const double *l, long nl, const double *c, long nc, const eko_rec *r,
                       double *prev, double *curr, int64_t *cells) {
    curr[0] = 0.0;
    for (long j = 1; j <= nc; j++) curr[j] = hbord(j, r);
    for (long i = 1; i <= nl; i++) {
        double *t = prev; prev = curr; curr = t;
        curr[0] = vbord(i, r);
        for (long j = 1; j <= nc; j++) curr[j] = cell3(prev[j - 1], prev[j], curr[j - 1], l, c, i, j, r);
    }
    *cells = (int64_t)nl * (int64_t)nc;
    return curr[nc];
}

static double eng_ea(const double *l, long nl, const double *c, long nc, long w, double cutoff,
                     const eko_rec *r, double *prev, double *curr, int64_t *cells) {
    *cells = 0;
    if (w < nl - nc) return EKO_INF;
    curr[0] = 0.0;
    long top = w + 1 < nc ? w + 1 : nc;
    for (long j = 1; j <= top; j++) curr[j] = hbord(j, r);
    for (long i = 1; i <= nl; i++) {
        double *t = prev; prev = curr; curr = t;
        long js = i - w > 1 ? i - w : 1;
        long je = i + w < nc ? i + w : nc;
        curr[js - 1] = js == 1 ? vbord(i, r) : EKO_INF;
        double rowmin = curr[js - 1];
        for (long j = js; j <= je; j++) {
            double v = cell3(prev[j - 1], prev[j], curr[j - 1], l, c, i, j, r);
            curr[j] = v;
            (*cells)++;
            if (v < rowmin) rowmin = v;
        }
        if (rowmin > cutoff) return EKO_INF;
    }
    return curr[nc];
}

static double eng_eapruned(const double *l, long nl, const double *c, long nc, long w, double cutoff,
                           const eko_rec *r, double *prev, double *curr, int64_t *cells) {
    *cells = 0;
    if (w < nl - nc) return EKO_INF;
    curr[0] = 0.0;
    long top = w + 1 < nc ? w + 1 : nc;
    long npp = 1;
    for (long j = 1; j <= top; j++) {
        curr[j] = hbord(j, r);
        if (curr[j] <= cutoff) npp = j + 1;
    }
    long ns = 1, pp = npp, j = 1;
    for (long i = 1; i <= nl; i++) {
        double *t = prev; prev = curr; curr = t;
        long js = i - w > ns ? i - w : ns;
        long je = i + w < nc ? i + w : nc;
        j = js;
        curr[js - 1] = js == 1 ? vbord(i, r) : EKO_INF;
        int alive = curr[js - 1] <= cutoff;
        /* discard points: left neighbour dead, diag + top only */
        if (curr[js - 1] > cutoff) {
            for (; j <= pp - 1 && j == ns; j++) {
                double v = prev[j - 1] + mv_canon(l, c, i, j, r);
                double a = prev[j] + mv_row(l, c, i, j, r);
                if (a < v) v = a;
                (*cells)++;
                curr[j] = v;
                if (v <= cutoff) { npp = j + 1; alive = 1; }
                else ns++;
            }
        }
        /* full cells up to the pruning point */
        for (; j <= pp - 1; j++) {
            double v = cell3(prev[j - 1], prev[j], curr[j - 1], l, c, i, j, r);
            (*cells)++;
            curr[j] = v;
            if (v <= cutoff) { npp = j + 1; alive = 1; }
        }
        /* the pruning point: top dependency dead */
        if (j <= je) {
            if (j == ns && curr[j - 1] > cutoff) {
                double v = prev[j - 1] + mv_canon(l, c, i, j, r);
                (*cells)++;
                curr[j] = v;
                if (v <= cutoff) { npp = j + 1; alive = 1; }
                else return EKO_INF;
            } else {
                double v = prev[j - 1] + mv_canon(l, c, i, j, r);
                double a = curr[j - 1] + mv_col(l, c, i, j, r);
                if (a < v) v = a;
                (*cells)++;
                curr[j] = v;
                if (v <= cutoff) { npp = j + 1; alive = 1; }
            }
            j++;
        } else if (j == ns) {
            return EKO_INF;
        }
        /* past the pruning point: left dependency only */
        for (; j <= je && j == npp; j++) {
            double v = curr[j - 1] + mv_col(l, c, i, j, r);
            (*cells)++;
            curr[j] = v;
            if (v <= cutoff) { npp = j + 1; alive = 1; }
        }
        if (!alive) return EKO_INF;
        pp = npp;
    }
    if (j <= nc) return EKO_INF;
    double cost = curr[nc];
    return cost > cutoff ? EKO_INF : cost;
}

/* ---- the engine entry (mirrors _speedups.run, pkg/src/elastik/_speedups.pyx:274-317) ---- */

static double run_engine(int engine, const double *l, long nl, const double *c, long nc,
                         long w, double cutoff, const eko_rec *r, double *buf, int64_t *cells) {
    for (long k = 0; k < 2 * (nc + 1); k++) buf[k] = EKO_INF;
    double *prev = buf, *curr = buf + nc + 1;
    if (engine == E_BASE) return eng_base(l, nl, c, nc, r, prev, curr, cells);
    if (engine == E_EA) return eng_ea(l, nl, c, nc, w, cutoff, r, prev, curr, cells);
    return eng_eapruned(l, nl, c, nc, w, cutoff, r, prev, curr, cells);
}

int eko_run(int engine, const double *lines, long nl, const double *cols, long nc, int kind, int mode,
            long window, double cutoff, double gap, double msm_c, double nu, double lam,
            const double *weights, const double *vb, const double *hb, double *out_cost,
            int64_t *out_cells) {
    if (nl < 1 || nc < 1) return -1;
    eko_rec r = {kind, mode, gap, msm_c, nu, lam, weights, vb, hb};
    double *buf = (double *)malloc(sizeof(double) * 2 * (size_t)(nc + 1));
    if (!buf) return -2;
    *out_cost = run_engine(engine, lines, nl, cols, nc, window, cutoff, &r, buf, out_cells);
    free(buf);
    return 0;
}

/* ---- make_recurrence + variant facade (kernels.py:157-277; engines.py:87-147) ---- */

typedef struct {
    int kind, mode, variant;
    long window;           /* <0 => None (unbounded) */
    double gap, msm_c, nu, lam;
    const double *const *wtabs; /* wdtw: wtabs[m] = table for longest length m */
} eko_spec;

typedef struct {
    double *buf;           /* 2*(cap+1) row buffer */
    double *vb, *hb;       /* erp borders, cap+1 each */
    long cap;
} eko_ws;

static int ws_reserve(eko_ws *ws, long n) {
    if (n <= ws->cap) return 0;
    free(ws->buf); free(ws->vb); free(ws->hb);
    ws->buf = (double *)malloc(sizeof(double) * 2 * (size_t)(n + 1));
    ws->vb = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    ws->hb = (double *)malloc(sizeof(double) * (size_t)(n + 1));
    ws->cap = n;
    return (ws->buf && ws->vb && ws->hb) ? 0 : -2;
}

static void ws_free(eko_ws *ws) { free(ws->buf); free(ws->vb); free(ws->hb); ws->cap = 0; }

/* _erp_border (kernels.py:280-289): sequential prefix of gap-alignment costs */
static void erp_border(const double *v, long n, double gap, int mode, int row, double *out) {
    double acc = 0.0;
    out[0] = 0.0;
    for (long k = 1; k <= n; k++) {
        acc = acc + (row ? pcost(v[k - 1], gap, mode) : pcost(gap, v[k - 1], mode));
        out[k] = acc;
    }
}

/* diagonal_upper_bound (engines.py:87-103), summed in the same order */
static double diag_ub(const double *l, long nl, const double *c, long nc, const eko_rec *r) {
    double total = 0.0;
    for (long k = 1; k <= nc; k++) total += mv_canon(l, c, k, k, r);
    for (long i = nc + 1; i <= nl; i++) total += mv_row(l, c, i, nc, r);
    return total;
}

/* engines.distance (engines.py:121-147): returns cost, writes cells */
static double facade(const eko_spec *sp, const double *s, long ls, const double *t, long lt,
                     double cutoff, eko_ws *ws, int64_t *cells) {
    const double *l = s, *c = t;
    long nl = ls, nc = lt;
    if (lt > ls) { l = t; nl = lt; c = s; nc = ls; } /* ties keep s on the rows */
    long w = sp->window >= 0 ? sp->window : nl;
    eko_rec r = {sp->kind, sp->mode, sp->gap, sp->msm_c, sp->nu, sp->lam, NULL, NULL, NULL};
    if (ws_reserve(ws, nl > nc ? nl : nc)) { *cells = -1; return NAN; }
    if (sp->kind == K_WDTW) r.wt = sp->wtabs[nl];
    if (sp->kind == K_ERP) {
        erp_border(l, nl, sp->gap, sp->mode, 1, ws->vb);
        erp_border(c, nc, sp->gap, sp->mode, 0, ws->hb);
        r.vb = ws->vb; r.hb = ws->hb;
    }
    switch (sp->variant) {
    case V_BASE:
        if (sp->window < 0) return run_engine(E_BASE, l, nl, c, nc, w, EKO_INF, &r, ws->buf, cells);
        return run_engine(E_EA, l, nl, c, nc, w, EKO_INF, &r, ws->buf, cells);
    case V_EA: return run_engine(E_EA, l, nl, c, nc, w, cutoff, &r, ws->buf, cells);
    case V_EAPRUNED: return run_engine(E_EAPRUNED, l, nl, c, nc, w, cutoff, &r, ws->buf, cells);
    default:
        if (w < nl - nc) { *cells = 0; return EKO_INF; }
        return run_engine(E_EAPRUNED, l, nl, c, nc, w, diag_ub(l, nl, c, nc, &r), &r, ws->buf, cells);
    }
}

int eko_distance(const eko_spec *sp, const double *s, long ls, const double *t, long lt, double cutoff,
                 double *out_cost, int64_t *out_cells) {
    eko_ws ws = {0};
    *out_cost = facade(sp, s, ls, t, lt, cutoff, &ws, out_cells);
    ws_free(&ws);
    return *out_cells < 0 ? -2 : 0;
}

double eko_diag_ub(const eko_spec *sp, const double *s, long ls, const double *t, long lt) {
    const double *l = s, *c = t;
    long nl = ls, nc = lt;
    if (lt > ls) { l = t; nl = lt; c = s; nc = ls; }
    eko_rec r = {sp->kind, sp->mode, sp->gap, sp->msm_c, sp->nu, sp->lam, NULL, NULL, NULL};
    if (sp->kind == K_WDTW) r.wt = sp->wtabs[nl];
    return diag_ub(l, nl, c, nc, &r);
}

/* ---- batched drivers, threaded over independent units (queries / rows) ---- */

typedef struct {
    const eko_spec *sp;
    const double *Q; const int64_t *qoff; const int64_t *qlen;
    const double *C; const int64_t *coff; const int64_t *clen;
    long nq, nc;
    int64_t *nn_idx; double *nn_dist; int64_t *cells; int64_t *computed; int64_t *abandoned;
    long next;
    pthread_mutex_t mu;
    int err;
} nn_job;

static long take(long *next, pthread_mutex_t *mu, long n) {
    pthread_mutex_lock(mu);
    long k = *next < n ? (*next)++ : -1;
    pthread_mutex_unlock(mu);
    return k;
}

static void *nn_worker(void *arg) {
    nn_job *jb = (nn_job *)arg;
    eko_ws ws = {0};
    long q;
    while ((q = take(&jb->next, &jb->mu, jb->nq)) >= 0) {
        /* search.nn_search (search.py:101-123): serial scan, running cutoff, strict < */
        double dnn = EKO_INF;
        int64_t best = -1, cells = 0, comp = 0, ab = 0;
        for (long k = 0; k < jb->nc; k++) {
            int64_t cc = 0;
            double d = facade(jb->sp, jb->Q + jb->qoff[q], jb->qlen[q], jb->C + jb->coff[k], jb->clen[k],
                              dnn, &ws, &cc);
            if (cc < 0) { jb->err = -2; break; }
            cells += cc;
            if (isinf(d)) { ab++; continue; }
            comp++;
            if (d < dnn) { dnn = d; best = k; }
        }
        jb->nn_idx[q] = best; jb->nn_dist[q] = dnn; jb->cells[q] = cells;
        jb->computed[q] = comp; jb->abandoned[q] = ab;
    }
    ws_free(&ws);
    return NULL;
}

static int run_threads(void *(*fn)(void *), void *job, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    if (!th) return -2;
    int started = 0;
    for (int k = 0; k < nthreads; k++)
        if (pthread_create(&th[k], NULL, fn, job) == 0) started++;
    for (int k = 0; k < started; k++) pthread_join(th[k], NULL);
    free(th);
    if (started == 0) fn(job);
    return 0;
}

int eko_nn(const eko_spec *sp, const double *Q, const int64_t *qoff, const int64_t *qlen, long nq,
           const double *C, const int64_t *coff, const int64_t *clen, long nc, int nthreads,
           int64_t *nn_idx, double *nn_dist, int64_t *cells, int64_t *computed, int64_t *abandoned) {
    nn_job jb = {sp, Q, qoff, qlen, C, coff, clen, nq, nc, nn_idx, nn_dist, cells, computed, abandoned, 0,
                 PTHREAD_MUTEX_INITIALIZER, 0};
    run_threads(nn_worker, &jb, nthreads);
    return jb.err;
}

typedef struct {
    const eko_spec *sp;
    const double *X; const int64_t *off; const int64_t *len;
    long n;
    double *D; int64_t *cells;
    long next;
    pthread_mutex_t mu;
    int err;
} pw_job;

static void *pw_worker(void *arg) {
    pw_job *jb = (pw_job *)arg;
    eko_ws ws = {0};
    long i;
    while ((i = take(&jb->next, &jb->mu, jb->n)) >= 0) {
        int64_t rc = 0;
        jb->D[i * jb->n + i] = 0.0;
        for (long j = i + 1; j < jb->n; j++) {
            int64_t cc = 0;
            double d = facade(jb->sp, jb->X + jb->off[i], jb->len[i], jb->X + jb->off[j], jb->len[j],
                              EKO_INF, &ws, &cc);
            if (cc < 0) { jb->err = -2; break; }
            rc += cc;
            jb->D[i * jb->n + j] = d;
            jb->D[j * jb->n + i] = d;
        }
        jb->cells[i] = rc;
    }
    ws_free(&ws);
    return NULL;
}

/* all-pairs matrix: distance(spec, variant, X[i], X[j]) for i<j, mirrored, diagonal 0.0
 * (the loop of SURVEY.md 3.4; d(a,b)==d(b,a) bit-exactly per SURVEY Appendix A probe 4) */
int eko_pairwise(const eko_spec *sp, const double *X, const int64_t *off, const int64_t *len, long n,
                 int nthreads, double *D, int64_t *cells_per_row) {
    pw_job jb = {sp, X, off, len, n, D, cells_per_row, 0, PTHREAD_MUTEX_INITIALIZER, 0};
    run_threads(pw_worker, &jb, nthreads);
    return jb.err;
}

/* numpy's float64 add.reduce order for a contiguous 1-D array: 8 accumulators,
 * blocks of 128, recursive halving at multiples of 8 (numpy pairwise_sum). */
static double np_pairwise_sum(const double *a, long n) {
    if (n < 8) {
        double res = 0.0;
        for (long i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int k = 0; k < 8; k++) r[k] = a[k];
        long i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int k = 0; k < 8; k++) r[k] += a[i + k];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

double eko_np_sum(const double *a, long n) { return np_pairwise_sum(a, n); }

/* series.znormalize (series.py:118-131) with numpy's mean/std arithmetic */
int eko_znormalize(const double *s, long n, double *out, double *tmp) {
    if (n < 2) return -1;
    double mean = np_pairwise_sum(s, n) / (double)n;
    for (long k = 0; k < n; k++) { double d = s[k] - mean; tmp[k] = d * d; }
    double sd = sqrt(np_pairwise_sum(tmp, n) / (double)n);
    if (sd < 1e-12) { for (long k = 0; k < n; k++) out[k] = 0.0; return 0; }
    for (long k = 0; k < n; k++) out[k] = (s[k] - mean) / sd;
    return 0;
}

typedef struct {
    const eko_spec *sp;
    const double *q; long lq;
    const double *ref; long nref;
    int normalize;
    long chunk, nchunks;
    int64_t *best_off; double *best_d; int64_t *cells;
    long next;
    pthread_mutex_t mu;
    int err;
} ss_job;

static void *ss_worker(void *arg) {
    ss_job *jb = (ss_job *)arg;
    eko_ws ws = {0};
    double *win = (double *)malloc(sizeof(double) * (size_t)jb->lq);
    double *tmp = (double *)malloc(sizeof(double) * (size_t)jb->lq);
    long k;
    long nwin = jb->nref - jb->lq + 1;
    while ((k = take(&jb->next, &jb->mu, jb->nchunks)) >= 0) {
        long o0 = k * jb->chunk, o1 = o0 + jb->chunk < nwin ? o0 + jb->chunk : nwin;
        double bd = EKO_INF;
        int64_t bo = -1, cells = 0;
        /* subsequence_search (search.py:191-213): per-offset scan, running cutoff */
        for (long o = o0; o < o1; o++) {
            const double *wv = jb->ref + o;
            if (jb->normalize) { eko_znormalize(wv, jb->lq, win, tmp); wv = win; }
            int64_t cc = 0;
            double d = facade(jb->sp, jb->q, jb->lq, wv, jb->lq, bd, &ws, &cc);
            cells += cc;
            if (!isinf(d) && d < bd) { bd = d; bo = o; }
        }
        jb->best_off[k] = bo; jb->best_d[k] = bd; jb->cells[k] = cells;
    }
    free(win); free(tmp);
    ws_free(&ws);
    return NULL;
}

/* Chunked subsequence scan: each chunk of offsets runs the reference's serial
 * scan with its own running cutoff; the caller merges chunks by the
 * lexicographic (distance, offset) minimum.  One chunk == the reference. */
int eko_subseq(const eko_spec *sp, const double *q_normed, long lq, const double *ref, long nref,
               int normalize, long chunk, int nthreads, int64_t *best_off, double *best_d,
               int64_t *cells) {
    if (lq > nref || chunk < 1) return -1;
    long nwin = nref - lq + 1;
    ss_job jb = {sp, q_normed, lq, ref, nref, normalize, chunk, (nwin + chunk - 1) / chunk,
                 best_off, best_d, cells, 0, PTHREAD_MUTEX_INITIALIZER, 0};
    run_threads(ss_worker, &jb, nthreads);
    return jb.err;
}
