/*
 * oracle/mrq_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what the MRQ query path computes
 * (arXiv 2411.06158, /root/reference/PAPER.md; citations "P:N" are its lines).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, table or constant with the
 * CUDA path in paper_2411_06158_b200/.
 *
 * Conventions:
 *   - every sum is a plain left-to-right loop  acc = acc + term  (no fma; the
 *     library is compiled with -O2 -ffp-contract=off, no fast-math);
 *   - per-vector values the index stores are rounded once to float32
 *     ("float32 data"; the paper stores them);
 *   - selections order by (value, id), all prune tests are strict '<'.
 *
 * Build-time inputs (mu, P, lambda, R, centroids, assignment) come from the
 * build file written by oracle/build.py (Alg.1 L1-L6).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (see DESIGN.md "oracle pins"); the absolute values of dis', bounds and
 * survivor counts are additionally "parity unpinned" by any printed paper
 * example (the paper prints none; SURVEY P-13).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ types */

typedef struct {
    int32_t N, D, d, k, W;          /* W = ceil(d/32) code words per vector      */
    const double *mu;               /* D        PCA mean                          */
    const double *P;                /* D x D    PCA rows, descending eigenvalue   */
    const double *lam;              /* D        eigenvalues sigma_i^2 (Eq.6)      */
    const double *R;                /* d x d    random rotation P_r, y = R t      */
    const double *C;                /* k x d    IVF centroids on the heads        */
    const uint32_t *assign;         /* N        cluster of each vector            */
    /* outputs of orc_encode (per vector id) */
    float *head;                    /* N x d      fp32(x_p[0:d])                  */
    float *tail;                    /* N x (D-d)  fp32(x_p[d:D])                  */
    float *xr2f;                    /* N          fp32(||x_r||^2)                 */
    uint32_t *code;                 /* N x W      sign bits of y = R (x_d - c)    */
    float *f1, *f2, *f3;            /* N          stored factors, see orc_encode  */
    int64_t *list_off;              /* k+1                                        */
    int64_t *list_ids;              /* N ids, ascending inside each list          */
    double *Rc;                     /* k x d   R c_j                              */
} orc_index;

typedef struct {
    int32_t K, nprobe;
    double eps0, m;
    int32_t mode;            /* 0 FULL, 1 STAGE1_ONLY, 2 EXACT, 3 NOCORR, 4 SEQ       */
    int32_t tau_schedule;    /* 0 TIGHT, 1 LOOSE                                      */
    int32_t seed_mult;       /* K' = seed_mult * K                                    */
    double resid_scale;      /* eps_r = (resid_scale * m) * sigma                     */
    int32_t Bq;              /* query bits; levels 0 .. 2^Bq - 1                      */
    int32_t est_kind;        /* 0 quantized query, 1 unquantized query r,
                                2 no quantization at all (exact <t, q_d - c>)         */
    int32_t seed_lists;      /* decision T: the seed pool spans >= seed_lists lists    */
} orc_params;

typedef struct {
    int64_t scanned, f1, f2, exact, s0, s1;
} orc_stats;

typedef struct {                 /* optional per-stage dumps (NULL = skip)             */
    double *qp, *qr2, *eps_r, *r0;          /* Q x D, Q, Q, Q x d                      */
    int32_t *probe; double *probe_qn2;      /* Q x np                                  */
    uint8_t *levels; double *qconst;        /* Q x np x d, Q x np x 5 (A,Bc,C0,g1,eb)  */
    double *tau0, *tau1;                    /* Q                                       */
    int64_t cap;                            /* per-query capacity of the lists below   */
    int64_t *scan_cnt, *scan_ids; double *scan_dis, *scan_lb1;
    int64_t *s0_cnt, *s0_ids; double *s0_exact;
    int64_t *s1_cnt, *s1_ids; double *s1_exact;
    int64_t *f1_cnt, *f1_ids; double *f1_diso;
    int64_t *f2_cnt, *f2_ids; double *f2_exact;
} orc_dump;

/* ------------------------------------------------------- L0: plain algebra */

/* <a, b> over n terms, left to right. */
static double dot(const double *a, const double *b, int n)
{
    double acc = 0.0;
    for (int i = 0; i < n; i++) acc = acc + a[i] * b[i];
    return acc;
}

/* ------------------------------------------- L1: RaBitQ-style head encoder */

/*
 * Encode one head residual t = x_d - c (length d).  Alg.1 L7-L8,
 * RaBitQ codebook {+-1/sqrt(d)}^d under the random rotation (read with
 * d in place of D, SURVEY A-3): y = R t, bit_j = [y_j >= 0] (sign(0) -> 1),
 * <x_bar, x_b> = sum_j |y_j| / (sqrt(d) ||t||)  (A-22: d-dim head).
 * Degenerate t = 0: u = 1 and all bits 1 (SURVEY A-23).
 * Returns u = <x_bar, x_b>; writes ||t||^2 to *nrm2.
 */
double orc_encode_head(int d, const double *R, const double *t, uint32_t *code, double *nrm2)
{
    int W = (d + 31) / 32;
    double n2 = 0.0;
    for (int i = 0; i < d; i++) n2 = n2 + t[i] * t[i];
    for (int w = 0; w < W; w++) code[w] = 0u;
    double abssum = 0.0;
    for (int j = 0; j < d; j++) {
        double y = dot(R + (size_t)j * d, t, d);
        if (y >= 0.0) code[j / 32] |= 1u << (j % 32);
        abssum = abssum + fabs(y);
    }
    *nrm2 = n2;
    if (n2 == 0.0) return 1.0;
    double u = abssum / (sqrt((double)d) * sqrt(n2));
    if (u > 1.0) u = 1.0;
    return u;
}

/*
 * Alg.1 L3-L8 for every vector.
 *   x_p = P (x - mu)                     (L3; centred PCA rotation, A-16)
 *   ||x_r||^2 = sum_{i>=d} x_p,i^2       (L4; squared, A-24)
 *   t = x_d - c_{a(x)}                   (L5-L7; own IVF centroid, A-14)
 *   code, u = <x_bar, x_b>               (L7-L8)
 * stored factors (Eq.4 P:245-250 with the ||q_d - c|| factor restored, A-1;
 * Eq.5 P:255 with <x_bar,x> and sqrt(d-1), A-2):
 *   f1 = fp32(||t||^2 + ||x_r||^2)       norm part of C1 that belongs to x
 *   f2 = fp32(||t|| / u)                 scale of the quantized cross term C2
 *   f3 = fp32(||t|| sqrt(1-u^2) / (u sqrt(d-1)))   Eq.5 radical times ||t||
 * Also builds the inverted lists (ids ascending, A-28) and R c_j.
 * orc_encode_subset: only the vectors of the lists with only[c] != 0 (a
 * search that probes only those lists reads nothing else; the full-size GPU
 * parity tests encode just the lists their sampled queries probe).
 */
void orc_encode_subset(orc_index *ix, const float *X, const uint8_t *only)
{
    const int N = ix->N, D = ix->D, d = ix->d, k = ix->k, W = ix->W;
    const double sqd1 = sqrt((double)(d - 1));
    #pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) {
        if (only && !only[ix->assign[n]]) continue;   /* a list no search will probe: left unencoded */
        double *u = (double *)malloc(sizeof(double) * D);
        double *xp = (double *)malloc(sizeof(double) * D);
        double *t = (double *)malloc(sizeof(double) * d);
        const float *x = X + (size_t)n * D;
        for (int j = 0; j < D; j++) u[j] = (double)x[j] - ix->mu[j];
        for (int i = 0; i < D; i++) xp[i] = dot(ix->P + (size_t)i * D, u, D);
        double xr2 = 0.0;
        for (int i = d; i < D; i++) xr2 = xr2 + xp[i] * xp[i];
        const double *c = ix->C + (size_t)ix->assign[n] * d;
        for (int i = 0; i < d; i++) t[i] = xp[i] - c[i];
        double nrm2;
        double uu = orc_encode_head(d, ix->R, t, ix->code + (size_t)n * W, &nrm2);
        double nrm = sqrt(nrm2);
        for (int i = 0; i < d; i++) ix->head[(size_t)n * d + i] = (float)xp[i];
        for (int i = d; i < D; i++) ix->tail[(size_t)n * (D - d) + (i - d)] = (float)xp[i];
        ix->xr2f[n] = (float)xr2;
        ix->f1[n] = (float)(nrm2 + xr2);
        ix->f2[n] = (float)(nrm / uu);
        ix->f3[n] = (float)(nrm * (sqrt(1.0 - uu * uu) / (uu * sqd1)));
        free(u); free(xp); free(t);
    }
    /* inverted lists: counting sort by cluster, ids ascending */
    for (int c = 0; c <= k; c++) ix->list_off[c] = 0;
    for (int64_t n = 0; n < N; n++) ix->list_off[ix->assign[n] + 1]++;
    for (int c = 0; c < k; c++) ix->list_off[c + 1] += ix->list_off[c];
    int64_t *fill = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    for (int64_t n = 0; n < N; n++) {
        uint32_t c = ix->assign[n];
        ix->list_ids[ix->list_off[c] + fill[c]++] = n;
    }
    free(fill);
    for (int c = 0; c < k; c++)
        for (int j = 0; j < d; j++)
            ix->Rc[(size_t)c * d + j] = dot(ix->R + (size_t)j * d, ix->C + (size_t)c * d, d);
}

void orc_encode(orc_index *ix, const float *X) { orc_encode_subset(ix, X, NULL); }

/* ------------------------------------------------ L1: query quantizer (A-12) */

/*
 * Uniform Bq-bit scalar quantization of the rotated head residual r (Alg.2 L5,
 * P:307; the paper gives no construction): lo = min r, hi = max r,
 * delta = (hi - lo) / (2^Bq - 1), L_j = clamp(floor((r_j - lo)/delta + 0.5)).
 * delta = 0 -> all levels 0.  Returns sum L_j.
 */
int64_t orc_quantize(int d, const double *r, int Bq, uint8_t *L, double *lo_out, double *delta_out)
{
    const int top = (1 << Bq) - 1;
    double lo = r[0], hi = r[0];
    for (int j = 1; j < d; j++) {
        if (r[j] < lo) lo = r[j];
        if (r[j] > hi) hi = r[j];
    }
    double delta = (hi - lo) / (double)top;
    int64_t sumL = 0;
    for (int j = 0; j < d; j++) {
        int v = 0;
        if (delta > 0.0) {
            double f = floor((r[j] - lo) / delta + 0.5);
            v = f < 0.0 ? 0 : (f > (double)top ? top : (int)f);
        }
        L[j] = (uint8_t)v;
        sumL += v;
    }
    *lo_out = lo;
    *delta_out = delta;
    return sumL;
}

/*
 * <x_hat, r_bar> where x_hat_j = (2 bit_j - 1)/sqrt(d) and r_bar_j = lo + delta L_j
 * (the RaBitQ inner product <x_bar_b, q_b> times ||q_d - c||).  With
 * pop = sum bit_j and S = sum_{bit_j = 1} L_j (plain loop) it equals
 *   ((2 lo pop + 2 delta S) - (d lo + delta sumL)) / sqrt(d).
 */
double orc_ip_quantized(int d, const uint32_t *code, const uint8_t *L,
                        double A, double Bc, double C0, double isd)
{
    int64_t pop = 0, S = 0;
    for (int j = 0; j < d; j++) {
        if ((code[j / 32] >> (j % 32)) & 1u) { pop += 1; S += L[j]; }
    }
    double t1 = A * (double)pop;
    double t2 = Bc * (double)S;
    double t4 = (t1 + t2) - C0;
    return t4 * isd;
}

/* <x_hat, r> without query quantization (est_kind 1). */
double orc_ip_unquantized(int d, const uint32_t *code, const double *r, double isd)
{
    double acc = 0.0;
    for (int j = 0; j < d; j++) {
        double s = ((code[j / 32] >> (j % 32)) & 1u) ? r[j] : -r[j];
        acc = acc + s;
    }
    return acc * isd;
}

/* ------------------------------------------------------ L2/L4: query side */

/*
 * Alg.2 L1-L4: q_p = P (q - mu), split at d, ||q_r||^2,
 * sigma^2 = sum_{i>=d} q_i^2 lambda_i (Eq.6; A-16/A-17),
 * eps_r = (resid_scale m) sigma (Alg.2 L11 P:313 with the distance-domain
 * factor 2 of A-5 when resid_scale = 2), r0 = R q_d.
 */
void orc_prepare_query(const orc_index *ix, const float *q, double rscale, double m,
                       double *qp, double *qr2, double *eps_r, double *r0)
{
    const int D = ix->D, d = ix->d;
    double *u = (double *)malloc(sizeof(double) * D);
    for (int j = 0; j < D; j++) u[j] = (double)q[j] - ix->mu[j];
    for (int i = 0; i < D; i++) qp[i] = dot(ix->P + (size_t)i * D, u, D);
    double a = 0.0, s2 = 0.0;
    for (int i = d; i < D; i++) {
        a = a + qp[i] * qp[i];
        s2 = s2 + (qp[i] * qp[i]) * ix->lam[i];
    }
    *qr2 = a;
    *eps_r = (rscale * m) * sqrt(s2);
    for (int j = 0; j < d; j++) r0[j] = dot(ix->R + (size_t)j * d, qp, d);
    free(u);
}

/* ||x_p - q_p||^2 over i = 0..n-1 (left to right). n = d gives HEAD, n = D exact. */
static double exact_partial(const orc_index *ix, int64_t id, const double *qp, int n)
{
    const int D = ix->D, d = ix->d;
    double acc = 0.0;
    for (int i = 0; i < n; i++) {
        double x = i < d ? (double)ix->head[(size_t)id * d + i]
                         : (double)ix->tail[(size_t)id * (D - d) + (i - d)];
        double t = x - qp[i];
        acc = acc + t * t;
    }
    return acc;
}

/* ------------------------------------------------------------- selections */

typedef struct { double v; int64_t id; int32_t slot; } vi_t;

static int cmp_vi(const void *a, const void *b)
{
    const vi_t *x = (const vi_t *)a, *y = (const vi_t *)b;
    if (x->v < y->v) return -1;
    if (x->v > y->v) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* --------------------------------------------------------------- search */

typedef struct {
    int64_t id; int32_t p;
    double dis, lb1, diso, exact;
    int have_head, have_exact, in_f1;
} cand_t;

static double cand_exact(const orc_index *ix, cand_t *c, const double *qp, orc_stats *st)
{
    if (!c->have_exact) {
        c->exact = exact_partial(ix, c->id, qp, ix->D);
        c->have_exact = 1;
        st->exact++;
    }
    return c->exact;
}

/* K-th smallest exact over the distinct candidates in idx[0..n) (+inf if < K). */
static double kth_exact(cand_t *cs, const int32_t *idx, int n, int K)
{
    if (n < K) return INFINITY;
    vi_t *v = (vi_t *)malloc(sizeof(vi_t) * (size_t)n);
    for (int i = 0; i < n; i++) { v[i].v = cs[idx[i]].exact; v[i].id = cs[idx[i]].id; }
    qsort(v, (size_t)n, sizeof(vi_t), cmp_vi);
    double r = v[K - 1].v;
    free(v);
    return r;
}

#define MAXDUMP(dmp, field) ((dmp) && (dmp)->field)

/*
 * Search one query.  Probe (Alg.2 L7): top-nprobe centroids by
 * (||q_d - c_j||^2, j).  Per probed list (Alg.2 L4-L5 per (q, list), A-27):
 * r = R q_d - R c_j, quantized.  Per candidate (Alg.2 L8-L12):
 *   dis' = (f1 + g1) - 2 f2 <x_hat, r_bar>,  g1 = ||q_d - c||^2 + ||q_r||^2
 *   eps_b = eb f3,  eb = 2 eps0 ||q_d - c||    (A-6)
 *   LB1 = (dis' - eps_b) - eps_r
 * Stage 2 (Alg.2 L13 P:315, "Optimization" P:327, A-7):
 *   dis_o' = (HEAD + ||x_r||^2) + ||q_r||^2,  HEAD = ||x_d - q_d||^2.
 * Exact (Alg.2 L14 P:316, A-8): ||x_p - q_p||^2.
 * Threshold tau (Alg.2 L9 P:311): SEQ mode follows it literally (+inf until
 * the queue holds K, A-9); FULL uses decision T.
 */
static void search_one(const orc_index *ix, const float *q, const orc_params *pr, int64_t qi,
                       int64_t *out_ids, float *out_dist, orc_stats *st, orc_dump *dp)
{
    const int D = ix->D, d = ix->d, k = ix->k;
    const int K = pr->K, np = pr->nprobe < k ? pr->nprobe : k;
    const int Kp = pr->seed_mult * K;
    const double isd = 1.0 / sqrt((double)d);
    double *qp = (double *)malloc(sizeof(double) * D);
    double *r0 = (double *)malloc(sizeof(double) * d);
    double *r = (double *)malloc(sizeof(double) * d);
    uint8_t *L = (uint8_t *)malloc((size_t)d);
    double qr2, eps_r;
    orc_prepare_query(ix, q, pr->resid_scale, pr->m, qp, &qr2, &eps_r, r0);
    if (dp) {
        if (dp->qp) memcpy(dp->qp + qi * D, qp, sizeof(double) * D);
        if (dp->qr2) dp->qr2[qi] = qr2;
        if (dp->eps_r) dp->eps_r[qi] = eps_r;
        if (dp->r0) memcpy(dp->r0 + qi * d, r0, sizeof(double) * d);
    }

    /* probe: all k distances, sort by (qn2, j) */
    vi_t *cd = (vi_t *)malloc(sizeof(vi_t) * (size_t)k);
    for (int j = 0; j < k; j++) {
        const double *c = ix->C + (size_t)j * d;
        double acc = 0.0;
        for (int i = 0; i < d; i++) { double t = qp[i] - c[i]; acc = acc + t * t; }
        cd[j].v = acc; cd[j].id = j;
    }
    qsort(cd, (size_t)k, sizeof(vi_t), cmp_vi);

    /* gather candidates in probe order */
    int64_t ncand = 0;
    for (int p = 0; p < np; p++) ncand += ix->list_off[cd[p].id + 1] - ix->list_off[cd[p].id];
    cand_t *cs = (cand_t *)calloc((size_t)(ncand > 0 ? ncand : 1), sizeof(cand_t));
    int32_t *listend = (int32_t *)malloc(sizeof(int32_t) * (size_t)np);
    int64_t nc = 0;
    for (int p = 0; p < np; p++) {
        int j = (int)cd[p].id;
        double qn2 = cd[p].v;
        const double *c = ix->C + (size_t)j * d;
        for (int i = 0; i < d; i++) r[i] = r0[i] - ix->Rc[(size_t)j * d + i];
        double lo, delta;
        int64_t sumL = orc_quantize(d, r, pr->Bq, L, &lo, &delta);
        double A = 2.0 * lo, Bc = 2.0 * delta;
        double C0 = (double)d * lo + delta * (double)sumL;
        double g1 = qn2 + qr2;
        double eb = (2.0 * pr->eps0) * sqrt(qn2);
        if (dp) {
            if (dp->probe) dp->probe[qi * np + p] = j;
            if (dp->probe_qn2) dp->probe_qn2[qi * np + p] = qn2;
            if (dp->levels) memcpy(dp->levels + ((size_t)qi * np + p) * d, L, (size_t)d);
            if (dp->qconst) {
                double *o = dp->qconst + ((size_t)qi * np + p) * 5;
                o[0] = A; o[1] = Bc; o[2] = C0; o[3] = g1; o[4] = eb;
            }
        }
        for (int64_t s = ix->list_off[j]; s < ix->list_off[j + 1]; s++) {
            int64_t id = ix->list_ids[s];
            const uint32_t *code = ix->code + (size_t)id * ix->W;
            double t6;
            if (pr->est_kind == 2) {
                /* no quantization at all: the cross term is <t, q_d - c> itself
                   (Eq.2), so dis' reduces to Eq.3 without C3 */
                double acc = 0.0;
                for (int i = 0; i < d; i++) {
                    double ti = (double)ix->head[(size_t)id * d + i] - c[i];
                    acc = acc + ti * (qp[i] - c[i]);
                }
                t6 = acc;
            } else {
                double ip = pr->est_kind == 0 ? orc_ip_quantized(d, code, L, A, Bc, C0, isd)
                                              : orc_ip_unquantized(d, code, r, isd);
                t6 = (double)ix->f2[id] * ip;
            }
            double t5 = (double)ix->f1[id] + g1;
            double dis = t5 - 2.0 * t6;
            double lb1 = (dis - eb * (double)ix->f3[id]) - eps_r;
            cs[nc].id = id; cs[nc].p = p; cs[nc].dis = dis; cs[nc].lb1 = lb1;
            nc++;
        }
        listend[p] = (int32_t)nc;
    }
    st->scanned += nc;
    if (dp && dp->scan_cnt) {
        dp->scan_cnt[qi] = nc;
        for (int64_t i = 0; i < nc && i < dp->cap; i++) {
            if (dp->scan_ids) dp->scan_ids[qi * dp->cap + i] = cs[i].id;
            if (dp->scan_dis) dp->scan_dis[qi * dp->cap + i] = cs[i].dis;
            if (dp->scan_lb1) dp->scan_lb1[qi * dp->cap + i] = cs[i].lb1;
        }
    }

    vi_t *res = (vi_t *)malloc(sizeof(vi_t) * (size_t)(nc > 0 ? nc : 1));
    int nres = 0;
    double tau0 = INFINITY, tau1 = INFINITY;

    if (pr->mode == 2) {                         /* EXACT: IVF*-restricted exact top-K */
        for (int64_t i = 0; i < nc; i++) {
            res[nres].v = cand_exact(ix, &cs[i], qp, st); res[nres].id = cs[i].id; nres++;
        }
    } else if (pr->mode == 3) {                  /* NOCORR: rank by dis' only        */
        for (int64_t i = 0; i < nc; i++) { res[nres].v = cs[i].dis; res[nres].id = cs[i].id; nres++; }
    } else if (pr->mode == 4) {                  /* SEQ: Alg.2 literally             */
        /* result queue: K smallest (exact, id); tau = its max when full, else +inf */
        vi_t *heap = (vi_t *)malloc(sizeof(vi_t) * (size_t)(K + 1));
        int hn = 0;
        for (int64_t i = 0; i < nc; i++) {
            double tau = (hn == K) ? heap[K - 1].v : INFINITY;            /* L9  */
            if (cs[i].lb1 < tau) {                                          /* L12 */
                st->f1++;
                double head = exact_partial(ix, cs[i].id, qp, d);
                double diso = (head + (double)ix->xr2f[cs[i].id]) + qr2;
                if (diso - eps_r < tau) {                                   /* L13 */
                    st->f2++;
                    double ex = cand_exact(ix, &cs[i], qp, st);             /* L14 */
                    vi_t nv = {ex, cs[i].id, 0};                            /* L15 */
                    if (hn < K || cmp_vi(&nv, &heap[K - 1]) < 0) {
                        int pos = hn < K ? hn++ : K - 1;
                        while (pos > 0 && cmp_vi(&nv, &heap[pos - 1]) < 0) { heap[pos] = heap[pos - 1]; pos--; }
                        heap[pos] = nv;
                    }
                }
            }
        }
        for (int i = 0; i < hn; i++) res[nres++] = heap[i];
        free(heap);
    } else {                                     /* FULL / STAGE1_ONLY: decision T   */
        /* seeds: first lists in probe order holding >= K' candidates */
        int64_t pool = 0;
        const int sl = pr->seed_lists > 0 ? pr->seed_lists : 1;
        for (int p = 0; p < np; p++) { pool = listend[p]; if (pool >= Kp && p + 1 >= sl) break; }
        vi_t *sv = (vi_t *)malloc(sizeof(vi_t) * (size_t)(pool > 0 ? pool : 1));
        for (int64_t i = 0; i < pool; i++) { sv[i].v = cs[i].dis; sv[i].id = cs[i].id; sv[i].slot = (int32_t)i; }
        qsort(sv, (size_t)pool, sizeof(vi_t), cmp_vi);
        int ns0 = (int)(pool < Kp ? pool : Kp);
        int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * Kp + 1));
        for (int i = 0; i < ns0; i++) { sel[i] = sv[i].slot; cand_exact(ix, &cs[sel[i]], qp, st); }
        free(sv);
        tau0 = kth_exact(cs, sel, ns0, K);
        st->s0 += ns0;
        if (dp && dp->s0_cnt) {
            dp->s0_cnt[qi] = ns0;
            for (int i = 0; i < ns0 && i < dp->cap; i++) {
                if (dp->s0_ids) dp->s0_ids[qi * dp->cap + i] = cs[sel[i]].id;
                if (dp->s0_exact) dp->s0_exact[qi * dp->cap + i] = cs[sel[i]].exact;
            }
        }
        /* stage 1: F1 = {LB1 < tau0} */
        int64_t nf1 = 0;
        for (int64_t i = 0; i < nc; i++) if (cs[i].lb1 < tau0) { cs[i].in_f1 = 1; nf1++; }
        st->f1 += nf1;
        int nsel = ns0;
        if (pr->mode == 1) {
            tau1 = tau0;
        } else {
            for (int64_t i = 0; i < nc; i++) if (cs[i].in_f1) {
                double head = exact_partial(ix, cs[i].id, qp, d);
                cs[i].diso = (head + (double)ix->xr2f[cs[i].id]) + qr2;
                cs[i].have_head = 1;
            }
            if (pr->tau_schedule == 0) {           /* TIGHT: S1 = K' smallest (dis_o', id) in F1 */
                vi_t *fv = (vi_t *)malloc(sizeof(vi_t) * (size_t)(nf1 > 0 ? nf1 : 1));
                int64_t m = 0;
                for (int64_t i = 0; i < nc; i++) if (cs[i].in_f1) { fv[m].v = cs[i].diso; fv[m].id = cs[i].id; fv[m].slot = (int32_t)i; m++; }
                qsort(fv, (size_t)m, sizeof(vi_t), cmp_vi);
                int ns1 = (int)(m < Kp ? m : Kp);
                if (dp && dp->s1_cnt) dp->s1_cnt[qi] = ns1;
                for (int i = 0; i < ns1; i++) {
                    int32_t s = fv[i].slot;
                    cand_exact(ix, &cs[s], qp, st);
                    if (dp && dp->s1_ids && i < dp->cap) dp->s1_ids[qi * dp->cap + i] = cs[s].id;
                    if (dp && dp->s1_exact && i < dp->cap) dp->s1_exact[qi * dp->cap + i] = cs[s].exact;
                    int dup = 0;
                    for (int t = 0; t < nsel; t++) if (sel[t] == s) { dup = 1; break; }
                    if (!dup) sel[nsel++] = s;
                }
                st->s1 += ns1;
                free(fv);
                tau1 = kth_exact(cs, sel, nsel, K);
            } else {
                tau1 = tau0;
                if (dp && dp->s1_cnt) dp->s1_cnt[qi] = 0;
            }
        }
        /* stage 2: F2 = {c in F1 : dis_o' - eps_r < tau1}; exact on F2 */
        int64_t nf2 = 0;
        for (int64_t i = 0; i < nc; i++) {
            if (!cs[i].in_f1) continue;
            int pass = (pr->mode == 1) ? 1 : (cs[i].diso - eps_r < tau1);
            if (pass) {
                cand_exact(ix, &cs[i], qp, st);
                if (dp && dp->f2_ids && nf2 < dp->cap) {
                    dp->f2_ids[qi * dp->cap + nf2] = cs[i].id;
                    if (dp->f2_exact) dp->f2_exact[qi * dp->cap + nf2] = cs[i].exact;
                }
                nf2++;
            }
        }
        st->f2 += nf2;
        if (dp && dp->f2_cnt) dp->f2_cnt[qi] = nf2;
        if (dp && dp->f1_cnt) {
            int64_t m = 0;
            for (int64_t i = 0; i < nc; i++) if (cs[i].in_f1) {
                if (m < dp->cap) {
                    if (dp->f1_ids) dp->f1_ids[qi * dp->cap + m] = cs[i].id;
                    if (dp->f1_diso) dp->f1_diso[qi * dp->cap + m] = cs[i].have_head ? cs[i].diso : NAN;
                }
                m++;
            }
            dp->f1_cnt[qi] = m;
        }
        /* result: K smallest (exact, id) over F2 u S0 u S1 (distinct ids) */
        for (int64_t i = 0; i < nc; i++) {
            int inres = 0;
            if (cs[i].in_f1 && ((pr->mode == 1) || (cs[i].diso - eps_r < tau1))) inres = 1;
            for (int t = 0; t < nsel && !inres; t++) if (sel[t] == i) inres = 1;
            if (inres) { res[nres].v = cs[i].exact; res[nres].id = cs[i].id; nres++; }
        }
        free(sel);
    }
    if (dp) {
        if (dp->tau0) dp->tau0[qi] = tau0;
        if (dp->tau1) dp->tau1[qi] = tau1;
    }
    qsort(res, (size_t)nres, sizeof(vi_t), cmp_vi);
    for (int i = 0; i < K; i++) {
        if (i < nres) { out_ids[qi * K + i] = res[i].id; out_dist[qi * K + i] = (float)res[i].v; }
        else { out_ids[qi * K + i] = -1; out_dist[qi * K + i] = INFINITY; }
    }
    free(res); free(cs); free(listend); free(cd); free(qp); free(r0); free(r); free(L);
}

int orc_search(const orc_index *ix, int64_t nq, const float *queries, const orc_params *pr,
               int64_t *out_ids, float *out_dist, orc_stats *st, orc_dump *dp)
{
    if (pr->K < 1 || pr->nprobe < 1 || pr->Bq < 1 || pr->Bq > 8 || ix->d < 2) return -1;
    orc_stats tot = {0, 0, 0, 0, 0, 0};
    #pragma omp parallel
    {
        orc_stats loc = {0, 0, 0, 0, 0, 0};
        #pragma omp for schedule(dynamic, 1)
        for (int64_t qi = 0; qi < nq; qi++)
            search_one(ix, queries + (size_t)qi * ix->D, pr, qi, out_ids, out_dist, &loc, dp);
        #pragma omp critical
        {
            tot.scanned += loc.scanned; tot.f1 += loc.f1; tot.f2 += loc.f2;
            tot.exact += loc.exact; tot.s0 += loc.s0; tot.s1 += loc.s1;
        }
    }
    if (st) *st = tot;
    return 0;
}

/*
 * Brute-force exact KNN in the original space: K smallest
 * (||x - q||^2, id), fp64, plain loops.  Ground truth for recall.
 */
void orc_bruteforce(int64_t N, int32_t D, const float *X, int64_t nq, const float *Qv, int32_t K,
                    int64_t *out_ids, double *out_dist)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < nq; qi++) {
        vi_t *best = (vi_t *)malloc(sizeof(vi_t) * (size_t)(K + 1));
        int hn = 0;
        const float *q = Qv + (size_t)qi * D;
        for (int64_t n = 0; n < N; n++) {
            const float *x = X + (size_t)n * D;
            double acc = 0.0;
            for (int i = 0; i < D; i++) { double t = (double)x[i] - (double)q[i]; acc = acc + t * t; }
            vi_t nv = {acc, n, 0};
            if (hn < K || cmp_vi(&nv, &best[K - 1]) < 0) {
                int pos = hn < K ? hn++ : K - 1;
                while (pos > 0 && cmp_vi(&nv, &best[pos - 1]) < 0) { best[pos] = best[pos - 1]; pos--; }
                best[pos] = nv;
            }
        }
        for (int i = 0; i < K; i++) {
            out_ids[qi * K + i] = i < hn ? best[i].id : -1;
            out_dist[qi * K + i] = i < hn ? best[i].v : INFINITY;
        }
        free(best);
    }
}

/* Exact squared distance of a candidate list (used for ground-truth rescoring). */
void orc_exact_original(int32_t D, const float *X, const float *q, int64_t n, const int64_t *ids, double *out)
{
    for (int64_t i = 0; i < n; i++) {
        const float *x = X + (size_t)ids[i] * D;
        double acc = 0.0;
        for (int j = 0; j < D; j++) { double t = (double)x[j] - (double)q[j]; acc = acc + t * t; }
        out[i] = acc;
    }
}
