/*
 * tmfg_oracle.c -- CPU restatement of the reference tmfgclust hot path.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / `--impl reference` legs may load this library,
 * and only as the checker / the timed CPU baseline.  The product library
 * (paper_2408_09399_b200/_lib/libtmfg_b200.so) never links or calls it.
 *
 * Every function restates one reference routine; the citation is
 * /root/reference/pkg/src/tmfgclust/<file>:<lines>.  Arithmetic follows the
 * reference operation for operation (compile with -ffp-contract=off so no
 * FMA contraction changes a rounding):
 *   - pearson: sequential k-order mul+add, exactly like the numba loop
 *     (verified bit-identical to _kernels.pearson_kernel);
 *   - Dijkstra / truncated Dijkstra: lazy-deletion binary heap;
 *   - heap TMFG: binary heap keyed (-gain, fid) like heapq over tuples.
 * Parity of this file with the reference is pinned by tests/golden/ (fixtures
 * produced by importing the reference itself, see tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

EXPORT int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

EXPORT void orc_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------------------ */
/* a1  _kernels.py:17-37  pearson_kernel(xc, inv_norm, out)                  */
/* ------------------------------------------------------------------------ */
EXPORT void orc_pearson(const double *xc, const double *inv, int64_t n, int64_t L, double *out) {
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < n; i++) {
        out[i * n + i] = 1.0;
        for (int64_t j = i + 1; j < n; j++) {
            double r;
            if (inv[i] == 0.0 || inv[j] == 0.0) {
                r = 0.0;
            } else {
                double s = 0.0;
                const double *xi = xc + i * L, *xj = xc + j * L;
                for (int64_t k = 0; k < L; k++) s += xi[k] * xj[k];
                r = s * inv[i] * inv[j];
                if (r > 1.0) r = 1.0;
                else if (r < -1.0) r = -1.0;
            }
            out[i * n + j] = r;
            out[j * n + i] = r;
        }
    }
}

/* numpy's pairwise summation (the float64 add.reduce inner loop), used by
 * tmfg.py:76 `S.sum(axis=1)`.  Block size 128, 8-way unroll. */
static double pairwise_sum(const double *a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
    }
}

/* a4  tmfg.py:71-79  select_initial_clique: row sums minus diagonal, stable
 * top-4 by (sum desc, id asc), returned ascending. */
EXPORT void orc_initial_clique(const double *S, int64_t n, int32_t *clique) {
    double *sums = (double *)malloc(sizeof(double) * n);
#pragma omp parallel for
    for (int64_t i = 0; i < n; i++) sums[i] = pairwise_sum(S + i * n, n) - S[i * n + i];
    int32_t top[4];
    for (int k = 0; k < 4; k++) {
        int64_t best = -1;
        for (int64_t i = 0; i < n; i++) {
            int used = 0;
            for (int q = 0; q < k; q++) used |= (top[q] == i);
            if (used) continue;
            /* argsort(-sums, stable): smaller -sum first, NaN last, ties lower id */
            if (best < 0) { best = i; continue; }
            double ki = -sums[i], kb = -sums[best];
            if ((isnan(kb) && !isnan(ki)) || ki < kb) best = i;
        }
        top[k] = (int32_t)best;
    }
    /* sorted ascending */
    for (int a = 0; a < 4; a++)
        for (int b = a + 1; b < 4; b++)
            if (top[b] < top[a]) { int32_t t = top[a]; top[a] = top[b]; top[b] = t; }
    memcpy(clique, top, sizeof(top));
    free(sums);
}

/* ------------------------------------------------------------------------ */
/* a3  simmatrix.py:225-249  sort_neighbor_lists: per row, ids ordered by     */
/* (S desc, id asc) -- argsort(-S[v]) with the lexsort((ids, -S[v])) rule for */
/* ties -- then v removed.  -0.0 == +0.0 (float compare); NaN sorts last.     */
/* ------------------------------------------------------------------------ */
static inline int key_before(double a, double b) {
    /* strict "a precedes b" on the value alone (descending) */
    if (isnan(a)) return 0;
    if (isnan(b)) return 1;
    return a > b;
}

static void merge_sort_idx(const double *row, int32_t *idx, int32_t *tmp, int64_t len) {
    /* bottom-up stable merge sort; stability keeps ascending-id ties */
    int32_t *src = idx, *dst = tmp;
    for (int64_t w = 1; w < len; w *= 2) {
        for (int64_t lo = 0; lo < len; lo += 2 * w) {
            int64_t mid = lo + w < len ? lo + w : len;
            int64_t hi = lo + 2 * w < len ? lo + 2 * w : len;
            int64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) {
                if (key_before(row[src[j]], row[src[i]])) dst[k++] = src[j++];
                else dst[k++] = src[i++];
            }
            while (i < mid) dst[k++] = src[i++];
            while (j < hi) dst[k++] = src[j++];
        }
        int32_t *t = src; src = dst; dst = t;
    }
    if (src != idx) memcpy(idx, src, sizeof(int32_t) * len);
}

EXPORT void orc_sort_rows(const double *S, int64_t n, int32_t *order) {
#pragma omp parallel
    {
        int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (n > 1 ? n : 1));
        int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (n > 1 ? n : 1));
#pragma omp for schedule(dynamic, 16)
        for (int64_t v = 0; v < n; v++) {
            int64_t len = 0;
            for (int64_t u = 0; u < n; u++)
                if (u != v) idx[len++] = (int32_t)u;
            merge_sort_idx(S + v * n, idx, tmp, len);
            memcpy(order + v * (n - 1), idx, sizeof(int32_t) * len);
        }
        free(idx);
        free(tmp);
    }
}

/* ------------------------------------------------------------------------ */
/* a5-a8  tmfg.py:344-436  build_tmfg_heap                                    */
/* ------------------------------------------------------------------------ */
typedef struct { double negg; int32_t fid; int32_t u; } hentry;

/* heapq orders the tuples (-g, fid, u); fid is unique among live entries */
static inline int hless(const hentry *x, const hentry *y) {
    if (x->negg < y->negg) return 1;
    if (x->negg == y->negg) return x->fid < y->fid;
    return 0;
}

static void hpush(hentry *h, int64_t *sz, hentry e) {
    int64_t j = (*sz)++;
    h[j] = e;
    while (j > 0) {
        int64_t p = (j - 1) >> 1;
        if (!hless(&h[j], &h[p])) break;
        hentry t = h[p]; h[p] = h[j]; h[j] = t;
        j = p;
    }
}

static hentry hpop(hentry *h, int64_t *sz) {
    hentry top = h[0];
    (*sz)--;
    if (*sz > 0) {
        h[0] = h[*sz];
        int64_t i = 0;
        for (;;) {
            int64_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < *sz && hless(&h[l], &h[m])) m = l;
            if (r < *sz && hless(&h[r], &h[m])) m = r;
            if (m == i) break;
            hentry t = h[m]; h[m] = h[i]; h[i] = t;
            i = m;
        }
    }
    return top;
}

typedef struct {
    const double *S;
    const int32_t *order;
    int64_t n;
    int32_t *cursors;
    uint8_t *inserted;
    int32_t *max_corrs;
    int64_t rem;
    int32_t (*fv)[3]; /* face vertices, sorted */
    uint8_t *alive;
    int64_t nf;
} tstate;

/* tmfg.py:169-182 refresh_max_corr */
static int32_t refresh(tstate *st, int32_t v) {
    const int32_t *row = st->order + (int64_t)v * (st->n - 1);
    int32_t cur = st->cursors[v];
    while (st->inserted[row[cur]]) cur++;
    st->cursors[v] = cur;
    st->max_corrs[v] = row[cur];
    return row[cur];
}

/* tmfg.py:266-277 _best_candidate */
static hentry make_entry(tstate *st, int32_t fid) {
    int32_t a = st->fv[fid][0], b = st->fv[fid][1], c = st->fv[fid][2];
    const double *S = st->S;
    int64_t n = st->n;
    double best_g = -INFINITY;
    int32_t best_v = -1;
    int32_t cand[3] = {st->max_corrs[a], st->max_corrs[b], st->max_corrs[c]};
    for (int k = 0; k < 3; k++) {
        int32_t u = cand[k];
        double g = S[(int64_t)a * n + u] + S[(int64_t)b * n + u];
        g = g + S[(int64_t)c * n + u];
        if (g > best_g || (g == best_g && u < best_v)) { best_g = g; best_v = u; }
    }
    hentry e = {-best_g, fid, best_v};
    return e;
}

static void sort3(int32_t *t) {
    int32_t x;
    if (t[1] < t[0]) { x = t[0]; t[0] = t[1]; t[1] = x; }
    if (t[2] < t[1]) { x = t[1]; t[1] = t[2]; t[2] = x; }
    if (t[1] < t[0]) { x = t[0]; t[0] = t[1]; t[1] = x; }
}

static int32_t add_face(tstate *st, int32_t x, int32_t y, int32_t z) {
    int32_t fid = (int32_t)st->nf++;
    int32_t t[3] = {x, y, z};
    sort3(t);
    st->fv[fid][0] = t[0]; st->fv[fid][1] = t[1]; st->fv[fid][2] = t[2];
    st->alive[fid] = 1;
    return fid;
}

/*
 * Outputs (caller-allocated): trace (n-4)*4, host_fid (n-4), edges (3n-6)*2,
 * faces (2n-4)*3, stats[3] = {pops, refreshes, gain_increases}.
 * Returns the number of trace rows.
 */
EXPORT int64_t orc_tmfg_heap(const double *S, const int32_t *order, int64_t n, const int32_t *clique,
                             int32_t *trace, int32_t *host_fid, int32_t *edges, int32_t *faces,
                             int64_t *stats) {
    tstate st;
    st.S = S; st.order = order; st.n = n;
    st.cursors = (int32_t *)calloc(n, sizeof(int32_t));
    st.inserted = (uint8_t *)calloc(n, 1);
    st.max_corrs = (int32_t *)malloc(sizeof(int32_t) * n);
    for (int64_t i = 0; i < n; i++) st.max_corrs[i] = -1;
    st.rem = n;
    int64_t cap = 3 * n + 8;
    st.fv = (int32_t(*)[3])malloc(sizeof(int32_t) * 3 * cap);
    st.alive = (uint8_t *)calloc(cap, 1);
    st.nf = 0;
    int32_t a = clique[0], b = clique[1], c = clique[2], d = clique[3];
    /* tmfg.py:104-113 _GraphAccum.__init__ */
    int64_t ne = 0, nt = 0;
    int32_t e0[6][2] = {{a, b}, {a, c}, {a, d}, {b, c}, {b, d}, {c, d}};
    for (int k = 0; k < 6; k++) { edges[2 * ne] = e0[k][0]; edges[2 * ne + 1] = e0[k][1]; ne++; }
    add_face(&st, a, b, c); add_face(&st, a, b, d); add_face(&st, a, c, d); add_face(&st, b, c, d);
    for (int k = 0; k < 4; k++) { st.inserted[clique[k]] = 1; st.rem--; }
    if (st.rem)
        for (int k = 0; k < 4; k++) refresh(&st, clique[k]);
    int64_t pops = 0, refreshes = 0, gain_inc = 0;
    hentry *heap = (hentry *)malloc(sizeof(hentry) * cap);
    int64_t hs = 0;
    for (int32_t fid = 0; fid < 4; fid++)
        if (st.rem) hpush(heap, &hs, make_entry(&st, fid));
    while (st.rem) {
        hentry top = hpop(heap, &hs);
        pops++;
        int32_t fid = top.fid, v = top.u;
        int32_t fa = st.fv[fid][0], fb = st.fv[fid][1], fc = st.fv[fid][2];
        if (!st.inserted[v]) {
            /* tmfg.py:121-131 _GraphAccum.insert */
            trace[4 * nt] = v; trace[4 * nt + 1] = fa; trace[4 * nt + 2] = fb; trace[4 * nt + 3] = fc;
            host_fid[nt] = fid;
            nt++;
            int32_t w3[3] = {fa, fb, fc};
            for (int k = 0; k < 3; k++) {
                int32_t w = w3[k];
                edges[2 * ne] = w < v ? w : v;
                edges[2 * ne + 1] = w < v ? v : w;
                ne++;
            }
            st.alive[fid] = 0;
            int32_t f1 = add_face(&st, v, fa, fb);
            int32_t f2 = add_face(&st, v, fa, fc);
            int32_t f3 = add_face(&st, v, fb, fc);
            st.inserted[v] = 1;
            st.rem--;
            if (st.rem == 0) break;
            refresh(&st, v); refresh(&st, fa); refresh(&st, fb); refresh(&st, fc);
            hpush(heap, &hs, make_entry(&st, f1));
            hpush(heap, &hs, make_entry(&st, f2));
            hpush(heap, &hs, make_entry(&st, f3));
        } else {
            refresh(&st, fa); refresh(&st, fb); refresh(&st, fc);
            hentry e = make_entry(&st, fid);
            refreshes++;
            /* tmfg.py:427: -entry[0] > -neg_g + GAIN_EPS */
            if (-e.negg > -top.negg + 1e-12) gain_inc++;
            hpush(heap, &hs, e);
        }
    }
    /* tmfg.py:133-144 finalize: alive faces in creation order */
    int64_t k = 0;
    for (int64_t f = 0; f < st.nf; f++)
        if (st.alive[f]) {
            faces[3 * k] = st.fv[f][0]; faces[3 * k + 1] = st.fv[f][1]; faces[3 * k + 2] = st.fv[f][2];
            k++;
        }
    stats[0] = pops; stats[1] = refreshes; stats[2] = gain_inc;
    free(heap); free(st.cursors); free(st.inserted); free(st.max_corrs); free(st.fv); free(st.alive);
    return nt;
}

/* ------------------------------------------------------------------------ */
/* a10  _kernels.py:40-99  Dijkstra rows (binary heap, lazy deletion)          */
/* a11  _kernels.py:102-181 radius-truncated Dijkstra, count then fill        */
/* ------------------------------------------------------------------------ */
typedef struct { double d; int64_t v; } dentry;

static void dpush(dentry *h, int64_t *sz, double d, int64_t v) {
    int64_t j = (*sz)++;
    h[j].d = d; h[j].v = v;
    while (j > 0) {
        int64_t p = (j - 1) >> 1;
        if (h[p].d <= h[j].d) break;
        dentry t = h[p]; h[p] = h[j]; h[j] = t;
        j = p;
    }
}

static dentry dpop(dentry *h, int64_t *sz) {
    dentry top = h[0];
    (*sz)--;
    h[0] = h[*sz];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *sz && h[l].d < h[m].d) m = l;
        if (r < *sz && h[r].d < h[m].d) m = r;
        if (m == i) break;
        dentry t = h[m]; h[m] = h[i]; h[i] = t;
        i = m;
    }
    return top;
}

static void dijkstra_into(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n, int64_t src,
                          double *dist, uint8_t *done, dentry *heap) {
    for (int64_t i = 0; i < n; i++) { dist[i] = INFINITY; done[i] = 0; }
    int64_t sz = 0;
    dpush(heap, &sz, 0.0, src);
    dist[src] = 0.0;
    while (sz > 0) {
        dentry t = dpop(heap, &sz);
        if (done[t.v]) continue;
        done[t.v] = 1;
        for (int64_t e = indptr[t.v]; e < indptr[t.v + 1]; e++) {
            int64_t u = nbr[e];
            double nd = t.d + wt[e];
            if (nd < dist[u]) {
                dist[u] = nd;
                dpush(heap, &sz, nd, u);
            }
        }
    }
}

EXPORT void orc_dijkstra_rows(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n,
                              const int64_t *sources, int64_t ns, double *out) {
#pragma omp parallel
    {
        uint8_t *done = (uint8_t *)malloc(n);
        dentry *heap = (dentry *)malloc(sizeof(dentry) * (indptr[n] + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t s = 0; s < ns; s++) dijkstra_into(indptr, nbr, wt, n, sources[s], out + s * n, done, heap);
        free(done);
        free(heap);
    }
}

static int64_t truncated_into(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n, int64_t src,
                              double radius, int64_t *ids, double *dists, int64_t base, double *dist,
                              uint8_t *done, dentry *heap, int64_t *touched) {
    int64_t nt = 0;
    int64_t sz = 0;
    dpush(heap, &sz, 0.0, src);
    dist[src] = 0.0;
    touched[nt++] = src;
    int64_t cnt = 0;
    while (sz > 0) {
        dentry t = dpop(heap, &sz);
        if (t.d > radius) break;
        if (done[t.v]) continue;
        done[t.v] = 1;
        if (ids) { ids[base + cnt] = t.v; dists[base + cnt] = t.d; }
        cnt++;
        for (int64_t e = indptr[t.v]; e < indptr[t.v + 1]; e++) {
            int64_t u = nbr[e];
            double nd = t.d + wt[e];
            if (nd <= radius && nd < dist[u]) {
                if (isinf(dist[u])) touched[nt++] = u;
                dist[u] = nd;
                dpush(heap, &sz, nd, u);
            }
        }
    }
    for (int64_t i = 0; i < nt; i++) { dist[touched[i]] = INFINITY; done[touched[i]] = 0; }
    return cnt;
}

static void truncated_all(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n,
                          const double *radii, int64_t *counts, const int64_t *offsets, int64_t *ids,
                          double *dists) {
#pragma omp parallel
    {
        double *dist = (double *)malloc(sizeof(double) * n);
        uint8_t *done = (uint8_t *)calloc(n, 1);
        int64_t *touched = (int64_t *)malloc(sizeof(int64_t) * n);
        dentry *heap = (dentry *)malloc(sizeof(dentry) * (indptr[n] + 1));
        for (int64_t i = 0; i < n; i++) dist[i] = INFINITY;
#pragma omp for schedule(dynamic, 16)
        for (int64_t v = 0; v < n; v++) {
            int64_t c = truncated_into(indptr, nbr, wt, n, v, radii[v], ids, dists, offsets ? offsets[v] : 0,
                                       dist, done, heap, touched);
            if (counts) counts[v] = c;
        }
        free(dist); free(done); free(touched); free(heap);
    }
}

EXPORT void orc_truncated_counts(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n,
                                 const double *radii, int64_t *counts) {
    truncated_all(indptr, nbr, wt, n, radii, counts, NULL, NULL, NULL);
}

EXPORT void orc_truncated_fill(const int64_t *indptr, const int64_t *nbr, const double *wt, int64_t n,
                               const double *radii, const int64_t *offsets, int64_t *ids, double *dists) {
    truncated_all(indptr, nbr, wt, n, radii, NULL, offsets, ids, dists);
}

/* ------------------------------------------------------------------------ */
/* a16  _kernels.py:184-201  segment_pair_max (exact oracle group max)        */
/* ------------------------------------------------------------------------ */
EXPORT void orc_segment_pair_max(const double *D, int64_t n, const int64_t *perm, const int64_t *starts,
                                 int64_t m, double *out) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t idx = 0; idx < m * m; idx++) {
        int64_t i = idx / m, j = idx % m;
        if (j < i) continue;
        double best = (i == j) ? 0.0 : -INFINITY;
        for (int64_t a = starts[i]; a < starts[i + 1]; a++) {
            const double *row = D + perm[a] * n;
            for (int64_t b = starts[j]; b < starts[j + 1]; b++) {
                double d = row[perm[b]];
                if (d > best) best = d;
            }
        }
        out[i * m + j] = best;
        out[j * m + i] = best;
    }
}

/*
 * a12+a16  apsp.py:138-158 HubOracle.block followed by the two reduceat maxima
 * of dbht.py:228-230, restated without materialising the |perm|^2 block:
 *   est(u, v) = near_v(u) if u in near(v)        (column override wins)
 *             = near_u(v) elif v in near(u)      (row override)
 *             = min_h hd[h,u] + hd[h,v]          otherwise
 *   out[gi, gj] = max over u in group gi, v in group gj of est(u, v).
 * rev_* is the transposed near table (for each u: the (v, near_v(u)) with
 * u in near(v)); the wrapper builds it with numpy.
 */
EXPORT void orc_hub_group_max(const double *hub_dist, int64_t H, int64_t n, const int64_t *near_indptr,
                              const int64_t *near_ids, const double *near_dist, const int64_t *rev_indptr,
                              const int64_t *rev_ids, const double *rev_dist, const int64_t *perm,
                              const int64_t *starts, int64_t m, double *out) {
    int64_t P = starts[m];
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *grp = (int64_t *)malloc(sizeof(int64_t) * (P > 0 ? P : 1));
    for (int64_t i = 0; i < n; i++) pos[i] = -1;
    for (int64_t g = 0; g < m; g++)
        for (int64_t a = starts[g]; a < starts[g + 1]; a++) { pos[perm[a]] = a; grp[a] = g; }
    for (int64_t i = 0; i < m * m; i++) out[i] = -INFINITY;
    /* hub columns gathered in perm order: hp[h*P + b] = hd[h, perm[b]] */
    double *hp = (double *)malloc(sizeof(double) * H * (P > 0 ? P : 1));
    for (int64_t h = 0; h < H; h++)
        for (int64_t b = 0; b < P; b++) hp[h * P + b] = hub_dist[h * n + perm[b]];
#pragma omp parallel
    {
        double *est = (double *)malloc(sizeof(double) * (P > 0 ? P : 1));
        double *acc = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
#pragma omp for schedule(dynamic, 4)
        for (int64_t a = 0; a < P; a++) {
            int64_t u = perm[a];
            for (int64_t b = 0; b < P; b++) est[b] = INFINITY;
            for (int64_t h = 0; h < H; h++) {
                double du = hub_dist[h * n + u];
                const double *row = hp + h * P;
                for (int64_t b = 0; b < P; b++) {
                    double s = du + row[b];
                    if (s < est[b]) est[b] = s;
                }
            }
            for (int64_t e = near_indptr[u]; e < near_indptr[u + 1]; e++) {
                int64_t p = pos[near_ids[e]];
                if (p >= 0) est[p] = near_dist[e];
            }
            for (int64_t e = rev_indptr[u]; e < rev_indptr[u + 1]; e++) {
                int64_t p = pos[rev_ids[e]];
                if (p >= 0) est[p] = rev_dist[e];
            }
            for (int64_t g = 0; g < m; g++) acc[g] = -INFINITY;
            for (int64_t b = 0; b < P; b++)
                if (est[b] > acc[grp[b]]) acc[grp[b]] = est[b];
            int64_t gi = grp[a];
#pragma omp critical
            for (int64_t g = 0; g < m; g++)
                if (acc[g] > out[gi * m + g]) out[gi * m + g] = acc[g];
        }
        free(est);
        free(acc);
    }
    free(hp); free(pos); free(grp);
}

/* ------------------------------------------------------------------------ */
/* a17  linkage.py:50-94  nearest-neighbour-chain complete linkage            */
/* Raw merges in discovery order: (slot cluster x, slot cluster y, height).   */
/* ------------------------------------------------------------------------ */
EXPORT int64_t orc_nn_chain(const double *D, int64_t m, int64_t *lefts, int64_t *rights, double *heights) {
    if (m < 2) return 0;
    double *W = (double *)malloc(sizeof(double) * m * m);
    memcpy(W, D, sizeof(double) * m * m);
    for (int64_t i = 0; i < m; i++) W[i * m + i] = INFINITY;
    uint8_t *active = (uint8_t *)malloc(m);
    int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * m);
    int64_t *chain = (int64_t *)malloc(sizeof(int64_t) * (m + 1));
    double *merged = (double *)malloc(sizeof(double) * m);
    for (int64_t i = 0; i < m; i++) { active[i] = 1; slot[i] = i; }
    int64_t nchain = 0, next_id = m, remaining = m, nm = 0;
    while (remaining > 1) {
        if (nchain == 0) {
            int64_t f = 0;
            while (!active[f]) f++;
            chain[nchain++] = f;
        }
        int64_t x = chain[nchain - 1];
        /* row = where(active, W[x], inf); row[x] = inf; y = argmin(row) */
        int64_t y = 0;
        double best = INFINITY;
        int first = 1;
        for (int64_t j = 0; j < m; j++) {
            double r = (active[j] && j != x) ? W[x * m + j] : INFINITY;
            if (first || r < best) { best = r; y = j; first = 0; }
        }
        if (nchain > 1) {
            int64_t p = chain[nchain - 2];
            double rp = (active[p] && p != x) ? W[x * m + p] : INFINITY;
            if (rp == best) y = p;
        }
        if (nchain > 1 && y == chain[nchain - 2]) {
            nchain -= 2;
            double h = W[x * m + y];
            int64_t lo = x < y ? x : y, hi = x < y ? y : x;
            lefts[nm] = slot[x]; rights[nm] = slot[y]; heights[nm] = h; nm++;
            for (int64_t j = 0; j < m; j++) {
                double p = W[lo * m + j], q = W[hi * m + j];
                merged[j] = p > q ? p : (q > p ? q : p); /* np.maximum (no NaN) */
            }
            for (int64_t j = 0; j < m; j++) W[lo * m + j] = merged[j];
            for (int64_t j = 0; j < m; j++) W[j * m + lo] = merged[j];
            W[lo * m + lo] = INFINITY;
            active[hi] = 0;
            slot[lo] = next_id++;
            remaining--;
        } else {
            if (nchain >= m) { nm = -1; break; }  /* chain cycles: the reference would not terminate */
            chain[nchain++] = y;
        }
    }
    free(W); free(active); free(slot); free(chain); free(merged);
    return nm;
}

/* ------------------------------------------------------------------------ */
/* a15  dbht.py:178-214  assign_vertices (per vertex, containing bubbles in   */
/* ascending id; mean = total/4.0 with `total += 0.0 if w == v else query`)  */
/* query: apsp.py:88-90 (exact) or apsp.py:127-136 (hub).                     */
/* ------------------------------------------------------------------------ */
static int near_lookup(const int64_t *ip, const int64_t *ids, const double *dd, int64_t u, int64_t v, double *out) {
    int64_t lo = ip[u], hi = ip[u + 1];
    /* np.searchsorted(ids, v) (left) */
    int64_t a = lo, b = hi;
    while (a < b) {
        int64_t mid = (a + b) >> 1;
        if (ids[mid] < v) a = mid + 1;
        else b = mid;
    }
    if (a < hi && ids[a] == v) { *out = dd[a]; return 1; }
    return 0;
}

static double hub_query(const double *hub_dist, int64_t H, int64_t n, const int64_t *ip, const int64_t *ids,
                        const double *dd, int64_t u, int64_t v) {
    if (u == v) return 0.0;
    if (v < u) { int64_t t = u; u = v; v = t; }
    double d;
    if (near_lookup(ip, ids, dd, u, v, &d)) return d;
    if (near_lookup(ip, ids, dd, v, u, &d)) return d;
    double best = INFINITY;
    int first = 1;
    for (int64_t h = 0; h < H; h++) {
        double s = hub_dist[h * n + u] + hub_dist[h * n + v];
        if (first || s < best) { best = s; first = 0; }
    }
    return best;
}

/* mode 0: exact (D n x n); mode 1: hub.  cont_* = CSR vertex -> containing
 * bubbles ascending.  bubbles (m x 4) sorted members. */
EXPORT void orc_assign(int mode, const double *D, const double *hub_dist, int64_t H, const int64_t *near_indptr,
                       const int64_t *near_ids, const double *near_dist, int64_t n, const int32_t *bubbles,
                       const int64_t *cont_indptr, const int64_t *cont_ids, int64_t *vertex_bubble) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t v = 0; v < n; v++) {
        int64_t best_bid = -1;
        double best_mean = INFINITY;
        for (int64_t e = cont_indptr[v]; e < cont_indptr[v + 1]; e++) {
            int64_t bid = cont_ids[e];
            double total = 0.0;
            for (int k = 0; k < 4; k++) {
                int64_t w = bubbles[bid * 4 + k];
                double q;
                if (w == v) q = 0.0;
                else if (mode == 0) q = D[v * n + w];
                else q = hub_query(hub_dist, H, n, near_indptr, near_ids, near_dist, v, w);
                total += q;
            }
            double mean = total / 4.0;
            if (mean < best_mean) { best_mean = mean; best_bid = bid; }
        }
        vertex_bubble[v] = best_bid;
    }
}
