// rowsort.cu -- the aggregated per-row neighbour sort and the initial-clique row sums.
//
// Replaces simmatrix.py:225-249 sort_neighbor_lists (per row v: ids by (S desc,
// id asc), v removed; numpy argsort + lexsort tie rule) and tmfg.py:71-79
// select_initial_clique (numpy pairwise row sums, stable top-4).
//
// B200 design (one CTA of 1024 threads per row, persistent over rows):
//   1. the row (8n bytes) is streamed into shared memory with 16-byte cp.async,
//      double-buffered so row v+grid loads while row v is sorted;
//   2. equalised two-level bucketing: a warp-aggregated histogram over 512
//      linear bins of [min, max] sizes each bin's share of fine buckets
//      (ceil(count/2)), and each bin is split linearly again -- about two keys
//      per fine bucket whatever the value distribution; bucket ids are monotone
//      in the value and equal values (incl. -0.0/+0.0) share a bucket;
//   3. one shared-memory atomicAdd per key yields its rank inside the fine
//      bucket; a block scan gives bucket starts and the ids (u16) are scattered;
//   4. every key's exact rank inside its bucket (value desc, id asc) is counted
//      against the other members (independent loads, cost = bucket size), and
//      the ids are placed once more -- so the result is deterministic even though
//      the atomic ranks are not; degenerate rows with huge tie groups stay
//      correct (quadratic in the group size only);
//   5. the ids stream out with 16-byte stores; optionally the same pass computes
//      numpy's pairwise row sum from the staged row (fused initial-clique input).
// Rows longer than the shared-memory budget (n > 16384) take the global-memory
// variant below (same algorithm, the row and the scatter buffer live in L2).
#include "common.cuh"

namespace {

constexpr int RS_T = 1024;
constexpr int PW_MAXNODES = 2048;   // n <= 131072
constexpr int PW_SMALLNODES = 512;  // n <= 16384

// ---------------------------------------------------------------- pairwise tree
// numpy's float64 add.reduce inner loop: pairwise_sum(a, n) with 8 accumulators,
// block 128, split n2 = n/2 - (n/2)%8 (numpy/_core/src/umath/loops_utils.h).
template <int N>
struct PwTree {
    int nnodes;
    int nlevels;
    int root;
    int a[N];    // leaf: offset        internal: left child
    int b[N];    // leaf: length (> 0)  internal: -(right child + 1)
    int lvl_off[33];
    int lvl[N];
};

template <int N>
__device__ int pw_build(PwTree<N> &t, int off, int len, int *height) {
    if (len <= 128) {
        int id = t.nnodes++;
        t.a[id] = off;
        t.b[id] = len;
        height[id] = 0;
        return id;
    }
    int n2 = len / 2;
    n2 -= n2 % 8;
    int l = pw_build(t, off, n2, height);
    int r = pw_build(t, off + n2, len - n2, height);
    int id = t.nnodes++;
    t.a[id] = l;
    t.b[id] = -(r + 1);
    height[id] = 1 + max(height[l], height[r]);
    return id;
}

// single thread; `height` is scratch of PW_MAXNODES ints
template <int N>
__device__ void pw_plan(PwTree<N> &t, int n, int *height) {
    t.nnodes = 0;
    t.root = pw_build(t, 0, n, height);
    int H = height[t.root];
    t.nlevels = H + 1;
    int cnt[33];
    for (int h = 0; h <= 32; h++) cnt[h] = 0;
    for (int i = 0; i < t.nnodes; i++) cnt[height[i]]++;
    t.lvl_off[0] = 0;
    for (int h = 0; h < 32; h++) t.lvl_off[h + 1] = t.lvl_off[h] + cnt[h];
    for (int h = 0; h <= 32; h++) cnt[h] = 0;
    for (int i = 0; i < t.nnodes; i++) {
        int h = height[i];
        t.lvl[t.lvl_off[h] + cnt[h]++] = i;
    }
}

template <class Load>
__device__ __forceinline__ double pw_leaf(Load ld, int off, int len) {
    if (len < 8) {
        double r = 0.0;
        for (int i = 0; i < len; i++) r = __dadd_rn(r, ld(off + i));
        return r;
    }
    double r0 = ld(off), r1 = ld(off + 1), r2 = ld(off + 2), r3 = ld(off + 3);
    double r4 = ld(off + 4), r5 = ld(off + 5), r6 = ld(off + 6), r7 = ld(off + 7);
    int i = 8;
    int lim = len - (len % 8);
    for (; i < lim; i += 8) {
        r0 = __dadd_rn(r0, ld(off + i));
        r1 = __dadd_rn(r1, ld(off + i + 1));
        r2 = __dadd_rn(r2, ld(off + i + 2));
        r3 = __dadd_rn(r3, ld(off + i + 3));
        r4 = __dadd_rn(r4, ld(off + i + 4));
        r5 = __dadd_rn(r5, ld(off + i + 5));
        r6 = __dadd_rn(r6, ld(off + i + 6));
        r7 = __dadd_rn(r7, ld(off + i + 7));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                           __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    for (; i < len; i++) res = __dadd_rn(res, ld(off + i));
    return res;
}

// all threads of the block; returns the root value to every thread
template <int N, class Load>
__device__ double pw_eval(const PwTree<N> &t, double *val, Load ld) {
    for (int i = threadIdx.x; i < t.lvl_off[1]; i += blockDim.x) {
        int id = t.lvl[i];
        val[id] = pw_leaf(ld, t.a[id], t.b[id]);
    }
    __syncthreads();
    for (int h = 1; h < t.nlevels; h++) {
        for (int i = t.lvl_off[h] + threadIdx.x; i < t.lvl_off[h + 1]; i += blockDim.x) {
            int id = t.lvl[i];
            val[id] = __dadd_rn(val[t.a[id]], val[-t.b[id] - 1]);
        }
        __syncthreads();
    }
    return val[t.root];
}

__global__ void row_sums_kernel(const double *__restrict__ S, int64_t n, double *__restrict__ rowsum) {
    __shared__ PwTree<PW_MAXNODES> tree;
    __shared__ double val[PW_MAXNODES];
    if (threadIdx.x == 0) pw_plan(tree, (int)n, reinterpret_cast<int *>(val));
    __syncthreads();
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const double *row = S + v * n;
        double root = pw_eval(tree, val, [&](int i) { return __ldg(row + i); });
        if (threadIdx.x == 0) rowsum[v] = __dsub_rn(root, row[v]);
        __syncthreads();
    }
}

// argsort(-sums, kind="stable")[:4] -> sorted ascending; NaN sorts last
__device__ __forceinline__ bool clique_better(double si, int64_t i, double sj, int64_t j) {
    double ki = -si, kj = -sj;
    bool ni = isnan(ki), nj = isnan(kj);
    if (ni != nj) return !ni;
    if (!ni && ki != kj) return ki < kj;
    return i < j;
}

__global__ void clique_kernel(const double *__restrict__ rowsum, int64_t n, int32_t *__restrict__ out) {
    __shared__ double bs[32];
    __shared__ int64_t bi[32];
    __shared__ int64_t chosen[4];
    for (int k = 0; k < 4; k++) {
        double best = 0.0;
        int64_t bid = -1;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
            bool used = false;
            for (int q = 0; q < k; q++) used |= (chosen[q] == i);
            if (used) continue;
            double s = rowsum[i];
            if (bid < 0 || clique_better(s, i, best, bid)) { best = s; bid = i; }
        }
        for (int o = 16; o; o >>= 1) {
            double s2 = __shfl_xor_sync(0xffffffffu, best, o);
            int64_t i2 = __shfl_xor_sync(0xffffffffu, bid, o);
            if (i2 >= 0 && (bid < 0 || clique_better(s2, i2, best, bid))) { best = s2; bid = i2; }
        }
        if ((threadIdx.x & 31) == 0) { bs[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = bid; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b0 = 0.0;
            int64_t i0 = -1;
            for (int w = 0; w < (int)(blockDim.x >> 5); w++)
                if (bi[w] >= 0 && (i0 < 0 || clique_better(bs[w], bi[w], b0, i0))) { b0 = bs[w]; i0 = bi[w]; }
            chosen[k] = i0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int64_t t[4] = {chosen[0], chosen[1], chosen[2], chosen[3]};
        for (int a = 0; a < 4; a++)
            for (int b = a + 1; b < 4; b++)
                if (t[b] < t[a]) { int64_t x = t[a]; t[a] = t[b]; t[b] = x; }
        for (int a = 0; a < 4; a++) out[a] = (int32_t)t[a];
    }
}

// ---------------------------------------------------------------- row sort
// strict "id a precedes id b" in a row: value desc, NaN last, then id asc
__device__ __forceinline__ bool rs_before(double xa, int ia, double xb, int ib) {
    bool na = isnan(xa), nb = isnan(xb);
    if (na != nb) return !na;
    if (!na) {
        if (xa > xb) return true;
        if (xa < xb) return false;
    }
    return ia < ib;
}

constexpr int RS_CMAX = 512;   // coarse (linear) bins

__host__ __device__ __forceinline__ int rs_coarse_bins(int m) {
    int c = m / 4;
    if (c > RS_CMAX) c = RS_CMAX;
    if (c < 1) c = 1;
    return c;
}
// fine buckets never exceed C + ceil(m/2) + C
__host__ __device__ __forceinline__ int rs_fine_cap(int m) { return 2 * rs_coarse_bins(m) + (m + 1) / 2 + 1; }

struct RsPlan {
    int n, C, NBcap, nbuf, stride;
    size_t off_sidx, off_fcnt, off_misc, smem;
};

struct RsMisc {
    double red[64];
    double rmin, rmax, cscale;
    uint32_t ccnt[RS_CMAX + 1];    // coarse counts -> fine base (exclusive scan of f_c)
    uint32_t cf[RS_CMAX];          // fine buckets per coarse bin
    uint32_t wsum[32];
    uint32_t nsamp;
};

__host__ RsPlan rs_plan(int64_t n, int nbuf) {
    RsPlan p;
    p.n = (int)n;
    int m = (int)n - 1;
    p.C = rs_coarse_bins(m);
    p.NBcap = rs_fine_cap(m);
    p.nbuf = nbuf;
    p.stride = (int)((n + 1) & ~1LL);   // keeps the second row buffer 16-byte aligned
    size_t off = tg_align_up((size_t)nbuf * p.stride * sizeof(double), 16);
    p.off_sidx = off;
    off = tg_align_up(off + (size_t)n * sizeof(uint16_t), 16);
    p.off_fcnt = off;
    off = tg_align_up(off + (size_t)(p.NBcap + 1) * sizeof(uint32_t), 16);
    p.off_misc = off;
    off += tg_align_up(sizeof(RsMisc), 16);
    p.smem = off;
    return p;
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16g(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void rs_issue_row(double *dst, const double *src, int n) {
    // 16-byte chunks when source and destination are 16-byte aligned, else 8-byte copies
    if (((((uintptr_t)src) | ((uintptr_t)dst)) & 15) == 0) {
        int nv = n >> 1;
        for (int i = threadIdx.x; i < nv; i += blockDim.x) cp_async16g(dst + 2 * i, src + 2 * i);
        if ((n & 1) && threadIdx.x == 0) cp_async8(dst + n - 1, src + n - 1);
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) cp_async8(dst + i, src + i);
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

// coarse bin of x in t-space: t = (rmax - x) * cscale in [0, C]
__device__ __forceinline__ int rs_coarse_of(double x, double rmax, double cscale, int C, double &t) {
    if (isnan(x)) { t = (double)C; return C - 1; }
    t = (rmax - x) * cscale;
    int c = (t >= 0.0) ? (t < (double)C ? (int)t : C - 1) : 0;
    return c;
}

__device__ __forceinline__ int rs_fine_of(double t, int c, const uint32_t *base, const uint32_t *cf) {
    int f = (int)cf[c];
    double frac = t - (double)c;
    int sub = (frac >= 0.0) ? (int)(frac * (double)f) : 0;
    if (sub > f - 1) sub = f - 1;
    return (int)base[c] + sub;
}

template <int EMAX>
__global__ void __launch_bounds__(RS_T, 1)
row_sort_smem_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                     double *__restrict__ rowsum, RsPlan pl) {
    extern __shared__ __align__(16) unsigned char rs_smem[];
    const int n = (int)n64;
    const int m = n - 1;
    double *vbuf = reinterpret_cast<double *>(rs_smem);
    uint16_t *sidx = reinterpret_cast<uint16_t *>(rs_smem + pl.off_sidx);
    uint32_t *fcnt = reinterpret_cast<uint32_t *>(rs_smem + pl.off_fcnt);
    RsMisc &ms = *reinterpret_cast<RsMisc *>(rs_smem + pl.off_misc);
    __shared__ PwTree<PW_SMALLNODES> tree;
    __shared__ double pwval[PW_SMALLNODES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = pl.C;

    if (rowsum) {
        int *height = reinterpret_cast<int *>(pwval);  // scratch before first use
        if (tid == 0) pw_plan(tree, n, height);
    }
    int it = 0;
    int64_t v = blockIdx.x;
    if (v < n && pl.nbuf == 2) rs_issue_row(vbuf, S + v * n64, n);
    for (; v < n; v += gridDim.x, it++) {
        double *vals = vbuf + (pl.nbuf == 2 ? (size_t)(it & 1) * pl.stride : 0);
        if (pl.nbuf == 1) rs_issue_row(vals, S + v * n64, n);
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        if (pl.nbuf == 2) {
            int64_t vn = v + gridDim.x;
            if (vn < n) rs_issue_row(vbuf + (size_t)((it + 1) & 1) * pl.stride, S + vn * n64, n);
        }
        // ---- A: zero coarse counters, row min/max (v excluded)
        for (int c = tid; c <= C; c += RS_T) ms.ccnt[c] = 0;
        if (tid == 0) ms.nsamp = 0;
        double mn = INFINITY, mx = -INFINITY;
        bool nan_seen = false;
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double x = vals[j];
            if (x < mn) mn = x;
            if (x > mx) mx = x;
            nan_seen |= (x != x);
        }
        const bool row_nan = __syncthreads_or(nan_seen);
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { ms.red[warp] = mn; ms.red[32 + warp] = mx; }
        __syncthreads();
        if (warp == 0) {
            double a = ms.red[lane], b = ms.red[32 + lane];
            for (int o = 16; o; o >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
            }
            if (lane == 0) {
                double w = b - a;
                ms.rmin = a;
                ms.rmax = b;
                ms.cscale = (w > 0.0 && w < INFINITY) ? (double)C / w : 0.0;
            }
        }
        __syncthreads();
        // ---- B: coarse histogram (linear bins over [min, max]) from a 1-in-4 sample
        // (it only sizes the fine buckets: accuracy affects speed, never the order)
        const double rmax = ms.rmax, cscale = ms.cscale;
        uint32_t pk[EMAX];
        int nsamp = 0;
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            int j = tid + e * RS_T;
            bool act = j < n && j != v;
            if (act && (e & 3) == 0) {
                double t;
                atomicAdd(&ms.ccnt[rs_coarse_of(vals[j], rmax, cscale, C, t)], 1u);
                nsamp++;
            }
            pk[e] = act ? 0u : 0xffffffffu;
        }
        nsamp = __reduce_add_sync(0xffffffffu, nsamp);
        if (lane == 0 && nsamp) atomicAdd(&ms.nsamp, (uint32_t)nsamp);
        __syncthreads();
        // ---- C: fine buckets per coarse bin (about two keys each), base offsets
        {
            const uint64_t den = 2ull * (ms.nsamp ? ms.nsamp : 1u);
            for (int c = tid; c < C; c += RS_T) {
                uint64_t h = ms.ccnt[c];
                uint32_t f = (uint32_t)((h * (uint64_t)m + den - 1) / den);
                ms.cf[c] = f > 1 ? f : 1u;
            }
        }
        __syncthreads();
        if (warp == 0) {
            // exclusive scan of cf -> ccnt (base), C <= 512: 16 per lane
            const int per = (C + 31) / 32;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int c = lane * per + q;
                if (c < C) s += ms.cf[c];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t run = incl - s;
            for (int q = 0; q < per; q++) {
                int c = lane * per + q;
                if (c < C) { ms.ccnt[c] = run; run += ms.cf[c]; }
            }
            if (lane == 31) ms.ccnt[C] = incl;
        }
        __syncthreads();
        const int NB = (int)ms.ccnt[C];
        for (int b = tid; b <= NB; b += RS_T) fcnt[b] = 0;
        __syncthreads();
        // ---- D: fine bucket + rank inside it (one shared atomic per key)
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            if (pk[e] != 0xffffffffu) {
                int j = tid + e * RS_T;
                double t;
                int c = rs_coarse_of(vals[j], rmax, cscale, C, t);
                int fb = rs_fine_of(t, c, ms.ccnt, ms.cf);
                uint32_t r = atomicAdd(&fcnt[fb], 1u);
                pk[e] = ((uint32_t)fb << 16) | r;
            }
        }
        __syncthreads();
        // ---- E: exclusive scan of the fine counters, scatter ids
        {
            const int len = NB + 1;
            const int per = (len + RS_T - 1) / RS_T;
            const int b0 = tid * per;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b < len) s += fcnt[b];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) ms.wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                uint32_t w = ms.wsum[lane];
                uint32_t wi = w;
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= o) wi += y;
                }
                ms.wsum[lane] = wi - w;
            }
            __syncthreads();
            uint32_t run = ms.wsum[warp] + incl - s;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b < len) {
                    uint32_t c = fcnt[b];
                    fcnt[b] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            if (pk[e] != 0xffffffffu) {
                int j = tid + e * RS_T;
                sidx[fcnt[pk[e] >> 16] + (pk[e] & 0xffffu)] = (uint16_t)j;
            }
        }
        __syncthreads();
        // ---- F: exact rank of every key inside its bucket (value desc, id asc):
        // independent loads, cost per key = its bucket size; ids placed once more.
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            if (pk[e] != 0xffffffffu) {
                const int j = tid + e * RS_T;
                const int b = (int)(pk[e] >> 16);
                const int s0 = (int)fcnt[b], s1 = (int)fcnt[b + 1];
                int rank = 0;
                if (s1 - s0 > 1) {
                    const double xj = vals[j];
                    if (!row_nan) {
                        for (int k = s0; k < s1; k++) {
                            const int o = sidx[k];
                            const double xo = vals[o];
                            rank += (xo > xj) | ((xo == xj) & (o < j));
                        }
                    } else {
                        for (int k = s0; k < s1; k++) {
                            const int o = sidx[k];
                            rank += rs_before(vals[o], o, xj, j);
                        }
                    }
                }
                pk[e] = (uint32_t)(s0 + rank);
            }
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < EMAX; e++)
            if (pk[e] != 0xffffffffu) sidx[pk[e]] = (uint16_t)(tid + e * RS_T);
        __syncthreads();
        // ---- G: write ids (16-byte stores on the aligned body)
        {
            int32_t *out = order + v * (int64_t)m;
            int head = (int)(((16 - (((uintptr_t)out) & 15)) & 15) >> 2);
            if (head > m) head = m;
            for (int p = tid; p < head; p += RS_T) out[p] = sidx[p];
            int body = (m - head) >> 2;
            int4 *o4 = reinterpret_cast<int4 *>(out + head);
            for (int q = tid; q < body; q += RS_T) {
                int p = head + 4 * q;
                o4[q] = make_int4(sidx[p], sidx[p + 1], sidx[p + 2], sidx[p + 3]);
            }
            for (int p = head + 4 * body + tid; p < m; p += RS_T) out[p] = sidx[p];
        }
        // ---- H: fused pairwise row sum (initial-clique input)
        if (rowsum) {
            double root = pw_eval(tree, pwval, [&](int i) { return vals[i]; });
            if (tid == 0) rowsum[v] = __dsub_rn(root, vals[v]);
        }
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---------------------------------------------------------------- large rows
// n > 16384: the same two-level bucket algorithm; the row is read through L2,
// the per-key (bucket, rank) pairs live in a per-CTA global scratch slice and
// the output row itself is the scatter buffer.  Counters stay in shared memory.
__global__ void __launch_bounds__(RS_T, 1)
row_sort_global_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                       double *__restrict__ rowsum, uint32_t *__restrict__ gpk_all) {
    const int n = (int)n64;
    const int m = n - 1;
    extern __shared__ __align__(16) unsigned char rs_smem[];
    uint32_t *fcnt = reinterpret_cast<uint32_t *>(rs_smem);
    __shared__ RsMisc ms;
    __shared__ PwTree<PW_MAXNODES> tree;
    __shared__ double pwval[PW_MAXNODES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = rs_coarse_bins(m);
    uint32_t *gpk = gpk_all + (size_t)blockIdx.x * 2 * n;   // [n] bucket, [n] rank/position
    if (rowsum) {
        int *height = reinterpret_cast<int *>(pwval);
        if (tid == 0) pw_plan(tree, n, height);
        __syncthreads();
    }
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const double *row = S + v * n64;
        int32_t *out = order + v * (int64_t)m;
        for (int c = tid; c <= C; c += RS_T) ms.ccnt[c] = 0;
        if (tid == 0) ms.nsamp = 0;
        double mn = INFINITY, mx = -INFINITY;
        bool nan_seen = false;
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double x = __ldg(row + j);
            if (x < mn) mn = x;
            if (x > mx) mx = x;
            nan_seen |= (x != x);
        }
        const bool row_nan = __syncthreads_or(nan_seen);
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { ms.red[warp] = mn; ms.red[32 + warp] = mx; }
        __syncthreads();
        if (warp == 0) {
            double a = ms.red[lane], b = ms.red[32 + lane];
            for (int o = 16; o; o >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
            }
            if (lane == 0) {
                double w = b - a;
                ms.rmin = a;
                ms.rmax = b;
                ms.cscale = (w > 0.0 && w < INFINITY) ? (double)C / w : 0.0;
            }
        }
        __syncthreads();
        const double rmax = ms.rmax, cscale = ms.cscale;
        int nsamp = 0;
        for (int j = tid; j < n; j += 4 * RS_T) {
            if (j == v) continue;
            double t;
            atomicAdd(&ms.ccnt[rs_coarse_of(__ldg(row + j), rmax, cscale, C, t)], 1u);
            nsamp++;
        }
        nsamp = __reduce_add_sync(0xffffffffu, nsamp);
        if (lane == 0 && nsamp) atomicAdd(&ms.nsamp, (uint32_t)nsamp);
        __syncthreads();
        {
            const uint64_t den = 2ull * (ms.nsamp ? ms.nsamp : 1u);
            for (int c = tid; c < C; c += RS_T) {
                uint64_t h = ms.ccnt[c];
                uint32_t f = (uint32_t)((h * (uint64_t)m + den - 1) / den);
                ms.cf[c] = f > 1 ? f : 1u;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int per = (C + 31) / 32;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int c = lane * per + q;
                if (c < C) s += ms.cf[c];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t run = incl - s;
            for (int q = 0; q < per; q++) {
                int c = lane * per + q;
                if (c < C) { ms.ccnt[c] = run; run += ms.cf[c]; }
            }
            if (lane == 31) ms.ccnt[C] = incl;
        }
        __syncthreads();
        const int NB = (int)ms.ccnt[C];
        for (int b = tid; b <= NB; b += RS_T) fcnt[b] = 0;
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double t;
            int c = rs_coarse_of(__ldg(row + j), rmax, cscale, C, t);
            int fb = rs_fine_of(t, c, ms.ccnt, ms.cf);
            gpk[j] = (uint32_t)fb;
            gpk[n + j] = atomicAdd(&fcnt[fb], 1u);
        }
        __syncthreads();
        {
            const int len = NB + 1;
            const int per = (len + RS_T - 1) / RS_T;
            const int b0 = tid * per;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b < len) s += fcnt[b];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) ms.wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                uint32_t w = ms.wsum[lane];
                uint32_t wi = w;
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= o) wi += y;
                }
                ms.wsum[lane] = wi - w;
            }
            __syncthreads();
            uint32_t run = ms.wsum[warp] + incl - s;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b < len) {
                    uint32_t c = fcnt[b];
                    fcnt[b] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            out[fcnt[gpk[j]] + gpk[n + j]] = j;
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            const int b = (int)gpk[j];
            const int s0 = (int)fcnt[b], s1 = (int)fcnt[b + 1];
            int rank = 0;
            if (s1 - s0 > 1) {
                const double xj = __ldg(row + j);
                for (int k = s0; k < s1; k++) {
                    const int o = out[k];
                    const double xo = __ldg(row + o);
                    rank += row_nan ? (int)rs_before(xo, o, xj, j) : (int)((xo > xj) | ((xo == xj) & (o < j)));
                }
            }
            gpk[n + j] = (uint32_t)(s0 + rank);
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            out[gpk[n + j]] = j;
        }
        __syncthreads();
        if (rowsum) {
            double root = pw_eval(tree, pwval, [&](int i) { return __ldg(row + i); });
            if (tid == 0) rowsum[v] = __dsub_rn(root, row[v]);
        }
        __syncthreads();
    }
}

constexpr size_t RS_SMEM_MAX = 227 * 1024 - sizeof(PwTree<PW_SMALLNODES>) - PW_SMALLNODES * sizeof(double) - 1024;

}  // namespace

TG_API size_t tg_row_sort_workspace_bytes(int64_t n) {
    if (n <= 16384) return 256;
    return (size_t)tg_num_sms() * 2 * (size_t)n * sizeof(uint32_t) + 4096;
}

TG_API int tg_row_sort_f64(const double *S, int64_t n, int32_t *order, double *rowsum, void *ws, size_t ws_bytes,
                           void *stream) {
    if (n < 2 || !S || !order) return TG_ERR_ARG;
    cudaStream_t st = tg_stream(stream);
    int grid = tg_num_sms();
    if (grid > n) grid = (int)n;
    if (n <= 16384) {
        RsPlan pl = rs_plan(n, 2);
        if (pl.smem > RS_SMEM_MAX) pl = rs_plan(n, 1);
        if (pl.smem > RS_SMEM_MAX) return TG_ERR_ARG;
        int E = (int)((n + RS_T - 1) / RS_T);
#define RS_LAUNCH(EM)                                                                                      \
    do {                                                                                                   \
        auto kfn = row_sort_smem_kernel<EM>;                                                               \
        TG_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem)); \
        kfn<<<grid, RS_T, pl.smem, st>>>(S, n, order, rowsum, pl); tg_count_launch(1);                                         \
    } while (0)
        if (E <= 2) RS_LAUNCH(2);
        else if (E <= 4) RS_LAUNCH(4);
        else if (E <= 8) RS_LAUNCH(8);
        else RS_LAUNCH(16);
#undef RS_LAUNCH
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    if (n > (int64_t)1 << 30) return TG_ERR_ARG;
    if (n > 128 * (PW_MAXNODES / 2) && rowsum) return TG_ERR_ARG;
    if (ws_bytes < tg_row_sort_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    uint32_t *gpk = reinterpret_cast<uint32_t *>(ws);
    int m = (int)n - 1;
    size_t smem = (size_t)(rs_fine_cap(m) + 1) * sizeof(uint32_t);
    if (smem > 160 * 1024) return TG_ERR_ARG;
    TG_CUDA_CHECK(cudaFuncSetAttribute(row_sort_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    row_sort_global_kernel<<<grid, RS_T, smem, st>>>(S, n, order, rowsum, gpk); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_row_sums_workspace_bytes(int64_t) { return 256; }

TG_API int tg_row_sums_f64(const double *S, int64_t n, double *rowsum, void *, size_t, void *stream) {
    if (n < 1 || !S || !rowsum) return TG_ERR_ARG;
    if (n > 128 * (PW_MAXNODES / 2)) return TG_ERR_ARG;
    int grid = tg_num_sms() * 4;
    if (grid > n) grid = (int)n;
    row_sums_kernel<<<grid, 256, 0, tg_stream(stream)>>>(S, n, rowsum); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_initial_clique(const double *rowsum, int64_t n, int32_t *clique, void *stream) {
    if (n < 4 || !rowsum || !clique) return TG_ERR_ARG;
    clique_kernel<<<1, 1024, 0, tg_stream(stream)>>>(rowsum, n, clique); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
