// rowsort.cu -- the aggregated per-row neighbour sort and the initial-clique row sums.
//
// Replaces simmatrix.py:225-249 sort_neighbor_lists (per row v: ids by (S desc,
// id asc), v removed; numpy argsort + lexsort tie rule) and tmfg.py:71-79
// select_initial_clique (numpy pairwise row sums, stable top-4).
//
// B200 design (one CTA of 1024 threads per row, persistent over rows):
//   1. the row (8n bytes) is streamed into shared memory with 16-byte cp.async,
//      double-buffered so row v+grid loads while row v is sorted;
//   2. equalised bucketing: 64 splitters sampled from the row (sorted by one
//      warp) cut it into 65 quantile bins, each split linearly into K
//      sub-buckets, giving ~2 keys per bucket; bucket ids are monotone in the
//      value and equal values (incl. -0.0/+0.0) share a bucket;
//   3. one shared-memory atomicAdd per key yields its rank inside the bucket;
//      a block scan gives bucket starts and the ids (u16) are scattered once;
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
constexpr int RS_PMAX = 64;
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

struct RsPlan {
    int n, P, K, NB, pow2, nbuf;
    size_t off_sidx, off_cnt, off_spl, off_ub, off_scl, off_misc, smem;
};

__host__ RsPlan rs_plan(int64_t n, int nbuf) {
    RsPlan p;
    p.n = (int)n;
    int m = (int)n - 1;
    int P = m / 16;
    if (P > RS_PMAX) P = RS_PMAX;
    if (P < 1) P = 1;
    p.P = P;
    int K = (int)((m + 2 * (P + 1) - 1) / (2 * (P + 1)));
    if (K < 1) K = 1;
    p.K = K;
    p.NB = (P + 1) * K;
    int pw = 1;
    while (pw < m) pw <<= 1;
    p.pow2 = pw;
    p.nbuf = nbuf;
    size_t off = tg_align_up((size_t)nbuf * n * sizeof(double), 16);
    p.off_sidx = off;
    off = tg_align_up(off + (size_t)n * sizeof(uint16_t), 16);
    p.off_cnt = off;
    off = tg_align_up(off + (size_t)(p.NB + 1) * sizeof(uint32_t), 16);
    p.off_spl = off;
    off = tg_align_up(off + (size_t)RS_PMAX * sizeof(double), 16);
    p.off_ub = off;
    off = tg_align_up(off + (size_t)(RS_PMAX + 1) * sizeof(double), 16);
    p.off_scl = off;
    off = tg_align_up(off + (size_t)(RS_PMAX + 1) * sizeof(double), 16);
    p.off_misc = off;
    off += 2048;
    p.smem = off;
    return p;
}

struct RsMisc {
    double red[64];
    double rmin, rmax;
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16g(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void rs_issue_row(double *dst, const double *src, int n) {
    // 16-byte chunks when the row start is 16-byte aligned, else 8-byte copies
    if ((((uintptr_t)src) & 15) == 0) {
        int nv = n >> 1;
        for (int i = threadIdx.x; i < nv; i += blockDim.x) cp_async16g(dst + 2 * i, src + 2 * i);
        if ((n & 1) && threadIdx.x == 0) cp_async8(dst + n - 1, src + n - 1);
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) cp_async8(dst + i, src + i);
    }
    asm volatile("cp.async.commit_group;\n" ::);
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
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rs_smem + pl.off_cnt);
    double *spl = reinterpret_cast<double *>(rs_smem + pl.off_spl);
    double *ub = reinterpret_cast<double *>(rs_smem + pl.off_ub);
    double *scl = reinterpret_cast<double *>(rs_smem + pl.off_scl);
    RsMisc &ms = *reinterpret_cast<RsMisc *>(rs_smem + pl.off_misc);
    __shared__ PwTree<PW_SMALLNODES> tree;
    __shared__ double pwval[PW_SMALLNODES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int P = pl.P, K = pl.K, NB = pl.NB;

    if (rowsum) {
        int *height = reinterpret_cast<int *>(pwval);  // scratch before first use
        if (tid == 0) pw_plan(tree, n, height);
    }
    int it = 0;
    int64_t v = blockIdx.x;
    if (v < n && pl.nbuf == 2) rs_issue_row(vbuf, S + v * n64, n);
    for (; v < n; v += gridDim.x, it++) {
        double *vals = vbuf + (pl.nbuf == 2 ? (size_t)(it & 1) * n : 0);
        if (pl.nbuf == 1) rs_issue_row(vals, S + v * n64, n);
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        if (pl.nbuf == 2) {
            int64_t vn = v + gridDim.x;
            if (vn < n) rs_issue_row(vbuf + (size_t)((it + 1) & 1) * n, S + vn * n64, n);
        }
        // ---- phase A: zero counters, row min/max (v excluded)
        for (int b = tid; b <= NB; b += RS_T) cnt[b] = 0;
        double mn = INFINITY, mx = -INFINITY;
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double x = vals[j];
            if (x < mn) mn = x;
            if (x > mx) mx = x;
        }
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { ms.red[warp] = mn; ms.red[32 + warp] = mx; }
        __syncthreads();
        // ---- phase B: splitters (warp 0) and per-bin linear maps
        if (warp == 0) {
            double a = ms.red[lane], b = ms.red[32 + lane];
            for (int o = 16; o; o >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
            }
            double xs[2];
            unsigned long long ks[2];
            for (int q = 0; q < 2; q++) {
                int k = lane + 32 * q;
                double x = 0.0;
                if (k < P) {
                    int j = (int)(((int64_t)(2 * k + 1) * n) / (2 * P));
                    if (j >= n) j = n - 1;
                    if (j == v) j = (j + 1 < n) ? j + 1 : j - 1;
                    x = vals[j];
                }
                xs[q] = x;
                ks[q] = isnan(x) ? 0ull : tg_order_key(x);
            }
            for (int q = 0; q < 2; q++) {
                int k = lane + 32 * q;
                int rank = 0;
                for (int mm = 0; mm < 2 * 32; mm++) {
                    unsigned long long km = __shfl_sync(0xffffffffu, ks[mm >> 5], mm & 31);
                    if (mm < P) rank += (km > ks[q]) || (km == ks[q] && mm < k);
                }
                if (k < P) spl[rank] = xs[q];
            }
            __syncwarp();
            if (lane == 0) { ms.rmin = a; ms.rmax = b; }
            for (int c = lane; c <= P; c += 32) {
                double u = (c == 0) ? b : spl[c - 1];
                double l = (c == P) ? a : spl[c];
                double w = u - l;
                ub[c] = u;
                scl[c] = (w > 0.0 && w < INFINITY) ? (double)K / w : 0.0;
            }
        }
        __syncthreads();
        // ---- phase C: bucket + rank (one shared atomic per key)
        uint32_t pk[EMAX];
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            int j = tid + e * RS_T;
            pk[e] = 0xffffffffu;
            if (j < n && j != v) {
                double x = vals[j];
                int b;
                if (isnan(x)) {
                    b = NB - 1;
                } else {
                    int lo = 0, hi = P;
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (spl[mid] > x) lo = mid + 1;
                        else hi = mid;
                    }
                    double t = (ub[lo] - x) * scl[lo];
                    int sub = (t >= 0.0) ? (t < (double)K ? (int)t : K - 1) : 0;
                    b = lo * K + sub;
                }
                uint32_t r = atomicAdd(&cnt[b], 1u);
                pk[e] = ((uint32_t)b << 16) | r;
            }
        }
        __syncthreads();
        // ---- phase D: exclusive scan of cnt[0..NB] (block)
        {
            const int per = (NB + 1 + RS_T - 1) / RS_T;
            int b0 = tid * per;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b <= NB) s += cnt[b];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t *wsum = reinterpret_cast<uint32_t *>(ms.red);
            __syncthreads();
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                uint32_t w = wsum[lane];
                uint32_t wi = w;
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= o) wi += y;
                }
                wsum[lane] = wi - w;
            }
            __syncthreads();
            uint32_t run = wsum[warp] + incl - s;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b <= NB) {
                    uint32_t c = cnt[b];
                    cnt[b] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
        // ---- phase E: scatter ids
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            if (pk[e] != 0xffffffffu) {
                int j = tid + e * RS_T;
                sidx[cnt[pk[e] >> 16] + (pk[e] & 0xffffu)] = (uint16_t)j;
            }
        }
        __syncthreads();
        // ---- phase F: exact rank of every key inside its bucket (value desc, id asc).
        // Independent loads, no dependent chains: cost per key = its bucket size.
#pragma unroll
        for (int e = 0; e < EMAX; e++) {
            if (pk[e] != 0xffffffffu) {
                const int j = tid + e * RS_T;
                const int b = (int)(pk[e] >> 16);
                const int s0 = (int)cnt[b], s1 = (int)cnt[b + 1];
                int rank = 0;
                if (s1 - s0 > 1) {
                    const double xj = vals[j];
                    for (int k = s0; k < s1; k++) {
                        const int o = sidx[k];
                        rank += rs_before(vals[o], o, xj, j);
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
        // ---- phase G: write ids (16-byte stores on the aligned body)
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
        // ---- phase H: fused pairwise row sum (initial-clique input)
        if (rowsum) {
            double root = pw_eval(tree, pwval, [&](int i) { return vals[i]; });
            if (tid == 0) rowsum[v] = __dsub_rn(root, vals[v]);
        }
        __syncthreads();
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
}

// ---------------------------------------------------------------- large rows
// n > 16384: the same bucket algorithm with the row, the ranks and the scatter
// buffer in global scratch (one slice per CTA; L2-resident while the CTA works
// on the row).  Counters stay in shared memory.
__global__ void __launch_bounds__(RS_T, 1)
row_sort_global_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                       double *__restrict__ rowsum, int P, int K, int NB, uint32_t *__restrict__ gcnt_all,
                       uint32_t *__restrict__ grank_all, int32_t *__restrict__ gidx_all) {
    const int n = (int)n64;
    const int m = n - 1;
    extern __shared__ __align__(16) unsigned char rs_smem[];
    uint32_t *cnt = reinterpret_cast<uint32_t *>(rs_smem);   // NB+1 (if it fits) else global
    __shared__ double spl[RS_PMAX], ub[RS_PMAX + 1], scl[RS_PMAX + 1];
    __shared__ double red[64];
    __shared__ PwTree<PW_MAXNODES> tree;
    __shared__ double pwval[PW_MAXNODES];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t *gcnt = gcnt_all ? gcnt_all + (size_t)blockIdx.x * (NB + 1) : cnt;
    uint32_t *grank = grank_all + (size_t)blockIdx.x * n;
    int32_t *gidx = gidx_all + (size_t)blockIdx.x * n;
    if (rowsum) {
        int *height = reinterpret_cast<int *>(pwval);
        if (tid == 0) pw_plan(tree, n, height);
        __syncthreads();
    }
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const double *row = S + v * n64;
        for (int b = tid; b <= NB; b += RS_T) gcnt[b] = 0;
        double mn = INFINITY, mx = -INFINITY;
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double x = __ldg(row + j);
            if (x < mn) mn = x;
            if (x > mx) mx = x;
        }
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) { red[warp] = mn; red[32 + warp] = mx; }
        __syncthreads();
        if (warp == 0) {
            double a = red[lane], b = red[32 + lane];
            for (int o = 16; o; o >>= 1) {
                a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
                b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
            }
            double xs[2];
            unsigned long long ks[2];
            for (int q = 0; q < 2; q++) {
                int k = lane + 32 * q;
                double x = 0.0;
                if (k < P) {
                    int j = (int)(((int64_t)(2 * k + 1) * n) / (2 * P));
                    if (j >= n) j = n - 1;
                    if (j == v) j = (j + 1 < n) ? j + 1 : j - 1;
                    x = row[j];
                }
                xs[q] = x;
                ks[q] = isnan(x) ? 0ull : tg_order_key(x);
            }
            for (int q = 0; q < 2; q++) {
                int k = lane + 32 * q;
                int rank = 0;
                for (int mm = 0; mm < 64; mm++) {
                    unsigned long long km = __shfl_sync(0xffffffffu, ks[mm >> 5], mm & 31);
                    if (mm < P) rank += (km > ks[q]) || (km == ks[q] && mm < k);
                }
                if (k < P) spl[rank] = xs[q];
            }
            __syncwarp();
            for (int c = lane; c <= P; c += 32) {
                double u = (c == 0) ? b : spl[c - 1];
                double l = (c == P) ? a : spl[c];
                double w = u - l;
                ub[c] = u;
                scl[c] = (w > 0.0 && w < INFINITY) ? (double)K / w : 0.0;
            }
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            double x = __ldg(row + j);
            int b;
            if (isnan(x)) {
                b = NB - 1;
            } else {
                int lo = 0, hi = P;
                while (lo < hi) {
                    int mid = (lo + hi) >> 1;
                    if (spl[mid] > x) lo = mid + 1;
                    else hi = mid;
                }
                double t = (ub[lo] - x) * scl[lo];
                int sub = (t >= 0.0) ? (t < (double)K ? (int)t : K - 1) : 0;
                b = lo * K + sub;
            }
            uint32_t r = atomicAdd(&gcnt[b], 1u);
            grank[j] = (uint32_t)b;
            gidx[j] = (int32_t)r;  // temporarily: rank within bucket
        }
        __syncthreads();
        // exclusive scan over NB+1 counters
        {
            const int per = (NB + 1 + RS_T - 1) / RS_T;
            int b0 = tid * per;
            uint32_t s = 0;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b <= NB) s += gcnt[b];
            }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            __shared__ uint32_t wsum[32];
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                uint32_t w = wsum[lane];
                uint32_t wi = w;
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                    if (lane >= o) wi += y;
                }
                wsum[lane] = wi - w;
            }
            __syncthreads();
            uint32_t run = wsum[warp] + incl - s;
            for (int q = 0; q < per; q++) {
                int b = b0 + q;
                if (b <= NB) {
                    uint32_t c = gcnt[b];
                    gcnt[b] = run;
                    run += c;
                }
            }
        }
        __syncthreads();
        // scatter into the output row directly (it is the scatter buffer)
        int32_t *out = order + v * (int64_t)m;
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            out[gcnt[grank[j]] + (uint32_t)gidx[j]] = j;
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            const int b = (int)grank[j];
            const int s0 = (int)gcnt[b], s1 = (int)gcnt[b + 1];
            int rank = 0;
            if (s1 - s0 > 1) {
                const double xj = __ldg(row + j);
                for (int k = s0; k < s1; k++) {
                    const int o = out[k];
                    rank += rs_before(__ldg(row + o), o, xj, j);
                }
            }
            gidx[j] = s0 + rank;
        }
        __syncthreads();
        for (int j = tid; j < n; j += RS_T) {
            if (j == v) continue;
            out[gidx[j]] = j;
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
    int sms = tg_num_sms();
    int m = (int)n - 1;
    int P = RS_PMAX;
    int K = (m + 2 * (P + 1) - 1) / (2 * (P + 1));
    size_t NB = (size_t)(P + 1) * K;
    return (size_t)sms * ((NB + 1) * 4 + (size_t)n * 8) + 4096;
}

TG_API int tg_row_sort_f64(const double *S, int64_t n, int32_t *order, double *rowsum, void *ws, size_t ws_bytes,
                           void *stream) {
    if (n < 2 || !S || !order) return TG_ERR_ARG;
    cudaStream_t st = tg_stream(stream);
    if (n <= 16384) {
        RsPlan pl = rs_plan(n, 2);
        if (pl.smem > RS_SMEM_MAX) pl = rs_plan(n, 1);
        if (pl.smem > RS_SMEM_MAX) return TG_ERR_ARG;
        int E = (int)((n + RS_T - 1) / RS_T);
        int grid = tg_num_sms();
        if (grid > n) grid = (int)n;
#define RS_LAUNCH(EM)                                                                                      \
    do {                                                                                                   \
        auto kfn = row_sort_smem_kernel<EM>;                                                               \
        TG_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem)); \
        kfn<<<grid, RS_T, pl.smem, st>>>(S, n, order, rowsum, pl);                                         \
    } while (0)
        if (E <= 2) RS_LAUNCH(2);
        else if (E <= 4) RS_LAUNCH(4);
        else if (E <= 8) RS_LAUNCH(8);
        else RS_LAUNCH(16);
#undef RS_LAUNCH
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    if (n > 65535 * 16) return TG_ERR_ARG;
    if (ws_bytes < tg_row_sort_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    int m = (int)n - 1;
    int P = RS_PMAX;
    int K = (m + 2 * (P + 1) - 1) / (2 * (P + 1));
    int NB = (P + 1) * K;
    int grid = tg_num_sms();
    TgArena ar(ws, ws_bytes);
    size_t smem_cnt = (size_t)(NB + 1) * 4;
    bool cnt_in_smem = smem_cnt <= 160 * 1024;
    uint32_t *gcnt = cnt_in_smem ? nullptr : ar.take<uint32_t>((size_t)grid * (NB + 1));
    uint32_t *grank = ar.take<uint32_t>((size_t)grid * n);
    int32_t *gidx = ar.take<int32_t>((size_t)grid * n);
    if (!grank || !gidx || (!cnt_in_smem && !gcnt)) return TG_ERR_WORKSPACE;
    size_t smem = cnt_in_smem ? smem_cnt : 16;
    TG_CUDA_CHECK(cudaFuncSetAttribute(row_sort_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    row_sort_global_kernel<<<grid, RS_T, smem, st>>>(S, n, order, rowsum, P, K, NB, gcnt, grank, gidx);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_row_sums_workspace_bytes(int64_t) { return 256; }

TG_API int tg_row_sums_f64(const double *S, int64_t n, double *rowsum, void *, size_t, void *stream) {
    if (n < 1 || !S || !rowsum) return TG_ERR_ARG;
    if (n > 128 * (PW_MAXNODES / 2)) return TG_ERR_ARG;
    int grid = tg_num_sms() * 4;
    if (grid > n) grid = (int)n;
    row_sums_kernel<<<grid, 256, 0, tg_stream(stream)>>>(S, n, rowsum);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_initial_clique(const double *rowsum, int64_t n, int32_t *clique, void *stream) {
    if (n < 4 || !rowsum || !clique) return TG_ERR_ARG;
    clique_kernel<<<1, 1024, 0, tg_stream(stream)>>>(rowsum, n, clique);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
