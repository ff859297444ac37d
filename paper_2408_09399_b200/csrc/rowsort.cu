// rowsort.cu -- the aggregated per-row neighbour sort and the initial-clique row sums.
//
// Replaces simmatrix.py:225-249 sort_neighbor_lists (per row v: ids by (S desc,
// id asc), v removed; numpy argsort + lexsort tie rule) and tmfg.py:71-79
// select_initial_clique (numpy pairwise row sums, stable top-4).
//
// B200 design (details at each kernel):
//   * n <= 24,576: row_sort_fk_kernel -- one 1024-thread CTA per SM, persistent over
//     rows, rows arriving by TMA bulk copies into two recycled row buffers; float keys,
//     an equalised two-level bucket map, one packed-u16 shared atomic per key, a block
//     scan, and the exact in-bucket rank by sorted position (warp shuffles); the same
//     pass emits the initial-clique row-sum screen;
//   * n > 24,576: row_part_kernel (value-bin partition of each row into segments of
//     <= 12,288 keys, through a scratch row) + row_seg_kernel (the same bucket sort per
//     segment in shared memory);
//   * rows with NaN / values outside [-1, 1] / one dominant value bin at n > 24,576:
//     row_sort_global_kernel (the bucket algorithm with the row in L2).
// The result is deterministic although the atomic arrival ranks are not: positions come
// from bucket offsets plus exact ranks (value desc, id asc, -0.0 == +0.0, NaN last).
#include "common.cuh"

#include <cmath>
#include <cstdlib>

namespace {

constexpr int RS_T = 1024;
constexpr int PW_MAXNODES = 2048;   // n <= 131072

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
__host__ __device__ int pw_build(PwTree<N> &t, int off, int len, int *height) {
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
__host__ __device__ void pw_plan(PwTree<N> &t, int n, int *height) {
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

// rowsum[k] = pairwise_sum(S[v]) - S[v, v] for v = rows[k] (rows == NULL: v = k, k < n)
// (the plan is built on the host and passed by value, copied to shared memory)
__global__ void row_sums_kernel(const double *__restrict__ S, int64_t n, double *__restrict__ rowsum,
                                const int32_t *__restrict__ rows, const int32_t *__restrict__ nrows,
                                const __grid_constant__ PwTree<PW_MAXNODES> plan) {
    __shared__ PwTree<PW_MAXNODES> tree;
    __shared__ double val[PW_MAXNODES];
    for (int i = threadIdx.x; i < plan.nnodes; i += blockDim.x) {
        tree.a[i] = plan.a[i];
        tree.b[i] = plan.b[i];
        tree.lvl[i] = plan.lvl[i];
    }
    if (threadIdx.x < 33) tree.lvl_off[threadIdx.x] = plan.lvl_off[threadIdx.x];
    if (threadIdx.x == 0) { tree.nnodes = plan.nnodes; tree.nlevels = plan.nlevels; tree.root = plan.root; }
    __syncthreads();
    const int64_t cnt = rows ? (int64_t)*nrows : n;
    for (int64_t k = blockIdx.x; k < cnt; k += gridDim.x) {
        const int64_t v = rows ? (int64_t)rows[k] : k;
        const double *row = S + v * n;
        double root = pw_eval(tree, val, [&](int i) { return __ldg(row + i); });
        if (threadIdx.x == 0) rowsum[k] = __dsub_rn(root, row[v]);
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

// top-4 of (sum desc, id asc) over rowsum[k], id = rows ? rows[k] : k
__global__ void clique_kernel(const double *__restrict__ rowsum, int64_t n, int32_t *__restrict__ out,
                              const int32_t *__restrict__ rows, const int32_t *__restrict__ nrows) {
    __shared__ double bs[32];
    __shared__ int64_t bi[32];
    __shared__ int64_t chosen[4];
    const int64_t cnt = rows ? (int64_t)*nrows : n;
    for (int k = 0; k < 4; k++) {
        double best = 0.0;
        int64_t bid = -1;
        for (int64_t kk = threadIdx.x; kk < cnt; kk += blockDim.x) {
            const int64_t i = rows ? (int64_t)rows[kk] : kk;
            bool used = false;
            for (int q = 0; q < k; q++) used |= (chosen[q] == i);
            if (used) continue;
            double s = rowsum[kk];
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

// Candidates for the initial clique from the sort's row-sum screen: screen[v] is
// the row sum in any summation order and screen[n + v] bounds its distance to
// numpy's pairwise result, so the exact sum lies in [lo_v, hi_v].  With L4 the
// 4th largest lo, a row with hi_v < L4 has 4 rows strictly above it and cannot
// be chosen; the rest (normally 4-6 rows) get exact pairwise sums.  Any NaN in
// the screen makes every row a candidate (numpy's NaN ordering is then exact).
__global__ void clique_screen_kernel(const double *__restrict__ screen, int64_t n, int32_t *__restrict__ cand,
                                     int32_t *__restrict__ ncand) {
    __shared__ double bs[32];
    __shared__ int64_t bi[32];
    __shared__ int64_t chosen[4];
    __shared__ double l4;
    __shared__ int cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    bool nan_seen = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        nan_seen |= isnan(screen[i]) | isnan(screen[n + i]);
    const bool any_nan = __syncthreads_or(nan_seen);
    if (threadIdx.x == 0) { cnt = 0; l4 = -INFINITY; }
    if (!any_nan) {
        for (int k = 0; k < 4; k++) {
            double best = -INFINITY;
            int64_t bid = -1;
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                bool used = false;
                for (int q = 0; q < k; q++) used |= (chosen[q] == i);
                if (used) continue;
                double lo = screen[i] - screen[n + i];
                if (lo != lo) lo = -INFINITY;   // inf - inf
                if (bid < 0 || lo > best) { best = lo; bid = i; }
            }
            for (int o = 16; o; o >>= 1) {
                const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
                const int64_t i2 = __shfl_xor_sync(0xffffffffu, bid, o);
                if (i2 >= 0 && (bid < 0 || b2 > best)) { best = b2; bid = i2; }
            }
            if (lane == 0) { bs[warp] = best; bi[warp] = bid; }
            __syncthreads();
            if (threadIdx.x == 0) {
                double b0 = -INFINITY;
                int64_t i0 = -1;
                for (int w = 0; w < (int)(blockDim.x >> 5); w++)
                    if (bi[w] >= 0 && (i0 < 0 || bs[w] > b0)) { b0 = bs[w]; i0 = bi[w]; }
                chosen[k] = i0;
                l4 = b0;
            }
            __syncthreads();
        }
    }
    __syncthreads();
    const double L4 = l4;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        if (any_nan || !(screen[i] + screen[n + i] < L4)) cand[atomicAdd(&cnt, 1)] = (int32_t)i;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ncand = cnt;
}

// Radius of the row-sum screen.  Recursive/tree summation of depth d is within
// gamma_d * sum|x| of the exact sum (gamma_d ~ d u, u = 2^-53).  Depth here:
// ceil(n/1024) per thread + 10 shuffle/block levels; numpy's pairwise tree: 16
// per accumulator + 3 + log2(n/128) + 1 <= 40; the final "- diagonal" adds <= 4u.
// Radius = 8x that sum of depths (+ 50) times u ~ 1.1e-16 -> 9e-16 per level.
__device__ __forceinline__ double rs_screen_radius(int n, double abs_sum) {
    return (double)((n + 1023) / 1024 + 60) * 9e-16 * abs_sum;
}
__device__ __forceinline__ double rs_screen_radius_t(int n, int threads, double abs_sum) {
    return (double)((n + threads - 1) / threads + 60) * 9e-16 * abs_sum;
}

struct RsMisc {
    double red[128];
    double rmin, rmax, cscale;
    uint32_t ccnt[RS_CMAX + 1];    // coarse counts -> fine base (exclusive scan of f_c)
    uint32_t cf[RS_CMAX];          // fine buckets per coarse bin
    uint32_t wsum[32];
    uint32_t nsamp;
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
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

#ifndef RS_DEBUG_PHASES
#define RS_DEBUG_PHASES 0
#endif
#if RS_DEBUG_PHASES
__device__ long long g_rs_phase[8];
#endif
__device__ __forceinline__ unsigned rt_smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void rt_bulk_row(double *buf, const double *row, int n, uint64_t *bar) {
    // thread 0 only: 16-byte-aligned body by TMA, the unaligned edge doubles by cp.async
    const int sh = (int)(((uintptr_t)row >> 3) & 1);
    double *vals = buf + sh;
    const int cnt2 = (n - sh) & ~1;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(rt_smem_u32(bar)),
                 "r"((unsigned)(cnt2 * 8))
                 : "memory");
    if (cnt2 > 0)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                         rt_smem_u32(vals + sh)),
                     "l"(row + sh), "r"((unsigned)(cnt2 * 8)), "r"(rt_smem_u32(bar))
                     : "memory");
    if (sh) cp_async8(vals, row);
    if (sh + cnt2 < n) cp_async8(vals + n - 1, row + n - 1);
    // second arrival of the phase: when this thread's cp.async copies have landed
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(rt_smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void rt_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n RT_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra RT_WAIT_%=;\n}\n" ::"r"(rt_smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---------------------------------------------------------------- float-key kernel
// The production sort for n <= FK_NMAX: one 1024-thread CTA per SM, persistent over rows.
//  * bucket arithmetic runs on float keys: fl(x) is monotone (non-strictly) in x,
//    and so is every float step of the bucket map, so bucket(x) is monotone and
//    equal doubles share a bucket; float-EQUAL keys are ordered by their doubles
//    re-read through L2 (only ties at float precision take that path);
//  * a row buffer is recycled: after the first pass the keys live in registers
//    as floats and the buffer holds the float keys (4n B) and the (bucket, id)
//    scatter array (4n B).  With two buffers (n <~ 12.5k) the TMA load of the
//    next row is issued as soon as the current row's doubles are consumed;
//  * correlation rows (every off-diagonal value in [-1, 1], no NaN) use the
//    fixed coarse map t = (1 - f) * C/2 -- no min/max reduction; other rows use
//    their float range, NaN keys go to the last bucket and are ordered exactly
//    (a separate instantiation, so the common path carries no NaN logic);
//  * float -> integer steps use the 1.5 * 2^23 magic add (round to nearest, a
//    monotone map) on the FMA pipe; coarse bin c covers t in [c - 1/2, c + 1/2],
//    d = t - c is exact, and fb = rn(d f_c + base_c + f_c / 2) lies in
//    [base_c, base_c + f_c], so the map stays monotone across bins;
//  * the coarse bins get fine buckets in proportion to a 1/4-sample histogram
//    (up to 3 per key), one packed-u16 shared atomic per key gives bucket +
//    arrival rank, a block scan the offsets, the (bucket, id) pairs are scattered;
//  * the exact rank inside a bucket runs by sorted POSITION: a bucket's members
//    are consecutive lanes of a warp, their keys come by shuffles; buckets that
//    cross a warp boundary walk shared memory.
constexpr int FK_T = 1024;
constexpr float FK_MAGIC = 12582912.0f;   // 1.5 * 2^23: x + MAGIC has rn(x) in its low 22 bits

struct FkPlan {
    int n, C, NBcap, stride, nbuf;
    float fs, hc;
    size_t off_sidx, off_cinfo, off_misc, off_bar, off_f16, smem;
    size_t off_sid;   // segments: slot -> id table (row_seg_kernel)
};

struct FkMisc {
    double rsum[32], rabs[32];
    float rmn[32], rmx[32];
    uint32_t wsum[32];
    double diag;
    int nb;
};

__host__ FkPlan fk_plan(int64_t n, int nbuf, size_t smem_max, double fs_cap) {
    FkPlan p;
    p.n = (int)n;
    p.nbuf = nbuf;
    const int m = (int)n - 1;
    p.C = rs_coarse_bins(m);   // coarse bins 0..C (C + 1 of them)
    p.hc = 0.5f * (float)p.C;
    p.stride = (int)((n + 2) & ~1LL);
    p.off_sidx = tg_align_up((size_t)n * sizeof(float), 16);
    {
        const int need = (int)((p.off_sidx + ((size_t)n + 64) * 4 + 15) / 8);   // + sentinel pad
        if (p.stride < need) p.stride = (need + 1) & ~1;
    }
    size_t off = (size_t)nbuf * p.stride * sizeof(double);
    p.off_cinfo = tg_align_up(off, 16);
    off = p.off_cinfo + (size_t)(p.C + 1) * sizeof(float2);
    p.off_misc = tg_align_up(off, 16);
    off = p.off_misc + sizeof(FkMisc);
    p.off_bar = tg_align_up(off, 16);
    off = p.off_bar + 16;
    p.off_f16 = tg_align_up(off, 16);
    const size_t fixed = p.off_f16 + 64;
    double room = smem_max > fixed ? (double)(smem_max - fixed) / 2.0 : 0.0;   // u16 entries
    double fs = (room - 2.0 * p.C - 16.0) / (double)(m > 0 ? m : 1);
    if (fs > fs_cap) fs = fs_cap;
    p.fs = (float)fs;
    p.NBcap = 2 * (p.C + 1) + (int)std::ceil(fs * m) + 4;
    p.smem = p.off_f16 + (size_t)(p.NBcap / 2 + 2 + 16) * sizeof(uint32_t);
    if (fs < 0.45 || p.NBcap >= 65535) p.smem = (size_t)-1;
    return p;
}

__device__ __forceinline__ int fk_rni(float x) {   // rn(x) for 0 <= x < 2^22
    return __float_as_int(x + FK_MAGIC) & 0x3fffff;
}

// coarse bin of key f: rn((hi - f) * scale) in [0, C]; general rows clamp, NaN -> C
template <bool ODD>
__device__ __forceinline__ int fk_coarse(float f, float hs, float scale, int C) {
    const float t = fmaf(f, -scale, hs);
    if (!ODD) return fk_rni(t);
    if (f != f) return C;
    const float tc = fminf(fmaxf(t, 0.0f), (float)C);
    return fk_rni(tc);
}

struct FkRow {
    float *fkey;
    uint32_t *sidx, *f16;
    float2 *cinfo;
    uint32_t *ccnt;
    FkMisc *ms;
    const double *row;
    int32_t *out;
    const int32_t *sid;   // slot -> column id (segments); nullptr: the slot is the id
    int n, m, vi, C, nsamp;
    float fs, hc;
};

// phases 2-5 of one row; ODD: rows with NaN or values outside [-1, 1]
template <bool ODD, int KPT>
__device__ __forceinline__ void fk_row(const FkRow &R, const float (&fk)[KPT]) {
    constexpr int NT = FK_T, W = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = R.n, m = R.m, vi = R.vi, C = R.C;
    float *fkey = R.fkey;
    uint32_t *sidx = R.sidx, *f16 = R.f16, *ccnt = R.ccnt;
    float2 *cinfo = R.cinfo;
    const uint16_t *o16 = reinterpret_cast<const uint16_t *>(f16);
    FkMisc &ms = *R.ms;
    float hs = R.hc, scale = R.hc;   // t = hs - f * scale
    if (ODD) {   // the row's float range, histogram again
        float fmn = INFINITY, fmx = -INFINITY;
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            const int j = tid + e * NT;
            if (j < n && j != vi) { fmn = fminf(fmn, fk[e]); fmx = fmaxf(fmx, fk[e]); }
        }
        for (int o = 16; o; o >>= 1) {
            fmn = fminf(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
            fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        }
        if (lane == 0) { ms.rmn[warp] = fmn; ms.rmx[warp] = fmx; }
        for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;
        __syncthreads();
        float lo = INFINITY, hi = -INFINITY;
        for (int w = 0; w < W; w++) { lo = fminf(lo, ms.rmn[w]); hi = fmaxf(hi, ms.rmx[w]); }
        const float wd = hi - lo;
        scale = (wd > 0.0f && wd < INFINITY) ? (float)C / wd : 0.0f;
        if (!(hi < INFINITY && hi > -INFINITY)) hi = 0.0f;
        hs = hi * scale;
#pragma unroll
        if (R.sid) {   // segment slots are grouped by value: sample every 4th slot (threads 4k)
            if ((tid & 3) == 0) {
#pragma unroll
                for (int e = 0; e < KPT; e++) {
                    const int j = tid + e * NT;
                    if (j < n) atomicAdd(&ccnt[fk_coarse<true>(fk[e], hs, scale, C)], 1u);
                }
            }
        } else {
#pragma unroll
            for (int e = 0; e < KPT; e += 4) {
                const int j = tid + e * NT;
                if (j < n && j != vi) atomicAdd(&ccnt[fk_coarse<true>(fk[e], hs, scale, C)], 1u);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < KPT; e++) {
        const int j = tid + e * NT;
        if (j < n) fkey[j] = fk[e];
    }
    // ---- 2: fine buckets per coarse bin (one thread per bin) -> per-bin (A, B)
    {
        const float fsc = (float)m * R.fs / (float)(R.nsamp > 0 ? R.nsamp : 1) * 0.9999f;
        const uint32_t f = tid <= C ? 1u + (uint32_t)((float)ccnt[tid] * fsc) : 0u;
        uint32_t incl = f;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) ms.wsum[warp] = incl;
        __syncthreads();   // B2
        if (tid <= C) {
            uint32_t off = 0;
            for (int w = 0; w < warp; w++) off += ms.wsum[w];
            const uint32_t base = off + incl - f;
            // d = t - c in [-1/2, 1/2] (exact): fb = rn(d f + base + f/2) in [base, base + f]
            cinfo[tid] = make_float2((float)base + 0.5f * (float)f, (float)f);
            if (tid == C) ms.nb = (int)(base + f) + 1;
        }
    }
    __syncthreads();   // B3
    // ---- 3: fine bucket + arrival rank (one packed-u16 shared atomic per key)
    uint32_t pk[KPT];
    const int nan_fb = ms.nb - 1;
#pragma unroll
    for (int e = 0; e < KPT; e++) {
        const int j = tid + e * NT;
        pk[e] = 0xffffffffu;
        if (j < n && j != vi) {
            const float f = fk[e];
            float t = fmaf(f, -scale, hs);
            if (ODD) t = fminf(fmaxf(t, 0.0f), (float)C);
            const float y = t + FK_MAGIC;
            const int c = __float_as_int(y) & 0x3fffff;
            const float d = t - (y - FK_MAGIC);   // exact
            const float2 ab = cinfo[c];
            int fb = fk_rni(fmaf(d, ab.y, ab.x));
            if (ODD && f != f) fb = nan_fb;
            const uint32_t sh = (fb & 1) << 4;
            const uint32_t old = atomicAdd(&f16[fb >> 1], 1u << sh);
            pk[e] = __byte_perm((uint32_t)fb, old >> sh, 0x1054);   // (fb << 16) | (old >> sh) & 0xffff
        }
    }
    __syncthreads();   // B4
    for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;   // next row's histogram (cinfo is dead)
    // ---- 4: exclusive scan of the packed counters, scatter (bucket, id)
    {
        const int nw = (ms.nb + 2) >> 1;
        const int per = (nw + NT - 1) / NT;
        const int w0 = tid * per;
        uint32_t s = 0;
        for (int q = 0; q < per; q++) {
            const int w = w0 + q;
            if (w < nw) { const uint32_t x = f16[w]; s += (x + (x << 16)) >> 16; }
        }
        uint32_t incl = s;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) ms.wsum[warp] = incl;
        __syncthreads();   // B5
        uint32_t wex;
        {
            const uint32_t wv = ms.wsum[lane];
            uint32_t wi = wv;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            wex = __shfl_sync(0xffffffffu, wi - wv, warp);
        }
        uint32_t run = wex + incl - s;
        for (int q = 0; q < per; q++) {
            const int w = w0 + q;
            if (w < nw) {
                const uint32_t x = f16[w];
                f16[w] = run * 0x10001u + (x << 16);    // (run, run + lo)
                run += (x + (x << 16)) >> 16;           // lo + hi
            }
        }
    }
    __syncthreads();   // B6
#pragma unroll
    for (int e = 0; e < KPT; e++) {
        if (pk[e] != 0xffffffffu)
            sidx[o16[pk[e] >> 16] + (pk[e] & 0xffffu)] = (pk[e] & 0xffff0000u) | (uint32_t)(tid + e * NT);
    }
    if (tid < 64) sidx[m + tid] = 0xffff0000u;   // sentinel bucket past the last position (never a real one)
    __syncthreads();   // B7
    // ---- 5: exact rank inside the bucket by sorted position, coalesced id store
    const double *row = R.row;
    int32_t *out = R.out;
    const int32_t *sid = R.sid;
    if (!ODD) {
        // Positions kb..kb+31 in the lanes; a bucket's members are a run of lanes.  Runs
        // inside the window rank by shuffles; a run touching the window edge whose bucket
        // continues outside (sentinel-padded reads of positions kb-1 / kb+32) walks its
        // bucket in shared memory.  Float ties go to the doubles.
        const unsigned le = 0xffffffffu >> (31 - lane), lt = le >> 1;
        for (int kb = warp * 32; kb < m; kb += NT) {
            const int k = kb + lane;
            const uint32_t sk = sidx[k];
            const uint32_t pv = kb > 0 ? sidx[kb - 1] : 0xfffe0000u;   // uniform address: broadcast
            const uint32_t nv = sidx[kb + 32];
            const int fb = (int)(sk >> 16), j = (int)(sk & 0xffffu);
            const float fj = fkey[j];
            const int fprev = __shfl_up_sync(0xffffffffu, fb, 1);
            const int fnext = __shfl_down_sync(0xffffffffu, fb, 1);
            const unsigned S0 = __ballot_sync(0xffffffffu, fprev != fb) | 1u;
            const unsigned E0 = __ballot_sync(0xffffffffu, fnext != fb) | 0x80000000u;
            const int first = 31 - __clz(S0 & le);
            const int last = __ffs(E0 & ~lt) - 1;
            const int sz = last - first + 1;
            const bool cross = (first == 0 && (int)(pv >> 16) == fb) || (last == 31 && (int)(nv >> 16) == fb);
            const int smax = __reduce_max_sync(0xffffffffu, cross ? 1 : sz);
            int rank = 0, ties = 0;
#pragma unroll 1
            for (int i = 0; i < smax; i++) {
                const float fo = __shfl_sync(0xffffffffu, fj, first + i);
                const bool in = i < sz;
                rank += in & (fo > fj);
                ties += in & (fo == fj);
            }
            int pos = kb + first + rank;
            if ((cross || ties > 1) && k < m) {   // rare: walk the bucket in shared memory
                const int s0 = o16[fb], s1 = o16[fb + 1];
                const int idj = sid ? sid[j] : j;
                double xj = 0.0;
                bool have = false;
                rank = 0;
                for (int q = s0; q < s1; q++) {
                    const int o = (int)(sidx[q] & 0xffffu);
                    if (o == j) continue;
                    const float fo = fkey[o];
                    if (fo != fj) {
                        rank += fo > fj;
                    } else {   // float tie: the doubles decide, then the id
                        if (!have) { xj = __ldg(row + idj); have = true; }
                        const int ido = sid ? sid[o] : o;
                        rank += rs_before(__ldg(row + ido), ido, xj, idj);
                    }
                }
                pos = s0 + rank;
            }
            if (k < m) out[pos] = sid ? sid[j] : j;
        }
        return;
    }
    for (int kb = warp * 32; kb < m; kb += NT) {
        const int k = kb + lane;
        const bool live = k < m;
        const uint32_t sk = live ? sidx[k] : (0xfffe0000u | (uint32_t)lane);
        const int fb = (int)(sk >> 16), j = (int)(sk & 0xffffu);
        const float fj = fkey[j];
        // the bucket's lanes: a run of equal fb (positions are bucket-sorted)
        const int fprev = __shfl_up_sync(0xffffffffu, fb, 1);
        const unsigned starts = __ballot_sync(0xffffffffu, lane == 0 || fprev != fb);
        const unsigned le = 0xffffffffu >> (31 - lane);   // lanes <= lane
        const int first = 31 - __clz(starts & le);
        const unsigned above = starts & ~le;
        const int sz = (above ? __ffs(above) - 1 : 32) - first;
        // does the first run continue before lane 0, the last one after lane 31?
        bool cross = false;
        if (first == 0 && kb > 0) cross = (int)(sidx[kb - 1] >> 16) == fb;
        if (first + sz == 32 && kb + 32 < m) cross |= (int)(sidx[kb + 32] >> 16) == fb;
        const int smax = __reduce_max_sync(0xffffffffu, (live && !cross) ? sz : 1);
        int rank = 0, ties = 0;
        for (int i = 0; i < smax; i++) {
            const float fo = __shfl_sync(0xffffffffu, fj, first + i);
            const bool in = i < sz;
            if (!ODD) {
                rank += in & (fo > fj);
                ties += in & (fo == fj);
            } else {
                const bool no = fo != fo, nj = fj != fj;
                rank += in & ((fo > fj) | (nj & !no));
                ties += in & ((fo == fj) | (nj & no));
            }
        }
        if (live) {
            int pos;
            if (!cross) {
                pos = kb + first + rank;
                if (ties > 1) {   // float ties (itself included): order by the doubles, then id
                    const int idj = sid ? sid[j] : j;
                    const double xj = __ldg(row + idj);
                    rank = 0;
                    for (int i = 0; i < sz; i++) {
                        const int q = kb + first + i;
                        if (q == k) continue;
                        const int o = (int)(sidx[q] & 0xffffu);
                        const int ido = sid ? sid[o] : o;
                        rank += rs_before(__ldg(row + ido), ido, xj, idj);
                    }
                    pos = kb + first + rank;
                }
            } else {
                const int s0 = o16[fb], s1 = o16[fb + 1];
                rank = 0;
                int tie = 0;
                for (int q = s0; q < s1; q++) {
                    const float fo = fkey[sidx[q] & 0xffffu];
                    if (!ODD) {
                        rank += fo > fj;
                        tie += fo == fj;
                    } else {
                        const bool no = fo != fo, nj = fj != fj;
                        rank += (fo > fj) | (nj & !no);
                        tie += (fo == fj) | (nj & no);
                    }
                }
                if (tie > 1) {
                    const int idj = sid ? sid[j] : j;
                    const double xj = __ldg(row + idj);
                    rank = 0;
                    for (int q = s0; q < s1; q++) {
                        const int o = (int)(sidx[q] & 0xffffu);
                        const int ido = sid ? sid[o] : o;
                        if (o != j) rank += rs_before(__ldg(row + ido), ido, xj, idj);
                    }
                }
                pos = s0 + rank;
            }
            out[pos] = sid ? sid[j] : j;
        }
    }
}

template <int KPT>
__global__ void __launch_bounds__(FK_T, 1)
row_sort_fk_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                   double *__restrict__ screen, FkPlan pl) {
    extern __shared__ __align__(16) unsigned char fk_smem[];
    constexpr int NT = FK_T, W = NT / 32;
    const int n = (int)n64;
    const int m = n - 1;
    uint32_t *ccnt = reinterpret_cast<uint32_t *>(fk_smem + pl.off_cinfo);   // histogram, then (A, B)
    FkMisc &ms = *reinterpret_cast<FkMisc *>(fk_smem + pl.off_misc);
    uint64_t *bar = reinterpret_cast<uint64_t *>(fk_smem + pl.off_bar);
    uint32_t *f16 = reinterpret_cast<uint32_t *>(fk_smem + pl.off_f16);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = pl.C;
    const int nw16 = pl.NBcap / 2 + 2;
    const size_t bstride = (size_t)pl.stride * sizeof(double);

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(rt_smem_u32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(rt_smem_u32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;
    __syncthreads();
    int64_t v = blockIdx.x;
    if (tid == 0 && v < n) rt_bulk_row(reinterpret_cast<double *>(fk_smem), S + v * n64, n, &bar[0]);
    int nsamp_all = 0;   // sampled keys: e % 4 == 0
#pragma unroll
    for (int e = 0; e < KPT; e += 4) {
        const int r = n - e * NT;
        nsamp_all += r < 0 ? 0 : (r < NT ? r : NT);
    }
    FkRow R;
    R.f16 = f16;
    R.cinfo = reinterpret_cast<float2 *>(ccnt);
    R.ccnt = ccnt;
    R.ms = &ms;
    R.n = n;
    R.m = m;
    R.C = C;
    R.fs = pl.fs;
    R.hc = pl.hc;
#if RS_DEBUG_PHASES
    long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long pt = clock64();
#define FK_PH(k) do { if (tid == 0) { const long long now = clock64(); ph[k] += now - pt; pt = now; } } while (0)
#else
#define FK_PH(k) do {} while (0)
#endif
    for (int it = 0; v < n; v += gridDim.x, it++) {
        const int b = pl.nbuf == 2 ? (it & 1) : 0;
        const unsigned parity = pl.nbuf == 2 ? (unsigned)((it >> 1) & 1) : (unsigned)(it & 1);
        unsigned char *buf = fk_smem + (size_t)b * bstride;
        const double *row = S + v * n64;
        const double *vals = reinterpret_cast<const double *>(buf) + (((uintptr_t)row >> 3) & 1);
        const int vi = (int)v;
        rt_wait(&bar[b], parity);
        FK_PH(0);
        // ---- 1: doubles -> float keys (registers), screen sums, sampled coarse histogram
        for (int i = tid; i < nw16; i += NT) f16[i] = 0u;
        float fk[KPT];
        double sm = 0.0, sa = 0.0;
        bool odd = false;
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            const int j = tid + e * NT;
            fk[e] = 0.0f;
            if (j < n) {
                const double x = vals[j];
                sm += x;
                sa += fabs(x);
                const float f = __double2float_rn(x);
                fk[e] = f;
                if (j != vi) {
                    odd |= !(fabsf(f) <= 1.0f);   // NaN or outside [-1, 1] at float precision
                    if ((e & 3) == 0) atomicAdd(&ccnt[fk_coarse<true>(f, pl.hc, pl.hc, C)], 1u);
                } else {
                    ms.diag = x;
                }
            }
        }
        if (screen) {
            for (int o = 16; o; o >>= 1) {
                sm += __shfl_xor_sync(0xffffffffu, sm, o);
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
            }
            if (lane == 0) { ms.rsum[warp] = sm; ms.rabs[warp] = sa; }
        }
        const bool row_odd = __syncthreads_or(odd);   // B1: every double of the row is consumed
        if (tid == 0) {
            const int64_t vn = v + gridDim.x;
            if (pl.nbuf == 2 && vn < n)
                rt_bulk_row(reinterpret_cast<double *>(fk_smem + (size_t)(b ^ 1) * bstride), S + vn * n64, n,
                            &bar[b ^ 1]);
        }
        if (screen && warp == W - 1) {
            double s1 = ms.rsum[lane], s2 = ms.rabs[lane];
            for (int o = 16; o; o >>= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            }
            if (lane == 0) {
                screen[vi] = __dsub_rn(s1, ms.diag);
                screen[n + vi] = rs_screen_radius_t(n, NT, s2);
            }
        }
        FK_PH(1);
        R.fkey = reinterpret_cast<float *>(buf);
        R.sidx = reinterpret_cast<uint32_t *>(buf + pl.off_sidx);
        R.row = row;
        R.out = order + v * (int64_t)m;
        R.sid = nullptr;
        R.vi = vi;
        R.nsamp = nsamp_all - (((vi / NT) & 3) == 0 ? 1 : 0);
        if (row_odd) fk_row<true, KPT>(R, fk);
        else fk_row<false, KPT>(R, fk);
        __syncthreads();   // B8: buffer b and the counters are free
        FK_PH(6);
        if (tid == 0 && pl.nbuf == 1) {
            const int64_t vn = v + gridDim.x;
            if (vn < n) rt_bulk_row(reinterpret_cast<double *>(fk_smem), S + vn * n64, n, &bar[0]);
        }
    }
#if RS_DEBUG_PHASES
    if (tid == 0)
        for (int k = 0; k < 7; k++) atomicAdd((unsigned long long *)&g_rs_phase[k], (unsigned long long)ph[k]);
#endif
#undef FK_PH
}

// ---------------------------------------------------------------- v2: rank by bucket walk
// The production sort for n <= FK_NMAX.  Same bucket map, counters and screen as the
// float-key kernel above, with fewer instructions per key where they were spent:
//  * the scatter writes (float key, column id) pairs, so the rank of a key inside its
//    bucket is a walk over the bucket's few pairs in shared memory by the key's own lane
//    (singleton buckets -- most of them -- cost nothing); no run detection, shuffles or
//    window-edge walks by sorted position;
//  * the ranked ids land in shared memory and leave by one TMA bulk store per row
//    (cp.async.bulk.global.shared::cta; the 16-byte aligned body, scalar edges), so the
//    id store costs one STS per key and the next row's TMA load into the buffer waits
//    only for that store's reads (cp.async.bulk.wait_group.read).
// Ties at float precision still go to the doubles (re-read through L2), then the id.
__device__ __forceinline__ void v2_bulk_store(int32_t *g, const void *smem, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g), "r"(rt_smem_u32(smem)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void v2_bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

template <bool ODD, int KPT>
__device__ __forceinline__ void v2_row(const FkRow &R, const float (&fk)[KPT], unsigned char *buf) {
    constexpr int NT = FK_T, W = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = R.n, m = R.m, vi = R.vi, C = R.C;
    uint32_t *f16 = R.f16, *ccnt = R.ccnt;
    uint32_t *cinfo32 = R.ccnt;   // per coarse bin: fine base | fine count << 16
    const uint16_t *o16 = reinterpret_cast<const uint16_t *>(f16);
    FkMisc &ms = *R.ms;
    uint2 *P = reinterpret_cast<uint2 *>(buf);   // scattered (float key bits, column id)
    float hs = R.hc, scale = R.hc;               // t = hs - f * scale
    if (ODD) {   // the row's float range, histogram again
        float fmn = INFINITY, fmx = -INFINITY;
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            const int j = tid + e * NT;
            if (j < n && j != vi) { fmn = fminf(fmn, fk[e]); fmx = fmaxf(fmx, fk[e]); }
        }
        for (int o = 16; o; o >>= 1) {
            fmn = fminf(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
            fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        }
        if (lane == 0) { ms.rmn[warp] = fmn; ms.rmx[warp] = fmx; }
        for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;
        __syncthreads();
        float lo = INFINITY, hi = -INFINITY;
        for (int w = 0; w < W; w++) { lo = fminf(lo, ms.rmn[w]); hi = fmaxf(hi, ms.rmx[w]); }
        const float wd = hi - lo;
        scale = (wd > 0.0f && wd < INFINITY) ? (float)C / wd : 0.0f;
        if (!(hi < INFINITY && hi > -INFINITY)) hi = 0.0f;
        hs = hi * scale;
#pragma unroll
        for (int e = 0; e < KPT; e += 4) {
            const int j = tid + e * NT;
            if (j < n && j != vi) atomicAdd(&ccnt[fk_coarse<true>(fk[e], hs, scale, C)], 1u);
        }
        __syncthreads();
    }
    // ---- 2: fine buckets per coarse bin (one thread per bin) -> per-bin (A, B)
    {
        const float fsc = (float)m * R.fs / (float)(R.nsamp > 0 ? R.nsamp : 1) * 0.9999f;
        const uint32_t f = tid <= C ? 1u + (uint32_t)((float)ccnt[tid] * fsc) : 0u;
        uint32_t incl = f;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) ms.wsum[warp] = incl;
        __syncthreads();
        if (tid <= C) {
            uint32_t off = 0;
            for (int w = 0; w < warp; w++) off += ms.wsum[w];
            const uint32_t base = off + incl - f;
            cinfo32[tid] = base | (f << 16);   // fb = rn((d + 1/2) f + base): the same value as v1's map
            if (tid == C) ms.nb = (int)(base + f) + 1;
        }
    }
    __syncthreads();
    // ---- 3: fine bucket + arrival rank (one packed-u16 shared atomic per key); the loads,
    // then the atomics, are issued back to back (independent across keys)
    uint32_t pk[KPT];
    const int nan_fb = ms.nb - 1;
    constexpr int G3 = 6;   // keys per batch
#pragma unroll
    for (int e0 = 0; e0 < KPT; e0 += G3) {
        uint32_t ab[G3];
        float dd[G3];
#pragma unroll
        for (int g = 0; g < G3; g++) {
            const int e = e0 + g;
            if (e >= KPT) break;
            float t = fmaf(fk[e], -scale, hs);
            if (ODD) t = fminf(fmaxf(t, 0.0f), (float)C);
            const float y = t + FK_MAGIC;
            const int c = __float_as_int(y) & 0x3fffff;
            dd[g] = t - (y - FK_MAGIC);   // exact
            const int j = tid + e * NT;
            ab[g] = (j < n) ? cinfo32[c] : 0u;
        }
#pragma unroll
        for (int g = 0; g < G3; g++) {
            const int e = e0 + g;
            if (e >= KPT) break;
            const int j = tid + e * NT;
            pk[e] = 0xffffffffu;
            if (j < n && j != vi) {
                int fb = fk_rni(fmaf(dd[g] + 0.5f, (float)(ab[g] >> 16), (float)(ab[g] & 0xffffu)));
                if (ODD && fk[e] != fk[e]) fb = nan_fb;
                const uint32_t sh = (fb & 1) << 4;
                const uint32_t old = atomicAdd(&f16[fb >> 1], 1u << sh);
                pk[e] = __byte_perm((uint32_t)fb, old >> sh, 0x1054);   // (fb << 16) | arrival
            }
        }
    }
    __syncthreads();
    for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;   // next row's histogram (cinfo is dead)
    // ---- 4: exclusive scan of the packed counters.  Warp w owns a contiguous range of words and
    // walks it 128 words (one 16-byte load per lane, conflict-free) at a time.
    {
        const int nw = (ms.nb + 2) >> 1;
        const int per = ((nw + W - 1) / W + 127) & ~127;   // words per warp
        const int w0 = warp * per;
        uint32_t s = 0;   // the warp's total (lane 31 after the loop)
        for (int q = 0; q < per; q += 128) {
            const int w = w0 + q + 4 * lane;
            uint32_t t = 0;
            if (w < nw) {
                const uint4 x = *reinterpret_cast<const uint4 *>(f16 + w);
                t = ((x.x + (x.x << 16)) >> 16) + ((x.y + (x.y << 16)) >> 16) + ((x.z + (x.z << 16)) >> 16) +
                    ((x.w + (x.w << 16)) >> 16);
            }
            s += __reduce_add_sync(0xffffffffu, t);
        }
        if (lane == 0) ms.wsum[warp] = s;
        __syncthreads();
        uint32_t run;
        {
            const uint32_t wv = ms.wsum[lane];
            uint32_t wi = wv;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            run = __shfl_sync(0xffffffffu, wi - wv, warp);   // words before this warp's range
        }
        for (int q = 0; q < per; q += 128) {
            const int w = w0 + q + 4 * lane;
            uint4 x = make_uint4(0u, 0u, 0u, 0u);
            if (w < nw) x = *reinterpret_cast<const uint4 *>(f16 + w);
            const uint32_t c0 = (x.x + (x.x << 16)) >> 16, c1 = (x.y + (x.y << 16)) >> 16;
            const uint32_t c2 = (x.z + (x.z << 16)) >> 16, c3 = (x.w + (x.w << 16)) >> 16;
            const uint32_t t = c0 + c1 + c2 + c3;
            uint32_t incl = t;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t r = run + incl - t;
            if (w < nw) {
                x.x = r * 0x10001u + (x.x << 16); r += c0;
                x.y = r * 0x10001u + (x.y << 16); r += c1;
                x.z = r * 0x10001u + (x.z << 16); r += c2;
                x.w = r * 0x10001u + (x.w << 16);
                *reinterpret_cast<uint4 *>(f16 + w) = x;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    __syncthreads();
    // ---- 5: scatter (key, id) to bucket offset + arrival (offset loads batched, then the stores);
    // pk becomes (bucket start s0, position of the key's pair)
    {
        uint32_t s0[KPT];
#pragma unroll
        for (int e = 0; e < KPT; e++) s0[e] = pk[e] != 0xffffffffu ? o16[pk[e] >> 16] : 0u;
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            if (pk[e] != 0xffffffffu) {
                const uint32_t p = s0[e] + (pk[e] & 0xffffu);
                P[p] = make_uint2(__float_as_uint(fk[e]), (uint32_t)(tid + e * NT));
                pk[e] = (pk[e] & 0xffff0000u) | s0[e];   // (bucket, bucket start)
            }
        }
    }
    __syncthreads();
    // ---- 6: rank inside the bucket: a fixed 4-slot compare (predicated loads, no loop) covers
    // buckets of <= 4 keys -- nearly all of them; larger buckets and float ties walk the bucket
    const double *row = R.row;
    constexpr int G = 4;   // keys per batch (bounds the registers of the batched loads)
#pragma unroll
    for (int e0 = 0; e0 < KPT; e0 += G) {
        int s0[G], cc[G];
        float kq[G][4];
#pragma unroll
        for (int g = 0; g < G; g++) {
            const int e = e0 + g;
            s0[g] = 0;
            cc[g] = 0;
            if (e < KPT && pk[e] != 0xffffffffu) {
                const int fb = (int)(pk[e] >> 16);
                s0[g] = (int)(pk[e] & 0xffffu);
                cc[g] = (int)o16[fb + 1] - s0[g];
            }
        }
#pragma unroll
        for (int g = 0; g < G; g++) {   // a singleton bucket holds only the key itself: no loads
#pragma unroll
            for (int i = 0; i < 4; i++)
                kq[g][i] = (cc[g] > 1 && i < cc[g]) ? __uint_as_float(P[s0[g] + i].x) : (ODD ? 0.0f : -INFINITY);
        }
#pragma unroll
        for (int g = 0; g < G; g++) {
            const int e = e0 + g;
            if (e >= KPT || pk[e] == 0xffffffffu) continue;
            const int j = tid + e * NT;
            const float fj = fk[e];
            const int c = cc[g];
            int rank = 0, tie = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const float fo = kq[g][i];
                const bool in = c > 1 && i < c;
                if (!ODD) {   // absent slots hold -inf: never above or equal to a key in [-1, 1]
                    rank += fo > fj;
                    tie += fo == fj;
                } else {
                    const bool no = fo != fo, nj = fj != fj;
                    rank += in & ((fo > fj) | (nj & !no));
                    tie += in & ((fo == fj) | (nj & no));
                }
            }
            if (c > 4) {
                for (int q = s0[g] + 4; q < s0[g] + c; q++) {
                    const float fo = __uint_as_float(P[q].x);
                    if (!ODD) {
                        rank += fo > fj;
                        tie += fo == fj;
                    } else {
                        const bool no = fo != fo, nj = fj != fj;
                        rank += (fo > fj) | (nj & !no);
                        tie += (fo == fj) | (nj & no);
                    }
                }
            }
            if (tie > 1) {   // float ties (itself included): the doubles decide, then the id
                // (segments: slots map to column ids through R.sid)
                const int idj = R.sid ? R.sid[j] : j;
                const double xj = __ldg(row + idj);
                rank = 0;
                for (int q = s0[g]; q < s0[g] + c; q++) {
                    const uint2 o = P[q];
                    if ((int)o.y == j) continue;
                    const float fo = __uint_as_float(o.x);
                    const bool feq = ODD ? ((fo == fj) | ((fo != fo) & (fj != fj))) : (fo == fj);
                    if (!feq) {
                        if (!ODD) rank += fo > fj;
                        else rank += (fo > fj) | ((fj != fj) & (fo == fo));
                    } else {
                        const int ido = R.sid ? R.sid[o.y] : (int)o.y;
                        rank += rs_before(__ldg(row + ido), ido, xj, idj);
                    }
                }
            }
            pk[e] = (uint32_t)(s0[g] + rank);
        }
    }
    __syncthreads();   // every walk is done: the buffer takes the ranked ids
    int32_t *out32 = reinterpret_cast<int32_t *>(buf) + (int)(((uintptr_t)R.out >> 2) & 3);
#pragma unroll
    for (int e = 0; e < KPT; e++)
        if (pk[e] != 0xffffffffu) out32[pk[e]] = R.sid ? R.sid[tid + e * NT] : tid + e * NT;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic writes -> bulk-store reads
    __syncthreads();
}

template <int KPT>
__global__ void __launch_bounds__(FK_T, 1)
row_sort_v2_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                   double *__restrict__ screen, FkPlan pl) {
    extern __shared__ __align__(16) unsigned char fk_smem[];
    constexpr int NT = FK_T, W = NT / 32;
    const int n = (int)n64;
    const int m = n - 1;
    uint32_t *ccnt = reinterpret_cast<uint32_t *>(fk_smem + pl.off_cinfo);   // histogram, then (A, B)
    FkMisc &ms = *reinterpret_cast<FkMisc *>(fk_smem + pl.off_misc);
    uint64_t *bar = reinterpret_cast<uint64_t *>(fk_smem + pl.off_bar);
    uint32_t *f16 = reinterpret_cast<uint32_t *>(fk_smem + pl.off_f16);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = pl.C;
    const int nw16 = pl.NBcap / 2 + 2;
    const size_t bstride = (size_t)pl.stride * sizeof(double);

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(rt_smem_u32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;\n" ::"r"(rt_smem_u32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int c = tid; c <= C; c += NT) ccnt[c] = 0u;
    __syncthreads();
    int64_t v = blockIdx.x;
    if (tid == 0 && v < n) rt_bulk_row(reinterpret_cast<double *>(fk_smem), S + v * n64, n, &bar[0]);
    int nsamp_all = 0;   // sampled keys: e % 4 == 0
#pragma unroll
    for (int e = 0; e < KPT; e += 4) {
        const int r = n - e * NT;
        nsamp_all += r < 0 ? 0 : (r < NT ? r : NT);
    }
    FkRow R;
    R.f16 = f16;
    R.cinfo = reinterpret_cast<float2 *>(ccnt);
    R.ccnt = ccnt;
    R.ms = &ms;
    R.n = n;
    R.m = m;
    R.C = C;
    R.fs = pl.fs;
    R.hc = pl.hc;
    R.sid = nullptr;
    R.fkey = nullptr;
    R.sidx = nullptr;
    for (int it = 0; v < n; v += gridDim.x, it++) {
        const int b = pl.nbuf == 2 ? (it & 1) : 0;
        const unsigned parity = pl.nbuf == 2 ? (unsigned)((it >> 1) & 1) : (unsigned)(it & 1);
        unsigned char *buf = fk_smem + (size_t)b * bstride;
        const double *row = S + v * n64;
        const double *vals = reinterpret_cast<const double *>(buf) + (((uintptr_t)row >> 3) & 1);
        const int vi = (int)v;
        for (int i = 4 * tid; i < nw16 + 8; i += 4 * NT)   // + the 16-byte scan's overhang
            *reinterpret_cast<uint4 *>(f16 + i) = make_uint4(0u, 0u, 0u, 0u);
        rt_wait(&bar[b], parity);
        // ---- 1: doubles -> float keys (registers), screen sums, sampled coarse histogram
        float fk[KPT];
        double sm = 0.0, sa = 0.0;
        bool odd = false;
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            const int j = tid + e * NT;
            fk[e] = 0.0f;
            if (j < n) {
                const double x = vals[j];
                sm += x;
                sa += fabs(x);
                const float f = __double2float_rn(x);
                fk[e] = f;
                if (j != vi) {
                    odd |= !(fabsf(f) <= 1.0f);   // NaN or outside [-1, 1] at float precision
                    if ((e & 3) == 0) atomicAdd(&ccnt[fk_coarse<true>(f, pl.hc, pl.hc, C)], 1u);
                } else {
                    ms.diag = x;
                }
            }
        }
        if (screen) {
            for (int o = 16; o; o >>= 1) {
                sm += __shfl_xor_sync(0xffffffffu, sm, o);
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
            }
            if (lane == 0) { ms.rsum[warp] = sm; ms.rabs[warp] = sa; }
        }
        const bool row_odd = __syncthreads_or(odd);   // every double of the row is consumed
        if (tid == 0) {
            const int64_t vn = v + gridDim.x;
            if (pl.nbuf == 2 && vn < n) {
                v2_bulk_wait_read();   // the previous row's id store out of the other buffer
                rt_bulk_row(reinterpret_cast<double *>(fk_smem + (size_t)(b ^ 1) * bstride), S + vn * n64, n,
                            &bar[b ^ 1]);
            }
        }
        if (screen && warp == W - 1) {
            double s1 = ms.rsum[lane], s2 = ms.rabs[lane];
            for (int o = 16; o; o >>= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            }
            if (lane == 0) {
                screen[vi] = __dsub_rn(s1, ms.diag);
                screen[n + vi] = rs_screen_radius_t(n, NT, s2);
            }
        }
        R.row = row;
        R.out = order + v * (int64_t)m;
        R.vi = vi;
        R.nsamp = nsamp_all - (((vi / NT) & 3) == 0 ? 1 : 0);
        if (row_odd) v2_row<true, KPT>(R, fk, buf);
        else v2_row<false, KPT>(R, fk, buf);
        // ---- 7: the ranked ids leave by a bulk store (16-byte aligned body) + scalar edges
        {
            int32_t *g = R.out;
            const int a = (int)(((uintptr_t)g >> 2) & 3);
            const int32_t *out32 = reinterpret_cast<const int32_t *>(buf) + a;
            const int h = (4 - a) & 3;
            const int p0 = h < m ? h : m;
            const int p1 = p0 + ((m - p0) & ~3);
            if (tid == 0 && p1 > p0) v2_bulk_store(g + p0, out32 + p0, (unsigned)((p1 - p0) * 4));
            if (warp == 1) {
                if (lane < p0) g[lane] = out32[lane];
                else if (lane >= 4 && lane - 4 < m - p1) g[p1 + lane - 4] = out32[p1 + lane - 4];
            }
        }
        if (pl.nbuf == 1) {
            __syncthreads();   // warp 1's edge reads of the buffer are done before it is refilled
            if (tid == 0) {
                const int64_t vn = v + gridDim.x;
                if (vn < n) {
                    v2_bulk_wait_read();
                    rt_bulk_row(reinterpret_cast<double *>(fk_smem), S + vn * n64, n, &bar[0]);
                }
            }
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------- long rows (n > FK_NMAX)
// Two passes per batch of rows, everything heavy in shared memory:
//  1. row_part_kernel (one CTA per row): float keys, screen sums, a histogram over
//     SP_C fixed bins of [-1, 1]; bins are grouped into segments of consecutive
//     bins (bin start position / T, T = SEG_MAX - largest bin + 1, so a segment
//     holds <= SEG_MAX keys) and every key is scattered as (float key, id) to its
//     bin's slice of a per-row scratch row -- a segment's keys are exactly the
//     output positions [P_s, P_s + cnt_s) of the row, in arbitrary order;
//  2. row_seg_kernel (persistent CTAs pulling (row, segment) items): the
//     float-key bucket sort of fk_row on the segment (range map from the
//     segment's own float min/max), ids through a slot -> id table.
// Rows with NaN / values outside [-1, 1] or one bin above SEG_MAX / 2 are listed
// and sorted by row_sort_global_kernel afterwards.
constexpr int SP_C = 4096;
constexpr int SEG_MAX = 12288;
constexpr int SEG_KPT = SEG_MAX / FK_T;
constexpr int SP_MAXSEG = 64;
constexpr int SP_U = 8;     // loads in flight per thread
constexpr int SP_PT = 512;  // partition CTA size (2 per SM)   // segments per row: n <= ~390k

struct SegItem {
    int32_t v, pos0, cnt, pad;
    int64_t soff;   // scratch offset (float2 entries)
};

template <int PT>
__global__ void __launch_bounds__(PT, 1024 / PT)
row_part_kernel(const double *__restrict__ S, int64_t n64, int64_t v0, int64_t v1, double *__restrict__ screen,
                float2 *__restrict__ scratch, SegItem *__restrict__ items, int *__restrict__ nitems,
                int32_t *__restrict__ slow, int *__restrict__ nslow) {
    __shared__ uint32_t hist[SP_C + 1];
    __shared__ uint32_t base[SP_C + 1];
    __shared__ double red[2][32];
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t maxbin;
    __shared__ double diag;
    __shared__ double seg_lo[SP_MAXSEG], seg_inv[SP_MAXSEG];
    __shared__ uint8_t segof[SP_C + 1];
    __shared__ uint32_t segcur[SP_MAXSEG], gcur[SP_MAXSEG], ccnt_s[SP_MAXSEG], coff[SP_MAXSEG];
    extern __shared__ __align__(16) unsigned char sp_dyn[];   // SP_U * PT * 9 bytes
    float2 *stage = reinterpret_cast<float2 *>(sp_dyn);
    uint8_t *stg_seg = sp_dyn + SP_U * PT * sizeof(float2);
    const int n = (int)n64, m = n - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int W = PT / 32;
    constexpr float HC = 0.5f * SP_C;
    for (int64_t v = v0 + blockIdx.x; v < v1; v += gridDim.x) {
        const double *row = S + v * n64;
        const int vi = (int)v;
        for (int c = tid; c <= SP_C; c += PT) hist[c] = 0u;
        if (tid == 0) maxbin = 0u;
        __syncthreads();
        double sm = 0.0, sa = 0.0;
        bool odd = false;
        for (int j0 = tid; j0 < n; j0 += SP_U * PT) {
            double x[SP_U];
#pragma unroll
            for (int u = 0; u < SP_U; u++) x[u] = j0 + u * PT < n ? __ldg(row + j0 + u * PT) : 0.0;
#pragma unroll
            for (int u = 0; u < SP_U; u++) {
                const int j = j0 + u * PT;
                if (j >= n) continue;
                sm += x[u];
                sa += fabs(x[u]);
                if (j == vi) { diag = x[u]; continue; }
                const float f = __double2float_rn(x[u]);
                odd |= !(fabsf(f) <= 1.0f);
                atomicAdd(&hist[fk_coarse<true>(f, HC, HC, SP_C)], 1u);
            }
        }
        for (int o = 16; o; o >>= 1) {
            sm += __shfl_xor_sync(0xffffffffu, sm, o);
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        if (lane == 0) { red[0][warp] = sm; red[1][warp] = sa; }
        const bool row_odd = __syncthreads_or(odd);
        if (warp == W - 1) {
            double s1 = lane < W ? red[0][lane] : 0.0, s2 = lane < W ? red[1][lane] : 0.0;
            for (int o = 16; o; o >>= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            }
            if (lane == 0 && screen) {
                screen[vi] = __dsub_rn(s1, diag);
                screen[n + vi] = rs_screen_radius_t(n, PT, s2);
            }
        }
        // exclusive scan of the bins (4 per thread) and the largest bin
        constexpr int BPT = SP_C / PT;   // bins per thread (+ bin SP_C on the last thread)
        uint32_t h[BPT + 1], s = 0, hm = 0;
#pragma unroll
        for (int q = 0; q < BPT; q++) {
            const int c = tid * BPT + q;
            h[q] = hist[c];
            s += h[q];
            hm = max(hm, h[q]);
        }
        h[BPT] = (tid == PT - 1) ? hist[SP_C] : 0u;
        s += h[BPT];
        hm = max(hm, h[BPT]);
        uint32_t incl = s;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        hm = __reduce_max_sync(0xffffffffu, hm);
        if (lane == 31) wsum[warp] = incl;
        if (lane == 0) atomicMax(&maxbin, hm);
        __syncthreads();
        uint32_t wex = 0;
        for (int w = 0; w < warp; w++) wex += wsum[w];   // W <= 32 warps
        uint32_t run = wex + incl - s;
#pragma unroll
        for (int q = 0; q < BPT; q++) { base[tid * BPT + q] = run; hist[tid * BPT + q] = run; run += h[q]; }
        if (tid == PT - 1) { base[SP_C] = run; hist[SP_C] = run; }
        __syncthreads();
        const uint32_t mb = maxbin;
        if (row_odd || mb > (uint32_t)(SEG_MAX / 2)) {
            if (tid == 0) slow[atomicAdd(nslow, 1)] = vi;
            __syncthreads();
            continue;
        }
        const uint32_t T = (uint32_t)SEG_MAX - mb + 1u;   // segment s: bins starting in [s T, (s+1) T)
        // segment s = positions [B_s, B_{s+1}), B_s = the first bin start >= s T (bin boundaries);
        // bin c belongs to segment base[c] / T.  Its keys are re-expressed relative to the
        // segment's value window, so float keys keep ~2^-24 of the window's width.
        const int nseg = (int)(((uint32_t)m + T - 1u) / T);
        for (int sg = tid; sg < nseg; sg += PT) {
            auto bound = [&](uint32_t lim) -> int {   // first bin index with start >= lim
                int lo = 0, hi = SP_C + 1;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (base[mid] < lim) lo = mid + 1;
                    else hi = mid;
                }
                return lo;
            };
            const int cA = sg == 0 ? 0 : bound((uint32_t)sg * T);
            const int cB = bound((uint32_t)(sg + 1) * T);   // exclusive
            const uint32_t b0 = cA <= SP_C ? base[cA] : (uint32_t)m;
            const uint32_t b1 = cB <= SP_C ? base[cB] : (uint32_t)m;
            // values of bins [cA, cB): f in [1 - (cB - 1/2)/HC, 1 - (cA - 1/2)/HC], padded
            const double vlo = 1.0 - ((double)cB - 0.5) / (double)HC - 1e-6;
            const double vhi = 1.0 - ((double)cA - 0.5) / (double)HC + 1e-6;
            seg_lo[sg] = vlo;
            seg_inv[sg] = 2.0 / (vhi - vlo);   // key = 2 (x - lo) / (hi - lo) - 1 in (-1, 1)
            if (b1 <= b0) continue;
            SegItem it;
            it.v = vi;
            it.pos0 = (int32_t)b0;
            it.cnt = (int32_t)(b1 - b0);
            it.pad = 0;
            it.soff = (v - v0) * (int64_t)m + b0;
            items[atomicAdd(nitems, 1)] = it;
        }
        __syncthreads();
        for (int c = tid; c <= SP_C; c += PT) segof[c] = (uint8_t)(base[c] / T);
        if (tid < SP_MAXSEG) segcur[tid] = 0u;
        __syncthreads();
        if (tid < nseg) {   // scratch cursor of segment tid = its first position
            int lo = 0, hi = SP_C + 1;
            const uint32_t lim = (uint32_t)tid * T;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (base[mid] < lim) lo = mid + 1;
                else hi = mid;
            }
            segcur[tid] = tid == 0 ? 0u : (lo <= SP_C ? base[lo] : (uint32_t)m);
        }
        // scatter in chunks of SP_U * PT keys: stage by segment in shared memory, then
        // write each segment's run of the chunk contiguously at its scratch cursor
        float2 *srow = scratch + (v - v0) * (int64_t)m;
        for (int j0 = 0; j0 < n; j0 += SP_U * PT) {
            if (tid < SP_MAXSEG) ccnt_s[tid] = 0u;
            __syncthreads();
            double x[SP_U];
#pragma unroll
            for (int u = 0; u < SP_U; u++) {
                const int j = j0 + u * PT + tid;
                x[u] = j < n ? __ldg(row + j) : 0.0;
            }
            int sgs[SP_U];
            uint32_t loc[SP_U];
#pragma unroll
            for (int u = 0; u < SP_U; u++) {
                const int j = j0 + u * PT + tid;
                sgs[u] = -1;
                if (j < n && j != vi) {
                    const int c = fk_coarse<true>(__double2float_rn(x[u]), HC, HC, SP_C);
                    sgs[u] = segof[c];
                    loc[u] = atomicAdd(&ccnt_s[sgs[u]], 1u);
                }
            }
            __syncthreads();
            if (warp == 0) {   // chunk-local segment offsets + global reservation (nseg <= 64)
                uint32_t c0 = ccnt_s[lane], c1 = ccnt_s[lane + 32];
                uint32_t i0 = c0, i1 = c1;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y0 = __shfl_up_sync(0xffffffffu, i0, o);
                    const uint32_t y1 = __shfl_up_sync(0xffffffffu, i1, o);
                    if (lane >= o) { i0 += y0; i1 += y1; }
                }
                const uint32_t t0 = __shfl_sync(0xffffffffu, i0, 31);
                coff[lane] = i0 - c0;
                coff[lane + 32] = t0 + i1 - c1;
                gcur[lane] = segcur[lane];
                gcur[lane + 32] = segcur[lane + 32];
                segcur[lane] += c0;
                segcur[lane + 32] += c1;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < SP_U; u++) {
                if (sgs[u] < 0) continue;
                const int sg = sgs[u];
                const int j = j0 + u * PT + tid;
                const float key = __double2float_rn(__dsub_rn(__dmul_rn(__dsub_rn(x[u], seg_lo[sg]), seg_inv[sg]), 1.0));
                stage[coff[sg] + loc[u]] = make_float2(key, __int_as_float(j));
                stg_seg[coff[sg] + loc[u]] = (uint8_t)sg;
            }
            __syncthreads();
            const int tot = (int)(coff[SP_MAXSEG - 1] + ccnt_s[SP_MAXSEG - 1]);
            for (int q = tid; q < tot; q += PT) {
                const int sg = stg_seg[q];
                srow[gcur[sg] + (uint32_t)q - coff[sg]] = stage[q];
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(FK_T, 1)
row_seg_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
               const float2 *__restrict__ scratch, const SegItem *__restrict__ items, const int *__restrict__ nitems,
               int *__restrict__ next_item, FkPlan pl) {
    extern __shared__ __align__(16) unsigned char fk_smem[];
    constexpr int NT = FK_T, KPT = SEG_KPT;
    uint32_t *ccnt = reinterpret_cast<uint32_t *>(fk_smem + pl.off_cinfo);
    FkMisc &ms = *reinterpret_cast<FkMisc *>(fk_smem + pl.off_misc);
    uint32_t *f16 = reinterpret_cast<uint32_t *>(fk_smem + pl.off_f16);
    int32_t *sid = reinterpret_cast<int32_t *>(fk_smem + pl.off_sid);
    __shared__ int sh_item;
    const int tid = threadIdx.x;
    const int nw16 = pl.NBcap / 2 + 2;
    const int m_row = (int)n64 - 1;
    for (int c = tid; c <= pl.C; c += NT) ccnt[c] = 0u;
    FkRow R;
    R.f16 = f16;
    R.cinfo = reinterpret_cast<float2 *>(ccnt);
    R.ccnt = ccnt;
    R.ms = &ms;
    R.fkey = reinterpret_cast<float *>(fk_smem);
    R.sidx = reinterpret_cast<uint32_t *>(fk_smem + pl.off_sidx);
    R.sid = sid;
    R.vi = -1;
    R.fs = pl.fs;
    const int total = *nitems;
    for (;;) {
        __syncthreads();   // the previous item is finished with shared memory
        if (tid == 0) sh_item = atomicAdd(next_item, 1);
        __syncthreads();
        const int k = sh_item;
        if (k >= total) break;
        const SegItem it = items[k];
        const int cnt = it.cnt;
        int32_t *out = order + (int64_t)it.v * m_row + it.pos0;
        const float2 *src = scratch + it.soff;
        if (cnt <= 1) {
            if (cnt == 1 && tid == 0) out[0] = __float_as_int(src[0].y);
            continue;
        }
        float fk[KPT];
#pragma unroll
        for (int e = 0; e < KPT; e++) {
            const int s = tid + e * NT;
            fk[e] = 0.0f;
            if (s < cnt) {
                const float2 pr = src[s];
                fk[e] = pr.x;
                sid[s] = __float_as_int(pr.y);
            }
        }
        const int Ci = rs_coarse_bins(cnt);
        const float hci = 0.5f * (float)Ci;
        for (int i = tid; i < nw16 + 8; i += NT) f16[i] = 0u;   // + the 16-byte scan's overhang
        int ns = 0;   // sampled slots: e % 4 == 0 (v2_row's histogram)
#pragma unroll
        for (int e = 0; e < KPT; e += 4) {
            const int rr = cnt - e * NT;
            ns += rr < 0 ? 0 : (rr < NT ? rr : NT);
        }
        R.row = S + (int64_t)it.v * n64;
        R.out = out;
        R.n = cnt;
        R.m = cnt;
        R.C = Ci;
        R.hc = hci;
        R.nsamp = ns;
        __syncthreads();   // sid and the cleared counters are visible
        // the segment's own float range (the general path): a fixed map over the segment
        // window degrades badly when the keys crowd into part of it.  v2_row ranks the
        // (key, slot) pairs and leaves the column ids (through sid) in the buffer
        v2_row<true, KPT>(R, fk, fk_smem);
        const int32_t *o32 = reinterpret_cast<const int32_t *>(fk_smem) + (int)(((uintptr_t)out >> 2) & 3);
        for (int i = tid; i < cnt; i += NT) out[i] = o32[i];
    }
}

// ---------------------------------------------------------------- large rows
// n > 16384: the same two-level bucket algorithm; the row is read through L2,
// the per-key (bucket, rank) pairs live in a per-CTA global scratch slice and
// the output row itself is the scatter buffer.  Counters stay in shared memory.
__global__ void __launch_bounds__(RS_T, 1)
row_sort_global_kernel(const double *__restrict__ S, int64_t n64, int32_t *__restrict__ order,
                       double *__restrict__ screen, uint32_t *__restrict__ gpk_all, const int32_t *__restrict__ rows,
                       const int *__restrict__ nrows) {
    const int n = (int)n64;
    const int m = n - 1;
    extern __shared__ __align__(16) unsigned char rs_smem[];
    uint32_t *fcnt = reinterpret_cast<uint32_t *>(rs_smem);
    __shared__ RsMisc ms;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = rs_coarse_bins(m);
    uint32_t *gpk = gpk_all + (size_t)blockIdx.x * 2 * n;   // [n] bucket, [n] rank/position
    const int64_t nv = rows ? (int64_t)*nrows : n64;
    for (int64_t vix = blockIdx.x; vix < nv; vix += gridDim.x) {
        const int64_t v = rows ? (int64_t)rows[vix] : vix;
        const double *row = S + v * n64;
        int32_t *out = order + v * (int64_t)m;
        for (int c = tid; c <= C; c += RS_T) ms.ccnt[c] = 0;
        if (tid == 0) ms.nsamp = 0;
        double mn = INFINITY, mx = -INFINITY, sm = 0.0, sa = 0.0;
        bool nan_seen = false;
        for (int j = tid; j < n; j += RS_T) {
            double x = __ldg(row + j);
            sm += x;
            sa += fabs(x);
            if (j == v) continue;
            if (x < mn) mn = x;
            if (x > mx) mx = x;
            nan_seen |= (x != x);
        }
        const bool row_nan = __syncthreads_or(nan_seen);
        for (int o = 16; o; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            sm += __shfl_xor_sync(0xffffffffu, sm, o);
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        if (lane == 0) { ms.red[warp] = mn; ms.red[32 + warp] = mx; ms.red[64 + warp] = sm; ms.red[96 + warp] = sa; }
        __syncthreads();
        if (screen && warp == 1) {
            double s1 = ms.red[64 + lane], s2 = ms.red[96 + lane];
            for (int o = 16; o; o >>= 1) {
                s1 += __shfl_xor_sync(0xffffffffu, s1, o);
                s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            }
            if (lane == 0) {
                screen[v] = __dsub_rn(s1, __ldg(row + v));
                screen[n + v] = rs_screen_radius(n, s2);
            }
        }
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
    }
}

constexpr size_t RS_SMEM_MAX = 227 * 1024;
constexpr int FK_NMAX = 24576;   // longer rows: row_part_kernel + row_seg_kernel

// numpy's pairwise plan for n (a pure function of n), cached per host thread
const PwTree<PW_MAXNODES> &pw_host_plan(int n) {
    static thread_local PwTree<PW_MAXNODES> tree;
    static thread_local int tree_n = -1;
    static thread_local int height[PW_MAXNODES];
    if (tree_n != n) {
        pw_plan(tree, n, height);
        tree_n = n;
    }
    return tree;
}

}  // namespace

// long rows: rows per partition batch (scratch = batch x (n-1) float2, <= ~512 MB)
static int64_t seg_batch_rows(int64_t n) {
    int64_t b = ((int64_t)512 << 20) / (8 * (n - 1));
    if (b < tg_num_sms()) b = tg_num_sms();
    return b < n ? b : n;
}
static int64_t seg_items_cap(int64_t n) { return seg_batch_rows(n) * (2 * (n - 1) / SEG_MAX + 3); }

TG_API size_t tg_row_sort_workspace_bytes(int64_t n) {
    if (n <= FK_NMAX) return 256;
    const size_t gk = tg_align_up((size_t)tg_num_sms() * 2 * (size_t)n * sizeof(uint32_t), 256);
    return gk + tg_align_up((size_t)seg_batch_rows(n) * (size_t)(n - 1) * sizeof(float2), 256) +
           tg_align_up((size_t)seg_items_cap(n) * sizeof(SegItem), 256) + tg_align_up((size_t)n * 4, 256) + 1024;
}

TG_API int tg_row_sort_f64(const double *S, int64_t n, int32_t *order, double *screen, void *ws, size_t ws_bytes,
                           void *stream) {
    if (n < 2 || !S || !order) return TG_ERR_ARG;
    if ((((uintptr_t)S) & 7) != 0 || (((uintptr_t)order) & 3) != 0) return TG_ERR_ARG;
    if (n > (int64_t)1 << 30) return TG_ERR_ARG;
    cudaStream_t st = tg_stream(stream);
    int grid = tg_num_sms();
    if (grid > n) grid = (int)n;
    if (n <= FK_NMAX) {
        // two row buffers (the next row's TMA overlaps this row) when they leave room
        // for >= 1.5 fine buckets per key, else one
        const char *fse = getenv("TG_SORT_FS");
        const double fcap = fse ? atof(fse) : 3.0;
        FkPlan pl = fk_plan(n, 2, RS_SMEM_MAX, fcap);
        if (pl.smem > RS_SMEM_MAX || pl.fs < 1.5f) pl = fk_plan(n, 1, RS_SMEM_MAX, fcap);
        if (pl.smem > RS_SMEM_MAX) return TG_ERR_ARG;
        const int K = (int)((n + FK_T - 1) / FK_T);
        static const bool v1 = getenv("TG_SORT_V1") != nullptr;   // A/B switch (development)
#define FK_LAUNCH(KK)                                                                                      \
    do {                                                                                                   \
        auto kfn = v1 ? row_sort_fk_kernel<KK> : row_sort_v2_kernel<KK>;                                   \
        TG_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem)); \
        kfn<<<grid, FK_T, pl.smem, st>>>(S, n, order, screen, pl); tg_count_launch(1);                      \
    } while (0)
        if (K <= 2) FK_LAUNCH(2);
        else if (K <= 4) FK_LAUNCH(4);
        else if (K <= 8) FK_LAUNCH(8);
        else if (K <= 10) FK_LAUNCH(10);
        else if (K <= 12) FK_LAUNCH(12);
        else if (K <= 16) FK_LAUNCH(16);
        else FK_LAUNCH(24);
#undef FK_LAUNCH
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    if (ws_bytes < tg_row_sort_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    if (2 * (n - 1) / SEG_MAX + 2 > SP_MAXSEG) return TG_ERR_ARG;
    TgArena ar(ws, ws_bytes);
    uint32_t *gpk = ar.take<uint32_t>((size_t)tg_num_sms() * 2 * (size_t)n);
    int m = (int)n - 1;
    size_t smem = (size_t)(rs_fine_cap(m) + 1) * sizeof(uint32_t);
    if (smem > 160 * 1024) return TG_ERR_ARG;
    TG_CUDA_CHECK(cudaFuncSetAttribute(row_sort_global_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // partition into segments per batch of rows, sort the segments in shared memory,
    // then the listed rows (NaN, out of range, one huge bin) with the global kernel
    const int64_t B = seg_batch_rows(n);
    float2 *scratch = ar.take<float2>((size_t)B * (size_t)m);
    SegItem *items = ar.take<SegItem>((size_t)seg_items_cap(n));
    int32_t *slow = ar.take<int32_t>((size_t)n);
    int *cnt = ar.take<int>(4);   // nitems, next_item, nslow
    if (!scratch || !items || !slow || !cnt) return TG_ERR_WORKSPACE;
    FkPlan sp = fk_plan(SEG_MAX, 1, RS_SMEM_MAX - (size_t)SEG_MAX * 4 - 64, 3.0);
    sp.off_sid = tg_align_up(sp.smem, 16);
    const size_t seg_smem = sp.off_sid + (size_t)SEG_MAX * 4;
    if (sp.smem > RS_SMEM_MAX || seg_smem > RS_SMEM_MAX) return TG_ERR_ARG;
    TG_CUDA_CHECK(cudaFuncSetAttribute(row_seg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)seg_smem));
    const size_t part_smem = (size_t)SP_U * SP_PT * 9;
    TG_CUDA_CHECK(cudaFuncSetAttribute(row_part_kernel<SP_PT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)part_smem));
    TG_CUDA_CHECK(cudaMemsetAsync(cnt + 2, 0, sizeof(int), st));
    for (int64_t v0 = 0; v0 < n; v0 += B) {
        const int64_t v1 = v0 + B < n ? v0 + B : n;
        TG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), st));
        row_part_kernel<SP_PT><<<2 * grid, SP_PT, part_smem, st>>>(S, n, v0, v1, screen, scratch, items, cnt, slow, cnt + 2);
        row_seg_kernel<<<grid, FK_T, seg_smem, st>>>(S, n, order, scratch, items, cnt, cnt + 1, sp);
        tg_count_launch(2);
    }
    row_sort_global_kernel<<<grid, RS_T, smem, st>>>(S, n, order, screen, gpk, slow, cnt + 2); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_row_sums_workspace_bytes(int64_t) { return 256; }

TG_API int tg_row_sums_f64(const double *S, int64_t n, double *rowsum, void *, size_t, void *stream) {
    if (n < 1 || !S || !rowsum) return TG_ERR_ARG;
    if (n > 128 * (PW_MAXNODES / 2)) return TG_ERR_ARG;
    int grid = tg_num_sms() * 4;
    if (grid > n) grid = (int)n;
    row_sums_kernel<<<grid, 256, 0, tg_stream(stream)>>>(S, n, rowsum, nullptr, nullptr, pw_host_plan((int)n));
    tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_initial_clique(const double *rowsum, int64_t n, int32_t *clique, void *stream) {
    if (n < 4 || !rowsum || !clique) return TG_ERR_ARG;
    clique_kernel<<<1, 1024, 0, tg_stream(stream)>>>(rowsum, n, clique, nullptr, nullptr); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_initial_clique_screened_workspace_bytes(int64_t n) {
    return tg_align_up((size_t)n * sizeof(double), 256) + tg_align_up((size_t)n * sizeof(int32_t), 256) + 256;
}

TG_API int tg_initial_clique_screened(const double *S, int64_t n, const double *screen, int32_t *clique, void *ws,
                                      size_t ws_bytes, void *stream) {
    if (n < 4 || !S || !screen || !clique) return TG_ERR_ARG;
    if (n > 128 * (PW_MAXNODES / 2)) return TG_ERR_ARG;
    if (!ws || ws_bytes < tg_initial_clique_screened_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    TgArena ar(ws, ws_bytes);
    double *sums = ar.take<double>((size_t)n);
    int32_t *cand = ar.take<int32_t>((size_t)n);
    int32_t *ncand = ar.take<int32_t>(1);
    clique_screen_kernel<<<1, 1024, 0, st>>>(screen, n, cand, ncand);
    int grid = tg_num_sms();
    row_sums_kernel<<<grid, 256, 0, st>>>(S, n, sums, cand, ncand, pw_host_plan((int)n));
    clique_kernel<<<1, 1024, 0, st>>>(sums, n, clique, cand, ncand);
    tg_count_launch(3);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

#if RS_DEBUG_PHASES
// debug build only: per-phase cycle sums (thread 0 of every CTA) since the last call
TG_API void tg_row_sort_debug_phases(long long *out) {
    cudaMemcpyFromSymbol(out, g_rs_phase, 8 * sizeof(long long));
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_rs_phase, z, sizeof(z));
}
#endif
