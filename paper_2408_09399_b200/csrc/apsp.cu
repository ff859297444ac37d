// apsp.cu -- shortest paths over the TMFG: CSR build, many-source SSSP, hubs,
// radius-truncated searches.
//
// Replaces apsp.py:52-77 to_weighted, 164-171 apsp_exact, 178-230 apsp_hub and
// the numba kernels _kernels.py:40-181 (binary-heap Dijkstra, truncated
// Dijkstra with count-then-fill).
//
// Exactness: Dijkstra in fp64 returns, for every target, the minimum over paths
// of the left-fold fl(fl(d + w1) + w2)...; fl(d + w) is monotone in d and never
// below d (w >= 0), so ANY label-correcting iteration that relaxes with the
// same additions reaches the same fixed point bit for bit.  The kernels below
// are frontier label-correcting searches (one CTA per source), so the distance
// rows and near tables are identical to the reference's.
#include "common.cuh"

namespace {

// ---------------------------------------------------------------- to_weighted
__global__ void deg_kernel(const int32_t *__restrict__ edges, int64_t m, int32_t *__restrict__ deg) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        atomicAdd(&deg[edges[2 * i]], 1);
        atomicAdd(&deg[edges[2 * i + 1]], 1);
    }
}

// single-CTA exclusive scan of int32 counts into int64 offsets (n+1 entries)
__global__ void scan_i32_to_i64_kernel(const int32_t *__restrict__ in, int64_t n, int64_t *__restrict__ out) {
    __shared__ long long wsum[32];
    __shared__ long long carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        int64_t i = base + tid;
        long long x = i < n ? in[i] : 0;
        long long incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            long long w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            long long wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                long long y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            wsum[lane] = wi - w;
        }
        __syncthreads();
        if (i < n) out[i] = carry + wsum[warp] + incl - x;
        __syncthreads();
        if (tid == blockDim.x - 1) carry += wsum[warp] + incl;
        __syncthreads();
    }
    if (tid == 0) out[n] = carry;
}

__global__ void scatter_edges_kernel(const int32_t *__restrict__ edges, int64_t m, const int64_t *__restrict__ indptr,
                                     int32_t *__restrict__ cursor, int32_t *__restrict__ slot_edge) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {
        int a = edges[2 * i], b = edges[2 * i + 1];
        slot_edge[indptr[a] + atomicAdd(&cursor[a], 1)] = (int32_t)i;
        slot_edge[indptr[b] + atomicAdd(&cursor[b], 1)] = (int32_t)i;
    }
}

// one CTA per vertex: order its incident edges by edge id (the reference fills
// the CSR in edge order, apsp.py:66-72), write neighbour + length, and fold
// strength exactly like np.add.at(e0) then np.add.at(e1) (apsp.py:73-75).
__global__ void fill_csr_kernel(const double *__restrict__ S, int64_t n, const int32_t *__restrict__ edges,
                                const int64_t *__restrict__ indptr, const int32_t *__restrict__ slot_edge,
                                int32_t *__restrict__ nbr, double *__restrict__ len, double *__restrict__ strength,
                                int smem_cap) {
    extern __shared__ int32_t fc_sh[];
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const int64_t beg = indptr[v];
        const int d = (int)(indptr[v + 1] - beg);
        const bool in_smem = d <= smem_cap;
        const int32_t *ids = in_smem ? fc_sh : slot_edge + beg;
        if (in_smem)
            for (int k = threadIdx.x; k < d; k += blockDim.x) fc_sh[k] = slot_edge[beg + k];
        __syncthreads();
        for (int k = threadIdx.x; k < d; k += blockDim.x) {
            const int e = ids[k];
            int r = 0;
            for (int q = 0; q < d; q++) r += ids[q] < e;
            const int a = edges[2 * e], b = edges[2 * e + 1];
            const double s = S[(int64_t)a * n + b];
            double t = 2.0 * (1.0 - s);
            t = t > 0.0 ? t : 0.0;  // np.maximum(., 0.0)
            nbr[beg + r] = (a == v) ? b : a;
            len[beg + r] = __dsqrt_rn(t);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double acc = 0.0;
            for (int k = 0; k < d; k++) {  // edges where v is e0 (the smaller id), in edge order
                int u = nbr[beg + k];
                if (u > v) acc = __dadd_rn(acc, S[(int64_t)v * n + u]);
            }
            for (int k = 0; k < d; k++) {  // then the edges where v is e1
                int u = nbr[beg + k];
                if (u < v) acc = __dadd_rn(acc, S[(int64_t)u * n + v]);
            }
            strength[v] = acc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- SSSP
// Frontier label-correcting search from one source per CTA iteration.
//   dist: shared memory (n <= SSSP_SMEM_N) or the output row in global memory;
//   queue: vertices improved in the previous round (deduplicated by a round
//   stamp); relaxation: atomicMin on the raw bits (all distances >= +0.0).
// Warps take 32 queued vertices at a time and flatten their edges so lanes stay
// busy on high-degree hubs.
constexpr int SS_T = 512;
constexpr int SSSP_SMEM_N = 10240;

template <bool SMEM>
struct SsState {
    double *dist;
    uint32_t *stamp;
    int32_t *q0, *q1;
};

__device__ __forceinline__ void relax_edges(int32_t u, double du, const int64_t *__restrict__ indptr,
                                            const int32_t *__restrict__ nbr, const double *__restrict__ len,
                                            double *dist, uint32_t *stamp, uint32_t round, int32_t *qnext,
                                            int *qn, double radius, int *eb_beg, int *eb_off, double *eb_du) {
    // warp-cooperative: every lane brings one vertex (u < 0 = none)
    const int lane = threadIdx.x & 31;
    int beg = 0, d = 0;
    if (u >= 0) {
        beg = (int)indptr[u];
        d = (int)(indptr[u + 1] - beg);
    }
    int incl = d;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    eb_beg[lane] = beg;
    eb_off[lane] = incl - d;
    eb_du[lane] = du;
    __syncwarp();
    for (int k = lane; k < total; k += 32) {
        int lo = 0, hi = 31;
        while (lo < hi) {  // last owner with off <= k
            int mid = (lo + hi + 1) >> 1;
            if (eb_off[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        int e = eb_beg[lo] + (k - eb_off[lo]);
        int v = nbr[e];
        double nd = __dadd_rn(eb_du[lo], len[e]);
        if (!(nd <= radius)) continue;
        unsigned long long nb = tg_dbits(nd);
        unsigned long long old = atomicMin((unsigned long long *)&dist[v], nb);
        if (nb < old) {
            if (atomicExch(&stamp[v], round) != round) qnext[atomicAdd(qn, 1)] = v;
        }
    }
    __syncwarp();
}

template <bool SMEM>
__global__ void __launch_bounds__(SS_T)
sssp_rows_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ nbr, const double *__restrict__ len,
                 int64_t n64, const int64_t *__restrict__ sources, int64_t n_src, double *__restrict__ out,
                 uint32_t *__restrict__ gstamp_all, int32_t *__restrict__ gq_all) {
    extern __shared__ __align__(16) unsigned char ss_sh[];
    const int n = (int)n64;
    __shared__ int qlen[2];
    __shared__ int eb_beg[SS_T / 32][32], eb_off[SS_T / 32][32];
    __shared__ double eb_du[SS_T / 32][32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double *sdist = reinterpret_cast<double *>(ss_sh);
    uint32_t *stamp;
    int32_t *qa, *qb;
    if (SMEM) {
        stamp = reinterpret_cast<uint32_t *>(sdist + n);
        qa = reinterpret_cast<int32_t *>(stamp + n);
        qb = qa + n;
    } else {
        stamp = gstamp_all + (size_t)blockIdx.x * n;
        qa = gq_all + (size_t)blockIdx.x * 2 * n;
        qb = qa + n;
        for (int i = tid; i < n; i += SS_T) stamp[i] = 0u;
    }
    uint32_t round = 0;
    for (int64_t s = blockIdx.x; s < n_src; s += gridDim.x) {
        const int src = (int)sources[s];
        double *dist = SMEM ? sdist : out + s * n64;
        for (int i = tid; i < n; i += SS_T) {
            dist[i] = INFINITY;
            if (SMEM) stamp[i] = 0u;
        }
        if (SMEM) round = 0;
        __syncthreads();
        if (tid == 0) {
            dist[src] = 0.0;
            qa[0] = src;
            qlen[0] = 1;
            qlen[1] = 0;
        }
        __syncthreads();
        int cur = 0;
        while (qlen[cur] > 0) {
            round++;
            int32_t *q = cur ? qb : qa;
            int32_t *qn = cur ? qa : qb;
            const int len_q = qlen[cur];
            for (int base = warp * 32; base < len_q; base += SS_T) {
                int idx = base + lane;
                int u = idx < len_q ? q[idx] : -1;
                double du = u >= 0 ? dist[u] : 0.0;
                relax_edges(u, du, indptr, nbr, len, dist, stamp, round, qn, &qlen[cur ^ 1], INFINITY, eb_beg[warp],
                            eb_off[warp], eb_du[warp]);
            }
            __syncthreads();
            if (tid == 0) qlen[cur] = 0;
            cur ^= 1;
            __syncthreads();
        }
        if (SMEM) {
            double *o = out + s * n64;
            for (int i = tid; i < n; i += SS_T) o[i] = dist[i];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- hubs
// top-H of (strength desc, id asc): radix select on the order key, then an
// exact rank sort of the selected set.  One CTA.
__global__ void select_hubs_kernel(const double *__restrict__ strength, int64_t n64, int64_t H,
                                   int64_t *__restrict__ hubs, int32_t *__restrict__ cand) {
    const int n = (int)n64;
    __shared__ int hist[256];
    __shared__ unsigned long long prefix;
    __shared__ int need, ncand;
    const int tid = threadIdx.x;
    if (tid == 0) { prefix = 0ull; need = (int)H; ncand = 0; }
    __syncthreads();
    // find the H-th largest key (64-bit order key, ties resolved by id later)
    for (int pass = 0; pass < 8; pass++) {
        const int shift = 56 - 8 * pass;
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long pf = prefix;
        for (int i = tid; i < n; i += blockDim.x) {
            unsigned long long k = tg_order_key(strength[i]);
            if (pass == 0 || (k >> (64 - 8 * pass)) == (pf >> (64 - 8 * pass))) atomicAdd(&hist[(k >> shift) & 255], 1);
        }
        __syncthreads();
        if (tid == 0) {
            int acc = 0, d = 255;
            for (; d > 0; d--) {
                if (acc + hist[d] >= need) break;
                acc += hist[d];
            }
            need -= acc;
            prefix = pf | ((unsigned long long)d << shift);
        }
        __syncthreads();
    }
    const unsigned long long thr = prefix;
    const int need_ties = need;  // how many keys == thr to take (lowest ids first)
    for (int i = tid; i < n; i += blockDim.x) {
        unsigned long long k = tg_order_key(strength[i]);
        if (k > thr) cand[atomicAdd(&ncand, 1)] = i;
    }
    __syncthreads();
    // ties at the threshold: the need_ties smallest ids
    __shared__ int nties;
    if (tid == 0) nties = 0;
    __syncthreads();
    int32_t *ties = cand + n;  // second half of the scratch
    for (int i = tid; i < n; i += blockDim.x)
        if (tg_order_key(strength[i]) == thr) ties[atomicAdd(&nties, 1)] = i;
    __syncthreads();
    const int base = ncand, T = nties;
    for (int a = tid; a < T; a += blockDim.x) {
        int ia = ties[a], r = 0;
        for (int b = 0; b < T; b++) r += ties[b] < ia;
        if (r < need_ties) cand[base + r] = ia;
    }
    __syncthreads();
    if (tid == 0) ncand = base + need_ties;
    __syncthreads();
    const int c = ncand;
    for (int a = tid; a < c; a += blockDim.x) {
        int ia = cand[a];
        double sa = strength[ia];
        int r = 0;
        for (int b = 0; b < c; b++) {
            int ib = cand[b];
            double sb = strength[ib];
            r += (sb > sa) || (sb == sa && ib < ia);
        }
        if (r < H) hubs[r] = ia;
    }
}

__global__ void nearest_hub_kernel(const double *__restrict__ hd, const int64_t *__restrict__ hubs, int64_t H,
                                   int64_t n, double c, int64_t *__restrict__ nh, double *__restrict__ nd,
                                   double *__restrict__ radii) {
    int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    int64_t best = 0;
    double bd = hd[u];
    for (int64_t h = 1; h < H; h++) {
        double x = hd[h * n + u];
        if (x < bd) { bd = x; best = h; }  // np.argmin: first minimum in hub-rank order
    }
    nh[u] = hubs[best];
    nd[u] = bd;
    radii[u] = c * bd;
}

// ---------------------------------------------------------------- truncated searches
// Every vertex u gets the ball {v : d(u, v) <= r(u)} with exact distances.
// One CTA per source (dynamic scheduling), tentative distances in a per-CTA
// global slice (only ball entries are ever touched, so it stays in L2), the
// ball recorded as it is first touched, then ordered by id with a bitmap rank
// and appended to a pool; a second kernel compacts the pool into the CSR.
constexpr int TR_T = 256;

__global__ void __launch_bounds__(TR_T)
truncated_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ nbr, const double *__restrict__ len,
                 int64_t n64, const double *__restrict__ radii, double *__restrict__ gdist_all,
                 uint32_t *__restrict__ gstamp_all, int32_t *__restrict__ gq_all, int32_t *__restrict__ gtouch_all,
                 unsigned long long *__restrict__ work, unsigned long long *__restrict__ pool_used, int64_t capacity,
                 int32_t *__restrict__ pool_ids, double *__restrict__ pool_dist, int64_t *__restrict__ src_off,
                 int64_t *__restrict__ counts) {
    extern __shared__ __align__(16) uint32_t tr_bits[];   // n bits
    const int n = (int)n64;
    const int nw = (n + 31) >> 5;
    __shared__ int qlen[2];
    __shared__ int ntouch;
    __shared__ int cur_src;
    __shared__ long long off;
    __shared__ uint32_t wsum[TR_T / 32];
    __shared__ int eb_beg[TR_T / 32][32], eb_off[TR_T / 32][32];
    __shared__ double eb_du[TR_T / 32][32];
    __shared__ uint32_t round_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    double *dist = gdist_all + (size_t)blockIdx.x * n;
    uint32_t *stamp = gstamp_all + (size_t)blockIdx.x * n;
    int32_t *qa = gq_all + (size_t)blockIdx.x * 2 * n;
    int32_t *qb = qa + n;
    int32_t *touch = gtouch_all + (size_t)blockIdx.x * n;
    for (int i = tid; i < n; i += TR_T) { dist[i] = INFINITY; stamp[i] = 0u; }
    for (int i = tid; i < nw; i += TR_T) tr_bits[i] = 0u;
    if (tid == 0) round_sh = 0;
    __syncthreads();
    for (;;) {
        if (tid == 0) cur_src = (int)atomicAdd(work, 1ull);
        __syncthreads();
        const int src = cur_src;
        if (src >= n) break;
        const double radius = radii[src];
        if (tid == 0) {
            dist[src] = 0.0;
            qa[0] = src;
            qlen[0] = 1;
            qlen[1] = 0;
            touch[0] = src;
            ntouch = 1;
        }
        __syncthreads();
        int cur = 0;
        uint32_t round = round_sh;
        while (qlen[cur] > 0) {
            round++;
            int32_t *q = cur ? qb : qa;
            int32_t *qn = cur ? qa : qb;
            const int len_q = qlen[cur];
            for (int base = warp * 32; base < len_q; base += TR_T) {
                int idx = base + lane;
                int u = idx < len_q ? q[idx] : -1;
                double du = u >= 0 ? dist[u] : 0.0;
                // same as relax_edges, plus first-touch recording
                int beg = 0, d = 0;
                if (u >= 0) {
                    beg = (int)indptr[u];
                    d = (int)(indptr[u + 1] - beg);
                }
                int incl = d;
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                eb_beg[warp][lane] = beg;
                eb_off[warp][lane] = incl - d;
                eb_du[warp][lane] = du;
                __syncwarp();
                for (int k = lane; k < total; k += 32) {
                    int lo = 0, hi = 31;
                    while (lo < hi) {
                        int mid = (lo + hi + 1) >> 1;
                        if (eb_off[warp][mid] <= k) lo = mid;
                        else hi = mid - 1;
                    }
                    int e = eb_beg[warp][lo] + (k - eb_off[warp][lo]);
                    int v = nbr[e];
                    double nd = __dadd_rn(eb_du[warp][lo], len[e]);
                    if (!(nd <= radius)) continue;
                    unsigned long long nb = tg_dbits(nd);
                    unsigned long long old = atomicMin((unsigned long long *)&dist[v], nb);
                    if (nb < old) {
                        if (old == 0x7ff0000000000000ull) touch[atomicAdd(&ntouch, 1)] = v;
                        if (atomicExch(&stamp[v], round) != round) qn[atomicAdd(&qlen[cur ^ 1], 1)] = v;
                    }
                }
                __syncwarp();
            }
            __syncthreads();
            if (tid == 0) qlen[cur] = 0;
            cur ^= 1;
            __syncthreads();
        }
        if (tid == 0) round_sh = round;
        // order the ball by id: bitmap + prefix popcount
        const int nt = ntouch;
        for (int i = tid; i < nt; i += TR_T) {
            int v = touch[i];
            atomicOr(&tr_bits[v >> 5], 1u << (v & 31));
        }
        if (tid == 0) {
            unsigned long long o = atomicAdd(pool_used, (unsigned long long)nt);
            off = (long long)o;
            src_off[src] = (int64_t)o;
            counts[src] = nt;
        }
        __syncthreads();
        const bool fits = off + nt <= capacity;
        if (fits) {
            // per-thread chunk of words: local popcount prefix, block scan
            const int per = (nw + TR_T - 1) / TR_T;
            const int w0 = tid * per;
            uint32_t s = 0;
            for (int q = 0; q < per; q++)
                if (w0 + q < nw) s += __popc(tr_bits[w0 + q]);
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) wsum[warp] = incl;
            __syncthreads();
            uint32_t wbase = 0;
            for (int w = 0; w < warp; w++) wbase += wsum[w];
            uint32_t run = wbase + incl - s;
            for (int q = 0; q < per; q++) {
                int wd = w0 + q;
                if (wd >= nw) break;
                uint32_t bits = tr_bits[wd];
                while (bits) {
                    int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    int v = wd * 32 + b;
                    pool_ids[off + run] = v;
                    pool_dist[off + run] = dist[v];
                    run++;
                }
            }
        }
        __syncthreads();
        for (int i = tid; i < nt; i += TR_T) {
            int v = touch[i];
            dist[v] = INFINITY;
            tr_bits[v >> 5] = 0u;
        }
        __syncthreads();
    }
}

__global__ void compact_pool_kernel(int64_t n, const int64_t *__restrict__ src_off, const int64_t *__restrict__ indptr,
                                    const int32_t *__restrict__ pool_ids, const double *__restrict__ pool_dist,
                                    int32_t *__restrict__ ids, double *__restrict__ dd) {
    for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
        int64_t a = src_off[u], b = indptr[u], c = indptr[u + 1] - b;
        for (int64_t k = threadIdx.x; k < c; k += blockDim.x) {
            ids[b + k] = pool_ids[a + k];
            dd[b + k] = pool_dist[a + k];
        }
    }
}

__global__ void scan_i64_kernel(const int64_t *__restrict__ in, int64_t n, int64_t *__restrict__ out) {
    __shared__ long long wsum[32];
    __shared__ long long carry;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        int64_t i = base + tid;
        long long x = i < n ? in[i] : 0;
        long long incl = x;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            long long w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
            long long wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                long long y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            wsum[lane] = wi - w;
        }
        __syncthreads();
        if (i < n) out[i] = carry + wsum[warp] + incl - x;
        __syncthreads();
        if (tid == blockDim.x - 1) carry += wsum[warp] + incl;
        __syncthreads();
    }
    if (tid == 0) out[n] = carry;
}

// transposed near table: rev(v) = {(u, near_u(v)) : v in near(u)}
__global__ void near_count_kernel(const int32_t *__restrict__ ids, int64_t E, int32_t *__restrict__ cnt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < E) atomicAdd(&cnt[ids[i]], 1);
}

__global__ void near_scatter_kernel(int64_t n, const int64_t *__restrict__ ip, const int32_t *__restrict__ ids,
                                    const double *__restrict__ dd, const int64_t *__restrict__ rip,
                                    int32_t *__restrict__ cursor, int32_t *__restrict__ rids, double *__restrict__ rdd) {
    for (int64_t u = blockIdx.x; u < n; u += gridDim.x) {
        for (int64_t k = ip[u] + threadIdx.x; k < ip[u + 1]; k += blockDim.x) {
            int v = ids[k];
            int64_t p = rip[v] + atomicAdd(&cursor[v], 1);
            rids[p] = (int32_t)u;
            rdd[p] = dd[k];
        }
    }
}

}  // namespace

// ============================================================== C ABI
TG_API size_t tg_weighted_workspace_bytes(int64_t n, int64_t m) {
    return tg_align_up((size_t)n * 4, 256) * 2 + tg_align_up((size_t)2 * m * 4, 256) + 1024;
}

TG_API int tg_to_weighted(const double *S, int64_t n, const int32_t *edges, int64_t m, int64_t *indptr,
                          int32_t *nbr, double *len, double *strength, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || m < 0 || !S || !edges || !indptr) return TG_ERR_ARG;
    if (ws_bytes < tg_weighted_workspace_bytes(n, m)) return TG_ERR_WORKSPACE;
    TgArena ar(ws, ws_bytes);
    int32_t *deg = ar.take<int32_t>(n);
    int32_t *cursor = ar.take<int32_t>(n);
    int32_t *slot_edge = ar.take<int32_t>((size_t)2 * m + 1);
    cudaStream_t st = tg_stream(stream);
    TG_CUDA_CHECK(cudaMemsetAsync(deg, 0, n * 4, st));
    TG_CUDA_CHECK(cudaMemsetAsync(cursor, 0, n * 4, st));
    if (m > 0) deg_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(edges, m, deg); tg_count_launch(1);
    scan_i32_to_i64_kernel<<<1, 1024, 0, st>>>(deg, n, indptr); tg_count_launch(1);
    if (m > 0) scatter_edges_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(edges, m, indptr, cursor, slot_edge); tg_count_launch(1);
    int grid = tg_num_sms() * 8;
    if (grid > n) grid = (int)n;
    const int cap = 4096;  // incident-edge ids cached in shared memory; larger degrees read global
    size_t smem = (size_t)cap * sizeof(int32_t);
    fill_csr_kernel<<<grid, 128, smem, st>>>(S, n, edges, indptr, slot_edge, nbr, len, strength, cap); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_sssp_workspace_bytes(int64_t n, int64_t) {
    if (n <= SSSP_SMEM_N) return 256;
    size_t grid = (size_t)tg_num_sms() * 2;
    return grid * (size_t)n * (4 + 8) + 1024;
}

TG_API int tg_sssp_rows(const int64_t *indptr, const int32_t *nbr, const double *len, int64_t n, const int64_t *sources,
                        int64_t n_src, double *dist, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || n_src < 0 || !indptr || !dist) return TG_ERR_ARG;
    if (n_src == 0) return TG_OK;
    cudaStream_t st = tg_stream(stream);
    if (n <= SSSP_SMEM_N) {
        size_t smem = (size_t)n * (8 + 4 + 8);
        TG_CUDA_CHECK(cudaFuncSetAttribute(sssp_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = (int)((220 * 1024) / (smem + 20 * 1024));
        if (per_sm < 1) per_sm = 1;
        if (per_sm > 4) per_sm = 4;
        int64_t grid = (int64_t)tg_num_sms() * per_sm;
        if (grid > n_src) grid = n_src;
        sssp_rows_kernel<true><<<(unsigned)grid, SS_T, smem, st>>>(indptr, nbr, len, n, sources, n_src, dist, nullptr,
                                                                   nullptr); tg_count_launch(1);
    } else {
        if (ws_bytes < tg_sssp_workspace_bytes(n, n_src)) return TG_ERR_WORKSPACE;
        int64_t grid = (int64_t)tg_num_sms() * 2;
        if (grid > n_src) grid = n_src;
        TgArena ar(ws, ws_bytes);
        uint32_t *stamp = ar.take<uint32_t>((size_t)grid * n);
        int32_t *q = ar.take<int32_t>((size_t)grid * 2 * n);
        if (!stamp || !q) return TG_ERR_WORKSPACE;
        sssp_rows_kernel<false><<<(unsigned)grid, SS_T, 0, st>>>(indptr, nbr, len, n, sources, n_src, dist, stamp, q); tg_count_launch(1);
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_select_hubs_workspace_bytes(int64_t n) { return tg_align_up((size_t)2 * n * 4, 256) + 256; }

TG_API int tg_select_hubs(const double *strength, int64_t n, int64_t H, int64_t *hubs, void *ws, size_t ws_bytes,
                          void *stream) {
    if (n < 1 || H < 1 || H > n || !strength || !hubs) return TG_ERR_ARG;
    if (ws_bytes < tg_select_hubs_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    select_hubs_kernel<<<1, 1024, 0, tg_stream(stream)>>>(strength, n, H, hubs, reinterpret_cast<int32_t *>(ws)); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_nearest_hub(const double *hub_dist, const int64_t *hubs, int64_t H, int64_t n, double radius_factor,
                          int64_t *nh, double *nd, double *radii, void *stream) {
    if (n < 1 || H < 1 || !hub_dist || !hubs) return TG_ERR_ARG;
    nearest_hub_kernel<<<(unsigned)((n + 255) / 256), 256, 0, tg_stream(stream)>>>(hub_dist, hubs, H, n, radius_factor,
                                                                                   nh, nd, radii); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

static int tr_grid(int64_t n) {
    int64_t g = (int64_t)tg_num_sms() * 8;
    if (g > n) g = n;
    return (int)g;
}

TG_API size_t tg_truncated_workspace_bytes(int64_t n) {
    size_t g = (size_t)tr_grid(n);
    size_t b = 0;
    b += tg_align_up(g * n * 8, 256);          // dist
    b += tg_align_up(g * n * 4, 256);          // stamp
    b += tg_align_up(g * 2 * n * 4, 256);      // queues
    b += tg_align_up(g * n * 4, 256);          // touched
    b += tg_align_up((size_t)n * 8, 256) * 2;  // src_off, counts
    b += 1024;
    return b;
}

// The pool is the caller's output buffers' size twice over: pool_ids/pool_dist
// are carved from `ws` after the fixed part; the call needs
// tg_truncated_workspace_bytes(n) + capacity * 12 (+alignment) bytes.
TG_API int tg_truncated(const int64_t *indptr, const int32_t *nbr, const double *len, int64_t n, const double *radii,
                        int64_t capacity, int64_t *near_indptr, int32_t *near_ids, double *near_dist, int64_t *total_out,
                        void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || capacity < 0 || !indptr || !radii || !near_indptr || !total_out) return TG_ERR_ARG;
    size_t fixed = tg_truncated_workspace_bytes(n);
    size_t need = fixed + tg_align_up((size_t)capacity * 4, 256) + tg_align_up((size_t)capacity * 8, 256) + 512;
    if (ws_bytes < need) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    const int grid = tr_grid(n);
    TgArena ar(ws, ws_bytes);
    double *gd = ar.take<double>((size_t)grid * n);
    uint32_t *gs = ar.take<uint32_t>((size_t)grid * n);
    int32_t *gq = ar.take<int32_t>((size_t)grid * 2 * n);
    int32_t *gt = ar.take<int32_t>((size_t)grid * n);
    int64_t *src_off = ar.take<int64_t>(n);
    int64_t *counts = ar.take<int64_t>(n);
    unsigned long long *ctr = ar.take<unsigned long long>(2);
    int32_t *pool_ids = ar.take<int32_t>((size_t)capacity + 1);
    double *pool_dist = ar.take<double>((size_t)capacity + 1);
    if (!gd || !gs || !gq || !gt || !src_off || !counts || !ctr || !pool_ids || !pool_dist) return TG_ERR_WORKSPACE;
    TG_CUDA_CHECK(cudaMemsetAsync(ctr, 0, 16, st));
    size_t smem = (size_t)((n + 31) / 32) * 4;
    TG_CUDA_CHECK(cudaFuncSetAttribute(truncated_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    truncated_kernel<<<grid, TR_T, smem, st>>>(indptr, nbr, len, n, radii, gd, gs, gq, gt, ctr, ctr + 1, capacity,
                                               pool_ids, pool_dist, src_off, counts); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    scan_i64_kernel<<<1, 1024, 0, st>>>(counts, n, near_indptr); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    int64_t total = 0;
    TG_CUDA_CHECK(cudaMemcpyAsync(&total, near_indptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    TG_CUDA_CHECK(cudaStreamSynchronize(st));
    *total_out = total;
    if (total > capacity) return TG_ERR_CAPACITY;
    compact_pool_kernel<<<tg_num_sms() * 8, 256, 0, st>>>(n, src_off, near_indptr, pool_ids, pool_dist, near_ids,
                                                         near_dist); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_near_transpose_workspace_bytes(int64_t n, int64_t) { return tg_align_up((size_t)n * 4, 256) * 2 + 256; }

TG_API int tg_near_transpose(int64_t n, const int64_t *ip, const int32_t *ids, const double *dd, int64_t *rip,
                             int32_t *rids, double *rdd, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || !ip || !rip) return TG_ERR_ARG;
    if (ws_bytes < tg_near_transpose_workspace_bytes(n, 0)) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    TgArena ar(ws, ws_bytes);
    int32_t *cnt = ar.take<int32_t>(n);
    int32_t *cur = ar.take<int32_t>(n);
    int64_t E = 0;
    TG_CUDA_CHECK(cudaMemcpyAsync(&E, ip + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    TG_CUDA_CHECK(cudaStreamSynchronize(st));
    TG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, n * 4, st));
    TG_CUDA_CHECK(cudaMemsetAsync(cur, 0, n * 4, st));
    if (E > 0) near_count_kernel<<<(unsigned)((E + 255) / 256), 256, 0, st>>>(ids, E, cnt); tg_count_launch(1);
    scan_i32_to_i64_kernel<<<1, 1024, 0, st>>>(cnt, n, rip); tg_count_launch(1);
    if (E > 0) near_scatter_kernel<<<tg_num_sms() * 8, 128, 0, st>>>(n, ip, ids, dd, rip, cur, rids, rdd); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
