// dbht.cu -- DBHT on the B200: bubble tree, orientation, converging sinks,
// vertex assignment, distance blocks, group-max matrices and NN-chain linkage.
//
// Replaces dbht.py:64-230 (build_bubble_tree, orient_edges, _next_hops,
// bubble_sinks, assign_vertices, _cluster_max_matrix), the oracle accessors
// apsp.py:88-158 (query / block) and linkage.py:50-94 (_nn_chain), plus
// _kernels.py:184-201 (segment_pair_max).
//
// The dominant kernel is the group max in hub mode: for every vertex pair of
// the (permuted) member list, est(u,v) = min_h hd[h,u] + hd[h,v] -- a min-plus
// "GEMM" over the H hub rows on the fp64 CUDA-core pipe (no tensor path exists
// for min-plus) -- overridden by the exact near-table distances, then reduced
// by max into the (group x group) matrix.  Tiles of 64x64 pairs, hub columns
// staged in shared memory 32 hubs at a time, 4x4 register micro-tiles.
#include "common.cuh"

#include <cooperative_groups.h>
#include <cstdlib>
#include <cstdlib>

namespace {

// ------------------------------------------------------------ oracle access
__device__ __forceinline__ bool near_find(const int64_t *ip, const int32_t *ids, const double *dd, int u, int v,
                                          double &out) {
    int64_t lo = ip[u], hi = ip[u + 1];
    while (lo < hi) {  // np.searchsorted(ids, v) (left)
        int64_t mid = (lo + hi) >> 1;
        if (ids[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    if (lo < ip[u + 1] && ids[lo] == v) {
        out = dd[lo];
        return true;
    }
    return false;
}

__device__ __forceinline__ double hub_min(const tg_oracle_t &o, int u, int v) {
    double best = INFINITY;
    for (int64_t h = 0; h < o.H; h++) {
        double s = __dadd_rn(o.hub_dist[h * o.n + u], o.hub_dist[h * o.n + v]);
        best = s < best ? s : best;
    }
    return best;
}

// apsp.py:127-136 HubOracle.query / apsp.py:88-90 ExactOracle.query
__device__ double oracle_query(const tg_oracle_t &o, int u, int v) {
    if (o.mode == 0) return o.matrix[(int64_t)u * o.n + v];
    if (u == v) return 0.0;
    int a = u < v ? u : v, b = u < v ? v : u;
    double d;
    if (near_find(o.near_indptr, o.near_ids, o.near_dist, a, b, d)) return d;
    if (near_find(o.near_indptr, o.near_ids, o.near_dist, b, a, d)) return d;
    return hub_min(o, a, b);
}

// apsp.py:138-158 HubOracle.block entry (column-vertex table wins over the row's)
__device__ double oracle_block(const tg_oracle_t &o, int u, int v) {
    if (o.mode == 0) return o.matrix[(int64_t)u * o.n + v];
    double d;
    if (near_find(o.near_indptr, o.near_ids, o.near_dist, v, u, d)) return d;
    if (near_find(o.near_indptr, o.near_ids, o.near_dist, u, v, d)) return d;
    return hub_min(o, u, v);
}

__device__ __forceinline__ void sort3i(int &x, int &y, int &z) {
    int t;
    if (y < x) { t = x; x = y; y = t; }
    if (z < y) { t = y; y = z; z = t; }
    if (y < x) { t = x; x = y; y = t; }
}

// ------------------------------------------------------------ bubble tree
__global__ void ins_time_kernel(int64_t n, int32_t *ins_t) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) ins_t[i] = -2;
}

__global__ void ins_time_set_kernel(const int32_t *clique, const int32_t *trace, int64_t nt, int32_t *ins_t) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 4) ins_t[clique[t]] = -1;
    if (t < nt) ins_t[trace[4 * t]] = (int32_t)t;
}

__device__ __forceinline__ unsigned long long face_key(int x, int y, int z, int64_t n) {
    return ((unsigned long long)x * (unsigned long long)n + (unsigned long long)y) * (unsigned long long)n +
           (unsigned long long)z + 1ull;
}

// dbht.py:64-89: the owner of a live face is the bubble created by the insertion
// of its latest-inserted vertex (0 for faces of the initial clique); a row is
// valid iff its face was created before it and not consumed by an earlier row.
__global__ void bubble_tree_kernel(const int32_t *clique, const int32_t *trace, int64_t nt, int64_t n,
                                   const int32_t *ins_t, unsigned long long *htab, int64_t hmask,
                                   int32_t *bubbles, int32_t *links, int32_t *link_faces,
                                   unsigned long long *bad_min) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) {
        int a = clique[0], b = clique[1], c = clique[2], d = clique[3];
        int q[4] = {a, b, c, d};
        for (int i = 0; i < 4; i++)
            for (int j = i + 1; j < 4; j++)
                if (q[j] < q[i]) { int x = q[i]; q[i] = q[j]; q[j] = x; }
        for (int i = 0; i < 4; i++) bubbles[i] = q[i];
    }
    if (t >= nt) return;
    int v = trace[4 * t], x = trace[4 * t + 1], y = trace[4 * t + 2], z = trace[4 * t + 3];
    sort3i(x, y, z);
    bool ok = true;
    int tx = ins_t[x], ty = ins_t[y], tz = ins_t[z];
    if (tx == -2 || ty == -2 || tz == -2) ok = false;
    int tw = max(tx, max(ty, tz));
    int owner = 0;
    if (ok && tw >= (int)t) ok = false;
    if (ok && tw >= 0) {
        int w = (tw == tx) ? x : ((tw == ty) ? y : z);
        int o1 = (w == x) ? y : x, o2 = (w == z) ? y : z;
        if (w == y) { o1 = x; o2 = z; }
        // F \ {w} must be two vertices of the host face of row tw, and w = v(tw)
        const int32_t *r = trace + 4 * (int64_t)tw;
        bool h1 = (o1 == r[1] || o1 == r[2] || o1 == r[3]);
        bool h2 = (o2 == r[1] || o2 == r[2] || o2 == r[3]);
        if (!(h1 && h2 && r[0] == w)) ok = false;
        owner = tw + 1;
    }
    // a face can be consumed once: the later duplicate row is invalid
    unsigned long long key = face_key(x, y, z, n);
    int64_t h = (int64_t)((key * 0x9E3779B97F4A7C15ull) >> 20) & hmask;
    for (;;) {
        unsigned long long prev = atomicCAS(&htab[2 * h], 0ull, key);
        if (prev == 0ull) {
            atomicMin(&htab[2 * h + 1], (unsigned long long)t);
            break;
        }
        if (prev == key) {
            atomicMin(&htab[2 * h + 1], (unsigned long long)t);
            break;
        }
        h = (h + 1) & hmask;
    }
    int q[4] = {v, x, y, z};
    for (int i = 0; i < 4; i++)
        for (int j = i + 1; j < 4; j++)
            if (q[j] < q[i]) { int s = q[i]; q[i] = q[j]; q[j] = s; }
    for (int i = 0; i < 4; i++) bubbles[4 * (t + 1) + i] = q[i];
    links[2 * t] = owner;
    links[2 * t + 1] = (int32_t)(t + 1);
    link_faces[3 * t] = x;
    link_faces[3 * t + 1] = y;
    link_faces[3 * t + 2] = z;
    if (!ok) atomicMin(bad_min, (unsigned long long)t);
}

__global__ void bubble_dup_kernel(const int32_t *trace, int64_t nt, int64_t n, const unsigned long long *htab,
                                  int64_t hmask, unsigned long long *bad_min) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int x = trace[4 * t + 1], y = trace[4 * t + 2], z = trace[4 * t + 3];
    sort3i(x, y, z);
    unsigned long long key = face_key(x, y, z, n);
    int64_t h = (int64_t)((key * 0x9E3779B97F4A7C15ull) >> 20) & hmask;
    while (htab[2 * h] != key) h = (h + 1) & hmask;
    if (htab[2 * h + 1] != (unsigned long long)t) atomicMin(bad_min, (unsigned long long)t);
}

// ------------------------------------------------------------ orientation
__device__ __forceinline__ int apex_of(const int32_t *bub, int f0, int f1, int f2) {
    for (int k = 0; k < 4; k++) {
        int w = bub[k];
        if (w != f0 && w != f1 && w != f2) return w;
    }
    return -1;
}

__global__ void orient_kernel(const double *S, int64_t n, const int32_t *bubbles, const int32_t *links,
                              const int32_t *faces, int64_t L, int64_t *src, int64_t *dst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    int b1 = links[2 * i], b2 = links[2 * i + 1];
    int f0 = faces[3 * i], f1 = faces[3 * i + 1], f2 = faces[3 * i + 2];
    int a1 = apex_of(bubbles + 4 * (int64_t)b1, f0, f1, f2);
    int a2 = apex_of(bubbles + 4 * (int64_t)b2, f0, f1, f2);
    // tmfg.py:82-85 gain: S[a,v] + S[b,v] + S[c,v], left to right
    double g1 = __dadd_rn(__dadd_rn(S[(int64_t)f0 * n + a1], S[(int64_t)f1 * n + a1]), S[(int64_t)f2 * n + a1]);
    double g2 = __dadd_rn(__dadd_rn(S[(int64_t)f0 * n + a2], S[(int64_t)f1 * n + a2]), S[(int64_t)f2 * n + a2]);
    int s, d;
    if (g2 > g1) { s = b1; d = b2; }
    else if (g1 > g2) { s = b2; d = b1; }
    else if (b2 < b1) { s = b1; d = b2; }
    else { s = b2; d = b1; }
    src[i] = s;
    dst[i] = d;
}

// ------------------------------------------------------------ next hops + sinks
__device__ __forceinline__ double edge_gain(const double *S, int64_t n, int f0, int f1, int f2, int apex) {
    // dbht.py:131-140: total = 0.0 then += weight of (w, apex) over the sorted face
    double t = 0.0;
    int f[3] = {f0, f1, f2};
    for (int k = 0; k < 3; k++) {
        int a = f[k] < apex ? f[k] : apex, b = f[k] < apex ? apex : f[k];
        t = __dadd_rn(t, S[(int64_t)a * n + b]);
    }
    return t;
}

__global__ void hop_gain_kernel(const double *S, int64_t n, const int32_t *bubbles, const int32_t *faces,
                                const int64_t *src, const int64_t *dst, int64_t L, double *g_out,
                                unsigned long long *best) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    int f0 = faces[3 * i], f1 = faces[3 * i + 1], f2 = faces[3 * i + 2];
    int d = (int)dst[i];
    int apex = apex_of(bubbles + 4 * (int64_t)d, f0, f1, f2);
    double g = edge_gain(S, n, f0, f1, f2, apex);
    g_out[i] = g;
    atomicMax(&best[src[i]], tg_order_key(g));
}

__global__ void hop_pick_kernel(const int64_t *src, const int64_t *dst, int64_t L, const double *g,
                                const unsigned long long *best, int64_t *hops) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    if (tg_order_key(g[i]) == best[src[i]]) atomicMin((unsigned long long *)&hops[src[i]], (unsigned long long)dst[i]);
}

__global__ void sink_init_kernel(int64_t m, int64_t *hops, int64_t *sink) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m) return;
    sink[b] = hops[b] < 0 ? b : hops[b];
}

__global__ void sink_jump_kernel(int64_t m, const int64_t *in, int64_t *out, int *changed) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= m) return;
    int64_t s = in[b];
    int64_t t = in[s];
    out[b] = t;
    if (t != s) *changed = 1;
}

// ------------------------------------------------------------ assignment
__global__ void assign_mean_kernel(tg_oracle_t o, const int32_t *bubbles, int64_t m, double *mean_out,
                                   unsigned long long *best) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (bubble, member) pair
    if (i >= 4 * m) return;
    int64_t bid = i >> 2;
    const int32_t *bub = bubbles + 4 * bid;
    int v = bub[i & 3];
    double total = 0.0;
    for (int k = 0; k < 4; k++) {
        int w = bub[k];
        double q = (w == v) ? 0.0 : oracle_query(o, v, w);
        total = __dadd_rn(total, q);
    }
    double mean = total / 4.0;
    mean_out[i] = mean;
    atomicMin(&best[v], tg_order_key(mean));
}

__global__ void assign_pick_kernel(const int32_t *bubbles, int64_t m, const double *mean,
                                   const unsigned long long *best, int64_t *vb) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 4 * m) return;
    int v = bubbles[i];
    if (tg_order_key(mean[i]) == best[v]) atomicMin((unsigned long long *)&vb[v], (unsigned long long)(i >> 2));
}

__global__ void assign_conv_kernel(int64_t n, const int64_t *vb, const int64_t *sinks, int64_t *vc) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) vc[v] = sinks[vb[v]];
}

// ------------------------------------------------------------ group blocks (layer 1)
__global__ void group_blocks_kernel(tg_oracle_t o, const int32_t *perm, const int64_t *starts, int64_t count,
                                    const int64_t *boff, double *out) {
    for (int64_t g = blockIdx.x; g < count; g += gridDim.x) {
        int64_t s0 = starts[g];
        int gsz = (int)(starts[g + 1] - s0);
        double *B = out + boff[g];
        for (int e = threadIdx.x; e < gsz * gsz; e += blockDim.x) {
            int i = e / gsz, j = e % gsz;
            B[e] = oracle_block(o, perm[s0 + i], perm[s0 + j]);
        }
    }
}

// ------------------------------------------------------------ group max (layers 2 and 3)
constexpr int NN_WARP_MAX = 48;  // larger matrices take the CTA-per-matrix NN-chain
constexpr int GM_T = 256;
constexpr int GM_TILE = 64;
constexpr int GM_HC = 32;   // hubs staged per chunk

struct GmTile {
    int sub;   // sub-problem
    int i0, j0;
};

struct GmSub {
    int64_t perm_off;   // into perm / gid
    int32_t len;        // vertices
    int32_t m;          // groups
    int64_t out_off;    // into out (m x m)
    int64_t tile_off;   // first tile of this sub-problem (row-major, nt x nt tiles)
};

// out is pre-filled with 0 bits (all distances >= 0); atomicMax on raw bits.
__global__ void __launch_bounds__(GM_T)
group_max_tile_kernel(tg_oracle_t o, const int32_t *__restrict__ perm, const int32_t *__restrict__ gid,
                      const int32_t *__restrict__ pos, const GmSub *__restrict__ subs, const GmTile *__restrict__ tiles,
                      int64_t ntiles, unsigned long long *__restrict__ out, const uint64_t *__restrict__ mask) {
    // the hub panels (A, B) and the pair tile E are never live together
    __shared__ __align__(16) double gm_raw[GM_TILE * (GM_TILE + 1)];
    double (*A)[GM_TILE] = reinterpret_cast<double (*)[GM_TILE]>(gm_raw);
    double (*B)[GM_TILE] = reinterpret_cast<double (*)[GM_TILE]>(gm_raw + GM_HC * GM_TILE);
    double (*E)[GM_TILE + 1] = reinterpret_cast<double (*)[GM_TILE + 1]>(gm_raw);
    __shared__ int ru[GM_TILE], cv[GM_TILE], rg[GM_TILE], cg[GM_TILE];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4x4 pairs each
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const GmTile tl = tiles[t];
        const GmSub sb = subs[tl.sub];
        const int rows = min(GM_TILE, sb.len - tl.i0), cols = min(GM_TILE, sb.len - tl.j0);
        if (tid < GM_TILE) {
            int i = tid;
            ru[i] = i < rows ? perm[sb.perm_off + tl.i0 + i] : -1;
            rg[i] = i < rows ? gid[sb.perm_off + tl.i0 + i] : -1;
            cv[i] = i < cols ? perm[sb.perm_off + tl.j0 + i] : -1;
            cg[i] = i < cols ? gid[sb.perm_off + tl.j0 + i] : -1;
        }
        __syncthreads();
        if (o.mode == 1) {
            double acc[4][4];
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c] = INFINITY;
            for (int64_t h0 = 0; h0 < o.H; h0 += GM_HC) {
                const int hc = (int)min((int64_t)GM_HC, o.H - h0);
                for (int e = tid; e < GM_HC * GM_TILE; e += GM_T) {
                    int h = e / GM_TILE, i = e % GM_TILE;
                    double a = INFINITY, b = INFINITY;
                    if (h < hc) {
                        if (ru[i] >= 0) a = o.hub_dist[(h0 + h) * o.n + ru[i]];
                        if (cv[i] >= 0) b = o.hub_dist[(h0 + h) * o.n + cv[i]];
                    }
                    A[h][i] = a;
                    B[h][i] = b;
                }
                __syncthreads();
                for (int h = 0; h < hc; h++) {
                    double a[4], b[4];
#pragma unroll
                    for (int r = 0; r < 4; r++) a[r] = A[h][ty + 16 * r];
#pragma unroll
                    for (int c = 0; c < 4; c++) b[c] = B[h][tx + 16 * c];
#pragma unroll
                    for (int r = 0; r < 4; r++)
#pragma unroll
                        for (int c = 0; c < 4; c++) acc[r][c] = fmin(acc[r][c], __dadd_rn(a[r], b[c]));
                }
                __syncthreads();
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) E[ty + 16 * r][tx + 16 * c] = acc[r][c];
            __syncthreads();
            // pairs carrying a near-table override were maxed by the override pass
            const uint64_t *mk = mask + (size_t)t * GM_TILE;
            for (int e = tid; e < GM_TILE * GM_TILE; e += GM_T) {
                int i = e / GM_TILE, j = e % GM_TILE;
                if ((mk[i] >> j) & 1ull) E[i][j] = 0.0;
            }
            __syncthreads();
        } else {
            for (int e = tid; e < GM_TILE * GM_TILE; e += GM_T) {
                int i = e / GM_TILE, j = e % GM_TILE;
                E[i][j] = (i < rows && j < cols) ? o.matrix[(int64_t)ru[i] * o.n + cv[j]] : 0.0;
            }
            __syncthreads();
        }
        // per (row group, column group) segment max -> atomicMax
        for (int i = tid; i < rows; i += GM_T) {
            int gi = rg[i];
            int j = 0;
            while (j < cols) {
                int gj = cg[j];
                double best = E[i][j];
                int k = j + 1;
                while (k < cols && cg[k] == gj) {
                    best = fmax(best, E[i][k]);
                    k++;
                }
                // exact mode: only the lower group's rows count (_kernels.py:188-201)
                if (o.mode == 1 || gi <= gj) atomicMax(&out[sb.out_off + (int64_t)gi * sb.m + gj], tg_dbits(best));
                j = k;
            }
        }
        __syncthreads();
    }
}

// Hub-mode group max with an fp32 screen.  For a pair (u, v) the hub estimate is
// D = min_h fl64(hd[h,u] + hd[h,v]) (apsp.py:136-143); in fp32, d' = min_h
// fl32(fl32(hd[h,u]) + fl32(hd[h,v])) satisfies |d' - D| <= 2^-22.8 D + 2^-147
// (all terms >= 0).  Per tile and per (row group run, column group run) the
// largest d' is taken; every pair with d' >= lmax' (1 - 2^-21) - 2^-140 -- a
// superset of the pairs attaining the tile-local maximum of D -- gets its exact
// fp64 D and only those are maxed into M.  The maximum over tiles of the exact
// tile-local maxima is M's exact entry.  The hub distances are first laid out
// vertex-major in the sub-problems' permuted order (hp_fill_kernel, fp32 and
// fp64 copies), so every panel load is a coalesced row segment.
constexpr int GH_T = 256;
constexpr int GH_MAXC = GM_TILE * GM_TILE;
constexpr int GH_LD = GM_HC + 2;   // panel row stride: 17 8-byte words (odd), so 16 consecutive rows'
                                   // float2 reads hit distinct 8-byte bank pairs

__global__ void hp_fill_kernel(tg_oracle_t o, const int32_t *__restrict__ perm, int64_t total, int Hp,
                               float *__restrict__ hpf, double *__restrict__ hpd) {
    const int64_t cnt = total * Hp;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = e / Hp;
        const int h = (int)(e - g * Hp);
        const double x = h < o.H ? o.hub_dist[(int64_t)h * o.n + perm[g]] : INFINITY;
        hpd[e] = x;
        hpf[e] = (float)x;
    }
}

__global__ void __launch_bounds__(GH_T, 3)
group_max_hub_kernel(tg_oracle_t o, const int32_t *__restrict__ gid, const GmSub *__restrict__ subs,
                     const GmTile *__restrict__ tiles, int64_t ntiles, int Hp, const float *__restrict__ hpf,
                     const double *__restrict__ hpd, unsigned long long *__restrict__ out,
                     const uint64_t *__restrict__ mask) {
    constexpr int PF = GM_TILE * GH_LD * 4;
    __shared__ __align__(16) unsigned char gh_raw[2 * PF + GM_TILE * GM_TILE * 4];
    float (*Af)[GH_LD] = reinterpret_cast<float (*)[GH_LD]>(gh_raw);     // [64 rows][32 hubs]
    float (*Bf)[GH_LD] = reinterpret_cast<float (*)[GH_LD]>(gh_raw + PF);
    unsigned *lmax = reinterpret_cast<unsigned *>(gh_raw + 2 * PF);      // [64 runs][64 runs]
    __shared__ uint16_t cand[GH_MAXC];
    __shared__ int ncand;
    __shared__ int rg[GM_TILE], cg[GM_TILE], lr[GM_TILE], lc[GM_TILE];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tid & 15, ty = tid >> 4;   // 16 x 16 threads, rows ty + 16 r, cols tx + 16 c
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const GmTile tl = tiles[t];
        // the hub estimate D(u, v) = min_h fl(hd[h,u] + hd[h,v]) is symmetric, and so is the
        // override set (u in near(v) or v in near(u)): a tile below the diagonal repeats the
        // transposed tile's pairs, whose maxima are written to both orientations instead
        if (tl.i0 > tl.j0) continue;
        const bool mirror = tl.i0 < tl.j0;
        const GmSub sb = subs[tl.sub];
        const int rows = min(GM_TILE, sb.len - tl.i0), cols = min(GM_TILE, sb.len - tl.j0);
        const int64_t rbase = sb.perm_off + tl.i0, cbase = sb.perm_off + tl.j0;
        if (tid < GM_TILE) {
            const int i = tid;
            rg[i] = i < rows ? gid[rbase + i] : -1;
            cg[i] = i < cols ? gid[cbase + i] : -1;
        }
        if (tid == 0) ncand = 0;
        for (int e = tid; e < GM_TILE * GM_TILE; e += GH_T) lmax[e] = 0u;
        __syncthreads();
        if (warp < 2) {   // run index of each row (warp 0) / column (warp 1) group
            const int *g = warp == 0 ? rg : cg;
            int *l = warp == 0 ? lr : lc;
            int carry = 0;
            for (int base = 0; base < GM_TILE; base += 32) {
                const int i = base + lane;
                const unsigned b = __ballot_sync(0xffffffffu, i > 0 && g[i] != g[i - 1]);
                l[i] = carry + __popc(b & (0xffffffffu >> (31 - lane)));
                carry += __popc(b);
            }
        }
        // ---- fp32 screen
        float acc[4][4];
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 4; c++) acc[r][c] = INFINITY;
        for (int h0 = 0; h0 < Hp; h0 += GM_HC) {
            // 16-byte panel loads (rows of Hp floats, Hp a multiple of 32: aligned), 8-byte stores
            for (int e = tid; e < GM_HC * GM_TILE / 4; e += GH_T) {
                const int i = e >> 3, h = (e & 7) * 4;
                const float4 inf4 = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
                const float4 a = i < rows ? *reinterpret_cast<const float4 *>(hpf + (rbase + i) * Hp + h0 + h) : inf4;
                const float4 b = i < cols ? *reinterpret_cast<const float4 *>(hpf + (cbase + i) * Hp + h0 + h) : inf4;
                *reinterpret_cast<float2 *>(&Af[i][h]) = make_float2(a.x, a.y);
                *reinterpret_cast<float2 *>(&Af[i][h + 2]) = make_float2(a.z, a.w);
                *reinterpret_cast<float2 *>(&Bf[i][h]) = make_float2(b.x, b.y);
                *reinterpret_cast<float2 *>(&Bf[i][h + 2]) = make_float2(b.z, b.w);
            }
            __syncthreads();
            // two hubs per step: one packed fp32x2 add (FADD2: two independent round-to-nearest
            // fp32 adds) and one three-input min (FMNMX3) per pair -- the same d' as two FADD +
            // two FMNMX, in half the instructions
#pragma unroll 4
            for (int h = 0; h < GM_HC; h += 2) {
                unsigned long long av[4], bv[4];
#pragma unroll
                for (int r = 0; r < 4; r++) av[r] = *reinterpret_cast<const unsigned long long *>(&Af[ty + 16 * r][h]);
#pragma unroll
                for (int c = 0; c < 4; c++) bv[c] = *reinterpret_cast<const unsigned long long *>(&Bf[tx + 16 * c][h]);
#pragma unroll
                for (int r = 0; r < 4; r++)
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        unsigned long long sum;
                        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(sum) : "l"(av[r]), "l"(bv[c]));
                        float m3;
                        asm("min.f32 %0, %1, %2, %3;"
                            : "=f"(m3)
                            : "f"(acc[r][c]), "f"(__uint_as_float((unsigned)sum)),
                              "f"(__uint_as_float((unsigned)(sum >> 32))));
                        acc[r][c] = m3;
                    }
            }
            __syncthreads();
        }
        // ---- tile-local maxima per (row run, column run); override pairs are excluded
        const uint64_t *mk = mask + (size_t)t * GM_TILE;
        uint32_t valid = 0;
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int i = ty + 16 * r;
            const uint64_t mrow = i < rows ? mk[i] : ~0ull;
#pragma unroll
            for (int c = 0; c < 4; c++) {
                const int j = tx + 16 * c;
                if (i < rows && j < cols && !((mrow >> j) & 1ull)) {
                    valid |= 1u << (r * 4 + c);
                    atomicMax(&lmax[lr[i] * GM_TILE + lc[j]], __float_as_uint(acc[r][c]));
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < 4; c++) {
                if (!((valid >> (r * 4 + c)) & 1u)) continue;
                const int i = ty + 16 * r, j = tx + 16 * c;
                // (an overflowed lmax' = inf still admits every pair near FLT_MAX)
                const float lm = fminf(__uint_as_float(lmax[lr[i] * GM_TILE + lc[j]]), 3.4028235e38f);
                // |d' - D| <= e D + t (e = 2^-22.8, t = 2^-147) gives, for a pair attaining the exact
                // maximum, d' >= lmax' (1 - 2e) - 2t; 1 - 2^-21 stays below 1 - 2e after the rounding
                // of the product (2^-21 - 2^-24 > 2^-21.8)
                const float thr = __fsub_rn(__fmul_rn(lm, 1.0f - 0x1p-21f), 0x1p-140f);
                if (acc[r][c] >= thr) cand[atomicAdd(&ncand, 1)] = (uint16_t)((i << 6) | j);
            }
        __syncthreads();
        // ---- exact fp64 estimate of the candidates: one warp per candidate, lanes over the
        // hubs of the two vertex-major rows (coalesced, L2-resident), then a warp min
        const int nc = ncand;
        for (int k = warp; k < nc; k += GH_T / 32) {
            const int ci = cand[k] >> 6, cj = cand[k] & 63;
            const double *ha = hpd + (rbase + ci) * Hp, *hb = hpd + (cbase + cj) * Hp;
            double ex = INFINITY;
            for (int h0 = 0; h0 < Hp; h0 += 256) {   // every load of a 256-hub chunk in flight at once
                double xa[8], xb[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int h = h0 + u * 32 + lane;
                    xa[u] = h < Hp ? ha[h] : INFINITY;
                    xb[u] = h < Hp ? hb[h] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 8; u++) ex = fmin(ex, __dadd_rn(xa[u], xb[u]));
            }
            for (int o = 16; o; o >>= 1) ex = fmin(ex, __shfl_xor_sync(0xffffffffu, ex, o));
            if (lane == 0) {
                atomicMax(&out[sb.out_off + (int64_t)rg[ci] * sb.m + cg[cj]], tg_dbits(ex));
                if (mirror) atomicMax(&out[sb.out_off + (int64_t)cg[cj] * sb.m + rg[ci]], tg_dbits(ex));
            }
        }
        __syncthreads();
    }
}

// Near-table overrides (apsp.py:147-157): for every pair (u, v) of a sub-problem
// with u in near(v) [column table, wins] or v in near(u) [row table], est(u, v)
// is the recorded exact distance.  Pass 0 walks the transposed tables (column
// overrides), pass 1 the row tables and skips pairs pass 0 already claimed.
// Each claimed pair sets its bit in the tile mask and maxes its value into M.
__global__ void group_max_override_kernel(tg_oracle_t o, const int32_t *__restrict__ perm,
                                          const int32_t *__restrict__ gid, const int32_t *__restrict__ pos,
                                          const int32_t *__restrict__ vsub, const GmSub *__restrict__ subs,
                                          int64_t nsub, int64_t total_len, int pass, uint64_t *__restrict__ mask,
                                          unsigned long long *__restrict__ out) {
    const int64_t *ip = pass == 0 ? o.rev_indptr : o.near_indptr;
    const int32_t *ids = pass == 0 ? o.rev_ids : o.near_ids;
    const double *dd = pass == 0 ? o.rev_dist : o.near_dist;
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t g = wid; g < total_len; g += nwarps) {
        const int u = perm[g];
        const int p = vsub[u];
        const GmSub sb = subs[p];
        const int i = (int)(g - sb.perm_off);
        const int nt = (sb.len + GM_TILE - 1) / GM_TILE;
        const int gi = gid[g];
        for (int64_t k = ip[u] + lane; k < ip[u + 1]; k += 32) {
            const int v = ids[k];
            if (vsub[v] != p) continue;
            const int j = (int)(pos[v] - sb.perm_off);
            const int64_t t = sb.tile_off + (int64_t)(i / GM_TILE) * nt + (j / GM_TILE);
            uint64_t *word = mask + (size_t)t * GM_TILE + (i % GM_TILE);
            const uint64_t bit = 1ull << (j % GM_TILE);
            if (pass == 1 && ((*word) & bit)) continue;   // a column override already owns the pair
            atomicOr((unsigned long long *)word, (unsigned long long)bit);
            atomicMax(&out[sb.out_off + (int64_t)gi * sb.m + gid[pos[v]]], tg_dbits(dd[k]));
        }
    }
}

// exact mode: the kernels fill the upper triangle only; mirror it (segment_pair_max is
// symmetric).  32x32 tiles through shared memory so both the read and the write coalesce;
// every block walks all sub-problems, taking every gridDim.x-th tile of each (the first
// tile rotating with the sub-problem so that many one-tile sub-problems spread out).
__global__ void group_max_finalize_kernel(const GmSub *subs, int64_t nsub, double *out) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    for (int64_t p = 0; p < nsub; p++) {
        const GmSub sb = subs[p];
        const int m = sb.m, nt = (m + 31) / 32;
        double *M = out + sb.out_off;
        const int64_t t0 = ((int64_t)blockIdx.x + gridDim.x - p % gridDim.x) % gridDim.x;
        for (int64_t t = t0; t < (int64_t)nt * nt; t += gridDim.x) {
            const int ti = (int)(t / nt), tj = (int)(t % nt);
            if (tj > ti) continue;
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {   // source rows j (tile tj), columns i (tile ti)
                const int j = tj * 32 + r, i = ti * 32 + tx;
                if (j < m && i < m) tile[r][tx] = M[(int64_t)j * m + i];
            }
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {   // destination rows i, columns j, i > j
                const int i = ti * 32 + r, j = tj * 32 + tx;
                if (i < m && j < m && i > j) M[(int64_t)i * m + j] = tile[tx][r];
            }
        }
    }
}

// ------------------------------------------------------------ NN-chain (linkage.py:50-94)
// One warp per matrix; the matrix itself is the working copy W.
__global__ void nn_chain_kernel(double *mats, const int64_t *mat_off, const int64_t *sizes, int64_t count,
                                const int64_t *merge_off, int64_t *lefts, int64_t *rights, double *heights,
                                uint8_t *active_all, int64_t *slot_all, int64_t *chain_all, const int64_t *aux_off) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = wid; b < count; b += nwarps) {
        const int64_t m = sizes[b];
        if (m < 2 || m > NN_WARP_MAX) continue;
        double *W = mats + mat_off[b];
        uint8_t *active = active_all + aux_off[b];
        int64_t *slot = slot_all + aux_off[b];
        int64_t *chain = chain_all + aux_off[b];
        int64_t *L = lefts + merge_off[b], *R = rights + merge_off[b];
        double *Hh = heights + merge_off[b];
        for (int64_t i = lane; i < m; i += 32) {
            active[i] = 1;
            slot[i] = i;
            W[i * m + i] = INFINITY;
        }
        __syncwarp();
        int64_t nchain = 0, next_id = m, remaining = m, nm = 0;
        while (remaining > 1) {
            if (nchain == 0) {
                int64_t f = -1;
                for (int64_t i0 = 0; i0 < m && f < 0; i0 += 32) {
                    int64_t i = i0 + lane;
                    unsigned bal = __ballot_sync(0xffffffffu, i < m && active[i]);
                    if (bal) f = i0 + __ffs(bal) - 1;
                }
                chain[nchain++] = f;
            }
            const int64_t x = chain[nchain - 1];
            // y = argmin over active j != x of W[x, j] (first index on ties)
            double bv = INFINITY;
            int64_t bi = INT64_MAX;
            for (int64_t j = lane; j < m; j += 32) {
                double r = (active[j] && j != x) ? W[x * m + j] : INFINITY;
                if (r < bv || (r == bv && j < bi)) { bv = r; bi = j; }
            }
            for (int o = 16; o; o >>= 1) {
                double r2 = __shfl_xor_sync(0xffffffffu, bv, o);
                int64_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (r2 < bv || (r2 == bv && i2 < bi)) { bv = r2; bi = i2; }
            }
            int64_t y = (bi == INT64_MAX) ? 0 : bi;  // all-inf row: np.argmin -> 0
            if (nchain > 1) {
                int64_t p = chain[nchain - 2];
                double rp = (active[p] && p != x) ? W[x * m + p] : INFINITY;
                double ry = (active[y] && y != x) ? W[x * m + y] : INFINITY;
                if (rp == ry) y = p;
            }
            if (nchain > 1 && y == chain[nchain - 2]) {
                nchain -= 2;
                const double h = W[x * m + y];
                const int64_t lo = x < y ? x : y, hi = x < y ? y : x;
                if (lane == 0) {
                    L[nm] = slot[x];
                    R[nm] = slot[y];
                    Hh[nm] = h;
                }
                nm++;
                // merged = max(W[lo], W[hi]); W[lo] = merged; W[:, lo] = merged; W[lo, lo] = inf
                for (int64_t j = lane; j < m; j += 32) {
                    double p = W[lo * m + j], q = W[hi * m + j];
                    double mg = p > q ? p : (q > p ? q : p);
                    W[lo * m + j] = mg;
                    W[j * m + lo] = mg;
                }
                __syncwarp();
                if (lane == 0) {
                    W[lo * m + lo] = INFINITY;
                    active[hi] = 0;
                    slot[lo] = next_id;
                }
                next_id++;
                remaining--;
                __syncwarp();
            } else {
                if (nchain >= m) {  // a non-reducible (asymmetric) matrix made the chain cycle
                    if (lane == 0) Hh[0] = __longlong_as_double(0x7ff8dead00000000ll);
                    break;
                }
                chain[nchain++] = y;
            }
        }
    }
}

__global__ void pos_fill_kernel(const GmSub *subs, int64_t nsub, const int32_t *perm, int32_t *pos, int32_t *vsub) {
    for (int64_t p = blockIdx.x; p < nsub; p += gridDim.x)
        for (int i = threadIdx.x; i < subs[p].len; i += blockDim.x) {
            const int v = perm[subs[p].perm_off + i];
            pos[v] = (int32_t)(subs[p].perm_off + i);  // global position
            vsub[v] = (int32_t)p;
        }
}

__global__ void oracle_block_kernel(tg_oracle_t o, const int32_t *rows, int64_t nr, const int32_t *cols, int64_t nc,
                                    int q, double *out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nr * nc) return;
    int u = rows[e / nc], v = cols[e % nc];
    out[e] = q ? oracle_query(o, u, v) : oracle_block(o, u, v);
}

// Larger matrices: one CTA per matrix, rows scanned by the whole block.  Chain,
// activity flags and slot ids live in shared memory (m <= NN_SMEM_MAX); each
// step is one coalesced row read (L2), a two-level argmin (shuffles, then warp 0)
// and two barriers.  The value at the chain's second-to-last entry -- needed by
// the tie rule -- is captured during the scan instead of re-read.
constexpr int NN_SMEM_MAX = 7168;
constexpr int NN_CL = 8;          // cluster NN-chain (below): CTAs per cluster
constexpr int NN_CL_T = 256;      //   threads per CTA
constexpr int NN_CL_U = 4;        //   row entries in flight per thread (one pass covers 1024 columns)
constexpr int NN_CL_MIN = 2048;   //   matrices with NN_CL_MIN <= m <= NN_SMEM_MAX (HBM-resident rows;
                                  //   L2-resident smaller ones step faster in one CTA)
constexpr int NN_BIG = 2048;   // larger matrices: 1024 threads, 8 row entries in flight per thread
#ifndef NN_SMALL_T_DEF
#define NN_SMALL_T_DEF 512
#define NN_SMALL_U_DEF 4
#endif
constexpr int NN_SMALL_T = NN_SMALL_T_DEF, NN_SMALL_U = NN_SMALL_U_DEF;

// Order key of a row entry for the argmin: unsigned order = double order for every non-NaN
// value (-0.0 keyed as +0.0: np.argmin compares them equal); NaN keys above +inf, so a NaN is
// never the minimum (as the compare-based scans treat it).
__device__ __forceinline__ unsigned long long nn_key(double r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(r == 0.0 ? 0.0 : r);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// (minimum key, first index attaining it) over the warp: three REDUX steps, no shuffle tree
__device__ __forceinline__ void nn_warp_argmin(unsigned long long k, unsigned i, unsigned &kh, unsigned &kl,
                                               unsigned &ki) {
    const unsigned h = (unsigned)(k >> 32), l = (unsigned)k;
    kh = __reduce_min_sync(0xffffffffu, h);
    kl = __reduce_min_sync(0xffffffffu, h == kh ? l : 0xffffffffu);
    ki = __reduce_min_sync(0xffffffffu, (h == kh && l == kl) ? i : 0xffffffffu);
}

template <int NN_CTA_T, int NN_U, bool BIG>
__global__ void __launch_bounds__(NN_CTA_T)
nn_chain_cta_kernel(double *mats, const int64_t *mat_off, const int64_t *sizes, int64_t count,
                    const int64_t *merge_off, int64_t *lefts, int64_t *rights, double *heights,
                    uint8_t *active_all, int64_t *slot_all, int64_t *chain_all, const int64_t *aux_off,
                    int cl_min) {
    extern __shared__ __align__(16) unsigned char nn_smem[];
    __shared__ uint4 part[2][NN_CTA_T / 32];   // per warp: (key hi, key lo, first index)
    __shared__ double sh_rp[2], sh_patch;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NN_CTA_T / 32;
    // the next chain top's row is read together with the merged rows (one L2 round trip per
    // merge instead of two); the big variant has no registers for a third row
    constexpr bool PREF = !BIG;
    int32_t *s_chain = reinterpret_cast<int32_t *>(nn_smem);
    int32_t *s_slot = s_chain + NN_SMEM_MAX;
    uint8_t *s_act = reinterpret_cast<uint8_t *>(s_slot + NN_SMEM_MAX);
    for (int64_t b = blockIdx.x; b < count; b += gridDim.x) {
        const int64_t m64 = sizes[b];
        if (m64 <= NN_WARP_MAX || BIG != (m64 > NN_BIG)) continue;
        if (cl_min > 0 && m64 >= cl_min && m64 <= NN_SMEM_MAX) continue;   // the cluster kernel's
        const int m = (int)m64;
        double *W = mats + mat_off[b];
        int64_t *L = lefts + merge_off[b], *R = rights + merge_off[b];
        double *Hh = heights + merge_off[b];
        const bool in_smem = m <= NN_SMEM_MAX;
        // state: shared memory when it fits, else the caller's scratch (int64 slot/chain)
        uint8_t *act = in_smem ? s_act : active_all + aux_off[b];
        int64_t *gslot = slot_all + aux_off[b];
        int64_t *gchain = chain_all + aux_off[b];
        auto slot_get = [&](int i) -> int64_t { return in_smem ? (int64_t)s_slot[i] : gslot[i]; };
        auto slot_set = [&](int i, int64_t v) { if (in_smem) s_slot[i] = (int32_t)v; else gslot[i] = v; };
        auto chain_get = [&](int i) -> int { return in_smem ? s_chain[i] : (int)gchain[i]; };
        auto chain_set = [&](int i, int v) { if (in_smem) s_chain[i] = v; else gchain[i] = v; };
        for (int i = tid; i < m; i += NN_CTA_T) {
            act[i] = 1;
            slot_set(i, i);
            W[(int64_t)i * m + i] = INFINITY;
        }
        __syncthreads();
        int nchain = 0, remaining = m, nm = 0, step = 0;
        int64_t next_id = m;
        // every thread reduces the warps' partials itself and so takes the same decision: the
        // chain's top two stay in registers, partials are double-buffered by step parity, and
        // a chain step costs one barrier (a merge: one more after its row / column pass)
        int x = 0, p = -1;
        double rr[NN_U];
        bool have = false;   // rr holds row x (read during the last merge; column `plo` patched)
        int plo = -1;
        while (remaining > 1) {
            if (nchain == 0) {
                // chain start: the first active cluster
                int f = INT_MAX;
                for (int i = tid; i < m; i += NN_CTA_T)
                    if (act[i]) { f = i; break; }
                f = __reduce_min_sync(0xffffffffu, (unsigned)f);
                if (lane == 0) part[0][warp].x = (unsigned)f;
                __syncthreads();
                unsigned g = lane < NW ? part[0][lane].x : 0xffffffffu;
                g = __reduce_min_sync(0xffffffffu, g);
                if (tid == 0) chain_set(0, (int)g);
                __syncthreads();   // part[0] is rewritten by the next step
                nchain = 1;
                x = (int)g;
                p = -1;
                have = false;
            }
            const int par = step & 1;
            const double *row = W + (int64_t)x * m;
            unsigned long long bk = ~0ull;
            unsigned bi = 0xffffffffu;
            for (int j0 = tid; j0 < m; j0 += NN_U * NN_CTA_T) {
                if (!(PREF && have && j0 == tid)) {
#pragma unroll
                    for (int u = 0; u < NN_U; u++) {   // all loads in flight before any use
                        const int j = j0 + u * NN_CTA_T;
                        rr[u] = j < m ? row[j] : INFINITY;
                    }
                }
#pragma unroll
                for (int u = 0; u < NN_U; u++) {
                    const int j = j0 + u * NN_CTA_T;
                    if (j < m) {
                        double r = (act[j] && j != x) ? rr[u] : INFINITY;
                        if (PREF && j == plo) r = sh_patch;   // W[x, lo] of the last merge
                        const unsigned long long k = nn_key(r);
                        if (k < bk) { bk = k; bi = (unsigned)j; }   // j ascends: first index on ties
                        if (j == p) sh_rp[par] = r;
                    }
                }
            }
            have = false;
            plo = -1;
            unsigned kh, kl, ki;
            nn_warp_argmin(bk, bi, kh, kl, ki);
            if (lane == 0) part[par][warp] = make_uint4(kh, kl, ki, 0u);
            __syncthreads();
            {
                const uint4 q = lane < NW ? part[par][lane] : make_uint4(~0u, ~0u, ~0u, 0u);
                nn_warp_argmin(((unsigned long long)q.x << 32) | q.y, q.z, kh, kl, ki);
            }
            const unsigned long long vk = ((unsigned long long)kh << 32) | kl;
            const double rp = p >= 0 ? sh_rp[par] : INFINITY;
            step++;
            int y = (int)ki;   // every column takes part (masked ones as +inf): np.argmin's index
            // linkage.py: prefer the previous chain element on ties (row[y] is the minimum v)
            if (p >= 0 && nn_key(rp) == vk) y = p;
            if (p >= 0 && y == p) {
                nchain -= 2;
                const int lo = x < y ? x : y, hi = x < y ? y : x;
                if (tid == 0) {
                    L[nm] = slot_get(x);
                    R[nm] = slot_get(y);
                    Hh[nm] = rp;
                    act[hi] = 0;          // read again only after the barrier below
                    slot_set(lo, next_id);
                }
                nm++;
                const int xn = nchain > 0 ? chain_get(nchain - 1) : -1;   // the next chain top
                double *Wlo = W + (int64_t)lo * m;
                const double *Whi = W + (int64_t)hi * m;
                const double *Wxn = W + (int64_t)(xn >= 0 ? xn : 0) * m;
                const bool pref = PREF && xn >= 0 && m <= NN_U * NN_CTA_T;
                for (int j0 = tid; j0 < m; j0 += NN_U * NN_CTA_T) {
                    double pv[NN_U], qv[NN_U];
#pragma unroll
                    for (int u = 0; u < NN_U; u++) {
                        const int j = j0 + u * NN_CTA_T;
                        pv[u] = j < m ? Wlo[j] : 0.0;
                        qv[u] = j < m ? Whi[j] : 0.0;
                        if (PREF && pref) rr[u] = j < m ? Wxn[j] : INFINITY;
                    }
#pragma unroll
                    for (int u = 0; u < NN_U; u++) {
                        const int j = j0 + u * NN_CTA_T;
                        if (j < m && j != lo) {   // W[lo, lo] stays inf (linkage.py:88)
                            const double mg = pv[u] > qv[u] ? pv[u] : (qv[u] > pv[u] ? qv[u] : pv[u]);
                            Wlo[j] = mg;
                            W[(int64_t)j * m + lo] = mg;
                            if (PREF && j == xn) sh_patch = mg;   // = the new W[xn, lo]
                        }
                    }
                }
                next_id++;
                remaining--;
                __syncthreads();   // the merged row / column, act[hi] and sh_patch are visible
                if (nchain > 0) {
                    x = xn;
                    p = nchain > 1 ? chain_get(nchain - 2) : -1;
                    have = pref;
                    plo = pref ? lo : -1;
                }
            } else {
                if (nchain >= m) {  // a non-reducible (asymmetric) matrix made the chain cycle
                    if (tid == 0) Hh[0] = __longlong_as_double(0x7ff8dead00000000ll);
                    break;
                }
                if (tid == 0) chain_set(nchain, y);   // read back only after a later barrier
                nchain++;
                p = x;
                x = y;
            }
        }
        __syncthreads();
    }
}


// ------------------------------------------------------------ NN-chain over a thread-block cluster
// For the large matrices (m >= NN_CL_MIN: layer 3 at n = 50k has m = 5906, layer 2 at n = 10k
// up to ~1000) one chain step was one CTA reading a whole row (47 KB at m = 5906) through one
// SM.  Here a cluster of NN_CL CTAs runs one chain: CTA c owns the columns [c m / NN_CL,
// (c + 1) m / NN_CL) of every row.  Per step each CTA scans its slice of row x, reduces it,
// and writes its partial (min value, first index, and W[x, chain[-2]] if it owns that
// column) into every CTA's shared memory (DSMEM; double-buffered by step parity); after one
// cluster barrier every CTA reduces the same partials in the same order, so all of them take
// the same decision and keep identical chain / activity state (linkage.py:50-94 semantics:
// first index on ties, chain[-2] preferred on an equal value, all-inf row -> index 0).  A merge
// updates row lo and column lo slice by slice (each CTA its own columns and its own rows) and
// ends with a second barrier; W is read through L2 (ld.global.cg) so no CTA sees a stale line.

struct NnPart {
    double v, rp;
    int i, has_p;
};

__device__ __forceinline__ void nn_cl_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(NN_CL_T)
nn_chain_cluster_kernel(double *mats, const int64_t *mat_off, const int64_t *sizes, int64_t count,
                        const int64_t *merge_off, int64_t *lefts, int64_t *rights, double *heights, int cl_min) {
    extern __shared__ __align__(16) unsigned char ncl_smem[];
    __shared__ NnPart part[2][NN_CL];
    __shared__ double rv[NN_CL_T / 32], rpv[NN_CL_T / 32];
    __shared__ int ri[NN_CL_T / 32], rph[NN_CL_T / 32];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int crank = (int)cl.block_rank();
    const int64_t cid = blockIdx.x / NN_CL, ncl = gridDim.x / NN_CL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = NN_CL_T / 32;
    int32_t *chain = reinterpret_cast<int32_t *>(ncl_smem);
    int32_t *slot = chain + NN_SMEM_MAX;
    uint8_t *act = reinterpret_cast<uint8_t *>(slot + NN_SMEM_MAX);
    for (int64_t b = cid; b < count; b += ncl) {
        const int m = (int)sizes[b];
        if (m < cl_min || m > NN_SMEM_MAX) continue;
        double *W = mats + mat_off[b];
        int64_t *L = lefts + merge_off[b], *R = rights + merge_off[b];
        double *Hh = heights + merge_off[b];
        const int c0 = (int)((int64_t)crank * m / NN_CL), c1 = (int)((int64_t)(crank + 1) * m / NN_CL);
        for (int i = tid; i < m; i += NN_CL_T) {
            act[i] = 1;
            slot[i] = i;
        }
        for (int i = c0 + tid; i < c1; i += NN_CL_T) W[(int64_t)i * m + i] = INFINITY;   // linkage.py:61
        __syncthreads();
        nn_cl_barrier();
        int nchain = 0, remaining = m, nm = 0, first = 0, step = 0;
        int next_id = m;
        bool cycled = false;
        while (remaining > 1) {
            if (nchain == 0) {
                while (!act[first]) first++;   // the first active slot only moves forward
                chain[0] = first;
                nchain = 1;
            }
            const int x = chain[nchain - 1];
            const int p = nchain > 1 ? chain[nchain - 2] : -1;
            const double *row = W + (int64_t)x * m;
            double bv = INFINITY, rp = INFINITY;
            int bi = INT_MAX, hp = 0;
            for (int j0 = c0 + tid; j0 < c1; j0 += NN_CL_U * NN_CL_T) {
                double rr[NN_CL_U];
#pragma unroll
                for (int u = 0; u < NN_CL_U; u++) {   // the slice's loads all in flight before any use
                    const int j = j0 + u * NN_CL_T;
                    rr[u] = j < c1 ? __ldcg(row + j) : INFINITY;
                }
#pragma unroll
                for (int u = 0; u < NN_CL_U; u++) {
                    const int j = j0 + u * NN_CL_T;
                    if (j < c1) {
                        const double r = (act[j] && j != x) ? rr[u] : INFINITY;
                        if (r < bv || (r == bv && j < bi)) { bv = r; bi = j; }
                        if (j == p) { rp = r; hp = 1; }
                    }
                }
            }
            for (int o = 16; o; o >>= 1) {
                const double r2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (r2 < bv || (r2 == bv && i2 < bi)) { bv = r2; bi = i2; }
                const double p2 = __shfl_xor_sync(0xffffffffu, rp, o);
                const int h2 = __shfl_xor_sync(0xffffffffu, hp, o);
                if (h2) { rp = p2; hp = 1; }
            }
            if (lane == 0) { rv[warp] = bv; ri[warp] = bi; rpv[warp] = rp; rph[warp] = hp; }
            __syncthreads();
            const int par = step & 1;
            if (warp == 0) {
                double v = lane < NW ? rv[lane] : INFINITY;
                int i = lane < NW ? ri[lane] : INT_MAX;
                double q = lane < NW ? rpv[lane] : INFINITY;
                int h = lane < NW ? rph[lane] : 0;
                for (int o = 16; o; o >>= 1) {
                    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
                    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
                    const double q2 = __shfl_xor_sync(0xffffffffu, q, o);
                    const int h2 = __shfl_xor_sync(0xffffffffu, h, o);
                    if (h2) { q = q2; h = 1; }
                }
                if (lane < NN_CL) {   // this CTA's partial into CTA `lane`'s slot crank (DSMEM)
                    NnPart *dst = cl.map_shared_rank(&part[par][crank], (unsigned)lane);
                    dst->v = v;
                    dst->i = i;
                    dst->rp = q;
                    dst->has_p = h;
                }
            }
            nn_cl_barrier();
            // every CTA reduces the same partials in the same order: identical decisions
            double v = INFINITY, q = INFINITY;
            int i = INT_MAX;
            for (int c = 0; c < NN_CL; c++) {
                const NnPart &pp = part[par][c];
                if (pp.v < v || (pp.v == v && pp.i < i)) { v = pp.v; i = pp.i; }
                if (pp.has_p) q = pp.rp;
            }
            step++;
            int y = v == INFINITY ? 0 : i;   // np.argmin: first index of the minimum (an all-inf row: 0)
            if (p >= 0 && q == v) y = p;   // linkage.py:76-77
            if (p >= 0 && y == p) {
                nchain -= 2;
                const int lo = x < y ? x : y, hi = x < y ? y : x;
                if (crank == 0 && tid == 0) {
                    L[nm] = slot[x];
                    R[nm] = slot[y];
                    Hh[nm] = q;   // W[x, y] with y = chain[-2]
                }
                nm++;
                double *Wlo = W + (int64_t)lo * m;
                const double *Whi = W + (int64_t)hi * m;
                for (int j0 = c0 + tid; j0 < c1; j0 += NN_CL_U * NN_CL_T) {
                    double a[NN_CL_U], c[NN_CL_U];
#pragma unroll
                    for (int u = 0; u < NN_CL_U; u++) {
                        const int j = j0 + u * NN_CL_T;
                        a[u] = j < c1 ? __ldcg(Wlo + j) : 0.0;
                        c[u] = j < c1 ? __ldcg(Whi + j) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < NN_CL_U; u++) {
                        const int j = j0 + u * NN_CL_T;
                        if (j < c1) {
                            const double mg = a[u] > c[u] ? a[u] : (c[u] > a[u] ? c[u] : a[u]);
                            Wlo[j] = mg;                      // row lo, own columns
                            W[(int64_t)j * m + lo] = mg;      // column lo, own rows
                        }
                    }
                }
                __syncthreads();
                if (tid == 0) {
                    if (lo >= c0 && lo < c1) Wlo[lo] = INFINITY;
                    act[hi] = 0;
                    slot[lo] = next_id;
                }
                next_id++;
                remaining--;
                __syncthreads();
                nn_cl_barrier();   // the merged row / column are visible to every CTA
            } else {
                if (nchain >= m) { cycled = true; break; }
                __syncthreads();   // every thread has read chain[] before it grows
                if (tid == 0) chain[nchain] = y;
                nchain++;
                __syncthreads();
            }
        }
        if (cycled && crank == 0 && tid == 0) Hh[0] = __longlong_as_double(0x7ff8dead00000000ll);
        __syncthreads();
        nn_cl_barrier();   // the cluster's shared state is reused by its next matrix
    }
}

}  // namespace

// ============================================================== C ABI
TG_API size_t tg_bubble_tree_workspace_bytes(int64_t n) {
    size_t hs = 1;
    while (hs < (size_t)(4 * n + 16)) hs <<= 1;
    return tg_align_up((size_t)n * 4, 256) + tg_align_up(hs * 16, 256) + 512;
}

TG_API int tg_bubble_tree(const int32_t *clique, const int32_t *trace, int64_t n, int32_t *bubbles, int32_t *links,
                          int32_t *link_faces, int64_t *bad_row, void *ws, size_t ws_bytes, void *stream) {
    if (n < 4 || !clique || !bubbles || !bad_row) return TG_ERR_ARG;
    if (ws_bytes < tg_bubble_tree_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    size_t hs = 1;
    while (hs < (size_t)(4 * n + 16)) hs <<= 1;
    TgArena ar(ws, ws_bytes);
    int32_t *ins_t = ar.take<int32_t>(n);
    unsigned long long *htab = ar.take<unsigned long long>(2 * hs);
    unsigned long long *bad = ar.take<unsigned long long>(1);
    const int64_t nt = n - 4;
    TG_CUDA_CHECK(cudaMemsetAsync(bad, 0xff, 8, st));
    // hash table of faces: key slots 0 (empty), first-row slots +inf
    TG_CUDA_CHECK(cudaMemsetAsync(htab, 0xff, hs * 16, st));
    TG_CUDA_CHECK(cudaMemset2DAsync(htab, 16, 0, 8, hs, st));
    const unsigned T = 256;
    ins_time_kernel<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(n, ins_t); tg_count_launch(1);
    ins_time_set_kernel<<<(unsigned)((max(nt, (int64_t)4) + T - 1) / T), T, 0, st>>>(clique, trace, nt, ins_t); tg_count_launch(1);
    if (nt > 0) {
        bubble_tree_kernel<<<(unsigned)((nt + T - 1) / T), T, 0, st>>>(clique, trace, nt, n, ins_t, htab,
                                                                     (int64_t)hs - 1, bubbles, links, link_faces, bad); tg_count_launch(1);
        bubble_dup_kernel<<<(unsigned)((nt + T - 1) / T), T, 0, st>>>(trace, nt, n, htab, (int64_t)hs - 1, bad); tg_count_launch(1);
    } else {
        bubble_tree_kernel<<<1, 32, 0, st>>>(clique, trace, 0, n, ins_t, htab, (int64_t)hs - 1, bubbles, links,
                                            link_faces, bad); tg_count_launch(1);
    }
    TG_LAUNCH_CHECK();
    unsigned long long b = 0;
    TG_CUDA_CHECK(cudaMemcpyAsync(&b, bad, 8, cudaMemcpyDeviceToHost, st));
    TG_CUDA_CHECK(cudaStreamSynchronize(st));
    *bad_row = (b == ~0ull) ? -1 : (int64_t)b;
    return *bad_row >= 0 ? TG_ERR_TRACE : TG_OK;
}

TG_API int tg_orient_edges(const double *S, int64_t n, const int32_t *bubbles, const int32_t *links,
                           const int32_t *link_faces, int64_t L, int64_t *src, int64_t *dst, void *stream) {
    if (!S || L < 0) return TG_ERR_ARG;
    if (L == 0) return TG_OK;
    orient_kernel<<<(unsigned)((L + 255) / 256), 256, 0, tg_stream(stream)>>>(S, n, bubbles, links, link_faces, L, src,
                                                                             dst); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_bubble_sinks_workspace_bytes(int64_t m) {
    return tg_align_up((size_t)(m + 1) * 8, 256) * 4 + tg_align_up((size_t)(m + 1) * 8, 256) + 512;
}

TG_API int tg_bubble_sinks(const double *S, int64_t n, const int32_t *bubbles, int64_t m, const int32_t *link_faces,
                           const int64_t *src, const int64_t *dst, int64_t L, int64_t *sinks, void *ws,
                           size_t ws_bytes, void *stream) {
    if (!S || m < 1 || !sinks) return TG_ERR_ARG;
    if (ws_bytes < tg_bubble_sinks_workspace_bytes(m)) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    TgArena ar(ws, ws_bytes);
    unsigned long long *best = ar.take<unsigned long long>(m);
    int64_t *hops = ar.take<int64_t>(m);
    int64_t *tmp = ar.take<int64_t>(m);
    double *g = ar.take<double>(L + 1);
    int *changed = ar.take<int>(2);
    TG_CUDA_CHECK(cudaMemsetAsync(best, 0, m * 8, st));
    TG_CUDA_CHECK(cudaMemsetAsync(hops, 0xff, m * 8, st));   // -1: no outgoing link (a sink)
    const unsigned T = 256;
    if (L > 0) {
        hop_gain_kernel<<<(unsigned)((L + T - 1) / T), T, 0, st>>>(S, n, bubbles, link_faces, src, dst, L, g, best); tg_count_launch(1);
        // unsigned atomicMin: the unset value 0xff..ff is the largest
        hop_pick_kernel<<<(unsigned)((L + T - 1) / T), T, 0, st>>>(src, dst, L, g, best, hops); tg_count_launch(1);
    }
    sink_init_kernel<<<(unsigned)((m + T - 1) / T), T, 0, st>>>(m, hops, sinks); tg_count_launch(1);
    // pointer jumping: the hops follow the oriented tree (acyclic), so after ceil(log2 m) + 1
    // doublings every bubble points at its sink (dbht.py:161-175) -- launched back to back, no
    // host round trip per doubling
    int64_t *a = sinks, *b = tmp;
    int iters = 1;
    while (((int64_t)1 << (iters - 1)) < m) iters++;
    for (int it = 0; it < iters; it++) {
        sink_jump_kernel<<<(unsigned)((m + T - 1) / T), T, 0, st>>>(m, a, b, changed); tg_count_launch(1);
        int64_t *t = a;
        a = b;
        b = t;
    }
    if (a != sinks) TG_CUDA_CHECK(cudaMemcpyAsync(sinks, a, m * 8, cudaMemcpyDeviceToDevice, st));
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_assign_workspace_bytes(int64_t n, int64_t m) {
    return tg_align_up((size_t)4 * m * 8, 256) + tg_align_up((size_t)n * 8, 256) + 512;
}

TG_API int tg_assign_vertices(const tg_oracle_t *o, const int32_t *bubbles, int64_t m, const int64_t *sinks,
                              int64_t *vb, int64_t *vc, void *ws, size_t ws_bytes, void *stream) {
    if (!o || !bubbles || m < 1 || !vb || !vc) return TG_ERR_ARG;
    const int64_t n = o->n;
    if (ws_bytes < tg_assign_workspace_bytes(n, m)) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    TgArena ar(ws, ws_bytes);
    double *mean = ar.take<double>(4 * m);
    unsigned long long *best = ar.take<unsigned long long>(n);
    TG_CUDA_CHECK(cudaMemsetAsync(best, 0xff, n * 8, st));
    TG_CUDA_CHECK(cudaMemsetAsync(vb, 0x7f, n * 8, st));
    const unsigned T = 256;
    assign_mean_kernel<<<(unsigned)((4 * m + T - 1) / T), T, 0, st>>>(*o, bubbles, m, mean, best); tg_count_launch(1);
    assign_pick_kernel<<<(unsigned)((4 * m + T - 1) / T), T, 0, st>>>(bubbles, m, mean, best, vb); tg_count_launch(1);
    assign_conv_kernel<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(n, vb, sinks, vc); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_group_blocks(const tg_oracle_t *o, const int32_t *perm, const int64_t *starts, int64_t count,
                           const int64_t *boff, double *out, void *stream) {
    if (!o || count < 0) return TG_ERR_ARG;
    if (count == 0) return TG_OK;
    int grid = (int)min((int64_t)tg_num_sms() * 16, count);
    group_blocks_kernel<<<grid, 128, 0, tg_stream(stream)>>>(*o, perm, starts, count, boff, out); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

namespace {
__global__ void group_tiles_fill_kernel(const GmSub *__restrict__ subs, int64_t nsub, GmTile *__restrict__ tiles,
                                        int64_t ntiles) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = nsub;   // the last sub-problem with tile_off <= t
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (subs[mid].tile_off <= t) lo = mid;
            else hi = mid;
        }
        const int64_t nt = (subs[lo].len + GM_TILE - 1) / GM_TILE, q = t - subs[lo].tile_off;
        tiles[t] = GmTile{(int)lo, (int)(q / nt) * GM_TILE, (int)(q % nt) * GM_TILE};
    }
}
}  // namespace

TG_API int tg_group_tiles_fill(const void *subs_v, int64_t nsub, void *tiles_v, int64_t ntiles, void *stream) {
    if (nsub < 0 || ntiles < 0 || (ntiles > 0 && (!subs_v || !tiles_v || nsub == 0))) return TG_ERR_ARG;
    if (ntiles == 0) return TG_OK;
    const int64_t blocks = std::min<int64_t>((ntiles + 255) / 256, (int64_t)tg_num_sms() * 8);
    group_tiles_fill_kernel<<<(unsigned)blocks, 256, 0, tg_stream(stream)>>>(
        reinterpret_cast<const GmSub *>(subs_v), nsub, reinterpret_cast<GmTile *>(tiles_v), ntiles);
    tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_group_max_workspace_bytes(int64_t n, int64_t ntiles, int64_t H) {
    const size_t Hp = (size_t)((H + GM_HC - 1) / GM_HC * GM_HC);
    return tg_align_up((size_t)n * 4, 256) * 2 + tg_align_up((size_t)ntiles * GM_TILE * 8 + 8, 256) +
           tg_align_up((size_t)n * Hp * 4, 256) + tg_align_up((size_t)n * Hp * 8, 256) + 1024;
}

TG_API int tg_group_max_batch(const tg_oracle_t *o, const int32_t *perm, const int32_t *gid, int64_t total_len,
                              const void *subs_v, int64_t nsub, const void *tiles_v, int64_t ntiles, double *out,
                              int64_t out_len, void *ws, size_t ws_bytes, void *stream) {
    if (!o || !perm || !gid || !subs_v || !tiles_v || !out || nsub < 0 || ntiles < 0 || total_len < 0) return TG_ERR_ARG;
    const int64_t n = o->n;
    if (ws_bytes < tg_group_max_workspace_bytes(n, ntiles, o->mode == 1 ? o->H : 0)) return TG_ERR_WORKSPACE;
    const GmSub *subs = reinterpret_cast<const GmSub *>(subs_v);
    const GmTile *tiles = reinterpret_cast<const GmTile *>(tiles_v);
    cudaStream_t st = tg_stream(stream);
    TgArena ar(ws, ws_bytes);
    int32_t *pos = ar.take<int32_t>(n);
    int32_t *vsub = ar.take<int32_t>(n);
    uint64_t *mask = ar.take<uint64_t>((size_t)ntiles * GM_TILE + 1);
    TG_CUDA_CHECK(cudaMemsetAsync(out, 0, (size_t)out_len * 8, st));
    if (nsub == 0) return TG_OK;
    TG_CUDA_CHECK(cudaMemsetAsync(pos, 0xff, (size_t)n * 4, st));
    TG_CUDA_CHECK(cudaMemsetAsync(vsub, 0xff, (size_t)n * 4, st));
    pos_fill_kernel<<<(unsigned)min(nsub, (int64_t)65535), 256, 0, st>>>(subs, nsub, perm, pos, vsub); tg_count_launch(1);
    if (o->mode == 1 && ntiles > 0) {
        TG_CUDA_CHECK(cudaMemsetAsync(mask, 0, (size_t)ntiles * GM_TILE * 8, st));
        const int64_t blocks = min((total_len * 32 + 255) / 256, (int64_t)tg_num_sms() * 16);
        for (int pass = 0; pass < 2; pass++) {
            group_max_override_kernel<<<(unsigned)blocks, 256, 0, st>>>(*o, perm, gid, pos, vsub, subs, nsub, total_len,
                                                                        pass, mask,
                                                                        reinterpret_cast<unsigned long long *>(out));
            tg_count_launch(1);
        }
    }
    if (ntiles > 0) {
        int grid = (int)min((int64_t)tg_num_sms() * 8, ntiles);
        if (o->mode == 1) {
            const int Hp = (int)((o->H + GM_HC - 1) / GM_HC * GM_HC);
            float *hpf = ar.take<float>((size_t)total_len * Hp);
            double *hpd = ar.take<double>((size_t)total_len * Hp);
            if (!hpf || !hpd) return TG_ERR_WORKSPACE;
            const int64_t cnt = total_len * Hp;
            hp_fill_kernel<<<(unsigned)min((cnt + 255) / 256, (int64_t)tg_num_sms() * 16), 256, 0, st>>>(
                *o, perm, total_len, Hp, hpf, hpd);
            tg_count_launch(1);
            group_max_hub_kernel<<<grid, GH_T, 0, st>>>(*o, gid, subs, tiles, ntiles, Hp, hpf, hpd,
                                                      reinterpret_cast<unsigned long long *>(out), mask);
        } else
            group_max_tile_kernel<<<grid, GM_T, 0, st>>>(*o, perm, gid, pos, subs, tiles, ntiles,
                                                       reinterpret_cast<unsigned long long *>(out), mask);
        tg_count_launch(1);
    }
    if (o->mode == 0) {   // hub mode evaluates every ordered pair: nothing to mirror
        group_max_finalize_kernel<<<(unsigned)tg_num_sms() * 8, 256, 0, st>>>(subs, nsub, out); tg_count_launch(1);
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_nn_chain_batch(double *mats, const int64_t *mat_off, const int64_t *sizes, int64_t count,
                             const int64_t *merge_off, int64_t *lefts, int64_t *rights, double *heights,
                             const int64_t *aux_off, uint8_t *active, int64_t *slot, int64_t *chain, void *stream) {
    if (count < 0 || !mats) return TG_ERR_ARG;
    if (count == 0) return TG_OK;
    int64_t warps = count;
    int threads = 128;
    int64_t blocks = (warps * 32 + threads - 1) / threads;
    if (blocks > (int64_t)tg_num_sms() * 32) blocks = (int64_t)tg_num_sms() * 32;
    cudaStream_t st = tg_stream(stream);
    int64_t cblocks = count < (int64_t)tg_num_sms() * 2 ? count : (int64_t)tg_num_sms() * 2;
    const size_t nn_smem = (size_t)NN_SMEM_MAX * 9;
    // m <= NN_BIG: 512 threads (two CTAs per SM); larger: 1024 threads, one row read in flight
    TG_CUDA_CHECK(cudaFuncSetAttribute(nn_chain_cta_kernel<NN_SMALL_T, NN_SMALL_U, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nn_smem));
    TG_CUDA_CHECK(cudaFuncSetAttribute(nn_chain_cta_kernel<1024, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)nn_smem));
    // matrices with cl_min <= m <= NN_SMEM_MAX take the cluster chain (TG_NN_CLMIN: development knob, 0 = off)
    static const int cl_min = std::getenv("TG_NN_CLMIN") ? std::atoi(std::getenv("TG_NN_CLMIN")) : NN_CL_MIN;
    const int cl_on = cl_min > 0;
    // the cluster chains (the large matrices) run on a side stream, beside the per-CTA chains
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (cl_on) {
        TG_CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        TG_CUDA_CHECK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
        TG_CUDA_CHECK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
        TG_CUDA_CHECK(cudaEventRecord(fork, st));
        TG_CUDA_CHECK(cudaStreamWaitEvent(side, fork, 0));
    }
    nn_chain_cta_kernel<NN_SMALL_T, NN_SMALL_U, false><<<(unsigned)cblocks, NN_SMALL_T, nn_smem, st>>>(mats, mat_off, sizes, count, merge_off, lefts,
                                                                        rights, heights, active, slot, chain, aux_off,
                                                                        cl_min);
    nn_chain_cta_kernel<1024, 8, true><<<(unsigned)cblocks, 1024, nn_smem, st>>>(mats, mat_off, sizes, count, merge_off,
                                                                          lefts, rights, heights, active, slot, chain,
                                                                          aux_off, cl_min);
    tg_count_launch(2);
    // the warp-per-matrix chains (m <= NN_WARP_MAX) last: the large matrices' chains are the
    // batch's critical path and should not queue behind them
    nn_chain_kernel<<<(unsigned)blocks, threads, 0, st>>>(mats, mat_off, sizes, count, merge_off, lefts, rights, heights,
                                                        active, slot, chain, aux_off); tg_count_launch(1);
    if (cl_on) {
        const int64_t ncl = count < (int64_t)tg_num_sms() / NN_CL ? count : (int64_t)tg_num_sms() / NN_CL;
        TG_CUDA_CHECK(cudaFuncSetAttribute(nn_chain_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)nn_smem));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = NN_CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)(ncl * NN_CL), 1, 1);
        cfg.blockDim = dim3(NN_CL_T, 1, 1);
        cfg.dynamicSmemBytes = nn_smem;
        cfg.stream = side;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        TG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, nn_chain_cluster_kernel, mats, mat_off, sizes, count, merge_off, lefts,
                                         rights, heights, cl_min));
        tg_count_launch(1);
        TG_CUDA_CHECK(cudaEventRecord(join, side));
        TG_CUDA_CHECK(cudaStreamWaitEvent(st, join, 0));
        cudaEventDestroy(fork);
        cudaEventDestroy(join);
        cudaStreamDestroy(side);   // released once its work completes
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

// public block / query accessors (apsp.py:88-94, 127-158)
TG_API int tg_oracle_block(const tg_oracle_t *o, const int32_t *rows, int64_t nr, const int32_t *cols, int64_t nc,
                           int32_t query_semantics, double *out, void *stream) {
    if (!o || nr < 0 || nc < 0 || !out) return TG_ERR_ARG;
    if (nr * nc == 0) return TG_OK;
    oracle_block_kernel<<<(unsigned)((nr * nc + 255) / 256), 256, 0, tg_stream(stream)>>>(*o, rows, nr, cols, nc,
                                                                                          query_semantics, out); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
