// tmfg_variants.cu -- the exact and corr TMFG builders (tmfg.py:185-341) on the B200.
//
// Replaces build_tmfg_exact (tmfg.py:208-263: every live face keeps its true best
// uninserted vertex, an argmax over all remaining vertices) and build_tmfg_corr
// (tmfg.py:280-341: each face considers only its three vertices' best uninserted
// neighbours, refreshed eagerly), both with the prefix rule of _select_round
// (tmfg.py:185-205: top prefix_size face-vertex pairs by (gain desc, face id asc),
// vertex conflicts resolved by keeping the first).  Face / edge / trace bookkeeping
// is _GraphAccum's (tmfg.py:94-144).
//
// One persistent 1024-thread CTA runs the rounds; the face table, gains and
// scan state live in global memory (L2-resident: ~40 n bytes).  Per round:
//   select     block argmax over the live faces (prefix > 1: repeated argmax with the
//              chosen faces and the already-taken vertices excluded, which visits the
//              faces in exactly _select_round's ranked order);
//   insert     thread 0 appends trace / edges / faces in pair order;
//   stale      faces whose cached vertex was just inserted, plus the new faces;
//   exact:     rescan each listed face: g(u) = (S[a,u] + S[b,u]) + S[c,u] over the
//              uninserted u, first max (u ascending) -- eight faces per pass, each
//              thread keeping eight (g, u) bests over its strided u range;
//   corr:      refresh the cursors of the listed faces' vertices (one warp per
//              vertex, 32 ids per step) and recompute each listed face's best of
//              its three candidates (tmfg.py:266-277 tie rule).
// Results are independent of the launch configuration: every reduction is an exact
// (gain desc, id asc) argmax and every update set is processed as a set.
#include "common.cuh"

#include <cmath>

namespace {

constexpr int VT = 1024;
constexpr int VW = VT / 32;
constexpr int KCH = 8;   // exact: faces rescanned per pass

struct VarWs {
    int32_t *fv;       // 3n x 3 face vertices (sorted)
    uint8_t *alive;    // 3n
    double *fgain;     // 3n
    int32_t *fvert;    // 3n (-1: never computed)
    int32_t *fpick;    // 3n: round in which the face was picked (prefix selection)
    uint8_t *ins;      // n
    int32_t *stamp;    // n: round in which the vertex was picked
    int32_t *vstamp;   // n: round in which the vertex's cursor was claimed for a refresh (corr)
    int32_t *cur;      // n cursors (corr)
    int32_t *mc;       // n max_corrs (corr)
    int32_t *list;     // 3n faces to update this round
    int32_t *vlist;    // n vertices to refresh this round (corr)
    int32_t *pairs;    // 2 n (fid, v) picked this round
};

// (g desc, id asc); id < 0 is "none"
__device__ __forceinline__ bool vb_better(double g1, int i1, double g2, int i2) {
    if (i1 < 0) return false;
    if (i2 < 0) return true;
    return g1 > g2 || (g1 == g2 && i1 < i2);
}

__device__ __forceinline__ void vb_warp(double &g, int &i) {
    for (int o = 16; o; o >>= 1) {
        const double g2 = __shfl_xor_sync(0xffffffffu, g, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        if (vb_better(g2, i2, g, i)) { g = g2; i = i2; }
    }
}

// block-wide best of (g, i); every thread gets the result
__device__ __forceinline__ void vb_block(double &g, int &i, double *sg, int *si) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    vb_warp(g, i);
    if (lane == 0) { sg[warp] = g; si[warp] = i; }
    __syncthreads();
    if (warp == 0) {
        g = sg[lane];
        i = si[lane];
        vb_warp(g, i);
        if (lane == 0) { sg[32] = g; si[32] = i; }
    }
    __syncthreads();
    g = sg[32];
    i = si[32];
    __syncthreads();
}

// tmfg.py:266-277 _best_candidate: candidates (mc[a], mc[b], mc[c]) in that order,
// g = S[a,u] + S[b,u] + S[c,u]; g > best or (g == best and u < best_v)
__device__ __forceinline__ void vb_best_candidate(const double *S, int64_t n, const int32_t *mc, int a, int b, int c,
                                                  double &bg, int &bv) {
    bg = -INFINITY;
    bv = -1;
    const int cand[3] = {mc[a], mc[b], mc[c]};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        const int u = cand[k];
        const double g = __dadd_rn(__dadd_rn(S[(int64_t)a * n + u], S[(int64_t)b * n + u]), S[(int64_t)c * n + u]);
        if (g > bg || (g == bg && u < bv)) { bg = g; bv = u; }
    }
}

// tmfg.py:169-182 refresh_max_corr by one warp: first uninserted id at or after the cursor
__device__ __forceinline__ void vb_refresh_warp(const int32_t *order, int64_t n, const uint8_t *ins, int32_t *cur,
                                                int32_t *mc, int w) {
    const int lane = threadIdx.x & 31;
    const int32_t *row = order + (int64_t)w * (n - 1);
    int c = cur[w];
    for (;;) {
        const int q = c + lane;
        const bool free = q < n - 1 && !ins[row[q]];
        const unsigned bal = __ballot_sync(0xffffffffu, free);
        if (bal) {
            c += __ffs(bal) - 1;
            break;
        }
        c += 32;
    }
    if (lane == 0) {
        cur[w] = c;
        mc[w] = row[c];
    }
}

template <int V>   // 0: exact, 1: corr
__global__ void __launch_bounds__(VT, 1)
tmfg_variant_kernel(const double *__restrict__ S, const int32_t *__restrict__ order, int64_t n64,
                    const int32_t *__restrict__ clique, int prefix, int32_t *__restrict__ trace,
                    int32_t *__restrict__ edges, int32_t *__restrict__ faces_out, VarWs w) {
    __shared__ double sg[33];
    __shared__ int si[33];
    __shared__ double kg[KCH][32];
    __shared__ int ki[KCH][32];
    __shared__ int s_nf, s_nlist, s_nv, s_npairs, s_cnt;
    const int n = (int)n64;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int F = 3 * n;
    for (int i = tid; i < n; i += VT) {
        w.ins[i] = 0;
        w.stamp[i] = -1;
        w.vstamp[i] = -1;
        w.cur[i] = 0;
        w.mc[i] = -1;
    }
    for (int f = tid; f < F; f += VT) {
        w.alive[f] = 0;
        w.fvert[f] = -1;
        w.fgain[f] = -INFINITY;
        w.fpick[f] = -1;
    }
    __syncthreads();
    const int a0 = clique[0], b0 = clique[1], c0 = clique[2], d0 = clique[3];
    if (tid == 0) {
        w.ins[a0] = w.ins[b0] = w.ins[c0] = w.ins[d0] = 1;
        const int t4[4][3] = {{a0, b0, c0}, {a0, b0, d0}, {a0, c0, d0}, {b0, c0, d0}};
        for (int f = 0; f < 4; f++) {
            for (int k = 0; k < 3; k++) w.fv[3 * f + k] = t4[f][k];
            w.alive[f] = 1;
        }
        const int e6[6][2] = {{a0, b0}, {a0, c0}, {a0, d0}, {b0, c0}, {b0, d0}, {c0, d0}};
        for (int e = 0; e < 6; e++) { edges[2 * e] = e6[e][0]; edges[2 * e + 1] = e6[e][1]; }
        s_nf = 4;
        s_nlist = 4;
        for (int f = 0; f < 4; f++) w.list[f] = f;
    }
    __syncthreads();
    int rem = n - 4, ntrace = 0, nedge = 6;
    int round = 0;
    while (rem > 0) {
        // ---- update the listed faces (round 0: the four clique faces)
        const int nlist = s_nlist;
        if (V == 0) {
            for (int k0 = 0; k0 < nlist; k0 += KCH) {
                const int kn = min(KCH, nlist - k0);
                int fa[KCH], fb[KCH], fc[KCH];
                double bg[KCH];
                int bu[KCH];
#pragma unroll
                for (int k = 0; k < KCH; k++) {
                    const int f = k < kn ? w.list[k0 + k] : w.list[k0];
                    fa[k] = w.fv[3 * f];
                    fb[k] = w.fv[3 * f + 1];
                    fc[k] = w.fv[3 * f + 2];
                    bg[k] = -INFINITY;
                    bu[k] = -1;
                }
                for (int u = tid; u < n; u += VT) {
                    if (w.ins[u]) continue;
#pragma unroll
                    for (int k = 0; k < KCH; k++) {
                        if (k >= kn) break;
                        const double g = __dadd_rn(__dadd_rn(S[(int64_t)fa[k] * n64 + u], S[(int64_t)fb[k] * n64 + u]),
                                                   S[(int64_t)fc[k] * n64 + u]);
                        if (bu[k] < 0 || g > bg[k]) { bg[k] = g; bu[k] = u; }   // u ascending per thread
                    }
                }
#pragma unroll
                for (int k = 0; k < KCH; k++) {
                    vb_warp(bg[k], bu[k]);
                    if (lane == 0) { kg[k][warp] = bg[k]; ki[k][warp] = bu[k]; }
                }
                __syncthreads();
                if (warp < kn) {
                    double g = kg[warp][lane];
                    int u = ki[warp][lane];
                    vb_warp(g, u);
                    if (lane == 0) {
                        const int f = w.list[k0 + warp];
                        w.fgain[f] = g;
                        w.fvert[f] = u;
                    }
                }
                __syncthreads();
            }
        } else {
            // verts_update: the listed faces' vertices, each refreshed once (tmfg.py:327-330)
            if (tid == 0) s_nv = 0;
            __syncthreads();
            for (int k = tid; k < 3 * nlist; k += VT) {
                const int v = w.fv[3 * w.list[k / 3] + k % 3];
                if (atomicExch(&w.vstamp[v], round) != round) w.vlist[atomicAdd(&s_nv, 1)] = v;
            }
            __syncthreads();
            const int nv = s_nv;
            for (int q = warp; q < nv; q += VW) vb_refresh_warp(order, n64, w.ins, w.cur, w.mc, w.vlist[q]);
            __syncthreads();
            for (int k = tid; k < nlist; k += VT) {
                const int f = w.list[k];
                double g;
                int u;
                vb_best_candidate(S, n64, w.mc, w.fv[3 * f], w.fv[3 * f + 1], w.fv[3 * f + 2], g, u);
                w.fgain[f] = g;
                w.fvert[f] = u;
            }
            __syncthreads();
        }
        // ---- select (tmfg.py:185-205)
        const int nf = s_nf;
        const int want = prefix < rem ? prefix : rem;
        if (tid == 0) s_npairs = 0;
        __syncthreads();
        for (int t = 0; t < want; t++) {
            double g = -INFINITY;
            int id = -1;
            for (int f = tid; f < nf; f += VT) {
                if (!w.alive[f]) continue;
                if (prefix > 1) {
                    if (w.fpick[f] == round) continue;
                    const int v = w.fvert[f];
                    if (w.stamp[v] == round) continue;   // its vertex is already taken this round
                }
                const double gf = w.fgain[f];
                if (vb_better(gf, f, g, id)) { g = gf; id = f; }
            }
            vb_block(g, id, sg, si);
            if (id < 0) break;   // every remaining live face's vertex is taken
            if (tid == 0) {
                const int v = w.fvert[id];
                w.pairs[2 * t] = id;
                w.pairs[2 * t + 1] = v;
                w.fpick[id] = round;
                w.stamp[v] = round;
                s_npairs = t + 1;
            }
            __syncthreads();
        }
        // ---- insert in pair order (tmfg.py:120-131)
        const int np = s_npairs;
        if (tid == 0) {
            int nf2 = nf;
            for (int t = 0; t < np; t++) {
                const int fid = w.pairs[2 * t], v = w.pairs[2 * t + 1];
                const int a = w.fv[3 * fid], b = w.fv[3 * fid + 1], c = w.fv[3 * fid + 2];
                int32_t *tr = trace + 4 * (int64_t)ntrace;
                tr[0] = v; tr[1] = a; tr[2] = b; tr[3] = c;
                ntrace++;
                const int fw[3] = {a, b, c};
                for (int k = 0; k < 3; k++) {
                    const int x = fw[k];
                    edges[2 * (int64_t)nedge] = x < v ? x : v;
                    edges[2 * (int64_t)nedge + 1] = x < v ? v : x;
                    nedge++;
                }
                w.alive[fid] = 0;
                w.ins[v] = 1;
                const int ch[3][3] = {{v, a, b}, {v, a, c}, {v, b, c}};
                for (int k = 0; k < 3; k++) {
                    int x = ch[k][0], y = ch[k][1], z = ch[k][2];   // sort the triple
                    if (x > y) { int s = x; x = y; y = s; }
                    if (y > z) { int s = y; y = z; z = s; }
                    if (x > y) { int s = x; x = y; y = s; }
                    w.fv[3 * nf2] = x; w.fv[3 * nf2 + 1] = y; w.fv[3 * nf2 + 2] = z;
                    w.alive[nf2] = 1;
                    w.fvert[nf2] = -1;
                    nf2++;
                }
            }
            s_nf = nf2;
            s_nlist = 0;
        } else {
            // the other threads keep the counters in step with thread 0
            ntrace += np;
            nedge += 3 * np;
        }
        rem -= np;
        __syncthreads();
        if (rem == 0) break;
        // ---- faces to update: live faces whose vertex was taken this round, then the new faces
        const int nf2 = s_nf;
        for (int f = tid; f < nf; f += VT) {
            if (!w.alive[f]) continue;
            const int v = w.fvert[f];
            if (v >= 0 && w.stamp[v] == round) w.list[atomicAdd(&s_nlist, 1)] = f;
        }
        __syncthreads();
        if (tid == 0) {
            int k = s_nlist;
            for (int f = nf; f < nf2; f++) w.list[k++] = f;
            s_nlist = k;
        }
        __syncthreads();
        round++;
    }
    // ---- faces alive at the end, in creation order (tmfg.py:133-144)
    const int nf = s_nf;
    if (tid == 0) s_cnt = 0;
    __syncthreads();
    for (int f0 = 0; f0 < nf; f0 += VT) {
        const int f = f0 + tid;
        const bool ok = f < nf && w.alive[f];
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) ki[0][warp] = __popc(bal);
        __syncthreads();
        int before = s_cnt;
        for (int q = 0; q < warp; q++) before += ki[0][q];
        if (ok) {
            const int o = before + __popc(bal & ((1u << lane) - 1u));
            faces_out[3 * o] = w.fv[3 * f];
            faces_out[3 * o + 1] = w.fv[3 * f + 1];
            faces_out[3 * o + 2] = w.fv[3 * f + 2];
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int q = 0; q < VW; q++) tot += ki[0][q];
            s_cnt += tot;
        }
        __syncthreads();
    }
}

VarWs carve(void *ws, int64_t n) {
    TgArena ar(ws, (size_t)-1);
    VarWs w;
    const size_t F = 3 * (size_t)n;
    w.fv = ar.take<int32_t>(3 * F);
    w.alive = ar.take<uint8_t>(F);
    w.fgain = ar.take<double>(F);
    w.fvert = ar.take<int32_t>(F);
    w.fpick = ar.take<int32_t>(F);
    w.ins = ar.take<uint8_t>(n);
    w.stamp = ar.take<int32_t>(n);
    w.vstamp = ar.take<int32_t>(n);
    w.cur = ar.take<int32_t>(n);
    w.mc = ar.take<int32_t>(n);
    w.list = ar.take<int32_t>(F);
    w.vlist = ar.take<int32_t>(n);
    w.pairs = ar.take<int32_t>(2 * (size_t)n);
    return w;
}

size_t carve_bytes(int64_t n) {
    const size_t F = 3 * (size_t)n;
    const size_t parts[] = {3 * F * 4, F, F * 8, F * 4, F * 4, (size_t)n, (size_t)n * 4, (size_t)n * 4,
                            (size_t)n * 4, (size_t)n * 4, F * 4, (size_t)n * 4, 2 * (size_t)n * 4};
    size_t s = 0;
    for (size_t p : parts) s += tg_align_up(p, 256) + 256;
    return s;
}

template <int V>
int launch(const double *S, const int32_t *order, int64_t n, const int32_t *clique, int64_t prefix, int32_t *trace,
           int32_t *edges, int32_t *faces, void *ws, size_t ws_bytes, void *stream) {
    if (!S || !clique || (n > 4 && !trace) || !edges || !faces || n < 4 || prefix < 1) return TG_ERR_ARG;
    if (V == 1 && !order) return TG_ERR_ARG;
    if (n > (int64_t)INT_MAX / 3) return TG_ERR_ARG;
    if (!ws || ws_bytes < carve_bytes(n)) return TG_ERR_WORKSPACE;
    const int p = prefix > n ? (int)n : (int)prefix;
    tmfg_variant_kernel<V><<<1, VT, 0, tg_stream(stream)>>>(S, order, n, clique, p, trace, edges, faces, carve(ws, n));
    tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

}  // namespace

TG_API size_t tg_tmfg_variant_workspace_bytes(int64_t n) { return n < 4 ? 256 : carve_bytes(n); }

TG_API int tg_tmfg_exact(const double *S, int64_t n, const int32_t *clique, int64_t prefix_size, int32_t *trace_out,
                         int32_t *edges_out, int32_t *faces_out, void *ws, size_t ws_bytes, void *stream) {
    return launch<0>(S, nullptr, n, clique, prefix_size, trace_out, edges_out, faces_out, ws, ws_bytes, stream);
}

TG_API int tg_tmfg_corr(const double *S, const int32_t *order, int64_t n, const int32_t *clique, int64_t prefix_size,
                        int32_t *trace_out, int32_t *edges_out, int32_t *faces_out, void *ws, size_t ws_bytes,
                        void *stream) {
    return launch<1>(S, order, n, clique, prefix_size, trace_out, edges_out, faces_out, ws, ws_bytes, stream);
}
