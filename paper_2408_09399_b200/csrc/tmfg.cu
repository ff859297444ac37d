// tmfg.cu -- the lazy-gain (heap) TMFG insertion loop as one persistent thread-block cluster
// (the leader CTA runs the rounds below; helper CTAs keep the per-vertex scan state two
// candidates deep and one prefetches the S values of the queue head into L2).
//
// Replaces tmfg.py:344-436 build_tmfg_heap with its helpers tmfg.py:94-144
// (_GraphAccum), 147-182 (TmfgState, refresh_max_corr), 266-277
// (_best_candidate).  Output is bit-identical: the same trace, edges, faces and
// debug counters as heapq over (-gain, fid, cand).
//
// Why the result is exact although work is speculative:
//   * every heap entry is (g, fid, cand) with fid unique among live entries, so
//     the pop sequence depends only on the SET of keys (g desc, fid asc): any
//     priority structure with that order pops the same sequence;
//   * refresh_max_corr(w) = first uninserted id of order[w] (cursors only skip
//     inserted ids), a pure function of the inserted set I.  Hence the
//     refreshed entry of a face, entry(face, I), is pure too: between two
//     insertions I is fixed and all stale entries near the top of the heap can
//     be refreshed IN PARALLEL, then the sequential pop/re-push sequence is
//     replayed exactly by a short scan (a stale pop pushes a fresh entry; the
//     first fresh thing on top wins).
//
// One round = [parallel] refresh the stale entries among the top K = 56 of the queue (two
// per window warp on the lean path, window_refresh2; a scan only when a vertex's scan-state
// word certifies no uninserted candidate) and build the entries
// of the 3 faces created by the last insertion (cursor scans: one 128-byte
// warp load of order[w] + a ballot against the inserted bitmap in shared
// memory; gains: 9 fp64 loads of S, summed (S[a,u]+S[b,u])+S[c,u] with
// __dadd_rn) -> [one warp] replay the pops, chunk of 28 window positions by chunk -> [block]
// update the queue and insert the winner.  About two dependent global-load latencies per
// insertion.
//
// Priority queue: the top B entries live sorted in shared memory (double
// buffered, merge-path insertion); the rest sit unsorted in a global pool whose
// keys are all below the buffer's; the buffer is refilled by a radix select
// over the pool when it runs short.
#include "common.cuh"
#include <cooperative_groups.h>
#include <cstdlib>

namespace {

// TM_PROFILE=1 (make PROFILE=1): per-warp phase clocks of the parallel phase
// (tools/tmfg_profile.py); the round-level phase clocks are always on.
#ifndef TM_PROFILE
#define TM_PROFILE 0
#endif

constexpr int TM_T = 1024;
constexpr int TM_WARPS = TM_T / 32;
#ifndef TM_BG_WARPS_DEF
#define TM_BG_WARPS_DEF 0   // the cluster helpers keep the scan state; all 32 warps serve the rounds
#endif
constexpr int TM_BG_WARPS = TM_BG_WARPS_DEF;      // background cursor-advancing warps
constexpr int TM_FG_WARPS = TM_WARPS - TM_BG_WARPS;
constexpr int TM_FG_T = TM_FG_WARPS * 32;
constexpr int TM_EPW = 1;                       // entries refreshed per warp
constexpr int TM_NEW_WARPS = 4;                 // warps that build new-face entries
constexpr int TM_CH = TM_FG_WARPS - TM_NEW_WARPS;  // window entries per replay chunk (one per window warp)
#ifndef TM_WPE_DEF
#define TM_WPE_DEF 2
#endif
constexpr int TM_WPE = TM_WPE_DEF;               // window entries per warp (one per half-warp): replay chunks per round
constexpr int TM_K = TM_WPE * TM_CH;             // top-K speculated per round
// After a round without a winner (every window entry popped stale: the lazy heap's stale streaks,
// 60-800 pops per insertion at the end of config 5) the next window is TM_PASSES times as wide:
// each window warp makes TM_PASSES passes of its two entries (nearly all refresh-cache hits then).
// Only with the scan state in global memory (large n): at n = 10k the wider arrays cost more
// than the 5 % of rounds they save (66.2 -> 67.6 ms), at n = 50k they pay (430 -> 418 ms).
#ifndef TM_PASSES_DEF
#define TM_PASSES_DEF 2
#endif
constexpr int TM_PASSES = TM_PASSES_DEF;
template <bool SMEM_ST>
__host__ __device__ constexpr int tm_kmax() { return SMEM_ST ? TM_K : TM_PASSES * TM_K; }
#ifndef TM_MERGE_WARPS_DEF
#define TM_MERGE_WARPS_DEF 28   // (the kernel picks per instantiation: see tm_merge_warps)
#endif
constexpr int TM_MERGE_WARPS = TM_MERGE_WARPS_DEF;            // replay + merge warps; the rest speculate meanwhile
// Scan state in shared memory (n <~ 17k): every foreground warp replays / merges (the merge
// then has ~one entry per thread).  Scan state in global memory (large n, 2048-entry queue):
// 4 warps speculate -- refresh the entries just past the window into the refresh cache --
// while the others replay and merge (measured: n = 10k 96 -> 89 ms; n = 50k 644 vs 592 ms).
template <bool SMEM_ST>
__host__ __device__ constexpr int tm_merge_warps() { return SMEM_ST ? TM_FG_WARPS : TM_MERGE_WARPS; }
#ifndef TM_B_DEF
// measured after the refill's counting-sort ranking and 3/4 take (refills got ~2x cheaper, so a shorter queue -- a
// shorter merge -- pays): 512 (1/2 take) / 608 / 640 / 704 / 768 / 896 / 1024 -> 75.4 / 69.4 / 69.3 / 69.3 / 69.4 /
// 70.1 / 71.8 ms at n = 10k, 503 / 511 / 449-452 / 455 / 455 / 463 / 469 ms at n = 50k (queue 2x these there);
// before: 640 / 768 / 896 / 1024 -> 87.6 / 86-88 / 86.2 / 87.6 ms at n = 10k
#define TM_B_DEF 640
#endif
constexpr int TM_B = TM_B_DEF;                  // shared-memory queue capacity (scan state in smem)
constexpr int TM_BMAX = 2 * TM_B;               // ... when the scan state lives in global memory (large n):
// the queue can then take the room, and a longer queue means fewer O(pool) refills
template <bool SMEM_ST>
__host__ __device__ constexpr int tm_qb() { return SMEM_ST ? TM_B : TM_BMAX; }
constexpr int TM_BATCH = TM_K + 8;   // (largest re-queued run of a narrow round; kernels size theirs from tm_kmax)
static_assert(TM_CH <= 32, "replay_warp maps one queue position of a chunk per lane");
static_assert(TM_WPE == 1 || TM_WPE == 2, "window_refresh2 serves one entry per half-warp");

struct Ent {
    double g;
    int fid;
    int cand;
    int a, b, c;
    int opt;     // check mode: g >= max over uninserted u of the face gain - 1e-12
};

__device__ __forceinline__ bool ent_gt(const Ent &x, const Ent &y) {
    // x pops before y: heapq order of (-g, fid)
    return (x.g > y.g) | ((x.g == y.g) & (x.fid < y.fid));
}

// refresh cache slot (direct-mapped by face id)
struct RcEnt {
    double g;
    int fid, cand;
    int m[3];
    int pad;
};
constexpr int TM_RC = 1024;

struct Ctl {
    int size;        // entries in the shared buffer
    int sel;         // which half of the double buffer is current
    int rem;         // uninserted vertices
    int nt;          // trace rows written
    int nf;          // faces created
    int ne_count;    // fresh entries built last round (not yet queued)
    int ne_fid[4];
    int ne_v[4][3];
    int L_count;
    int removed;     // buffer head entries consumed by the scan
    int nbatch;
    int nbuf_new;    // batch entries headed for the buffer
    int exhausted;
    int winner;      // 0 none, 1 yes
    Ent win;
    long long pops, refreshes, gain_inc;
    int pool_count;
    unsigned long long pool_minkey;   // <= the smallest pool key (order key of the gain)
    int pool_has_max;
    Ent pool_max;
    int refill_take;
    int need_refill;
    int nsurv;
    int stop;
    unsigned long long sel_prefix;
    int sel_room;
    int hist[256];
    int done;
    int bad;
    int bg_stop;
    long long t_par, t_replay, t_merge, t_insert, t_refill, t_tail, rounds, refills;
    int it_round_max;
    int ph[4];
    long long phs[4];
    long long pops_dbg;
    long long rf_t[4];   // refill phases: select, take, place, hole fill (TM_PROFILE)
    unsigned rc_hit;     // refresh-cache hits (TM_PROFILE)
    long long it_total, it_maxsum;
    int wide;        // the last round had no winner: this round's window is TM_PASSES times as wide
};

struct TmArgs {
    const double *S;
    const int32_t *order;
    int n;
    const int32_t *clique;
    int32_t *trace;
    int32_t *host_fid;
    int32_t *edges;
    int32_t *faces;
    int64_t *stats;
    int4 *fv;            // face vertices (a, b, c) + alive flag, 3n entries
    double *pool_g;      // global pool (struct of arrays): gain
    int2 *pool_fc;       //   (fid, cand); capacity 3n + B

    unsigned long long *gvst;  // per-vertex scan state when it does not fit in shared memory
    int check;           // check_invariants mode (tmfg.py:375-399)
    int prefetch;        // the last helper CTA prefetches S for the queue head into L2
};

__device__ __forceinline__ bool is_ins(const uint32_t *bits, int v) { return (bits[v >> 5] >> (v & 31)) & 1u; }

// named barrier 1 over the foreground warps only (background warps never wait on it)
__device__ __forceinline__ void fg_sync() { asm volatile("bar.sync 1, %0;" ::"r"(TM_FG_T) : "memory"); }
// same barrier with a reduction result: the clock read after it really follows the release
__device__ __forceinline__ long long fg_sync_clock() {
    unsigned r;
    asm volatile("bar.red.popc.u32 %0, 1, %1, 1;" : "=r"(r) : "r"(TM_FG_T) : "memory");
    return clock64() + (long long)(r & 0u);
}

// Per-vertex scan state, one 64-bit word (tmfg.py:169-182 cursors + max_corrs):
//   bits  0-20  mc + 1   the first uninserted id of order[w] when computed (0: unknown)
//   bits 21-41  mc2 + 1  the next uninserted id after it (0: unknown)
//   bits 42-63  cursor   where a scan restarts: the position of mc2 (of mc if mc2 is unknown)
// "every id before pos(mc) is inserted" and "every id between mc and mc2 is
// inserted" are monotone facts, so a word stays a valid certificate forever:
// mc if uninserted, else mc2 if known and uninserted, is the first uninserted id,
// and once both are inserted every id before the cursor is.  A word is written
// with one atomicMax (cursor in the top bits: the furthest scan wins), so readers
// never see a cursor from one scan with ids from another.  n <= 2^21 - 1.
#if TM_PROFILE
__device__ unsigned long long g_rp[4];
__shared__ unsigned long long g_mw_round;   // slowest merge warp this round   // replay segments: prefix scan, winner, re-queue split, sort
__device__ unsigned long long g_tm_prof[8];   // fg vertices looked up, scanned, tail batches; bg scans
#endif
struct VSt {
    int mc, mc2, cur;
};
__device__ __forceinline__ VSt vst_unpack(unsigned long long x) {
    VSt r;
    r.mc = (int)(x & 0x1fffffull) - 1;
    r.mc2 = (int)((x >> 21) & 0x1fffffull) - 1;
    r.cur = (int)(x >> 42);
    return r;
}
__device__ __forceinline__ unsigned long long vst_pack(int mc, int mc2, int cur) {
    return ((unsigned long long)(uint32_t)cur << 42) | ((unsigned long long)(uint32_t)(mc2 + 1) << 21) |
           (unsigned long long)(uint32_t)(mc + 1);
}
// the first uninserted id certified by the word, or -1 (scan from r.cur)
__device__ __forceinline__ int vst_pick(const uint32_t *bits, const VSt &r) {
    if (r.mc < 0) return -1;
    if (!is_ins(bits, r.mc)) return r.mc;
    if (r.mc2 >= 0 && !is_ins(bits, r.mc2)) return r.mc2;
    return -1;
}

// Warp probe of NQ x 32 consecutive ids of a sorted row (val[q] = id at offset
// q*32 + lane, -1 past the end; ok[q] = uninserted): offset of the first
// uninserted id (>= NQ*32: none), that id and the next uninserted one (or -1).
template <int NQ>
__device__ __forceinline__ unsigned probe_two(const int (&val)[NQ], const bool (&ok)[NQ], int &hit, int &hit2,
                                              unsigned &off2) {
    const int lane = threadIdx.x & 31;
    int q1 = NQ, q2 = NQ, h1 = -1, h2 = -1;
#pragma unroll
    for (int q = NQ - 1; q >= 0; q--)
        if (ok[q]) { q2 = q1; h2 = h1; q1 = q; h1 = val[q]; }
    const unsigned k1 = (unsigned)(q1 * 32 + lane);
    const unsigned best = __reduce_min_sync(0xffffffffu, k1);
    const bool mine = best < (unsigned)(NQ * 32) && (int)(best & 31u) == lane;
    const unsigned second = __reduce_min_sync(0xffffffffu, mine ? (unsigned)(q2 * 32 + lane) : k1);
    const int src = mine ? h2 : h1;
    hit = __shfl_sync(0xffffffffu, h1, best & 31u);
    const int s2 = __shfl_sync(0xffffffffu, src, second & 31u);
    if (best >= (unsigned)(NQ * 32)) hit = -1;
    hit2 = second < (unsigned)(NQ * 32) ? s2 : -1;
    off2 = second;
    return best;
}

// Long-tail cursor probe (16 x 32 ids of one sorted row), kept out of line: its 16
// loads in flight would otherwise raise the register pressure of every refresh and
// push the face / candidate ids of the common path into local memory.
__device__ __noinline__ unsigned tail_probe(const int32_t *row, int c, int m, const uint32_t *bits, int &hit,
                                            int &hit2, unsigned &o2) {
    const int lane = threadIdx.x & 31;
    int val[16];
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const int idx = c + q * 32 + lane;
        val[q] = idx < m ? __ldg(row + idx) : -1;
    }
    bool ok[16];
#pragma unroll
    for (int q = 0; q < 16; q++) ok[q] = val[q] >= 0 && !is_ins(bits, val[q]);
    return probe_two<16>(val, ok, hit, hit2, o2);
}

__shared__ int g_went[TM_WARPS][10 * TM_EPW];   // warp_entries scratch (per hardware warp)

// One warp builds up to TM_EPW entries: refresh the 3 vertices of each face
// (first uninserted id of order[w], tmfg.py:169-182) and pick the best of the
// three candidates (tmfg.py:266-277).  Cursor probes: 4 x 32 ids per vertex in
// one batch of independent loads; rare long tails continue 16 x 32 at a time.

template <bool SMEM_ST>
__device__ void warp_entries(const TmArgs &A, const uint32_t *bits, unsigned long long *vst, int cnt,
                             const int (*fverts)[3], const int *fids, Ent *out, int *iters, int *mc_out) {
    const int lane = threadIdx.x & 31;
    const int n = A.n, m = n - 1;
    constexpr int NV = 3 * TM_EPW;
    unsigned long long *st = SMEM_ST ? vst : A.gvst;
    // warp-uniform face vertices / candidates live in a per-warp shared-memory slot across the
    // (register-hungry) cursor probes instead of spilling to local memory (L2 latency)
    int *F = g_went[threadIdx.x >> 5];   // [0,NV) vertex, [NV,2NV) mc, [2NV,3NV) mc2, [3NV,..) fid
    int vv[NV], cur[NV], found[NV], found2[NV];
    const int nv = 3 * cnt;
    // a vertex whose certified max-corr (or the id after it) is still uninserted needs no scan
    unsigned pending = 0u;
    // vertex k's word is read and decided by lane k (all of them at once, not one after the
    // other on lane 0) and broadcast: background warps rewrite the word and the winner's bit
    // may be set concurrently (speculative refreshes), and every lane must take the same scan
    // decision (full-mask collectives follow)
    int c_mine = 0, f_mine = -1;
    if (lane < nv && lane < NV) {
        const VSt r = vst_unpack(st[fverts[lane / 3][lane % 3]]);
        c_mine = r.cur;
        f_mine = vst_pick(bits, r);
    }
#pragma unroll
    for (int k = 0; k < NV; k++) {
        vv[k] = k < nv ? fverts[k / 3][k % 3] : 0;
        cur[k] = __shfl_sync(0xffffffffu, c_mine, k);
        const int mcv = __shfl_sync(0xffffffffu, f_mine, k);
        found[k] = -1;
        found2[k] = -1;
        if (k < nv) {
            if (mcv >= 0) found[k] = mcv;
            else pending |= 1u << k;
        }
    }
    const unsigned scanned = pending;
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NV; q++) { F[q] = vv[q]; F[NV + q] = found[q]; F[2 * NV + q] = found2[q]; }
#pragma unroll
        for (int q = 0; q < TM_EPW; q++) F[3 * NV + q] = q < cnt ? fids[q] : -1;
    }
    __syncwarp();
#if TM_PROFILE
    long long tw0 = clock64();
    if (lane == 0) { atomicAdd(&g_tm_prof[0], (unsigned long long)nv); atomicAdd(&g_tm_prof[1], (unsigned long long)__popc(pending)); }
#endif
    {
        // one vertex at a time (a refresh rarely has more than one to scan): keeps the
        // probe's registers small enough that the face / candidate ids are not spilled
#pragma unroll
        for (int k = 0; k < NV; k++) {
            if ((pending >> k) & 1u) {
                int val[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int idx = cur[k] + q * 32 + lane;
                    val[q] = idx < m ? __ldg(A.order + (int64_t)F[k] * m + idx) : -1;
                }
                bool ok[4];
#pragma unroll
                for (int q = 0; q < 4; q++) ok[q] = val[q] >= 0 && !is_ins(bits, val[q]);
                int h1, h2;
                unsigned o2;
                const unsigned best = probe_two<4>(val, ok, h1, h2, o2);
                if (best < 128u) {
                    __syncwarp();
                    if (lane == 0) { F[NV + k] = h1; F[2 * NV + k] = h2; }
                    __syncwarp();
                    cur[k] += (int)(h2 >= 0 ? o2 : best);
                    pending &= ~(1u << k);
                } else {
                    cur[k] += 128;
                }
            }
        }
    }
#if TM_PROFILE
    long long tw1 = clock64();
#endif
    while (pending) {
        (*iters)++;
#if TM_PROFILE
        if (lane == 0) atomicAdd(&g_tm_prof[2], 1ull);
#endif
        const int k = __ffs(pending) - 1;
        int w = 0, c = 0;
#pragma unroll
        for (int q = 0; q < NV; q++)
            if (q == k) c = cur[q];
        w = F[k];
        int hit, hit2;
        unsigned o2;
        const unsigned best = tail_probe(A.order + (int64_t)w * m, c, m, bits, hit, hit2, o2);
        const int adv = best < 512u ? (int)(hit2 >= 0 ? o2 : best) : 512;
        const int cn = min(c + adv, m);
#pragma unroll
        for (int q = 0; q < NV; q++)
            if (q == k) cur[q] = cn;
        if (hit >= 0) {
            __syncwarp();
            if (lane == 0) { F[NV + k] = hit; F[2 * NV + k] = hit2; }
            __syncwarp();
        }
        if (hit >= 0 || cn >= m) pending &= ~(1u << k);
    }
    if (lane == 0) {
        if (mc_out) {
#pragma unroll
            for (int k = 0; k < NV; k++)
                if (k < nv) mc_out[k] = F[NV + k];
        }
#pragma unroll
        for (int k = 0; k < NV; k++)
            if ((scanned >> k) & 1u) atomicMax(st + F[k], vst_pack(F[NV + k], F[2 * NV + k], min(cur[k], m)));
    }
#if TM_PROFILE
    long long tw2 = clock64();
#endif
    // 9 similarity loads per entry: lane = e*9 + ci*3 + vi loads S[face_vi, cand_ci]
    double sv = 0.0;
    int my_u = -1;
    {
        const int e = lane / 9, r = lane % 9, ci = r / 3, vi = r % 3;
        const int u = e < cnt ? F[NV + e * 3 + ci] : -1;
        const int w = e < cnt ? F[e * 3 + vi] : 0;
        if (e < cnt && u >= 0) sv = __ldg(A.S + (int64_t)w * n + u);
        my_u = u;
    }
    // lanes with vi == 0 form g = (S[a,u] + S[b,u]) + S[c,u]  (tmfg.py:273, left to right)
    const double s1 = __shfl_down_sync(0xffffffffu, sv, 1);
#if TM_PROFILE
    long long tw3 = clock64() + (long long)(s1 != s1);
    if (lane == 0) { iters[1] = (int)(tw1 - tw0); iters[2] = (int)(tw2 - tw1); iters[3] = (int)(tw3 - tw2); }
#endif
    const double s2 = __shfl_down_sync(0xffffffffu, sv, 2);
    const double g = __dadd_rn(__dadd_rn(sv, s1), s2);
    // entry leader (lane e*9) picks the best of its 3 candidates: g desc, u asc
    const double g1 = __shfl_down_sync(0xffffffffu, g, 3), g2 = __shfl_down_sync(0xffffffffu, g, 6);
    const int u1 = __shfl_down_sync(0xffffffffu, my_u, 3), u2 = __shfl_down_sync(0xffffffffu, my_u, 6);
    if (lane % 9 == 0 && lane / 9 < cnt) {
        const int e = lane / 9;
        double best_g = -INFINITY;   // candidates in (mc[a], mc[b], mc[c]) order (tmfg.py:272-276)
        int best_v = -1;
        if (g > best_g || (g == best_g && my_u < best_v)) { best_g = g; best_v = my_u; }
        if (g1 > best_g || (g1 == best_g && u1 < best_v)) { best_g = g1; best_v = u1; }
        if (g2 > best_g || (g2 == best_g && u2 < best_v)) { best_g = g2; best_v = u2; }
        Ent x;
        x.g = best_g;
        x.fid = F[3 * NV + e];
        x.cand = best_v;
        x.a = F[e * 3 + 0];
        x.b = F[e * 3 + 1];
        x.c = F[e * 3 + 2];
        x.opt = 0;
        out[e] = x;
    }
    __syncwarp();
    if (A.check) {
        // tmfg.py:377-380 true_best_gain: brute force over every uninserted vertex
        for (int e = 0; e < cnt; e++) {
            const double *Sa = A.S + (int64_t)fverts[e][0] * n;
            const double *Sb = A.S + (int64_t)fverts[e][1] * n;
            const double *Sc = A.S + (int64_t)fverts[e][2] * n;
            double best = -INFINITY;
            for (int u = lane; u < n; u += 32) {
                if (is_ins(bits, u)) continue;
                double gg = __dadd_rn(__dadd_rn(Sa[u], Sb[u]), Sc[u]);
                best = fmax(best, gg);
            }
            for (int o = 16; o; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (lane == 0) out[e].opt = out[e].g >= __dsub_rn(best, 1e-12);
            __syncwarp();
        }
    }
}

// Fast path of one entry refresh.  When all three vertices' scan-state words certify an
// uninserted max-corr (the common case: the cluster helpers keep the words two deep), lanes
// 0..8 each read the word of "their" candidate's vertex (lanes of one candidate read the same
// address in the same instruction, so they agree), load their S value and reduce -- no
// shuffle broadcast of the words, no per-warp staging slot, no local-memory face arrays.

// lane (ci, vi) = (lane / 3, lane % 3), lane < 9, holds candidate u = mc[face vertex ci] and
// w = face vertex vi: 9 loads of S, g = (S[a,u] + S[b,u]) + S[c,u] per candidate (tmfg.py:273,
// left to right), best of the three in (mc[a], mc[b], mc[c]) order: g desc, u asc (tmfg.py:272-276)
__device__ __forceinline__ void entry_from_cands(const TmArgs &A, int a, int b, int c, int fid, int u, int w, Ent *out,
                                                 int *mc_out, int *iters) {
    const int lane = threadIdx.x & 31;
#if TM_PROFILE
    const long long tf1 = clock64();
#endif
    const double sv = lane < 9 ? __ldg(A.S + (int64_t)w * A.n + u) : 0.0;
    const double s1 = __shfl_down_sync(0xffffffffu, sv, 1);
#if TM_PROFILE
    const long long tf2 = clock64() + (long long)(s1 != s1);
    if (iters && lane == 0) iters[3] = (int)(tf2 - tf1);
#endif
    const double s2 = __shfl_down_sync(0xffffffffu, sv, 2);
    const double g = __dadd_rn(__dadd_rn(sv, s1), s2);
    const double g1 = __shfl_down_sync(0xffffffffu, g, 3), g2 = __shfl_down_sync(0xffffffffu, g, 6);
    const int u1 = __shfl_down_sync(0xffffffffu, u, 3), u2 = __shfl_down_sync(0xffffffffu, u, 6);
    if (mc_out && (lane == 0 || lane == 3 || lane == 6)) mc_out[lane / 3] = u;
    if (lane == 0) {
        double best_g = g;
        int best_v = u;
        if (g1 > best_g || (g1 == best_g && u1 < best_v)) { best_g = g1; best_v = u1; }
        if (g2 > best_g || (g2 == best_g && u2 < best_v)) { best_g = g2; best_v = u2; }
        Ent x;
        x.g = best_g;
        x.fid = fid;
        x.cand = best_v;
        x.a = a;
        x.b = b;
        x.c = c;
        x.opt = 0;
        *out = x;
    }
    __syncwarp();
}

// Returns false (nothing written) when a vertex needs a scan: the caller runs warp_entries.
template <bool SMEM_ST>
__device__ __forceinline__ bool warp_entry_fast(const TmArgs &A, const uint32_t *bits, unsigned long long *vst,
                                                int a, int b, int c, int fid, Ent *out, int *mc_out,
                                                int *iters = nullptr) {
    const int lane = threadIdx.x & 31;
    const unsigned long long *st = SMEM_ST ? vst : A.gvst;
    const int l9 = lane < 9 ? lane : 0;
    const int ci = l9 / 3, vi = l9 - 3 * ci;
    const int xc = ci == 0 ? a : (ci == 1 ? b : c);
    const int w = vi == 0 ? a : (vi == 1 ? b : c);
    const VSt r = vst_unpack(st[xc]);
    // both certificates' bitmap words in flight at once
    const bool i1 = r.mc < 0 || is_ins(bits, max(r.mc, 0));
    const bool i2 = r.mc2 < 0 || is_ins(bits, max(r.mc2, 0));
    const int u = !i1 ? r.mc : (!i2 ? r.mc2 : -1);
    if (__any_sync(0xffffffffu, u < 0)) return false;
#if TM_PROFILE
    if (lane == 0) atomicAdd(&g_tm_prof[0], 3ull);
#endif
    entry_from_cands(A, a, b, c, fid, u, w, out, mc_out, iters);
    return true;
}

// One window position (queue entry *hp at position i) of the parallel phase, one warp:
// fresh -> flags only; stale -> the refresh cache's entry if its three max-corr candidates
// are still uninserted (a refreshed entry stays exact while they are: each is a monotone
// fact; the cache is written only between rounds, so this read is stable), else the fast
// refresh.  With the scan state in shared memory the cache's candidates (lanes 9..11) and
// the scan-state words' (lanes 0..8) go through the inserted bitmap in one instruction
// stream, so the cache check is not a dependent step before the refresh.  Returns false
// (nothing written) when a vertex needs a scan.
template <bool SMEM_ST>
__device__ __forceinline__ bool window_refresh(const TmArgs &A, const uint32_t *bits, unsigned long long *vst,
                                               const RcEnt *rcache, const Ent *hp, int i, Ent *Lref, int *Lstale,
                                               int *Lcomp, int (*Lmc)[3], int *iters, unsigned *rc_hits) {
    const int lane = threadIdx.x & 31;
    const int2 fc = *reinterpret_cast<const int2 *>(&hp->fid);   // (fid, cand)
    if (!is_ins(bits, fc.y)) {
        if (lane == 0) { Lstale[i] = 0; Lcomp[i] = 0; }
        return true;
    }
    const int4 fa = *reinterpret_cast<const int4 *>(&hp->a);     // (a, b, c, opt)
    const int a = fa.x, b = fa.y, c = fa.z, fid = fc.x;
    const RcEnt &rc = rcache[fid & (TM_RC - 1)];
    const int l9 = lane < 9 ? lane : 0;
    const int ci = l9 / 3, vi = l9 - 3 * ci;
    const int xc = ci == 0 ? a : (ci == 1 ? b : c);
    const int w = vi == 0 ? a : (vi == 1 ? b : c);
    const bool rcl = lane >= 9 && lane < 12;
    int id1, id2 = -1;
    bool rc_ok;
    int u;
    if (SMEM_ST) {
        if (rcl) {
            id1 = rc.fid == fid ? rc.m[lane - 9] : -1;
        } else {
            const VSt r = vst_unpack(vst[xc]);
            id1 = r.mc;
            id2 = r.mc2;
        }
        const bool i1 = id1 < 0 || is_ins(bits, max(id1, 0));
        const bool i2 = id2 < 0 || is_ins(bits, max(id2, 0));
        u = !i1 ? id1 : (!i2 ? id2 : -1);
        const unsigned okb = __ballot_sync(0xffffffffu, u >= 0);
        rc_ok = (okb & 0xe00u) == 0xe00u;
        if (!rc_ok && (okb & 0x1ffu) != 0x1ffu) return false;
    } else {
        id1 = (lane < 3 && rc.fid == fid) ? rc.m[lane] : -1;
        const bool okc = id1 >= 0 && !is_ins(bits, id1);
        rc_ok = (__ballot_sync(0xffffffffu, okc) & 7u) == 7u;
        u = -1;
        if (!rc_ok) {
            const VSt r = vst_unpack(A.gvst[xc]);
            const bool i1 = r.mc < 0 || is_ins(bits, max(r.mc, 0));
            const bool i2 = r.mc2 < 0 || is_ins(bits, max(r.mc2, 0));
            u = !i1 ? r.mc : (!i2 ? r.mc2 : -1);
            if (__any_sync(0xffffffffu, u < 0)) return false;
        }
    }
    if (rc_ok) {
        if (lane == 0) {
            Ent x;
            x.g = rc.g;
            x.fid = fid;
            x.cand = rc.cand;
            x.a = a;
            x.b = b;
            x.c = c;
            x.opt = 0;
            Lref[i] = x;
            Lstale[i] = 1;
            Lcomp[i] = 0;
#if TM_PROFILE
            atomicAdd(rc_hits, 1u);
#endif
        }
        return true;
    }
#if TM_PROFILE
    if (lane == 0) atomicAdd(&g_tm_prof[0], 3ull);
#endif
    if (lane == 0) { Lstale[i] = 1; Lcomp[i] = 1; }
    entry_from_cands(A, a, b, c, fid, u, w, &Lref[i], Lmc[i], iters);
    return true;
}

// Two window entries per warp, one per half-warp (entry of half h at queue position base + h * TM_CH):
// window_refresh's logic with lanes 16 h + (0..8) on the scan-state words and 16 h + (9..11) on the
// refresh cache, so a round speculates over TM_K = 2 TM_CH queue positions in the latency of one
// refresh.  Returns the halves (bits 0..1) whose entry needs a scan (nothing written for them).
template <bool SMEM_ST>
__device__ __forceinline__ unsigned window_refresh2(const TmArgs &A, const uint32_t *bits, unsigned long long *vst,
                                                    const RcEnt *rcache, const Ent *cur, int base, int cntL,
                                                    Ent *Lref, int *Lstale, int *Lcomp, int (*Lmc)[3],
                                                    unsigned *rc_hits) {
    const int lane = threadIdx.x & 31;
    const int h = lane >> 4, l = lane & 15;
    const int i = base + h * TM_CH;
    const bool valid = i < cntL;
    const Ent *hp = cur + (valid ? i : base);
    // (fid, cand) and (a, b, c, opt) in flight together: one dependent shared-memory step less
    const int2 fc = *reinterpret_cast<const int2 *>(&hp->fid);
    const int4 fa = *reinterpret_cast<const int4 *>(&hp->a);
    const bool stale = valid && is_ins(bits, fc.y);
    if (!__any_sync(0xffffffffu, stale)) {
        if (valid && l == 0) { Lstale[i] = 0; Lcomp[i] = 0; }
        return 0u;
    }
    const int a = fa.x, b = fa.y, c = fa.z, fid = fc.x;
    const RcEnt &rc = rcache[fid & (TM_RC - 1)];
    const int l9 = l < 9 ? l : 0;
    const int ci = l9 / 3, vi = l9 - 3 * ci;
    int xc = c, w = c;   // selects, not branches
    xc = ci == 1 ? b : xc;
    xc = ci == 0 ? a : xc;
    w = vi == 1 ? b : w;
    w = vi == 0 ? a : w;
    const bool rcl = l >= 9 && l < 12;
    int id1 = -1, id2 = -1;
    bool rc_ok, fast_ok;
    int u;
    if (SMEM_ST) {
        if (stale) {
            if (rcl) {
                id1 = rc.fid == fid ? rc.m[l - 9] : -1;
            } else {
                const VSt r = vst_unpack(vst[xc]);
                id1 = r.mc;
                id2 = r.mc2;
            }
        }
        const bool i1 = id1 < 0 || is_ins(bits, max(id1, 0));
        const bool i2 = id2 < 0 || is_ins(bits, max(id2, 0));
        u = !i1 ? id1 : (!i2 ? id2 : -1);
        const unsigned okb = (__ballot_sync(0xffffffffu, u >= 0) >> (16 * h)) & 0xffffu;
        rc_ok = (okb & 0xe00u) == 0xe00u;
        fast_ok = (okb & 0x1ffu) == 0x1ffu;
    } else {
        id1 = (stale && l < 3 && rc.fid == fid) ? rc.m[l] : -1;
        const bool okc = id1 >= 0 && !is_ins(bits, id1);
        rc_ok = ((__ballot_sync(0xffffffffu, okc) >> (16 * h)) & 7u) == 7u;
        u = -1;
        if (stale && !rc_ok) {
            const VSt r = vst_unpack(A.gvst[xc]);
            const bool i1 = r.mc < 0 || is_ins(bits, max(r.mc, 0));
            const bool i2 = r.mc2 < 0 || is_ins(bits, max(r.mc2, 0));
            u = !i1 ? r.mc : (!i2 ? r.mc2 : -1);
        }
        fast_ok = ((__ballot_sync(0xffffffffu, u >= 0) >> (16 * h)) & 0x1ffu) == 0x1ffu;
    }
    const bool need_S = stale && !rc_ok && fast_ok;
    const bool slow = stale && !rc_ok && !fast_ok;
    const double sv = (need_S && l < 9) ? __ldg(A.S + (int64_t)w * A.n + u) : 0.0;
    const double s1 = __shfl_down_sync(0xffffffffu, sv, 1);
    const double s2 = __shfl_down_sync(0xffffffffu, sv, 2);
    const double g = __dadd_rn(__dadd_rn(sv, s1), s2);   // (S[a,u] + S[b,u]) + S[c,u]  (tmfg.py:273)
    const double g1 = __shfl_down_sync(0xffffffffu, g, 3), g2 = __shfl_down_sync(0xffffffffu, g, 6);
    const int u1 = __shfl_down_sync(0xffffffffu, u, 3), u2 = __shfl_down_sync(0xffffffffu, u, 6);
    if (need_S && l < 9 && vi == 0) Lmc[i][ci] = u;
    if (valid && l == 0 && !slow) {
        Lstale[i] = stale;
        Lcomp[i] = need_S;
        if (stale) {
            Ent x;
            if (rc_ok) {
                x.g = rc.g;
                x.cand = rc.cand;
#if TM_PROFILE
                atomicAdd(rc_hits, 1u);
#endif
            } else {
                double best_g = g;   // (mc[a], mc[b], mc[c]) order: g desc, u asc (tmfg.py:272-276)
                int best_v = u;
                if (g1 > best_g || (g1 == best_g && u1 < best_v)) { best_g = g1; best_v = u1; }
                if (g2 > best_g || (g2 == best_g && u2 < best_v)) { best_g = g2; best_v = u2; }
                x.g = best_g;
                x.cand = best_v;
            }
            x.fid = fid;
            x.a = a;
            x.b = b;
            x.c = c;
            x.opt = 0;
            Lref[i] = x;
        }
    }
    const unsigned sb = __ballot_sync(0xffffffffu, slow && l == 0);
    return (sb & 1u) | ((sb >> 15) & 2u);
}

__device__ __forceinline__ void sort3(int &x, int &y, int &z) {
    int t;
    if (y < x) { t = x; x = y; y = t; }
    if (z < y) { t = y; y = z; z = t; }
    if (y < x) { t = x; x = y; y = t; }
}

__device__ __forceinline__ void pool_put(const TmArgs &A, unsigned long long *minkey, int idx, const Ent &x) {
    A.pool_g[idx] = x.g;
    A.pool_fc[idx] = make_int2(x.fid, x.cand);
    atomicMin(minkey, tg_order_key(x.g));
}

// Move the largest pool entries into the (short) shared buffer.  The pool is
// struct-of-arrays (gain | fid, cand; face vertices come back from fv[fid]) so
// the selection passes stream 8 bytes per entry.  Threshold by a most-
// significant-digit radix walk over the 96-bit key (gain, ~fid) that starts at
// the first byte where the pool's smallest and largest gain keys differ; stop at
// the first digit boundary whose "all keys above" set is non-empty and fits.
// Keys are unique and the pool order is irrelevant, so the result is exact.
// Taken entries leave holes that are refilled from the pool's tail (O(taken)).
constexpr int RF_U = 8;   // pool loads in flight per thread in the selection passes
constexpr int RF_LOG = 11, RF_BINS = 1 << RF_LOG;   // selection histogram bins
constexpr int RF_RB = 1024;   // bins of the counting sort that ranks the taken entries
// Entries one refill may take: 3/4 of the queue (a refill costs about the same whatever it takes
// -- its passes over the whole pool dominate -- so fewer, larger refills; 1/2 before)
#ifndef TM_RF_NUM
#define TM_RF_NUM 3
#define TM_RF_DEN 4
#endif
constexpr int rf_room(int qb) { return qb * TM_RF_NUM / TM_RF_DEN; }
static_assert(2 * RF_RB <= RF_BINS, "the rank bins reuse the selection histogram");
static_assert(RF_BINS * 4 + rf_room(TM_B) * 24 <= TM_B * (int)sizeof(Ent), "refill scratch overflows the spare buffer");
static_assert(RF_BINS * 4 + rf_room(TM_BMAX) * 24 <= TM_BMAX * (int)sizeof(Ent), "refill scratch overflows the spare buffer");

template <int NT, int QB>
__device__ void refill(const TmArgs &A, Ctl &ctl, Ent *cur, Ent *scratch, Ent *red_e, int *red_ok, int tid) {
    const int lane = tid & 31, warp = tid >> 5;
    const int P = ctl.pool_count;
    constexpr int RM = rf_room(QB);
    const int room = min(QB - ctl.size, RM);
#if TM_PROFILE
    long long rc0 = fg_sync_clock(), rc1;
#endif
    int *takeidx = reinterpret_cast<int *>(scratch) + RF_BINS;   // room entries (after the histogram)
    int *holes = takeidx + RM;                         // room entries
    double *tgv = reinterpret_cast<double *>(holes + RM);
    int *tfv = reinterpret_cast<int *>(tgv + RM);
    int *binned = tfv + RM;                            // room entries: taken entries grouped by rank bin
    unsigned long long thr_hi = 0ull, thr_lo = 0ull;
    const bool take_all = P <= room;
    if (!take_all) {
        // Threshold key: linear 2048-bin histograms over the pool's key window
        // [pool min, pool max] (kept incrementally), refined inside the top bin
        // only when that bin alone is larger than the room; exact gain ties that
        // straddle the room fall through to a byte-radix walk over ~fid.
        int *hist = reinterpret_cast<int *>(scratch);
        if (tid == 0) { ctl.sel_room = room; ctl.stop = 0; }
        unsigned long long lo = ctl.pool_minkey, hi = tg_order_key(ctl.pool_max.g);
        bool need_fid = false, done = false;
        for (int it = 0; it < 8 && !done; it++) {
            if (lo >= hi) { thr_hi = hi; need_fid = true; break; }
            const int nb = 64 - __clzll(hi - lo);
            const int shift = nb > RF_LOG ? nb - RF_LOG : 0;
            for (int i = tid; i < RF_BINS; i += NT) hist[i] = 0;
            fg_sync();
            for (int i0 = tid; i0 < P; i0 += RF_U * NT) {
                double gv[RF_U];
#pragma unroll
                for (int u = 0; u < RF_U; u++) gv[u] = i0 + u * NT < P ? A.pool_g[i0 + u * NT] : -INFINITY;
#pragma unroll
                for (int u = 0; u < RF_U; u++) {
                    const unsigned long long key = tg_order_key(gv[u]);
                    if (i0 + u * NT < P && key >= lo && key <= hi) atomicAdd(&hist[(int)((key - lo) >> shift)], 1);
                }
            }
            fg_sync();
            if (warp == 0) {
                // lane l owns bins [RF_BINS - (l+1)*PB, RF_BINS - l*PB): suffix sums from the top
                constexpr int PB = RF_BINS / 32;
                const int b0 = RF_BINS - (lane + 1) * PB;
                int s = 0, topnz = -1;
                for (int q = PB - 1; q >= 0; q--) {
                    s += hist[b0 + q];
                    if (topnz < 0 && hist[b0 + q]) topnz = b0 + q;
                }
                int incl = s;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int excl = incl - s;   // keys in bins above this lane's chunk
                const int room_now = ctl.sel_room;
                // lowest bin whose suffix still fits: inside the first lane whose total exceeds the room
                const unsigned over = __ballot_sync(0xffffffffu, incl > room_now);
                const int fl = over ? __ffs(over) - 1 : 31;
                int best = -1;
                if (lane == fl) {
                    int acc = excl;
                    best = acc > 0 ? b0 + PB : -1;   // everything above this chunk fits
                    for (int q = PB - 1; q >= 0; q--) {
                        if (acc + hist[b0 + q] > room_now) break;
                        acc += hist[b0 + q];
                        if (acc > 0) best = b0 + q;
                    }
                }
                best = __shfl_sync(0xffffffffu, best, fl);
                const unsigned nzb = __ballot_sync(0xffffffffu, topnz >= 0);
                const int top = nzb ? __shfl_sync(0xffffffffu, topnz, __ffs(nzb) - 1) : -1;
                if (lane == 0) {
                    if (best >= 0) {
                        ctl.sel_prefix = lo + ((unsigned long long)best << shift);
                        ctl.stop = 1;
                    } else {
                        ctl.sel_prefix = lo + ((unsigned long long)top << shift);   // refine inside the top bin
                        ctl.stop = 0;
                    }
                }
            }
            fg_sync();
            if (ctl.stop) {
                thr_hi = ctl.sel_prefix;
                thr_lo = 0ull;
                done = true;
            } else {
                const unsigned long long nlo = ctl.sel_prefix;
                const unsigned long long nhi = nlo + ((1ull << shift) - 1ull);
                lo = nlo;
                hi = nhi < hi ? nhi : hi;
            }
            fg_sync();
#if TM_PROFILE
            if (tid == 0) atomicAdd(&g_tm_prof[7], 1ull);   // selection passes over the pool (reported as spec_refreshes)
#endif
        }
        if (need_fid) {
            // all remaining candidates share one gain: select on ~fid bytes
            if (tid == 0) { ctl.sel_prefix = 0ull; ctl.stop = 0; }
            fg_sync();
            for (int pass = 8; pass < 16; pass++) {
                const int p = pass & 7;
                const int shift = 56 - 8 * p;
                for (int i = tid; i < 256; i += NT) ctl.hist[i] = 0;
                fg_sync();
                const unsigned long long pref = ctl.sel_prefix;
                for (int i = tid; i < P; i += NT) {
                    if (tg_order_key(A.pool_g[i]) != thr_hi) continue;
                    const unsigned long long key = ~(unsigned long long)(unsigned)A.pool_fc[i].x;
                    if (p > 0 && (key >> (64 - 8 * p)) != (pref >> (64 - 8 * p))) continue;
                    atomicAdd(&ctl.hist[(key >> shift) & 255], 1);
                }
                fg_sync();
                if (tid == 0) {
                    int acc = 0, d = 255, last_fit = -1;
                    for (; d >= 0; d--) {
                        if (acc + ctl.hist[d] > ctl.sel_room) break;
                        acc += ctl.hist[d];
                        if (ctl.hist[d]) last_fit = d;
                    }
                    if (acc > 0) {
                        ctl.sel_prefix = pref | ((unsigned long long)last_fit << shift);
                        ctl.stop = 1;
                    } else {
                        ctl.sel_prefix = pref | ((unsigned long long)d << shift);
                    }
                }
                fg_sync();
                if (ctl.stop) break;
            }
            thr_lo = ctl.sel_prefix;
        }
    }
#if TM_PROFILE
    rc1 = fg_sync_clock();
    if (tid == 0) { ctl.rf_t[0] += rc1 - rc0; rc0 = rc1; }
#endif
    fg_sync();
    if (tid == 0) { ctl.refill_take = 0; ctl.nsurv = 0; }
    fg_sync();
    // take pass: indices of the selected entries; best (max) of the rest
    double bg = 0.0;
    int bf = 0;
    bool ok = false;
    for (int i0 = tid; i0 < P; i0 += RF_U * NT) {
        double gv[RF_U];
        int fv[RF_U];
#pragma unroll
        for (int u = 0; u < RF_U; u++) {
            const int i = i0 + u * NT;
            gv[u] = i < P ? A.pool_g[i] : 0.0;
            fv[u] = i < P ? A.pool_fc[i].x : 0;
        }
#pragma unroll
        for (int u = 0; u < RF_U; u++) {
            const int i = i0 + u * NT;
            if (i >= P) continue;
            const double g = gv[u];
            const int f = fv[u];
            const unsigned long long kh = tg_order_key(g), kl = ~(unsigned long long)(unsigned)f;
            const bool take = take_all || kh > thr_hi || (kh == thr_hi && kl >= thr_lo);
            if (take) {
                const int s = atomicAdd(&ctl.refill_take, 1);
                takeidx[s] = i;
                tgv[s] = g;
                tfv[s] = f;
            } else if (!ok || (g > bg) || (g == bg && f < bf)) {
                bg = g; bf = f; ok = true;
            }
        }
    }
    for (int o = 16; o; o >>= 1) {
        const double g2 = __shfl_xor_sync(0xffffffffu, bg, o);
        const int f2 = __shfl_xor_sync(0xffffffffu, bf, o);
        const int ok2 = __shfl_xor_sync(0xffffffffu, (int)ok, o);
        if (ok2 && (!ok || g2 > bg || (g2 == bg && f2 < bf))) { bg = g2; bf = f2; ok = true; }
    }
    if (lane == 0) { red_e[warp].g = bg; red_e[warp].fid = bf; red_ok[warp] = ok; }
    fg_sync();
#if TM_PROFILE
    rc1 = fg_sync_clock();
    if (tid == 0) { ctl.rf_t[1] += rc1 - rc0; rc0 = rc1; }
#endif
    const int nt = ctl.refill_take;
    const int sz = ctl.size;
    const int keep = P - nt;
    // Pop-order rank of each taken entry by a counting sort over RF_RB linear bins of the taken
    // keys' range [threshold (or pool min), pool max] (bin 0 = largest keys), then an exact
    // (gain desc, fid asc) rank among the few entries of its own bin -- instead of comparing
    // every taken entry with every other (nt^2 / NT compares per thread: 15k cycles of a 38k-cycle
    // refill at n = 10k, 38k of 128k at n = 50k).
    int *bcnt = reinterpret_cast<int *>(scratch);   // the selection histogram is dead by now
    int *bstart = bcnt + RF_RB;
    const unsigned long long kmin = take_all ? ctl.pool_minkey : thr_hi;
    const unsigned long long kspan = tg_order_key(ctl.pool_max.g) - kmin;
    const int knb = 64 - __clzll(kspan);
    const int kshift = knb > 10 ? knb - 10 : 0;
    for (int i = tid; i < 2 * RF_RB; i += NT) bcnt[i] = 0;
    // the entries' (fid, cand) and face vertices: two dependent global round trips, under the ranking
    constexpr int PT = (RM + NT - 1) / NT;   // taken entries per thread
    int2 my_fc[PT];
    int4 my_fv[PT];
#pragma unroll
    for (int q = 0; q < PT; q++) {
        my_fc[q] = make_int2(0, 0);
        if (tid + q * NT < nt) my_fc[q] = A.pool_fc[takeidx[tid + q * NT]];
    }
#pragma unroll
    for (int q = 0; q < PT; q++) {
        my_fv[q] = make_int4(0, 0, 0, 0);
        if (tid + q * NT < nt) my_fv[q] = A.fv[my_fc[q].x];
    }
    fg_sync();
    int mybin[PT];
#pragma unroll
    for (int q = 0; q < PT; q++) {
        const int s = tid + q * NT;
        if (s < nt) {
            const unsigned long long d = (tg_order_key(tgv[s]) - kmin) >> kshift;
            mybin[q] = RF_RB - 1 - (int)(d < (unsigned long long)(RF_RB - 1) ? d : (unsigned long long)(RF_RB - 1));
            atomicAdd(&bcnt[mybin[q]], 1);
        }
    }
    fg_sync();
    if (warp == 0) {
        // exclusive prefix sums of the bin counts: lane l owns bins [32 l, 32 l + 32)
        constexpr int PB = RF_RB / 32;
        int sum = 0;
        for (int q = 0; q < PB; q++) sum += bcnt[lane * PB + q];
        int incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int acc = incl - sum;
        for (int q = 0; q < PB; q++) {
            bstart[lane * PB + q] = acc;
            acc += bcnt[lane * PB + q];
            bcnt[lane * PB + q] = 0;   // becomes the bin's fill cursor
        }
    }
    fg_sync();
#pragma unroll
    for (int q = 0; q < PT; q++) {
        const int s = tid + q * NT;
        if (s < nt) binned[bstart[mybin[q]] + atomicAdd(&bcnt[mybin[q]], 1)] = s;
    }
    fg_sync();
    // selected entries -> sorted tail of the buffer; holes below `keep` listed
#pragma unroll
    for (int q = 0; q < PT; q++) {
        const int s = tid + q * NT;
        if (s >= nt) continue;
        const double g = tgv[s];
        const int f = tfv[s];
        const int b0 = bstart[mybin[q]], b1 = b0 + bcnt[mybin[q]];
        int rank = b0;
        for (int pj = b0; pj < b1; pj++) {
            const int j = binned[pj];
            rank += (tgv[j] > g) | ((tgv[j] == g) & (tfv[j] < f));
        }
        const int i = takeidx[s];
        const int2 fc = my_fc[q];
        const int4 fvv = my_fv[q];
        Ent x;
        x.g = g;
        x.fid = fc.x;
        x.cand = fc.y;
        x.a = fvv.x;
        x.b = fvv.y;
        x.c = fvv.z;
        x.opt = 0;
        cur[sz + rank] = x;
        if (i < keep) holes[atomicAdd(&ctl.nsurv, 1)] = i;
    }
    fg_sync();
    // fill the holes with the surviving entries of the tail [keep, P) (any pairing)
#if TM_PROFILE
    rc1 = fg_sync_clock();
    if (tid == 0) { ctl.rf_t[2] += rc1 - rc0; rc0 = rc1; }
#endif
    if (tid == 0) ctl.nsurv = 0;
    fg_sync();
    for (int i = keep + tid; i < P; i += NT) {
        const double g = A.pool_g[i];
        const int2 fc = A.pool_fc[i];
        const unsigned long long kh = tg_order_key(g), kl = ~(unsigned long long)(unsigned)fc.x;
        if (!(take_all || kh > thr_hi || (kh == thr_hi && kl >= thr_lo))) {
            const int h = holes[atomicAdd(&ctl.nsurv, 1)];
            A.pool_g[h] = g;
            A.pool_fc[h] = fc;
        }
    }
    fg_sync();
#if TM_PROFILE
    rc1 = fg_sync_clock();
    if (tid == 0) { ctl.rf_t[3] += rc1 - rc0; rc0 = rc1; }
#endif
    if (tid == 0) {
        ctl.size = sz + nt;
        ctl.pool_count = keep;
        if (keep == 0) ctl.pool_minkey = ~0ull;
        bool any = false;
        Ent b;
        for (int w = 0; w < NT / 32; w++)
            if (red_ok[w] && (!any || red_e[w].g > b.g || (red_e[w].g == b.g && red_e[w].fid < b.fid))) {
                b = red_e[w];
                any = true;
            }
        ctl.pool_has_max = any;
        if (any) ctl.pool_max = b;
    }
    fg_sync();
}


// Branch-free key compare: (g1, f1) pops before (g2, f2) -- heapq order of (-g, fid).
__device__ __forceinline__ bool kgt(double g1, int f1, double g2, int f2) {
    return (g1 > g2) | ((g1 == g2) & (f1 < f2));
}

// Replays the lazy heap's pops for one round (chunks of TM_CH window positions, one lane per
// position).  Entries L[0..Lc) are the queue head in pop order; Lstale/Lref
// say which are stale and their refreshed entry under the current inserted
// set; NE are the fresh entries of the faces made by the last insertion (not
// queued yet).  Sequentially: pop the max of (L[i], best refreshed so far, best
// new); a stale L[i] pushes Lref[i]; the first fresh thing popped wins.  Only
// that first fresh pop can be a refreshed or a new entry, so the round ends at
// the first i where L[i] is fresh or is beaten by the running max of the
// refreshed entries or by the best new entry: a prefix max + a ballot.
__device__ void replay_warp(const TmArgs &A, Ctl &ctl, const Ent *L, const Ent *Lref, const int *Lstale,
                            const Ent *NE, Ent *tobuf, double *kg, int *kf, int *ksrc, double *tkg,
                            int *tkf) {
    const int lane = threadIdx.x & 31;
#if TM_PROFILE
    const long long rp0 = clock64();
#endif
    const int Lc = ctl.L_count, nec = ctl.ne_count;
    // best new entry (<= 4, every lane)
    double ng = 0.0;
    int nf = 0, ni = -1;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (k < nec) {
            const double g = NE[k].g;
            const int f = NE[k].fid;
            if ((ni < 0) | kgt(g, f, ng, nf)) { ng = g; nf = f; ni = k; }
        }
    }
    const bool have_ne = ni >= 0;
    // The window is replayed in chunks of TM_CH positions (one lane per position); a chunk in which
    // nothing fresh pops hands the best of its refreshed entries on to the next as the carry
    // (cg, cf, cix): every one of its entries popped stale and pushed its refreshed entry.
    double cg = 0.0;
    int cf = 0, cix = -1;
    bool cok = false;
    int istar = Lc;               // window position of the first fresh pop (Lc: none)
    int kind = 0, widx = -1;      // 1 = queue entry, 2 = refreshed entry, 3 = new entry
    int ginc = 0;
    for (int c0 = 0; c0 < Lc; c0 += TM_CH) {
        const int pos = c0 + lane;
        const bool v = lane < TM_CH && pos < Lc;
        const bool st = v && Lstale[pos];
        const double hg = v ? L[pos].g : 0.0;
        const int hf = v ? L[pos].fid : 0;
        const double rg = st ? Lref[pos].g : 0.0;
        const int rf = st ? Lref[pos].fid : 0;
        // inclusive prefix max of the chunk's refreshed entries, carrying their window position
        double ig = rg;
        int ifd = rf, iix = pos;
        bool iok = st;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double g2 = __shfl_up_sync(0xffffffffu, ig, o);
            const int f2 = __shfl_up_sync(0xffffffffu, ifd, o);
            const int x2 = __shfl_up_sync(0xffffffffu, iix, o);
            const bool k2 = __shfl_up_sync(0xffffffffu, (int)iok, o) != 0;
            const bool take = (lane >= o) & k2 & ((!iok) | kgt(g2, f2, ig, ifd));
            ig = take ? g2 : ig;
            ifd = take ? f2 : ifd;
            iix = take ? x2 : iix;
            iok = iok | take;
        }
        // exclusive prefix, then the carry of the earlier chunks
        double eg = __shfl_up_sync(0xffffffffu, ig, 1);
        int ef = __shfl_up_sync(0xffffffffu, ifd, 1);
        int eix = __shfl_up_sync(0xffffffffu, iix, 1);
        bool eok = (lane > 0) & (__shfl_up_sync(0xffffffffu, (int)iok, 1) != 0);
        if (cok && (!eok || kgt(cg, cf, eg, ef))) { eg = cg; ef = cf; eix = cix; eok = true; }
        const bool c = v & ((!st) | (eok & kgt(eg, ef, hg, hf)) | (have_ne & kgt(ng, nf, hg, hf)));
        const unsigned bc = __ballot_sync(0xffffffffu, c);
        const int nv = min(TM_CH, Lc - c0);
        const int il = bc ? __ffs(bc) - 1 : nv;   // stale pops of this chunk
        // tmfg.py:425-431 counters over the stale pops (+ the check_invariants assertion)
        const bool rose = st & (lane < il) & (rg > __dadd_rn(hg, 1e-12));
        ginc += __popc(__ballot_sync(0xffffffffu, rose));
        if (A.check) {
            const unsigned bb = __ballot_sync(0xffffffffu, rose && Lref[pos].opt);
            if (bb) {
                if (lane == __ffs(bb) - 1) {
                    ctl.bad = 2;
                    A.stats[4] = rf;
                    A.stats[5] = __double_as_longlong(hg);
                    A.stats[6] = __double_as_longlong(rg);
                    ctl.winner = 0;
                    ctl.exhausted = 0;
                    ctl.removed = 0;
                    ctl.nbuf_new = 0;
                }
                __syncwarp();
                return;
            }
        }
        if (bc) {
            // the winner: evaluated by the lane at the first fresh pop
            int k_l = 1, w_l = pos;
            double tg = hg;
            int tf = hf;
            if (have_ne & kgt(ng, nf, tg, tf)) { tg = ng; tf = nf; k_l = 3; w_l = ni; }
            if (eok & kgt(eg, ef, tg, tf)) { k_l = 2; w_l = eix; }
            kind = __shfl_sync(0xffffffffu, k_l, il);
            widx = __shfl_sync(0xffffffffu, w_l, il);
            istar = c0 + il;
            break;
        }
        // nothing fresh popped: the chunk's best refreshed entry joins the carry
        const double ag = __shfl_sync(0xffffffffu, ig, 31);
        const int af = __shfl_sync(0xffffffffu, ifd, 31);
        const int ax = __shfl_sync(0xffffffffu, iix, 31);
        const bool aok = __shfl_sync(0xffffffffu, (int)iok, 31) != 0;
        if (aok && (!cok || kgt(ag, af, cg, cf))) { cg = ag; cf = af; cix = ax; cok = true; }
    }
#if TM_PROFILE
    const long long rp1 = clock64() + (istar & 0);
#endif
    const bool more = (ctl.size > Lc) || (ctl.pool_count > 0);
    if (istar >= Lc && !more) {
        // the whole queue popped stale and nothing is left behind it: the best of the refreshed
        // and new entries is the next pop, and it is fresh
        if (have_ne && ((!cok) | kgt(ng, nf, cg, cf))) { kind = 3; widx = ni; }
        else if (cok) { kind = 2; widx = cix; }
    }
    const int npop = istar < Lc ? istar : Lc;   // stale pops
    if (lane == 0) {
        ctl.pops += npop + (kind ? 1 : 0);
        ctl.refreshes += npop;
        ctl.gain_inc += ginc;
        ctl.removed = npop + (kind == 1 ? 1 : 0);
        ctl.winner = kind != 0;
        ctl.exhausted = kind == 0;
        if (kind == 0 && !more) ctl.bad = 1;
        if (kind == 1) ctl.win = L[widx];
        else if (kind == 2) ctl.win = Lref[widx];
        else if (kind == 3) ctl.win = NE[widx];
    }
    // re-queue: refreshed entries of the stale pops (minus a refreshed winner) and
    // new entries (minus a new winner); above the pool max -> shared buffer, else pool
#if TM_PROFILE
    const long long rp2 = clock64() + (kind & 0);
#endif
    const bool pm = ctl.pool_has_max;
    const double pg = ctl.pool_max.g;
    const int pf = ctl.pool_max.fid;
    const unsigned lt = (1u << lane) - 1u;
    const int pc = ctl.pool_count;
    int nk = 0, npool = 0;   // buffer-bound keys listed, pool entries written
    static_assert(TM_CH + 4 <= 32, "the new entries ride on the first chunk's spare lanes");
    for (int c0 = 0; c0 < max(npop, 1); c0 += TM_CH) {
        const int pos = c0 + lane;
        const int nk_l = lane - TM_CH;   // lanes TM_CH.. of the first chunk: the new entries
        const bool bn = c0 == 0 && nk_l >= 0 && nk_l < nec && !((kind == 3) & (widx == nk_l));
        const bool br = lane < TM_CH && pos < npop && Lstale[pos] && !((kind == 2) & (widx == pos));
        const Ent *src = bn ? &NE[nk_l] : &Lref[pos];
        const bool any = br | bn;
        const double rg = any ? src->g : 0.0;
        const int rf = any ? src->fid : 0;
        const bool fr = any & ((!pm) | kgt(rg, rf, pg, pf));
        const bool pr = any & !fr;
        const unsigned bfr = __ballot_sync(0xffffffffu, fr), bpr = __ballot_sync(0xffffffffu, pr);
        // keys of the buffer-bound entries (src >= 0: Lref index, src < 0: ~NE index)
        if (fr) { const int o = nk + __popc(bfr & lt); kg[o] = rg; kf[o] = rf; ksrc[o] = bn ? ~nk_l : pos; }
        if (pr) pool_put(A, &ctl.pool_minkey, pc + npool + __popc(bpr & lt), *src);
        nk += __popc(bfr);
        npool += __popc(bpr);
    }
    const int nbuf = nk;
    __syncwarp();
    if (lane == 0) {
        ctl.pool_count = pc + npool;
        ctl.nbuf_new = nbuf;
    }
#if TM_PROFILE
    const long long rp3 = clock64() + (nbuf & 0);
#endif
    for (int k = lane; k < nbuf; k += 32) {
        const double g = kg[k];
        const int f = kf[k];
        int r = 0;
#pragma unroll 4
        for (int j = 0; j < nbuf; j++) r += kgt(kg[j], kf[j], g, f);
        const int sidx = ksrc[k];
        tobuf[r] = sidx >= 0 ? Lref[sidx] : NE[~sidx];
        tkg[r] = g;   // compact sorted keys for the merge's searches
        tkf[r] = f;
    }
    __syncwarp();
#if TM_PROFILE
    const long long rp4 = clock64();
    if (lane == 0) {
        g_rp[0] += rp1 - rp0;   // scan + winner
        g_rp[0] += rp2 - rp1;
        g_rp[1] += rp3 - rp2;
        g_rp[2] += rp4 - rp3;
    }
#endif
}

// Background warp: sweep the vertices (32 per step, lane-parallel check), and for
// every vertex whose cached max-corr is unknown or already inserted, advance its
// cursor to the first uninserted id of its sorted row (16 x 32 ids per load batch).
// Background warp: sweep the vertices 32 at a time; every lane whose vertex's
// certified max-corr is unknown or inserted scans its own sorted row from the
// cursor (8 ids per batch, up to 64 ids per visit), so 32 rows are in flight per
// warp.  The result -- first two uninserted ids, or just the advanced cursor --
// is published with one atomicMax: scan-state words only ever move forward.
template <bool SMEM_ST>
__device__ void bg_sweep(const TmArgs &A, const uint32_t *bits_, unsigned long long *vst, const int *stop_, int bgw) {
    const int lane = threadIdx.x & 31;
    const int n = A.n, m = n - 1;
    volatile const uint32_t *bits = bits_;
    volatile unsigned long long *st = SMEM_ST ? vst : A.gvst;
    volatile const int *stop = stop_;
    int w0 = bgw * 32;
    // the loop decision is lane 0's read, broadcast: lanes must leave together
    while (!__shfl_sync(0xffffffffu, lane == 0 ? *stop : 0, 0)) {
        const int w = w0 + lane;
        if (w < n) {
            const VSt r = vst_unpack(st[w]);
            // a vertex that is itself inserted may still be refreshed (face vertex)
            if (r.cur < m && (r.mc < 0 || ((bits[r.mc >> 5] >> (r.mc & 31)) & 1u))) {
                const int32_t *row = A.order + (int64_t)w * m;
                int c = r.cur, hit = -1, hit2 = -1, p1 = 0, p2 = 0;
                for (int it = 0; it < 8 && hit2 < 0 && c < m; it++) {
                    int val[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) val[q] = c + q < m ? __ldg(row + c + q) : -1;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int u = val[q];
                        if (u >= 0 && !((bits[u >> 5] >> (u & 31)) & 1u)) {
                            if (hit < 0) { hit = u; p1 = c + q; }
                            else if (hit2 < 0) { hit2 = u; p2 = c + q; }
                        }
                    }
                    c = min(c + 8, m);
                }
                const int cur = hit2 >= 0 ? p2 : (hit >= 0 ? p1 : c);
                atomicMax((unsigned long long *)st + w, vst_pack(hit, hit2, cur));
#if TM_PROFILE
                atomicAdd(&g_tm_prof[3], 1ull);
#endif
            }
        }
        __syncwarp();
        w0 += TM_BG_WARPS * 32;
        if (w0 >= n) w0 = bgw * 32;
    }
}

// Helper CTA of the cluster (ranks 1..): keeps every vertex's scan-state word
// two candidates deep -- mc and mc2 both certified uninserted -- so the
// foreground refreshes of the leader CTA (rank 0) find their max-corr without a
// dependent global scan.  The words live in the leader's shared memory (or in
// global memory for large n).  Each pass a helper copies the leader's inserted
// bitmap into its own shared memory (any snapshot is a subset of the truth, so
// every "inserted" it sees is a fact) and works on its own copy of its vertex
// slice's words, touching the leader only to re-read a word that looks out of
// date and to publish improvements -- the leader's shared memory serves its own
// critical path.  A lane scans 16 ids of its own row; rows still unresolved are
// scanned by the whole warp, 512 ids per coalesced batch.  Every write is an
// atomicMax of a valid certificate (see VSt).
__host__ __device__ __forceinline__ int tm_helper_slice(int n, int nslots) {
    const int stride = nslots * TM_T;
    return (n + stride - 1) / stride * TM_T;   // words per helper
}

template <bool SMEM_ST>
__device__ void cluster_helper(const TmArgs &A, const uint32_t *bits_r, unsigned long long *vst_r,
                               const int *stop_r, int slot, int nslots, unsigned char *lsmem) {
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    const int n = A.n, m = n - 1;
    const int nwords = (n + 31) >> 5;
    uint32_t *bits = reinterpret_cast<uint32_t *>(lsmem);                                    // local snapshot
    unsigned long long *lst = reinterpret_cast<unsigned long long *>(bits + ((nwords + 1) & ~1));   // local words
    volatile const uint32_t *rbits = bits_r;
    volatile unsigned long long *st = SMEM_ST ? vst_r : A.gvst;
    volatile const int *stop = stop_r;
    const int stride = nslots * TM_T;
    const int nloc = tm_helper_slice(n, nslots);
    for (int i = tid; i < nloc; i += TM_T) lst[i] = 0ull;
#if TM_PROFILE
    long long passes = 0;
#endif
    for (;;) {
        for (int i = tid; i < nwords; i += TM_T) bits[i] = rbits[i];
        __syncthreads();
        if (__syncthreads_or(tid == 0 ? *stop : 0)) break;
#if TM_PROFILE
        passes++;
#endif
        for (int k = 0, w0 = slot * TM_T + (tid & ~31); w0 < n; k++, w0 += stride) {
            const int w = w0 + lane;
            const int li = k * TM_T + tid;
            int a = -1, c = 0;
            bool need = false;
            if (w < n) {
                VSt r = vst_unpack(lst[li]);
                bool mc_in = r.mc >= 0 && is_ins(bits, r.mc);
                bool mc2_in = r.mc2 >= 0 && is_ins(bits, r.mc2);
                need = r.cur < m && !(r.mc >= 0 && !mc_in && r.mc2 >= 0 && !mc2_in);
                if (need) {
                    // the leader may have advanced it (its own scans): take the newer word
                    const unsigned long long x = max(lst[li], (unsigned long long)st[w]);
                    lst[li] = x;
                    r = vst_unpack(x);
                    mc_in = r.mc >= 0 && is_ins(bits, r.mc);
                    mc2_in = r.mc2 >= 0 && is_ins(bits, r.mc2);
                    need = r.cur < m && !(r.mc >= 0 && !mc_in && r.mc2 >= 0 && !mc2_in);
                }
                if (need) {
#if TM_PROFILE
                    atomicAdd(&g_tm_prof[3], 1ull);
#endif
                    // mc stays when uninserted; look for the id(s) after the cursor
                    const int32_t *row = A.order + (int64_t)w * m;
                    a = (r.mc >= 0 && !mc_in) ? r.mc : -1;
                    c = r.cur;
                    int b = -1, pb = 0;
                    int val[16];
#pragma unroll
                    for (int q = 0; q < 16; q++) val[q] = c + q < m ? __ldg(row + c + q) : -1;
#pragma unroll
                    for (int q = 0; q < 16; q++) {
                        const int u = val[q];
                        if (u >= 0 && u != r.mc && !is_ins(bits, u)) {
                            if (a < 0) a = u;
                            else if (b < 0) { b = u; pb = c + q; }
                        }
                    }
                    c = min(c + 16, m);
                    if (b >= 0 || c >= m) {
                        // cursor: at mc2 when found, else past everything scanned
                        const unsigned long long x = vst_pack(a, b, b >= 0 ? pb : c);
                        lst[li] = x;
                        atomicMax((unsigned long long *)st + w, x);
                        need = false;
                    }
                }
            }
            unsigned todo = __ballot_sync(0xffffffffu, need);
#if TM_PROFILE
            if (lane == 0 && todo) atomicAdd(&g_tm_prof[5], (unsigned long long)__popc(todo));
#endif
            while (todo) {
                const int l = __ffs(todo) - 1;
                todo &= todo - 1;
                const int ww = w0 + l;
                int cc = __shfl_sync(0xffffffffu, c, l), aa = __shfl_sync(0xffffffffu, a, l);
                int bb = -1, pbb = 0;
                const int32_t *row = A.order + (int64_t)ww * m;
                for (int it = 0; it < 4 && bb < 0 && cc < m; it++) {
#if TM_PROFILE
                    if (lane == 0) atomicAdd(&g_tm_prof[6], 1ull);
#endif
                    int val[16];
#pragma unroll
                    for (int q = 0; q < 16; q++) {
                        const int idx = cc + q * 32 + lane;
                        val[q] = idx < m ? __ldg(row + idx) : -1;
                    }
                    bool ok[16];
#pragma unroll
                    for (int q = 0; q < 16; q++) ok[q] = val[q] >= 0 && !is_ins(bits, val[q]);
                    int h1, h2;
                    unsigned o2;
                    const unsigned best = probe_two<16>(val, ok, h1, h2, o2);
                    if (best < 512u) {
                        if (aa < 0) {
                            aa = h1;
                            if (h2 >= 0) { bb = h2; pbb = cc + (int)o2; }
                        } else {
                            bb = h1;
                            pbb = cc + (int)best;
                        }
                    }
                    cc = min(cc + 512, m);
                }
                const unsigned long long x = vst_pack(aa, bb, bb >= 0 ? pbb : cc);
                if (lane == l) lst[k * TM_T + (tid & ~31) + l] = x;
                if (lane == 0) atomicMax((unsigned long long *)st + ww, x);
            }
        }
    }
#if TM_PROFILE
    if (threadIdx.x == 0 && slot == 0) A.stats[30] = passes;   // helper passes over the vertices
#endif
}

// Prefetcher CTA of the cluster (the last rank when A.prefetch): sweeps the head of the
// leader's shared-memory queue and, for each face (a, b, c) there, issues L2 prefetches of
// S[x, u] for x in the face and u in the certified max-corr candidates (mc, mc2) of its
// vertices -- the 9 (or 18) values the face's next refresh will read (tmfg.py:266-277), so
// that refresh finds them in L2 instead of HBM.  Reads are racy snapshots and only steer
// prefetches (every id is range-checked); nothing it does affects results.
constexpr int TM_PF_DEPTH = 384;   // queue entries swept per pass

template <bool SMEM_ST>
__device__ void cluster_prefetcher(const TmArgs &A, const Ent *qbuf_r, const int *sel_r, const int *size_r,
                                   const unsigned long long *vst_r, const int *stop_r) {
    const int tid = threadIdx.x;
    const int n = A.n;
    volatile const int *stop = stop_r;
    volatile const int *selp = sel_r;
    volatile const int *sizep = size_r;
    volatile const unsigned long long *st = SMEM_ST ? vst_r : A.gvst;
    // 3 threads per entry: thread (i, q) prefetches row x = vertex q of entry i at the 6 candidates
    const int i = tid / 3, q = tid % 3;
    while (!*stop) {
        const int sel = *selp, size = *sizep;
        if (i < TM_PF_DEPTH && i < size && tid < 3 * TM_PF_DEPTH) {
            const volatile Ent *e = qbuf_r + (sel ? tm_qb<SMEM_ST>() : 0) + i;
            const int a = e->a, b = e->b, c = e->c;
            if (a >= 0 && a < n && b >= 0 && b < n && c >= 0 && c < n) {
                const int x = q == 0 ? a : (q == 1 ? b : c);
                const double *row = A.S + (int64_t)x * n;
                const int vv[3] = {a, b, c};
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    const VSt r = vst_unpack(st[vv[k]]);
                    if (r.mc >= 0 && r.mc < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + r.mc));
                    if (r.mc2 >= 0 && r.mc2 < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + r.mc2));
                }
            }
        }
        __nanosleep(200);
    }
}

template <bool SMEM_ST>
__global__ void __launch_bounds__(TM_T, 1) tmfg_heap_kernel(const __grid_constant__ TmArgs A) {
    constexpr int QB = tm_qb<SMEM_ST>();
    constexpr int MW = tm_merge_warps<SMEM_ST>();
    extern __shared__ __align__(16) unsigned char tm_smem[];
    const int n = A.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ Ctl ctl;
    constexpr int KM = tm_kmax<SMEM_ST>();   // widest window
    constexpr int BT = KM + 8;               // longest re-queued run (+ new entries)
    // static shared memory must stay under 48 KB: with the wide window (scan state in global
    // memory) the refreshed entries and the re-queued run move to the dynamic part
    __shared__ Ent Lref_s[SMEM_ST ? KM : 1];
    __shared__ Ent tobuf_s[SMEM_ST ? BT : 1];
    __shared__ Ent Lout[TM_WARPS - TM_NEW_WARPS][TM_EPW];
    __shared__ int Lstale[KM];
    __shared__ Ent NE[4];
    __shared__ Ent red_e[TM_WARPS];
    __shared__ double rk_g[BT];
    __shared__ int rk_f[BT], rk_src[BT];
    __shared__ double tk_g[BT];   // tobuf's keys (gain, fid), sorted
    __shared__ int tk_f[BT];
    __shared__ int red_ok[TM_WARPS];
    __shared__ RcEnt rcache[TM_RC];
    __shared__ int rc_claim[TM_RC];   // round that last wrote the slot: one writer per slot per round
    __shared__ int Lmc[KM][3];
    __shared__ int Lcomp[KM];

    Ent *Lref = SMEM_ST ? Lref_s : reinterpret_cast<Ent *>(tm_smem);
    Ent *tobuf = SMEM_ST ? tobuf_s : Lref + KM;
    Ent *buf0 = SMEM_ST ? reinterpret_cast<Ent *>(tm_smem) : tobuf + BT;
    Ent *buf1 = buf0 + QB;
    uint32_t *bits = reinterpret_cast<uint32_t *>(buf1 + QB);
    const int nwords = (n + 31) >> 5;
    unsigned long long *vst = reinterpret_cast<unsigned long long *>(bits + ((nwords + 1) & ~1));
    // merge scratch: # re-pushed entries popping before each old queue entry (QB shorts)
    short *mlo = reinterpret_cast<short *>(reinterpret_cast<unsigned char *>(vst) + (SMEM_ST ? (size_t)n * 8 : 0));

    namespace cg = cooperative_groups;
    const unsigned ncl = cg::this_cluster().num_blocks(), crank = cg::this_cluster().block_rank();
    if (crank != 0) {
        cg::this_cluster().sync();   // the leader has initialised its state
        const bool pf = A.prefetch && ncl > 2;
        if (pf && crank == ncl - 1)
            cluster_prefetcher<SMEM_ST>(A, cg::this_cluster().map_shared_rank(buf0, 0),
                                        cg::this_cluster().map_shared_rank(&ctl.sel, 0),
                                        cg::this_cluster().map_shared_rank(&ctl.size, 0),
                                        cg::this_cluster().map_shared_rank(vst, 0),
                                        cg::this_cluster().map_shared_rank(&ctl.bg_stop, 0));
        else
            cluster_helper<SMEM_ST>(A, cg::this_cluster().map_shared_rank(bits, 0),
                                    cg::this_cluster().map_shared_rank(vst, 0),
                                    cg::this_cluster().map_shared_rank(&ctl.bg_stop, 0), (int)crank - 1,
                                    (int)ncl - 1 - (pf ? 1 : 0), tm_smem);
        cg::this_cluster().sync();   // the leader's shared memory stays alive until here
        return;
    }
    for (int i = tid; i < nwords; i += TM_T) bits[i] = 0u;
#if TM_PROFILE
    if (tid < 8) g_tm_prof[tid] = 0ull;
    if (tid < 4) g_rp[tid] = 0ull;
    if (tid == 0) g_mw_round = 0ull;
#endif
    {
        unsigned long long *st0 = SMEM_ST ? vst : A.gvst;
        for (int i = tid; i < n; i += TM_T) st0[i] = 0ull;
    }
    for (int i = tid; i < 3 * n; i += TM_T) A.fv[i] = make_int4(0, 0, 0, 0);
    for (int i = tid; i < TM_RC; i += TM_T) { rcache[i].fid = -1; rc_claim[i] = -1; }
    __syncthreads();
    if (tid == 0) {
        int a = A.clique[0], b = A.clique[1], c = A.clique[2], d = A.clique[3];
        int e0[6][2] = {{a, b}, {a, c}, {a, d}, {b, c}, {b, d}, {c, d}};
        for (int k = 0; k < 6; k++) { A.edges[2 * k] = e0[k][0]; A.edges[2 * k + 1] = e0[k][1]; }
        int fcs[4][3] = {{a, b, c}, {a, b, d}, {a, c, d}, {b, c, d}};
        for (int f = 0; f < 4; f++) {
            A.fv[f] = make_int4(fcs[f][0], fcs[f][1], fcs[f][2], 1);
            ctl.ne_fid[f] = f;
            for (int q = 0; q < 3; q++) ctl.ne_v[f][q] = fcs[f][q];
        }
        bits[a >> 5] |= 1u << (a & 31);
        bits[b >> 5] |= 1u << (b & 31);
        bits[c >> 5] |= 1u << (c & 31);
        bits[d >> 5] |= 1u << (d & 31);
        ctl.size = 0;
        ctl.sel = 0;
        ctl.rem = n - 4;
        ctl.nt = 0;
        ctl.nf = 4;
        ctl.ne_count = (n > 4) ? 4 : 0;
        ctl.L_count = 0;
        ctl.wide = 0;
        ctl.pops = ctl.refreshes = ctl.gain_inc = 0;
        ctl.pool_count = 0;
        ctl.pool_minkey = ~0ull;
        ctl.pool_has_max = 0;
        ctl.done = (n <= 4);
        ctl.bad = 0;
        ctl.bg_stop = 0;
        ctl.t_par = ctl.t_replay = ctl.t_merge = ctl.t_insert = ctl.t_refill = ctl.t_tail = ctl.rounds = ctl.refills = 0;
        ctl.it_round_max = 0;
        for (int q = 0; q < 4; q++) { ctl.ph[q] = 0; ctl.phs[q] = 0; }
        ctl.pops_dbg = 0;
        ctl.rf_t[0] = ctl.rf_t[1] = ctl.rf_t[2] = ctl.rf_t[3] = 0;
        ctl.rc_hit = 0;
        ctl.it_total = ctl.it_maxsum = 0;
    }
    __syncthreads();
    if (ncl > 1) cg::this_cluster().sync();

    if (warp < TM_BG_WARPS) {
        // with helper CTAs the background warps stay idle (the helpers keep the states)
        if (ncl == 1)
        // ============ background: keep every vertex's cached max-corr fresh so the
        // foreground refreshes rarely scan (cursor / max-corr writes are monotone
        // facts -- "all ids before the cursor are inserted" -- valid in any order).
        // Background warps have the LOWEST ids: the scheduler favours high warp ids,
        // so the latency-critical foreground (replay on warp 31) keeps priority.
        bg_sweep<SMEM_ST>(A, bits, vst, &ctl.bg_stop, warp);
    } else {
    // foreground numbering: warp 31 is foreground warp 0 (replay, insertion, leader)
    const int warp = (TM_WARPS - 1) - (threadIdx.x >> 5);
    const int tid = warp * 32 + lane;
#if TM_PROFILE
    long long tc0 = clock64(), tc1;   // round-level phase clocks (profile build only)
#endif
    int sel = 0;   // which half of the queue buffer is current (tracked by every foreground thread)
    while (!ctl.done) {
        const int Lc_round = ctl.L_count, size_round = ctl.size;   // stable until the merge
        if (tid == 0) {
#if TM_PROFILE
            tc0 = clock64();
#endif
            ctl.rounds++;
        }
        // ================= parallel phase: new-face entries + speculative refresh of the top-K
        int my_iters[4] = {0, 0, 0, 0};
#if TM_PROFILE
        long long tpw0 = clock64();
#endif
        {
            Ent *cur = sel ? buf1 : buf0;
            if (warp < TM_NEW_WARPS) {
                if (warp < ctl.ne_count) {
                    const int na = ctl.ne_v[warp][0], nb_ = ctl.ne_v[warp][1], nc = ctl.ne_v[warp][2], nfid = ctl.ne_fid[warp];
                    if (A.check || !warp_entry_fast<SMEM_ST>(A, bits, vst, na, nb_, nc, nfid, &NE[warp], nullptr)) {
                        int fids[1] = {nfid};
                        int fvv[1][3] = {{na, nb_, nc}};
                        warp_entries<SMEM_ST>(A, bits, vst, 1, fvv, fids, &NE[warp], my_iters, nullptr);
                    }
                }
            } else {
                // window warp j serves queue positions j and j + TM_CH (one per half-warp) on the lean
                // path; what needs a scan (or check_invariants mode) goes through warp_entries
                const int j0 = warp - TM_NEW_WARPS;
                const int cntL = ctl.L_count;
#pragma unroll
                for (int ps = 0; ps < KM / TM_K; ps++) {   // one pass; TM_PASSES in a wide round
                const int j = j0 + ps * TM_K;
                if (j >= cntL) break;
                unsigned todo = 0u;
                if (A.check) {
                    todo = (j < cntL ? 1u : 0u) | ((TM_WPE > 1 && j + TM_CH < cntL) ? 2u : 0u);
                } else if (j < cntL) {
                    if (TM_WPE == 2)
                        todo = window_refresh2<SMEM_ST>(A, bits, vst, rcache, cur, j, cntL, Lref, Lstale, Lcomp, Lmc,
                                                        &ctl.rc_hit);
                    else
                        todo = window_refresh<SMEM_ST>(A, bits, vst, rcache, cur + j, j, Lref, Lstale, Lcomp, Lmc,
                                                       my_iters, &ctl.rc_hit) ? 0u : 1u;
                }
                for (int hh = 0; hh < TM_WPE; hh++) {
                    if (!((todo >> hh) & 1u)) continue;
                    const int i = j + hh * TM_CH;
                    const Ent h = cur[i];
                    const bool stale = is_ins(bits, h.cand);
                    // refresh cache (written only between rounds, so this read is stable):
                    // a refreshed entry stays exact while its three max-corr candidates
                    // are still uninserted (each is a monotone fact).  Decided on lane 0.
                    int hit = 0;
                    if (lane == 0) {
                        Lstale[i] = stale;
                        Lcomp[i] = 0;
                        if (stale && !A.check) {
                            const RcEnt &rc = rcache[h.fid & (TM_RC - 1)];
                            if (rc.fid == h.fid && rc.m[0] >= 0 && rc.m[1] >= 0 && rc.m[2] >= 0 &&
                                !is_ins(bits, rc.m[0]) && !is_ins(bits, rc.m[1]) && !is_ins(bits, rc.m[2])) {
                                Ent x = h;
                                x.g = rc.g;
                                x.cand = rc.cand;
                                x.opt = 0;
                                Lref[i] = x;
                                hit = 1;
#if TM_PROFILE
                                atomicAdd(&ctl.rc_hit, 1u);
#endif
                            }
                        }
                    }
                    hit = __shfl_sync(0xffffffffu, hit, 0);
                    if (stale && !hit) {
                        int fids[1] = {h.fid};
                        int fvv[1][3] = {{h.a, h.b, h.c}};
                        // the refreshed entry and its max-corrs straight into the window arrays
                        warp_entries<SMEM_ST>(A, bits, vst, 1, fvv, fids, &Lref[i], my_iters, Lmc[i]);
                        if (lane == 0) Lcomp[i] = 1;
                    }
                }
                }
            }
        }
#if TM_PROFILE
        if (lane == 0 && my_iters[0]) atomicMax(&ctl.it_round_max, my_iters[0]);
        if (lane == 0) {
            const int tw = (int)(clock64() - tpw0);
            atomicMax(&ctl.ph[warp < TM_NEW_WARPS ? 1 : 2], tw);
            atomicMax(&ctl.ph[3], my_iters[3]);
            atomicMax(&ctl.ph[0], tw);
        }
#endif
#if TM_PROFILE
        tc1 = fg_sync_clock();
        if (tid == 0) {
            ctl.t_par += tc1 - tc0;
            tc0 = tc1;
        }
#else
        fg_sync();
#endif
        // ================= replay the pops (warp 0, exact sequential semantics)
        // Warps 0..MW-1 replay, publish and merge (named barrier 2 between
        // replay and merge); the other foreground warps meanwhile refresh the queue
        // entries just past the window (the likely stale head of the next round) into
        // the refresh cache, and only meet the others at the end of the round.  Nobody
        // reads the cache before then; two writers of one slot in a round would tear
        // it, so the first to claim a slot writes it.  The winner's bit is set while
        // the speculative refreshes run: they stay exact (every fact they use is
        // monotone) and the cache's candidate check rejects what the winner voids.
        if (warp == 0) replay_warp(A, ctl, sel ? buf1 : buf0, Lref, Lstale, NE, tobuf, rk_g, rk_f, rk_src, tk_g, tk_f);
        else if (!A.check && (warp == 1 || warp >= MW)) {
            const int round = (int)ctl.rounds;
            if (warp == 1) {
                for (int i0 = 0; i0 < ctl.L_count; i0 += 32) {
                    const int i = i0 + lane;
                    if (i < ctl.L_count && Lcomp[i]) {
                        const Ent &x = Lref[i];
                        const int slot = x.fid & (TM_RC - 1);
                        if (atomicExch(&rc_claim[slot], round) != round) {
                            RcEnt &rc = rcache[slot];
                            rc.g = x.g;
                            rc.fid = x.fid;
                            rc.cand = x.cand;
                            rc.m[0] = Lmc[i][0];
                            rc.m[1] = Lmc[i][1];
                            rc.m[2] = Lmc[i][2];
                        }
                    }
                }
            } else {
                const int pos = Lc_round + (warp - MW);
                const Ent *curb = sel ? buf1 : buf0;
                if (pos < size_round) {
                    const Ent h = curb[pos];
                    int need = 0;
                    if (lane == 0) {
                        need = is_ins(bits, h.cand);
                        if (need) {
                            const RcEnt &rc = rcache[h.fid & (TM_RC - 1)];
                            if (rc.fid == h.fid && rc.m[0] >= 0 && rc.m[1] >= 0 && rc.m[2] >= 0 &&
                                !is_ins(bits, rc.m[0]) && !is_ins(bits, rc.m[1]) && !is_ins(bits, rc.m[2]))
                                need = 0;
                        }
                    }
                    if (__shfl_sync(0xffffffffu, need, 0)) {
                        int fids[1] = {h.fid};
                        int fvv[1][3] = {{h.a, h.b, h.c}};
                        int its[4] = {0, 0, 0, 0};
                        Ent *o = &Lout[warp - MW][0];
                        warp_entries<SMEM_ST>(A, bits, vst, 1, fvv, fids, o, its, nullptr);
                        const int *mcs = &g_went[threadIdx.x >> 5][3 * TM_EPW];
                        if (lane == 0) {
                            const int slot = h.fid & (TM_RC - 1);
                            if (atomicExch(&rc_claim[slot], round) != round) {
                                RcEnt &rc = rcache[slot];
                                rc.g = o->g;
                                rc.fid = o->fid;
                                rc.cand = o->cand;
                                rc.m[0] = mcs[0];
                                rc.m[1] = mcs[1];
                                rc.m[2] = mcs[2];
                            }
#if TM_PROFILE
                            atomicAdd(&g_tm_prof[7], 1ull);
#endif
                        }
                    }
                }
            }
        }
        if (warp < MW) {
        asm volatile("bar.sync 2, %0;" ::"r"(MW * 32) : "memory");
#if TM_PROFILE
        tc1 = clock64();
        if (tid == 0) {
            ctl.t_replay += tc1 - tc0;
            tc0 = tc1;
            ctl.it_maxsum += ctl.it_round_max;
            ctl.it_total += ctl.it_round_max ? 1 : 0;
            ctl.it_round_max = 0;
            for (int q = 0; q < 4; q++) { ctl.phs[q] += ctl.ph[q]; ctl.ph[q] = 0; }
        }
#endif
        // ================= merge buffer[removed..size) + tobuf -> other half (warps 1..),
        // while thread 0 inserts the winner and settles the queue size: both only
        // depend on the replay's results, so one barrier closes the round
        {
            const int r = ctl.removed, sz = ctl.size, nb = ctl.nbuf_new, pc0 = ctl.pool_count;
            // thread 0 rewrites ctl.size / sel / L_count / pool_count below: every merge warp has its copy first
            asm volatile("bar.sync 2, %0;" ::"r"(MW * 32) : "memory");
            if (warp > 0) {
#if TM_PROFILE
                const long long tm0 = clock64();
#endif
                Ent *cur = sel ? buf1 : buf0;
                Ent *nxt = sel ? buf0 : buf1;
                const int old = sz - r;
                const int mt = tid - 32;
                constexpr int MT = MW * 32 - 32;
                // Positions >= QB spill to the pool.  They are the merged sequence's tail, so
                // the spill at position p takes pool slot pc0 + (p - QB): no atomics here
                // (thread 0 settles pool_count and the pool's minimum key, the key of the
                // sequence's last entry); the entry at exactly QB becomes the pool maximum.
                auto place = [&](const Ent &x, int pos) {
                    if (pos < QB) {
                        nxt[pos] = x;
                    } else {
                        const int idx = pc0 + (pos - QB);
                        A.pool_g[idx] = x.g;
                        A.pool_fc[idx] = make_int2(x.fid, x.cand);
                        if (pos == QB) { ctl.pool_max = x; ctl.pool_has_max = 1; }
                    }
                };
                // old entry i -> i + lo_i (lo_i = # re-pushed entries popping before it); the
                // re-pushed entries k in [lo_{i-1}, lo_i) sit right before it, at k + i, and the
                // ones after the last old entry at k + old: one short search per old entry, the
                // lo_i exchanged through shared memory (no search of the long old run)
                for (int i = mt; i < old; i += MT) {
                    Ent x = cur[r + i];
                    int lo = 0, hi = nb;  // # of tobuf entries popping before x
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (kgt(tk_g[mid], tk_f[mid], x.g, x.fid)) lo = mid + 1;
                        else hi = mid;
                    }
                    place(x, i + lo);
                    mlo[i] = (short)lo;
                }
                if (nb > 0) {
                    asm volatile("bar.sync 3, %0;" ::"r"(MT) : "memory");
                    for (int i = mt; i < old; i += MT) {
                        const int lo = mlo[i], lp = i > 0 ? mlo[i - 1] : 0;
                        for (int k = lp; k < lo; k++) place(tobuf[k], k + i);
                        if (i == old - 1)
                            for (int k = lo; k < nb; k++) place(tobuf[k], k + old);
                    }
                    if (old == 0)
                        for (int k = mt; k < nb; k += MT) place(tobuf[k], k);
                }
#if TM_PROFILE
                if (lane == 0) atomicMax(&g_mw_round, (unsigned long long)(clock64() - tm0));
#endif
            } else if (lane == 0) {
#if TM_PROFILE
                long long tin0 = clock64();
#endif
                // spilled entries (total > B) are the smallest of the buffer; then no refill
                const int total = min(sz - r + nb, QB);
                const int spill = sz - r + nb - total;
                if (spill > 0) {
                    // the merged sequence's last entry: the later-popping of the two runs' tails
                    const Ent *curq = sel ? buf1 : buf0;
                    double lg;
                    if (nb == 0) lg = curq[sz - 1].g;
                    else if (sz - r == 0) lg = tobuf[nb - 1].g;
                    else lg = ent_gt(curq[sz - 1], tobuf[nb - 1]) ? tobuf[nb - 1].g : curq[sz - 1].g;
                    const unsigned long long lk = tg_order_key(lg);
                    if (lk < ctl.pool_minkey) ctl.pool_minkey = lk;
                    ctl.pool_count += spill;
                }
                ctl.size = total;
                ctl.sel = sel ^ 1;
                ctl.need_refill = total < TM_K && ctl.pool_count > 0;
                if (KM > TM_K) {
                    ctl.wide = !ctl.winner;
                    ctl.L_count = min(ctl.wide ? KM : TM_K, total);
                } else {
                    ctl.L_count = min(TM_K, total);
                }
                // ================= insert the winner (tmfg.py:94-143 bookkeeping)
                ctl.ne_count = 0;
                if (ctl.winner) {
                    Ent w = ctl.win;
                    int v = w.cand, fid = w.fid;
                    int a = w.a, b = w.b, c = w.c;
                    int t = ctl.nt;
                    A.trace[4 * t] = v;
                    A.trace[4 * t + 1] = a;
                    A.trace[4 * t + 2] = b;
                    A.trace[4 * t + 3] = c;
#if TM_PROFILE && defined(TM_TS)
                    // per-insertion timeline for tools/tmfg_timeline.py: clock (64-cycle units) / rounds / refills / pops
                    A.host_fid[t] = TM_TS == 1 ? (int)(clock64() >> 6) : TM_TS == 2 ? (int)ctl.rounds : TM_TS == 3 ? (int)ctl.refills : (int)ctl.pops;
#else
                    A.host_fid[t] = fid;
#endif
                    int e = 6 + 3 * t;
                    int wv[3] = {a, b, c};
                    for (int q = 0; q < 3; q++) {
                        A.edges[2 * (e + q)] = min(wv[q], v);
                        A.edges[2 * (e + q) + 1] = max(wv[q], v);
                    }
                    A.fv[fid] = make_int4(a, b, c, 0);   // the entry carries the face's sorted vertices
                    int f0 = ctl.nf;
                    int ch[3][3] = {{v, a, b}, {v, a, c}, {v, b, c}};
                    for (int q = 0; q < 3; q++) {
                        int x = ch[q][0], y = ch[q][1], z = ch[q][2];
                        sort3(x, y, z);
                        A.fv[f0 + q] = make_int4(x, y, z, 1);
                        ctl.ne_fid[q] = f0 + q;
                        ctl.ne_v[q][0] = x;
                        ctl.ne_v[q][1] = y;
                        ctl.ne_v[q][2] = z;
                    }
                    ctl.nf = f0 + 3;
                    bits[v >> 5] |= 1u << (v & 31);
                    ctl.nt = t + 1;
                    ctl.rem -= 1;
                    if (ctl.rem == 0) ctl.done = 1;
                    else ctl.ne_count = 3;
                }
                if (ctl.bad) ctl.done = 1;
#if TM_PROFILE
                ctl.t_insert += clock64() - tin0;
#endif
            }
        }
        }
        sel ^= 1;
#if TM_PROFILE
        tc1 = fg_sync_clock();
        if (tid == 0) { ctl.t_merge += tc1 - tc0; tc0 = tc1; g_rp[3] += g_mw_round; g_mw_round = 0; }
#else
        fg_sync();
#endif
        if (ctl.done) break;
        // ================= refill the shared buffer from the pool when short
        if (ctl.need_refill) {
            refill<TM_FG_T, QB>(A, ctl, sel ? buf1 : buf0, sel ? buf0 : buf1, red_e, red_ok, tid);
            if (tid == 0) ctl.L_count = min((KM > TM_K && ctl.wide) ? KM : TM_K, ctl.size);
#if TM_PROFILE
            tc1 = fg_sync_clock();
            if (tid == 0) { ctl.t_refill += tc1 - tc0; tc0 = tc1; }
#else
            fg_sync();
#endif
            if (tid == 0) ctl.refills++;
        }
    }
    fg_sync();
        if (tid == 0) *((volatile int *)&ctl.bg_stop) = 1;
    }
    __syncthreads();
    // ================= alive faces in creation order
    {
        const int nf = ctl.nf;
        __shared__ int wsum[TM_WARPS];
        __shared__ int carry;
        if (tid == 0) carry = 0;
        __syncthreads();
        for (int base = 0; base < nf; base += TM_T) {
            int f = base + tid;
            int4 x = f < nf ? A.fv[f] : make_int4(0, 0, 0, 0);
            int alive = (f < nf) ? x.w : 0;
            unsigned bal = __ballot_sync(0xffffffffu, alive);
            int pre = __popc(bal & ((1u << lane) - 1u));
            if (lane == 0) wsum[warp] = __popc(bal);
            __syncthreads();
            int off = carry;
            for (int w = 0; w < warp; w++) off += wsum[w];
            if (alive) {
                int k = off + pre;
                A.faces[3 * k] = x.x;
                A.faces[3 * k + 1] = x.y;
                A.faces[3 * k + 2] = x.z;
            }
            __syncthreads();
            if (tid == 0) {
                int s = 0;
                for (int w = 0; w < TM_WARPS; w++) s += wsum[w];
                carry += s;
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        A.stats[0] = ctl.pops;
        A.stats[1] = ctl.refreshes;
        A.stats[2] = ctl.gain_inc;
        A.stats[3] = ctl.bad;
        A.stats[7] = ctl.it_total * 100000 + ctl.it_maxsum;
        A.stats[8] = ctl.rounds;
        A.stats[9] = ctl.refills;
        A.stats[10] = ctl.phs[0];   // sum over rounds of the slowest warp's refresh time
        A.stats[11] = ctl.phs[1];   //   ... of the slowest new-face warp
        A.stats[12] = ctl.phs[2];   //   ... of the slowest window-refresh warp
        A.stats[13] = ctl.phs[3];   //   ... of its similarity loads
        A.stats[14] = ctl.t_refill;
        A.stats[15] = ctl.pool_count;
        A.stats[16] = ctl.t_par;
        A.stats[17] = ctl.t_replay;
        A.stats[18] = ctl.t_merge;
        A.stats[19] = ctl.t_insert;
        A.stats[20] = ctl.t_tail;
#if TM_PROFILE
        for (int q = 0; q < 3; q++) A.stats[21 + q] = (long long)g_tm_prof[q];
        A.stats[29] = (long long)g_tm_prof[3];
        A.stats[31] = (long long)(g_tm_prof[5] << 32 | g_tm_prof[6]);   // helper warp-phase vertices, batches
        A.stats[20] = (long long)g_tm_prof[7];
        for (int q = 0; q < 4; q++) A.stats[4 + q] = (long long)g_rp[q];   // (slot 7: it_total overwritten)
#endif
        A.stats[24] = ctl.rf_t[0];
        A.stats[25] = ctl.rf_t[1];
        A.stats[26] = ctl.rf_t[2];
        A.stats[27] = ctl.rf_t[3];
        A.stats[28] = ctl.rc_hit;
    }
    if (ncl > 1) cooperative_groups::this_cluster().sync();   // helpers read this CTA's shared memory until here
}

size_t tm_smem_bytes(int64_t n, bool smem_st) {
    size_t b = (size_t)2 * (smem_st ? tm_qb<true>() : tm_qb<false>()) * sizeof(Ent);
    if (!smem_st) b += (size_t)(2 * tm_kmax<false>() + 8) * sizeof(Ent);   // Lref + tobuf (wide window)
    b += (size_t)(((n + 31) / 32 + 1) & ~1LL) * 4;
    if (smem_st) b += (size_t)n * 8;
    b += (size_t)(smem_st ? tm_qb<true>() : tm_qb<false>()) * sizeof(short);   // merge scratch
    return tg_align_up(b, 16) + 64;
}

__global__ void edge_weights_kernel(const double *__restrict__ S, int64_t n, const int32_t *__restrict__ edges,
                                    int64_t m, double *__restrict__ w) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) w[i] = S[(int64_t)edges[2 * i] * n + edges[2 * i + 1]];
}

}  // namespace

TG_API int tg_edge_weights(const double *S, int64_t n, const int32_t *edges, int64_t m, double *w, void *stream) {
    if (!S || !edges || !w || m < 0) return TG_ERR_ARG;
    if (m == 0) return TG_OK;
    edge_weights_kernel<<<(unsigned)((m + 255) / 256), 256, 0, tg_stream(stream)>>>(S, n, edges, m, w); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API size_t tg_tmfg_workspace_bytes(int64_t n) {
    size_t b = 0;
    b += tg_align_up((size_t)3 * n * sizeof(int4), 256);
    b += tg_align_up((size_t)(3 * n + TM_BMAX + 64) * sizeof(double), 256);
    b += tg_align_up((size_t)(3 * n + TM_BMAX + 64) * sizeof(int2), 256);
    b += tg_align_up((size_t)n * sizeof(unsigned long long), 256);
    return b + 1024;
}

TG_API int tg_tmfg_heap(const double *S, const int32_t *order, int64_t n, const int32_t *clique, int32_t *trace,
                        int32_t *host_fid, int32_t *edges, int32_t *faces, int64_t *stats, int32_t check,
                        void *ws, size_t ws_bytes, void *stream) {
    if (n < 4 || !S || !order || !clique || !edges || !faces || !stats) return TG_ERR_ARG;
    if (ws_bytes < tg_tmfg_workspace_bytes(n)) return TG_ERR_WORKSPACE;
    TgArena ar(ws, ws_bytes);
    TmArgs A;
    A.S = S;
    A.order = order;
    A.n = (int)n;
    A.clique = clique;
    A.trace = trace;
    A.host_fid = host_fid;
    A.edges = edges;
    A.faces = faces;
    A.stats = stats;
    A.check = check;
    A.fv = ar.take<int4>((size_t)3 * n);
    A.pool_g = ar.take<double>((size_t)3 * n + TM_BMAX + 64);
    A.pool_fc = ar.take<int2>((size_t)3 * n + TM_BMAX + 64);
    A.gvst = ar.take<unsigned long long>((size_t)n);
    if (!A.fv || !A.pool_g || !A.pool_fc || !A.gvst) return TG_ERR_WORKSPACE;
    cudaStream_t st = tg_stream(stream);
    if (n >= (1 << 21)) return TG_ERR_ARG;   // scan-state word packs ids in 21 bits
    A.prefetch = 1;
    if (const char *e = std::getenv("TG_TMFG_PREFETCH")) A.prefetch = std::atoi(e);
    // dynamic shared memory budget: the per-block opt-in maximum minus the kernel's static arrays
    // (a fixed 200 KB would overflow the block's 227 KB for n ~ 13k-17k with ~46 KB of static data)
    int dev = 0, optin = 0;
    TG_CUDA_CHECK(cudaGetDevice(&dev));
    TG_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa_st, fa_gl;
    TG_CUDA_CHECK(cudaFuncGetAttributes(&fa_st, tmfg_heap_kernel<true>));
    TG_CUDA_CHECK(cudaFuncGetAttributes(&fa_gl, tmfg_heap_kernel<false>));
    const size_t budget_st = (size_t)optin - fa_st.sharedSizeBytes, budget_gl = (size_t)optin - fa_gl.sharedSizeBytes;
    const bool smem_st = tm_smem_bytes(n, true) <= budget_st;
    const size_t smem_leader = tm_smem_bytes(n, smem_st);
    const size_t budget = smem_st ? budget_st : budget_gl;
    if (smem_leader > budget) return TG_ERR_ARG;
    // a cluster of 1 leader + helper CTAs (TG_TMFG_CLUSTER, default 12: a non-portable size,
    // measured against 8 / 10 / 14 / 16 -- n = 10k 80.3 -> 79.1 ms, n = 50k 518 -> 510.5 ms;
    // 1 disables the helpers); smaller clusters are tried when it cannot be placed
    int ncl = 12;
    if (const char *e = std::getenv("TG_TMFG_CLUSTER")) ncl = std::atoi(e);
    if (ncl < 1) ncl = 1;
    if (ncl > 16) ncl = 16;   // > 8 needs the non-portable cluster size attribute (set below)
    // helpers reuse the dynamic shared memory for a bitmap snapshot + their slice's words
    size_t smem = smem_leader;
    for (; ncl > 1; ncl--) {
        const int vslots = ncl - 1 - ((A.prefetch && ncl > 2) ? 1 : 0);
        const size_t hs = (size_t)((((n + 31) / 32) + 1) & ~1LL) * 4 + (size_t)tm_helper_slice((int)n, vslots) * 8 + 64;
        if (hs <= budget) { smem = std::max(smem_leader, hs); break; }
    }
#define TM_LAUNCH(M)                                                                                      \
    do {                                                                                                  \
        TG_CUDA_CHECK(cudaFuncSetAttribute(tmfg_heap_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)smem));                                                  \
        if (ncl > 8) cudaFuncSetAttribute(tmfg_heap_kernel<M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
        cudaGetLastError();                                                                               \
        cudaLaunchConfig_t cfg = {};                                                                      \
        cudaLaunchAttribute attr[1];                                                                      \
        cfg.blockDim = dim3(TM_T, 1, 1);                                                                  \
        cfg.dynamicSmemBytes = smem;                                                                      \
        cfg.stream = st;                                                                                  \
        attr[0].id = cudaLaunchAttributeClusterDimension;                                                 \
        attr[0].val.clusterDim.y = 1;                                                                     \
        attr[0].val.clusterDim.z = 1;                                                                     \
        cfg.attrs = attr;                                                                                 \
        cfg.numAttrs = 1;                                                                                 \
        int k = ncl;                                                                                      \
        for (; k > 1; k--) {                                                                              \
            cfg.gridDim = dim3(k, 1, 1);                                                                  \
            attr[0].val.clusterDim.x = k;                                                                 \
            int nc = 0;                                                                                   \
            if (cudaOccupancyMaxActiveClusters(&nc, tmfg_heap_kernel<M>, &cfg) == cudaSuccess && nc > 0) break; \
            cudaGetLastError();                                                                           \
        }                                                                                                 \
        cfg.gridDim = dim3(k, 1, 1);                                                                      \
        attr[0].val.clusterDim.x = k;                                                                     \
        TG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, tmfg_heap_kernel<M>, A));                                  \
        tg_count_launch(1);                                                                               \
    } while (0)
    if (smem_st) TM_LAUNCH(true);
    else TM_LAUNCH(false);
#undef TM_LAUNCH
    TG_LAUNCH_CHECK();
    return TG_OK;
}
