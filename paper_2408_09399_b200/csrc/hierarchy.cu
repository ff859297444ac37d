// hierarchy.cu -- DBHT's three-layer complete-linkage hierarchy, native driver.
//
// Replaces dbht.py:233-339 build_hierarchy (+ linkage.py:97-116 canonicalisation
// and linkage.py:136-148 sizes).  The heavy parts stay on the GPU and are the
// kernels behind tg_group_blocks (layer-1 oracle blocks), tg_group_max_batch
// (layer-2/3 pairwise group maxima) and tg_nn_chain_batch (every linkage of a
// layer in one launch); this file is the host bookkeeping between them, in C++:
// grouping vertices by bubble / converging bubble, the stable height sort and
// renumbering of each linkage's merges, the merge records, and the emission
// with the running height floor.  One stream synchronisation per layer.
#include "common.cuh"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <mutex>
#include <vector>
#include <thread>
#include <string>
#include <functional>

// The hierarchy's per-layer buffers come from a pool owned by this library (one per device),
// not from the process-wide default pool: it keeps up to 16 GiB cached between calls (the
// n = 50k layer-3 buffers exceed 1 GiB, and a release threshold of 0 would unmap and remap them
// on every call) without changing the default pool's policy for anyone else.
// tg_release_cached_memory() trims it.
static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64];

static cudaError_t tg_hier_pool(cudaMemPool_t *out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pools[dev]) {
        cudaMemPoolProps props;
        std::memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t pool;
        if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
        uint64_t thr = 16ull << 30;
        if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess) return e;
        g_pools[dev] = pool;
    }
    *out = g_pools[dev];
    return cudaSuccess;
}

namespace {

constexpr double HEIGHT_BUMP = 1e-12;                       // dbht.py HEIGHT_BUMP
constexpr uint64_t NN_CYCLE_SENTINEL = 0x7ff8dead00000000ull;   // tg_nn_chain_batch: chain did not terminate

// stream-ordered device buffer
struct DevBuf {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t s) {
        st = s;
        cudaMemPool_t pool;
        cudaError_t e = tg_hier_pool(&pool);
        if (e != cudaSuccess) return e;
        return cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, pool, s);
    }
    template <class T>
    T *as() const { return reinterpret_cast<T *>(p); }
};

// a non-blocking side stream that starts after everything already queued on `main`
struct SideStream {
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    // priority: 0 = default; the stream's blocks are scheduled first when SMs free up
    cudaError_t open(cudaStream_t main, bool high_priority = false) {
        int lo = 0, hi = 0;
        if (high_priority) cudaDeviceGetStreamPriorityRange(&lo, &hi);
        cudaError_t e = cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, high_priority ? hi : 0);
        if (e != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev, main)) != cudaSuccess) return e;
        return cudaStreamWaitEvent(st, ev, 0);
    }
    ~SideStream() {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        if (ev) cudaEventDestroy(ev);
    }
};

static const bool g_hprof = std::getenv("TG_HIER_PROFILE") != nullptr;
static std::chrono::steady_clock::time_point g_hprof_t;
#define HPROF(name)                                                                                      \
    do {                                                                                                 \
        if (g_hprof) {                                                                                   \
            auto _t = std::chrono::steady_clock::now();                                                  \
            if (std::strcmp(name, "t0")) std::fprintf(stderr, "[hier] %s +%.3f ms\n", name,                \
                                        std::chrono::duration<double, std::milli>(_t - g_hprof_t).count()); \
            g_hprof_t = _t;                                                                              \
        }                                                                                                \
    } while (0)

struct Rec {
    int64_t l, r;
    double h;
};
// a vertex group: a run of a flat member array (ascending vertex ids)
struct Span {
    const int32_t *p;
    int64_t len;
    int64_t size() const { return len; }
    const int32_t *begin() const { return p; }
    const int32_t *end() const { return p + len; }
    int32_t operator[](int64_t i) const { return p[i]; }
};
struct Row {
    int64_t handle;
    double h;
};

struct Ctx {
    int64_t n;
    const tg_oracle_t *oracle;
    cudaStream_t st;
    std::vector<Rec> records;
};

#define HC(expr)                                          \
    do {                                                  \
        cudaError_t _e = (expr);                          \
        if (_e != cudaSuccess) {                          \
            tg_set_last_error(_e, __FILE__, __LINE__);    \
            return TG_ERR_CUDA;                           \
        }                                                 \
    } while (0)
#define HR(expr)                   \
    do {                           \
        int _r = (expr);           \
        if (_r != TG_OK) return _r; \
    } while (0)

// A batch of linkages in flight on one stream: the NN-chain of every matrix runs on the
// device (in place); collect() waits, canonicalises (stable height sort, renumbering) and
// appends the records.  Launch and collect are split so that two layers' device work can
// overlap (layers 2 and 3 are independent until their records are labelled).
struct LinkJob {
    cudaStream_t st = nullptr;
    DevBuf gm_buf, nn_buf;   // group-max inputs / output matrices, NN-chain outputs / scratch
    std::vector<int64_t> sizes, mat_off, merge_off;
    int64_t total = 0;
    int64_t *d_l = nullptr, *d_r = nullptr;
    double *d_h = nullptr;
};

int launch_linkages(Ctx &cx, LinkJob &job, double *mats_dev) {
    const size_t count = job.sizes.size();
    job.merge_off.assign(count + 1, 0);
    std::vector<int64_t> aux_off(count + 1, 0);
    for (size_t k = 0; k < count; k++) {
        job.merge_off[k + 1] = job.merge_off[k] + std::max<int64_t>(job.sizes[k] - 1, 0);
        aux_off[k + 1] = aux_off[k] + job.sizes[k];
    }
    job.total = job.merge_off[count];
    const int64_t naux = aux_off[count];
    if (job.total == 0) return TG_OK;
    // one device block: [mat_off | sizes | merge_off | aux_off] int64, then outputs / scratch
    const size_t nidx = 4 * (count + 1);
    const size_t b_idx = tg_align_up(nidx * 8, 256), b_l = tg_align_up((size_t)job.total * 8, 256);
    const size_t b_h = b_l, b_slot = tg_align_up((size_t)naux * 8, 256), b_chain = tg_align_up((size_t)(naux + 1) * 8, 256);
    const size_t b_act = tg_align_up((size_t)naux, 256);
    HC(job.nn_buf.alloc(b_idx + 2 * b_l + b_h + b_slot + b_chain + b_act, job.st));
    char *base = job.nn_buf.as<char>();
    int64_t *d_idx = reinterpret_cast<int64_t *>(base);
    job.d_l = reinterpret_cast<int64_t *>(base + b_idx);
    job.d_r = reinterpret_cast<int64_t *>(base + b_idx + b_l);
    job.d_h = reinterpret_cast<double *>(base + b_idx + 2 * b_l);
    int64_t *d_slot = reinterpret_cast<int64_t *>(base + b_idx + 2 * b_l + b_h);
    int64_t *d_chain = reinterpret_cast<int64_t *>(base + b_idx + 2 * b_l + b_h + b_slot);
    uint8_t *d_act = reinterpret_cast<uint8_t *>(base + b_idx + 2 * b_l + b_h + b_slot + b_chain);
    std::vector<int64_t> idx(nidx, 0);
    std::copy(job.mat_off.begin(), job.mat_off.end(), idx.begin());
    std::copy(job.sizes.begin(), job.sizes.end(), idx.begin() + (count + 1));
    std::copy(job.merge_off.begin(), job.merge_off.end(), idx.begin() + 2 * (count + 1));
    std::copy(aux_off.begin(), aux_off.end(), idx.begin() + 3 * (count + 1));
    HC(cudaMemcpyAsync(d_idx, idx.data(), nidx * 8, cudaMemcpyHostToDevice, job.st));
    HR(tg_nn_chain_batch(mats_dev, d_idx, d_idx + (count + 1), (int64_t)count, d_idx + 2 * (count + 1), job.d_l,
                         job.d_r, job.d_h, d_idx + 3 * (count + 1), d_act, d_slot, d_chain, job.st));
    return TG_OK;
}

int collect_linkages(Ctx &cx, LinkJob &job, const std::vector<std::vector<int64_t>> &handles,
                     std::vector<int64_t> &roots, std::vector<Row> &rows_out) {
    const size_t count = job.sizes.size();
    roots.assign(count, -1);
    const int64_t total = job.total;
    if (total == 0) {
        for (size_t k = 0; k < count; k++) roots[k] = handles[k][0];
        return TG_OK;
    }
    HC(cudaStreamSynchronize(job.st));
    std::vector<int64_t> L(total), R(total);
    std::vector<double> Hh(total);
    // on the job's own stream: a legacy-stream cudaMemcpy would also wait for the other layers
    HC(cudaMemcpyAsync(L.data(), job.d_l, total * 8, cudaMemcpyDeviceToHost, job.st));
    HC(cudaMemcpyAsync(R.data(), job.d_r, total * 8, cudaMemcpyDeviceToHost, job.st));
    HC(cudaMemcpyAsync(Hh.data(), job.d_h, total * 8, cudaMemcpyDeviceToHost, job.st));
    HC(cudaStreamSynchronize(job.st));
    for (int64_t q = 0; q < total; q++) {
        uint64_t bits;
        std::memcpy(&bits, &Hh[q], 8);
        if (bits == NN_CYCLE_SENTINEL) return TG_ERR_NOT_REDUCIBLE;
    }
    std::vector<int64_t> ord, rank, local;
    for (size_t k = 0; k < count; k++) {
        const int64_t m = job.sizes[k], lo = job.merge_off[k], nm = job.merge_off[k + 1] - lo;
        // linkage.py:97-116: stable sort of the raw merges by height, id m+t -> m+rank(t)
        ord.resize(nm);
        for (int64_t t = 0; t < nm; t++) ord[t] = t;
        std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return Hh[lo + a] < Hh[lo + b]; });
        rank.resize(nm);
        for (int64_t q = 0; q < nm; q++) rank[ord[q]] = q;
        local.assign(handles[k].begin(), handles[k].end());
        int64_t root = handles[k][0];
        for (int64_t q = 0; q < nm; q++) {
            const int64_t t = ord[q];
            int64_t a = L[lo + t], b = R[lo + t];
            if (a >= m) a = m + rank[a - m];
            if (b >= m) b = m + rank[b - m];
            const int64_t lo_id = std::min(a, b), hi_id = std::max(a, b);
            const double h = Hh[lo + t];
            const int64_t rec = cx.n + (int64_t)cx.records.size();
            cx.records.push_back({local[lo_id], local[hi_id], h});
            local.push_back(rec);
            rows_out.push_back({rec, h});
            root = rec;
        }
        roots[k] = root;
    }
    return TG_OK;
}

// dbht.py:217-230 group maxima for vertex-disjoint sub-problems (one launch) on job.st, then
// the linkages (launched; collect_linkages finishes them)
int launch_group_linkages(Ctx &cx, LinkJob &job, const std::vector<std::vector<Span>> &subproblems) {
    std::vector<int32_t> perm, gid;
    std::vector<tg_gm_sub_t> subs;
    int64_t out_off = 0, total_len = 0, total_tiles = 0;
    for (const auto &groups : subproblems) {
        int64_t len = 0;
        for (const auto &g : groups) len += g.size();
        total_len += len;
        total_tiles += ((len + 63) / 64) * ((len + 63) / 64);
    }
    perm.reserve(total_len);
    gid.reserve(total_len);
    // the tile list (n = 50k layer 3: 611k tiles, 7 MB) is built on the device from subs
    int64_t tile_off = 0;
    for (size_t p = 0; p < subproblems.size(); p++) {
        const auto &groups = subproblems[p];
        const int64_t perm_off = (int64_t)perm.size();
        for (size_t g = 0; g < groups.size(); g++) {
            perm.insert(perm.end(), groups[g].begin(), groups[g].end());
            gid.insert(gid.end(), (size_t)groups[g].size(), (int32_t)g);
        }
        const int32_t len = (int32_t)(perm.size() - perm_off), m = (int32_t)groups.size();
        tg_gm_sub_t sd;
        sd.perm_off = perm_off;
        sd.len = len;
        sd.m = m;
        sd.out_off = out_off;
        sd.tile_off = tile_off;
        subs.push_back(sd);
        tile_off += (int64_t)((len + 63) / 64) * ((len + 63) / 64);
        job.sizes.push_back(m);
        job.mat_off.push_back(out_off);
        out_off += (int64_t)m * m;
    }
    HPROF("gl_host");
    const int64_t ntiles = total_tiles;
    const size_t ws_bytes = tg_group_max_workspace_bytes(cx.n, ntiles, cx.oracle->mode == 1 ? cx.oracle->H : 0);
    const size_t b_perm = tg_align_up(perm.size() * 4, 256), b_sub = tg_align_up(subs.size() * sizeof(tg_gm_sub_t), 256);
    const size_t b_tile = tg_align_up((size_t)ntiles * sizeof(tg_gm_tile_t), 256);
    const size_t b_out = tg_align_up((size_t)std::max<int64_t>(out_off, 1) * 8, 256);
    HC(job.gm_buf.alloc(2 * b_perm + b_sub + b_tile + b_out + ws_bytes, job.st));
    HPROF("gl_alloc");
    char *base = job.gm_buf.as<char>();
    int32_t *d_perm = reinterpret_cast<int32_t *>(base);
    int32_t *d_gid = reinterpret_cast<int32_t *>(base + b_perm);
    void *d_sub = base + 2 * b_perm;
    void *d_tile = base + 2 * b_perm + b_sub;
    double *d_out = reinterpret_cast<double *>(base + 2 * b_perm + b_sub + b_tile);
    void *d_ws = base + 2 * b_perm + b_sub + b_tile + b_out;
    HC(cudaMemcpyAsync(d_perm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, job.st));
    HC(cudaMemcpyAsync(d_gid, gid.data(), gid.size() * 4, cudaMemcpyHostToDevice, job.st));
    HC(cudaMemcpyAsync(d_sub, subs.data(), subs.size() * sizeof(tg_gm_sub_t), cudaMemcpyHostToDevice, job.st));
    HR(tg_group_tiles_fill(d_sub, (int64_t)subs.size(), d_tile, ntiles, job.st));
    HPROF("gl_h2d");
    HR(tg_group_max_batch(cx.oracle, d_perm, d_gid, (int64_t)perm.size(), d_sub, (int64_t)subs.size(), d_tile, ntiles,
                          d_out, out_off, d_ws, ws_bytes, job.st));
    HPROF("gl_gm");
    return launch_linkages(cx, job, d_out);
}

void stable_sort_rows(std::vector<Row> &rows) {
    std::stable_sort(rows.begin(), rows.end(), [](const Row &a, const Row &b) { return a.h < b.h; });
}

int build(Ctx &cx, const int64_t *vb_dev, const int64_t *vc_dev, int64_t *lefts, int64_t *rights, double *heights,
          int64_t *sizes_out, int64_t *n_merges) {
    const int64_t n = cx.n;
    std::vector<int64_t> vb(n), vc(n);
    HPROF("t0");
    HC(cudaMemcpyAsync(vb.data(), vb_dev, n * 8, cudaMemcpyDeviceToHost, cx.st));
    HC(cudaMemcpyAsync(vc.data(), vc_dev, n * 8, cudaMemcpyDeviceToHost, cx.st));
    HC(cudaStreamSynchronize(cx.st));
    int64_t nb = 0;
    for (int64_t v = 0; v < n; v++) {
        if (vb[v] < 0) return TG_ERR_ARG;
        nb = std::max(nb, vb[v] + 1);
    }
    // vertices by (bubble, id): a counting sort into one flat array, members[b] ascending
    std::vector<int64_t> moff(nb + 1, 0);
    for (int64_t v = 0; v < n; v++) moff[vb[v] + 1]++;
    for (int64_t b = 0; b < nb; b++) moff[b + 1] += moff[b];
    std::vector<int32_t> mflat(n);
    {
        std::vector<int64_t> fill(moff.begin(), moff.end() - 1);
        for (int64_t v = 0; v < n; v++) mflat[fill[vb[v]]++] = (int32_t)v;
    }
    std::vector<Span> members(nb);
    for (int64_t b = 0; b < nb; b++) members[b] = Span{mflat.data() + moff[b], moff[b + 1] - moff[b]};
    std::vector<int64_t> bubble_ids;
    for (int64_t b = 0; b < nb; b++)
        if (members[b].size() > 0) bubble_ids.push_back(b);
    std::vector<int64_t> group_root(nb, -1);

    // All three layers' device work is independent: layer 1 (bubble groups) reads oracle
    // blocks, layers 2 and 3 read group maxima of the same oracle; only the record labels
    // chain them (layer 2's handles are layer 1's roots, layer 3's are layer 2's).  So layer 3
    // is launched on one side stream, layer 2 on the caller's stream and layer 1 on another
    // side stream, and they are collected in layer order (record numbering unchanged).
    std::vector<Row> rows1, rows2, rows3;
    SideStream side1, side3;   // destroyed after the jobs / buffers that free on them
    std::vector<int64_t> multi;
    for (int64_t b : bubble_ids) {
        if (members[b].size() > 1) multi.push_back(b);
        else group_root[b] = members[b][0];
    }
    DevBuf blocks_buf;
    LinkJob j1, j2, j3;
    static const bool l1_serial = std::getenv("TG_HIER_SERIAL") != nullptr;   // A/B switch
    std::vector<std::vector<int64_t>> handles1(multi.size());
    // fork layer 1's stream BEFORE anything of layers 2/3 is queued on cx.st: its event then
    // covers only the work that produced the assignment, so layer 1 never waits for layer 2
    if (!multi.empty()) HC(side1.open(cx.st));
    HPROF("tL1");
    // ---- layers 2 (bubbles inside each converging group, dbht.py:264-300) and 3 (converging
    // groups against each other, dbht.py:302-324)
    std::vector<int64_t> conv_ids;
    std::vector<std::vector<int64_t>> conv_bubbles;   // parallel to conv_ids
    std::vector<int64_t> conv_root;
    std::vector<std::vector<Span>> subproblems;
    std::vector<size_t> which;
    {
        // bubbles grouped by converging id (ascending), bubble order inside: a stable counting
        // sort (converging ids are bubble indices)
        int64_t ncv = 0;
        for (int64_t b : bubble_ids) ncv = std::max(ncv, vc[members[b][0]] + 1);
        std::vector<int64_t> cnt(ncv, 0);
        for (int64_t b : bubble_ids) cnt[vc[members[b][0]]]++;
        std::vector<int64_t> slot_of(ncv, -1);
        for (int64_t c = 0; c < ncv; c++)
            if (cnt[c] > 0) {
                slot_of[c] = (int64_t)conv_ids.size();
                conv_ids.push_back(c);
            }
        conv_bubbles.resize(conv_ids.size());
        for (size_t c = 0; c < conv_ids.size(); c++) conv_bubbles[c].reserve((size_t)cnt[conv_ids[c]]);
        for (int64_t b : bubble_ids) conv_bubbles[slot_of[vc[members[b][0]]]].push_back(b);
        conv_root.assign(conv_ids.size(), -1);
        for (size_t c = 0; c < conv_ids.size(); c++) {
            if (conv_bubbles[c].size() == 1) continue;
            std::vector<Span> groups;
            groups.reserve(conv_bubbles[c].size());
            for (int64_t b : conv_bubbles[c]) groups.push_back(members[b]);
            subproblems.push_back(std::move(groups));
            which.push_back(c);
        }
    }
    const bool layer3 = conv_ids.size() > 1;
    std::vector<int32_t> cflat;
    std::vector<Span> groups3;
    if (layer3) {
        // group c's vertices = the union of its bubbles' members, ascending: a counting sort of
        // the vertices (in id order) by group into one flat array
        const size_t ng = conv_ids.size();
        std::vector<int32_t> conv_of_bubble(nb, -1);
        std::vector<int64_t> coff(ng + 1, 0);
        for (size_t c = 0; c < ng; c++)
            for (int64_t b : conv_bubbles[c]) {
                conv_of_bubble[b] = (int32_t)c;
                coff[c + 1] += members[b].size();
            }
        for (size_t c = 0; c < ng; c++) coff[c + 1] += coff[c];
        cflat.resize((size_t)n);
        std::vector<int64_t> fill(coff.begin(), coff.end() - 1);
        for (int64_t v = 0; v < n; v++) cflat[fill[conv_of_bubble[vb[v]]]++] = (int32_t)v;
        groups3.reserve(ng);
        for (size_t c = 0; c < ng; c++) groups3.push_back(Span{cflat.data() + coff[c], coff[c + 1] - coff[c]});
        HPROF("cmem");
        // the side stream forks from the caller's stream here, before any layer is queued on it
        HC(side3.open(cx.st, true));
        HPROF("open3");
        j3.st = side3.st;
    }
    // The layer with the largest matrix is the critical path (its NN-chain is serial in the
    // matrix size): layer 3 at n = 50k (one 5,906-group matrix), layer 2 at n = 10k (1,056 groups
    // against a few hundred converging groups).  Its group maxima are queued first, so its chain
    // starts before the other layer's group maxima occupy the GPU.
    size_t m2max = 0;
    for (const auto &sp : subproblems) m2max = std::max(m2max, sp.size());
    const bool l3_first = layer3 && conv_ids.size() >= m2max;
    if (layer3 && l3_first) HR(launch_group_linkages(cx, j3, {groups3}));
    HPROF("tL3");
    j2.st = cx.st;
    if (!subproblems.empty()) HR(launch_group_linkages(cx, j2, subproblems));
    if (layer3 && !l3_first) HR(launch_group_linkages(cx, j3, {groups3}));
    // layer 1 last: its linkages are never the critical path (layer 2 is at n = 10k, layer 3
    // at n = 50k), so its host preparation overlaps their device work
    if (!multi.empty()) {   // ---- layer 1: complete linkage inside every bubble group (dbht.py:247-262)
        j1.st = side1.st;
        const size_t cnt = multi.size();
        std::vector<int32_t> perm;
        std::vector<int64_t> gst(cnt + 1, 0), boff(cnt + 1, 0);
        for (size_t k = 0; k < cnt; k++) {
            const auto &mem = members[multi[k]];
            const int64_t s = (int64_t)mem.size();
            perm.insert(perm.end(), mem.begin(), mem.end());
            gst[k + 1] = gst[k] + s;
            boff[k + 1] = boff[k] + s * s;
            j1.sizes.push_back(s);
            j1.mat_off.push_back(boff[k]);
            handles1[k].assign(mem.begin(), mem.end());
        }
        const size_t b_perm = tg_align_up(perm.size() * 4, 256), b_idx = tg_align_up((cnt + 1) * 8, 256);
        HC(blocks_buf.alloc(b_perm + 2 * b_idx + (size_t)boff[cnt] * 8, j1.st));
        char *base = blocks_buf.as<char>();
        int32_t *d_perm = reinterpret_cast<int32_t *>(base);
        int64_t *d_gst = reinterpret_cast<int64_t *>(base + b_perm);
        int64_t *d_boff = reinterpret_cast<int64_t *>(base + b_perm + b_idx);
        double *d_blocks = reinterpret_cast<double *>(base + b_perm + 2 * b_idx);
        HC(cudaMemcpyAsync(d_perm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, j1.st));
        HC(cudaMemcpyAsync(d_gst, gst.data(), (cnt + 1) * 8, cudaMemcpyHostToDevice, j1.st));
        HC(cudaMemcpyAsync(d_boff, boff.data(), (cnt + 1) * 8, cudaMemcpyHostToDevice, j1.st));
        HR(tg_group_blocks(cx.oracle, d_perm, d_gst, (int64_t)cnt, d_boff, d_blocks, j1.st));
        HR(launch_linkages(cx, j1, d_blocks));
        if (l1_serial) {
            std::vector<int64_t> roots;
            HR(collect_linkages(cx, j1, handles1, roots, rows1));
            for (size_t k = 0; k < multi.size(); k++) group_root[multi[k]] = roots[k];
        }
    }


    if (!multi.empty() && !l1_serial) {
        std::vector<int64_t> roots;
        HR(collect_linkages(cx, j1, handles1, roots, rows1));
        for (size_t k = 0; k < multi.size(); k++) group_root[multi[k]] = roots[k];
    }
    HPROF("tC1");
    stable_sort_rows(rows1);
    for (size_t c = 0; c < conv_ids.size(); c++)
        if (conv_bubbles[c].size() == 1) conv_root[c] = group_root[conv_bubbles[c][0]];
    if (!subproblems.empty()) {
        std::vector<std::vector<int64_t>> handles2;
        for (size_t c : which) {
            std::vector<int64_t> hs;
            for (int64_t b : conv_bubbles[c]) hs.push_back(group_root[b]);
            handles2.push_back(std::move(hs));
        }
        std::vector<int64_t> roots;
        HR(collect_linkages(cx, j2, handles2, roots, rows2));
        for (size_t k = 0; k < which.size(); k++) conv_root[which[k]] = roots[k];
    }
    HPROF("tC2");
    stable_sort_rows(rows2);
    if (layer3) {
        std::vector<int64_t> hs, roots;
        for (size_t c = 0; c < conv_ids.size(); c++) hs.push_back(conv_root[c]);
        HR(collect_linkages(cx, j3, {hs}, roots, rows3));
        stable_sort_rows(rows3);
    }

    HPROF("tC3");
    // ---- emission with the running height floor (dbht.py:326-339) + sizes (linkage.py:136-148)
    const int64_t nrec = (int64_t)cx.records.size();
    std::vector<int64_t> final_id(n + nrec);
    for (int64_t i = 0; i < n + nrec; i++) final_id[i] = i;
    std::vector<int64_t> size_of(n + nrec, 1);
    double floor_h = -INFINITY;
    int64_t k = 0;
    for (const std::vector<Row> *rows : {&rows1, &rows2, &rows3}) {
        for (const Row &row : *rows) {
            const Rec &rc = cx.records[row.handle - n];
            double h = rc.h;
            if (h < floor_h) h = floor_h + HEIGHT_BUMP;
            floor_h = h;
            const int64_t li = final_id[rc.l], ri = final_id[rc.r];
            final_id[row.handle] = n + k;
            if (k >= n - 1) return TG_ERR_ARG;   // more merges than a binary tree over n leaves has
            lefts[k] = std::min(li, ri);
            rights[k] = std::max(li, ri);
            heights[k] = h;
            const int64_t s = size_of[lefts[k]] + size_of[rights[k]];
            size_of[n + k] = s;
            sizes_out[k] = s;
            k++;
        }
    }
    *n_merges = k;
    HPROF("emit");
    return TG_OK;
}

}  // namespace

TG_API int tg_build_hierarchy(const tg_oracle_t *oracle, const int64_t *vertex_bubble, const int64_t *vertex_converging,
                              int64_t n, int64_t *lefts_out, int64_t *rights_out, double *heights_out,
                              int64_t *sizes_out, int64_t *n_merges_out, void *stream) {
    if (!oracle || !vertex_bubble || !vertex_converging || !n_merges_out || n < 1) return TG_ERR_ARG;
    if (n > 1 && (!lefts_out || !rights_out || !heights_out || !sizes_out)) return TG_ERR_ARG;
    *n_merges_out = 0;
    Ctx cx;
    cx.n = n;
    cx.oracle = oracle;
    cx.st = tg_stream(stream);
    try {
        return build(cx, vertex_bubble, vertex_converging, lefts_out, rights_out, heights_out, sizes_out,
                     n_merges_out);
    } catch (...) {   // std::bad_alloc: no C++ exception crosses the ABI
        return TG_ERR_ARG;
    }
}

// linkage.py:181-187 serialize_dendrogram: "left right height size\n" per merge,
// height with 17 significant digits (Python's "{:.17g}" == C's "%.17g": both
// correctly rounded, same exponent style).  Host arrays; writes at most `cap`
// bytes to out and the needed length to *len_out (TG_ERR_CAPACITY if larger).
TG_API int tg_serialize_dendrogram(const int64_t *lefts, const int64_t *rights, const double *heights,
                                   const int64_t *sizes, int64_t k, char *out, size_t cap, size_t *len_out) {
    if (k < 0 || !len_out || (k > 0 && (!lefts || !rights || !heights || !sizes))) return TG_ERR_ARG;
    // rows formatted in parallel chunks (std::to_chars(general, 17) is printf's "%.17g",
    // correctly rounded, ~0.2 us per row: 1.8 ms for a 10k-leaf dendrogram on one thread)
    auto fmt = [&](int64_t t0, int64_t t1, std::string &dst) {
        dst.clear();
        dst.reserve((size_t)(t1 - t0) * 40);
        char line[128];
        for (int64_t t = t0; t < t1; t++) {
            char *p = line, *end = line + sizeof(line);
            p = std::to_chars(p, end, (long long)lefts[t]).ptr;
            *p++ = ' ';
            p = std::to_chars(p, end, (long long)rights[t]).ptr;
            *p++ = ' ';
            p = std::to_chars(p, end, heights[t], std::chars_format::general, 17).ptr;
            *p++ = ' ';
            p = std::to_chars(p, end, (long long)sizes[t]).ptr;
            *p++ = '\n';
            dst.append(line, (size_t)(p - line));
        }
    };
    int nt = (int)std::min<int64_t>(16, std::max<int64_t>(1, k / 640));
    const unsigned hw = std::thread::hardware_concurrency();
    if (hw > 0 && (unsigned)nt > hw) nt = (int)hw;
    std::vector<std::string> parts((size_t)nt);
    if (nt == 1) {
        fmt(0, k, parts[0]);
    } else {
        std::vector<std::thread> th;
        th.reserve((size_t)nt - 1);
        for (int i = 1; i < nt; i++)
            th.emplace_back(fmt, k * i / nt, k * (i + 1) / nt, std::ref(parts[(size_t)i]));
        fmt(0, k / nt, parts[0]);
        for (auto &t : th) t.join();
    }
    size_t used = 0;
    for (const auto &pt : parts) {
        if (out && used + pt.size() <= cap) std::memcpy(out + used, pt.data(), pt.size());
        used += pt.size();
    }
    *len_out = used;
    return (out && used > cap) ? TG_ERR_CAPACITY : TG_OK;
}

// linkage.py:151-178 cut: flat labels after the first n - k merges, by the reference's own
// union-find (path halving, parent[find(child)] = node), labels in order of first appearance
// over the leaves (= ascending smallest member id).  Host arrays; `scratch` holds 2 (2n - 1)
// int64.  TG_ERR_ARG when a child id is outside [0, 2n - 1) (the reference raises IndexError).
TG_API int tg_cut_labels(const int64_t *lefts, const int64_t *rights, int64_t n, int64_t k, int64_t *labels,
                         int64_t *scratch) {
    if (n < 1 || k < 1 || k > n || !labels || !scratch || (n - k > 0 && (!lefts || !rights))) return TG_ERR_ARG;
    const int64_t nn = 2 * n - 1;
    int64_t *parent = scratch, *lab = scratch + nn;
    for (int64_t x = 0; x < nn; x++) {
        parent[x] = x;
        lab[x] = -1;
    }
    auto find = [&](int64_t x) {
        while (parent[x] != x) {
            parent[x] = parent[parent[x]];
            x = parent[x];
        }
        return x;
    };
    for (int64_t t = 0; t < n - k; t++) {
        const int64_t node = n + t, c[2] = {lefts[t], rights[t]};
        for (int q = 0; q < 2; q++) {
            if (c[q] < 0 || c[q] >= nn) return TG_ERR_ARG;
            parent[find(c[q])] = node;
        }
    }
    int64_t next = 0;
    for (int64_t leaf = 0; leaf < n; leaf++) {
        const int64_t r = find(leaf);
        if (lab[r] < 0) lab[r] = next++;
        labels[leaf] = lab[r];
    }
    return TG_OK;
}

// Return the hierarchy pool's cached memory (kept between tg_build_hierarchy calls) to the device.
TG_API int tg_release_cached_memory(void) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    for (int d = 0; d < 64; d++)
        if (g_pools[d]) {
            cudaError_t e = cudaMemPoolTrimTo(g_pools[d], 0);
            if (e != cudaSuccess) {
                tg_set_last_error(e, __FILE__, __LINE__);
                return TG_ERR_CUDA;
            }
        }
    return TG_OK;
}
