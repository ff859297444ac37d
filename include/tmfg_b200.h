/*
 * tmfg_b200.h -- C ABI of the B200-native TMFG-DBHT hot path (libtmfg_b200.so).
 *
 * Every entry point replaces one function of the reference package
 * (arxiv 2408.09399 reference, pkg/src/tmfgclust); the comment above each
 * prototype cites the reference interface it stands in for (file:line).
 *
 * Conventions (mirroring the reference kernels' out-parameter style,
 * _kernels.py:18,96,178,185):
 *   - all array arguments are DEVICE pointers (cudaMalloc / torch CUDA storage),
 *     C-contiguous, allocated by the caller; the library never frees them;
 *   - scratch comes from a caller-provided workspace `ws` of `ws_bytes`
 *     (query the size with the matching *_workspace_bytes function);
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     unless documented as synchronous;
 *   - return value: TG_OK or a TG_ERR_* code (no C++ exception crosses the ABI);
 *     tg_last_error() describes the last failure on this thread.
 *   - `workers` arguments of the reference have no equivalent: results are
 *     independent of launch configuration by construction.
 */
#ifndef TMFG_B200_H
#define TMFG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 1

#define TG_OK 0
#define TG_ERR_ARG 1         /* bad argument (shape, null pointer, unsupported size) */
#define TG_ERR_CUDA 2        /* CUDA runtime error */
#define TG_ERR_WORKSPACE 3   /* workspace too small */
#define TG_ERR_CAPACITY 5    /* variable-size output larger than the given capacity */
#define TG_ERR_TRACE 6       /* trace references a non-live face (tmfg.py:67-68 TraceError) */
#define TG_ERR_NOT_REDUCIBLE 7 /* NN-chain cannot terminate: distances not reducible (linkage.py:50-94) */

/* validation flags written by tg_validate_f64 (simmatrix.py:126-139 DataError causes) */
#define TG_BAD_NAN 1
#define TG_BAD_ASYM 2
#define TG_BAD_DIAG 4
#define TG_BAD_RANGE 8

int tg_abi_version(void);
const char *tg_last_error(void);
/* kernels launched by this library so far (process-wide counter) */
long long tg_launch_count(void);

/* ---------------------------------------------------------------- similarity */

/* simmatrix.py:105-123 pearson_similarity + _kernels.py:17-37 pearson_kernel.
 * X (n, L) float64 -> S (n, n) float64: centred rows, zero-norm rows correlate 0,
 * clamp to [-1, 1], unit diagonal, exactly symmetric. fp64 DMMA SYRK. */
size_t tg_pearson_workspace_bytes(int64_t n, int64_t L);
int tg_pearson_f64(const double *X, int64_t n, int64_t L, double *S_out, void *ws, size_t ws_bytes,
                   void *stream);

/* _kernels.py:17-37 in the reference's arithmetic order (sequential k, product
 * and sum rounded separately, (s * inv_i) * inv_j, clamp): bit-identical to the
 * reference's S from the same centred rows xc (n, L) and inverse norms inv (n)
 * (its numpy prologue, simmatrix.py:113-118).  FP64-pipe bound; the DMMA path
 * above is the fast one (within 1e-12). */
int tg_pearson_refexact_f64(const double *xc, const double *inv, int64_t n, int64_t L, double *S_out,
                            void *stream);

/* simmatrix.py:126-139 validate_similarity: writes a TG_BAD_* bitmask to
 * *flags_out (device int32). */
int tg_validate_f64(const double *S, int64_t n, int32_t *flags_out, void *stream);

/* simmatrix.py:225-249 sort_neighbor_lists: order_out (n, n-1) int32, each row the
 * ids by (S desc, id asc) with the row's own id removed.  If screen_out (2n
 * doubles) is not NULL the same pass writes the initial-clique screen:
 * screen_out[v] = sum_j S[v, j] - S[v, v] in this kernel's summation order and
 * screen_out[n + v] = a rigorous bound on its distance to numpy's pairwise sum
 * (tmfg.py:76), consumed by tg_initial_clique_screened. */
size_t tg_row_sort_workspace_bytes(int64_t n);
int tg_row_sort_f64(const double *S, int64_t n, int32_t *order_out, double *screen_out, void *ws,
                    size_t ws_bytes, void *stream);

/* tmfg.py:76: rowsum_out[v] = pairwise_sum(S[v, :]) - S[v, v] (numpy order, bit-identical). */
size_t tg_row_sums_workspace_bytes(int64_t n);
int tg_row_sums_f64(const double *S, int64_t n, double *rowsum_out, void *ws, size_t ws_bytes, void *stream);

/* tmfg.py:71-79 select_initial_clique from the row sums: 4 ids (sum desc, id asc),
 * written ascending to clique_out (device int32[4]). */
int tg_initial_clique(const double *rowsum, int64_t n, int32_t *clique_out, void *stream);

/* tmfg.py:71-79 select_initial_clique from the row-sort screen: rows that cannot
 * reach the top 4 under any value inside their bound are dropped, the rest get
 * exact numpy pairwise sums (same result as tg_row_sums_f64 + tg_initial_clique). */
size_t tg_initial_clique_screened_workspace_bytes(int64_t n);
int tg_initial_clique_screened(const double *S, int64_t n, const double *screen, int32_t *clique_out, void *ws,
                               size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- TMFG */

/* tmfg.py:344-436 build_tmfg_heap (+ tmfg.py:94-182 bookkeeping).
 * Outputs: trace (n-4, 4), host_fid (n-4) face id each row subdivided,
 * edges (3n-6, 2), faces (2n-4, 3) int32; stats int64[32] =
 * {pops, refreshes, gain_increases, status, assert_fid, assert_old_gain_bits,
 *  assert_new_gain_bits, then kernel self-profile counters (rounds, refills,
 *  per-phase cycles; see tools/tmfg_profile.py)}.  status 0 = ok, 2 = the check_invariants
 * assertion of tmfg.py:429 fired (check != 0 only).  One persistent thread-block
 * cluster (the leader CTA runs the insertion rounds, the other CTAs keep the per-vertex
 * scan state current and prefetch S into L2); check != 0 adds the brute-force optimality
 * test of tmfg.py:377-399. */
size_t tg_tmfg_workspace_bytes(int64_t n);
int tg_tmfg_heap(const double *S, const int32_t *order, int64_t n, const int32_t *clique, int32_t *trace_out,
                 int32_t *host_fid_out, int32_t *edges_out, int32_t *faces_out, int64_t *stats_out, int32_t check,
                 void *ws, size_t ws_bytes, void *stream);

/* tmfg.py:208-263 build_tmfg_exact and tmfg.py:280-341 build_tmfg_corr, with the
 * prefix rule of tmfg.py:185-205 _select_round (prefix_size >= 1).  S validated by the
 * caller; clique from tg_initial_clique*; order (corr only) from tg_row_sort_f64.
 * Outputs trace (n-4, 4), edges (3n-6, 2), faces (2n-4, 3) int32 exactly as the
 * reference's _GraphAccum (tmfg.py:94-144).  One persistent CTA; the workspace holds
 * the face table and the scan state (~40 n bytes). */
size_t tg_tmfg_variant_workspace_bytes(int64_t n);
int tg_tmfg_exact(const double *S, int64_t n, const int32_t *clique, int64_t prefix_size, int32_t *trace_out,
                  int32_t *edges_out, int32_t *faces_out, void *ws, size_t ws_bytes, void *stream);
int tg_tmfg_corr(const double *S, const int32_t *order, int64_t n, const int32_t *clique, int64_t prefix_size,
                 int32_t *trace_out, int32_t *edges_out, int32_t *faces_out, void *ws, size_t ws_bytes,
                 void *stream);

/* tmfg.py:137-143 finalize weights: w[i] = S[edges[i,0], edges[i,1]]. */
int tg_edge_weights(const double *S, int64_t n, const int32_t *edges, int64_t m, double *w_out, void *stream);

/* ---------------------------------------------------------------------- APSP */

/* apsp.py:52-77 to_weighted: CSR in edge order (indptr n+1 int64, nbr int32,
 * len = sqrt(max(2(1-s),0)) float64), strength (n) float64 accumulated like
 * np.add.at(e0) then np.add.at(e1).  edges (m, 2) int32. */
size_t tg_weighted_workspace_bytes(int64_t n, int64_t m);
int tg_to_weighted(const double *S, int64_t n, const int32_t *edges, int64_t m, int64_t *indptr_out,
                   int32_t *nbr_out, double *len_out, double *strength_out, void *ws, size_t ws_bytes,
                   void *stream);

/* _kernels.py:40-99 dijkstra_rows / apsp.py:164-171 apsp_exact: dist_out
 * (n_src, n) float64, row s = exact shortest-path distances from sources[s]
 * (bit-identical to binary-heap Dijkstra: same fl(d + w) fixed point). */
size_t tg_sssp_workspace_bytes(int64_t n, int64_t n_src);
int tg_sssp_rows(const int64_t *indptr, const int32_t *nbr, const double *len, int64_t n, const int64_t *sources,
                 int64_t n_src, double *dist_out, void *ws, size_t ws_bytes, void *stream);

/* apsp.py:178-186 select_hubs: first H ids by (strength desc, id asc). */
size_t tg_select_hubs_workspace_bytes(int64_t n);
int tg_select_hubs(const double *strength, int64_t n, int64_t H, int64_t *hubs_out, void *ws, size_t ws_bytes,
                   void *stream);

/* apsp.py:206-209: first argmin over hub rows, nearest hub id/dist, radii = c * dist. */
int tg_nearest_hub(const double *hub_dist, const int64_t *hubs, int64_t H, int64_t n, double radius_factor,
                   int64_t *nearest_hub_out, double *nearest_dist_out, double *radii_out, void *stream);

/* _kernels.py:102-181 + apsp.py:211-220: radius-truncated searches from every
 * vertex, recorded as a CSR sorted by id within each segment.  Synchronous.
 * If the total exceeds `capacity`, returns TG_ERR_CAPACITY with *total_out
 * set (call again with a larger buffer). */
size_t tg_truncated_workspace_bytes(int64_t n);
int tg_truncated(const int64_t *indptr, const int32_t *nbr, const double *len, int64_t n, const double *radii,
                 int64_t capacity, int64_t *near_indptr_out, int32_t *near_ids_out, double *near_dist_out,
                 int64_t *total_out, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------- DBHT */

/* Distance oracle view (apsp.py:80-158).  mode 0 = ExactOracle (matrix n x n),
 * mode 1 = HubOracle (hub_dist H x n + near CSR; rev_* is the transposed near
 * table: for each u the pairs (v, near_v(u)) with u in near(v)). */
typedef struct {
    int32_t mode;
    int64_t n;
    const double *matrix;
    int64_t H;
    const double *hub_dist;
    const int64_t *near_indptr;
    const int32_t *near_ids;
    const double *near_dist;
    const int64_t *rev_indptr;
    const int32_t *rev_ids;
    const double *rev_dist;
} tg_oracle_t;

/* transposed near table for tg_oracle_t.rev_* (E = near_indptr[n]). */
size_t tg_near_transpose_workspace_bytes(int64_t n, int64_t E);
int tg_near_transpose(int64_t n, const int64_t *near_indptr, const int32_t *near_ids, const double *near_dist,
                      int64_t *rev_indptr_out, int32_t *rev_ids_out, double *rev_dist_out, void *ws,
                      size_t ws_bytes, void *stream);

/* dbht.py:64-89 build_bubble_tree from the clique and the trace.  Synchronous:
 * returns TG_ERR_TRACE (and *bad_row_out) when a row's host face is not live. */
size_t tg_bubble_tree_workspace_bytes(int64_t n);
int tg_bubble_tree(const int32_t *clique, const int32_t *trace, int64_t n, int32_t *bubbles_out,
                   int32_t *links_out, int32_t *link_faces_out, int64_t *bad_row_out, void *ws, size_t ws_bytes,
                   void *stream);

/* dbht.py:100-117 orient_edges (sources/targets int64, n-4 links). */
int tg_orient_edges(const double *S, int64_t n, const int32_t *bubbles, const int32_t *links,
                    const int32_t *link_faces, int64_t n_links, int64_t *sources_out, int64_t *targets_out,
                    void *stream);

/* dbht.py:143-175 _next_hops + bubble_sinks (m bubbles). */
size_t tg_bubble_sinks_workspace_bytes(int64_t m);
int tg_bubble_sinks(const double *S, int64_t n, const int32_t *bubbles, int64_t m, const int32_t *link_faces,
                    const int64_t *sources, const int64_t *targets, int64_t n_links, int64_t *sinks_out,
                    void *ws, size_t ws_bytes, void *stream);

/* dbht.py:178-214 assign_vertices. */
size_t tg_assign_workspace_bytes(int64_t n, int64_t m);
int tg_assign_vertices(const tg_oracle_t *oracle, const int32_t *bubbles, int64_t m, const int64_t *sinks,
                       int64_t *vertex_bubble_out, int64_t *vertex_converging_out, void *ws, size_t ws_bytes,
                       void *stream);

/* apsp.py:92-94 / 138-158 oracle.block(mem, mem) for a batch of groups:
 * group g = perm[starts[g] : starts[g+1]], its g x g block written row-major at
 * blocks_out + block_offsets[g]. */
int tg_group_blocks(const tg_oracle_t *oracle, const int32_t *perm, const int64_t *starts, int64_t count,
                    const int64_t *block_offsets, double *blocks_out, void *stream);

/* apsp.py:88-94 / 127-158: out (nr x nc) = oracle.block(rows, cols)
 * (query_semantics = 0) or [oracle.query(u, v)] (query_semantics = 1). */
int tg_oracle_block(const tg_oracle_t *oracle, const int32_t *rows, int64_t nr, const int32_t *cols, int64_t nc,
                    int32_t query_semantics, double *out, void *stream);

/* dbht.py:217-230 _cluster_max_matrix (+ _kernels.py:184-201 segment_pair_max),
 * batched over vertex-disjoint sub-problems.  Sub-problem p covers positions
 * [perm_off, perm_off + len) of perm/gid (gid = group index of each position,
 * groups contiguous and ascending) and writes its m x m result at out + out_off.
 * Tiles (sub, i0, j0) of 64 x 64 positions cover every sub-problem.  Hub mode:
 * min-plus over the hub rows + near-table overrides (column table wins), max per
 * group pair; exact mode: D entries, rows from the lower group, mirrored. */
typedef struct {
    int64_t perm_off;
    int32_t len;
    int32_t m;
    int64_t out_off;
    int64_t tile_off;   /* index of the sub-problem's first tile (row-major nt x nt, nt = ceil(len/64)) */
} tg_gm_sub_t;
typedef struct {
    int32_t sub;
    int32_t i0;
    int32_t j0;
} tg_gm_tile_t;
/* H: the hub count of a hub-mode oracle (0 in exact mode); the workspace holds the
 * permuted vertex-major fp32/fp64 copies of hub_dist used by the hub-mode tiles. */
size_t tg_group_max_workspace_bytes(int64_t n, int64_t ntiles, int64_t H);
/* The tile list of tg_group_max_batch built on the device: tile t of sub-problem p (row-major
 * over its nt x nt grid) = {p, 64 (t / nt), 64 (t % nt)} at tiles[subs[p].tile_off + t]
 * (dbht.py:217-230 sub-problem layout; the host no longer builds and uploads it). */
int tg_group_tiles_fill(const void *subs, int64_t nsub, void *tiles, int64_t ntiles, void *stream);
/* total_len: the number of perm / gid entries (the sub-problems lie back to back). */
int tg_group_max_batch(const tg_oracle_t *oracle, const int32_t *perm, const int32_t *gid, int64_t total_len,
                       const void *subs, int64_t nsub, const void *tiles, int64_t ntiles, double *out, int64_t out_len,
                       void *ws, size_t ws_bytes, void *stream);

/* linkage.py:50-94 _nn_chain over a batch of dense matrices (matrix b: sizes[b]
 * x sizes[b] at mats + mat_offsets[b]; it is overwritten as the working copy).
 * Raw merges (slot cluster ids, discovery order) at merge_offsets[b]
 * (sizes[b]-1 rows).  active/slot/chain: scratch of sizes[b] entries at
 * aux_offsets[b]. */
int tg_nn_chain_batch(double *mats, const int64_t *mat_offsets, const int64_t *sizes, int64_t count,
                      const int64_t *merge_offsets, int64_t *lefts_out, int64_t *rights_out, double *heights_out,
                      const int64_t *aux_offsets, uint8_t *active, int64_t *slot, int64_t *chain, void *stream);

/* dbht.py:233-339 build_hierarchy (+ linkage.py:97-116 canonicalisation,
 * linkage.py:136-148 sizes): the three complete-linkage layers over the bubble
 * assignment, emitted with the running height floor.  vertex_bubble /
 * vertex_converging are DEVICE arrays (n); the dendrogram rows are written to
 * HOST arrays of n-1 entries (lefts, rights, heights, sizes) and *n_merges_out.
 * Host-orchestrated (a few stream synchronisations); the oracle blocks, group
 * maxima and NN-chains run on the GPU.  Scratch comes from a memory pool owned by
 * the library (one per device, up to 16 GiB kept cached between calls; the
 * process's default pool is not touched). */
int tg_build_hierarchy(const tg_oracle_t *oracle, const int64_t *vertex_bubble, const int64_t *vertex_converging,
                       int64_t n, int64_t *lefts_out, int64_t *rights_out, double *heights_out, int64_t *sizes_out,
                       int64_t *n_merges_out, void *stream);

/* Trim the library's hierarchy pool to zero (returns its cached memory to the device). */
int tg_release_cached_memory(void);

/* linkage.py:181-187 serialize_dendrogram (HOST arrays): "left right height size\n"
 * per merge, height as %.17g (== Python "{:.17g}").  Needed length in *len_out;
 * TG_ERR_CAPACITY when it exceeds cap. */
int tg_serialize_dendrogram(const int64_t *lefts, const int64_t *rights, const double *heights, const int64_t *sizes,
                            int64_t k, char *out, size_t cap, size_t *len_out);

/* linkage.py:151-178 cut (HOST arrays): flat labels 0..k-1 after the first n - k merges (the
 * reference's union-find; labels by ascending smallest member id).  scratch: 2 (2n - 1) int64.
 * TG_ERR_ARG for k outside 1..n or a child id outside [0, 2n - 1). */
int tg_cut_labels(const int64_t *lefts, const int64_t *rights, int64_t n, int64_t k, int64_t *labels,
                  int64_t *scratch);

#ifdef __cplusplus
}
#endif

#endif /* TMFG_B200_H */
