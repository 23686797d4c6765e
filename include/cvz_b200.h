/*
 * cvz_b200.h -- C-ABI of libcvz_b200.so, the B200 (sm_100a) implementation of
 * the BigGraphVis hot path (reference: commviz, /root/reference/pkg/src).
 *
 * The reference has no FFI; its native seam is a set of numba @njit kernels
 * called from Python.  Every entry point below replaces one of
 * those kernels or one numpy bulk operation on the path, and cites it as
 * C/<file>:<line> (C/ = /root/reference/pkg/src/commviz/).  The Python
 * drop-in package (paper_2108_00529_b200) binds these with ctypes; a
 * maintainer of the reference would bind them the same way.
 *
 * Conventions
 *  - Plain pointers + sizes, no torch types.  Pointers marked [dev] are
 *    device pointers, [host] host pointers.  Ids on device are int32
 *    (node ids < 2^31); public arrays stay int64/float64 like the reference.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Work is stream-ordered; scratch is cudaMallocAsync'ed on that stream.
 *  - Every function returns a cvz_status (0 = OK).  cvz_last_error() gives a
 *    message.  CVZ_ERR_VALUE maps to the reference's ValueError,
 *    CVZ_ERR_LAYOUT to LayoutError.
 *  - Functions whose output size is data-dependent synchronise the stream
 *    and say so.
 */
#ifndef CVZ_B200_H
#define CVZ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum cvz_status {
    CVZ_OK = 0,
    CVZ_ERR_CUDA = -1,   /* CUDA runtime / launch failure                    */
    CVZ_ERR_VALUE = -2,  /* bad argument (reference raises ValueError)       */
    CVZ_ERR_LAYOUT = -3, /* non-finite layout positions (LayoutError)        */
    CVZ_ERR_OOM = -4,    /* device allocation failed                          */
    CVZ_ERR_RANGE = -5   /* node id outside [0, 2^31) / label out of range    */
};

enum cvz_scoda_mode { CVZ_SCODA_DETERMINISTIC = 0, CVZ_SCODA_FAST = 1 };

int cvz_version(void);
const char *cvz_last_error(void);
/* Number of kernels this library has launched so far (process-wide).     */
long long cvz_launch_count(void);
/* Copy bytes (<= 256) of device memory to host memory after all work queued
 * on `stream`, without the copy engines (a one-CTA kernel writes mapped
 * pinned memory): small control reads (counts, flags) do not queue behind a
 * bulk transfer in flight on another stream.  No reference counterpart
 * (numpy scalars are host values). */
int cvz_read_small(void *host, const void *dev, int64_t bytes, void *stream);

/* Per-kernel device timing.  Between begin and end every library kernel
 * (and every CUB primitive, by region name) launched on a stream that is not
 * being captured is bracketed by CUDA events on its own stream; layout runs
 * launch their iterations directly instead of replaying a CUDA graph.  end
 * synchronises the device and builds the report: one line per kernel,
 * "name<TAB>launches<TAB>total_ms".  No reference counterpart (the
 * reference has only wall-clock stage timing, C/cli.py:106-117). */
int cvz_profile_begin(void);
int cvz_profile_end(void);
const char *cvz_profile_report(void);

/* Barnes-Hut walk statistics ("report BH interactions").
 * enable = 1 zeroes two device counters and makes every following per-thread
 * walk launch the instrumented kernel variant, which adds its node visits and
 * accepted interactions (force terms) to them; enable = 0 turns it off and
 * writes {visits, interactions} to totals (may be NULL).  Synchronises the
 * device.  Measurement only: the timed walk is never the counting variant.
 * No reference counterpart. */
int cvz_bh_stats(int enable, unsigned long long *totals);

/* FP64 FMA throughput probe (the Barnes-Hut walk's compute roofline, which
 * MEASURED_PEAKS.json does not carry): 8 independent DFMA chains per thread
 * at full occupancy on every SM, best of 3 timed launches; *gflops [host].
 * Synchronises `stream`.  Measurement only.  No reference counterpart. */
int cvz_probe_fp64(double *gflops, void *stream);

/* ---------------------------------------------------------------- graph */

/* Host (m,2) edge array [host, pageable or pinned; int64 or int32 per
 * in_is_int32] -> dev_out [dev] int32 pairs, same order.  The drop-in input
 * path of C/graph.py:114-122 (the reference takes int64 numpy arrays): ids
 * are range-checked and narrowed to int32 on the host by a thread pool into
 * page-locked staging buffers whose DMA overlaps the next chunk's
 * conversion.  Ids outside [0, 2^31) -> CVZ_ERR_RANGE.  Returns with the
 * copies queued on `stream` (the host array may be reused immediately). */
int cvz_edges_upload(const void *host_edges, int in_is_int32, int64_t m, int32_t *dev_out,
                     void *stream);

/* C/graph.py:114-122 from_edge_array (mask u==v keeping stream order) and
 * C/graph.py:121 np.bincount.  Stable single-pass compaction of an (m,2)
 * edge array ([dev] int64 or int32, in_is_int32 selects) into int32 pairs,
 * plus the maximum id.  d_m_out/d_max_id: [dev] int64 scalars.
 * Ids < 0 or >= 2^31 -> CVZ_ERR_RANGE (checked after a stream sync only when
 * check_range != 0). */
int cvz_edges_compact(const void *edges, int in_is_int32, int64_t m,
                      int32_t *edges_out, int64_t *d_m_out, int64_t *d_max_id,
                      int check_range, void *stream);

/* C/graph.py:121 degree = bincount(edges.ravel(), minlength=n).
 * degree [dev] int64[n] is overwritten. */
int cvz_degree_count(const int32_t *edges, int64_t m, int64_t n, int64_t *degree,
                     void *stream);

/* C/graph.py:125-136 degree_stats: out3 [dev] int64[3] = {mode of nonzero
 * degrees (ties -> smaller), sum, max}.  mode = 0 when all degrees are 0. */
int cvz_degree_stats(const int64_t *degree, int64_t n, int64_t *out3, void *stream);

/* C/graph.py:50-92 parse_edge_list, host tokenizer (multi-threaded C++).
 * text [host] ASCII bytes; threads <= 0 = all hardware threads.  Lines are
 * str.splitlines(), stripped, '#'/'%' comments and blank lines skipped,
 * exactly two Python-int tokens per line, u == v dropped.  Result:
 *   *err_code 0 ok (*m_out pairs kept, *handle to take them), 1 wrong token
 *   count (*err_tokens = K, "expected two tokens, got K"), 2 non-integer
 *   token, 3 input outside the native subset (non-ASCII byte, id outside
 *   int64: the caller uses the reference's Python loop); *err_line = the
 *   1-based line of the first error.
 * cvz_parse_take copies the 2*m external ids (u, v interleaved, line order)
 * into pairs_out [host] and frees the handle (pairs_out NULL: just free). */
int cvz_parse_begin(const char *text, int64_t len, int threads, void **handle, int64_t *m_out,
                    int64_t *err_line, int *err_code, int *err_tokens);
int cvz_parse_take(void *handle, int64_t *pairs_out);

/* C/graph.py:80-81 first-seen remap on the GPU: ext [dev] int64[count]
 * (u, v interleaved in line order) -> dense [dev] int32[count], dense id =
 * order of first appearance; *n_out [host] = number of distinct ids.
 * count < 2^31.  SYNCHRONISES. */
int cvz_first_seen_remap(const int64_t *ext, int64_t count, int32_t *dense, int64_t *n_out,
                         void *stream);

/* ------------------------------------------------------------ community */

/* C/community.py:98-120 _scoda_pass followed by C/community.py:123-161
 * _resolve_labels -- one streaming pass over edges[order[k]], k < m.
 *   order     [dev] int64[m] or NULL (identity; C/community.py:164-172)
 *   deg       [dev] int64[n] in/out counters (C/community.py:211)
 *   lab       [dev] int64[n] in: labels (values in [0,n)), out: RESOLVED
 *             representatives (min id on the reached cycle)
 *   lab_raw   [dev] int64[n] or NULL: receives the unresolved pass labels
 *   mode      CVZ_SCODA_DETERMINISTIC reproduces the sequential edge-order
 *             semantics bit-exactly; CVZ_SCODA_FAST is the racy 1-thread-per-
 *             edge pass (tolerance-gated). */
int cvz_scoda_pass(const int32_t *edges, int64_t m, const int64_t *order, int64_t n,
                   int64_t threshold, int tie_code, int mode, int64_t *deg, int64_t *lab,
                   int64_t *lab_raw, void *stream);

/* C/community.py:123-161 _resolve_labels alone: out[x] = min id on the cycle
 * reached from x.  lab values must lie in [0,n) (else CVZ_ERR_RANGE, after a
 * stream sync). */
int cvz_resolve_labels(const int64_t *lab, int64_t n, int64_t *out, void *stream);

/* C/community.py:164-195 make_schedule on the host (C++): out [host]
 * int64[m] = edge-processing order of `workers` chunked readers;
 * interleave 0 = "random" (numpy Generator(PCG64).integers replayed from the
 * state numpy's SeedSequence gives: 128-bit state/increment, has_uint32 /
 * uinteger buffer), 1 = "roundrobin".  workers <= 1 or m < 2: identity.
 * workers < 2^32. */
int cvz_make_schedule(int64_t m, int workers, int interleave, uint64_t state_hi,
                      uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int has_uint32,
                      uint32_t uinteger, int64_t *out);

/* One round of C/community.py:253-278 detect_communities on device:
 *   size-seeded counters (round > 1), pass over cur_edges (order or NULL),
 *   resolve, compose node_lab = lab[node_lab], history snapshot, early-stop
 *   test against prev_lab, then the next round's stream: contract
 *   (round_stream 0: relabelled crossing edges of cur_edges, stable) or
 *   restream (1: orig_edges relabelled by node_lab, crossing only).
 * node_lab [dev] int64[n] in/out; prev_lab [dev] int64[n] (in, ignored in
 * round 1; then overwritten with the new node_lab); deg_out [dev] int64[n];
 * history_out [dev] int64[n] or NULL; next_edges [dev] int32 capacity
 * max(m_cur, m_orig) pairs.  SYNCHRONISES: *next_m and *changed [host].
 * next_threshold >= 0 (contract stream, identity order, every later round's
 * threshold == next_threshold): crossing edges whose two communities both
 * have >= next_threshold + 2 members are no-ops in every later round and are
 * dropped from next_edges; *next_dead [host] counts them (the reference's
 * stream still holds them: m_{r+1} = *next_m + dropped so far).  -1 keeps
 * every crossing edge. */
int cvz_detect_round(const int32_t *cur_edges, int64_t m_cur, const int64_t *order,
                     const int32_t *orig_edges, int64_t m_orig, int64_t n,
                     int64_t threshold, int tie_code, int mode, int round_index,
                     int round_stream, int64_t *node_lab, int64_t *prev_lab,
                     int64_t *deg_out, int64_t *history_out, int32_t *next_edges,
                     int64_t *next_m, int *changed, int64_t next_threshold,
                     int64_t *next_dead, void *stream);

/* --------------------------------------------------------------- sketch */

/* C/sketch.py:39-44 CountMinSketch._indices: idx[r*k + j] = ((a_r*(x mod p)
 * + b_r) mod p) mod cols, p = 2^31-1, numpy non-negative mod. [dev] all. */
int cvz_sketch_indices(const int64_t *hash_a, const int64_t *hash_b, int rows,
                       int64_t cols, const int64_t *keys, int64_t k, int64_t *idx,
                       void *stream);

/* C/sketch.py:71-86 sketch_add_many (C/supergraph.py:42-46 accumulate_sizes):
 * table[r, idx_r(key_j)] += amount_j with int64 wrap-around, then every
 * negative cell is set to INT64_MAX.  n_amounts is the length of amounts:
 * k, or 1 to broadcast amounts[0] to every key (numpy's np.add.at
 * broadcasting); anything else is CVZ_ERR_VALUE.  amounts must be >= 0 (validate != 0
 * checks first and returns CVZ_ERR_VALUE without touching the table; this
 * synchronises).  *d_saturated [dev] int32 is set to 1 if any cell wrapped.
 * Shared-memory-staged table when rows*cols fits, warp-aggregated global
 * atomics otherwise. */
int cvz_sketch_add(int64_t *table, int rows, int64_t cols, const int64_t *hash_a,
                   const int64_t *hash_b, const int64_t *keys, const int64_t *amounts,
                   int64_t k, int64_t n_amounts, int validate, int32_t *d_saturated,
                   void *stream);

/* Sharded sketch building.  accumulate: delta[r, idx_r(key_j)]
 * += amount_j with u64 wrap-around and NO saturation (a rank-local delta
 * table, to be summed across ranks).  accumulate_edges: the edge-based form
 * of C/supergraph.py:42-46 -- +1 under labels[u] and +1 under labels[v] for
 * every edge (u, v) of edges [dev] int32[m*2]; labels [dev] int64[n].
 * merge: table += delta (wrap), then the C/sketch.py:80-86 saturation;
 * *d_saturated [dev] int32 set to 1 if a cell wrapped.  Since the adds are
 * integer additions mod 2^64, shard + all-reduce(SUM) + merge gives exactly
 * the single-process table. */
int cvz_sketch_accumulate(int64_t *delta, int rows, int64_t cols, const int64_t *hash_a,
                          const int64_t *hash_b, const int64_t *keys, const int64_t *amounts,
                          int64_t k, void *stream);
int cvz_sketch_accumulate_edges(int64_t *delta, int rows, int64_t cols, const int64_t *hash_a,
                                const int64_t *hash_b, const int32_t *edges, int64_t m,
                                const int64_t *labels, void *stream);
int cvz_sketch_merge(int64_t *table, const int64_t *delta, int rows, int64_t cols,
                     int32_t *d_saturated, void *stream);

/* C/sketch.py:93-98 sketch_estimate_many: out[j] = min_r table[r, idx_r]. */
int cvz_sketch_estimate(const int64_t *table, int rows, int64_t cols,
                        const int64_t *hash_a, const int64_t *hash_b,
                        const int64_t *keys, int64_t k, int64_t *out, void *stream);

/* ----------------------------------------------------------- supergraph */

typedef struct {
    int64_t k;         /* supernodes                                   */
    int64_t se;        /* superedges                                   */
    int64_t *comm_id;  /* [dev] int64[k] ascending community labels    */
    int64_t *weight;   /* [dev] int64[k] sketch estimates              */
    int64_t *se_edges; /* [dev] int64[se*2] (lo, hi), lexicographic    */
    int64_t *mult;     /* [dev] int64[se] multiplicities               */
} cvz_contract_result;

/* C/supergraph.py:49-76 contract: dense ids = rank of label among the
 * sorted unique labels; weights from the sketch; crossing edges -> (lo,hi)
 * 64-bit keys, radix sort + run-length encode.  labels [dev] int64[n]
 * (arbitrary int64 values).  Outputs are library-owned device buffers;
 * release with cvz_contract_release.  SYNCHRONISES. */
int cvz_contract(const int32_t *edges, int64_t m, const int64_t *labels, int64_t n,
                 const int64_t *table, int rows, int64_t cols, const int64_t *hash_a,
                 const int64_t *hash_b, cvz_contract_result *res, void *stream);
int cvz_contract_release(cvz_contract_result *res, void *stream);

/* --------------------------------------------------------------- layout */

typedef struct {
    int64_t iterations;
    double gravity, repulsion, jitter_tolerance, theta, max_step;
    int speed_form;      /* 0 product, 1 sum      (C/layout.py:384-387) */
    int attraction_form; /* 0 canonical, 1 reversed (C/layout.py:362)   */
} cvz_layout_params;

/* C/layout.py:312-328 repulsion_forces: theta <= 0 -> exact O(n^2) tiles
 * (C/layout.py:273-290), else GPU Barnes-Hut over the reference's quadtree
 * (C/layout.py:97-270).  pos [dev] f64[n*2], mass [dev] f64[n], out [dev]
 * f64[n*2] (overwritten). */
int cvz_repulsion(const double *pos, const double *mass, int64_t n, double repulsion,
                  double theta, double *out, void *stream);

/* C/layout.py:293-304 _attraction: out[u] += w*s*(p_v-p_u),
 * out[v] -= w*s*(p_v-p_u), accumulated per node in edge order (CSR gather,
 * no atomics).  edges [dev] int32[m*2], weight [dev] f64[m] or NULL (=1). */
int cvz_attraction(const double *pos, int64_t n, const int32_t *edges, int64_t m,
                   const double *weight, double sign, double *out, void *stream);

/* C/layout.py:341-402 layout loop, every iteration on device (one CUDA graph
 * per iteration, replayed).  pos [dev] f64[n*2] in/out; mass [dev] f64[n];
 * edges [dev] int32[m*2]; weight [dev] f64[m] or NULL; prev_force [dev]
 * f64[n*2] in/out (zeros for a fresh run, C/layout.py:363); speed [dev]
 * f64[1] in/out (1.0 fresh, :364); disp_hist [dev] f64[iterations].
 * On non-finite positions returns CVZ_ERR_LAYOUT and *bad_iteration [host]
 * = the 1-based iteration (C/layout.py:395-397).  SYNCHRONISES. */
int cvz_layout_run(double *pos, const double *mass, int64_t n, const int32_t *edges,
                   int64_t m, const double *weight, const cvz_layout_params *params,
                   double *prev_force, double *speed, double *disp_hist,
                   int64_t *bad_iteration, void *stream);

/* Node-sharded layout (one rank per GPU).  The single-process
 * loop C/layout.py:363-398 split at its two reductions.  Every rank keeps
 * ALL positions (pos [dev] f64[n*2], identical on every rank at the start of
 * an iteration), builds the full tree, and owns original node ids [lo, hi):
 * it computes their repulsion / springs / gravity / swing and moves only
 * them.  Per iteration the caller runs
 *     cvz_fa2_shard_forces(h, pos, sums)     sums [dev] f64[2] rank-local
 *     all-reduce(sums, SUM)                   -> Σswing, Σtraction
 *     cvz_fa2_shard_update(h, pos, sums, red) red [dev] f64[6] rank-local
 *     all-reduce(red, MAX)                    {-minx,maxx,-miny,maxy,maxdisp,bad}
 *     all-gather(pos rows [lo,hi))
 *     cvz_fa2_shard_absorb(h, red, disp_hist) next bbox, disp_hist[it], bad
 * then cvz_fa2_shard_finish (SYNCHRONISES).  Nothing synchronises inside the
 * loop.  ref_cell_ids = 1 numbers cells like the reference for coincident-
 * cell jitter (C/layout.py:258); run with 0 first and rerun with 1 when any
 * rank's finish reports *jitter_seen.  create SYNCHRONISES (CSR build). */
typedef struct cvz_fa2_shard cvz_fa2_shard;
int cvz_fa2_shard_create(const double *pos, const double *mass, int64_t n, const int32_t *edges,
                         int64_t m, const double *weight, const cvz_layout_params *params,
                         int64_t lo, int64_t hi, int ref_cell_ids, cvz_fa2_shard **out,
                         void *stream);
int cvz_fa2_shard_forces(cvz_fa2_shard *h, const double *pos, double *sums_out, void *stream);
int cvz_fa2_shard_update(cvz_fa2_shard *h, double *pos, const double *sums, double *red_out,
                         void *stream);
int cvz_fa2_shard_absorb(cvz_fa2_shard *h, const double *red, double *disp_hist, void *stream);
int cvz_fa2_shard_finish(cvz_fa2_shard *h, double *speed_out, int64_t *bad_iteration,
                         int *jitter_seen, void *stream);
int cvz_fa2_shard_destroy(cvz_fa2_shard *h, void *stream);

/* ------------------------------------------------------------------ rng */

/* numpy Generator(PCG64).uniform(low, low + range, count) on the device,
 * bit-exact: out[i] = low + range * ((next_u64 >> 11) * 2^-53), the i-th
 * draw of the generator whose 128-bit state/increment are given (take them
 * from numpy: default_rng(seed).bit_generator.state).  Replaces the host
 * draw of C/layout.py:78-82 init_positions.  out [dev] f64[count]. */
int cvz_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                      double low, double range, int64_t count, double *out, void *stream);

/* Synthetic input for BASELINE config C5 (not a reference function): edges
 * [start, start + count) of a counter-based R-MAT stream (draw l of edge k =
 * splitmix64(seed * 0x9E3779B97F4A7C15 + 64k + l), top 53 bits; quadrant
 * thresholds a, a+b, a+b+c), written as int32 pairs to edges_out [dev].
 * Shard-independent: any split of [0, m) over ranks gives the same stream.
 * Self-loops are kept (from_edge_array drops them, C/graph.py:117-118). */
int cvz_rmat_edges(int scale, double a, double b, double c, uint64_t seed, int64_t start,
                   int64_t count, int32_t *edges_out, void *stream);

/* -------------------------------------------------------------- metrics */

/* C/metrics.py:34-46 modularity ingredients: intra[c] and degsum[c] over
 * dense community ids.  dense [dev] int32[n] in [0,k); intra/degsum [dev]
 * int64[k] (overwritten). */
int cvz_modularity_parts(const int32_t *edges, int64_t m, const int32_t *dense,
                         const int64_t *degree, int64_t n, int64_t k, int64_t *intra,
                         int64_t *degsum, void *stream);

/* Dense community ids for arbitrary int64 labels (rank among the sorted
 * unique labels, np.unique(return_inverse=True)): dense [dev] int32[n],
 * *k_out [host] = number of communities.  SYNCHRONISES. */
int cvz_dense_labels(const int64_t *labels, int64_t n, int32_t *dense, int64_t *k_out,
                     void *stream);

/* C/metrics.py:70-75 community_size_histogram on device: sizes [dev]
 * int64[k] = members per dense id; hist [dev] int64[n+1] or NULL: hist[s] =
 * number of communities of size s. */
int cvz_community_sizes(const int32_t *dense, int64_t n, int64_t k, int64_t *sizes,
                        int64_t *hist, void *stream);

/* C/metrics.py:34-46 modularity: *q [dev] f64 = sum_c intra_c/m -
 * (degsum_c / 2m)^2 over dense ids (m > 0, else CVZ_ERR_VALUE). */
int cvz_modularity(const int32_t *edges, int64_t m, const int32_t *dense, const int64_t *degree,
                   int64_t n, int64_t k, double *q, void *stream);

/* ------------------------------------------------------------- writers */

/* Output formats, host C++, multi-threaded.  Results
 * are library-owned text: *handle + *bytes; cvz_text_take copies the text
 * into out [host, bytes long] (NULL: discard) and frees the handle.
 * format_table: nrows rows of ncols `sep`-separated fields + '\n'; kinds[c]
 * 0 = int64 column cols[c], 1 = double column "%.3f", 2 = the row index
 * (cols[c] unused) -- C/supergraph.py:79-91, C/community.py:284-294,
 * C/graph.py:100-111, C/sketch.py:101-102, C/cli.py:200-215.
 * format_svg: C/render.py:96-139 byte for byte (viewBox from positions and
 * radii, optional edges with multiplicity opacity, circles in (class,
 * index) order); pos [host] f64[n*2], classes in [0, ncolors). */
int cvz_format_table(int64_t nrows, int ncols, const int *kinds, const void *const *cols,
                     char sep, void **handle, int64_t *bytes);
int cvz_format_svg(int64_t n, const double *pos, const double *radii, const int64_t *classes,
                   const char *const *palette, int ncolors, int64_t ne, const int64_t *edges,
                   const double *mult, double margin, void **handle, int64_t *bytes);
int cvz_text_take(void *handle, char *out);

#ifdef __cplusplus
}
#endif
#endif /* CVZ_B200_H */
