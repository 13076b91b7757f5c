/*
 * gts.h -- C ABI of the B200-native GTS batch similarity-search engine.
 *
 * This is the drop-in boundary under the reference's Python index API
 * (arXiv 2404.00966 reference package `metrictree`).  Each entry point
 * names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/metrictree/).  Plain pointers and sizes only --
 * no torch or C++ types cross this boundary, no C++ exception escapes it.
 *
 * Status codes (the Python shim maps them to the reference's exception
 * types, search.py:231-234, 246-268, data.py:220-229):
 *   GTS_OK        0
 *   GTS_EINVAL    1  invalid argument            -> ValueError
 *   GTS_EBUDGET   2  memory-unit budget          -> BudgetError
 *   GTS_EMETRIC   3  payload / metric mismatch   -> MetricMismatchError
 *   GTS_ECUDA     4  CUDA runtime error          -> RuntimeError
 *   GTS_EOOM      5  device allocation failed    -> MemoryError
 * gts_last_error() returns a thread-local message for the last failure.
 *
 * Ownership: the caller owns every input and output buffer; an index
 * handle owns its device tables; a result handle owns its device CSR until
 * gts_result_free.  Query calls on one index are reentrant (each call
 * allocates its workspace stream-ordered on the stream it is given);
 * tombstone updates must not overlap queries on the same index
 * (single writer).
 */
#ifndef GTS_H
#define GTS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GTS_OK 0
#define GTS_EINVAL 1
#define GTS_EBUDGET 2
#define GTS_EMETRIC 3
#define GTS_ECUDA 4
#define GTS_EOOM 5
#define GTS_EREBUILD 6   /* cache insert needs a rebuild (symbol outside the index alphabet) */

/* gts_batch_host flags */
#define GTS_FLAG_PRUNING 1   /* BatchSearcher pruning=True (search.py:225) */
#define GTS_FLAG_CACHE 2     /* also scan the pending-insert cache (StreamingIndex queries) */

/* metric codes = the reference snapshot codes (io.py:30-35) */
#define GTS_EDIT 0
#define GTS_L1 1
#define GTS_L2 2
#define GTS_ANGULAR 3

/* A payload collection in dataset-row order (reference data.py:59-126:
 * _VectorStore float64 matrix / _StringStore int32 code points + offsets). */
typedef struct {
    int32_t metric;
    int64_t n;
    int64_t dim;               /* vectors: D; strings: 0 */
    const double *vectors;     /* [n*dim] row-major float64, host */
    const int32_t *codes;      /* strings: UTF-32 code points, host */
    const int64_t *offsets;    /* strings: [n+1], host */
    const int64_t *ids;        /* [n] strictly increasing object ids */
} gts_dataset;

/* FlatPivotTree arrays (reference tree.py:155-175).  Node arrays have
 * nodes+1 slots (slot 0 unused); table arrays have n slots. */
typedef struct {
    int64_t nc, levels, split_rounds, nodes, n;
    int64_t *pivot_id, *pivot_row, *pos, *size;
    double *min_dis, *max_dis;
    int64_t *rows;
    double *dis;
    uint8_t *tombstone;
} gts_tree;

/* tree_height (tree.py:60-78) */
int gts_tree_height(int64_t n, int64_t nc, int64_t *max_h, int64_t *split_rounds);
/* node_count_for (tree.py:106-108) */
int64_t gts_node_count(int64_t levels, int64_t nc);

/* build (tree.py:370-385, _Builder 241-367) into caller-allocated arrays.
 * root_row is the reference's seeded draw rng.integers(0, n)
 * (tree.py:263, 288-291), made by the caller.  nthreads <= 0: all cores. */
int gts_build_tree(const gts_dataset *ds, int64_t root_row, int nthreads, gts_tree *tree);

/* The same build on the device: per level a segmented
 * reduction picks the pivots, one thread per entry maps its float64 (numpy
 * pairwise order) or exact edit distance, two stable radix sorts order the
 * level by (dis / (max + 1) + ordinal, id).  Bit-identical to gts_build_tree
 * and to the reference (tree.py:241-385).  Metrics edit, l1, l2 (angular
 * stays on gts_build_tree: numpy's arccos is not the device's). */
int gts_build_tree_device(const gts_dataset *ds, int64_t root_row, int device, gts_tree *tree);
/* Device build over device-resident float32 vectors x[n][dim] on `device`
 * (e.g. gts_generate_clustered output); ids: host [n]; metric l1 or l2. */
int gts_build_tree_device_f32(int32_t metric, int64_t n, int64_t dim, const float *x, const int64_t *ids,
                              int64_t root_row, int device, gts_tree *tree);

/* Device index: uploads the flattened list tables (node table, pivot ids
 * and ranges, object table with pivot distances, payloads in table order).
 * Replaces the state BatchSearcher.__init__ binds (search.py:225-234). */
typedef struct gts_index gts_index;
int gts_index_create(const gts_dataset *ds, const gts_tree *tree, int device, gts_index **out);
int gts_index_destroy(gts_index *ix);
/* Index over device-resident float32 vectors x[n][dim] (dataset row order,
 * on `device`): the same tables as gts_index_create, with the payload
 * gathers done on the device.  Metrics l1, l2. */
int gts_index_create_f32dev(const gts_tree *tree, int32_t metric, int64_t dim, const float *x,
                            const int64_t *ids, int device, gts_index **out);
/* Synthetic clustered float32 vectors on the device (SURVEY.md §8(d) C5,
 * a generate_clustered-equivalent, data.py:403-412): object i of an n_total
 * collection = centre[c] + N(0, spread), c uniform in [0, clusters), centres
 * U(0,1]^dim, all from a counter-based Philox4x32-10 stream, so any range
 * [first, first + count) is generated independently (one shard per GPU).
 * query_seed != 0: query i = a uniformly drawn object + N(0, noise). */
int gts_generate_clustered(uint64_t seed, int64_t n_total, int64_t dim, int64_t clusters, float spread,
                           int64_t first, int64_t count, uint64_t query_seed, float noise, float *out,
                           void *stream);

/* In-place insert into leaf slack (the reference buffers
 * inserts in a pending list and rebuilds on overflow, updates.py:109-158,
 * PAPER.md:436-448).  Every leaf of the device layout is followed by free
 * slots; each item descends the tree (the ring holding its distance to each
 * pivot, else the nearest; at the last split the nearest leaf with room),
 * takes that leaf's next free slot, and widens the leaf's own-pivot range and
 * every chosen node's parent-pivot range to its distances, so pruning stays
 * exact.  slots[i] = the slot of item i, or -1 if it cannot be placed (leaf
 * full, string longer than a slot or with a symbol outside the index
 * alphabet, payload not float32-exact over float32-exact data, angular):
 * the caller keeps those in the pending cache (gts_index_cache_set). */
int gts_index_insert(gts_index *ix, const gts_dataset *items, int32_t *slots, void *stream);
/* Delete inserted objects by slot (a delete of a pending id, updates.py:124-135). */
int gts_index_erase(gts_index *ix, const int32_t *slots, int64_t n, void *stream);

/* tombstone marks in table order (tree.tombstone, updates.py:124-135) */
int gts_index_set_tombstones(gts_index *ix, const uint8_t *tombstone, void *stream);

/* A query batch (the prepared payloads of search.py:280 / data.py:220-229).
 * Host buffers; gts_queries_upload makes a device-resident copy. */
typedef struct {
    int32_t metric;
    int64_t nq;
    int64_t dim;
    const double *vectors;    /* [nq*dim] float64 */
    const int32_t *codes;     /* strings: code points */
    const int64_t *offsets;   /* strings: [nq+1] */
} gts_query_batch;

typedef struct gts_queries gts_queries;   /* device-resident prepared batch */
int gts_queries_upload(gts_index *ix, const gts_query_batch *qb, void *stream, gts_queries **out);
int gts_queries_free(gts_queries *q);

typedef struct gts_result gts_result;     /* device CSR + stats */

/* BatchSearcher.range_batch (search.py:238-248): radii[nq] >= 0.
 * memory_units: row budget (search.py:229, runtime.py:18); 0 = the device
 * default of 1<<24 rows (the reference's CPU default is 1<<20).
 * Answers per query are every live object with d <= r, sorted by
 * (distance, id) (search.py:298-314). */
int gts_range_batch(gts_index *ix, const gts_queries *q, const double *radii,
                    int64_t memory_units, int pruning, void *stream, gts_result **out);
/* BatchSearcher.knn_batch (search.py:250-260): ks[nq] >= 1.  Answers are
 * the k smallest (distance, id) pairs over live objects (oracle.py:30-36). */
int gts_knn_batch(gts_index *ix, const gts_queries *q, const int64_t *ks,
                  int64_t memory_units, int pruning, void *stream, gts_result **out);
/* kNN in two phases, for a collection sharded over several indexes
 * (SURVEY.md §8(e) collective 2; the reference has one index, search.py:250-296):
 * gts_knn_probe writes each query's probe radius -- an upper bound of the
 * k-th distance within this index -- into radius_out[nq] (device float32).
 * The MIN of those radii over all shards bounds the global k-th distance;
 * gts_knn_batch_bounded then searches with that radius instead of probing
 * (radius NULL = probe as gts_knn_batch does).  flags as gts_batch_host. */
int gts_knn_probe(gts_index *ix, const gts_queries *q, const int64_t *ks, void *stream, float *radius_out);
int gts_knn_batch_bounded(gts_index *ix, const gts_queries *q, const int64_t *ks, const float *radius,
                          int64_t memory_units, int flags, void *stream, gts_result **out);

/* One-call host path: upload + search + download (the e2e boundary). */
int gts_range_batch_host(gts_index *ix, const gts_query_batch *qb, const double *radii,
                         int64_t memory_units, int pruning, void *stream, gts_result **out);
int gts_knn_batch_host(gts_index *ix, const gts_query_batch *qb, const int64_t *ks,
                       int64_t memory_units, int pruning, void *stream, gts_result **out);

/* Generic host entry point: mode 0 = range (radii), 1 = kNN (ks); flags as
 * above.  With GTS_FLAG_CACHE the answers are exact over tree entries that
 * are not tombstoned plus the pending-insert cache, i.e. StreamingIndex
 * query_range / query_knn (updates.py:167-196). */
int gts_batch_host(gts_index *ix, const gts_query_batch *qb, int mode, const double *radii,
                   const int64_t *ks, int64_t memory_units, int flags, void *stream, gts_result **out);
/* Replace the device copy of the pending-insert cache (StreamingIndex.pending,
 * updates.py:109-122) with `items` (ids + payloads).  Returns GTS_EREBUILD when
 * a string holds a symbol the index alphabet lacks. */
int gts_index_cache_set(gts_index *ix, const gts_dataset *items, void *stream);

/* Result access: sizes, then a copy into caller buffers (host or device,
 * decided by the pointer).  offsets[nq+1], ids[total], dis[total],
 * verified[nq], pruned[nq] (SearchStats, search.py:98-113); any may be NULL.
 * size_limits[64]: per split layer, 0 = layer not visited. */
int gts_result_info(const gts_result *r, int64_t *nq, int64_t *total, int64_t *peak_units,
                    int64_t *size_limits64);
int gts_result_copy(const gts_result *r, int64_t *offsets, int64_t *ids, double *dis,
                    int64_t *verified, int64_t *pruned, void *stream);
/* Device pointers of the result CSR (valid until gts_result_free). */
int gts_result_device(const gts_result *r, const int64_t **offsets, const int64_t **ids,
                      const double **dis);
int gts_result_free(gts_result *r);

/* ---- sharded collections ------------------------------
 * A collection split into shards, one GTS tree (one gts_index) per shard.
 * Exact answers over the union are the union of exact per-shard answers
 * (PAPER.md:213-222); the merge keeps, per query, the k smallest (kNN,
 * _KnnPool.merge search.py:116-144) or all (range) answers ordered by
 * (distance, id) (_collect search.py:298-314).
 *
 * gts_merge_results: the owner side of an all-to-all exchange.  nsrc sorted
 * answer lists per query, all device pointers on the current device:
 * counts[nsrc][nq]; ids / dis: source-major, then query-major (each
 * (source, query) list sorted by (distance, id)); ks[nq] (kNN) or NULL
 * (range); verified / pruned [nsrc][nq] or NULL (summed).  The merged CSR is
 * a result handle (gts_result_copy / gts_result_device / gts_result_free). */
int gts_merge_results(int nsrc, int64_t nq, const int64_t *counts, const int64_t *ids, const double *dis,
                      const int64_t *ks, const int64_t *verified, const int64_t *pruned, void *stream,
                      gts_result **out);

/* One handle over several shard indexes (the SURVEY.md §8(b) multi-device
 * handle: the shards' devices form its device set).  The shard indexes stay
 * owned by the caller and must outlive the handle.  gts_multi_batch_host runs
 * one host thread per shard (upload, search on the shard's device), kNN with
 * the MIN-radius exchange, gathers the answers to shards[0]'s device over
 * peer copies and merges them there. */
typedef struct gts_multi gts_multi;
int gts_multi_create(int nshards, gts_index *const *shards, gts_multi **out);
int gts_multi_destroy(gts_multi *m);
int gts_multi_batch_host(gts_multi *m, const gts_query_batch *qb, int mode, const double *radii,
                         const int64_t *ks, int64_t memory_units, int flags, gts_result **out);

/* Exact single-pair and row-pair distances on the device (metrics.py:196-223
 * and data.py:245-263 row_to_row), float64 result, for tests and the cache
 * scan of StreamingIndex (updates.py:206-215). */
int gts_pair_distances(int32_t metric, int64_t npairs, int64_t dim,
                       const double *a_vec, const double *b_vec,
                       const int32_t *a_codes, const int64_t *a_off,
                       const int32_t *b_codes, const int64_t *b_off,
                       double *out, void *stream);

/* Number of visible CUDA devices (0 when none). */
int gts_device_count(void);
/* Count of this library's kernel launches since load (bench evidence). */
int64_t gts_launch_count(void);
/* Per-kernel CUDA-event timing + algorithmic work counters (bench.py's
 * roofline).  gts_profile_read writes a JSON object into buf. */
int gts_profile_enable(int on);
int gts_profile_read(char *buf, int64_t cap, int reset);
/* Integer-pipe throughput microbenchmark (LOP3 + IMAD chains), ops/s. */
int gts_bench_int_peak(double *ops_per_s, void *stream);
/* FP32-pipe throughput microbenchmark (FADD / FFMA chains), lane-ops/s. */
int gts_bench_fp32_peak(double *ops_per_s, void *stream);
const char *gts_last_error(void);
const char *gts_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GTS_H */
