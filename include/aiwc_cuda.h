/* aiwc_cuda.h -- C-ABI of the B200-native random-forest path (libaiwc_cuda.so).
 *
 * Drop-in boundary for the reference's forest API.  Every entry
 * point takes plain pointers and sizes; there are no C++ or torch types here.
 * The reference interface each one replaces (paths under /root/reference/proj/include/aiwc):
 *
 *   aiwc_ctx_create      <- PreparedDataset(const Dataset&, ResponseTransform)  forest.hpp:458-475
 *                           (FitContext column store + p argsorts, forest.hpp:134-161)
 *   aiwc_fit             <- Forest fit(const PreparedDataset&, const ForestParams&, jobs)
 *                           forest.hpp:480-509 (TreeGrower::grow :179-376, compute_oob :393-454)
 *   aiwc_forest_*export  <- Forest::trees / Forest::inbag / Forest::oob        forest.hpp:66-74
 *   aiwc_forest_import   <- Forest::from_json (model load)                     forest.hpp:556-594
 *   aiwc_oob             <- OobStats compute_oob(const Forest&, const FitContext&) forest.hpp:393
 *                           and oob_error(const Forest&, const Dataset&)        forest.hpp:518-522
 *   aiwc_predict         <- double Forest::predict_response(span<const double>) forest.hpp:77-81
 *                           (Tree::predict forest.hpp:42-50), batched over q rows
 *   aiwc_evaluate        <- EvaluateResult evaluate(const Dataset&, ...)       experiments.hpp:383-408
 *   aiwc_synth_*         <- synthesize(SynthConfig) + make_dataset            synth.hpp:126, dataset.hpp:280
 *
 * Error convention (error.hpp:8-9 + CLI exit codes main.cpp:33-37): every function
 * returns an int status -- 0 ok, 2 ParseError, 3 ExecutionError, 4 IoError,
 * 5 SchemaError, 6 CUDA error (incl. "no device" / extension unusable), 7 bad
 * argument -- and sets a thread-local message readable with aiwc_last_error().
 * There is no CPU fallback: without a usable sm_100 device every compute entry
 * point fails with status 6.
 *
 * Thread safety: handles are independent; concurrent calls on distinct handles are
 * safe (each call uses its own stream and scratch).  A forest is immutable after
 * aiwc_fit returns.
 */
#ifndef AIWC_CUDA_H
#define AIWC_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AIWC_OK 0
#define AIWC_EPARSE 2
#define AIWC_EEXEC 3
#define AIWC_EIO 4
#define AIWC_ESCHEMA 5
#define AIWC_ECUDA 6
#define AIWC_EARG 7

typedef struct aiwc_ctx aiwc_ctx;       /* device-resident PreparedDataset */
typedef struct aiwc_forest aiwc_forest; /* device-resident Forest (+ host mirrors) */

/* OobStats (forest.hpp:57-64) */
typedef struct aiwc_oob_stats {
  int32_t degenerate;
  double mse;
  double response_variance;
  double error_pct;
  double r_squared;
  uint64_t rows_evaluated;
} aiwc_oob_stats;

const char* aiwc_last_error(void);
/* library version string, e.g. "aiwc-b200 1 sm_100a" */
const char* aiwc_version(void);
/* number of usable CUDA devices (0 on a host without a GPU) */
int aiwc_device_count(int* out);

/* ---- PreparedDataset ------------------------------------------------------
 * col: column-major predictors, col[c*n + i] = Dataset::predictor_value(i, c)
 *      (dataset.hpp:134-138);  y: responses (log10 seconds for Log10, dataset.hpp:150-155).
 * Presorts every column by (value asc, row asc) (forest.hpp:148-159) and builds dense
 * value ranks; uploads everything to `device`.  n >= 2, 1 <= p <= 1024. */
int aiwc_ctx_create(const double* col, const double* y, uint64_t n, uint32_t p,
                    int device, aiwc_ctx** out);
int aiwc_ctx_free(aiwc_ctx* ctx);
int aiwc_ctx_info(const aiwc_ctx* ctx, uint64_t* n, uint32_t* p, int* device);
/* on != 0: fits on this dataset also copy their in-bag draws into a pinned host mirror
 * while later tree batches grow, so aiwc_forest_host_view only has to move the nodes. */
int aiwc_ctx_set_host_mirror(aiwc_ctx* ctx, int on);

/* ---- fit -------------------------------------------------------------------
 * Grows trees [tree_begin, tree_end) of the forest keyed by (seed, tree index)
 * (forest.hpp:182).  Parameter checks mirror forest.hpp:482-490 (status 3).
 * When compute_oob != 0 and the range is the whole forest, OOB stats are computed
 * as compute_oob does (forest.hpp:393-454); for a partial range the per-row OOB
 * leaf values are kept on the device for aiwc_oob_accumulate (multi-GPU chaining). */
int aiwc_fit(aiwc_ctx* ctx, uint32_t num_trees, uint32_t mtry, uint32_t min_node_size,
             uint64_t seed, uint32_t tree_begin, uint32_t tree_end, int compute_oob,
             aiwc_forest** out);
int aiwc_forest_free(aiwc_forest* f);

/* tree count held, total node count, per-tree node counts (len = trees) */
int aiwc_forest_info(const aiwc_forest* f, uint32_t* trees, uint64_t* total_nodes,
                     uint32_t* tree_begin);
int aiwc_forest_node_counts(const aiwc_forest* f, uint64_t* counts);
/* concatenated BFS node SoA (TreeNode, forest.hpp:31-37); offsets len trees+1.
 * Any output pointer may be NULL. */
int aiwc_forest_export(const aiwc_forest* f, uint64_t* offsets, int32_t* feature,
                       double* threshold, int32_t* left, int32_t* right, double* value);
/* in-bag draws (forest.hpp:73), trees x n uint32, draw order */
int aiwc_forest_export_inbag(const aiwc_forest* f, uint32_t* inbag);
/* The same SoA and in-bag draws as host memory the forest owns: on first call the
 * device arrays are DMA'd straight into a pinned host mirror (no bounce copy into
 * pageable memory); the pointers stay valid until aiwc_forest_free.  inbag is set to
 * NULL when the forest holds no in-bag lists.  Any output pointer may be NULL. */
int aiwc_forest_host_view(aiwc_forest* f, const int32_t** feature, const double** threshold,
                          const int32_t** left, const int32_t** right, const double** value,
                          const uint32_t** inbag);
int aiwc_forest_oob_stats(const aiwc_forest* f, aiwc_oob_stats* out);

/* Build a device forest from host SoA (Forest::load path).  inbag may be NULL
 * (then OOB is unavailable).  n = rows of the training set (for inbag). */
int aiwc_forest_import(uint32_t trees, const uint64_t* offsets, const int32_t* feature,
                       const double* threshold, const int32_t* left, const int32_t* right,
                       const double* value, const uint32_t* inbag, uint64_t n, int device,
                       aiwc_forest** out);

/* Device-to-device forms of export / import, for gathering the tree-seed shards of a
 * multi-GPU fit over NCCL: the SoA arrays (and inbag, trees x n) are DEVICE
 * pointers on the forest's device; offsets stay on the host.  import_device checks the
 * canonical BFS layout on the device (same AIWC_EPARSE as aiwc_forest_import). */
int aiwc_forest_export_device(const aiwc_forest* f, int32_t* d_feature, double* d_threshold,
                              int32_t* d_left, double* d_value, uint32_t* d_inbag);
int aiwc_forest_import_device(uint32_t trees, const uint64_t* offsets, const int32_t* d_feature,
                              const double* d_threshold, const int32_t* d_left,
                              const double* d_value, const uint32_t* d_inbag, uint64_t n,
                              int device, aiwc_forest** out);

/* Device selection (cmd_rank, tools/main.cpp:338-349): for each of q feature rows
 * (row-major q x nfeat, host) predict the response on every device, i.e. on
 * Forest::make_row(features, device) (forest.hpp:98-115: the nfeat features, then a
 * one-hot over ndev device columns; nfeat + ndev = the forest's column count), expanded
 * on the device in chunks and scored by the predict kernels.  out_best[i] = the first-ranked device column offset (smallest
 * predict_time, lowest device name on ties).  out_response (q x ndev) may be NULL. */
int aiwc_rank(aiwc_forest* f, const double* features, uint64_t q, uint32_t nfeat,
              uint32_t ndev, double* out_response, uint32_t* out_best);

/* ---- OOB ---------------------------------------------------------------------
 * compute_oob over (forest, ctx): stats + optional per-row tree-ordered sum/count. */
int aiwc_oob(aiwc_ctx* ctx, aiwc_forest* f, aiwc_oob_stats* out, double* row_sum,
             uint32_t* row_count);
/* Multi-GPU chaining: continue per-row (sum, count) with this forest's trees in
 * tree order, starting from the given host arrays (in/out, length n).  Chaining
 * rank 0 -> 1 -> ... reproduces the single-forest tree-order sum bit-exactly. */
int aiwc_oob_accumulate(aiwc_ctx* ctx, aiwc_forest* f, double* row_sum,
                        uint32_t* row_count);
/* The same on DEVICE buffers (n doubles, n uint32 on the forest's device): the multi-GPU
 * OOB chain passes (row_sum, row_count) rank to rank over NCCL without host copies.
 * The caller's writes to the buffers must be complete (its stream synchronised); the
 * call returns when the sums are updated.  Replaces the same loop as above. */
int aiwc_oob_accumulate_device(aiwc_ctx* ctx, aiwc_forest* f, double* d_row_sum,
                               uint32_t* d_row_count);
/* OOB statistics of the forest's first tree_counts[i] trees, i < k (ascending counts,
 * forest grown from tree 0): compute_oob (forest.hpp:393-454) of every T-tree fit of
 * the same (data, mtry, min.node.size, seed) at once -- by the tree-prefix property a
 * T-tree fit is the first T trees of a longer one (forest.hpp:182, 477-479).  This is
 * the objective of tune_forest / heatmap_scan (tuner.hpp:247-253, experiments.hpp:
 * 79-108) over the num.trees axis. */
int aiwc_oob_prefix(aiwc_ctx* ctx, aiwc_forest* f, const uint32_t* tree_counts, uint32_t k,
                    aiwc_oob_stats* out);
/* Grid cells in one launch: ncells forests of num_trees trees
 * each, forest c grown exactly as aiwc_fit(ctx, num_trees, mtry[c], min_node_size[c],
 * seed, 0, num_trees, ...) would (tree t of every forest keyed by (seed, t)); the trees of
 * forest c are [c*num_trees, (c+1)*num_trees) of the returned handle.  OOB statistics
 * are not computed here: aiwc_oob_prefix_cells gives them for every tree prefix. */
int aiwc_fit_cells(aiwc_ctx* ctx, uint32_t ncells, const uint32_t* mtry,
                   const uint32_t* min_node_size, uint32_t num_trees, uint64_t seed,
                   aiwc_forest** out);
/* aiwc_oob_prefix for each forest of an aiwc_fit_cells handle: out[c*k + i] */
int aiwc_oob_prefix_cells(aiwc_ctx* ctx, aiwc_forest* f, const uint32_t* tree_counts,
                          uint32_t k, aiwc_oob_stats* out);
/* finalize OOB stats from per-row sum/count (forest.hpp:396-453) */
int aiwc_oob_finalize(const double* y, uint64_t n, const double* row_sum,
                      const uint32_t* row_count, aiwc_oob_stats* out);

/* ---- predict -----------------------------------------------------------------
 * rows: q x p row-major HOST array; out: q responses (mean over trees in tree
 * order, forest.hpp:77-81).  predict_time is the host-side pow(10, r).  Rows narrower
 * than the forest's largest split column fail with AIWC_ESCHEMA (predict, predict_device,
 * rank). */
int aiwc_predict(aiwc_forest* f, const double* rows, uint64_t q, uint32_t p,
                 double* out_response);
/* same with DEVICE pointers (inputs already resident in HBM) on the forest's device */
int aiwc_predict_device(aiwc_forest* f, const double* d_rows, uint64_t q, uint32_t p,
                        double* d_out);

/* ---- evaluate (hold-one-kernel-out, experiments.hpp:383-408) -------------------
 * kernel_of_row: kernel index per row (rows in canonical order); K kernels.
 * predicted_seconds[i] = predict_time of row i by the fold that held out its kernel;
 * fold k uses seed derive_seed(seed, "holdout", k).  Rows are the dataset's own
 * predictor rows (col, column-major). */
int aiwc_evaluate(const double* col, const double* y, uint64_t n, uint32_t p,
                  const uint32_t* kernel_of_row, uint32_t K, uint32_t num_trees,
                  uint32_t mtry, uint32_t min_node_size, uint64_t seed, int device,
                  double* predicted_seconds);

/* folds [fold_begin, fold_end) only (rows of other folds are left untouched): the
 * multi-GPU split of evaluate -- rank r takes a fold range and the predictions of the
 * ranks are combined row-wise (each row belongs to exactly one fold). */
int aiwc_evaluate_folds(const double* col, const double* y, uint64_t n, uint32_t p,
                        const uint32_t* kernel_of_row, uint32_t K, uint32_t fold_begin,
                        uint32_t fold_end, uint32_t num_trees, uint32_t mtry,
                        uint32_t min_node_size, uint64_t seed, int device,
                        double* predicted_seconds);

/* Hands the device's recycled fit memory (the grower's slot arena, idle per-fit blocks,
 * the stream-ordered pool's reserve) and the process's idle pinned host buffers back to
 * the driver, e.g. before other libraries allocate large buffers.  The next large fit
 * re-allocates what it needs. */
int aiwc_release_cached(int device);

/* ---- measurement (not part of the reference API) ----------------------------------
 * grow-kernel device time of the fit (CUDA events on the launching stream), whole fit
 * device time, sum over split nodes of their in-bag row counts (SURVEY 8d unit),
 * number of grow launches (1, or 2 after a pool-overflow retry). */
int aiwc_forest_profile(const aiwc_forest* f, double* grow_ms, double* fit_ms,
                        uint64_t* split_rows, uint32_t* grow_launches);
/* total kernels this library has launched in the process */
uint64_t aiwc_launch_count(void);
/* C5 device-selection queries: d_out[i*p + c] = d_rows[r_i*p + c] with
 * r_i = Rng(derive_seed(seed, "query", i)).bounded(n); device pointers, row-major */
int aiwc_make_queries(const double* d_rows, uint64_t n, uint32_t p, uint64_t q, uint64_t seed,
                      int device, double* d_out);

/* ---- seeds (rng.hpp) ----------------------------------------------------------- */
uint64_t aiwc_derive_seed(uint64_t seed, const char* tag, uint64_t index);

/* ---- synthetic AIWC tables (synth.hpp + dataset.hpp; host-side input generator) --
 * Produces the canonical-order dataset: n = kernels*4*devices rows,
 * p = 27 + devices predictors. */
typedef struct aiwc_table aiwc_table;
int aiwc_synth(uint64_t kernel_count, uint64_t device_count, double noise, uint64_t seed,
               aiwc_table** out);
int aiwc_table_free(aiwc_table* t);
int aiwc_table_info(const aiwc_table* t, uint64_t* n, uint32_t* p, uint32_t* kernels,
                    uint64_t* fingerprint);
/* any output may be NULL: col (p*n col-major), y (log10 s), seconds, kernel index */
int aiwc_table_export(const aiwc_table* t, double* col, double* y, double* seconds,
                      uint32_t* kernel_of_row);

#ifdef __cplusplus
}
#endif
#endif /* AIWC_CUDA_H */
