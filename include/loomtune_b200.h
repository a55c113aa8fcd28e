/*
 * loomtune-b200 — C-ABI of the B200-native Ansor hot path.
 *
 * Drop-in boundary for the reference `loomtune` (arXiv 2006.06762 restatement):
 *   (A) measuring candidate programs  — replaces loomtune.machine.measure_batch
 *       (reference pkg/src/loomtune/machine.py:249-285)
 *   (B) scoring the evolutionary population — replaces CostModel.predict /
 *       predict_rows / predict_matrix (model.py:98-108) and extract_features
 *       (features.py:420-425).
 * Plain pointers and sizes only; callers own every host array; the library
 * owns device memory and frees it on lt_release_scratch / lt_task_destroy /
 * lt_model_destroy.  Every function returns 0 on success (or a non-zero
 * handle) and sets a thread-local message readable with lt_last_error().
 * Per-candidate failures are statuses in lt_measure_record, never errors.
 * Python binding: paper_2006_06762_b200/runtime.py (ctypes; GIL released).
 */
#ifndef LOOMTUNE_B200_H
#define LOOMTUNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ------------------------------------------------------------ */
const char* lt_last_error(void);
int lt_version(void);
int lt_device_count(void);
int lt_set_device(int device);
void lt_release_scratch(void);
/* Setup: checks that n_gpus devices are visible, creates
 * their contexts and starts the compile pool (n_workers <= 0: host cores - 1)
 * with an on-disk cubin cache in cache_dir (NULL/"": none). */
int lt_init(int n_gpus, const char* cache_dir, int n_workers);
/* Teardown before process exit: compile pool stopped (workers reaped), scratch
 * freed.  Task, module, model and training handles stay valid until their
 * destroy calls. */
int lt_shutdown(void);

/* ---- (B) feature extraction --------------------------------------------
 * Replaces extract_features / analyze_program / statement_features
 * (features.py:161-425).  Input: one int32 record per live statement, produced
 * by paper_2006_06762_b200/encode.py (layout documented there); stmt_off[n+1]
 * are word offsets.  Output: rows[n_stmt][164] float64, bit-identical to the
 * reference up to the last ulp of log2 (tolerance 1e-6).                      */
int lt_features_batch(const int32_t* words, const int64_t* stmt_off, int64_t n_stmt, double* out_rows);
int lt_features_device(const int32_t* d_words, const int64_t* d_stmt_off, int64_t n_stmt, double* d_rows,
                       int* d_err, void* stream);
/* Same features written column-major, d_cols[164][n_stmt] (coalesced stores; the
 * layout the fused scoring path uses), and the transpose to rows[n][164]. */
int lt_features_device_cm(const int32_t* d_words, const int64_t* d_stmt_off, int64_t n_stmt, double* d_cols,
                          int* d_err, void* stream);
int lt_cols_to_rows_device(const double* d_cols, int64_t n_stmt, double* d_rows, void* stream);

/* ---- (B) GBDT inference --------------------------------------------------
 * Model arrays are CostModel.to_json (model.py:110-125) concatenated over
 * trees; tree_node_off[n_trees+1]; node ids tree-local; n_features must be 164.
 * Scores follow numpy's order exactly: per row base + sum over trees in order
 * of value*eta; per program numpy's pairwise sum of its rows (model.py:98-105). */
int64_t lt_model_create(int n_trees, const int64_t* tree_node_off, const int32_t* feature,
                        const double* threshold, const int32_t* left, const int32_t* right,
                        const double* value, const double* eta, double base, int n_features);
void lt_model_destroy(int64_t model);
int lt_model_info(int64_t model, int* n_trees, int* n_used_features);
/* CostModel.predict_matrix over many programs: rows[n_rows][164], prog_row_off[n_prog+1]. */
int lt_predict_batch(int64_t model, const double* rows, const int64_t* prog_row_off, int64_t n_prog,
                     double* out_scores);
int lt_predict_rows_device(int64_t model, const double* d_rows, int64_t n_rows, double* d_row_scores,
                           void* stream);
int lt_predict_cols_device(int64_t model, const double* d_cols, int64_t n_rows, double* d_row_scores,
                           void* stream);
int lt_segment_sum_device(const double* d_row_scores, const int64_t* d_prog_off, int64_t n_prog,
                          double* d_scores, void* stream);
/* CostModel.predict over a population without leaving the device:
 * encoded statements -> features -> trees -> per-program scores (evolve.py:453-454).
 * out_rows may be NULL. */
int lt_score_batch(int64_t model, const int32_t* words, const int64_t* stmt_off, int64_t n_stmt,
                   const int64_t* prog_row_off, int64_t n_prog, double* out_scores, double* out_rows);

/* ---- (B) GBDT training ------------------------------------------------------
 * Replaces `_fit_tree` (model.py:158-255), the inner loop of `train`
 * (model.py:275-320).  lt_gbdt_create uploads a training matrix rows[n][nf]
 * (host) and sorts every feature column once; lt_gbdt_fit_tree fits one tree
 * for target[n], w[n] with the reference's exact split rule and numbering
 * (arrays of capacity cap >= 2^(depth+1)-1; *n_nodes = node count).
 * Bit-identical to the reference (numpy's summation orders).                 */
int64_t lt_gbdt_create(const double* rows, int64_t n, int nf);
void lt_gbdt_destroy(int64_t handle);
int lt_gbdt_fit_tree(int64_t handle, const double* target, const double* w, int depth, int cap,
                     int32_t* feature, double* threshold, int32_t* left, int32_t* right, double* value,
                     int32_t* n_nodes);

/* ---- (A) compile service ---------------------------------------------------
 * N NVRTC worker processes + on-disk cubin cache keyed by (options, source).
 * Candidate kernels are generated by paper_2006_06762_b200/lower.py. */
int lt_pool_start(int n_workers, const char* cache_dir, double timeout_s);
void lt_pool_stop(void);
int lt_pool_size(void);
int64_t lt_compile_submit(const char* src, int64_t len, const char* opts_newline_separated);
/* queued behind every job with a lower prio (the next batch, compiled ahead of time) */
int64_t lt_compile_submit_prio(const char* src, int64_t len, const char* opts_newline_separated, int64_t prio);
int lt_compile_wait(int64_t job, int* status, double* seconds, int* cache_hit, int64_t* out_len);
int lt_compile_ready(int64_t job);                             /* 1 done, 0 pending, -1 unknown */
int lt_compile_wait_any(const int64_t* jobs, int n, double timeout_s);  /* index of a finished job, -1: timeout */
int lt_compile_fetch(int64_t job, char* buf, int64_t cap);   /* cubin, or log when status != 0 */

/* ---- (A) runner --------------------------------------------------------------
 * Replaces the per-program body of measure_batch (machine.py:257-274): a
 * candidate is a launch list over task buffer slots; lt_measure poisons the
 * outputs, runs once, verifies every output against its fp64 ground-truth slot
 * (max |got-ref|/max(|ref|,1e-30), machine.py:193-208), then times repeats. */
typedef struct {
  int64_t func;         /* from lt_module_function */
  uint32_t grid[3];
  uint32_t block[3];
  uint32_t smem;        /* dynamic shared memory bytes */
  int32_t n_args;
  int32_t arg_slot[16]; /* each kernel argument is a slot's device pointer */
} lt_launch;

typedef struct {
  double cost_us;       /* mean device time of the launch list */
  double first_us;      /* warm-up run */
  float max_rel_err;    /* worst relative error over checked outputs (inf if NaN) */
  int32_t repeats;
  int32_t status;       /* 0 ok, 1 launch refused (resources), 2 kernel fault: the process's CUDA
                           state is lost (every context on the device), restart the process */
  char detail[200];
} lt_measure_record;

int64_t lt_module_load(int device, const void* cubin, int64_t len);
int lt_module_unload(int64_t module);
int64_t lt_module_function(int64_t module, const char* name);
int lt_function_info(int64_t func, int* regs, int* local_bytes, int* max_threads, int* static_smem);
int64_t lt_task_create(int device);
void lt_task_destroy(int64_t task);
void* lt_task_stream(int64_t task);
int lt_task_slot(int64_t task, int slot, int64_t bytes);
int64_t lt_task_slot_ptr(int64_t task, int slot);
int lt_task_upload(int64_t task, int slot, const void* host, int64_t bytes);
int lt_task_download(int64_t task, int slot, void* host, int64_t bytes);
/* page-lock / release a host buffer that is uploaded repeatedly (the DAG's inputs) */
int lt_host_register(void* host, int64_t bytes);
int lt_host_unregister(void* host);
/* fill n 32-bit words of a slot with `value`, stream-ordered (NaN-poisoning scratch) */
int lt_task_fill(int64_t task, int slot, int64_t n, uint32_t value);
/* physical copy of a packed constant on the device (replaces the host-side packing of
   LayoutRewrite constants, src/ir.py:747-760): dst[i] = src[sum_j digit_j(i) * src_mult[j]],
   digits of i over phys_ext (outer to inner, n_phys <= 16) */
int lt_task_pack(int64_t task, int dst_slot, int src_slot, int n_phys, const int64_t* phys_ext,
                 const int64_t* src_mult);
int lt_task_run(int64_t task, const lt_launch* launches, int n);
int lt_measure(int64_t task, const lt_launch* launches, int n_launch, const int32_t* check_pairs,
               const int64_t* numel, int n_check, int min_repeat, int max_repeat, double min_ms,
               lt_measure_record* rec);

/* ---- multi-GPU exchange ---------------------------
 * One process per GPU; each measures its shard of a batch (lt_measure) and
 * scores its shard of a population (lt_score_batch); only fixed-size records,
 * the fitness vector and the serialised model cross GPUs, over NCCL (opened at
 * run time: libnccl.so.2).  Replaces nothing in the reference (single process,
 * src/machine.py:257-274 and src/evolve.py:453-454 are serial loops); the
 * Python path does the same exchange with torch.distributed (dist.py).
 * Shards are padded to the largest shard: out has world * n_local_max entries. */
int lt_comm_unique_id(char* out128);                      /* rank 0, sent to the others out of band */
int64_t lt_comm_create(const char* id128, int rank, int world, int device);
void lt_comm_destroy(int64_t comm);
int lt_comm_rank(int64_t comm, int* rank, int* world);
int lt_comm_allgather(int64_t comm, const void* local, int64_t bytes_per_rank, void* out);
int lt_comm_allgather_records(int64_t comm, const lt_measure_record* local, int64_t n_local_max,
                              lt_measure_record* out);
int lt_comm_allgather_f64(int64_t comm, const double* local, int64_t n_local_max, double* out);
int lt_comm_broadcast(int64_t comm, void* buf, int64_t bytes, int root);   /* e.g. the model after train */

/* FP32 FFMA peak of the device (TFLOP/s), the roofline denominator for candidate kernels. */
int lt_ffma_peak(int device, double* tflops, double* ms);
/* Same with register (non-immediate) FFMA operands: the GEMM inner-product form. */
int lt_ffma_peak_reg(int device, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* LOOMTUNE_B200_H */
