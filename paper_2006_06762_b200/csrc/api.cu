// C-ABI entry points that take HOST buffers (the reference-facing drop-in
// boundary, declared in include/loomtune_b200.h).  Each copies its inputs to
// the device, runs the device-pointer entry points on one stream, and copies
// the results back.  Callers own every host array; the library owns device
// scratch (grow-only, per thread) and frees it at lt_shutdown().

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <mutex>
#include <unistd.h>
#include "common.h"

extern "C" int lt_features_device(const int32_t*, const int64_t*, int64_t, double*, int*, void*);
extern "C" int lt_features_device_cm(const int32_t*, const int64_t*, int64_t, double*, int*, void*);
extern "C" int lt_cols_to_rows_device(const double*, int64_t, double*, void*);
extern "C" int lt_predict_rows_device(int64_t, const double*, int64_t, double*, void*);
extern "C" int lt_predict_cols_device(int64_t, const double*, int64_t, double*, void*);
extern "C" int lt_segment_sum_device(const double*, const int64_t*, int64_t, double*, void*);
extern "C" int lt_pool_start(int, const char*, double);
extern "C" void lt_pool_stop(void);

namespace lt {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(const std::string& msg) { g_err = msg; return -1; }

struct Scratch {
  DevBuf words, stmt_off, rows, cols, row_scores, prog_off, scores, err;
  cudaStream_t stream = nullptr;
  int init() {
    if (!stream && check_cuda(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream")) return -1;
    return 0;
  }
  void release() {
    for (DevBuf* b : {&words, &stmt_off, &rows, &cols, &row_scores, &prog_off, &scores, &err}) {
      if (b->ptr) cudaFree(b->ptr);
      b->ptr = nullptr;
      b->cap = 0;
    }
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
  }
};
static Scratch g_s;
static std::mutex g_mu;

// features of the uploaded records into g_s.cols ([164][n_stmt], column-major)
static int upload_features(const int32_t* words, const int64_t* stmt_off, int64_t n_stmt) {
  int64_t n_words = stmt_off[n_stmt];
  if (g_s.init() || g_s.words.reserve((size_t)n_words * 4 + 4) ||
      g_s.stmt_off.reserve((size_t)(n_stmt + 1) * 8) || g_s.cols.reserve((size_t)n_stmt * 164 * 8 + 8) ||
      g_s.err.reserve(4))
    return -1;
  cudaMemcpyAsync(g_s.words.ptr, words, (size_t)n_words * 4, cudaMemcpyHostToDevice, g_s.stream);
  cudaMemcpyAsync(g_s.stmt_off.ptr, stmt_off, (size_t)(n_stmt + 1) * 8, cudaMemcpyHostToDevice, g_s.stream);
  cudaMemsetAsync(g_s.err.ptr, 0, 4, g_s.stream);
  return lt_features_device_cm(g_s.words.as<int32_t>(), g_s.stmt_off.as<int64_t>(), n_stmt, g_s.cols.as<double>(),
                               g_s.err.as<int>(), g_s.stream);
}

// g_s.cols -> g_s.rows ([n_stmt][164]) for callers that want rows on the host
static int rows_from_cols(int64_t n_stmt) {
  if (g_s.rows.reserve((size_t)n_stmt * 164 * 8 + 8)) return -1;
  return lt_cols_to_rows_device(g_s.cols.as<double>(), n_stmt, g_s.rows.as<double>(), g_s.stream);
}

static int check_feature_err() {
  int err = 0;
  cudaMemcpyAsync(&err, g_s.err.ptr, 4, cudaMemcpyDeviceToHost, g_s.stream);
  if (check_cuda(cudaStreamSynchronize(g_s.stream), "features sync")) return -1;
  if (err == 1) return fail("statement record exceeds kernel limits (nest/loops/iterators/views)");
  if (err == 2) return fail("malformed decode AST in statement record");
  return 0;
}

}  // namespace lt

extern "C" {

const char* lt_last_error(void) { return lt::g_err.c_str(); }

int lt_version(void) { return 1; }

int lt_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int lt_set_device(int device) { return lt::check_cuda(cudaSetDevice(device), "cudaSetDevice"); }

// Features for n_stmt encoded statement records -> out_rows[n_stmt][164] (host).
int lt_features_batch(const int32_t* words, const int64_t* stmt_off, int64_t n_stmt, double* out_rows) {
  std::lock_guard<std::mutex> g(lt::g_mu);
  if (n_stmt <= 0) return 0;
  if (lt::upload_features(words, stmt_off, n_stmt) || lt::rows_from_cols(n_stmt)) return -1;
  if (lt::check_feature_err()) return -1;
  cudaMemcpyAsync(out_rows, lt::g_s.rows.ptr, (size_t)n_stmt * 164 * 8, cudaMemcpyDeviceToHost, lt::g_s.stream);
  return lt::check_cuda(cudaStreamSynchronize(lt::g_s.stream), "features copy-back");
}

// Program scores from feature rows (host): rows[n_rows][164], prog_row_off[n_prog+1].
int lt_predict_batch(int64_t model, const double* rows, const int64_t* prog_row_off, int64_t n_prog,
                     double* out_scores) {
  std::lock_guard<std::mutex> g(lt::g_mu);
  if (n_prog <= 0) return 0;
  int64_t n_rows = prog_row_off[n_prog];
  auto& s = lt::g_s;
  if (s.init() || s.rows.reserve((size_t)n_rows * 164 * 8 + 8) || s.row_scores.reserve((size_t)n_rows * 8 + 8) ||
      s.prog_off.reserve((size_t)(n_prog + 1) * 8) || s.scores.reserve((size_t)n_prog * 8))
    return -1;
  if (n_rows) cudaMemcpyAsync(s.rows.ptr, rows, (size_t)n_rows * 164 * 8, cudaMemcpyHostToDevice, s.stream);
  cudaMemcpyAsync(s.prog_off.ptr, prog_row_off, (size_t)(n_prog + 1) * 8, cudaMemcpyHostToDevice, s.stream);
  if (lt_predict_rows_device(model, s.rows.as<double>(), n_rows, s.row_scores.as<double>(), s.stream)) return -1;
  if (lt_segment_sum_device(s.row_scores.as<double>(), s.prog_off.as<int64_t>(), n_prog, s.scores.as<double>(),
                            s.stream))
    return -1;
  cudaMemcpyAsync(out_scores, s.scores.ptr, (size_t)n_prog * 8, cudaMemcpyDeviceToHost, s.stream);
  return lt::check_cuda(cudaStreamSynchronize(s.stream), "predict copy-back");
}

// Population scoring without leaving the device: encoded statements -> features ->
// trees -> per-program scores.  out_rows may be NULL (rows stay on the device).
int lt_score_batch(int64_t model, const int32_t* words, const int64_t* stmt_off, int64_t n_stmt,
                   const int64_t* prog_row_off, int64_t n_prog, double* out_scores, double* out_rows) {
  std::lock_guard<std::mutex> g(lt::g_mu);
  if (n_prog <= 0) return 0;
  auto& s = lt::g_s;
  if (prog_row_off[n_prog] != n_stmt) return lt::fail("program row offsets do not cover the statements");
  if (n_stmt > 0 && lt::upload_features(words, stmt_off, n_stmt)) return -1;
  if (s.row_scores.reserve((size_t)n_stmt * 8 + 8) || s.prog_off.reserve((size_t)(n_prog + 1) * 8) ||
      s.scores.reserve((size_t)n_prog * 8))
    return -1;
  cudaMemcpyAsync(s.prog_off.ptr, prog_row_off, (size_t)(n_prog + 1) * 8, cudaMemcpyHostToDevice, s.stream);
  if (n_stmt > 0 && lt_predict_cols_device(model, s.cols.as<double>(), n_stmt, s.row_scores.as<double>(), s.stream))
    return -1;
  if (lt_segment_sum_device(s.row_scores.as<double>(), s.prog_off.as<int64_t>(), n_prog, s.scores.as<double>(),
                            s.stream))
    return -1;
  if (n_stmt > 0 && lt::check_feature_err()) return -1;
  cudaMemcpyAsync(out_scores, s.scores.ptr, (size_t)n_prog * 8, cudaMemcpyDeviceToHost, s.stream);
  if (out_rows && n_stmt > 0) {
    if (lt::rows_from_cols(n_stmt)) return -1;
    cudaMemcpyAsync(out_rows, s.rows.ptr, (size_t)n_stmt * 164 * 8, cudaMemcpyDeviceToHost, s.stream);
  }
  return lt::check_cuda(cudaStreamSynchronize(s.stream), "score copy-back");
}

// Library setup: check the devices, create each device's primary context and
// start the compile pool (n_workers <= 0: host cores - 1) on `cache_dir`
// (NULL or "": no on-disk cubin cache).
int lt_init(int n_gpus, const char* cache_dir, int n_workers) {
  int n = lt_device_count();
  if (n_gpus < 1 || n_gpus > n) return lt::fail("lt_init: " + std::to_string(n_gpus) + " GPUs asked, " +
                                                std::to_string(n) + " visible");
  for (int d = 0; d < n_gpus; ++d)
    if (lt::check_cuda(cudaSetDevice(d), "lt_init: cudaSetDevice") || lt::check_cuda(cudaFree(0), "lt_init: context"))
      return -1;
  if (n_workers <= 0) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    n_workers = c > 1 ? (int)c - 1 : 1;
  }
  return lt_pool_start(n_workers, cache_dir, 120.0);
}

// Library teardown, before process exit: stop the compile pool (joins its
// dispatcher thread and reaps the workers) and free the scoring scratch.  Task,
// module, model and training handles stay valid until their destroy calls.
int lt_shutdown(void) {
  lt_pool_stop();
  std::lock_guard<std::mutex> g(lt::g_mu);
  lt::g_s.release();
  return 0;
}

void lt_release_scratch(void) {
  std::lock_guard<std::mutex> g(lt::g_mu);
  lt::g_s.release();
}

}  // extern "C"
