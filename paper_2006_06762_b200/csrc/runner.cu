// Candidate runner: the B200 replacement for the reference's CPU measurement
// seam (`measure_batch`, src/machine.py:249-285).
//
// A candidate is a list of launches of NVRTC-compiled kernels whose only
// arguments are device buffers ("slots" of a task).  lt_measure():
//   1. poisons the candidate's output slots with NaN (unwritten cells fail),
//   2. runs the launch list once (warm-up, also times it),
//   3. verifies every output against its fp64 ground-truth slot on the device:
//      max |got - ref| / max(|ref|, 1e-30) (the reference's _check_outputs
//      metric, src/machine.py:193-208) reduced to one float,
//   4. re-runs the list r >= min_repeat times between CUDA events on the task's
//      stream, r chosen so the timed region lasts >= min_ms, and reports mean
//      microseconds (the runner passes min_repeat 1: the warm-up run carries
//      first-launch costs and is never the measurement).
// Launch failures (e.g. too many registers x threads) are statuses, not errors.

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>
#include <mutex>
#include "common.h"

namespace lt {

// Driver-API entry points resolved through the runtime (cudaGetDriverEntryPoint),
// so the library loads on hosts without libcuda (the CPU build container).
struct Drv {
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*FuncGetAttribute)(int*, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           CUstream, void**, void**) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  bool ok = false;
};
static Drv g_drv;
static std::mutex g_drv_mu;

template <class F>
static bool resolve(const char* name, F& fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

static const Drv* drv() {
  std::lock_guard<std::mutex> g(g_drv_mu);
  if (!g_drv.ok) {
    bool ok = resolve("cuModuleLoadData", g_drv.ModuleLoadData) && resolve("cuModuleUnload", g_drv.ModuleUnload) &&
              resolve("cuModuleGetFunction", g_drv.ModuleGetFunction) &&
              resolve("cuFuncGetAttribute", g_drv.FuncGetAttribute) &&
              resolve("cuFuncSetAttribute", g_drv.FuncSetAttribute) &&
              resolve("cuLaunchKernel", g_drv.LaunchKernel) && resolve("cuGetErrorString", g_drv.GetErrorString);
    if (!ok) {
      fail("CUDA driver entry points unavailable (no driver / no device)");
      return nullptr;
    }
    g_drv.ok = true;
  }
  return &g_drv;
}

static const char* cu_str(CUresult r) {
  const char* s = nullptr;
  if (g_drv.GetErrorString) g_drv.GetErrorString(r, &s);
  return s ? s : "unknown CUDA driver error";
}

static int check_cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return 0;
  return fail(std::string(what) + ": " + cu_str(r));
}

// A faulting candidate (illegal address, ...) leaves a sticky error that kills
// every CUDA context of the process on that device (measured on the B200: the
// primary context and a fresh cuCtxCreate both fail afterwards).  Faults are
// therefore contained by a process boundary: lt_measure reports status 2 and
// the caller restarts its measuring process (the Python runner measures in a
// child process, paper_2006_06762_b200/measure.py).
static std::mutex g_mod_mu;
static std::unordered_map<CUmodule, int> g_mod;   // module -> device

struct Task {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::unordered_map<int, std::pair<void*, int64_t>> slots;
  unsigned int* d_err = nullptr;
};

static std::mutex g_fn_mu;
static std::unordered_set<CUfunction> g_smem_set;

void runner_forget() {
  std::lock_guard<std::mutex> g(g_fn_mu);
  g_smem_set.clear();
}

__global__ void relerr_kernel(const float* __restrict__ got, const double* __restrict__ ref, int64_t n,
                              unsigned int* __restrict__ out_bits) {
  float local = 0.0f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r = ref[i];
    double g = (double)got[i];
    double den = fabs(r) > 1e-30 ? fabs(r) : 1e-30;
    double e = fabs(g - r) / den;
    float ef = (e <= 3.0e38) ? (float)e : INFINITY;   // NaN and overflow -> inf
    local = fmaxf(local, ef);
  }
  for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
  __shared__ float warp_max[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) warp_max[w] = local;
  __syncthreads();
  if (w == 0) {
    float v = lane < (int)(blockDim.x >> 5) ? warp_max[lane] : 0.0f;
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) atomicMax(out_bits, __float_as_uint(v));   // non-negative floats order as uints
  }
}

__global__ void fill_u32_kernel(unsigned int* p, int64_t n, unsigned int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// Physical copy of a packed constant (LayoutRewrite, src/ir.py:747-760): physical
// element i, decomposed over the descriptor's extents (innermost last), reads the
// logical element sum_j digit_j * mult_j.  Pure data movement: equal bit for bit to
// the host restatement measure.pack.  Consecutive threads write consecutive
// physical words (coalesced stores; the gather is the layout change itself).
constexpr int PACK_MAX_DIMS = 16;
struct PackDesc {
  int n;
  int64_t ext[PACK_MAX_DIMS];
  int64_t mult[PACK_MAX_DIMS];
};

__global__ void pack_kernel(float* __restrict__ dst, const float* __restrict__ src, int64_t n, PackDesc d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i, off = 0;
    for (int j = d.n - 1; j >= 0; --j) {
      int64_t q = r / d.ext[j];
      off += (r - q * d.ext[j]) * d.mult[j];
      r = q;
    }
    dst[i] = src[off];
  }
}

}  // namespace lt

using lt::Task;

extern "C" {

typedef struct {
  int64_t func;
  uint32_t grid[3];
  uint32_t block[3];
  uint32_t smem;
  int32_t n_args;
  int32_t arg_slot[16];
} lt_launch;

typedef struct {
  double cost_us;       // mean device time of the whole launch list
  double first_us;      // warm-up run
  float max_rel_err;    // worst over all checked outputs
  int32_t repeats;
  int32_t status;       // 0 ok, 1 launch failed (resources), 2 kernel fault
  char detail[200];
} lt_measure_record;

int64_t lt_module_load(int device, const void* image, int64_t len) {
  (void)len;
  if (lt::check_cuda(cudaSetDevice(device), "cudaSetDevice")) return 0;
  cudaFree(0);  // make the primary context current for the driver API
  const lt::Drv* d = lt::drv();
  if (!d) return 0;
  CUmodule m;
  if (lt::check_cu(d->ModuleLoadData(&m, image), "cuModuleLoadData")) return 0;
  std::lock_guard<std::mutex> g(lt::g_mod_mu);
  lt::g_mod[m] = device;
  return (int64_t)(intptr_t)m;
}

int lt_module_unload(int64_t module) {
  CUmodule m = (CUmodule)(intptr_t)module;
  int device;
  {
    std::lock_guard<std::mutex> g(lt::g_mod_mu);
    auto it = lt::g_mod.find(m);
    if (it == lt::g_mod.end()) return lt::fail("cuModuleUnload: unknown module");
    device = it->second;
    lt::g_mod.erase(it);
  }
  const lt::Drv* d = lt::drv();
  if (!d || lt::check_cuda(cudaSetDevice(device), "cudaSetDevice")) return -1;
  return lt::check_cu(d->ModuleUnload(m), "cuModuleUnload");
}

int64_t lt_module_function(int64_t module, const char* name) {
  const lt::Drv* d = lt::drv();
  if (!d) return 0;
  CUfunction f;
  if (lt::check_cu(d->ModuleGetFunction(&f, (CUmodule)(intptr_t)module, name), "cuModuleGetFunction")) return 0;
  {
    // a handle value can be reused by a module loaded after another was unloaded
    // (the runner's LRU evicts modules): its dynamic shared-memory grant is new
    std::lock_guard<std::mutex> g(lt::g_fn_mu);
    lt::g_smem_set.erase(f);
  }
  return (int64_t)(intptr_t)f;
}

// registers per thread, local (spill+stack) bytes per thread, max threads per block, static smem
int lt_function_info(int64_t func, int* regs, int* local_bytes, int* max_threads, int* static_smem) {
  CUfunction f = (CUfunction)(intptr_t)func;
  const lt::Drv* d = lt::drv();
  if (!d) return -1;
  if (lt::check_cu(d->FuncGetAttribute(regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f), "attr") ||
      lt::check_cu(d->FuncGetAttribute(local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f), "attr") ||
      lt::check_cu(d->FuncGetAttribute(max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, f), "attr") ||
      lt::check_cu(d->FuncGetAttribute(static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, f), "attr"))
    return -1;
  return 0;
}

int64_t lt_task_create(int device) {
  if (lt::check_cuda(cudaSetDevice(device), "cudaSetDevice")) return 0;
  Task* t = new Task();
  t->device = device;
  if (lt::check_cuda(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking), "stream") ||
      lt::check_cuda(cudaEventCreate(&t->ev0), "event") || lt::check_cuda(cudaEventCreate(&t->ev1), "event") ||
      lt::check_cuda(cudaMalloc(&t->d_err, 16), "cudaMalloc")) {
    delete t;
    return 0;
  }
  return (int64_t)(intptr_t)t;
}

void lt_task_destroy(int64_t handle) {
  Task* t = (Task*)(intptr_t)handle;
  if (!t) return;
  cudaSetDevice(t->device);
  cudaStreamSynchronize(t->stream);
  for (auto& kv : t->slots) cudaFree(kv.second.first);
  cudaFree(t->d_err);
  cudaEventDestroy(t->ev0);
  cudaEventDestroy(t->ev1);
  cudaStreamDestroy(t->stream);
  delete t;
}

void* lt_task_stream(int64_t handle) { return ((Task*)(intptr_t)handle)->stream; }

#define TASK_SCOPE(t) \
  if (lt::check_cuda(cudaSetDevice((t)->device), "cudaSetDevice")) return -1

static int slot_alloc(Task* t, int slot, int64_t bytes) {
  auto it = t->slots.find(slot);
  if (it != t->slots.end()) {
    if (it->second.second >= bytes) return 0;
    cudaFree(it->second.first);
    t->slots.erase(it);
  }
  void* p = nullptr;
  if (lt::check_cuda(cudaMalloc(&p, bytes > 0 ? (size_t)bytes : 16), "cudaMalloc slot")) return -1;
  t->slots[slot] = {p, bytes};
  return 0;
}

// (Re)allocate slot `slot` with `bytes` bytes (contents undefined).
int lt_task_slot(int64_t handle, int slot, int64_t bytes) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  return slot_alloc(t, slot, bytes);
}

int64_t lt_task_slot_ptr(int64_t handle, int slot) {
  Task* t = (Task*)(intptr_t)handle;
  auto it = t->slots.find(slot);
  return it == t->slots.end() ? 0 : (int64_t)(intptr_t)it->second.first;
}

int lt_task_upload(int64_t handle, int slot, const void* host, int64_t bytes) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  if (slot_alloc(t, slot, bytes)) return -1;
  if (lt::check_cuda(cudaMemcpyAsync(t->slots[slot].first, host, (size_t)bytes, cudaMemcpyHostToDevice, t->stream),
                     "upload"))
    return -1;
  return lt::check_cuda(cudaStreamSynchronize(t->stream), "upload sync");
}

// Page-lock a host buffer (the DAG's inputs), so uploads from it are DMA from
// pinned memory; unregister before freeing it.
int lt_host_register(void* host, int64_t bytes) {
  if (bytes <= 0) return 0;
  return lt::check_cuda(cudaHostRegister(host, (size_t)bytes, cudaHostRegisterPortable), "cudaHostRegister");
}

int lt_host_unregister(void* host) {
  return lt::check_cuda(cudaHostUnregister(host), "cudaHostUnregister");
}

int lt_task_download(int64_t handle, int slot, void* host, int64_t bytes) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  auto it = t->slots.find(slot);
  if (it == t->slots.end() || it->second.second < bytes) return lt::fail("download: bad slot");
  if (lt::check_cuda(cudaMemcpyAsync(host, it->second.first, (size_t)bytes, cudaMemcpyDeviceToHost, t->stream),
                     "download"))
    return -1;
  return lt::check_cuda(cudaStreamSynchronize(t->stream), "download sync");
}

// Fill `n` 32-bit words of slot `slot` with `value`, ordered on the task stream
// before whatever runs next on it (the runner NaN-poisons a candidate's
// intermediate buffers before its verified warm-up, as the reference's
// interpreter NaN-fills stage buffers, src/interp.py:339-340).
int lt_task_fill(int64_t handle, int slot, int64_t n, uint32_t value) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  auto it = t->slots.find(slot);
  if (it == t->slots.end() || it->second.second < n * 4) return lt::fail("fill: bad slot");
  lt::fill_u32_kernel<<<256, 256, 0, t->stream>>>((unsigned int*)it->second.first, n, value);
  return lt::check_launch("fill");
}

// Pack slot `src_slot` (fp32, logical row-major) into `dst_slot` through the
// physical descriptor: n_phys extents (outer to inner) and per-extent multipliers
// into the logical flat offset.  Stream-ordered on the task stream.
int lt_task_pack(int64_t handle, int dst_slot, int src_slot, int n_phys, const int64_t* phys_ext,
                 const int64_t* src_mult) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  if (n_phys < 1 || n_phys > lt::PACK_MAX_DIMS) return lt::fail("pack: 1..16 physical dims");
  auto dst = t->slots.find(dst_slot), src = t->slots.find(src_slot);
  if (dst == t->slots.end() || src == t->slots.end()) return lt::fail("pack: bad slot");
  lt::PackDesc d;
  d.n = n_phys;
  int64_t n = 1, hi = 0;
  for (int j = 0; j < n_phys; ++j) {
    if (phys_ext[j] < 1 || src_mult[j] < 0) return lt::fail("pack: bad descriptor");
    d.ext[j] = phys_ext[j];
    d.mult[j] = src_mult[j];
    n *= phys_ext[j];
    hi += (phys_ext[j] - 1) * src_mult[j];
  }
  if (dst->second.second < n * 4 || src->second.second < (hi + 1) * 4) return lt::fail("pack: slot too small");
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  lt::pack_kernel<<<(int)blocks, 256, 0, t->stream>>>((float*)dst->second.first, (const float*)src->second.first, n, d);
  return lt::check_launch("pack");
}

static int launch_list(Task* t, const lt_launch* ls, int n, std::string& why) {
  const lt::Drv* d = lt::drv();
  if (!d) { why = "CUDA driver unavailable"; return 2; }
  for (int i = 0; i < n; ++i) {
    const lt_launch& L = ls[i];
    CUfunction f = (CUfunction)(intptr_t)L.func;
    void* ptrs[16];
    void* args[16];
    if (L.n_args > 16) { why = "too many kernel arguments"; return 1; }
    for (int a = 0; a < L.n_args; ++a) {
      auto it = t->slots.find(L.arg_slot[a]);
      if (it == t->slots.end()) { why = "launch references an unallocated slot"; return 1; }
      ptrs[a] = it->second.first;
      args[a] = &ptrs[a];
    }
    if (L.smem > 48 * 1024) {
      std::lock_guard<std::mutex> g(lt::g_fn_mu);
      if (!lt::g_smem_set.count(f)) {
        CUresult r = d->FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)L.smem);
        if (r != CUDA_SUCCESS) {
          why = std::string("dynamic shared memory not granted: ") + lt::cu_str(r);
          return 1;
        }
        lt::g_smem_set.insert(f);
      }
    }
    CUresult r = d->LaunchKernel(f, L.grid[0], L.grid[1], L.grid[2], L.block[0], L.block[1], L.block[2], L.smem,
                                 (CUstream)t->stream, args, nullptr);
    if (r != CUDA_SUCCESS) {
      why = std::string("launch failed: ") + lt::cu_str(r);
      return r == CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES || r == CUDA_ERROR_INVALID_VALUE ? 1 : 2;
    }
  }
  return 0;
}

// Run a launch list once, synchronously (ground truth, packing, warm-ups).
int lt_task_run(int64_t handle, const lt_launch* launches, int n) {
  Task* t = (Task*)(intptr_t)handle;
  TASK_SCOPE(t);
  std::string why;
  if (launch_list(t, launches, n, why)) return lt::fail(why);
  return lt::check_cuda(cudaStreamSynchronize(t->stream), "run");
}

// A sticky error after launching: the candidate faulted and the process's CUDA
// state is lost.  Reported as status 2 (the caller restarts the measuring
// process); never an error return, so measure_batch keeps its never-raises contract.
static int faulted(lt_measure_record* rec, const char* where, cudaError_t e) {
  rec->status = 2;
  snprintf(rec->detail, sizeof rec->detail, "kernel fault (%s): %s", where, cudaGetErrorString(e));
  return 0;
}

int lt_measure(int64_t handle, const lt_launch* launches, int n_launch, const int32_t* check_pairs,
               const int64_t* numel, int n_check, int min_repeat, int max_repeat, double min_ms,
               lt_measure_record* rec) {
  Task* t = (Task*)(intptr_t)handle;
  memset(rec, 0, sizeof *rec);
  TASK_SCOPE(t);
  std::string why;
  // 1. poison outputs
  for (int c = 0; c < n_check; ++c) {
    auto it = t->slots.find(check_pairs[2 * c]);
    if (it == t->slots.end()) return lt::fail("measure: output slot missing");
    lt::fill_u32_kernel<<<256, 256, 0, t->stream>>>((unsigned int*)it->second.first, numel[c], 0x7fc00000u);
  }
  // 2. warm-up (timed)
  cudaEventRecord(t->ev0, t->stream);
  int st = launch_list(t, launches, n_launch, why);
  if (st) {
    rec->status = st;
    snprintf(rec->detail, sizeof rec->detail, "%s", why.c_str());
    cudaError_t e = cudaStreamSynchronize(t->stream);
    if (e != cudaSuccess) return faulted(rec, "launch", e);
    cudaGetLastError();
    return 0;
  }
  cudaEventRecord(t->ev1, t->stream);
  cudaError_t e = cudaStreamSynchronize(t->stream);
  if (e != cudaSuccess) return faulted(rec, "warm-up", e);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t->ev0, t->ev1);
  rec->first_us = ms * 1000.0;
  // 3. verify against the fp64 ground truth
  cudaMemsetAsync(t->d_err, 0, 4, t->stream);
  for (int c = 0; c < n_check; ++c) {
    const float* got = (const float*)t->slots[check_pairs[2 * c]].first;
    auto it = t->slots.find(check_pairs[2 * c + 1]);
    if (it == t->slots.end()) return lt::fail("measure: reference slot missing");
    int64_t n = numel[c];
    int blocks = (int)((n + 255) / 256);
    if (blocks > 1184) blocks = 1184;
    if (blocks < 1) blocks = 1;
    lt::relerr_kernel<<<blocks, 256, 0, t->stream>>>(got, (const double*)it->second.first, n, t->d_err);
  }
  unsigned int bits = 0;
  cudaMemcpyAsync(&bits, t->d_err, 4, cudaMemcpyDeviceToHost, t->stream);
  e = cudaStreamSynchronize(t->stream);
  if (e != cudaSuccess) return faulted(rec, "verify", e);
  float err;
  memcpy(&err, &bits, 4);
  rec->max_rel_err = err;
  // 4. timed repeats: a run at least min_ms long is its own measurement (min_repeat
  //    0); shorter kernels are re-run until the timed region spans min_ms
  double first_ms = ms > 1e-4 ? ms : 1e-4;
  int r = (int)ceil(min_ms / first_ms);
  if (first_ms >= min_ms) r = 0;
  if (r < min_repeat) r = min_repeat;
  if (r > max_repeat) r = max_repeat;
  if (r == 0) {
    rec->repeats = 0;
    rec->cost_us = first_ms * 1000.0;
    return 0;
  }
  cudaEventRecord(t->ev0, t->stream);
  for (int k = 0; k < r; ++k) {
    st = launch_list(t, launches, n_launch, why);
    if (st) {
      rec->status = st;
      snprintf(rec->detail, sizeof rec->detail, "timed run: %s", why.c_str());
      e = cudaStreamSynchronize(t->stream);
      if (e != cudaSuccess) return faulted(rec, "timed runs", e);
      return 0;
    }
  }
  cudaEventRecord(t->ev1, t->stream);
  e = cudaStreamSynchronize(t->stream);
  if (e != cudaSuccess) return faulted(rec, "timed runs", e);
  cudaEventElapsedTime(&ms, t->ev0, t->ev1);
  rec->repeats = r;
  rec->cost_us = ms * 1000.0 / r;
  return 0;
}

}  // extern "C"

// ---- FP32 FFMA peak (the roofline denominator for candidate kernels) --------
// 8 independent FFMA chains per thread, 8 resident warps per SMSP: issue-bound.
namespace lt {
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters, float m, float c) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (float)(threadIdx.x + k) * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 123.456f) out[threadIdx.x] = s;   // keep the chains live
}

// register-operand form (a = a*b + c, b and c runtime registers): the FFMA shape
// of a GEMM inner product, which may issue at a lower rate than the immediate form
__global__ void __launch_bounds__(256) ffma_reg_kernel(float* out, const float* in, int iters) {
  float a[8], b[8], c[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = (float)(threadIdx.x + k) * 1e-3f;
    b[k] = in[k];
    c[k] = in[8 + k];
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b[(k + u) & 7], c[(k + 3 * u) & 7]);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 123.456f) out[threadIdx.x] = s;
}
}  // namespace lt

extern "C" int lt_ffma_peak_reg(int device, double* tflops, double* ms_out) {
  if (lt::check_cuda(cudaSetDevice(device), "cudaSetDevice")) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float *out = nullptr, *in = nullptr;
  if (lt::check_cuda(cudaMalloc(&out, 1024 * sizeof(float)), "cudaMalloc") ||
      lt::check_cuda(cudaMalloc(&in, 64 * sizeof(float)), "cudaMalloc"))
    return -1;
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = (i < 8) ? 0.9999f : 1e-4f;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  lt::ffma_reg_kernel<<<blocks, threads>>>(out, in, 64);
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    lt::ffma_reg_kernel<<<blocks, threads>>>(out, in, iters);
    cudaEventRecord(e1);
    if (lt::check_cuda(cudaEventSynchronize(e1), "ffma reg peak")) return -1;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *tflops = 2.0 * (double)blocks * threads * iters * 16 * 8 / (best * 1e-3) / 1e12;
  *ms_out = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaFree(in);
  return 0;
}


extern "C" int lt_ffma_peak(int device, double* tflops, double* ms_out) {
  if (lt::check_cuda(cudaSetDevice(device), "cudaSetDevice")) return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (lt::check_cuda(cudaMalloc(&out, 1024 * sizeof(float)), "cudaMalloc")) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  lt::ffma_peak_kernel<<<blocks, threads>>>(out, 64, 0.9999f, 1e-4f);   // warm-up / clocks up
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    lt::ffma_peak_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(e1);
    if (lt::check_cuda(cudaEventSynchronize(e1), "ffma peak")) return -1;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double flops = 2.0 * (double)blocks * threads * iters * 16 * 8;
  *tflops = flops / (best * 1e-3) / 1e12;
  *ms_out = best;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return 0;
}
