// Shared helpers for the loomtune-b200 C-ABI library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

namespace lt {

// thread-local last error, surfaced through lt_last_error()
void set_error(const std::string& msg);
int fail(const std::string& msg);            // set_error + return -1

inline int check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}
inline int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

void runner_forget();       // drop cached per-function state (runner.cu)

// Feature columns kept raw (reference src/features.py:74-78): position one-hots of the
// vectorize/unroll/parallel blocks (cols 19-26, 30-37, 41-48) and, per buffer block b
// starting at 69+18b, the access one-hot (+0..2) and reuse one-hot (+7..9).
__host__ __device__ inline bool is_onehot(int k) {
  if ((k >= 19 && k <= 26) || (k >= 30 && k <= 37) || (k >= 41 && k <= 48)) return true;
  if (k >= 69 && k < 159) {
    int o = (k - 69) % 18;
    return o < 3 || (o >= 7 && o <= 9);
  }
  return false;
}

// grow-only device scratch buffer
struct DevBuf {
  void* ptr = nullptr;
  size_t cap = 0;
  int reserve(size_t bytes) {
    if (bytes <= cap) return 0;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    size_t want = bytes < 4096 ? 4096 : bytes + bytes / 4;
    if (check_cuda(cudaMalloc(&ptr, want), "cudaMalloc")) return -1;
    cap = want;
    return 0;
  }
  template <class T> T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace lt
