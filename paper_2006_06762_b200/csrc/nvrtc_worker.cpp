// NVRTC compile worker process (one of N, spawned by compile_pool.cpp).
//
// NVRTC serialises inside one process (measured 1.19x on 8 threads, SURVEY.md
// §7 hard part 3), so candidate kernels are compiled in separate processes.
// Protocol on stdin/stdout, little-endian:
//   request : u32 n_opts, n_opts x (u32 len, bytes), u32 src_len, src bytes
//   response: i32 status (0 ok, else nvrtcResult or -1), f64 seconds,
//             u32 len, bytes (cubin when ok, compile log otherwise)
// The worker exits when stdin closes.  When the first option is "--ptx" the
// source is PTX and is assembled in-process with nvPTXCompiler (ptxas as a
// library) using the remaining options.

#include <nvrtc.h>
#include <nvPTXCompiler.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>
#include <chrono>
#include <string>
#include <vector>

static bool read_all(void* buf, size_t n) {
  char* p = (char*)buf;
  while (n) {
    ssize_t r = read(0, p, n);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
  }
  return true;
}

static bool write_all(const void* buf, size_t n) {
  const char* p = (const char*)buf;
  while (n) {
    ssize_t r = write(1, p, n);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
  }
  return true;
}

static bool read_str(std::string& s) {
  uint32_t n;
  if (!read_all(&n, 4)) return false;
  s.resize(n);
  return n == 0 || read_all(&s[0], n);
}

int main() {
  for (;;) {
    uint32_t n_opts;
    if (!read_all(&n_opts, 4)) return 0;
    std::vector<std::string> opts(n_opts);
    for (auto& o : opts)
      if (!read_str(o)) return 0;
    std::string src;
    if (!read_str(src)) return 0;

    auto t0 = std::chrono::steady_clock::now();
    int32_t status = 0;
    std::string out;
    if (!opts.empty() && opts[0] == "--ptx") {
      nvPTXCompilerHandle h = nullptr;
      nvPTXCompileResult r = nvPTXCompilerCreate(&h, src.size(), src.data());
      if (r == NVPTXCOMPILE_SUCCESS) {
        std::vector<const char*> argv;
        for (size_t i = 1; i < opts.size(); ++i) argv.push_back(opts[i].c_str());
        r = nvPTXCompilerCompile(h, (int)argv.size(), argv.data());
        if (r == NVPTXCOMPILE_SUCCESS) {
          size_t n = 0;
          nvPTXCompilerGetCompiledProgramSize(h, &n);
          out.resize(n);
          if (n) nvPTXCompilerGetCompiledProgram(h, &out[0]);
        } else {
          size_t n = 0;
          nvPTXCompilerGetErrorLogSize(h, &n);
          out.resize(n);
          if (n) nvPTXCompilerGetErrorLog(h, &out[0]);
        }
      }
      status = (int32_t)r;
      if (h) nvPTXCompilerDestroy(&h);
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      uint32_t len = (uint32_t)out.size();
      if (!write_all(&status, 4) || !write_all(&secs, 8) || !write_all(&len, 4) ||
          (len && !write_all(out.data(), len)))
        return 0;
      continue;
    }
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "candidate.cu", 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) {
      status = (int32_t)r;
      out = nvrtcGetErrorString(r);
    } else {
      std::vector<const char*> argv;
      for (auto& o : opts) argv.push_back(o.c_str());
      r = nvrtcCompileProgram(prog, (int)argv.size(), argv.data());
      if (r != NVRTC_SUCCESS) {
        status = (int32_t)r;
        size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        out.resize(n);
        if (n) nvrtcGetProgramLog(prog, &out[0]);
      } else {
        size_t n = 0;
        nvrtcGetCUBINSize(prog, &n);
        out.resize(n);
        if (n) nvrtcGetCUBIN(prog, &out[0]);
      }
      nvrtcDestroyProgram(&prog);
    }
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint32_t len = (uint32_t)out.size();
    if (!write_all(&status, 4) || !write_all(&secs, 8) || !write_all(&len, 4) ||
        (len && !write_all(out.data(), len)))
      return 0;
  }
}
