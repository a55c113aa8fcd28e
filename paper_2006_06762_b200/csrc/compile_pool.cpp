// Multi-process NVRTC compile pool with a persistent on-disk cubin cache.
//
// Candidate kernels are instantiated with their exact tile constants, so most
// candidates need a fresh compile (64-85% distinct keys) and the
// measured-candidates/sec rate is bound by compile throughput.  NVRTC does not
// scale across threads of one process, so the pool runs N `lt_nvrtc_worker`
// processes (posix_spawn, pipes) fed by one dispatcher thread.  Results are
// keyed by a 64-bit FNV-1a hash of (options, source); hits are served from
// `<cache_dir>/<key>.cubin` without compiling.

#include <dlfcn.h>
#include <fcntl.h>
#include <poll.h>
#include <signal.h>
#include <spawn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.h"

extern char** environ;

namespace lt {

struct Job {
  std::string src;
  std::vector<std::string> opts;
  std::string key;
  int state = 0;  // 0 queued, 1 running, 2 done
  int status = 0;
  double secs = 0.0;
  bool cache_hit = false;
  int64_t prio = 0;  // lower runs first (the batch a job belongs to); then longest first
  std::string result;
  std::chrono::steady_clock::time_point started;
};

struct Worker {
  pid_t pid = -1;
  int to = -1, from = -1;
  int64_t job = 0;  // 0 = idle
};

class Pool {
 public:
  ~Pool() { stop(); }
  int start(int n, const std::string& cache_dir, double timeout_s);
  void stop();
  int64_t submit(const char* src, int64_t len, const char* opts, int64_t prio = 0);
  int wait_any(const int64_t* ids, int n, double timeout_s);
  int wait(int64_t id, int* status, double* secs, int* hit, int64_t* len);
  int fetch(int64_t id, char* buf, int64_t cap);
  int ready(int64_t id) {
    std::lock_guard<std::mutex> g(mu_);
    auto it = jobs_.find(id);
    return it == jobs_.end() ? -1 : (it->second.state == 2 ? 1 : 0);
  }
  int size() const { return (int)workers_.size(); }

 private:
  int spawn(Worker& w);
  void kill_worker(Worker& w);
  void loop();
  bool send(Worker& w, Job& j);
  void finish(int64_t id, Job& j);

  std::string exe_, cache_dir_;
  double timeout_s_ = 120.0;
  std::vector<Worker> workers_;
  std::deque<int64_t> queue_;
  std::unordered_map<int64_t, Job> jobs_;
  int64_t next_id_ = 1;
  bool running_ = false;
  std::thread thr_;
  std::mutex mu_;
  std::condition_variable cv_done_, cv_work_;
  int wake_[2] = {-1, -1};
};

static std::string lib_dir() {
  Dl_info info;
  if (dladdr((void*)&lib_dir, &info) && info.dli_fname) {
    std::string p = info.dli_fname;
    size_t s = p.rfind('/');
    if (s != std::string::npos) return p.substr(0, s);
  }
  return ".";
}

static uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ULL) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}

static bool write_all(int fd, const void* buf, size_t n) {
  const char* p = (const char*)buf;
  while (n) {
    ssize_t r = write(fd, p, n);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
  }
  return true;
}

static bool read_all(int fd, void* buf, size_t n) {
  char* p = (char*)buf;
  while (n) {
    ssize_t r = read(fd, p, n);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
  }
  return true;
}

int Pool::spawn(Worker& w) {
  int in_p[2], out_p[2];
  if (pipe(in_p) || pipe(out_p)) return fail("pipe failed");
  posix_spawn_file_actions_t fa;
  posix_spawn_file_actions_init(&fa);
  posix_spawn_file_actions_adddup2(&fa, in_p[0], 0);
  posix_spawn_file_actions_adddup2(&fa, out_p[1], 1);
  posix_spawn_file_actions_addclose(&fa, in_p[1]);
  posix_spawn_file_actions_addclose(&fa, out_p[0]);
  char* argv[] = {(char*)exe_.c_str(), nullptr};
  pid_t pid;
  int rc = posix_spawn(&pid, exe_.c_str(), &fa, nullptr, argv, environ);
  posix_spawn_file_actions_destroy(&fa);
  close(in_p[0]);
  close(out_p[1]);
  if (rc != 0) {
    close(in_p[1]);
    close(out_p[0]);
    return fail("posix_spawn of " + exe_ + " failed: " + strerror(rc));
  }
  fcntl(in_p[1], F_SETFD, FD_CLOEXEC);
  fcntl(out_p[0], F_SETFD, FD_CLOEXEC);
  w.pid = pid;
  w.to = in_p[1];
  w.from = out_p[0];
  w.job = 0;
  return 0;
}

void Pool::kill_worker(Worker& w) {
  if (w.pid > 0) {
    kill(w.pid, SIGKILL);
    waitpid(w.pid, nullptr, 0);
  }
  if (w.to >= 0) close(w.to);
  if (w.from >= 0) close(w.from);
  w = Worker();
}

int Pool::start(int n, const std::string& cache_dir, double timeout_s) {
  std::lock_guard<std::mutex> g(mu_);
  if (running_) return 0;
  signal(SIGPIPE, SIG_IGN);
  exe_ = lib_dir() + "/lt_nvrtc_worker";
  if (access(exe_.c_str(), X_OK) != 0) return fail("compile worker not found: " + exe_);
  cache_dir_ = cache_dir;
  if (!cache_dir_.empty()) mkdir(cache_dir_.c_str(), 0755);
  timeout_s_ = timeout_s > 0 ? timeout_s : 120.0;
  if (pipe(wake_)) return fail("pipe failed");
  fcntl(wake_[0], F_SETFL, O_NONBLOCK);
  workers_.resize(n < 1 ? 1 : n);
  for (auto& w : workers_)
    if (spawn(w)) return -1;
  running_ = true;
  thr_ = std::thread([this] { loop(); });
  return 0;
}

void Pool::stop() {
  {
    std::lock_guard<std::mutex> g(mu_);
    if (!running_) return;
    running_ = false;
  }
  char c = 1;
  if (write(wake_[1], &c, 1) < 0) {}
  cv_work_.notify_all();
  if (thr_.joinable()) thr_.join();
  for (auto& w : workers_) kill_worker(w);
  workers_.clear();
  close(wake_[0]);
  close(wake_[1]);
  std::lock_guard<std::mutex> g(mu_);
  for (auto& kv : jobs_)
    if (kv.second.state != 2) {
      kv.second.state = 2;
      kv.second.status = -3;
      kv.second.result = "compile pool stopped";
    }
  cv_done_.notify_all();
}

int64_t Pool::submit(const char* src, int64_t len, const char* opts, int64_t prio) {
  Job j;
  j.prio = prio;
  j.src.assign(src, (size_t)len);
  std::string o = opts ? opts : "";
  size_t p = 0;
  while (p < o.size()) {
    size_t e = o.find('\n', p);
    if (e == std::string::npos) e = o.size();
    if (e > p) j.opts.push_back(o.substr(p, e - p));
    p = e + 1;
  }
  char key[32];
  snprintf(key, sizeof key, "%016llx", (unsigned long long)fnv1a(j.src, fnv1a(o)));
  j.key = key;
  if (!cache_dir_.empty()) {
    std::string path = cache_dir_ + "/" + j.key + ".cubin";
    FILE* f = fopen(path.c_str(), "rb");
    if (f) {
      fseek(f, 0, SEEK_END);
      long n = ftell(f);
      fseek(f, 0, SEEK_SET);
      j.result.resize((size_t)n);
      bool ok = n > 0 && fread(&j.result[0], 1, (size_t)n, f) == (size_t)n;
      fclose(f);
      if (ok) {
        j.state = 2;
        j.cache_hit = true;
      }
    }
  }
  std::lock_guard<std::mutex> g(mu_);
  int64_t id = next_id_++;
  bool queued = j.state != 2;
  jobs_.emplace(id, std::move(j));
  if (queued) {
    if (!running_) {
      Job& jj = jobs_[id];
      jj.state = 2;
      jj.status = -3;
      jj.result = "compile pool not started";
    } else {
      queue_.push_back(id);
      char c = 1;
      if (write(wake_[1], &c, 1) < 0) {}
    }
  }
  return id;
}

bool Pool::send(Worker& w, Job& j) {
  uint32_t n = (uint32_t)j.opts.size();
  if (!write_all(w.to, &n, 4)) return false;
  for (auto& o : j.opts) {
    uint32_t l = (uint32_t)o.size();
    if (!write_all(w.to, &l, 4) || !write_all(w.to, o.data(), l)) return false;
  }
  uint32_t l = (uint32_t)j.src.size();
  return write_all(w.to, &l, 4) && write_all(w.to, j.src.data(), l);
}

void Pool::finish(int64_t id, Job& j) {
  j.state = 2;
  if (j.status == 0 && !cache_dir_.empty() && !j.result.empty()) {
    std::string path = cache_dir_ + "/" + j.key + ".cubin";
    std::string tmp = path + ".tmp" + std::to_string((long long)getpid()) + "_" + std::to_string((long long)id);
    FILE* f = fopen(tmp.c_str(), "wb");
    if (f) {
      bool ok = fwrite(j.result.data(), 1, j.result.size(), f) == j.result.size();
      fclose(f);
      if (ok) rename(tmp.c_str(), path.c_str());
      else unlink(tmp.c_str());
    }
  }
  j.src.clear();
  j.src.shrink_to_fit();
}

void Pool::loop() {
  for (;;) {
    std::vector<pollfd> fds;
    {
      std::unique_lock<std::mutex> g(mu_);
      if (!running_) return;
      // hand queued jobs to idle workers
      for (auto& w : workers_) {
        if (w.job || queue_.empty()) continue;
        if (w.pid < 0 && spawn(w)) continue;
        // the oldest batch first, and within it the longest job first (source
        // size ~ ptxas time): shortens a batch's tail
        auto best = queue_.begin();
        for (auto it = queue_.begin(); it != queue_.end(); ++it) {
          const Job& a = jobs_[*it];
          const Job& b = jobs_[*best];
          if (a.prio < b.prio || (a.prio == b.prio && a.src.size() > b.src.size())) best = it;
        }
        int64_t id = *best;
        queue_.erase(best);
        Job& j = jobs_[id];
        j.state = 1;
        j.started = std::chrono::steady_clock::now();
        w.job = id;
        if (!send(w, j)) {  // worker died: respawn and requeue
          kill_worker(w);
          j.state = 0;
          queue_.push_front(id);
        }
      }
      fds.push_back({wake_[0], POLLIN, 0});
      for (auto& w : workers_)
        if (w.job) fds.push_back({w.from, POLLIN, 0});
    }
    int rc = poll(fds.data(), fds.size(), 200);
    if (rc < 0) continue;
    if (fds[0].revents & POLLIN) {
      char buf[256];
      while (read(wake_[0], buf, sizeof buf) > 0) {}
    }
    std::unique_lock<std::mutex> g(mu_);
    if (!running_) return;
    auto now = std::chrono::steady_clock::now();
    for (auto& w : workers_) {
      if (!w.job) continue;
      Job& j = jobs_[w.job];
      bool ready = false;
      for (size_t k = 1; k < fds.size(); ++k)
        if (fds[k].fd == w.from && (fds[k].revents & (POLLIN | POLLHUP | POLLERR))) ready = true;
      if (ready) {
        int32_t st;
        double secs;
        uint32_t len;
        bool ok = read_all(w.from, &st, 4) && read_all(w.from, &secs, 8) && read_all(w.from, &len, 4);
        if (ok) {
          j.result.resize(len);
          ok = len == 0 || read_all(w.from, &j.result[0], len);
        }
        if (!ok) {
          j.status = -2;
          j.result = "compile worker crashed";
          kill_worker(w);
        } else {
          j.status = st;
          j.secs = secs;
        }
        int64_t id = w.job;
        w.job = 0;
        finish(id, j);
        cv_done_.notify_all();
      } else if (std::chrono::duration<double>(now - j.started).count() > timeout_s_) {
        int64_t id = w.job;
        kill_worker(w);
        j.status = -4;
        j.secs = timeout_s_;
        j.result = "compile timeout";
        finish(id, j);
        cv_done_.notify_all();
      }
    }
  }
}

int Pool::wait(int64_t id, int* status, double* secs, int* hit, int64_t* len) {
  std::unique_lock<std::mutex> g(mu_);
  auto it = jobs_.find(id);
  if (it == jobs_.end()) return fail("unknown compile job");
  cv_done_.wait(g, [&] { return it->second.state == 2; });
  *status = it->second.status;
  *secs = it->second.secs;
  *hit = it->second.cache_hit ? 1 : 0;
  *len = (int64_t)it->second.result.size();
  return 0;
}

int Pool::wait_any(const int64_t* ids, int n, double timeout_s) {
  std::unique_lock<std::mutex> g(mu_);
  int hit = -1;
  auto any_done = [&] {
    for (int i = 0; i < n; ++i) {
      auto it = jobs_.find(ids[i]);
      if (it == jobs_.end() || it->second.state == 2) { hit = i; return true; }
    }
    return false;
  };
  cv_done_.wait_for(g, std::chrono::duration<double>(timeout_s), any_done);
  return hit;
}

int Pool::fetch(int64_t id, char* buf, int64_t cap) {
  std::lock_guard<std::mutex> g(mu_);
  auto it = jobs_.find(id);
  if (it == jobs_.end()) return fail("unknown compile job");
  if (it->second.state != 2) return fail("compile job not finished");
  int64_t n = (int64_t)it->second.result.size();
  if (buf && cap >= n && n) memcpy(buf, it->second.result.data(), (size_t)n);
  jobs_.erase(it);
  return 0;
}

static Pool g_pool;

}  // namespace lt

extern "C" {

int lt_pool_start(int n_workers, const char* cache_dir, double timeout_s) {
  return lt::g_pool.start(n_workers, cache_dir ? cache_dir : "", timeout_s);
}

void lt_pool_stop(void) { lt::g_pool.stop(); }

int lt_pool_size(void) { return lt::g_pool.size(); }

// opts: newline-separated NVRTC options.  Returns a job id (> 0).
int64_t lt_compile_submit(const char* src, int64_t len, const char* opts) { return lt::g_pool.submit(src, len, opts); }

// Block until one of the jobs has finished (or is unknown): its index, or -1
// after timeout_s.  Lets the measuring thread sleep instead of polling.
int lt_compile_wait_any(const int64_t* jobs, int n, double timeout_s) {
  return lt::g_pool.wait_any(jobs, n, timeout_s);
}

// As lt_compile_submit, queued behind every job of a lower priority value (a
// later batch compiled ahead of time waits for the current batch's jobs).
int64_t lt_compile_submit_prio(const char* src, int64_t len, const char* opts, int64_t prio) {
  return lt::g_pool.submit(src, len, opts, prio);
}

int lt_compile_wait(int64_t job, int* status, double* secs, int* cache_hit, int64_t* out_len) {
  return lt::g_pool.wait(job, status, secs, cache_hit, out_len);
}

// 1 when the job has finished (wait/fetch will not block), 0 if not, -1 if unknown.
int lt_compile_ready(int64_t job) { return lt::g_pool.ready(job); }

// Copy the finished job's output (cubin, or the compile log on failure) and release the job.
int lt_compile_fetch(int64_t job, char* buf, int64_t cap) { return lt::g_pool.fetch(job, buf, cap); }

}  // extern "C"
