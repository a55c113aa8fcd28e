// Exact-greedy regression-tree fitting on sm_100a.
//
// Replaces `_fit_tree` (reference src/model.py:158-255), the inner loop of the
// reference's `train` (src/model.py:275-320; 45-70% of tuning wall time).  The
// result is bit-identical to the reference, so every floating-point operation
// follows numpy's order (compiled with --fmad=false):
//
//   * per feature, the frontier's rows in (node id, feature value, row) order:
//     the per-feature stable argsort (segmented radix sort of the column, -0.0
//     folded into +0.0 and NaN made canonical so ties keep row order exactly as
//     numpy's stable sort does) filtered and stably bucketed by node;
//   * ONE running float64 sum of w and of w*target along that concatenation,
//     sequential like np.cumsum; left/right sums are differences against the
//     value before the node's first row (src/model.py:179-191);
//   * gain ((sl*sl/max(wl,1e-300)) + (sr*sr/max(wr,1e-300))) - gs*gs/max(gw,1e-300)
//     between distinct neighbouring values with wl>0 and wr>0; per node the
//     FIRST position of the maximum (NaN in a node disqualifies it); features
//     compared in order, replaced only by a strictly larger gain;
//   * leaf value = numpy pairwise sum of w*target over the leaf's rows (row
//     order) / numpy pairwise sum of w (src/model.py:239-247).
//
// Layout: X column-major [nf][n] (one feature = one contiguous column), the
// per-feature sort order, and per-feature scratch columns (bucketed rows, w,
// w*target, value, running sums, gains) all resident in HBM for the whole
// `train` call (one handle per training matrix).  One block per feature does
// the bucketing and gain evaluation in parallel; the running sums are one
// sequential chain per feature (the exactness contract), 164 chains in flight.

#include <cuda_runtime.h>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <vector>
#include "common.h"
#include "npsum.cuh"

namespace lt {

constexpr int GB_THREADS = 128;
constexpr int GB_MAX_FRONTIER = 64;     // depth <= 7
constexpr double GB_TINY = 1e-300;
constexpr double GB_EPS_GAIN = 1e-12;

struct SplitRes {
  double gain;
  double thr;
  int valid;
  int pad;
};

struct Gbdt {
  int64_t n = 0;
  int nf = 0;
  cudaStream_t stream = nullptr;
  double* X = nullptr;          // [nf][n]
  int32_t* order = nullptr;     // [nf][n]
  double* target = nullptr;     // [n]
  double* w = nullptr;          // [n]
  double* wt = nullptr;         // [n]  w * target
  int32_t* node_of = nullptr;   // [n]
  int32_t* grp = nullptr;       // [nf][n] bucketed rows
  double* sw = nullptr;         // [nf][n] running sum of w
  double* swt = nullptr;        // [nf][n] running sum of w*target
  double* gain = nullptr;       // [nf][n]
  SplitRes* res = nullptr;      // [nf][GB_MAX_FRONTIER]
  int32_t* choice_f = nullptr;  // [GB_MAX_FRONTIER]
  double* choice_thr = nullptr;
  int32_t* child = nullptr;     // [GB_MAX_FRONTIER] left child id (or -1)
  double* leaf_buf = nullptr;   // [2][n]
  double* leaf_val = nullptr;   // [2^(depth+1)]
};

__global__ void rows_to_cols_kernel(const double* __restrict__ rows, int64_t n, int nf, double* __restrict__ cols,
                                    double* __restrict__ keys, int32_t* __restrict__ idx) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * nf) return;
  int64_t r = e / nf;
  int f = (int)(e - r * nf);
  double x = rows[e];
  cols[(int64_t)f * n + r] = x;
  // sort key: numpy orders -0.0 == +0.0 and NaN last
  double k = (x == 0.0) ? 0.0 : x;
  if (k != k) k = __longlong_as_double(0x7ff8000000000000LL);
  keys[(int64_t)f * n + r] = k;
  idx[(int64_t)f * n + r] = (int32_t)r;
}

// np.maximum(a, tiny): NaN propagates (fmax would drop it)
__device__ __forceinline__ double npmax(double a, double b) { return (a != a) ? a : fmax(a, b); }

__device__ __forceinline__ unsigned long long ord_key(double g) {
  unsigned long long b = (unsigned long long)__double_as_longlong(g);
  return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// One block per feature: best split of every frontier node [lo, lo+K) on it.
__global__ void __launch_bounds__(GB_THREADS)
split_kernel(Gbdt g, int lo, int K) {
  const int f = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t n = g.n;
  const int32_t* ord = g.order + (int64_t)f * n;
  const double* xf = g.X + (int64_t)f * n;
  int32_t* grp = g.grp + (int64_t)f * n;
  double* sw = g.sw + (int64_t)f * n;
  double* swt = g.swt + (int64_t)f * n;
  double* gain = g.gain + (int64_t)f * n;

  __shared__ int cnt[GB_MAX_FRONTIER][GB_THREADS + 1];
  __shared__ int64_t start[GB_MAX_FRONTIER + 1];
  __shared__ unsigned long long gmax[GB_MAX_FRONTIER];
  __shared__ int gfirst[GB_MAX_FRONTIER];
  __shared__ int gnan[GB_MAX_FRONTIER];

  const int64_t chunk = (n + GB_THREADS - 1) / GB_THREADS;
  const int64_t c0 = t * chunk, c1 = min(n, c0 + chunk);
  for (int k = 0; k < K; ++k) cnt[k][t] = 0;
  for (int64_t i = c0; i < c1; ++i) {
    int k = g.node_of[ord[i]] - lo;
    if (k >= 0 && k < K) cnt[k][t]++;
  }
  __syncthreads();
  if (t < K) {            // within-node offsets of each thread's chunk
    int run = 0;
    for (int u = 0; u < GB_THREADS; ++u) {
      int c = cnt[t][u];
      cnt[t][u] = run;
      run += c;
    }
    cnt[t][GB_THREADS] = run;
    gmax[t] = ord_key(-INFINITY);
    gfirst[t] = 0x7fffffff;
    gnan[t] = 0;
  }
  __syncthreads();
  if (t == 0) {
    int64_t s = 0;
    for (int k = 0; k < K; ++k) { start[k] = s; s += cnt[k][GB_THREADS]; }
    start[K] = s;
  }
  __syncthreads();
  const int64_t n_act = start[K];
  // stable bucketing by node, value order kept inside a node
  {
    int off[GB_MAX_FRONTIER];
    for (int k = 0; k < K; ++k) off[k] = cnt[k][t];
    for (int64_t i = c0; i < c1; ++i) {
      int r = ord[i];
      int k = g.node_of[r] - lo;
      if (k >= 0 && k < K) {
        int64_t pos = start[k] + off[k]++;
        grp[pos] = r;
        sw[pos] = g.w[r];        // gathered now; prefix-summed in place below
        swt[pos] = g.wt[r];
      }
    }
  }
  __syncthreads();
  if (n_act < 2) {
    if (t < K) g.res[f * GB_MAX_FRONTIER + t].valid = 0;
    return;
  }
  // the sequential running sums (np.cumsum order)
  if (t == 0) {
    double a = 0.0, b = 0.0;
    for (int64_t i = 0; i < n_act; ++i) {
      a = __dadd_rn(a, sw[i]);
      b = __dadd_rn(b, swt[i]);
      sw[i] = a;
      swt[i] = b;
    }
  }
  __syncthreads();
  // gains, per-node maximum (first position), NaN flags
  for (int64_t i = t; i < n_act; i += GB_THREADS) {
    int k = 0;
    while (k + 1 < K && start[k + 1] <= i) ++k;
    const int64_t a = start[k], b = start[k + 1];
    double gv = -INFINITY;
    if (i < b - 1) {
      const double bw = a > 0 ? sw[a - 1] : 0.0, bs = a > 0 ? swt[a - 1] : 0.0;
      const double gw = __dsub_rn(sw[b - 1], bw), gs = __dsub_rn(swt[b - 1], bs);
      const double wl = __dsub_rn(sw[i], bw), sl = __dsub_rn(swt[i], bs);
      const double wr = __dsub_rn(gw, wl), sr = __dsub_rn(gs, sl);
      const double x0 = xf[grp[i]], x1 = xf[grp[i + 1]];
      if (x0 != x1 && wl > 0.0 && wr > 0.0) {
        const double parent = __ddiv_rn(__dmul_rn(gs, gs), npmax(gw, GB_TINY));
        gv = __dsub_rn(__dadd_rn(__ddiv_rn(__dmul_rn(sl, sl), npmax(wl, GB_TINY)),
                                 __ddiv_rn(__dmul_rn(sr, sr), npmax(wr, GB_TINY))),
                       parent);
      }
    }
    gain[i] = gv;
    if (gv != gv) gnan[k] = 1;
    else atomicMax(&gmax[k], ord_key(gv));
  }
  __syncthreads();
  for (int64_t i = t; i < n_act; i += GB_THREADS) {
    int k = 0;
    while (k + 1 < K && start[k + 1] <= i) ++k;
    double gv = gain[i];
    if (gv == gv && ord_key(gv) == gmax[k]) atomicMin(&gfirst[k], (int)i);
  }
  __syncthreads();
  if (t < K) {
    SplitRes r;
    r.valid = 0;
    r.gain = 0.0;
    r.thr = 0.0;
    r.pad = 0;
    const unsigned long long m = gmax[t];
    const double gm = __longlong_as_double((long long)((m & 0x8000000000000000ULL) ? (m & 0x7fffffffffffffffULL)
                                                                                     : ~m));
    if (!gnan[t] && start[t + 1] > start[t] && gm > GB_EPS_GAIN && isfinite(gm) && gfirst[t] != 0x7fffffff) {
      const int p = gfirst[t];
      r.valid = 1;
      r.gain = gm;
      r.thr = __dmul_rn(0.5, __dadd_rn(xf[grp[p]], xf[grp[p + 1]]));
    }
    g.res[f * GB_MAX_FRONTIER + t] = r;
  }
}

// Best feature per frontier node: features in order, strictly larger gain wins.
__global__ void choose_kernel(Gbdt g, int K) {
  const int k = threadIdx.x;
  if (k >= K) return;
  int bf = -1;
  double bg = 0.0, bt = 0.0;
  for (int f = 0; f < g.nf; ++f) {
    const SplitRes r = g.res[f * GB_MAX_FRONTIER + k];
    if (r.valid && (bf < 0 || r.gain > bg)) { bf = f; bg = r.gain; bt = r.thr; }
  }
  g.choice_f[k] = bf;
  g.choice_thr[k] = bt;
}

__global__ void route_kernel(Gbdt g, int lo, int K) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= g.n) return;
  const int k = g.node_of[r] - lo;
  if (k < 0 || k >= K) return;
  const int f = g.choice_f[k];
  if (f < 0) return;
  const int c = g.child[k];
  g.node_of[r] = (g.X[(int64_t)f * g.n + r] <= g.choice_thr[k]) ? c : c + 1;
}

__global__ void wt_kernel(Gbdt g) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < g.n) g.wt[r] = __dmul_rn(g.w[r], g.target[r]);
}

// One block per leaf: the leaf's rows in row order, then numpy's sums.
__global__ void __launch_bounds__(GB_THREADS)
leaf_kernel(Gbdt g, const int32_t* __restrict__ leaves, int n_leaves) {
  const int L = blockIdx.x;
  if (L >= n_leaves) return;
  const int nd = leaves[L];
  double* bw = g.leaf_buf + (int64_t)L * 2 * g.n;
  double* bwt = bw + g.n;
  __shared__ int64_t tot[GB_THREADS + 1];
  const int t = threadIdx.x;
  const int64_t chunk = (g.n + GB_THREADS - 1) / GB_THREADS;
  const int64_t c0 = t * chunk, c1 = min(g.n, c0 + chunk);
  int64_t c = 0;
  for (int64_t r = c0; r < c1; ++r) c += g.node_of[r] == nd;
  tot[t] = c;
  __syncthreads();
  if (t == 0) {
    int64_t s = 0;
    for (int u = 0; u < GB_THREADS; ++u) { int64_t v = tot[u]; tot[u] = s; s += v; }
    tot[GB_THREADS] = s;
  }
  __syncthreads();
  int64_t pos = tot[t];
  for (int64_t r = c0; r < c1; ++r)
    if (g.node_of[r] == nd) { bw[pos] = g.w[r]; bwt[pos] = g.wt[r]; ++pos; }
  __syncthreads();
  if (t == 0) {
    const int64_t m = tot[GB_THREADS];
    const double s = np_pairwise(bw, m);
    g.leaf_val[nd] = s > 0.0 ? __ddiv_rn(np_pairwise(bwt, m), s) : 0.0;
  }
}

}  // namespace lt

using lt::Gbdt;

extern "C" {

void lt_gbdt_destroy(int64_t h) {
  Gbdt* g = (Gbdt*)(intptr_t)h;
  if (!g) return;
  for (void* p : {(void*)g->X, (void*)g->order, (void*)g->target, (void*)g->w, (void*)g->wt, (void*)g->node_of,
                  (void*)g->grp, (void*)g->sw, (void*)g->swt, (void*)g->gain, (void*)g->res, (void*)g->choice_f,
                  (void*)g->choice_thr, (void*)g->child, (void*)g->leaf_buf, (void*)g->leaf_val})
    if (p) cudaFree(p);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

// Upload a training matrix (host rows[n][nf]) and sort every feature column once
// (the matrix is shared by all trees of one `train` call).
int64_t lt_gbdt_create(const double* rows, int64_t n, int nf) {
  if (n <= 0 || nf <= 0 || n * nf > 0x7fffffff) { lt::fail("gbdt: bad matrix shape"); return 0; }
  Gbdt* g = new Gbdt();
  g->n = n;
  g->nf = nf;
  const size_t cells = (size_t)n * nf;
  double* d_rows = nullptr;
  double *keys = nullptr, *keys_out = nullptr;
  int32_t* idx = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  std::vector<int64_t> seg(nf + 1);
  int64_t* d_seg = nullptr;
  bool ok = !lt::check_cuda(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking), "gbdt stream") &&
            !lt::check_cuda(cudaMalloc(&g->X, cells * 8), "gbdt X") &&
            !lt::check_cuda(cudaMalloc(&g->order, cells * 4), "gbdt order") &&
            !lt::check_cuda(cudaMalloc(&g->grp, cells * 4), "gbdt grp") &&
            !lt::check_cuda(cudaMalloc(&g->sw, cells * 8), "gbdt sw") &&
            !lt::check_cuda(cudaMalloc(&g->swt, cells * 8), "gbdt swt") &&
            !lt::check_cuda(cudaMalloc(&g->gain, cells * 8), "gbdt gain") &&
            !lt::check_cuda(cudaMalloc(&g->target, n * 8), "gbdt target") &&
            !lt::check_cuda(cudaMalloc(&g->w, n * 8), "gbdt w") &&
            !lt::check_cuda(cudaMalloc(&g->wt, n * 8), "gbdt wt") &&
            !lt::check_cuda(cudaMalloc(&g->node_of, n * 4), "gbdt node_of") &&
            !lt::check_cuda(cudaMalloc(&g->res, (size_t)nf * lt::GB_MAX_FRONTIER * sizeof(lt::SplitRes)), "res") &&
            !lt::check_cuda(cudaMalloc(&g->choice_f, lt::GB_MAX_FRONTIER * 4), "choice") &&
            !lt::check_cuda(cudaMalloc(&g->choice_thr, lt::GB_MAX_FRONTIER * 8), "choice") &&
            !lt::check_cuda(cudaMalloc(&g->child, lt::GB_MAX_FRONTIER * 4), "child") &&
            !lt::check_cuda(cudaMalloc(&g->leaf_buf, (size_t)lt::GB_MAX_FRONTIER * 2 * 2 * n * 8), "leaf buf") &&
            !lt::check_cuda(cudaMalloc(&g->leaf_val, 512 * 8), "leaf val") &&
            !lt::check_cuda(cudaMalloc(&d_rows, cells * 8), "gbdt rows") &&
            !lt::check_cuda(cudaMalloc(&keys, cells * 8), "gbdt keys") &&
            !lt::check_cuda(cudaMalloc(&keys_out, cells * 8), "gbdt keys") &&
            !lt::check_cuda(cudaMalloc(&idx, cells * 4), "gbdt idx") &&
            !lt::check_cuda(cudaMalloc(&d_seg, (nf + 1) * 8), "gbdt seg");
  if (ok) {
    for (int f = 0; f <= nf; ++f) seg[f] = (int64_t)f * n;
    cudaMemcpyAsync(d_seg, seg.data(), (nf + 1) * 8, cudaMemcpyHostToDevice, g->stream);
    cudaMemcpyAsync(d_rows, rows, cells * 8, cudaMemcpyHostToDevice, g->stream);
    lt::rows_to_cols_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, g->stream>>>(d_rows, n, nf, g->X, keys, idx);
    // stable per-column sort (radix sort is stable: ties keep row order)
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_out, idx, g->order, (int)cells, nf,
                                             d_seg, d_seg + 1, 0, 64, g->stream);
    ok = !lt::check_cuda(cudaMalloc(&tmp, tmp_bytes > 0 ? tmp_bytes : 16), "gbdt sort tmp");
    if (ok) {
      cub::DeviceSegmentedRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_out, idx, g->order, (int)cells, nf,
                                               d_seg, d_seg + 1, 0, 64, g->stream);
      ok = !lt::check_cuda(cudaStreamSynchronize(g->stream), "gbdt sort");
    }
  }
  for (void* p : {(void*)d_rows, (void*)keys, (void*)keys_out, (void*)idx, tmp, (void*)d_seg})
    if (p) cudaFree(p);
  if (!ok) {
    lt_gbdt_destroy((int64_t)(intptr_t)g);
    return 0;
  }
  return (int64_t)(intptr_t)g;
}

// One tree (src/model.py:158-255) for targets/weights target[n], w[n].  Node
// arrays (capacity `cap` >= 2^(depth+1)-1) are written in the reference's
// numbering; *n_nodes receives the node count.
int lt_gbdt_fit_tree(int64_t h, const double* target, const double* w, int depth, int cap, int32_t* feature,
                     double* threshold, int32_t* left, int32_t* right, double* value, int32_t* n_nodes) {
  Gbdt* g = (Gbdt*)(intptr_t)h;
  if (!g) return lt::fail("gbdt: null handle");
  if (depth < 1 || depth > 7 || cap < (2 << depth) - 1) return lt::fail("gbdt: depth must be 1..7 with room for nodes");
  const int64_t n = g->n;
  cudaStream_t s = g->stream;
  cudaMemcpyAsync(g->target, target, n * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(g->w, w, n * 8, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(g->node_of, 0, n * 4, s);
  const unsigned rb = (unsigned)((n + 255) / 256);
  lt::wt_kernel<<<rb, 256, 0, s>>>(*g);
  std::vector<int32_t> feat(1, -1), lf(1, 0), rt(1, 0);
  std::vector<double> thr(1, 0.0);
  int lo = 0, K = 1;
  int32_t h_choice_f[lt::GB_MAX_FRONTIER];
  double h_choice_thr[lt::GB_MAX_FRONTIER];
  for (int level = 0; level < depth && K > 0; ++level) {
    lt::split_kernel<<<g->nf, lt::GB_THREADS, 0, s>>>(*g, lo, K);
    lt::choose_kernel<<<1, lt::GB_MAX_FRONTIER, 0, s>>>(*g, K);
    cudaMemcpyAsync(h_choice_f, g->choice_f, K * 4, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h_choice_thr, g->choice_thr, K * 8, cudaMemcpyDeviceToHost, s);
    if (lt::check_cuda(cudaStreamSynchronize(s), "gbdt split")) return -1;
    int32_t h_child[lt::GB_MAX_FRONTIER];
    int next_lo = (int)feat.size(), next_k = 0;
    for (int k = 0; k < K; ++k) {          // children numbered in frontier order
      const int nd = lo + k;
      if (h_choice_f[k] < 0) { h_child[k] = -1; continue; }
      const int li = (int)feat.size();
      feat[nd] = h_choice_f[k];
      thr[nd] = h_choice_thr[k];
      lf[nd] = li;
      rt[nd] = li + 1;
      feat.insert(feat.end(), {-1, -1});
      thr.insert(thr.end(), {0.0, 0.0});
      lf.insert(lf.end(), {0, 0});
      rt.insert(rt.end(), {0, 0});
      h_child[k] = li;
      next_k += 2;
    }
    cudaMemcpyAsync(g->child, h_child, K * 4, cudaMemcpyHostToDevice, s);
    lt::route_kernel<<<rb, 256, 0, s>>>(*g, lo, K);
    lo = next_lo;
    K = next_k;
  }
  const int nn = (int)feat.size();
  if (nn > cap) return lt::fail("gbdt: node capacity exceeded");
  std::vector<int32_t> leaves;
  for (int i = 0; i < nn; ++i)
    if (feat[i] < 0) leaves.push_back(i);
  int32_t* d_leaves = nullptr;
  if (lt::check_cuda(cudaMalloc(&d_leaves, leaves.size() * 4), "gbdt leaves")) return -1;
  cudaMemcpyAsync(d_leaves, leaves.data(), leaves.size() * 4, cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(g->leaf_val, 0, nn * 8, s);
  lt::leaf_kernel<<<(unsigned)leaves.size(), lt::GB_THREADS, 0, s>>>(*g, d_leaves, (int)leaves.size());
  std::vector<double> val(nn);
  cudaMemcpyAsync(val.data(), g->leaf_val, nn * 8, cudaMemcpyDeviceToHost, s);
  int st = lt::check_cuda(cudaStreamSynchronize(s), "gbdt leaves");
  cudaFree(d_leaves);
  if (st) return -1;
  for (int i = 0; i < nn; ++i) {
    feature[i] = feat[i];
    threshold[i] = thr[i];
    left[i] = lf[i];
    right[i] = rt[i];
    value[i] = feat[i] < 0 ? val[i] : 0.0;
  }
  *n_nodes = nn;
  return 0;
}

}  // extern "C"
