// GBDT inference over whole populations on sm_100a.
//
// Replaces `Tree.predict` / `CostModel.predict_rows` / `predict_matrix`
// (reference src/model.py:75-108).  Exactness contract, matching numpy:
//   * routing `x <= threshold` -> left, else right (NaN goes right), in fp64;
//   * per row: acc = base, then acc += value[leaf] * eta tree by tree in list
//     order (the product is precomputed on the host with the same IEEE multiply);
//   * per program: numpy's add.reduce order over its rows (plain loop below 8
//     rows, numpy's 8-accumulator pairwise scheme above).
// Layout (predict_trees_kernel, the default): one tree per warp.  Each block
// copies the whole model into shared memory once (16 B per node: 61 KB at 30
// trees x 127 nodes) and loops over tiles of TILE_ROWS rows (persistent grid):
// the tile's tested feature columns are staged into shared memory with
// coalesced loads; warp w walks trees w, w+W, ... for the tile's rows (one row
// per lane), every level a shared-memory node load and a shared-memory feature
// load, and writes each (tree, row) leaf into a shared partials table; then one
// thread per row adds base + partials in tree order — the reference's
// summation order, so results are bit-identical.  Models too large for shared
// memory use predict_rows_kernel (thread per row, nodes read through L1).
// Compiled with --fmad=false.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <vector>
#include <tuple>
#include <string>
#include "common.h"
#include "npsum.cuh"

namespace lt {

constexpr int NF = 164;
constexpr int ROWS_PER_BLOCK = 128;

struct Node {
  double x;        // threshold (internal) or value*eta (leaf)
  int32_t feat;    // compact feature column, -1 at leaves
  int32_t lr;      // left | right << 16 (tree-local node ids)
};

struct Model {
  int n_trees = 0;
  int n_nodes = 0;
  int depth = -1;              // perfect layout depth D (-1: not available)
  double* d_pthr = nullptr;    // [n_trees][2^D - 1] thresholds
  int32_t* d_pfeat = nullptr;  // [n_trees][2^D - 1] compact feature columns
  double* d_pval = nullptr;    // [n_trees][2^D] leaf value*eta
  int n_used = 0;          // compact feature columns
  double base = 0.0;
  Node* d_nodes = nullptr;
  int32_t* d_tree_off = nullptr;
  int32_t* d_used = nullptr;   // compact col -> original feature index
};

__global__ void __launch_bounds__(ROWS_PER_BLOCK)
predict_rows_kernel(const double* __restrict__ X, int64_t n_rows, bool col_major, const Node* __restrict__ nodes,
                    const int32_t* __restrict__ tree_off, int n_trees, const int32_t* __restrict__ used,
                    int n_used, double base, double* __restrict__ out) {
  extern __shared__ double tile[];             // ROWS_PER_BLOCK x (n_used + 1)
  const int ld = n_used + 1;                   // odd stride: conflict-free row access
  const int64_t row0 = (int64_t)blockIdx.x * ROWS_PER_BLOCK;
  const int rows_here = (int)min((int64_t)ROWS_PER_BLOCK, n_rows - row0);
  if (col_major) {            // X[164][n_rows]: consecutive threads read consecutive rows
    for (int e = threadIdx.x; e < rows_here * n_used; e += blockDim.x) {
      int c = e / rows_here, r = e - c * rows_here;
      tile[r * ld + c] = X[(int64_t)used[c] * n_rows + row0 + r];
    }
  } else {
    for (int e = threadIdx.x; e < rows_here * n_used; e += blockDim.x) {
      int r = e / n_used, c = e - r * n_used;
      tile[r * ld + c] = X[(row0 + r) * NF + used[c]];
    }
  }
  __syncthreads();
  const int r = threadIdx.x;
  if (r >= rows_here) return;
  const double* x = tile + r * ld;
  double acc = base;
  for (int t = 0; t < n_trees; ++t) {
    const Node* nd = nodes + tree_off[t];
    Node cur = nd[0];
    for (int lvl = 0; lvl < 64 && cur.feat >= 0; ++lvl) {
      int nxt = (x[cur.feat] <= cur.x) ? (cur.lr & 0xffff) : (cur.lr >> 16);
      cur = nd[nxt];
    }
    acc = __dadd_rn(acc, cur.x);
  }
  out[row0 + r] = acc;
}

constexpr int TILE_ROWS = 64;
constexpr int TREE_WARPS = 16;

__global__ void __launch_bounds__(TREE_WARPS * 32)
predict_trees_kernel(const double* __restrict__ X, int64_t n_rows, bool col_major, const Node* __restrict__ nodes,
                     int n_nodes, const int32_t* __restrict__ tree_off, int n_trees,
                     const int32_t* __restrict__ used, int n_used, double base, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Node* s_nodes = (Node*)smem_raw;                                   // n_nodes
  double* tile = (double*)(s_nodes + n_nodes);                       // n_used x TILE_ROWS (column-major)
  double* part = tile + (size_t)n_used * TILE_ROWS;                  // n_trees x TILE_ROWS
  int32_t* s_off = (int32_t*)(part + (size_t)n_trees * TILE_ROWS);   // n_trees + 1
  for (int i = threadIdx.x; i < n_nodes; i += blockDim.x) s_nodes[i] = nodes[i];
  for (int i = threadIdx.x; i <= n_trees; i += blockDim.x) s_off[i] = tree_off[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t row0 = (int64_t)blockIdx.x * TILE_ROWS; row0 < n_rows; row0 += (int64_t)gridDim.x * TILE_ROWS) {
    const int rows_here = (int)min((int64_t)TILE_ROWS, n_rows - row0);
    __syncthreads();                      // previous tile fully consumed (and the model staged)
    if (col_major) {                      // X[164][n_rows]: a column's rows are contiguous
      for (int e = threadIdx.x; e < n_used * TILE_ROWS; e += blockDim.x) {
        const int c = e / TILE_ROWS, r = e - c * TILE_ROWS;
        if (r < rows_here) tile[e] = X[(int64_t)used[c] * n_rows + row0 + r];
      }
    } else {
      for (int e = threadIdx.x; e < n_used * TILE_ROWS; e += blockDim.x) {
        const int r = e / n_used, c = e - r * n_used;
        if (r < rows_here) tile[c * TILE_ROWS + r] = X[(row0 + r) * NF + used[c]];
      }
    }
    __syncthreads();
    for (int t = warp; t < n_trees; t += TREE_WARPS) {
      const Node* nd = s_nodes + s_off[t];
      for (int r = lane; r < rows_here; r += 32) {
        Node cur = nd[0];
        for (int lvl = 0; lvl < 64 && cur.feat >= 0; ++lvl) {
          const int nxt = (tile[cur.feat * TILE_ROWS + r] <= cur.x) ? (cur.lr & 0xffff) : (cur.lr >> 16);
          cur = nd[nxt];
        }
        part[t * TILE_ROWS + r] = cur.x;
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rows_here; r += blockDim.x) {
      double acc = base;
      for (int t = 0; t < n_trees; ++t) acc = __dadd_rn(acc, part[t * TILE_ROWS + r]);
      out[row0 + r] = acc;
    }
  }
}

// Perfect-tree walk: every tree padded to a complete tree of depth D (a leaf
// above the bottom level is replicated into all bottom leaves below it, so the
// direction taken under it does not matter, NaN included).  Each level is one
// shared threshold load, one shared feature load and a compare: child =
// 2*i + 1 + !(x <= thr), no per-node child indices, no data-dependent trip count
// (the warp stays converged).  Same comparisons, leaf values and per-row
// summation order as the other kernels: bit-identical scores.
constexpr int MAX_PERFECT_DEPTH = 7;

__global__ void __launch_bounds__(TREE_WARPS * 32)
predict_perfect_kernel(const double* __restrict__ X, int64_t n_rows, bool col_major, const double* __restrict__ pthr,
                       const int32_t* __restrict__ pfeat, const double* __restrict__ pval, int depth, int n_trees,
                       const int32_t* __restrict__ used, int n_used, double base, double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n_int = (1 << depth) - 1, n_leaf = 1 << depth;
  double* s_thr = (double*)smem_raw;                                  // n_trees x n_int
  double* s_val = s_thr + (size_t)n_trees * n_int;                    // n_trees x n_leaf
  double* tile = s_val + (size_t)n_trees * n_leaf;                    // n_used x TILE_ROWS
  double* part = tile + (size_t)n_used * TILE_ROWS;                   // n_trees x TILE_ROWS
  int32_t* s_feat = (int32_t*)(part + (size_t)n_trees * TILE_ROWS);   // n_trees x n_int
  for (int i = threadIdx.x; i < n_trees * n_int; i += blockDim.x) {
    s_thr[i] = pthr[i];
    s_feat[i] = pfeat[i] * TILE_ROWS;                                 // pre-scaled tile column offset
  }
  for (int i = threadIdx.x; i < n_trees * n_leaf; i += blockDim.x) s_val[i] = pval[i];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t row0 = (int64_t)blockIdx.x * TILE_ROWS; row0 < n_rows; row0 += (int64_t)gridDim.x * TILE_ROWS) {
    const int rows_here = (int)min((int64_t)TILE_ROWS, n_rows - row0);
    __syncthreads();
    if (col_major) {
      for (int e = threadIdx.x; e < n_used * TILE_ROWS; e += blockDim.x) {
        const int c = e / TILE_ROWS, r = e - c * TILE_ROWS;
        if (r < rows_here) tile[e] = X[(int64_t)used[c] * n_rows + row0 + r];
      }
    } else {
      for (int e = threadIdx.x; e < n_used * TILE_ROWS; e += blockDim.x) {
        const int r = e / n_used, c = e - r * n_used;
        if (r < rows_here) tile[c * TILE_ROWS + r] = X[(row0 + r) * NF + used[c]];
      }
    }
    __syncthreads();
    for (int t = warp; t < n_trees; t += TREE_WARPS) {
      const double* thr = s_thr + t * n_int;
      const int32_t* feat = s_feat + t * n_int;
      for (int r = lane; r < rows_here; r += 32) {
        int i = 0;
        for (int lvl = 0; lvl < depth; ++lvl) i = 2 * i + 1 + (tile[feat[i] + r] <= thr[i] ? 0 : 1);
        part[t * TILE_ROWS + r] = s_val[t * n_leaf + (i - n_int)];
      }
    }
    __syncthreads();
    for (int r = threadIdx.x; r < rows_here; r += blockDim.x) {
      double acc = base;
      for (int t = 0; t < n_trees; ++t) acc = __dadd_rn(acc, part[t * TILE_ROWS + r]);
      out[row0 + r] = acc;
    }
  }
}

__global__ void segment_sum_kernel(const double* __restrict__ row_scores, const int64_t* __restrict__ prog_off,
                                   int64_t n_prog, double* __restrict__ out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_prog) return;
  int64_t lo = prog_off[p], hi = prog_off[p + 1];
  out[p] = np_pairwise(row_scores + lo, hi - lo);
}

}  // namespace lt

using lt::Model;
using lt::Node;

extern "C" {

// Build a device-resident model from the reference's CostModel.to_json arrays
// (src/model.py:110-125), trees concatenated; node ids are tree-local.
int64_t lt_model_create(int n_trees, const int64_t* tree_node_off, const int32_t* feature,
                        const double* threshold, const int32_t* left, const int32_t* right,
                        const double* value, const double* eta, double base, int n_features) {
  if (n_features != lt::NF) { lt::fail("model was built for a different feature layout"); return 0; }
  std::vector<int> remap(lt::NF, -1);
  std::vector<int32_t> used;
  int64_t total = tree_node_off[n_trees];
  std::vector<Node> nodes((size_t)(total > 0 ? total : 1));
  std::vector<int32_t> toff(n_trees + 1);
  for (int t = 0; t < n_trees; ++t) {
    int64_t o = tree_node_off[t], n = tree_node_off[t + 1] - o;
    if (n <= 0 || n > 65535) { lt::fail("tree node count out of range"); return 0; }
    toff[t] = (int32_t)o;
    for (int64_t i = 0; i < n; ++i) {
      int32_t f = feature[o + i];
      Node nd;
      if (f >= 0) {
        if (f >= lt::NF) { lt::fail("feature index out of range"); return 0; }
        if (remap[f] < 0) { remap[f] = (int)used.size(); used.push_back(f); }
        int32_t l = left[o + i], r = right[o + i];
        if (l < 0 || l >= n || r < 0 || r >= n) { lt::fail("child index out of range"); return 0; }
        nd.x = threshold[o + i];
        nd.feat = remap[f];
        nd.lr = l | (r << 16);
      } else {
        volatile double v = value[o + i];
        volatile double e = eta[t];
        nd.x = v * e;                 // IEEE product, same as numpy's value[idx] * eta
        nd.feat = -1;
        nd.lr = 0;
      }
      nodes[o + i] = nd;
    }
  }
  toff[n_trees] = (int32_t)total;
  if (used.empty()) used.push_back(0);
  // perfect layout (see predict_perfect_kernel) when every tree is at most 7 deep
  int depth = 0;
  bool perfect = true;
  std::vector<int> level;
  for (int t = 0; t < n_trees && perfect; ++t) {
    int64_t o = tree_node_off[t], n = tree_node_off[t + 1] - o;
    level.assign((size_t)n, -1);
    level[0] = 0;
    for (int64_t i = 0; i < n; ++i) {            // children follow their parent (breadth-first ids)
      if (level[i] < 0) { perfect = false; break; }
      if (feature[o + i] >= 0) {
        for (int32_t c : {left[o + i], right[o + i]}) {
          if (c <= i || level[c] >= 0) { perfect = false; break; }
          level[c] = level[i] + 1;
        }
        if (!perfect) break;
      } else if (level[i] > depth) {
        depth = level[i];
      }
    }
    if (depth > lt::MAX_PERFECT_DEPTH) perfect = false;
  }
  std::vector<double> pthr, pval;
  std::vector<int32_t> pfeat;
  if (perfect && n_trees > 0) {
    const int n_int = (1 << depth) - 1, n_leaf = 1 << depth;
    pthr.assign((size_t)n_trees * n_int, 0.0);
    pfeat.assign((size_t)n_trees * n_int, 0);
    pval.assign((size_t)n_trees * n_leaf, 0.0);
    for (int t = 0; t < n_trees; ++t) {
      const int64_t o = tree_node_off[t];
      // (node, perfect position, level) work list
      std::vector<std::tuple<int64_t, int, int>> work{{0, 0, 0}};
      while (!work.empty()) {
        auto [nd, pos, lv] = work.back();
        work.pop_back();
        if (feature[o + nd] >= 0) {
          pthr[(size_t)t * n_int + pos] = nodes[o + nd].x;
          pfeat[(size_t)t * n_int + pos] = nodes[o + nd].feat;
          work.push_back({left[o + nd], 2 * pos + 1, lv + 1});
          work.push_back({right[o + nd], 2 * pos + 2, lv + 1});
        } else {
          // replicate the leaf into every bottom position under pos
          int first = pos, span = 1;
          for (int k = lv; k < depth; ++k) { first = 2 * first + 1; span *= 2; }
          for (int j = 0; j < span; ++j) pval[(size_t)t * n_leaf + (first - n_int) + j] = nodes[o + nd].x;
        }
      }
    }
  }
  Model* m = new Model();
  m->n_trees = n_trees;
  m->n_nodes = (int)nodes.size();
  m->n_used = (int)used.size();
  m->base = base;
  if (lt::check_cuda(cudaMalloc(&m->d_nodes, nodes.size() * sizeof(Node)), "cudaMalloc nodes") ||
      lt::check_cuda(cudaMalloc(&m->d_tree_off, toff.size() * sizeof(int32_t)), "cudaMalloc toff") ||
      lt::check_cuda(cudaMalloc(&m->d_used, used.size() * sizeof(int32_t)), "cudaMalloc used")) {
    delete m;
    return 0;
  }
  cudaMemcpy(m->d_nodes, nodes.data(), nodes.size() * sizeof(Node), cudaMemcpyHostToDevice);
  cudaMemcpy(m->d_tree_off, toff.data(), toff.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(m->d_used, used.data(), used.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (!pthr.empty()) {
    if (lt::check_cuda(cudaMalloc(&m->d_pthr, pthr.size() * sizeof(double)), "cudaMalloc pthr") ||
        lt::check_cuda(cudaMalloc(&m->d_pfeat, pfeat.size() * sizeof(int32_t)), "cudaMalloc pfeat") ||
        lt::check_cuda(cudaMalloc(&m->d_pval, pval.size() * sizeof(double)), "cudaMalloc pval")) {
      delete m;
      return 0;
    }
    cudaMemcpy(m->d_pthr, pthr.data(), pthr.size() * sizeof(double), cudaMemcpyHostToDevice);
    cudaMemcpy(m->d_pfeat, pfeat.data(), pfeat.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    cudaMemcpy(m->d_pval, pval.data(), pval.size() * sizeof(double), cudaMemcpyHostToDevice);
    m->depth = depth;
  }
  if (lt::check_cuda(cudaGetLastError(), "model upload")) { delete m; return 0; }
  return (int64_t)(intptr_t)m;
}

void lt_model_destroy(int64_t handle) {
  Model* m = (Model*)(intptr_t)handle;
  if (!m) return;
  cudaFree(m->d_nodes);
  cudaFree(m->d_tree_off);
  cudaFree(m->d_used);
  if (m->d_pthr) cudaFree(m->d_pthr);
  if (m->d_pfeat) cudaFree(m->d_pfeat);
  if (m->d_pval) cudaFree(m->d_pval);
  delete m;
}

int lt_model_info(int64_t handle, int* n_trees, int* n_used_features) {
  Model* m = (Model*)(intptr_t)handle;
  if (!m) return lt::fail("null model");
  *n_trees = m->n_trees;
  *n_used_features = m->n_used;
  return 0;
}

static int device_props(int* sms, size_t* smem_optin) {
  static int cached_dev = -1, cached_sms = 0;
  static size_t cached_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    int v = 0;
    cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cached_smem = (size_t)v;
    cached_dev = dev;
  }
  *sms = cached_sms;
  *smem_optin = cached_smem;
  return dev;
}

static int predict_device(int64_t handle, const double* d_rows, int64_t n_rows, bool col_major,
                          double* d_row_scores, void* stream) {
  Model* m = (Model*)(intptr_t)handle;
  if (!m) return lt::fail("null model");
  if (n_rows <= 0) return 0;
  int sms = 0;
  size_t optin = 0;
  const int tdev = device_props(&sms, &optin);
  if (m->depth >= 0 && getenv("LT_PREDICT_IRREGULAR") == nullptr && getenv("LT_PREDICT_THREAD_PER_ROW") == nullptr) {
    const size_t n_int = ((size_t)1 << m->depth) - 1, n_leaf = (size_t)1 << m->depth;
    const size_t psmem = (size_t)m->n_trees * (n_int + n_leaf) * sizeof(double) +
                         (size_t)(m->n_used + m->n_trees) * lt::TILE_ROWS * sizeof(double) +
                         (size_t)m->n_trees * n_int * sizeof(int32_t);
    if (psmem <= optin) {
      static size_t pconfigured[64] = {};
      if (psmem > 48 * 1024 && (tdev < 0 || tdev >= 64 || psmem > pconfigured[tdev])) {
        if (lt::check_cuda(cudaFuncSetAttribute(lt::predict_perfect_kernel,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem),
                           "smem attr"))
          return -1;
        if (tdev >= 0 && tdev < 64) pconfigured[tdev] = psmem;
      }
      const int per_sm = psmem <= optin / 2 ? 2 : 1;
      int64_t tiles = (n_rows + lt::TILE_ROWS - 1) / lt::TILE_ROWS;
      int64_t blocks = (int64_t)sms * per_sm;
      if (blocks > tiles) blocks = tiles;
      lt::predict_perfect_kernel<<<(unsigned)blocks, lt::TREE_WARPS * 32, psmem, (cudaStream_t)stream>>>(
          d_rows, n_rows, col_major, m->d_pthr, m->d_pfeat, m->d_pval, m->depth, m->n_trees, m->d_used, m->n_used,
          m->base, d_row_scores);
      return lt::check_launch("predict_perfect_kernel");
    }
  }
  const size_t tsmem = (size_t)m->n_nodes * sizeof(Node) +
                       (size_t)(m->n_used + m->n_trees) * lt::TILE_ROWS * sizeof(double) +
                       (size_t)(m->n_trees + 1) * sizeof(int32_t);
  if (tsmem <= optin && getenv("LT_PREDICT_THREAD_PER_ROW") == nullptr) {
    static size_t tconfigured[64] = {};
    if (tsmem > 48 * 1024 && (tdev < 0 || tdev >= 64 || tsmem > tconfigured[tdev])) {
      if (lt::check_cuda(cudaFuncSetAttribute(lt::predict_trees_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)tsmem), "smem attr"))
        return -1;
      if (tdev >= 0 && tdev < 64) tconfigured[tdev] = tsmem;
    }
    const int per_sm = tsmem <= optin / 2 ? 2 : 1;
    int64_t tiles = (n_rows + lt::TILE_ROWS - 1) / lt::TILE_ROWS;
    int64_t blocks = (int64_t)sms * per_sm;
    if (blocks > tiles) blocks = tiles;
    lt::predict_trees_kernel<<<(unsigned)blocks, lt::TREE_WARPS * 32, tsmem, (cudaStream_t)stream>>>(
        d_rows, n_rows, col_major, m->d_nodes, m->n_nodes, m->d_tree_off, m->n_trees, m->d_used, m->n_used,
        m->base, d_row_scores);
    return lt::check_launch("predict_trees_kernel");
  }
  size_t smem = (size_t)lt::ROWS_PER_BLOCK * (m->n_used + 1) * sizeof(double);
  // the opt-in shared-memory grant is per device (function attributes are per context)
  static size_t configured[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && (dev < 0 || dev >= 64 || smem > configured[dev])) {
    if (lt::check_cuda(cudaFuncSetAttribute(lt::predict_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem), "smem attr"))
      return -1;
    if (dev >= 0 && dev < 64) configured[dev] = smem;
  }
  int64_t blocks = (n_rows + lt::ROWS_PER_BLOCK - 1) / lt::ROWS_PER_BLOCK;
  lt::predict_rows_kernel<<<(unsigned)blocks, lt::ROWS_PER_BLOCK, smem, (cudaStream_t)stream>>>(
      d_rows, n_rows, col_major, m->d_nodes, m->d_tree_off, m->n_trees, m->d_used, m->n_used, m->base,
      d_row_scores);
  return lt::check_launch("predict_rows_kernel");
}

// rows[n_rows][164]
int lt_predict_rows_device(int64_t handle, const double* d_rows, int64_t n_rows, double* d_row_scores,
                           void* stream) {
  return predict_device(handle, d_rows, n_rows, false, d_row_scores, stream);
}

// cols[164][n_rows] (the layout lt_features_device_cm writes)
int lt_predict_cols_device(int64_t handle, const double* d_cols, int64_t n_rows, double* d_row_scores,
                           void* stream) {
  return predict_device(handle, d_cols, n_rows, true, d_row_scores, stream);
}

int lt_segment_sum_device(const double* d_row_scores, const int64_t* d_prog_off, int64_t n_prog,
                          double* d_scores, void* stream) {
  if (n_prog <= 0) return 0;
  int64_t blocks = (n_prog + 255) / 256;
  lt::segment_sum_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_row_scores, d_prog_off, n_prog,
                                                                             d_scores);
  return lt::check_launch("segment_sum_kernel");
}

}  // extern "C"
