// Batched per-statement feature extraction on sm_100a.
//
// Replaces `extract_features` / `analyze_program` / `statement_features`
// (reference src/features.py:161-425).  One thread per statement record (the
// record format is produced by paper_2006_06762_b200/encode.py and documented in
// include/loomtune_b200.h).  All structural resolution (attach chains, id-based
// loop identity, first-access views, packing strides, name ranks) is done by the
// encoder; this kernel performs every interval / evaluation / product the
// reference does, in the same order and with the same fp64 rounding:
//   * decode-AST intervals with the DMod same-block rule (src/ir.py:122-149),
//     floor division semantics of Python for negative operands;
//   * hull widths, unique bytes/lines, reuse classification, strides, working
//     sets (src/features.py:143-158,202-274);
//   * annotation / unroll blocks, intensity curve, ranked buffer blocks,
//     log2(1+max(x,0)) compression (src/features.py:296-417).
// Compiled with --fmad=false so no product/sum pair is contracted into an FMA.

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include <stdlib.h>
#include "common.h"

namespace lt {

constexpr int HDR = 18;
constexpr int NF = 164;
constexpr int MAX_NEST = 32;
constexpr int MAX_LOOPS = 64;
constexpr int MAX_ITERS = 24;
constexpr int MAX_VIEWS = 12;
constexpr int MAX_STACK = 32;

struct Iv { long long lo, hi; };

__device__ __forceinline__ long long fdiv(long long a, long long c) {
  long long q = a / c;
  if ((a % c != 0) && ((a < 0) != (c < 0))) --q;
  return q;
}
__device__ __forceinline__ long long fmod_(long long a, long long c) {
  long long r = a % c;
  if (r != 0 && ((r < 0) != (c < 0))) r += c;
  return r;
}

// upper bound of own loop j (lo = 0): its full range when pos < 0, else its range
// only if the loop sits inside nest position pos (`ws_inside`, src/features.py:266-274)
__device__ __forceinline__ long long loop_hi(const int32_t* loops, int j, int pos) {
  return (pos < 0 || loops[3 * j + 2] > pos) ? (long long)loops[3 * j] - 1 : 0;
}

// interval of one postfix decode AST given per-own-loop upper bounds (lo = 0)
__device__ bool ast_interval(const int32_t* nodes, int cnt, const int32_t* loops, int pos, Iv& out) {
  Iv st[MAX_STACK];
  int sp = 0;
  for (int n = 0; n < cnt; ++n) {
    int op = nodes[2 * n], arg = nodes[2 * n + 1];
    switch (op) {
      case 0: if (sp >= MAX_STACK) return false; st[sp].lo = 0; st[sp].hi = loop_hi(loops, arg, pos); ++sp; break;
      case 1: if (sp >= MAX_STACK) return false; st[sp].lo = arg; st[sp].hi = arg; ++sp; break;
      case 2: { if (sp < 2) return false; Iv b = st[--sp]; st[sp - 1].lo += b.lo; st[sp - 1].hi += b.hi; break; }
      case 3: { if (sp < 1) return false; Iv a = st[sp - 1]; long long c = arg;
                st[sp - 1] = c >= 0 ? Iv{a.lo * c, a.hi * c} : Iv{a.hi * c, a.lo * c}; break; }
      case 4: { if (sp < 1) return false; Iv a = st[sp - 1]; st[sp - 1] = Iv{fdiv(a.lo, arg), fdiv(a.hi, arg)}; break; }
      case 5: { if (sp < 1) return false; Iv a = st[sp - 1];
                if (fdiv(a.lo, arg) == fdiv(a.hi, arg)) st[sp - 1] = Iv{fmod_(a.lo, arg), fmod_(a.hi, arg)};
                else st[sp - 1] = Iv{0, (long long)arg - 1};
                break; }
      default: return false;
    }
  }
  if (sp != 1) return false;
  out = st[0];
  return true;
}

// value of a decode AST with every own loop at 0 except loop `one_at` at 1
__device__ bool ast_eval(const int32_t* nodes, int cnt, int one_at, long long& out) {
  long long st[MAX_STACK];
  int sp = 0;
  for (int n = 0; n < cnt; ++n) {
    int op = nodes[2 * n], arg = nodes[2 * n + 1];
    switch (op) {
      case 0: if (sp >= MAX_STACK) return false; st[sp++] = (arg == one_at) ? 1 : 0; break;
      case 1: if (sp >= MAX_STACK) return false; st[sp++] = arg; break;
      case 2: if (sp < 2) return false; --sp; st[sp - 1] += st[sp]; break;
      case 3: if (sp < 1) return false; st[sp - 1] *= arg; break;
      case 4: if (sp < 1) return false; st[sp - 1] = fdiv(st[sp - 1], arg); break;
      case 5: if (sp < 1) return false; st[sp - 1] = fmod_(st[sp - 1], arg); break;
      default: return false;
    }
  }
  if (sp != 1) return false;
  out = st[0];
  return true;
}

// Decode-AST evaluation used by both feature kernels: same operations as ast_interval /
// ast_eval, with the top three stack entries in registers (the decode ASTs of
// real States need depth <= 4; deeper entries go to a small local array).
struct RegStack {
  Iv a, b, c;          // a = top
  Iv deep[MAX_STACK];
  int sp;
  __device__ __forceinline__ void push(Iv v) {
    if (sp >= 3) deep[sp - 3] = c;
    c = b; b = a; a = v; ++sp;
  }
  __device__ __forceinline__ Iv pop() {
    Iv v = a;
    a = b; b = c;
    if (sp > 3) c = deep[sp - 4];
    --sp;
    return v;
  }
};

__device__ __forceinline__ bool ast_interval_w(const int32_t* nodes, int cnt, const int32_t* loops, int pos,
                                               Iv& out) {
  RegStack st;
  st.sp = 0;
  for (int n = 0; n < cnt; ++n) {
    const int op = nodes[2 * n], arg = nodes[2 * n + 1];
    if (op == 0) {
      if (st.sp >= MAX_STACK) return false;
      st.push(Iv{0, loop_hi(loops, arg, pos)});
    } else if (op == 1) {
      if (st.sp >= MAX_STACK) return false;
      st.push(Iv{arg, arg});
    } else if (op == 2) {
      if (st.sp < 2) return false;
      Iv b = st.pop();
      st.a.lo += b.lo; st.a.hi += b.hi;
    } else {
      if (st.sp < 1) return false;
      Iv a = st.a;
      const long long c = arg;
      if (op == 3) st.a = c >= 0 ? Iv{a.lo * c, a.hi * c} : Iv{a.hi * c, a.lo * c};
      else if (op == 4) st.a = Iv{fdiv(a.lo, c), fdiv(a.hi, c)};
      else if (op == 5) {
        if (fdiv(a.lo, c) == fdiv(a.hi, c)) st.a = Iv{fmod_(a.lo, c), fmod_(a.hi, c)};
        else st.a = Iv{0, c - 1};
      } else return false;
    }
  }
  if (st.sp != 1) return false;
  out = st.a;
  return true;
}

__device__ __forceinline__ bool ast_eval_w(const int32_t* nodes, int cnt, int one_at, long long& out) {
  RegStack st;        // lo carries the value
  st.sp = 0;
  for (int n = 0; n < cnt; ++n) {
    const int op = nodes[2 * n], arg = nodes[2 * n + 1];
    if (op == 0) {
      if (st.sp >= MAX_STACK) return false;
      st.push(Iv{(arg == one_at) ? 1 : 0, 0});
    } else if (op == 1) {
      if (st.sp >= MAX_STACK) return false;
      st.push(Iv{arg, 0});
    } else if (op == 2) {
      if (st.sp < 2) return false;
      Iv b = st.pop();
      st.a.lo += b.lo;
    } else {
      if (st.sp < 1) return false;
      if (op == 3) st.a.lo *= arg;
      else if (op == 4) st.a.lo = fdiv(st.a.lo, arg);
      else if (op == 5) st.a.lo = fmod_(st.a.lo, arg);
      else return false;
    }
  }
  if (st.sp != 1) return false;
  out = st.a.lo;
  return true;
}

struct View {
  const int32_t* dims;   // -> first dim record
  int n_marks, has_w, rank, n_dims;
  unsigned long long present;  // bitmask over own loops
};

// next dim record: (size, st, pext, const, n_terms, (it, c) * n_terms)
__device__ __forceinline__ const int32_t* dim_next(const int32_t* d) { return d + 5 + 2 * d[4]; }

__device__ __forceinline__ Iv dim_interval(const int32_t* d, const Iv* iv) {
  long long lo = d[3], hi = d[3];
  for (int t = 0; t < d[4]; ++t) {
    int it = d[5 + 2 * t];
    long long c = d[6 + 2 * t];
    if (c >= 0) { lo += c * iv[it].lo; hi += c * iv[it].hi; }
    else { lo += c * iv[it].hi; hi += c * iv[it].lo; }
  }
  int st = d[1], pext = d[2];
  if (pext > 0) {
    if (st > 1) { lo = fdiv(lo, st); hi = fdiv(hi, st); }
    if (fdiv(lo, pext) == fdiv(hi, pext)) { lo = fmod_(lo, pext); hi = fmod_(hi, pext); }
    else { lo = 0; hi = pext - 1; }
  }
  return Iv{lo, hi};
}

__device__ __forceinline__ long long dim_value(const int32_t* d, const long long* val) {
  long long v = d[3];
  for (int t = 0; t < d[4]; ++t) v += (long long)d[6 + 2 * t] * val[d[5 + 2 * t]];
  int st = d[1], pext = d[2];
  if (pext > 0) {
    if (st > 1) v = fdiv(v, st);
    v = fmod_(v, pext);
  }
  return v;
}

__device__ __forceinline__ long long hull_width(const int32_t* d, const Iv* iv) {
  Iv r = dim_interval(d, iv);
  long long size = d[0];
  long long lo = r.lo > 0 ? r.lo : 0;
  long long hi = r.hi < size - 1 ? r.hi : size - 1;
  long long w = hi - lo + 1;
  return w > 1 ? w : 1;
}

// position tag of nest entry i among same-kind loops (src/features.py:296-305)
__device__ int position(const int32_t* nest, int n_nest, int i) {
  int kind = nest[4 * i + 1];
  int cnt = 0, rank = 0;
  for (int j = 0; j < n_nest; ++j)
    if (nest[4 * j + 1] == kind) { if (j < i) ++rank; ++cnt; }
  int base = kind == 0 ? 1 : 4;                 // inner_spatial / inner_reduce
  if (rank == cnt - 1) return base;
  if (rank == 0 && cnt > 1) return base + 2;    // outer
  return base + 1;                              // middle
}

struct Row {
  double* v;
  __device__ void set(int i, double x) { v[i] = x; }
};

__device__ void annotation_block(const int32_t* nest, int n_nest, int ann, double* b) {
  for (int i = 0; i < 11; ++i) b[i] = 0.0;
  int hits = 0, last = -1, tag = -1;
  double prod = 1.0;
  for (int i = 0; i < n_nest; ++i) {
    if (nest[4 * i + 2] != ann) continue;
    int p = position(nest, n_nest, i);
    tag = (hits == 0) ? p : (tag == p ? tag : 7);
    prod *= (double)nest[4 * i];
    last = i;
    ++hits;
  }
  if (!hits) { b[1] = 1.0; return; }
  b[0] = (double)nest[4 * last];
  b[1 + tag] = 1.0;
  b[9] = prod;
  b[10] = (double)hits;
}

// One statement's 164-wide row.  Element (statement s, column k) lives at
// rows[s * ld_row + k * ld_col]: row-major (ld_col 1) or column-major (ld_col
// n_stmt, coalesced across the warp).
__device__ __forceinline__ void feature_row(const int32_t* __restrict__ words, const int64_t* __restrict__ stmt_off,
                                            int64_t s, double* __restrict__ rows, int64_t ld_col,
                                            int* __restrict__ err) {
  const int32_t* r = words + stmt_off[s];
  const int64_t ld_row = ld_col == 1 ? NF : 1;
  double* out = rows + s * ld_row;
#define O(k) out[(int64_t)(k) * ld_col]

  const int n_nest = r[0], own_start = r[1], n_loops = r[2], n_iter = r[3], n_views = r[4];
  const int unroll = r[5], n_live = r[6], has_reduce = r[7] & 1, gpu_feats = r[7] & 2;
  const int32_t* ops = r + 8;
  const int n_nodes = r[17];
  if (n_nest > MAX_NEST || n_loops > MAX_LOOPS || n_iter > MAX_ITERS || n_views > MAX_VIEWS) {
    for (int i = 0; i < NF; ++i) O(i) = __longlong_as_double(0x7ff8000000000000ULL);
    atomicExch(err, 1);
    return;
  }
  const int32_t* nest = r + HDR;
  const int32_t* loops = nest + 4 * n_nest;
  const int32_t* itab = loops + 3 * n_loops;
  const int32_t* nodes = itab + 2 * n_iter;
  const int32_t* vp = nodes + 2 * n_nodes;

  View views[MAX_VIEWS];
  unsigned long long iter_mask[MAX_ITERS];
  for (int it = 0; it < n_iter; ++it) {
    unsigned long long m = 0;
    const int32_t* nd = nodes + 2 * itab[2 * it];
    for (int n = 0; n < itab[2 * it + 1]; ++n)
      if (nd[2 * n] == 0) m |= 1ULL << nd[2 * n + 1];
    iter_mask[it] = m;
  }
  for (int v = 0; v < n_views; ++v) {
    View& w = views[v];
    w.n_marks = vp[0]; w.has_w = vp[1]; w.rank = vp[2]; w.n_dims = vp[3];
    w.dims = vp + 4;
    const int32_t* d = w.dims;
    unsigned long long m = 0;
    for (int k = 0; k < w.n_dims; ++k) {
      for (int t = 0; t < d[4]; ++t) m |= iter_mask[d[5 + 2 * t]];
      d = dim_next(d);
    }
    w.present = m;
    vp = d;
  }

  // own-range intervals of every iterator decode
  Iv iv[MAX_ITERS];
  bool ok = true;
  for (int it = 0; it < n_iter; ++it)
    ok &= ast_interval_w(nodes + 2 * itab[2 * it], itab[2 * it + 1], loops, -1, iv[it]);

  double total = 1.0;
  for (int i = 0; i < n_nest; ++i) total *= (double)nest[4 * i];
  double red_prod = 1.0, alloc = 4.0;
  for (int i = own_start; i < n_nest; ++i) {
    if (nest[4 * i + 1] == 1) red_prod *= (double)nest[4 * i];
    else alloc *= (double)nest[4 * i];
  }
  int ops_total = 0;
  for (int k = 0; k < 9; ++k) ops_total += ops[k];

  // per-view access statistics
  double tb[MAX_VIEWS], ub[MAX_VIEWS], ul[MAX_VIEWS], cnt[MAX_VIEWS], di[MAX_VIEWS], db[MAX_VIEWS],
      strd[MAX_VIEWS];
  int acc[MAX_VIEWS], reuse[MAX_VIEWS];
  const int inner_own = (n_nest > own_start) ? nest[4 * (n_nest - 1) + 3] : -1;
  long long val0[MAX_ITERS], val1[MAX_ITERS];
  if (inner_own >= 0) {
    for (int it = 0; it < n_iter; ++it) ok &= ast_eval_w(nodes + 2 * itab[2 * it], itab[2 * it + 1], -1, val0[it]);
    for (int it = 0; it < n_iter; ++it)
      ok &= ast_eval_w(nodes + 2 * itab[2 * it], itab[2 * it + 1], inner_own, val1[it]);
  }
  for (int v = 0; v < n_views; ++v) {
    const View& w = views[v];
    const bool has_w = w.has_w != 0;
    const bool has_r = (w.n_marks > w.has_w) || (has_w && red_prod > 1.0);
    acc[v] = (has_w && has_r) ? 2 : (has_w ? 1 : 0);
    long long uprod = 1, last = 1;
    double lines = 1.0;
    const int32_t* d = w.dims;
    for (int k = 0; k < w.n_dims; ++k) {
      long long wd = hull_width(d, iv);
      uprod *= wd;
      if (k < w.n_dims - 1) lines *= (double)wd; else last = wd;
      d = dim_next(d);
    }
    ub[v] = (double)uprod * 4.0;
    double lc = ceil((double)(last * 4) / 64.0);
    ul[v] = lines * (lc > 1.0 ? lc : 1.0);
    tb[v] = ((double)w.n_marks * total) * 4.0;
    // reuse (src/features.py:224-242)
    int absent_last = -1;
    double counter = 1.0;
    for (int i = 0; i < n_nest; ++i) {
      int oi = nest[4 * i + 3];
      bool present = oi >= 0 && ((w.present >> oi) & 1ULL);
      if (!present && nest[4 * i] > 1) { counter *= (double)nest[4 * i]; absent_last = i; }
    }
    if (has_w && has_reduce && red_prod > 1.0) {
      reuse[v] = 1; cnt[v] = red_prod; di[v] = 1.0; db[v] = (double)(4 * w.n_marks);
    } else if (absent_last >= 0) {
      reuse[v] = 0; cnt[v] = counter;
      double dit = 1.0;
      for (int i = absent_last + 1; i < n_nest; ++i) dit *= (double)nest[4 * i];
      di[v] = dit; db[v] = (dit * 4.0) * (double)w.n_marks;
    } else {
      reuse[v] = 2; cnt[v] = 1.0; di[v] = 0.0; db[v] = 0.0;
    }
    // stride (src/features.py:244-259)
    strd[v] = 0.0;
    if (inner_own >= 0 && ((w.present >> inner_own) & 1ULL)) {
      long long a0 = 0, a1 = 0, fs = 1;
      // dims are walked inner->outer for row-major flat strides
      const int32_t* dd[16];
      const int32_t* q = w.dims;
      int nd = w.n_dims < 16 ? w.n_dims : 16;
      for (int k = 0; k < nd; ++k) { dd[k] = q; q = dim_next(q); }
      for (int k = nd - 1; k >= 0; --k) {
        long long size = dd[k][0];
        long long x0 = dim_value(dd[k], val0), x1 = dim_value(dd[k], val1);
        x0 = x0 < 0 ? 0 : (x0 > size - 1 ? size - 1 : x0);
        x1 = x1 < 0 ? 0 : (x1 > size - 1 ? size - 1 : x1);
        a0 += x0 * fs; a1 += x1 * fs;
        fs *= size;
      }
      long long dlt = a1 - a0;
      strd[v] = (double)((dlt < 0 ? -dlt : dlt) * 4);
    }
  }

  // working set inside each nest position (src/features.py:266-274)
  // An iterator's interval at position pos depends only on which of ITS own loops
  // sit inside pos (key = iter_mask & inside), so it is recomputed only when that
  // key changes, and the working set only when some interval changed.
  double ws[MAX_NEST];
  {
    Iv iv2[MAX_ITERS];
    unsigned long long seen[MAX_ITERS];
    double acc_ws = 0.0;
    for (int pos = 0; pos < n_nest; ++pos) {
      unsigned long long inside = 0;
      for (int j = 0; j < n_loops; ++j)
        if (loops[3 * j + 2] > pos) inside |= 1ULL << j;
      bool changed = false;
      for (int it = 0; it < n_iter; ++it) {
        const unsigned long long key = iter_mask[it] & inside;
        if (pos > 0 && key == seen[it]) continue;
        ok &= ast_interval_w(nodes + 2 * itab[2 * it], itab[2 * it + 1], loops, pos, iv2[it]);
        seen[it] = key;
        changed = true;
      }
      if (changed) {
        acc_ws = 0.0;
        for (int v = 0; v < n_views; ++v) {
          long long p = 1;
          const int32_t* d = views[v].dims;
          for (int k = 0; k < views[v].n_dims; ++k) { p *= hull_width(d, iv2); d = dim_next(d); }
          acc_ws += (double)p * 4.0;
        }
      }
      ws[pos] = acc_ws;
    }
  }

  // ---- row assembly (src/features.py:388-417) ----
  // every column is written once, already compressed: log2(1 + max(x, 0)) on the
  // non-one-hot columns (src/features.py:416)
  auto W = [&](int k, double x) { O(k) = is_onehot(k) ? x : log2(1.0 + (x > 0.0 ? x : 0.0)); };
  double b[11];
  for (int k = 0; k < 9; ++k) W(k, (double)ops[k] * total);
  for (int k = 9; k < 18; ++k) O(k) = 0.0;
  annotation_block(nest, n_nest, 2, b);
  for (int k = 0; k < 11; ++k) W(18 + k, b[k]);
  {  // unroll block
    for (int k = 0; k < 11; ++k) b[k] = 0.0;
    long long prod = 1;
    int n_cov = 0, first = -1, tag = -1;
    if (unroll > 0 && n_nest > own_start) {
      for (int i = n_nest - 1; i >= own_start; --i) {
        if (prod * nest[4 * i] > unroll) break;
        prod *= nest[4 * i];
        int p = position(nest, n_nest, i);
        tag = (n_cov == 0) ? p : (tag == p ? tag : 7);
        if (n_cov == 0) first = i;
        ++n_cov;
      }
    }
    if (!n_cov) b[1] = 1.0;
    else { b[0] = (double)nest[4 * first]; b[1 + tag] = 1.0; b[9] = (double)prod; b[10] = (double)n_cov; }
    for (int k = 0; k < 11; ++k) W(29 + k, b[k]);
  }
  annotation_block(nest, n_nest, 1, b);
  for (int k = 0; k < 11; ++k) W(40 + k, b[k]);
  if (gpu_feats) {          // opt-in: the kernel binding the encoder appended (8 trailing words)
    const int32_t* gw = words + stmt_off[s + 1] - 8;
    for (int k = 0; k < 8; ++k) W(51 + k, (double)gw[k]);
  } else {
    for (int k = 51; k < 59; ++k) O(k) = 0.0;     // the reference leaves the gpu_* slots zero
  }
  if (n_nest == 0 || ops_total == 0) {
    for (int k = 59; k < 69; ++k) O(k) = 0.0;
  } else {
    double inside[MAX_NEST + 1];
    inside[n_nest] = 1.0;
    for (int i = n_nest - 1; i >= 0; --i) inside[i] = inside[i + 1] * (double)nest[4 * i];
    for (int j = 1; j <= 10; ++j) {
      int depth = (int)ceil((double)j / 10.0 * (double)n_nest);
      if (depth < 1) depth = 1;
      int pos = n_nest - depth;
      double by;
      if (pos == 0) { by = 0.0; for (int v = 0; v < n_views; ++v) by += ub[v]; }
      else by = ws[pos - 1];
      double flops = (double)ops_total * inside[pos];
      W(58 + j, flops / (by > 1.0 ? by : 1.0));
    }
  }
  // ranked buffer blocks: by (-total_bytes, name)
  bool used[MAX_VIEWS];
  for (int v = 0; v < n_views; ++v) used[v] = false;
  int n_rank = n_views < 5 ? n_views : 5;
  for (int slot = 0; slot < 5; ++slot) {
    const int o = 69 + 18 * slot;
    if (slot >= n_rank) { for (int k = 0; k < 18; ++k) O(o + k) = 0.0; continue; }
    int best = -1;
    for (int v = 0; v < n_views; ++v) {
      if (used[v]) continue;
      if (best < 0 || tb[v] > tb[best] || (tb[v] == tb[best] && views[v].rank < views[best].rank)) best = v;
    }
    used[best] = true;
    const int v = best;
    for (int k = 0; k < 3; ++k) O(o + k) = (k == acc[v]) ? 1.0 : 0.0;
    double ln = tb[v] / 64.0;
    W(o + 3, tb[v]); W(o + 4, ub[v]); W(o + 5, ln); W(o + 6, ul[v]);
    for (int k = 0; k < 3; ++k) O(o + 7 + k) = (k == reuse[v]) ? 1.0 : 0.0;
    W(o + 10, di[v]); W(o + 11, db[v]); W(o + 12, cnt[v]); W(o + 13, strd[v]);
    double c = cnt[v] > 1.0 ? cnt[v] : 1.0;
    W(o + 14, tb[v] / c); W(o + 15, ub[v] / c); W(o + 16, ln / c); W(o + 17, ul[v] / c);
  }
  W(159, alloc);
  W(160, (double)n_live);
  W(161, (double)n_nest);
  W(162, total);
  W(163, (double)unroll);
  if (!ok) {
    for (int i = 0; i < NF; ++i) O(i) = __longlong_as_double(0x7ff8000000000000ULL);
    atomicExch(err, 2);
  }
#undef O
}

// ---------------------------------------------------------------------------
// Warp-per-statement kernel (the default).  The thread-per-statement kernel
// above keeps ~4 KB of per-statement scratch (decode stacks, intervals, per-view
// statistics, working sets) in local memory, which at full occupancy spills to
// HBM (r01 ncu: 7.4 KB read + 2.5 KB written per statement for 2.3 KB of
// algorithmic bytes).  Here a warp owns one statement: the per-statement tables
// live in shared memory and the lanes split the work — one lane per iterator
// (masks, own-range intervals, the two stride evaluations), per view (access
// statistics, reuse, stride), per nest position (working set, each lane
// evaluating the intervals it needs on the fly), per intensity point and per
// ranked buffer slot.  Every value is computed by exactly the expression the
// thread kernel uses (same operand order, --fmad=false), so rows are identical.
// A block of FW_WARPS warps stages FW_CHUNK rows in shared memory and writes
// them out coalesced (column-major: FW_CHUNK consecutive statements per column).
constexpr int FW_WARPS = 4;
constexpr int FW_CHUNK = 16;
constexpr int FW_LD = NF + 1;            // odd row stride: conflict-free lane-per-column access

constexpr int FW_REC = 768;        // statement record words staged in shared memory (longest seen: 635)
constexpr int FW_TAB = 192;        // memoised (position, iterator) intervals (largest seen: 14 x 8)

struct WarpScratch {
  unsigned long long iter_mask[MAX_ITERS];
  Iv iv[MAX_ITERS];
  long long val0[MAX_ITERS], val1[MAX_ITERS];
  unsigned long long present[MAX_VIEWS];
  int vdims[MAX_VIEWS], vmarks[MAX_VIEWS], vhasw[MAX_VIEWS], vrank[MAX_VIEWS], vndims[MAX_VIEWS];
  double tb[MAX_VIEWS], ub[MAX_VIEWS], ul[MAX_VIEWS], cnt[MAX_VIEWS], di[MAX_VIEWS], db[MAX_VIEWS],
      strd[MAX_VIEWS];
  int acc[MAX_VIEWS], reuse[MAX_VIEWS];
  double ws[MAX_NEST];
  unsigned long long inside[MAX_NEST];
  int ok;
  Iv tab[FW_TAB];                  // interval of iterator it at position pos: tab[pos * n_iter + it]
  int32_t rec[FW_REC];
};

// interval of iterator `it` at nest position pos (pos < 0: own ranges)
__device__ __forceinline__ Iv iter_interval(const int32_t* nodes, const int32_t* itab, const int32_t* loops, int it,
                                            int pos, bool& ok) {
  Iv r{0, 0};
  ok &= ast_interval_w(nodes + 2 * itab[2 * it], itab[2 * it + 1], loops, pos, r);
  return r;
}

__device__ __forceinline__ double wcol(int k, double x) {
  return is_onehot(k) ? x : log2(1.0 + (x > 0.0 ? x : 0.0));
}

__device__ void warp_feature_row(const int32_t* __restrict__ words, const int64_t* __restrict__ stmt_off, int64_t s,
                                 double* __restrict__ row, WarpScratch& S, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int32_t* r = words + stmt_off[s];
  {
    const int64_t len = stmt_off[s + 1] - stmt_off[s];
    if (len <= FW_REC) {                 // the record in shared memory: every later read is on-chip
      for (int i = lane; i < len; i += 32) S.rec[i] = r[i];
      __syncwarp();
      r = S.rec;
    }
  }
  const int n_nest = r[0], own_start = r[1], n_loops = r[2], n_iter = r[3], n_views = r[4];
  const int unroll = r[5], n_live = r[6], has_reduce = r[7] & 1, gpu_feats = r[7] & 2;
  const int32_t* ops = r + 8;
  const int n_nodes = r[17];
  if (n_nest > MAX_NEST || n_loops > MAX_LOOPS || n_iter > MAX_ITERS || n_views > MAX_VIEWS) {
    for (int i = lane; i < NF; i += 32) row[i] = __longlong_as_double(0x7ff8000000000000ULL);
    if (lane == 0) atomicExch(err, 1);
    return;
  }
  const int32_t* nest = r + HDR;
  const int32_t* loops = nest + 4 * n_nest;
  const int32_t* itab = loops + 3 * n_loops;
  const int32_t* nodes = itab + 2 * n_iter;
  const int inner_own = (n_nest > own_start) ? nest[4 * (n_nest - 1) + 3] : -1;
  bool ok = true;

  // ---- lane per iterator: own-loop mask, own-range interval, stride evaluations
  if (lane < n_iter) {
    const int it = lane;
    unsigned long long m = 0;
    const int32_t* nd = nodes + 2 * itab[2 * it];
    for (int n = 0; n < itab[2 * it + 1]; ++n)
      if (nd[2 * n] == 0) m |= 1ULL << nd[2 * n + 1];
    S.iter_mask[it] = m;
    S.iv[it] = iter_interval(nodes, itab, loops, it, -1, ok);
    if (inner_own >= 0) {
      long long v0 = 0, v1 = 0;
      ok &= ast_eval_w(nd, itab[2 * it + 1], -1, v0);
      ok &= ast_eval_w(nd, itab[2 * it + 1], inner_own, v1);
      S.val0[it] = v0;
      S.val1[it] = v1;
    }
  }
  // ---- lane 0: view record offsets (variable-length, sequential)
  if (lane == 0) {
    const int32_t* vp = nodes + 2 * n_nodes;
    for (int v = 0; v < n_views; ++v) {
      S.vmarks[v] = vp[0]; S.vhasw[v] = vp[1]; S.vrank[v] = vp[2]; S.vndims[v] = vp[3];
      const int32_t* d = vp + 4;
      S.vdims[v] = (int)(d - r);
      for (int k = 0; k < vp[3]; ++k) d = dim_next(d);
      vp = d;
    }
  }
  __syncwarp();

  double total = 1.0;
  for (int i = 0; i < n_nest; ++i) total *= (double)nest[4 * i];
  double red_prod = 1.0, alloc = 4.0;
  for (int i = own_start; i < n_nest; ++i) {
    if (nest[4 * i + 1] == 1) red_prod *= (double)nest[4 * i];
    else alloc *= (double)nest[4 * i];
  }
  int ops_total = 0;
  for (int k = 0; k < 9; ++k) ops_total += ops[k];

  // ---- lane per view: access statistics, reuse, stride (src/features.py:202-259)
  if (lane < n_views) {
    const int v = lane;
    const int32_t* d = r + S.vdims[v];
    const int nd_ = S.vndims[v];
    unsigned long long m = 0;
    {
      const int32_t* q = d;
      for (int k = 0; k < nd_; ++k) {
        for (int t = 0; t < q[4]; ++t) m |= S.iter_mask[q[5 + 2 * t]];
        q = dim_next(q);
      }
    }
    S.present[v] = m;
    const bool has_w = S.vhasw[v] != 0;
    const bool has_r = (S.vmarks[v] > S.vhasw[v]) || (has_w && red_prod > 1.0);
    S.acc[v] = (has_w && has_r) ? 2 : (has_w ? 1 : 0);
    long long uprod = 1, last = 1;
    double lines = 1.0;
    {
      const int32_t* q = d;
      for (int k = 0; k < nd_; ++k) {
        long long wd = hull_width(q, S.iv);
        uprod *= wd;
        if (k < nd_ - 1) lines *= (double)wd; else last = wd;
        q = dim_next(q);
      }
    }
    S.ub[v] = (double)uprod * 4.0;
    double lc = ceil((double)(last * 4) / 64.0);
    S.ul[v] = lines * (lc > 1.0 ? lc : 1.0);
    S.tb[v] = ((double)S.vmarks[v] * total) * 4.0;
    int absent_last = -1;
    double counter = 1.0;
    for (int i = 0; i < n_nest; ++i) {
      int oi = nest[4 * i + 3];
      bool present = oi >= 0 && ((m >> oi) & 1ULL);
      if (!present && nest[4 * i] > 1) { counter *= (double)nest[4 * i]; absent_last = i; }
    }
    if (has_w && has_reduce && red_prod > 1.0) {
      S.reuse[v] = 1; S.cnt[v] = red_prod; S.di[v] = 1.0; S.db[v] = (double)(4 * S.vmarks[v]);
    } else if (absent_last >= 0) {
      S.reuse[v] = 0; S.cnt[v] = counter;
      double dit = 1.0;
      for (int i = absent_last + 1; i < n_nest; ++i) dit *= (double)nest[4 * i];
      S.di[v] = dit; S.db[v] = (dit * 4.0) * (double)S.vmarks[v];
    } else {
      S.reuse[v] = 2; S.cnt[v] = 1.0; S.di[v] = 0.0; S.db[v] = 0.0;
    }
    double sv = 0.0;
    if (inner_own >= 0 && ((m >> inner_own) & 1ULL)) {
      long long a0 = 0, a1 = 0, fs = 1;
      const int32_t* dd[16];
      const int32_t* q = d;
      int ndc = nd_ < 16 ? nd_ : 16;
      for (int k = 0; k < ndc; ++k) { dd[k] = q; q = dim_next(q); }
      for (int k = ndc - 1; k >= 0; --k) {
        long long size = dd[k][0];
        long long x0 = dim_value(dd[k], S.val0), x1 = dim_value(dd[k], S.val1);
        x0 = x0 < 0 ? 0 : (x0 > size - 1 ? size - 1 : x0);
        x1 = x1 < 0 ? 0 : (x1 > size - 1 ? size - 1 : x1);
        a0 += x0 * fs; a1 += x1 * fs;
        fs *= size;
      }
      long long dlt = a1 - a0;
      sv = (double)((dlt < 0 ? -dlt : dlt) * 4);
    }
    S.strd[v] = sv;
  }
  // ---- working set inside each nest position (src/features.py:266-274).  An
  // iterator's interval at position pos depends only on which of ITS own loops
  // sit inside pos; lane = iterator walks the positions and re-evaluates only
  // when that set changes (memoised into S.tab), then lane = position sums the
  // views' hull products from the table.
  for (int pos = lane; pos < n_nest; pos += 32) {
    unsigned long long in = 0;
    for (int j = 0; j < n_loops; ++j)
      if (loops[3 * j + 2] > pos) in |= 1ULL << j;
    S.inside[pos] = in;
  }
  __syncwarp();
  const bool memo = n_nest * n_iter <= FW_TAB;
  if (memo && lane < n_iter) {
    const int it = lane;
    unsigned long long seen = 0;
    Iv cur{0, 0};
    for (int pos = 0; pos < n_nest; ++pos) {
      const unsigned long long key = S.iter_mask[it] & S.inside[pos];
      if (pos == 0 || key != seen) {
        cur = iter_interval(nodes, itab, loops, it, pos, ok);
        seen = key;
      }
      S.tab[pos * n_iter + it] = cur;
    }
  }
  __syncwarp();
  for (int pos = lane; pos < n_nest; pos += 32) {
    double acc_ws = 0.0;
    for (int v = 0; v < n_views; ++v) {
      long long pr = 1;
      const int32_t* d = r + S.vdims[v];
      for (int k = 0; k < S.vndims[v]; ++k) {
        if (memo) {
          pr *= hull_width(d, S.tab + pos * n_iter);
        } else {
          long long lo = d[3], hi = d[3];
          for (int t = 0; t < d[4]; ++t) {
            const Iv a = iter_interval(nodes, itab, loops, d[5 + 2 * t], pos, ok);
            long long c = d[6 + 2 * t];
            if (c >= 0) { lo += c * a.lo; hi += c * a.hi; }
            else { lo += c * a.hi; hi += c * a.lo; }
          }
          int st = d[1], pext = d[2];
          if (pext > 0) {
            if (st > 1) { lo = fdiv(lo, st); hi = fdiv(hi, st); }
            if (fdiv(lo, pext) == fdiv(hi, pext)) { lo = fmod_(lo, pext); hi = fmod_(hi, pext); }
            else { lo = 0; hi = pext - 1; }
          }
          long long size = d[0];
          long long l2 = lo > 0 ? lo : 0;
          long long h2 = hi < size - 1 ? hi : size - 1;
          long long w = h2 - l2 + 1;
          pr *= (w > 1 ? w : 1);
        }
        d = dim_next(d);
      }
      acc_ws += (double)pr * 4.0;
    }
    S.ws[pos] = acc_ws;
  }
  __syncwarp();

  // ---- row assembly (src/features.py:388-417), lanes over column groups
  for (int k = lane; k < 9; k += 32) row[k] = wcol(k, (double)ops[k] * total);
  for (int k = 9 + lane; k < 18; k += 32) row[k] = 0.0;
  if (lane < 3) {                          // lane 0 vectorize, 1 unroll, 2 parallel block
    double b[11];
    const int base_col = lane == 0 ? 18 : (lane == 1 ? 29 : 40);
    if (lane == 1) {
      for (int k = 0; k < 11; ++k) b[k] = 0.0;
      long long prod = 1;
      int n_cov = 0, first = -1, tag = -1;
      if (unroll > 0 && n_nest > own_start) {
        for (int i = n_nest - 1; i >= own_start; --i) {
          if (prod * nest[4 * i] > unroll) break;
          prod *= nest[4 * i];
          int p = position(nest, n_nest, i);
          tag = (n_cov == 0) ? p : (tag == p ? tag : 7);
          if (n_cov == 0) first = i;
          ++n_cov;
        }
      }
      if (!n_cov) b[1] = 1.0;
      else { b[0] = (double)nest[4 * first]; b[1 + tag] = 1.0; b[9] = (double)prod; b[10] = (double)n_cov; }
    } else {
      annotation_block(nest, n_nest, lane == 0 ? 2 : 1, b);
    }
    for (int k = 0; k < 11; ++k) row[base_col + k] = wcol(base_col + k, b[k]);
  }
  if (lane >= 3 && lane < 11) {            // gpu_* slots
    const int k = 51 + (lane - 3);
    if (gpu_feats) row[k] = wcol(k, (double)(words + stmt_off[s + 1] - 8)[lane - 3]);
    else row[k] = 0.0;                     // the reference leaves the gpu_* slots zero
  }
  if (lane >= 11 && lane < 21) {           // intensity curve point j
    const int j = lane - 10;
    if (n_nest == 0 || ops_total == 0) {
      row[58 + j] = 0.0;
    } else {
      int depth = (int)ceil((double)j / 10.0 * (double)n_nest);
      if (depth < 1) depth = 1;
      const int pos = n_nest - depth;
      double inside = 1.0;                 // same left-to-right product as inside[pos]
      for (int i = n_nest - 1; i >= pos; --i) inside = inside * (double)nest[4 * i];
      double by;
      if (pos == 0) { by = 0.0; for (int v = 0; v < n_views; ++v) by += S.ub[v]; }
      else by = S.ws[pos - 1];
      double flops = (double)ops_total * inside;
      row[58 + j] = wcol(58 + j, flops / (by > 1.0 ? by : 1.0));
    }
  }
  if (lane >= 21 && lane < 26) {           // ranked buffer slot
    const int slot = lane - 21;
    const int o = 69 + 18 * slot;
    const int n_rank = n_views < 5 ? n_views : 5;
    if (slot >= n_rank) {
      for (int k = 0; k < 18; ++k) row[o + k] = 0.0;
    } else {
      // the view of rank `slot` under (-total_bytes, name)
      int v = -1;
      for (int u = 0; u < n_views && v < 0; ++u) {
        int before = 0;
        for (int w2 = 0; w2 < n_views; ++w2)
          if (S.tb[w2] > S.tb[u] || (S.tb[w2] == S.tb[u] && S.vrank[w2] < S.vrank[u])) ++before;
        if (before == slot) v = u;
      }
      for (int k = 0; k < 3; ++k) row[o + k] = (k == S.acc[v]) ? 1.0 : 0.0;
      double ln = S.tb[v] / 64.0;
      row[o + 3] = wcol(o + 3, S.tb[v]); row[o + 4] = wcol(o + 4, S.ub[v]);
      row[o + 5] = wcol(o + 5, ln); row[o + 6] = wcol(o + 6, S.ul[v]);
      for (int k = 0; k < 3; ++k) row[o + 7 + k] = (k == S.reuse[v]) ? 1.0 : 0.0;
      row[o + 10] = wcol(o + 10, S.di[v]); row[o + 11] = wcol(o + 11, S.db[v]);
      row[o + 12] = wcol(o + 12, S.cnt[v]); row[o + 13] = wcol(o + 13, S.strd[v]);
      double c = S.cnt[v] > 1.0 ? S.cnt[v] : 1.0;
      row[o + 14] = wcol(o + 14, S.tb[v] / c); row[o + 15] = wcol(o + 15, S.ub[v] / c);
      row[o + 16] = wcol(o + 16, ln / c); row[o + 17] = wcol(o + 17, S.ul[v] / c);
    }
  }
  if (lane == 26) {
    row[159] = wcol(159, alloc);
    row[160] = wcol(160, (double)n_live);
    row[161] = wcol(161, (double)n_nest);
    row[162] = wcol(162, total);
    row[163] = wcol(163, (double)unroll);
  }
  const unsigned bad = __ballot_sync(0xffffffffu, !ok);
  __syncwarp();
  if (bad) {
    for (int i = lane; i < NF; i += 32) row[i] = __longlong_as_double(0x7ff8000000000000ULL);
    if (lane == 0) atomicExch(err, 2);
  }
}

__global__ void __launch_bounds__(FW_WARPS * 32)
features_warp_kernel(const int32_t* __restrict__ words, const int64_t* __restrict__ stmt_off, int64_t n_stmt,
                     double* __restrict__ out, int64_t ld_col, int* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char fw_smem[];
  double* rows = (double*)fw_smem;                                     // FW_CHUNK x FW_LD
  WarpScratch* scratch = (WarpScratch*)(rows + FW_CHUNK * FW_LD);
  const int warp = threadIdx.x >> 5;
  WarpScratch& S = scratch[warp];
  for (int64_t s0 = (int64_t)blockIdx.x * FW_CHUNK; s0 < n_stmt; s0 += (int64_t)gridDim.x * FW_CHUNK) {
    const int here = (int)min((int64_t)FW_CHUNK, n_stmt - s0);
    for (int i = warp; i < here; i += FW_WARPS) {
      warp_feature_row(words, stmt_off, s0 + i, rows + i * FW_LD, S, err);
      __syncwarp();
    }
    __syncthreads();
    if (ld_col == 1) {                     // rows[n][164]: the chunk is one contiguous run
      double* dst = out + s0 * NF;
      for (int e = threadIdx.x; e < here * NF; e += blockDim.x) {
        const int i = e / NF, k = e - i * NF;
        dst[e] = rows[i * FW_LD + k];
      }
    } else {                               // cols[164][n]: `here` consecutive statements per column
      for (int e = threadIdx.x; e < here * NF; e += blockDim.x) {
        const int k = e / here, i = e - k * here;
        out[(int64_t)k * ld_col + s0 + i] = rows[i * FW_LD + k];
      }
    }
    __syncthreads();
  }
}

// Persistent grid-stride loop: the grid is sized so that each thread's local
// working set (intervals, per-view statistics, decode stacks) stays L1/L2
// resident instead of spilling to HBM (SM count x blocks_per_sm blocks).
__global__ void __launch_bounds__(128)
features_kernel(const int32_t* __restrict__ words, const int64_t* __restrict__ stmt_off,
                int64_t n_stmt, double* __restrict__ rows, int64_t ld_col, int* __restrict__ err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_stmt; s += stride)
    feature_row(words, stmt_off, s, rows, ld_col, err);
}

}  // namespace lt

static int launch_features(const int32_t* d_words, const int64_t* d_stmt_off, int64_t n_stmt, double* d_out,
                           int64_t ld_col, int* d_err, void* stream) {
  if (n_stmt <= 0) return 0;
  // the thread-per-statement kernel is the default: the warp-per-statement kernel
  // moves 1.02x the algorithmic DRAM bytes (vs 4.2x) but is ~9x slower (r02 ncu,
  // profiles/r02_scoring_kernels_ncu.txt): the per-statement work is a serial
  // chain of decode-AST interpretation that a warp cannot spread over its lanes
  if (getenv("LT_FEATURES_WARP") != nullptr) {
    static int wsms = -1, wdev = -1;
    const size_t smem = (size_t)lt::FW_CHUNK * lt::FW_LD * sizeof(double) + lt::FW_WARPS * sizeof(lt::WarpScratch);
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != wdev) {
      cudaDeviceGetAttribute(&wsms, cudaDevAttrMultiProcessorCount, dev);
      if (lt::check_cuda(cudaFuncSetAttribute(lt::features_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem), "features smem attr"))
        return -1;
      wdev = dev;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lt::features_warp_kernel, lt::FW_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t chunks = (n_stmt + lt::FW_CHUNK - 1) / lt::FW_CHUNK;
    int64_t blocks = (int64_t)wsms * per_sm;
    if (blocks > chunks) blocks = chunks;
    lt::features_warp_kernel<<<(unsigned)blocks, lt::FW_WARPS * 32, smem, (cudaStream_t)stream>>>(
        d_words, d_stmt_off, n_stmt, d_out, ld_col, d_err);
    return lt::check_launch("features_warp_kernel");
  }
  const int threads = 128;
  static int sms = 0, per_sm = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = getenv("LT_FEAT_BLOCKS_PER_SM");
    per_sm = e ? atoi(e) : 0;
    cudaFuncSetAttribute(lt::features_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  }
  int64_t blocks = (n_stmt + threads - 1) / threads;
  if (per_sm > 0 && blocks > (int64_t)sms * per_sm) blocks = (int64_t)sms * per_sm;
  lt::features_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(d_words, d_stmt_off, n_stmt,
                                                                             d_out, ld_col, d_err);
  return lt::check_launch("features_kernel");
}

// rows[n_stmt][164] (row-major)
extern "C" int lt_features_device(const int32_t* d_words, const int64_t* d_stmt_off, int64_t n_stmt,
                                  double* d_rows, int* d_err, void* stream) {
  return launch_features(d_words, d_stmt_off, n_stmt, d_rows, 1, d_err, stream);
}

// cols[164][n_stmt] (column-major: each warp's stores are contiguous)
extern "C" int lt_features_device_cm(const int32_t* d_words, const int64_t* d_stmt_off, int64_t n_stmt,
                                     double* d_cols, int* d_err, void* stream) {
  return launch_features(d_words, d_stmt_off, n_stmt, d_cols, n_stmt, d_err, stream);
}

namespace lt {
// [164][n] -> [n][164] through a shared-memory tile (coalesced on both sides)
__global__ void __launch_bounds__(256) cols_to_rows_kernel(const double* __restrict__ cols, int64_t n,
                                                          double* __restrict__ rows) {
  __shared__ double tile[32][33];
  const int64_t s0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    int k = k0 + dy;
    int64_t s = s0 + threadIdx.x;
    if (k < NF && s < n) tile[dy][threadIdx.x] = cols[(int64_t)k * n + s];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += 8) {
    int64_t s = s0 + dy;
    int k = k0 + threadIdx.x;
    if (k < NF && s < n) rows[s * NF + k] = tile[threadIdx.x][dy];
  }
}
}  // namespace lt

extern "C" int lt_cols_to_rows_device(const double* d_cols, int64_t n, double* d_rows, void* stream) {
  if (n <= 0) return 0;
  dim3 grid((unsigned)((n + 31) / 32), (lt::NF + 31) / 32), block(32, 8);
  lt::cols_to_rows_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(d_cols, n, d_rows);
  return lt::check_launch("cols_to_rows_kernel");
}
