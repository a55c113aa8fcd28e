// Native State encoder: Program objects -> the flat int32 statement records of
// csrc/features.cu, bit-identical to paper_2006_06762_b200/encode.py (which stays
// as the readable specification and the gpu_features path).  The encoder walks the
// reference's own frozen dataclasses (loomtune.ir Program / Stage / Loop / decode
// ASTs, loomtune.expr nodes) through the CPython API, so host-side scoring is no
// longer bound by Python bytecode (`src/features.py:161-284` is the structure it
// resolves; see encode.py's docstring for the record layout and every citation).
//
// Entry point: _lt_encode.encode_batch(programs) -> (words: bytes of int32,
// stmt_offsets: bytes of int64, prog_offsets: bytes of int64).
// Errors raise ValueError with encode.py's EncodeError messages.

#define PY_SSIZE_T_CLEAN
#include <Python.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <functional>
#include <unordered_map>
#include <utility>
#include <vector>

namespace {

enum { OP_VAR = 0, OP_CONST = 1, OP_ADD = 2, OP_MUL = 3, OP_DIV = 4, OP_MOD = 5 };
// node kinds, resolved from the class name once per type object
enum Kind { K_OTHER = 0, K_DVAR, K_DCONST, K_DADD, K_DMUL, K_DDIV, K_DMOD,
            K_CONST, K_ITERVAL, K_READ, K_BIN, K_CALL, K_SELECT, K_REDUCE };
// op-count buckets in encode.KINDS order
enum { C_ADD = 0, C_SUB, C_MUL, C_DIV, C_MINMAX, C_CMP, C_MATH, C_SELECT, C_OTHER, N_KINDS };

struct EncodeError {
  std::string msg;
};

struct Names {
  PyObject *stages, *layouts, *dag, *name, *inlined, *compute_at, *loops, *id, *extent, *kind, *annotation,
      *index_map, *space, *reduce, *expr, *pragma_unroll, *loop, *value, *a, *b, *c, *buffer, *index, *terms,
      *const_, *lhs, *rhs, *arg, *cond, *then, *other, *body, *op, *node, *shape;
} N;

bool init_names() {
#define I(f, s) if (!(N.f = PyUnicode_InternFromString(s))) return false;
  I(stages, "stages") I(layouts, "layouts") I(dag, "dag") I(name, "name") I(inlined, "inlined")
  I(compute_at, "compute_at") I(loops, "loops") I(id, "id") I(extent, "extent") I(kind, "kind")
  I(annotation, "annotation") I(index_map, "index_map") I(space, "space") I(reduce, "reduce") I(expr, "expr")
  I(pragma_unroll, "pragma_unroll") I(loop, "loop") I(value, "value") I(a, "a") I(b, "b") I(c, "c")
  I(buffer, "buffer") I(index, "index") I(terms, "terms") I(const_, "const") I(lhs, "lhs") I(rhs, "rhs")
  I(arg, "arg") I(cond, "cond") I(then, "then") I(other, "other") I(body, "body") I(op, "op") I(node, "node")
  I(shape, "shape")
#undef I
  return true;
}

// Owned reference with automatic release.
struct Ref {
  PyObject* p = nullptr;
  Ref() = default;
  explicit Ref(PyObject* o) : p(o) {}
  Ref(const Ref&) = delete;
  Ref(Ref&& o) noexcept : p(o.p) { o.p = nullptr; }
  Ref& operator=(Ref&& o) noexcept { std::swap(p, o.p); return *this; }
  ~Ref() { Py_XDECREF(p); }
  PyObject* get() const { return p; }
};

struct PyErrSet {};     // a Python exception is already set

Ref attr(PyObject* o, PyObject* name) {
  PyObject* r = PyObject_GetAttr(o, name);
  if (!r) throw PyErrSet{};
  return Ref(r);
}

int64_t as_i64(PyObject* o) {
  // int(x): ints and integral floats (the reference stores ints; DConst.value may be an int-like)
  if (PyLong_Check(o)) {
    int64_t v = PyLong_AsLongLong(o);
    if (v == -1 && PyErr_Occurred()) throw PyErrSet{};
    return v;
  }
  Ref i(PyNumber_Long(o));
  if (!i.get()) throw PyErrSet{};
  int64_t v = PyLong_AsLongLong(i.get());
  if (v == -1 && PyErr_Occurred()) throw PyErrSet{};
  return v;
}

// UTF-8 view of a str attribute plus its (cached) Python hash; the objects it points
// into are owned by the programs being encoded, which the caller keeps alive for the
// whole call.  Equality tests the hash first, so the small linear maps below cost an
// integer compare per entry.
struct Str {
  std::string_view v;
  Py_hash_t h = 0;
  bool operator==(const Str& o) const { return h == o.h && v == o.v; }
  bool operator==(const char* lit) const { return v == lit; }
  bool operator<(const Str& o) const { return v < o.v; }
  explicit operator std::string() const { return std::string(v); }
};

Str as_str(PyObject* o) {
  Py_ssize_t n;
  const char* s = PyUnicode_AsUTF8AndSize(o, &n);
  if (!s) throw PyErrSet{};
  Py_hash_t h = PyObject_Hash(o);
  if (h == -1) throw PyErrSet{};
  return Str{std::string_view(s, (size_t)n), h};
}

// small insertion-ordered map with dict assignment semantics (d[k] = v overwrites)
template <class V>
struct FlatMap {
  std::vector<std::pair<Str, V>> v;
  V* find(Str k) {
    for (auto& e : v)
      if (e.first == k) return &e.second;
    return nullptr;
  }
  const V* find(Str k) const {
    for (auto& e : v)
      if (e.first == k) return &e.second;
    return nullptr;
  }
  void set(Str k, V val) {
    if (V* x = find(k)) *x = std::move(val);
    else v.emplace_back(k, std::move(val));
  }
};

bool truthy(PyObject* o) {
  int t = PyObject_IsTrue(o);
  if (t < 0) throw PyErrSet{};
  return t != 0;
}

std::unordered_map<PyTypeObject*, int> g_kinds;

int kind_of(PyObject* o) {
  PyTypeObject* t = Py_TYPE(o);
  auto it = g_kinds.find(t);
  if (it != g_kinds.end()) return it->second;
  const char* full = t->tp_name;
  const char* dot = strrchr(full, '.');
  std::string nm = dot ? dot + 1 : full;
  static const std::pair<const char*, int> table[] = {
      {"DVar", K_DVAR}, {"DConst", K_DCONST}, {"DAdd", K_DADD}, {"DMul", K_DMUL}, {"DDiv", K_DDIV},
      {"DMod", K_DMOD}, {"Const", K_CONST}, {"IterVal", K_ITERVAL}, {"Read", K_READ}, {"Bin", K_BIN},
      {"Call", K_CALL}, {"Select", K_SELECT}, {"Reduce", K_REDUCE}};
  int k = K_OTHER;
  for (auto& e : table)
    if (nm == e.first) k = e.second;
  g_kinds[t] = k;
  return k;
}

// Python sequences (tuples / lists) as a vector of borrowed items kept alive by `hold`.
struct Seq {
  Ref hold;
  PyObject** items = nullptr;
  Py_ssize_t n = 0;
  explicit Seq(PyObject* o) : hold(PySequence_Fast(o, "expected a sequence")) {
    if (!hold.get()) throw PyErrSet{};
    items = PySequence_Fast_ITEMS(hold.get());
    n = PySequence_Fast_GET_SIZE(hold.get());
  }
};

struct LoopInfo {
  Str id;
  int64_t extent;      // int(extent or 1)
  int kind;            // 0 space, 1 reduce
  int ann;             // 0 None/other, 1 parallel, 2 vectorize
};

struct StageInfo {
  PyObject* obj;       // borrowed (the program's stage tuple holds it)
  Str name;
  bool inlined;
  bool has_at;
  Str at_stage, at_loop;
  bool loaded = false;          // loops / shape read (live stages, attach targets, read buffers)
  std::vector<LoopInfo> loops;
  std::vector<int64_t> shape;   // tuple(e for _, e in space)
};

LoopInfo read_loop(PyObject* l);

void load_loops(StageInfo& S) {
  if (S.loaded) return;
  S.loaded = true;
  Seq loops(attr(S.obj, N.loops).get());
  for (Py_ssize_t j = 0; j < loops.n; ++j) S.loops.push_back(read_loop(loops.items[j]));
  Seq space(attr(S.obj, N.space).get());
  for (Py_ssize_t j = 0; j < space.n; ++j) {
    Seq ax(space.items[j]);
    S.shape.push_back(as_i64(ax.items[1]));
  }
}

LoopInfo read_loop(PyObject* l) {
  LoopInfo L;
  L.id = as_str(attr(l, N.id).get());
  Ref e = attr(l, N.extent);
  L.extent = (e.get() == Py_None) ? 1 : as_i64(e.get());
  if (L.extent == 0) L.extent = 1;          // `extent or 1`
  L.kind = as_str(attr(l, N.kind).get()) == "space" ? 0 : 1;
  Ref an = attr(l, N.annotation);
  L.ann = 0;
  if (an.get() != Py_None) {
    Str s = as_str(an.get());
    L.ann = s == "parallel" ? 1 : s == "vectorize" ? 2 : 0;
  }
  return L;
}

// postfix form of a decode AST (encode._postfix): operands before operators
void postfix(PyObject* d, const FlatMap<int>& loop_idx, std::vector<int32_t>& out) {
  int k = kind_of(d);
  switch (k) {
    case K_DVAR: {
      Ref lpo = attr(d, N.loop);
      const int* it = loop_idx.find(as_str(lpo.get()));
      if (!it) {
        std::string r = PyUnicode_AsUTF8(Ref(PyObject_Repr(attr(d, N.loop).get())).get());
        throw EncodeError{"decode references unknown loop " + r};
      }
      out.push_back(OP_VAR);
      out.push_back(*it);
      return;
    }
    case K_DCONST:
      out.push_back(OP_CONST);
      out.push_back((int32_t)as_i64(attr(d, N.value).get()));
      return;
    case K_DADD:
      postfix(attr(d, N.a).get(), loop_idx, out);
      postfix(attr(d, N.b).get(), loop_idx, out);
      out.push_back(OP_ADD);
      out.push_back(0);
      return;
    case K_DMUL:
    case K_DDIV:
    case K_DMOD: {
      Ref c = attr(d, N.c);
      if (c.get() == Py_None) throw EncodeError{"symbolic factor in decode"};
      postfix(attr(d, N.a).get(), loop_idx, out);
      out.push_back(k == K_DMUL ? OP_MUL : k == K_DDIV ? OP_DIV : OP_MOD);
      out.push_back((int32_t)as_i64(c.get()));
      return;
    }
    default:
      throw EncodeError{std::string("unknown decode node ") + Py_TYPE(d)->tp_name};
  }
}

// one pre-order walk (expr.walk): Read nodes in order and op_counts buckets
void walk_expr(PyObject* e, std::vector<PyObject*>& reads, int32_t* ops, std::vector<Ref>& keep) {
  int k = kind_of(e);
  switch (k) {
    case K_READ:
      reads.push_back(e);
      return;
    case K_BIN: {
      Ref opo = attr(e, N.op);
      Str op = as_str(opo.get());
      int b = C_OTHER;
      if (op == "add") b = C_ADD;
      else if (op == "sub") b = C_SUB;
      else if (op == "mul") b = C_MUL;
      else if (op == "div") b = C_DIV;
      else if (op == "max" || op == "min") b = C_MINMAX;
      else if (op == "lt" || op == "le" || op == "gt" || op == "ge" || op == "eq") b = C_CMP;
      else throw EncodeError{"unknown binary op " + std::string(op)};
      ops[b]++;
      Ref l = attr(e, N.lhs), r = attr(e, N.rhs);
      walk_expr(l.get(), reads, ops, keep);
      walk_expr(r.get(), reads, ops, keep);
      keep.push_back(std::move(l));
      keep.push_back(std::move(r));
      return;
    }
    case K_CALL: {
      ops[C_MATH]++;
      Ref a = attr(e, N.arg);
      walk_expr(a.get(), reads, ops, keep);
      keep.push_back(std::move(a));
      return;
    }
    case K_SELECT: {
      ops[C_SELECT]++;
      Ref c = attr(e, N.cond), t = attr(e, N.then), o = attr(e, N.other);
      walk_expr(c.get(), reads, ops, keep);
      walk_expr(t.get(), reads, ops, keep);
      walk_expr(o.get(), reads, ops, keep);
      keep.push_back(std::move(c));
      keep.push_back(std::move(t));
      keep.push_back(std::move(o));
      return;
    }
    case K_REDUCE: {
      ops[as_str(attr(e, N.op).get()) == "sum" ? C_ADD : C_MINMAX]++;
      Ref b = attr(e, N.body);
      walk_expr(b.get(), reads, ops, keep);
      keep.push_back(std::move(b));
      return;
    }
    default:
      return;     // Const, IterVal: leaves without reads or ops
  }
}

struct Dim {
  int64_t size, st, pext, cnst;
  std::vector<std::pair<int, int64_t>> terms;
};

struct View {
  int n_marks = 0, has_w = 0;
  std::vector<Dim> dims;
};

class Encoder {
 public:
  std::vector<int32_t> words;
  std::vector<int64_t> stmt_off{0};

  int64_t encode_program(PyObject* p) {
    Seq stages_seq(attr(p, N.stages).get());
    std::vector<StageInfo> stages(stages_seq.n);
    FlatMap<int> smap;
    for (Py_ssize_t i = 0; i < stages_seq.n; ++i) {
      PyObject* s = stages_seq.items[i];
      StageInfo& S = stages[i];
      S.obj = s;
      S.name = as_str(attr(s, N.name).get());
      S.inlined = truthy(attr(s, N.inlined).get());
      Ref at = attr(s, N.compute_at);
      S.has_at = at.get() != Py_None;
      if (S.has_at) {
        Seq t(at.get());
        S.at_stage = as_str(t.items[0]);
        S.at_loop = as_str(t.items[1]);
      }
      if (!S.inlined) load_loops(S);
      smap.set(S.name, (int)i);   // dict: the last stage of a name wins
    }
    // layouts: buffer -> descriptor (dim, extent) pairs
    FlatMap<std::vector<std::pair<int, int64_t>>> layouts;
    {
      Seq lay(attr(p, N.layouts).get());
      for (Py_ssize_t i = 0; i < lay.n; ++i) {
        Seq kv(lay.items[i]);
        std::vector<std::pair<int, int64_t>> desc;
        Seq ds(kv.items[1]);
        for (Py_ssize_t j = 0; j < ds.n; ++j) {
          Seq de(ds.items[j]);
          desc.emplace_back((int)as_i64(de.items[0]), as_i64(de.items[1]));
        }
        layouts.set(as_str(kv.items[0]), std::move(desc));
      }
    }
    int n_live = 0;
    for (auto& S : stages) n_live += S.inlined ? 0 : 1;
    Ref dag = attr(p, N.dag);
    FlatMap<std::vector<int64_t>> node_shapes;
    int64_t emitted = 0;
    for (auto& S : stages) {
      if (S.inlined) continue;
      encode_stage(S, stages, smap, layouts, n_live, dag.get(), node_shapes);
      ++emitted;
    }
    return emitted;
  }

 private:
  void nest_above(const StageInfo& s, std::vector<StageInfo>& stages,
                  const FlatMap<int>& smap, std::vector<const LoopInfo*>& out, int depth) {
    if (!s.has_at) return;
    if (depth > 256) throw EncodeError{"compute_at cycle"};
    const int* it = smap.find(s.at_stage);
    if (!it) throw EncodeError{"compute_at references unknown stage " + std::string(s.at_stage)};
    StageInfo& t = stages[*it];
    load_loops(t);
    nest_above(t, stages, smap, out, depth + 1);
    int upto = -1;
    for (size_t j = 0; j < t.loops.size(); ++j)
      if (t.loops[j].id == s.at_loop) { upto = (int)j; break; }       // list.index: first match
    if (upto < 0) throw EncodeError{"compute_at references unknown loop " + std::string(s.at_loop)};
    for (int j = 0; j <= upto; ++j) out.push_back(&t.loops[j]);
  }

  void encode_stage(const StageInfo& S, std::vector<StageInfo>& stages,
                    const FlatMap<int>& smap, const FlatMap<std::vector<std::pair<int, int64_t>>>& layouts,
                    int n_live, PyObject* dag, FlatMap<std::vector<int64_t>>& node_shapes) {
    PyObject* s = S.obj;
    std::vector<const LoopInfo*> above_all, above, nest;
    nest_above(S, stages, smap, above_all, 0);
    for (auto* l : above_all)
      if (l->extent > 1) above.push_back(l);
    nest = above;
    for (auto& l : S.loops)
      if (l.extent > 1) nest.push_back(&l);
    FlatMap<int> loop_idx, last_pos;
    for (size_t j = 0; j < S.loops.size(); ++j) loop_idx.set(S.loops[j].id, (int)j);
    for (size_t q = 0; q < nest.size(); ++q) last_pos.set(nest[q]->id, (int)q);

    // index_map: iterator names in order, decode per name (dict: last wins)
    Seq imap(attr(s, N.index_map).get());
    std::vector<Str> iters;
    FlatMap<PyObject*> dmap;
    FlatMap<int> iter_idx;
    std::vector<Seq> kvs;
    kvs.reserve(imap.n);
    for (Py_ssize_t j = 0; j < imap.n; ++j) {
      kvs.emplace_back(imap.items[j]);
      Str nm = as_str(kvs.back().items[0]);
      iters.push_back(nm);
      dmap.set(nm, kvs.back().items[1]);
      iter_idx.set(nm, (int)j);
    }
    std::vector<int32_t> nodes, iter_tab;
    for (auto& nm : iters) {
      int start = (int)(nodes.size() / 2);
      postfix(*dmap.find(nm), loop_idx, nodes);
      iter_tab.push_back(start);
      iter_tab.push_back((int)(nodes.size() / 2) - start);
    }
    int n_extra = 0;
    auto iter_slot = [&](Str name) -> int {
      if (const int* it = iter_idx.find(name)) return *it;
      const int* li = loop_idx.find(name);
      if (!li) throw EncodeError{"iterator '" + std::string(name) + "' has no decode and no loop"};
      int slot = (int)iters.size() + n_extra++;
      iter_idx.set(name, slot);
      int start = (int)(nodes.size() / 2);
      nodes.push_back(OP_VAR);
      nodes.push_back(*li);
      iter_tab.push_back(start);
      iter_tab.push_back(1);
      return slot;
    };

    // accesses: reads (pre-order) then the write; op counts in the same walk
    Ref expr = attr(s, N.expr);
    std::vector<PyObject*> rd;
    std::vector<Ref> keep;
    int32_t ops[N_KINDS] = {0};
    if (expr.get() != Py_None) walk_expr(expr.get(), rd, ops, keep);
    FlatMap<int> vpos;
    std::vector<Str> order;
    std::vector<View> views;
    auto access = [&](Str buf, PyObject* index, int is_w) {
      const int* it = vpos.find(buf);
      int vi;
      if (!it) {
        // logical (const, [(iter slot, coeff)]) per dim, iter_slot called in dim / term order
        std::vector<std::pair<int64_t, std::vector<std::pair<int, int64_t>>>> logical;
        if (index == nullptr) {
          Seq space(attr(s, N.space).get());
          for (Py_ssize_t d = 0; d < space.n; ++d) {
            Seq ax(space.items[d]);
            logical.push_back({0, {{iter_slot(as_str(ax.items[0])), 1}}});
          }
        } else {
          Seq idx(index);
          for (Py_ssize_t d = 0; d < idx.n; ++d) {
            Ref cst = attr(idx.items[d], N.const_);
            Seq terms(attr(idx.items[d], N.terms).get());
            std::vector<std::pair<int, int64_t>> ts;
            for (Py_ssize_t t = 0; t < terms.n; ++t) {
              Seq nc(terms.items[t]);
              ts.emplace_back(iter_slot(as_str(nc.items[0])), as_i64(nc.items[1]));
            }
            logical.push_back({as_i64(cst.get()), std::move(ts)});
          }
        }
        View V;
        if (const auto* lay = layouts.find(buf)) {
          const auto& desc = *lay;
          for (size_t i = 0; i < desc.size(); ++i) {
            int64_t st = 1;
            for (size_t i2 = i + 1; i2 < desc.size(); ++i2)
              if (desc[i2].first == desc[i].first) st *= desc[i2].second;
            int d = desc[i].first;
            if (d < 0 || d >= (int)logical.size()) throw EncodeError{"layout dim out of range for " + std::string(buf)};
            V.dims.push_back({desc[i].second, st, desc[i].second, logical[d].first, logical[d].second});
          }
        } else {
          const std::vector<int64_t>* shape = nullptr;
          if (const int* si = smap.find(buf)) {
            load_loops(stages[*si]);
            shape = &stages[*si].shape;
          } else {
            const std::vector<int64_t>* ns = node_shapes.find(buf);
            if (!ns) {
              Ref bname(PyUnicode_FromStringAndSize(buf.v.data(), (Py_ssize_t)buf.v.size()));
              Ref node(PyObject_CallMethodObjArgs(dag, N.node, bname.get(), nullptr));
              if (!node.get()) throw PyErrSet{};
              Seq sh(attr(node.get(), N.shape).get());
              std::vector<int64_t> v;
              for (Py_ssize_t d = 0; d < sh.n; ++d) v.push_back(as_i64(sh.items[d]));
              node_shapes.set(buf, std::move(v));
              ns = node_shapes.find(buf);
            }
            shape = ns;
          }
          if (shape->size() < logical.size()) throw EncodeError{"access rank exceeds the shape of " + std::string(buf)};
          for (size_t d = 0; d < logical.size(); ++d)
            V.dims.push_back({(*shape)[d], 1, 0, logical[d].first, logical[d].second});
        }
        vi = (int)views.size();
        views.push_back(std::move(V));
        vpos.set(buf, vi);
        order.push_back(buf);
      } else {
        vi = *it;
      }
      views[vi].n_marks += 1;
      views[vi].has_w |= is_w;
    };
    for (PyObject* r : rd) {
      Ref buf = attr(r, N.buffer);
      Ref index = attr(r, N.index);
      access(as_str(buf.get()), index.get(), 0);
    }
    access(S.name, nullptr, 1);
    std::vector<Str> sorted_names = order;
    std::sort(sorted_names.begin(), sorted_names.end());
    FlatMap<int> rank;
    for (size_t r = 0; r < sorted_names.size(); ++r) rank.set(sorted_names[r], (int)r);

    // record
    std::vector<int32_t>& w = words;
    size_t rec0 = w.size();
    w.push_back((int32_t)nest.size());
    w.push_back((int32_t)above.size());
    w.push_back((int32_t)S.loops.size());
    w.push_back((int32_t)(iter_tab.size() / 2));
    w.push_back((int32_t)order.size());
    w.push_back((int32_t)as_i64(attr(s, N.pragma_unroll).get()));
    w.push_back(n_live);
    w.push_back(truthy(attr(s, N.reduce).get()) ? 1 : 0);
    for (int k = 0; k < N_KINDS; ++k) w.push_back(ops[k]);
    w.push_back((int32_t)(nodes.size() / 2));
    for (auto* l : nest) {
      const int* li = loop_idx.find(l->id);
      w.push_back((int32_t)l->extent);
      w.push_back(l->kind);
      w.push_back(l->ann);
      w.push_back(li ? *li : -1);
    }
    for (auto& l : S.loops) {
      const int* lp = last_pos.find(l.id);
      w.push_back((int32_t)l.extent);
      w.push_back(l.kind);
      w.push_back(lp ? *lp : -1);
    }
    w.insert(w.end(), iter_tab.begin(), iter_tab.end());
    w.insert(w.end(), nodes.begin(), nodes.end());
    for (auto& b : order) {
      const View& V = views[*vpos.find(b)];
      w.push_back(V.n_marks);
      w.push_back(V.has_w);
      w.push_back(*rank.find(b));
      w.push_back((int32_t)V.dims.size());
      for (auto& d : V.dims) {
        w.push_back((int32_t)d.size);
        w.push_back((int32_t)d.st);
        w.push_back((int32_t)d.pext);
        w.push_back((int32_t)d.cnst);
        w.push_back((int32_t)d.terms.size());
        for (auto& t : d.terms) {
          w.push_back(t.first);
          w.push_back((int32_t)t.second);
        }
      }
    }
    (void)rec0;
    stmt_off.push_back((int64_t)w.size());
  }
};

PyObject* g_encode_error = nullptr;

PyObject* encode_batch(PyObject*, PyObject* args) {
  PyObject* programs;
  if (!PyArg_ParseTuple(args, "O", &programs)) return nullptr;
  Encoder enc;
  std::vector<int64_t> prog_off{0};
  try {
    Seq ps(programs);
    for (Py_ssize_t i = 0; i < ps.n; ++i) prog_off.push_back(prog_off.back() + enc.encode_program(ps.items[i]));
  } catch (const EncodeError& e) {
    PyErr_SetString(g_encode_error ? g_encode_error : PyExc_ValueError, e.msg.c_str());
    return nullptr;
  } catch (const PyErrSet&) {
    return nullptr;
  }
  PyObject* w = PyBytes_FromStringAndSize((const char*)enc.words.data(), (Py_ssize_t)(enc.words.size() * 4));
  PyObject* so = PyBytes_FromStringAndSize((const char*)enc.stmt_off.data(), (Py_ssize_t)(enc.stmt_off.size() * 8));
  PyObject* po = PyBytes_FromStringAndSize((const char*)prog_off.data(), (Py_ssize_t)(prog_off.size() * 8));
  if (!w || !so || !po) {
    Py_XDECREF(w);
    Py_XDECREF(so);
    Py_XDECREF(po);
    return nullptr;
  }
  return Py_BuildValue("(NNN)", w, so, po);
}

PyObject* set_error(PyObject*, PyObject* args) {
  PyObject* cls;
  if (!PyArg_ParseTuple(args, "O", &cls)) return nullptr;
  Py_XINCREF(cls);
  Py_XDECREF(g_encode_error);
  g_encode_error = cls;
  Py_RETURN_NONE;
}

PyMethodDef methods[] = {
    {"encode_batch", encode_batch, METH_VARARGS,
     "encode_batch(programs) -> (words int32 bytes, stmt_offsets int64 bytes, prog_offsets int64 bytes)"},
    {"set_error", set_error, METH_VARARGS, "set the exception class raised for malformed States"},
    {nullptr, nullptr, 0, nullptr}};

PyModuleDef moddef = {PyModuleDef_HEAD_INIT, "_lt_encode", "Native State encoder (see encode.py)", -1, methods};

}  // namespace

PyMODINIT_FUNC PyInit__lt_encode(void) {
  if (!init_names()) return nullptr;
  return PyModule_Create(&moddef);
}
