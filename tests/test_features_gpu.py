"""GPU feature kernel and tree kernel vs the reference's own outputs (golden) and the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-6   # north star: features within 1e-6 (absolute on the log2-compressed row)


def test_features_match_reference_golden(corpus):
    from paper_2006_06762_b200.features import extract_features_batch
    got = extract_features_batch(corpus.programs)
    worst, exact = 0.0, 0
    for i, g in enumerate(got):
        w = corpus.features_of(i)
        assert g.shape == w.shape, i
        assert np.isfinite(g).all(), i
        d = float(np.max(np.abs(g - w))) if g.size else 0.0
        worst = max(worst, d)
        exact += bool(np.array_equal(g, w))
    assert worst <= TOL, worst
    print(f"features: {exact}/{len(got)} programs bit-exact, worst abs diff {worst:.3g}")


def test_scores_match_reference_golden(corpus):
    from paper_2006_06762_b200.model import GpuCostModel
    m = GpuCostModel.from_json(corpus.model_json)
    got = m.predict_batch(corpus.programs)
    want = corpus.scores
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-12)
    assert float(rel.max()) <= 1e-5, float(rel.max())
    print(f"scores: {int((got == want).sum())}/{len(got)} bit-exact")


def test_predict_rows_matches_oracle_on_golden_rows(corpus):
    from oracle import predict as OP
    from paper_2006_06762_b200.model import GpuCostModel
    m = GpuCostModel.from_json(corpus.model_json)
    X = corpus.rows
    got = m.predict_rows(X)
    want = OP.predict_rows(OP.load_model(corpus.model_json), X)
    assert np.array_equal(got, want)


def test_empty_model_scores_zero(corpus):
    from paper_2006_06762_b200.model import GpuCostModel
    assert (GpuCostModel().predict_batch(corpus.programs[:10]) == 0.0).all()


def test_pairwise_sum_order_many_rows():
    """Programs with >= 8 rows must follow numpy's pairwise summation."""
    from paper_2006_06762_b200.model import GpuCostModel
    rng = np.random.default_rng(0)
    model = GpuCostModel.from_json({"base": 0.0, "n_features": 164, "shrinkage": 0.3, "depth": 1, "trees": [
        {"eta": 1.0, "feature": [0, -1, -1], "threshold": [0.5, 0.0, 0.0], "left": [1, 0, 0], "right": [2, 0, 0],
         "value": [0.0, 1e16, 1.0]}]})
    mats = []
    for n in (1, 3, 7, 8, 11, 127, 129, 300):
        X = rng.random((n, 164))
        X[0, 0] = 0.1  # first row -> 1e16 leaf, the rest mostly 1.0 or 1e16
        mats.append(X)
    got = model.predict_matrices(mats)
    for g, X in zip(got, mats):
        rows = np.where(X[:, 0] <= 0.5, 1e16, 1.0)
        assert g == float(rows.sum())


def test_column_major_features_and_predict_match_row_major(corpus):
    """lt_features_device_cm (+ lt_cols_to_rows_device) and lt_predict_cols_device
    are bit-identical to the row-major entry points on the golden corpus."""
    import torch
    from paper_2006_06762_b200 import runtime as rt
    from paper_2006_06762_b200.encode import encode_batch
    from paper_2006_06762_b200.model import GpuCostModel
    lib = rt.load()
    words, soff, _ = encode_batch(corpus.programs)
    n = len(soff) - 1
    dev = torch.device("cuda", 0)
    d_w, d_so = torch.from_numpy(words).to(dev), torch.from_numpy(soff).to(dev)
    rows = torch.empty((n, 164), dtype=torch.float64, device=dev)
    cols = torch.empty((164, n), dtype=torch.float64, device=dev)
    back = torch.empty((n, 164), dtype=torch.float64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    sp = torch.cuda.current_stream().cuda_stream
    rt.check(lib.lt_features_device(d_w.data_ptr(), d_so.data_ptr(), n, rows.data_ptr(), err.data_ptr(), sp), "rm")
    rt.check(lib.lt_features_device_cm(d_w.data_ptr(), d_so.data_ptr(), n, cols.data_ptr(), err.data_ptr(), sp), "cm")
    rt.check(lib.lt_cols_to_rows_device(cols.data_ptr(), n, back.data_ptr(), sp), "transpose")
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert torch.equal(rows, back)
    assert torch.equal(rows.t().contiguous(), cols)
    m = GpuCostModel.from_json(corpus.model_json)
    a = torch.empty(n, dtype=torch.float64, device=dev)
    b = torch.empty(n, dtype=torch.float64, device=dev)
    rt.check(lib.lt_predict_rows_device(m.handle(), rows.data_ptr(), n, a.data_ptr(), sp), "rows")
    rt.check(lib.lt_predict_cols_device(m.handle(), cols.data_ptr(), n, b.data_ptr(), sp), "cols")
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_opt_in_gpu_feature_slots(corpus):
    """gpu_features=True fills columns 51-58 with log2(1 + kernel binding) and
    leaves every other column exactly as the reference's layout."""
    from paper_2006_06762_b200.features import extract_features_batch
    from paper_2006_06762_b200.lower import gpu_binding
    progs = corpus.programs[:64]
    base = extract_features_batch(progs)
    gpu = extract_features_batch(progs, gpu_features=True)
    for p, a, b in zip(progs, base, gpu):
        keep = [k for k in range(164) if not 51 <= k <= 58]
        assert np.array_equal(a[:, keep], b[:, keep])
        assert not a[:, 51:59].any()
        live = [s for s in p.stages if not s.inlined]
        for row, s in zip(b, live):
            nb, nt, nv, smem = gpu_binding(p, s)
            want = np.log2(1.0 + np.asarray([nb, 1, 1, nt, 1, 1, nv, smem], np.float64))
            assert np.allclose(row[51:59], want, rtol=0, atol=1e-12)


def _stream_programs(n_per_cfg=256):
    import bench
    from paper_2006_06762_b200.state import replay
    progs = []
    for cfg in ("RC", "CL", "G10", "TBG"):
        dag, stream = bench.load_stream(cfg)
        progs += [replay(dag, h) for h in stream[:n_per_cfg]]
    return progs


def test_warp_and_thread_feature_kernels_agree_bitwise(corpus, monkeypatch):
    """The thread-per-statement kernel (default) and the warp-per-statement
    kernel compute every row identically (golden corpus + stream States)."""
    from paper_2006_06762_b200.features import extract_features_batch
    progs = list(corpus.programs) + _stream_programs()
    thread = extract_features_batch(progs)
    monkeypatch.setenv("LT_FEATURES_WARP", "1")
    warp = extract_features_batch(progs)
    monkeypatch.delenv("LT_FEATURES_WARP")
    for i, (a, b) in enumerate(zip(warp, thread)):
        assert np.array_equal(a, b), i


def test_tree_per_warp_and_thread_per_row_predict_agree_bitwise(corpus, monkeypatch):
    """The three predict kernels — perfect-tree walk (default), irregular
    tree-per-warp, thread-per-row — give bit-identical scores, equal to the
    golden scores; also for a model with early leaves, a depth-0 tree and NaN
    features (the padded subtrees must not change the leaf)."""
    from paper_2006_06762_b200.model import GpuCostModel
    progs = list(corpus.programs) + _stream_programs()
    ragged = {"base": 0.25, "n_features": 164, "shrinkage": 0.3, "depth": 3, "trees": [
        {"eta": 0.3, "feature": [5, -1, 7, -1, -1], "threshold": [0.5, 0, 1.5, 0, 0], "left": [1, 0, 3, 0, 0],
         "right": [2, 0, 4, 0, 0], "value": [0, 0.125, 0, -2.0, 3.5]},
        {"eta": 0.3, "feature": [-1], "threshold": [0.0], "left": [0], "right": [0], "value": [0.75]},
        {"eta": 0.3, "feature": [161, 162, -1, 9, -1, -1, -1], "threshold": [2.0, 1.0, 0, 0.0, 0, 0, 0],
         "left": [1, 3, 0, 5, 0, 0, 0], "right": [2, 4, 0, 6, 0, 0, 0],
         "value": [0, 0, 1.0, 0, 2.0, -1.0, 4.0]}]}
    for mj in (corpus.model_json, ragged):
        m = GpuCostModel.from_json(mj)
        X = np.vstack([corpus.features_of(i) for i in range(len(corpus.programs))])
        X[::7, 5] = np.nan
        X[::5, 161] = np.nan
        got = []
        for env in (None, "LT_PREDICT_IRREGULAR", "LT_PREDICT_THREAD_PER_ROW"):
            if env:
                monkeypatch.setenv(env, "1")
            got.append((m.predict_batch(progs), m.predict_rows(X)))
            if env:
                monkeypatch.delenv(env)
        for a, b in got[1:]:
            assert np.array_equal(got[0][0], a) and np.array_equal(got[0][1], b, equal_nan=True)
        from oracle import predict as OP
        assert np.array_equal(got[0][1], OP.predict_rows(OP.load_model(mj), X), equal_nan=True)
        if mj is corpus.model_json:
            assert np.array_equal(got[0][0][:len(corpus.scores)], corpus.scores)


def test_c_abi_comm_single_rank_roundtrip():
    """The C-ABI multi-GPU exchange (csrc/comm.cu, NCCL) on a one-rank
    communicator: all-gather and broadcast are the identity."""
    import ctypes
    from paper_2006_06762_b200 import runtime as rt
    lib = rt.load()
    uid = ctypes.create_string_buffer(128)
    rt.check(lib.lt_comm_unique_id(uid), "unique id")
    comm = lib.lt_comm_create(uid.raw, 0, 1, 0)
    assert comm, lib.lt_last_error().decode()
    try:
        rank, world = ctypes.c_int(), ctypes.c_int()
        rt.check(lib.lt_comm_rank(comm, ctypes.byref(rank), ctypes.byref(world)), "rank")
        assert (rank.value, world.value) == (0, 1)
        fit = np.arange(37, dtype=np.float64) * 0.5
        out = np.zeros_like(fit)
        rt.check(lib.lt_comm_allgather_f64(comm, rt.ptr(fit, rt.c_f64p), len(fit), rt.ptr(out, rt.c_f64p)), "gather")
        assert np.array_equal(out, fit)
        recs = (rt.MeasureRecord * 3)()
        for i in range(3):
            recs[i].cost_us, recs[i].status = 10.0 + i, i % 2
        got = (rt.MeasureRecord * 3)()
        rt.check(lib.lt_comm_allgather_records(comm, ctypes.addressof(recs), 3, ctypes.addressof(got)), "records")
        assert [(r.cost_us, r.status) for r in got] == [(10.0, 0), (11.0, 1), (12.0, 0)]
        blob = np.frombuffer(b"model-json" * 100, dtype=np.uint8).copy()
        rt.check(lib.lt_comm_broadcast(comm, blob.ctypes.data, blob.nbytes, 0), "broadcast")
        assert blob.tobytes() == b"model-json" * 100
    finally:
        lib.lt_comm_destroy(comm)
