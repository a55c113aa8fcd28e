"""Every template path on real candidates: the first States of each golden stream
(the reference sampler's own candidates for RC, G10, CL, TBG) are measured on the
B200 and every one must verify against the fp64 ground truth (max relative error
<= 1e-4, north star).  The sample is checked to cover the naive template, tiled
kernels with cp.async staging, synchronous staging, and -O1 (register-overflow)
modules, so a regression in any of them fails here."""

import pytest

pytestmark = pytest.mark.gpu

N = 24


@pytest.fixture(scope="module")
def runner():
    from paper_2006_06762_b200 import measure
    r = measure.configure(device=0, cache_dir="")
    yield r
    measure._shutdown()


def test_stream_candidates_verify_on_every_template_path(runner):
    from bench import load_stream
    from paper_2006_06762_b200.state import replay
    paths = set()
    for cfg in ("RC", "G10", "CL", "TBG"):
        dag, stream = load_stream(cfg)
        recs = runner.measure_programs([replay(dag, h) for h in stream[:N]])
        for i, rec in enumerate(recs):
            assert rec.status == "valid", (cfg, i, rec.detail)
            assert rec.max_rel_err <= 1e-4, (cfg, i, rec.max_rel_err)
            for k in rec.info.get("kernels", []):
                if k["template"] == "naive":
                    paths.add("naive")
                elif k.get("async_copy"):
                    paths.add("async")
                else:
                    paths.add("sync")
                if k.get("ptxas"):
                    paths.add("O1")
    assert {"naive", "async", "sync", "O1"} <= paths, paths
