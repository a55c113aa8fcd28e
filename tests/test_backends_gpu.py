"""The PTX backend and the CUDA-C (NVRTC) backend implement the same templates:
same legality verdicts, both correct on every candidate, same kernel shapes
(except the cross-thread reduction of rule-6 States, PTX only: NVRTC keeps the
two naive kernels)."""

import pytest

pytestmark = pytest.mark.gpu


def test_ptx_and_nvrtc_agree(corpus):
    from paper_2006_06762_b200 import measure
    idx = [i for i, e in enumerate(corpus.entries) if i % 4 == 0]
    progs = [corpus.programs[i] for i in idx]
    r_ptx = measure.configure(device=0, cache_dir="", backend="ptx").measure_programs(progs)
    r_c = measure.configure(device=0, cache_dir="", backend="nvrtc").measure_programs(progs)
    for k, (a, b) in enumerate(zip(r_ptx, r_c)):
        assert a.status == b.status, (idx[k], a.detail, b.detail)
        if a.status == "valid":
            assert a.max_rel_err <= 1e-4 and b.max_rel_err <= 1e-4
            if any(x["template"] == "xreduce" for x in a.info["kernels"]):
                assert [x["template"] for x in b.info["kernels"]][:2] == ["naive", "naive"]
                continue
            ka = [(x["template"], x.get("threads"), x.get("blocks"), x.get("acc")) for x in a.info["kernels"]]
            kb = [(x["template"], x.get("threads"), x.get("blocks"), x.get("acc")) for x in b.info["kernels"]]
            assert ka == kb
    measure._shutdown()
