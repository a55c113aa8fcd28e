"""Run the scoring kernels (features, trees, segment sums) over a 2^16-program
population inside NVTX range "profile" (for ncu --nvtx-include profile/), and
print their CUDA-event times.

  python tools/profile_scoring.py [REPS]
"""

import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import load_stream  # noqa: E402
from paper_2006_06762_b200 import runtime as rt  # noqa: E402
from paper_2006_06762_b200.encode import encode_batch  # noqa: E402
from paper_2006_06762_b200.model import GpuCostModel  # noqa: E402
from paper_2006_06762_b200.state import replay  # noqa: E402


def main() -> None:
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    lib = rt.load()
    dag, stream = load_stream("RC")
    programs = [replay(dag, h) for h in stream[:256]]
    model = GpuCostModel.from_json(json.load(open(os.path.join(ROOT, "tests", "golden", "model.json"))))
    w, so, po = encode_batch(programs)
    n_rep = (1 << 16) // len(programs)
    words = np.tile(w, n_rep)
    soff = np.concatenate([so[:-1] + i * len(w) for i in range(n_rep)] + [[len(words)]])
    poff = np.concatenate([po[:-1] + i * po[-1] for i in range(n_rep)] + [[po[-1] * n_rep]]).astype(np.int64)
    n_stmt, n_prog = len(soff) - 1, len(poff) - 1
    dev = torch.device("cuda", 0)
    d_w, d_so, d_po = (torch.from_numpy(x).to(dev) for x in (words, soff, poff))
    rows = torch.empty((n_stmt, 164), dtype=torch.float64, device=dev)
    rs = torch.empty(n_stmt, dtype=torch.float64, device=dev)
    sc = torch.empty(n_prog, dtype=torch.float64, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    h = model.handle()
    sp = torch.cuda.current_stream().cuda_stream

    def run():
        rt.check(lib.lt_features_device_cm(d_w.data_ptr(), d_so.data_ptr(), n_stmt, rows.data_ptr(), err.data_ptr(),
                                        sp), "features")
        rt.check(lib.lt_predict_cols_device(h, rows.data_ptr(), n_stmt, rs.data_ptr(), sp), "trees")
        rt.check(lib.lt_segment_sum_device(rs.data_ptr(), d_po.data_ptr(), n_prog, sc.data_ptr(), sp), "sum")
    run()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("profile")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(json.dumps({"programs": n_prog, "statements": n_stmt, "ms_per_pass": e0.elapsed_time(e1) / reps,
                      "err": int(err.item())}))


if __name__ == "__main__":
    main()
