"""Whole-network config (BASELINE.json configs[4]): the
reference's unchanged multi-task `tune` over the ResNet-50 task list
(convolutions, classifier, max-pool, global average pool) with the B200 path
installed — a few units through tools/tune_network.py."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tune_network_smoke():
    out = os.path.join(ROOT, "gpurun_out", "tune_network.json")
    if os.path.exists(out):
        os.remove(out)
    # 26 tasks: the first unit of every task measures its naive program and one batch
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tune_network.py"), "28", "0",
                        "--gpu-sampler", "--gpu-rules"], capture_output=True, text=True, timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.load(open(out))
    assert res["tasks"] == 26
    names = {t["task"] for t in res["per_task"]}
    assert {"maxpool112_64_k3s2", "avgpool7_2048", "dense2048_1000"} <= names
    assert res["valid"] > 0.5 * res["measured"]
    for t in res["per_task"]:
        assert t["best_us"] > 0 and t["best_us"] <= t["naive_us"] * 1.0001, t
    assert res["network_latency_us"] < res["naive_network_latency_us"]
