"""ResNet-50 (batch 16, NHWC) task list for the whole-network config
(BASELINE.json configs[4]).

The reference has no graph frontend (`SPEC.md:8`); the distinct conv subgraphs
were extracted from torchvision's resnet50 (v1.5: stride on the 3x3) by the
survey: 26 conv shapes with their instance counts (= `Task.weight`), plus the
classifier.  Each is built with the reference's own builders (`conv2d`,
`matmul`), so `make_task(name, dag, weight, structure="SSSRRSRS")` applies.
"""

from __future__ import annotations

from .state.workloads import build

# (input H=W, Ci, Co, kernel, stride, pad, count)
CONVS = [
    (224, 3, 64, 7, 2, 3, 1),
    (56, 64, 64, 1, 1, 0, 1),
    (56, 64, 64, 3, 1, 1, 3),
    (56, 64, 256, 1, 1, 0, 4),
    (56, 128, 128, 3, 2, 1, 1),
    (56, 256, 64, 1, 1, 0, 2),
    (56, 256, 128, 1, 1, 0, 1),
    (56, 256, 512, 1, 2, 0, 1),
    (28, 128, 512, 1, 1, 0, 4),
    (28, 128, 128, 3, 1, 1, 3),
    (28, 256, 256, 3, 2, 1, 1),
    (28, 512, 128, 1, 1, 0, 3),
    (28, 512, 256, 1, 1, 0, 1),
    (28, 512, 1024, 1, 2, 0, 1),
    (14, 256, 1024, 1, 1, 0, 6),
    (14, 256, 256, 3, 1, 1, 5),
    (14, 512, 512, 3, 2, 1, 1),
    (14, 1024, 256, 1, 1, 0, 5),
    (14, 1024, 512, 1, 1, 0, 1),
    (14, 1024, 2048, 1, 2, 0, 1),
    (7, 512, 2048, 1, 1, 0, 3),
    (7, 512, 512, 3, 1, 1, 2),
    (7, 2048, 512, 1, 1, 0, 2),
]


def tasks(batch: int = 16):
    """[(name, dag, weight)] for every distinct subgraph."""
    out = []
    for h, ci, co, k, s, p, cnt in CONVS:
        name = f"conv{h}_{ci}_{co}_k{k}s{s}"
        out.append((name, build("conv2d", h=h, w=h, ci=ci, co=co, kernel=k, stride=s, pad=p, n=batch), cnt))
    out.append(("dense2048_1000", build("matmul", n=batch, m=1000, k=2048), 1))
    return out


def flops(dag) -> int:
    """Algorithmic multiply-add FLOPs (2 per MAC) of the DAG's reducing node."""
    for n in dag.nodes:
        if n.reduce:
            v = 2
            for _, e in (*n.space, *n.reduce):
                v *= e
            return v
    return 0
