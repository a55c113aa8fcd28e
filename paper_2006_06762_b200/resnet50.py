"""ResNet-50 (batch 16, NHWC) task list for the whole-network config
(BASELINE.json configs[4]).

The reference has no graph frontend (`SPEC.md:8`); the distinct conv subgraphs
were extracted from torchvision's resnet50 (v1.5: stride on the 3x3) by the
survey: 26 conv shapes with their instance counts (= `Task.weight`), plus the
classifier.  Each is built with the reference's own builders (`conv2d`,
`matmul`), so `make_task(name, dag, weight, structure="SSSRRSRS")` applies.
"""

from __future__ import annotations

from .state import Bin, ComputeDAG, Const, IterVal, Lin, Read, Reduce, compute, placeholder
from .state.workloads import build

v = Lin.var

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


def max_pool(n: int = 16, h: int = 112, c: int = 64, kernel: int = 3, stride: int = 2, pad: int = 1):
    """M[n,y,x,c] = max over a kernel x kernel window of the padded input.

    The pad stage mirrors the reference's conv padding (`src/workloads.py:45-67`,
    a `Select` over the in-bounds test); its fill is 0, which equals
    max-pooling's -inf padding here because the pooled tensor is a ReLU output
    (>= 0) and every window holds at least one real element."""
    from .state import Select
    hp = h + 2 * pad
    ho = (hp - kernel) // stride + 1
    inb = Bin("mul",
              Bin("mul", Bin("ge", IterVal(v("ph")), Const(float(pad))), Bin("lt", IterVal(v("ph")), Const(float(h + pad)))),
              Bin("mul", Bin("ge", IterVal(v("pw")), Const(float(pad))), Bin("lt", IterVal(v("pw")), Const(float(h + pad)))))
    x = placeholder("x", (n, h, h, c), iters=("x0", "x1", "x2", "x3"))
    pnode = compute("P", (("pn", n), ("ph", hp), ("pw", hp), ("pc", c)),
                    Select(inb, Read("x", (v("pn"), v("ph").shift(-pad), v("pw").shift(-pad), v("pc"))), Const(0.0)))
    body = Reduce("max", ("rh", "rw"), Read("P", (v("mn"), v("mh").scale(stride) + v("rh"),
                                                  v("mw").scale(stride) + v("rw"), v("mc"))))
    m = compute("M", (("mn", n), ("mh", ho), ("mw", ho), ("mc", c)), body, reduce=(("rh", kernel), ("rw", kernel)))
    return ComputeDAG((x, pnode, m))


def global_avg_pool(n: int = 16, h: int = 7, c: int = 2048):
    """G[n,c] = (sum over the h x h window) * 1/h²: a sum reduction and a scale."""
    x = placeholder("x", (n, h, h, c), iters=("x0", "x1", "x2", "x3"))
    s = compute("S", (("sn", n), ("sc", c)), Reduce("sum", ("rh", "rw"), Read("x", (v("sn"), v("rh"), v("rw"), v("sc")))),
                reduce=(("rh", h), ("rw", h)))
    g = compute("G", (("gn", n), ("gc", c)), Bin("mul", Read("S", (v("gn"), v("gc"))), Const(1.0 / (h * h))))
    return ComputeDAG((x, s, g))


def tasks(batch: int = 16, pools: bool = True, fusion: str = "conv"):
    """[(name, dag, weight)] for every distinct subgraph.

    fusion: "conv" — each convolution alone (inference: BN folds into the
    weights; the residual add and ReLU are elementwise consumers); "conv_bn_relu"
    — each convolution with its batch-norm affine and ReLU fused as one subgraph
    (the ConvLayer config's DAG, `state.workloads.conv_bn_relu`), the fusion the
    paper's Relay partitioning produces for the non-residual convolutions."""
    if fusion not in ("conv", "conv_bn_relu"):
        raise ValueError(f"unknown fusion {fusion!r}")
    out = []
    for h, ci, co, k, s, p, cnt in CONVS:
        name = f"conv{h}_{ci}_{co}_k{k}s{s}" + ("_bn_relu" if fusion == "conv_bn_relu" else "")
        out.append((name, build(fusion if fusion == "conv_bn_relu" else "conv2d", h=h, w=h, ci=ci, co=co, kernel=k,
                                stride=s, pad=p, n=batch), cnt))
    out.append(("dense2048_1000", build("matmul", n=batch, m=1000, k=2048), 1))
    if pools:
        out.append(("maxpool112_64_k3s2", max_pool(n=batch), 1))
        out.append(("avgpool7_2048", global_avg_pool(n=batch), 1))
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
