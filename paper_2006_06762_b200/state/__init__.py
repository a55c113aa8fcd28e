"""The host data model: the reference's own State types, imported unchanged.

`measure_batch` receives reference `Program`s and the cost model scores them,
so this package reads the reference's objects directly (`loomtune.expr`,
`loomtune.graph`, `loomtune.ir`; found by `paper_2006_06762_b200.reference`).
Only two things are defined here: `kind` (class-name dispatch used by the
lowering and the encoder) and, in `workloads`, the DAG builders for the two
BASELINE configs the reference's registry lacks (TBG, ConvLayer).
"""

from ..reference import loomtune  # noqa: F401  (puts the reference on sys.path)

from loomtune.expr import (  # noqa: E402
    Bin, Call, Const, IterVal, Lin, Read, Reduce, Select, op_counts, reads,
)
from loomtune.graph import ComputeDAG, ComputeNode, compute, placeholder, topological_order  # noqa: E402
from loomtune.ir import (  # noqa: E402
    REDUCE, SPACE, Annotate, CacheWrite, ComputeAt, DAdd, DConst, DDiv, DMod, DMul, DVar, Fuse,
    Inline, IRError, LayoutRewrite, Loop, Program, Reorder, Rfactor, SetPragma, Simplify, Split,
    Stage, apply_step, d_eval, d_interval, d_vars, history_from_json, history_to_json,
    lin_to_decode, naive_program, replay, simplify, validate,
)

from .workloads import CONFIGS, REGISTRY, build, config_dag  # noqa: E402


def kind(e) -> str:
    """Class-name dispatch over expression / decode nodes."""
    return type(e).__name__
