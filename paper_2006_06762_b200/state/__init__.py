"""Host-side mirror of the reference's State data model (expr, DAG, loop-nest IR).

These are the types that cross the drop-in boundary: `measure_batch` receives
`Program`s, the cost model scores them.  The reference's own objects work
everywhere this package takes a Program; this mirror exists so the package (and
its GPU tests and bench) run without the reference installed.
"""

from .expr import Bin, Call, Const, IterVal, Lin, Read, Reduce, Select, op_counts, reads
from .graph import ComputeDAG, ComputeNode, compute, placeholder, topological_order
from .ir import (
    REDUCE, SPACE, Annotate, CacheWrite, ComputeAt, DAdd, DConst, DDiv, DMod, DMul, DVar, Fuse,
    Inline, IRError, LayoutRewrite, Loop, Program, Reorder, Rfactor, SetPragma, Simplify, Split,
    Stage, apply_step, d_eval, d_interval, d_vars, history_from_json, history_to_json,
    lin_to_decode, naive_program, replay, simplify, validate,
)
from .workloads import CONFIGS, REGISTRY, build, config_dag
