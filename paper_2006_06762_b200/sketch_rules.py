"""The paper's two GPU sketch derivation rules (Ansor §4.3 "GPU Support",
`/root/reference/PAPER.md:687`), as `DerivationRule`s for the reference's own
rule engine (`generate_sketches(dag, extra_rules=GPU_RULES, structure=
"SSSRRSRS")`, `src/sketch.py:212-232,345-388`).  Opt-in: they change the
search space.

* `SharedMemoryCacheRule` — "utilizing shared memory by inserting a caching
  node (similar to Rule 5)".  A multi-level-tiled GPU kernel stages every
  operand of a reduction step (R0) through shared memory (ptxgen's tiled
  template).  When an operand is a computed producer (the conv padding stage
  `P`) rather than a placeholder, the rule makes that producer the caching
  node: it is attached at the consumer's innermost R0 loop, so each staging
  step computes exactly the producer's slice the tile reads, straight into
  shared memory (Ansor's `cache_read(…, "shared")` + `compute_at` R0), instead
  of materialising the whole producer in a separate kernel.  The reference's
  IR has no cache-read step; `ComputeAt` to the R0 loop is its exact
  equivalent for a computed operand, and placeholders are staged by every
  tiled kernel already.
* `CrossThreadReductionRule` — "cross-thread reduction (similar to Rule 6)".
  Like the reference's reduction factorisation (fuse the reduction loops,
  `Rfactor`), but with the GPU condition: a naive stage whose reduction
  offers at least a warp of parallelism and more parallelism than its space
  (Ansor's GPU rule; the CPU rule 6 needs a space below `small_space`).  The
  factored pair lowers to one kernel that binds rf to threadIdx.x and combines
  with warp shuffles (`ptxgen._xreduce`).
"""

from __future__ import annotations

from .reference import loomtune  # noqa: F401  (puts the reference on sys.path)

from loomtune.ir import IRError, ComputeAt, Fuse, Rfactor, apply_step  # noqa: E402
from loomtune.sketch import DerivationRule, generate_sketches, generate_sketches_traced  # noqa: E402

WARP = 32


def _tiled(stage) -> bool:
    """Multi-level tiled by rule 3/4: split loops (ids with a level suffix)."""
    return stage.compute_at is None and not stage.is_naive() and any("." in l.id for l in stage.loops)


class SharedMemoryCacheRule(DerivationRule):
    name = "gpu_shared_memory_cache"
    rule_id = "gpu_smem"

    def _target(self, state, ctx):
        p = state.program
        stage = state.focus_of(ctx.node_at(state))
        if not p.has_stage(stage):
            return None
        s = p.stage(stage)
        if s.inlined or s.compute_at is not None or s.reduce or p.attached_to(stage):
            return None
        readers = [r for r in p.readers_of(stage) if r.name != stage]
        if len(readers) != 1 or not readers[0].reduce or not _tiled(readers[0]):
            return None
        t = readers[0]
        r0 = f"{t.reduce[-1][0]}.0"
        if not any(l.id == r0 for l in t.loops):
            return None
        return stage, t.name, r0

    def applies(self, state, ctx):
        return self._target(state, ctx) is not None

    def expand(self, state, ctx):
        stage, host, loop = self._target(state, ctx)
        try:
            p = apply_step(state.program, ComputeAt(stage, host, loop))
        except IRError:
            return []
        return [self._advance(state, p)]


class CrossThreadReductionRule(DerivationRule):
    name = "gpu_cross_thread_reduction"
    rule_id = "gpu_ctr"

    def applies(self, state, ctx):
        p = state.program
        stage = state.focus_of(ctx.node_at(state))
        if not p.has_stage(stage):
            return False
        s = p.stage(stage)
        if s.inlined or s.compute_at is not None or not s.is_naive() or not s.reduce:
            return False
        if p.has_stage(f"{stage}.rf") or p.attached_to(stage):
            return False
        space = red = 1
        for _, e in s.space:
            space *= e or 1
        for _, e in s.reduce:
            red *= e or 1
        return red >= WARP and red > space

    def expand(self, state, ctx):
        stage = state.focus_of(ctx.node_at(state))
        p = state.program
        red = [l.id for l in p.stage(stage).loops if l.kind == "reduce"]
        fused = red[0]
        try:
            for nxt in red[1:]:
                p = apply_step(p, Fuse(stage, fused, nxt))
                fused = f"{fused}@{nxt}"
            p = apply_step(p, Rfactor(stage, fused, None))
        except IRError:
            return []
        return [self._advance(state, p)]


GPU_RULES = (SharedMemoryCacheRule(), CrossThreadReductionRule())


def gpu_sketches(dag, structure: str = "SSSRRSRS") -> list:
    """The reference's sketch generator with the two GPU rules added."""
    return generate_sketches(dag, extra_rules=GPU_RULES, structure=structure)


def gpu_sketches_traced(dag, structure: str = "SSSRRSRS") -> list:
    return generate_sketches_traced(dag, extra_rules=GPU_RULES, structure=structure)
