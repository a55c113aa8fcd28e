"""Plug the B200 path into an unchanged reference tuning loop.

`install(loomtune)` rebinds the module-level names the reference's tuner calls
(`src/sched.py:24-30`, `src/cli.py:25`):

* `measure_batch`  -> `paper_2006_06762_b200.measure.measure_batch` (GPU runner);
* `train`          -> `gbdt.train`: the same interface and a bit-identical model,
                      with every tree fitted on the GPU (`csrc/gbdt.cu`);
                      `install(..., gpu_train=False)` keeps the reference's own
                      `train` and wraps its result as `GpuCostModel`;
* `cli.cmd_replay` -> `replay.cmd_replay` (status parity exact, costs within a
                      tolerance, device recorded) and tune-log headers gain a
                      `runner` block (device, cost unit µs);
* `evolve`         -> `evolve_batched`: the reference's evolution loop
                      (`src/evolve.py:442-502`) verbatim in its random-number use,
                      except that each population is scored with one
                      `model.predict_batch(programs)` device pass instead of one
                      `model.predict(p)` per program (`src/evolve.py:453-454`).

Search semantics are untouched: with identical scores the batched evolve makes
the same draws and returns the same candidates as the reference's (tested in
tests/test_integrate.py).

Opt-in (`install(loomtune, gpu_features=True)`): the
8 `gpu_*` feature slots the reference leaves zero carry each statement's kernel
binding (blockIdx, threadIdx, vthread, shared bytes) in training rows and in
population scoring, so the cost model can tell launch shapes apart.

Opt-in (`install(loomtune, gpu_sampler=True)`): fresh
samples go through `make_gpu_sampler`, which draws the sketch's tile sizes with
the reference's own `random_factorization` until the tiled stages have a legal
launch shape (the reference's CPU-oriented draws give ~1-2% of those for tiled
sketches), then runs the reference's `sample_program` on that State.  This
changes the search distribution and is off by default.

Opt-in (`gpu_sketch_policy(loomtune, task, gpu_rules=True)`, SURVEY.md §8(f)
row 3): the task's sketches are derived with the paper's two GPU rules added to
the reference's rule table (`sketch_rules.py`: a shared-memory caching node for
computed operands, a cross-thread reduction) and only the sketches derived
through a GPU rule are kept (multi-level tiling — every tiled kernel stages its
operands through shared memory — reduction factorization, or the two GPU rules).
"""

from __future__ import annotations

import numpy as np

from .measure import measure_batch
from .model import GpuCostModel
from .replay import cmd_replay


def make_evolve_batched(ev, score_population=None):
    """Build the batched twin of `ev.evolve` from the reference module `ev`.

    `score_population(model, programs) -> fitness list` replaces the default
    one-pass `model.predict_batch(programs)` (the sharded scorer under
    torch.distributed, `dist.score_batch_sharded`)."""

    def evolve_batched(initial, model, config, rng=None, stats=None):
        if not initial:
            raise ValueError("empty initial population")
        if stats is None:
            stats = ev.EvolveStats()
        root = config.seed if rng is None else int(rng.integers(2 ** 62))

        gm = model if hasattr(model, "predict_batch") else GpuCostModel.wrap(model)

        def score(programs):
            fits = score_population(gm, programs) if score_population else gm.predict_batch(programs)
            return [ev.Candidate(p, float(f)) for p, f in zip(programs, fits)]

        pool: dict = {}
        order: dict = {}

        def absorb(cands):
            for c in cands:
                key = ev._state_key(c.program)
                if key not in pool or c.fitness > pool[key].fitness:
                    if key not in order:
                        order[key] = len(order)
                    pool[key] = c

        population = score(initial)
        absorb(population)
        for gen in range(config.generations):
            children = []
            for slot in range(config.population):
                r = np.random.default_rng((root, gen, slot))
                if r.random() < config.mutation_prob:
                    parent = ev.select_parent(population, r, stats)
                    child = ev._mutate_child(parent, config, r, stats)
                else:
                    pa = ev.select_parent(population, r, stats)
                    pb = ev.select_parent(population, r, stats)
                    out = ev.crossover(pa.program, pb.program, r)
                    stats.crossovers += 1
                    if isinstance(out, ev.Infeasible):
                        stats.infeasible_crossovers += 1
                        child = ev._mutate_child(pa, config, r, stats)
                    else:
                        child = out
                if r.random() < config.validate_fraction:
                    stats.validated += 1
                    problems = ev.validate(child)
                    if problems:
                        raise AssertionError(f"evolved child failed validation: {problems}")
                children.append(child)
            population = score(children)
            absorb(population)
            fits = sorted(c.fitness for c in population)
            stats.generation_best.append(fits[-1])
            stats.generation_median.append(fits[len(fits) // 2])
        ranked = sorted(pool, key=lambda k: (-pool[k].fitness, order[k]))
        return [pool[k] for k in ranked[: config.k]]

    return evolve_batched


def gpu_sane(p, min_threads: int = 32) -> bool:
    """A State whose lowering is legal and whose tiled kernels use a sane thread block."""
    from .lower import LoweringError, lower
    try:
        lo = lower(p)
    except LoweringError:
        return False
    return all(k.info.get("template") != "tiled" or k.info["threads"] >= min_threads for k in lo.kernels)


def _launch_ok(parts_by_stage: dict) -> bool:
    """Launch shape of the multi-level tiled stages from their 5-level space
    splits alone (S0 blockIdx, S1 vthread, S2 threadIdx, S3, S4): 32-1024
    threads, <= 8 vthreads, <= 256 accumulators (lower.py's limits)."""
    for splits in parts_by_stage.values():
        threads = vt = acc = 1
        for parts in splits:
            threads *= parts[2]
            vt *= parts[1]
            acc *= parts[1] * parts[3] * parts[4]
        if not (32 <= threads <= 1024 and vt <= 8 and acc <= 256):
            return False
    return True


def make_gpu_sampler(sample_program, tries: int = 64, factor_tries: int = 2048):
    """GPU-aware sampling around the reference's `sample_program` (src/annotate.py:346).

    The sketch's symbolic tile sizes are drawn with the reference's own
    `random_factorization` (as `resolve_factors`, src/annotate.py:84-102, deals
    them) until the tiled stages have a legal launch shape; the resolved State
    then goes through the unchanged `sample_program` (whose `resolve_factors`
    finds nothing left to draw: layout packing, compute-location moves and
    annotations are the reference's), and the result is kept when `gpu_sane`.
    Rejection at the factor level samples the same conditional distribution as
    rejecting whole programs, ~20x cheaper per draw."""
    import sys
    ann = sys.modules[sample_program.__module__]

    def resolve(sketch, rng):
        axes = {}
        for st in sketch.stages:
            axes[st.name] = dict((*st.space, *st.reduce))
        plan = []
        for step in sketch.history:
            if type(step).__name__ == "Split" and any(f is None for f in step.inner):
                ext = axes.get(step.stage, {}).get(step.loop)
                if ext is None:
                    return None                 # not an original axis: let the reference resolve
                plan.append((step, ext))
            elif type(step).__name__ == "Rfactor" and step.factor is None:
                return None
        parts_of = None
        for _ in range(factor_tries):
            parts_of = [ann.random_factorization(ext, len(step.inner) + 1, rng) for step, ext in plan]
            by_stage: dict = {}
            for (step, _), parts in zip(plan, parts_of):
                if len(parts) == 5:
                    by_stage.setdefault(step.stage, []).append(parts)
            if _launch_ok(by_stage):
                break
        it = iter(parts_of or [])
        p = ann.naive_program(sketch.dag)
        for step in sketch.history:
            if type(step).__name__ == "Split" and any(f is None for f in step.inner):
                step = ann.Split(step.stage, step.loop, tuple(next(it)[1:]))
            p = ann.apply_step(p, step)
        return p

    def sample(sketch, policy, rng):
        p = None
        for _ in range(tries):
            q = resolve(sketch, rng)
            p = sample_program(q if q is not None else sketch, policy, rng)
            if gpu_sane(p):
                return p
        return p
    return sample


# rule ids that give a stage a GPU kernel shape: the reference's multi-level
# tiling, tiling with fusion and reduction factorization (src/sketch.py:260-329;
# lowered as a cross-thread reduction, ptxgen._xreduce), and the paper's two GPU
# rules (sketch_rules.py: shared-memory caching node, cross-thread reduction)
GPU_SKETCH_RULES = frozenset((3, 4, 6, "gpu_smem", "gpu_ctr"))


def gpu_sketch_policy(loomtune, task, structure: str = "SSSRRSRS", gpu_rules: bool = False) -> list:
    """Opt-in GPU sketch policy: Ansor's GPU sketches
    always tile a data-reuse stage (multi-level tiling staged through shared
    memory) or bind a factored reduction to threads; the reference's CPU rule
    table also keeps the untiled derivations (rule 1 `skip` on every node).

    gpu_rules: derive the task's sketches again with the paper's two GPU rules
    added to the reference's rule table (`sketch_rules.GPU_RULES` through
    `generate_sketches(extra_rules=...)`).  Then keeps, in place and in order,
    the sketches whose rule path uses a GPU rule, when there is one; returns
    the kept rule paths.  Changes the search space, so it is off by default."""
    import importlib
    sk = importlib.import_module(loomtune.__name__ + ".sketch")
    if gpu_rules:
        from .sketch_rules import GPU_RULES
        traced = sk.generate_sketches_traced(task.dag, extra_rules=GPU_RULES, structure=structure)
        task.sketches[:] = [p for p, _ in traced]
    else:
        traced = sk.generate_sketches_traced(task.dag, structure=structure)
    if len(traced) != len(task.sketches):
        raise ValueError(f"task {task.name}: sketch list does not match its rule paths")
    keep = [i for i, (_, path) in enumerate(traced) if any(r in GPU_SKETCH_RULES for r in path)]
    if keep and len(keep) < len(traced):
        task.sketches[:] = [task.sketches[i] for i in keep]
        return [traced[i][1] for i in keep]
    return [path for _, path in traced]


def _world() -> int:
    try:
        import torch.distributed as dist
    except ImportError:
        return 1
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def install(loomtune, gpu_sampler: bool = False, gpu_train: bool = True, gpu_features: bool = False,
            sharded: bool | None = None, stand_in: dict | None = None) -> dict:
    """Rebind the reference's hot-path call sites; returns the originals.

    gpu_train: `train` fits its trees on the GPU (`gbdt.train`, bit-identical
    models; trees deeper than `gbdt.MAX_DEPTH` — the
    device kernel's frontier limit — are fitted by the reference's own `train`);
    False keeps the reference's own `train` and only wraps its result.

    sharded (default: a torch.distributed group with more than one rank is
    initialised): every measurement batch (`dist.measure_batch_sharded`) and
    every evolution population (`dist.score_batch_sharded`) is partitioned
    across the ranks, one GPU each; only the (status, cost) records and the
    fitness vector are all-gathered.  Every rank runs the same
    deterministic scheduler on the same gathered results, so the tune is
    identical on all ranks and to the single-GPU tune.

    stand_in: device-free replacements for the two device calls, for the CPU
    multi-process tests only — {"measure_records": fn(programs, seed) ->
    [measure.Record], "score": fn(model, programs) -> fitness list}."""
    import importlib
    sched = importlib.import_module(loomtune.__name__ + ".sched")
    cli = importlib.import_module(loomtune.__name__ + ".cli")
    ev = importlib.import_module(loomtune.__name__ + ".evolve")
    orig = {"measure_batch": sched.measure_batch, "train": sched.train, "evolve": sched.evolve,
            "cli.measure_batch": cli.measure_batch, "sample_program": sched.sample_program}
    ref_train = sched.train

    def train(records, hyper=None):
        from . import gbdt
        if gpu_train and (hyper is None or hyper.depth <= gbdt.MAX_DEPTH):
            m = gbdt.train(records, hyper)
        else:
            m = GpuCostModel.wrap(ref_train(records, hyper) if hyper is not None else ref_train(records))
        m.gpu_features = gpu_features
        return m

    orig["attach_features"] = sched.attach_features
    if gpu_features:            # opt-in: training rows carry the kernel binding
        from .features import extract_features

        def attach_features(record, program):
            record.feats = extract_features(program, gpu_features=True)
            return record
        sched.attach_features = attach_features

    logio = importlib.import_module(loomtune.__name__ + ".logio")
    orig["cli.cmd_replay"] = cli.cmd_replay
    orig["logio.LogWriter.write"] = logio.LogWriter.write
    ref_write = logio.LogWriter.write

    def write(self, record):            # header records name the B200 runner (cost unit µs)
        if record.get("kind") == "header" and "runner" not in record:
            from .replay import runner_header
            record = {**record, "runner": runner_header()}
        return ref_write(self, record)
    logio.LogWriter.write = write
    cli.cmd_replay = cmd_replay         # wall-clock replay
    stand_in = stand_in or {}
    if sharded is None:
        sharded = _world() > 1
    score_population = None
    mb = measure_batch
    if sharded:
        from . import dist as D
        records = stand_in.get("measure_records")

        def mb(programs, spec=None, limits=None, best_cost=None):
            return D.measure_batch_sharded(programs, spec, limits, best_cost, measure_records=records)
        scorer = stand_in.get("score")

        def score_population(gm, programs):
            if scorer is not None:
                return D.score_batch_sharded(gm, programs, score_fn=lambda ps: scorer(gm, ps))
            return D.score_batch_sharded(gm, programs)
    elif stand_in:
        if "measure_records" in stand_in:
            from .measure import MeasureLimits, normalise

            def mb(programs, spec=None, limits=None, best_cost=None):
                lim = limits or MeasureLimits()
                return normalise(stand_in["measure_records"](list(programs), lim.check_seed), best_cost,
                                 lim.cost_ceiling)
        if "score" in stand_in:
            score_population = stand_in["score"]
    sched.measure_batch = mb
    cli.measure_batch = mb
    sched.train = train
    sched.evolve = make_evolve_batched(ev, score_population)
    if gpu_sampler:
        sched.sample_program = make_gpu_sampler(orig["sample_program"])
    return orig


def uninstall(loomtune, orig: dict) -> None:
    import importlib
    sched = importlib.import_module(loomtune.__name__ + ".sched")
    cli = importlib.import_module(loomtune.__name__ + ".cli")
    sched.measure_batch = orig["measure_batch"]
    sched.train = orig["train"]
    sched.evolve = orig["evolve"]
    cli.measure_batch = orig["cli.measure_batch"]
    sched.sample_program = orig["sample_program"]
    if "attach_features" in orig:
        sched.attach_features = orig["attach_features"]
    if "cli.cmd_replay" in orig:
        cli.cmd_replay = orig["cli.cmd_replay"]
        importlib.import_module(loomtune.__name__ + ".logio").LogWriter.write = orig["logio.LogWriter.write"]
