"""Batches of independent load-perturbed ACOPF instances (config C5).

SURVEY.md §8(e): a single instance does not shard, but a batch of
independent instances does. A batch of B instances is partitioned into
contiguous blocks: instance i goes to rank floor(i * G / B) of G ranks,
one process per GPU. Every rank

* builds its instances (host),
* computes the symbolic plan ONCE (condensed pattern, ordering, symbolic
  factorisation and device plans). Load perturbations change parameter
  values only, never the sparsity, so every instance
  on the rank reuses it,
* solves its instances back to back on its GPU.

There is no inter-GPU traffic until a single final gather. Each instance is
a fixed-size float64 record [x (n), objective, status code, iterations,
residual, constraint violation]; all ranks' records are all-gathered to
every rank with one NCCL collective (`gather_records`).

The reference has no batch solver. Its only multi-instance mechanism is
`run_suite(paths, parallel=P)` (src/bench.py:166-186), a process pool of
independent `solve_case` calls that redoes every symbolic step per case.
"""
from __future__ import annotations

import numpy as np

from .ipm import SolveReport, SolverOptions, solve

STATUS_CODES = {"optimal": 0, "max_iter": 1, "regularization_exhausted": 2,
                "line_search_failure": 3, "eval_error": 4}
STATUS_NAMES = {v: k for k, v in STATUS_CODES.items()}
N_META = 5   # objective, status, iterations, residual, violation


def partition(n_items: int, world: int, rank: int) -> range:
    """Contiguous block of instance indices of `rank` (i -> floor(i*G/B))."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank out of range")
    lo = -(-rank * n_items // world)           # ceil(rank * B / G)
    hi = -(-(rank + 1) * n_items // world)
    return range(lo, hi)


def perturbed_instances(tiles: int, seeds, limits: bool = True):
    """AcopfModels of the Appendix-B grid with per-bus load factors drawn
    from np.random.default_rng(seed) for each seed (host, once)."""
    from .acopf import build_acopf
    from .grids import tiled_case
    from .matpower import parse_matpower

    return [build_acopf(parse_matpower(tiled_case(tiles, limits=limits, seed=int(s))))
            for s in seeds]


def share_symbolic(models) -> None:
    """Let every model reuse the first model's symbolic plan and device
    workspace (identical sparsity is checked, not assumed)."""
    if not models:
        return
    ref = models[0]
    for m in models[1:]:
        for f in ("jac_rows", "jac_cols", "hess_rows", "hess_cols"):
            if not np.array_equal(getattr(m, f), getattr(ref, f)):
                raise ValueError(f"instances differ in sparsity ({f})")
    for m in models[1:]:
        m._kkt_cache = getattr(ref, "_kkt_cache", None)


def solve_batch(instances, options: SolverOptions | None = None) -> list[SolveReport]:
    """Solve AcopfModels back to back on the current GPU with one shared
    symbolic plan (computed by the first solve)."""
    opts = options if options is not None else SolverOptions()
    models = [am.model for am in instances]
    reports = []
    for i, am in enumerate(instances):
        if i > 0:
            share_symbolic([models[0], am.model])
        reports.append(solve(am.model, opts, constraint_ranges=am.ranges))
    return reports


def solve_batch_concurrent(instances, options: SolverOptions | None = None,
                           workers: int = 4) -> list[SolveReport]:
    """Solve the instances with `workers` host threads, each driving its own
    CUDA stream and its own symbolic plan; a 1,358-bus solve is
    latency-bound and leaves most of the GPU idle, so independent solves
    overlap.  Every persistent kernel is sized to 1/workers of the device
    (gn_set_concurrency) so concurrent kernels stay co-resident.  Results
    are bitwise those of solve_batch (the kernels are deterministic)."""
    import threading

    import torch

    from . import _lib as L

    opts = options if options is not None else SolverOptions()
    n = len(instances)
    workers = max(1, min(int(workers), n))
    if workers == 1:
        return solve_batch(instances, opts)
    dev = torch.cuda.current_device()
    results: list = [None] * n
    errors: list = []
    groups = [list(range(w, n, workers)) for w in range(workers)]

    def run(idxs):
        try:
            torch.cuda.set_device(dev)
            L.check(L.lib().gn_set_concurrency(workers))
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                first = None
                for i in idxs:
                    am = instances[i]
                    if first is not None:
                        share_symbolic([first, am.model])
                    results[i] = solve(am.model, opts, constraint_ranges=am.ranges)
                    first = first or am.model
            stream.synchronize()
        except BaseException as exc:   # surfaced in the caller
            errors.append(exc)
        finally:
            L.lib().gn_set_concurrency(1)

    threads = [threading.Thread(target=run, args=(g,)) for g in groups]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results


def pack_records(reports, n_var: int) -> np.ndarray:
    """[len(reports), n_var + N_META] float64 records."""
    out = np.full((len(reports), n_var + N_META), np.nan)
    for k, r in enumerate(reports):
        if r.x is not None:
            out[k, :n_var] = r.x
        out[k, n_var:] = (r.objective, STATUS_CODES.get(r.status, -1), r.iterations,
                          r.residual_scaled, r.constraint_violation)
    return out


def unpack_record(rec: np.ndarray, n_var: int) -> dict:
    return {"x": rec[:n_var].copy(), "objective": float(rec[n_var]),
            "status": STATUS_NAMES.get(int(rec[n_var + 1]), "unknown"),
            "iterations": int(rec[n_var + 2]), "residual_scaled": float(rec[n_var + 3]),
            "constraint_violation": float(rec[n_var + 4])}


def gather_records(local: np.ndarray, n_items: int, world: int, rank: int, device=None) -> np.ndarray:
    """All-gather every rank's records into [n_items, width] (one collective).

    Blocks have different lengths (contiguous partition), so each rank pads
    to the largest block; padding rows are dropped after the gather.
    """
    import torch
    import torch.distributed as dist

    width = local.shape[1]
    sizes = [len(partition(n_items, world, r)) for r in range(world)]
    cap = max(sizes)
    buf = np.full((cap, width), np.nan)
    buf[:local.shape[0]] = local
    dev = device if device is not None else torch.device("cpu")
    t = torch.as_tensor(buf, device=dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return np.concatenate([parts[r].cpu().numpy()[:sizes[r]] for r in range(world)], axis=0)
