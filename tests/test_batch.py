"""Batch (config C5) host logic: contiguous partition, record packing and the
final gather over a real 2-process gloo group (CPU), plus a GPU check that
a batched solve with a shared symbolic plan equals solving alone."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2307_16830_b200 import batch as B


def test_partition_is_contiguous_and_complete():
    for n in (1, 7, 256):
        for g in (1, 2, 3, 4, 8):
            blocks = [B.partition(n, g, r) for r in range(g)]
            flat = [i for b in blocks for i in b]
            assert flat == list(range(n))
            # i -> floor(i * G / B)
            for r, b in enumerate(blocks):
                assert all((i * g) // n == r for i in b)


def test_pack_unpack_roundtrip():
    class R:
        x = np.arange(5.0)
        objective, status, iterations = 12.5, "optimal", 17
        residual_scaled, constraint_violation = 1e-7, 2e-8

    rec = B.pack_records([R()], 5)
    u = B.unpack_record(rec[0], 5)
    assert u["status"] == "optimal" and u["iterations"] == 17 and u["objective"] == 12.5
    np.testing.assert_array_equal(u["x"], R.x)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_items, width, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = list(B.partition(n_items, world, rank))
    local = np.array([[i * 10.0 + c for c in range(width)] for i in idx]).reshape(len(idx), width)
    full = B.gather_records(local, n_items, world, rank)
    if rank == 0:
        np.save(out, full)
    dist.destroy_process_group()


@pytest.mark.parametrize("n_items", [7, 8])
def test_gather_records_gloo_world2(tmp_path, n_items):
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), n_items, 3, out), nprocs=2, join=True)
    full = np.load(out)
    expect = np.array([[i * 10.0 + c for c in range(3)] for i in range(n_items)])
    np.testing.assert_array_equal(full, expect)


@pytest.mark.gpu
def test_batched_solve_equals_single_solves():
    from paper_2307_16830_b200 import SolverOptions, solve

    inst = B.perturbed_instances(4, [0, 1, 2])
    opts = SolverOptions(tol=1e-6)
    reps = B.solve_batch(inst, opts)
    for am, r in zip(B.perturbed_instances(4, [0, 1, 2]), reps):
        alone = solve(am.model, opts, constraint_ranges=am.ranges)
        assert r.status == alone.status == "optimal"
        assert r.iterations == alone.iterations
        np.testing.assert_array_equal(r.x, alone.x)   # deterministic, shared plan


@pytest.mark.gpu
def test_concurrent_batch_is_bitwise_sequential():
    from paper_2307_16830_b200 import SolverOptions

    opts = SolverOptions(tol=1e-6)
    seq = B.solve_batch(B.perturbed_instances(4, range(6)), opts)
    con = B.solve_batch_concurrent(B.perturbed_instances(4, range(6)), opts, workers=3)
    for a, b in zip(seq, con):
        assert a.status == b.status == "optimal" and a.iterations == b.iterations
        np.testing.assert_array_equal(a.x, b.x)


@pytest.mark.gpu
@pytest.mark.parametrize("tiles,seeds", [(4, range(5)), (97, range(6))])
def test_instance_batched_solve_is_bitwise_single(tiles, seeds):
    """K12: ONE batched solve (one launch per kernel for all instances, shared
    plans) gives every instance exactly the iterates of solving it alone:
    same status, iteration count, per-iteration trace and x (bitwise)."""
    from paper_2307_16830_b200 import SolverOptions, solve
    from paper_2307_16830_b200.batch_ipm import solve_batched

    opts = SolverOptions(tol=1e-6)
    reps = solve_batched(B.perturbed_instances(tiles, list(seeds)), opts)
    for am, r in zip(B.perturbed_instances(tiles, list(seeds)), reps):
        alone = solve(am.model, opts, constraint_ranges=am.ranges)
        assert r.status == alone.status == "optimal"
        assert r.iterations == alone.iterations
        assert r.trace == alone.trace
        np.testing.assert_array_equal(r.x, alone.x)
        assert r.objective == alone.objective
        assert r.constraint_violation == alone.constraint_violation


@pytest.mark.gpu
def test_instance_batched_c5_matches_reference(end_to_end):
    """The three C5 instances with reference goldens (make_golden.py), solved
    inside one batch: objective 1e-6 relative, iterations +-2."""
    from paper_2307_16830_b200 import SolverOptions
    from paper_2307_16830_b200.batch_ipm import solve_batched

    reps = solve_batched(B.perturbed_instances(97, [0, 1, 2]), SolverOptions(tol=1e-6))
    for seed, r in enumerate(reps):
        ref = end_to_end[f"C5s{seed}@1e-06"]
        assert r.status == ref["status"] == "optimal"
        assert r.objective == pytest.approx(ref["objective"], rel=1e-6)
        assert abs(r.iterations - ref["iterations"]) <= 2


@pytest.mark.gpu
def test_instance_batched_regularization_and_masking():
    """Instances that need the inertia correction (concave objective) and
    instances that converge at different iterations, in one batch: every
    instance equals its single solve (the delta_w schedule per instance, the
    finished ones masked out of every state-changing kernel)."""
    from paper_2307_16830_b200 import SolverOptions, solve
    from paper_2307_16830_b200.batch_ipm import solve_batched
    from paper_2307_16830_b200.expressions import param, var
    from paper_2307_16830_b200.model import ModelBuilder

    def model(w):
        b = ModelBuilder()
        b.add_variables(3, np.full(3, -1.0), np.full(3, 2.0), np.zeros(3))
        b.add_objective(-(var(0) - param(0)) ** 2 + param(1) * var(0) * var(1),
                        np.array([[0, 1], [1, 2], [2, 0]]), np.array([[0.3, w], [0.1, w], [-0.2, w]]))
        b.add_constraints(var(0) + var(1) + var(2) - 1.0, np.array([[0, 1, 2]]), np.zeros((1, 0)))
        return b.finalize()

    ws = (0.5, -0.4, 0.1, 1.5)
    opts = SolverOptions(tol=1e-8)
    reps = solve_batched([(model(w), None) for w in ws], opts)
    its = set()
    for w, r in zip(ws, reps):
        alone = solve(model(w), opts)
        assert r.status == alone.status
        assert r.iterations == alone.iterations
        assert [t[6] for t in r.trace] == [t[6] for t in alone.trace]
        np.testing.assert_array_equal(r.x, alone.x)
        its.add(r.iterations)
    assert any(t[6] > 0 for r in reps for t in r.trace)
