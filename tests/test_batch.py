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
