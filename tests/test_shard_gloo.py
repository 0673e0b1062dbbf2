"""Multi-process (world_size 2, gloo, CPU) tests of the query partitioner and result gather.

The per-rank compute here is a stand-in (the CPU oracle, which the tests may use); what is
under test is the host logic of paper_2605_18566_b200.shard: balanced contiguous partitions,
global-query-id bases, gathers along the right axes, and the residual all-reduce. Because
results depend only on global query ids, the gathered slice must be bit-identical to a single
unsharded solve.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_18566_b200 import shard
from paper_2605_18566_b200 import inputs as I


def test_partition_properties():
    for M in (0, 1, 7, 10201, 524288):
        for world in (1, 2, 3, 8):
            ranges = [shard.partition(M, world, r) for r in range(world)]
            assert sum(c for _, c in ranges) == M
            assert ranges[0][0] == 0
            for (s0, c0), (s1, _) in zip(ranges, ranges[1:]):
                assert s1 == s0 + c0
            cs = [c for _, c in ranges]
            assert max(cs) - min(cs) <= 1
    with pytest.raises(ValueError):
        shard.partition(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O

        p = I.C2.with_(N=300, K=2, Kp=2)
        P = O.Problem.from_preset(p)
        x = I.queries(p)[::211]                      # 49 queries: ragged over 2 ranks

        def solve(xl, base):
            r = O.solve_slice(P, xl, qid_base=base)
            return {k: torch.from_numpy(np.asarray(v)) for k, v in r.items() if k != "status"}

        full, (start, count) = shard.solve_sharded(solve, x)
        eps = shard.residuals_sharded(
            np.asarray(solve(x[start:start + count], start)["vhist"], dtype=np.float32),
            np.asarray(solve(x[start:start + count], start)["g0"], dtype=np.float32))
        if rank == 0:
            q.put(({k: v.numpy() for k, v in full.items()}, eps))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_is_bit_identical(oracle_mod):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got, eps = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    O = oracle_mod
    p = I.C2.with_(N=300, K=2, Kp=2)
    P = O.Problem.from_preset(p)
    x = I.queries(p)[::211]
    ref = O.solve_slice(P, x)
    for k in ("v", "dv", "c", "tube", "vhist", "chist", "g0"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    part = O.residual_partials(ref["vhist"].astype(np.float32).astype(np.float64),
                               ref["g0"].astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(eps, np.sqrt(part[..., 0] / part[..., 1]), rtol=1e-10)


def _allreduce_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_18566_b200.picard import torch_allreduce

        part = np.array([[1.0 + rank, 10.0 * (rank + 1), 0.5 * rank],
                         [2.0, 3.0, 7.0 - rank]], dtype=np.float64)
        out = torch_allreduce()(part)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_picard_partials_allreduce():
    """Algorithm 1's slice-wide stopping test across ranks: sums of (num, den), max of sup-norm."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allreduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    np.testing.assert_array_equal(out, [[3.0, 30.0, 0.5], [4.0, 6.0, 7.0]])
