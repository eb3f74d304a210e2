"""Multi-process sharding logic on CPU (gloo, world_size 2), no GPU.

The product kernels need CUDA; here the per-rank "solve" is the CPU oracle
(test infrastructure) so the host-side partition + gather path of
paper_2604_10377_b200.shard is exercised end to end: every rank solves its
contiguous pair range, rank 0 gathers, and the result is bitwise identical to
the single-process solve (SURVEY §8(e) determinism requirement).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10377_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_chunks_cover_exactly():
    for n in (1, 2, 7, 64, 65):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard.chunk(n, world, r) for r in range(world)]
            covered = [i for rg in ranges for i in range(rg.lo, rg.hi)]
            assert covered == list(range(n))
    assert shard.system_range(3, 200, 8, 7).hi == 600


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    b, k = 5, 12
    probs = [oracle.random_problem(k, 2 * k, 300 + q, kind=1) for q in range(b)]
    G = np.stack([p[0] for p in probs]).astype(np.float32)
    R = np.stack([p[1] for p in probs]).astype(np.float32)
    M = np.stack([p[2] for p in probs]).astype(np.float32)
    rg = shard.pair_range(b, world, rank)
    local = oracle.solve(G[rg.lo:rg.hi], R[rg.lo:rg.hi], M[rg.lo:rg.hi], 100.0, dtype=np.float32).maps \
        if rg.size else np.zeros((0, k, k), np.float32)
    full = shard.gather_maps(torch.from_numpy(np.ascontiguousarray(local)), b, k, world, rank)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_and_gather_bitwise(tmp_path, world):
    import oracle
    out = tmp_path / "c.npy"
    mp.spawn(_worker, args=(world, _free_port(), str(out)), nprocs=world, join=True)
    got = np.load(out)
    b, k = 5, 12
    probs = [oracle.random_problem(k, 2 * k, 300 + q, kind=1) for q in range(b)]
    G = np.stack([p[0] for p in probs]).astype(np.float32)
    R = np.stack([p[1] for p in probs]).astype(np.float32)
    M = np.stack([p[2] for p in probs]).astype(np.float32)
    ref = oracle.solve(G, R, M, 100.0, dtype=np.float32).maps
    assert got.shape == (b, k, k)
    assert np.array_equal(got, ref)


def _gather_worker(rank, world, port, out_path, b, k):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = shard.MapGather(b, k, world, rank, "cpu")
    rg = g.mine
    # each rank writes its pairs' "maps" (pair index encoded) into its slot
    for j, q in enumerate(range(rg.lo, rg.hi)):
        g.local[j].fill_(float(q))
    for _ in range(3):  # reusable across timed steps
        g()
    if rank == 0:
        np.save(out_path, g.out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,b", [(2, 5), (2, 64), (3, 7)])
def test_map_gather_preallocated(tmp_path, world, b):
    # bench.py's timed gather: uneven contiguous ranges, padded slots, global order
    out = tmp_path / "g.npy"
    k = 3
    mp.spawn(_gather_worker, args=(world, _free_port(), str(out), b, k), nprocs=world, join=True)
    got = np.load(out)
    assert got.shape == (b, k, k)
    assert np.array_equal(got[:, 0, 0], np.arange(b, dtype=np.float32))
    assert np.all(got == got[:, :1, :1])


def _gpu_worker(rank, world, port, out_path):
    # a real CUDA solve per rank (both ranks on cuda:0, independent kernels — no
    # kernel waits on another rank), gathered with gloo on host tensors
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2604_10377_b200 as fm
    b, k = 6, 40
    probs = [oracle.random_problem(k, 2 * k, 500 + q, kind=1) for q in range(b)]
    G = np.stack([p[0] for p in probs]).astype(np.float32)
    R = np.stack([p[1] for p in probs]).astype(np.float32)
    M = np.stack([p[2] for p in probs]).astype(np.float32)
    g = shard.MapGather(b, k, world, rank, "cpu")
    rg = g.mine
    local = fm.solve_host(G[rg.lo:rg.hi], R[rg.lo:rg.hi], M[rg.lo:rg.hi], 100.0).maps
    g.local.copy_(torch.from_numpy(local))
    g()
    if rank == 0:
        np.save(out_path, g.out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_bitwise_vs_single_process(tmp_path):
    import oracle
    import paper_2604_10377_b200 as fm
    out = tmp_path / "c.npy"
    mp.spawn(_gpu_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    got = np.load(out)
    b, k = 6, 40
    probs = [oracle.random_problem(k, 2 * k, 500 + q, kind=1) for q in range(b)]
    G = np.stack([p[0] for p in probs]).astype(np.float32)
    R = np.stack([p[1] for p in probs]).astype(np.float32)
    M = np.stack([p[2] for p in probs]).astype(np.float32)
    single = fm.solve_host(G, R, M, 100.0).maps
    assert np.array_equal(got, single)
