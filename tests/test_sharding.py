"""Host logic of the multi-GPU paths, on CPU: the config-2/4 recipes, the batch
sharding (contiguous slices, no collective on the data path), and a
world_size-2 gloo run of the sharded batch whose gathered results must equal
the single-process ones.  (The per-shard factorization here is the CPU oracle
standing in for the GPU; the GPU path is covered by tests/test_gpu_*.)"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_1112_5717_b200 import workloads as WL
from tests.helpers import c2_style, c4_batch, matmul_mod


def test_splitmix_matches_reference_stream():
    assert WL.splitmix64(0, 3) == [int(x) for x in O.splitmix64(0, 3)]
    assert WL.splitmix64(12345, 50) == [int(x) for x in O.splitmix64(12345, 50)]


@pytest.mark.parametrize("n", [0, 1, 7, 100, 4096])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(n, world):
    spans = [WL.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_c4_recipe_matches_test_generator():
    ranks, ls, rs = WL.c4_recipe(16)
    _, ref_ranks = c4_batch(4)
    assert ranks[:4] == ref_ranks
    assert all(128 <= r <= 256 for r in ranks)


def test_c2_shuffle_matches_test_generator():
    m, n, inner, seed, p = 60, 90, 20, 7, 65521
    L = O.port_random_matrix(m, inner, seed, p)
    R = O.port_random_matrix(inner, n, seed + 1, p)
    A = matmul_mod(L, R, p)
    A[2::3, :] = 0
    s = WL.c2_row_shuffle(m, seed + 2)
    assert np.array_equal(A[s, :], c2_style(m, n, inner, seed, p))


def _c4_small(t, seed=4, p=8388593):
    ranks, ls, rs = WL.c4_recipe(t + 1, seed)
    return matmul_mod(O.port_random_matrix(256, ranks[t], ls[t], p),
                      O.port_random_matrix(ranks[t], 256, rs[t], p), p)


def _worker(rank, world, port, total, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = WL.shard_range(total, rank, world)
    mine = []
    for t in range(lo, hi):
        r = O.port_cup(_c4_small(t), 8388593)
        mine.append((t, r.rank, r.rrp.tolist()))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out_q.put(sorted(x for part in gathered for x in part))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_batch_equals_single_process():
    import torch.multiprocessing as mp
    total, world = 6, 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    single = []
    for t in range(total):
        r = O.port_cup(_c4_small(t), 8388593)
        single.append((t, r.rank, r.rrp.tolist()))
    assert got == single
    assert [g[1] for g in got] == WL.c4_recipe(total)[0]
