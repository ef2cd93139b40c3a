"""GPU parity of the distributed single-matrix CUP (paper_1112_5717_b200/dist.py)
with the device compute (DeviceOps: rl_cup_u32_dev / rl_trsm_u32_dev /
rl_mm_u32_dev).  Only one GPU is available here: world 1 in-process, and
world 2 over gloo with both ranks on cuda:0 (independent kernels, host-side
collectives -- no kernel waits on another rank).  Bit-exact against the
single-GPU engine and the oracle."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
import paper_1112_5717_b200 as G
from paper_1112_5717_b200 import dist as D
from tests.helpers import c2_style

pytestmark = pytest.mark.gpu


def _cases():
    out = [
        ("full_1536", O.port_random_matrix(1536, 1536, 21, 65521), 65521, 128, 512),
        ("wide_p23", O.port_random_matrix(700, 1300, 22, 8388593), 8388593, 128, 256),
        ("tall_early_return", O.port_random_matrix(1200, 333, 23, 65521), 65521, 64, 256),
        ("c2_style", c2_style(1024, 2048, 512, 24, 65521), 65521, 256, 256),
    ]
    rnd = np.random.default_rng(25)
    a = rnd.integers(0, 2, (600, 520)).astype(np.uint32)
    a[:, :40] = 0
    out.append(("gf2_zero_cols", a, 2, 64, 128))
    out.append(("p31", O.port_random_matrix(520, 600, 26, 2147483647), 2147483647, 64, 192))
    return out


def _run(a, p, tile, block, world, rank, sb=None):
    tiles = D.ColumnTiles(a.shape[1], world, tile)
    full = torch.from_numpy(a.view(np.int32).copy()).cuda()
    x = D.scatter_columns(full, tiles, rank)
    res = D.dist_cup(x, a.shape[0], a.shape[1], p, tiles, block=block,
                      superblock=sb or 2 * block)
    body = D.gather_columns(x, a.shape[0], tiles).cpu().numpy().view(np.uint32)
    return res, body


def _check(name, a, p, res, body):
    ref = a.copy()
    g = G.cup(ref, p)
    assert res.rank == g.rank, name
    assert np.array_equal(res.row_profile, g.row_profile), name
    assert np.array_equal(res.col_perm, g.col_perm), name
    assert np.array_equal(body, ref), name
    if a.size <= 400_000:
        o = a.copy()
        orr = O.port_cup(o, p)
        assert res.rank == orr.rank and np.array_equal(body, o), name


@pytest.mark.parametrize("name,a,p,tile,block", _cases(), ids=[c[0] for c in _cases()])
def test_dist_world1_equals_engine(name, a, p, tile, block):
    torch.cuda.set_device(0)
    res, body = _run(a, p, tile, block, 1, 0)
    _check(name, a, p, res, body)


def test_random_matrix_local_columns():
    torch.cuda.set_device(0)
    m, n, p = 777, 1000, 65521
    full = torch.empty((m, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(full, m, n, 5, p)
    tiles = D.ColumnTiles(n, 3, 64)
    for g in range(3):
        x = D.random_matrix_local(m, n, 5, p, tiles, g, "cuda", chunk_rows=100)
        assert torch.equal(x, D.scatter_columns(full, tiles, g))


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        for name, a, p, tile, block in _cases():
            res, body = _run(a, p, tile, block, world, rank)
            if rank == 0:
                _check(name, a, p, res, body)
                out.append(name)
        if rank == 0:
            q.put(out)
    except Exception as e:
        if rank == 0:
            q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def test_dist_world2_gloo_on_one_gpu():
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=900)
    for pr in procs:
        pr.join(timeout=120)
    assert got == [c[0] for c in _cases()], got


@pytest.mark.parametrize("n,p,block,sb", [(8192, 65521, 1024, 4096), (6000, 8388593, 512, 2048)])
def test_dist_world1_large_equals_engine(n, p, block, sb):
    """Full-size-class sizes through the driver (super-blocks, lookahead, zero-copy
    views): every body entry equals the single-GPU engine's on the device."""
    torch.cuda.set_device(0)
    src = torch.empty((n, n), dtype=torch.int32, device="cuda")
    G.random_matrix_dev(src, n, n, 31, p)
    eng = src.clone()
    g = G.cup_dev(eng, n, n, p)
    tiles = D.ColumnTiles(n, 1, 1024)
    x = src.clone()
    res = D.dist_cup(x, n, n, p, tiles, block=block, superblock=sb)
    assert res.rank == g.rank
    assert np.array_equal(res.row_profile, g.row_profile)
    assert np.array_equal(res.col_perm, g.col_perm)
    assert torch.equal(x, eng)


def test_data_plane_kernels_match_tensor_ops():
    """csrc/dist.cu (pack / unpack / select / U-row shift) against the tensor-op
    formulation the CPU tests use, on strided views and both wire formats."""
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randint(0, 65521, (300, 700), dtype=torch.int32, device="cuda", generator=g)
    v = x[17:217, 33:433]
    for wire16, dt in ((True, torch.float16), (False, torch.int32)):
        w = torch.empty(v.shape, dtype=dt, device="cuda")
        G.dist_pack_dev(v, w, wire16)
        want = (v - 32768).to(torch.int16).view(torch.float16) if wire16 else v.contiguous()
        assert torch.equal(w.view(torch.int16) if wire16 else w, want.view(torch.int16) if wire16 else want)
        cm = torch.randperm(600, device="cuda", generator=g)[:400].to(torch.int64) + 50
        out = torch.zeros((200, 700), dtype=torch.int32, device="cuda")
        G.dist_unpack_dev(w, out, wire16, cm, 50)
        ref = torch.zeros_like(out)
        ref.index_copy_(1, cm - 50, v.contiguous())
        assert torch.equal(out, ref)
    cm = torch.randperm(700, device="cuda", generator=g)[:256].to(torch.int64) + 9
    dst = x[40:140, 100:356]
    ref = x[40:140].index_select(1, cm - 9)  # computed before dst is overwritten
    src = x[40:140].clone()
    G.dist_select_cols_dev(src, cm, dst, 9)
    assert torch.equal(x[40:140, 100:356], ref)
    # U-row shift with overlapping source / target rows (i0 - r < rt)
    for r, i0, rt in ((10, 30, 50), (5, 300 - 64, 64), (0, 1, 120)):
        y = torch.randint(0, 65521, (300, 500), dtype=torch.int32, device="cuda", generator=g)
        gp = torch.sort(torch.randperm(2000, device="cuda", generator=g)[:420]).values.to(torch.int64)
        ls = 80
        want = y.clone()
        src_ = want[i0:i0 + rt, ls:]
        j = torch.arange(rt, device="cuda", dtype=torch.int64)
        mask = gp[None, :] > (r + j)[:, None]
        moved = torch.where(mask, src_, torch.zeros_like(src_))
        src_.masked_fill_(mask, 0)
        d = want[r:r + rt, ls:]
        d.copy_(torch.where(mask, moved, d))
        G.dist_shift_u_rows_dev(y, ls, r, i0, rt, gp)
        assert torch.equal(y, want), (r, i0, rt)
