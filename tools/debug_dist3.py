#!/usr/bin/env python3
"""Debug the lookahead path: world 1 and world 2 (gloo, one GPU) on the wide_p23
case with lookahead on, window off; repeated; prints mismatching rows vs oracle."""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1112_5717_b200 import dist as D  # noqa: E402

A = O.port_random_matrix(700, 1300, 22, 8388593)
P = 8388593
REF = A.copy()
O.port_cup(REF, P)


def run(world, rank, la=True, win=0, sync_each=False):
    tiles = D.ColumnTiles(1300, world, 128)
    full = torch.from_numpy(A.view(np.int32).copy()).cuda()
    x = D.scatter_columns(full, tiles, rank)
    res = D.dist_cup(x, 700, 1300, P, tiles, block=256, superblock=512, lookahead=la, window=win)
    body = D.gather_columns(x, 700, tiles).cpu().numpy().view(np.uint32)
    bad = np.argwhere(body != REF)
    rows = sorted(set(bad[:, 0].tolist())) if len(bad) else []
    return len(bad), rows[:3], rows[-3:] if rows else []


def worker(rank, world, port, q, la, win):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = [run(world, rank, la, win) for _ in range(3)]
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    print("world1 la win0", [run(1, 0, True, 0) for _ in range(3)], flush=True)
    print("world1 la win512", [run(1, 0, True, 512) for _ in range(3)], flush=True)
    for la, win in ((True, 0), (True, None), (False, 0)):
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, port, q, la, win)) for r in range(2)]
        for pr in ps:
            pr.start()
        print("world2 lookahead", la, "window", win, q.get(timeout=300), flush=True)
        for pr in ps:
            pr.join()
