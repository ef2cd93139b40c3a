#!/usr/bin/env python3
"""Debug: world-2 gloo dist_cup on one GPU for one case, compared with the oracle
port; variants with lookahead/window toggled.  Usage: debug_dist2.py"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1112_5717_b200 import dist as D  # noqa: E402


def worker(rank, world, port, q, la, win):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, p = O.port_random_matrix(700, 1300, 22, 8388593), 8388593
    tiles = D.ColumnTiles(1300, world, 128)
    full = torch.from_numpy(a.view(np.int32).copy()).cuda()
    x = D.scatter_columns(full, tiles, rank)
    res = D.dist_cup(x, 700, 1300, p, tiles, block=256, superblock=512, lookahead=la,
                     window=None if win else 0)
    body = D.gather_columns(x, 700, tiles).cpu().numpy().view(np.uint32)
    if rank == 0:
        o = a.copy()
        r = O.port_cup(o, p)
        bad = np.argwhere(body != o)
        q.put((res.rank, r.rank, len(bad), bad[:10].tolist(),
               sorted(set(bad[:, 0].tolist()))[:20] if len(bad) else []))
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    for la in (True, False):
        for win in (True, False):
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            ctx = mp.get_context("spawn")
            q = ctx.Queue()
            ps = [ctx.Process(target=worker, args=(r, 2, port, q, la, win)) for r in range(2)]
            for pr in ps:
                pr.start()
            print("lookahead", la, "window", win, q.get(timeout=300), flush=True)
            for pr in ps:
                pr.join()
