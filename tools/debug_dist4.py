#!/usr/bin/env python3
"""world-2 gloo dist_cup (wide_p23, window mode, lookahead) repeated N times
under RL_DIST_DEBUG_SYNC variants; counts mismatching runs vs the oracle."""
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


def worker(rank, world, port, q, reps, dbg):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RL_DIST_DEBUG_SYNC"] = dbg
    if "nopdl" in dbg:
        os.environ["RL_NO_PDL"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bad = []
    for _ in range(reps):
        tiles = D.ColumnTiles(1300, world, 128)
        full = torch.from_numpy(A.view(np.int32).copy()).cuda()
        x = D.scatter_columns(full, tiles, rank)
        D.dist_cup(x, 700, 1300, P, tiles, block=256, superblock=512)
        body = D.gather_columns(x, 700, tiles).cpu().numpy().view(np.uint32)
        nb = int((body != REF).sum())
        if nb:
            rows = np.nonzero((body != REF).any(1))[0]
            bad.append((nb, int(rows[0]), int(rows[-1])))
        else:
            bad.append(0)
    if rank == 0:
        q.put(bad)
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    variants = sys.argv[2].split(";") if len(sys.argv) > 2 else ["", "pre", "evall", "nopdl"]
    for dbg in variants:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        ps = [ctx.Process(target=worker, args=(r, 2, port, q, reps, dbg)) for r in range(2)]
        for pr in ps:
            pr.start()
        print("sync", repr(dbg), q.get(timeout=600), flush=True)
        for pr in ps:
            pr.join()
