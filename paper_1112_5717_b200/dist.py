"""Multi-GPU CUP of ONE large matrix (config 5): 1D block-cyclic column tiles.

SURVEY.md 8(e): the columns of the m x n matrix are cut into tiles of ``tile``
columns; rank g owns the tiles t = g (mod world).  Rows are not split.  Each
rank keeps its tiles as one local row-major m x n_g matrix (columns in
increasing global position, so "global position >= c" is a suffix of the local
columns).  The factorization walks row blocks R = rows [i0, i0 + b):

1. every rank receives the active part of R (columns [r, n) in the current
   column order, r = rank so far) -- one NCCL broadcast per owning rank;
2. every rank factors R redundantly with the single-GPU CUP engine
   (``rl_cup_u32_dev``): rank r_t, row profile, the block's column permutation
   sigma_t, and R's packed [C\\U] block (the b x (n - r) CUP is the serial part);
3. sigma_t is applied to the columns of the other rows (the transpositions of
   the reference's ``perm_apply_cols``, factor.cpp:49-50/perm.cpp:115-125);
   a column whose source lives on another rank travels by an all-reduce of a
   zero-padded column buffer (rare: sigma_t = id for generic inputs);
4. the U rows of R move to global rows [r, r + r_t) on every rank's columns
   (the reference's U-row shift, factor.cpp:62-70, applied per step);
5. the rows below R receive their C columns G = B1 * U11^{-1} (``trsm``,
   factor.cpp:45-46), B1 broadcast by the owners of columns [r, r + r_t);
6. every rank updates its own columns right of the pivots:
   B2 <- B2 - G * U12 (the Schur complement, ``mm``, factor.cpp:51-53) -- the
   tensor-core GEMM, embarrassingly parallel over the column tiles.

The result is bit-exact with ``ranklab::cup`` (factor.cpp:30-85): with the
reference's pivot rule (first nonzero of each row in the current column order)
the packed [C\\U], the row profile and sigma are unique, and the row-block
sweep is the same elimination in a different grouping (SURVEY.md 8(c),
"iterative formulation").  The data path's collectives are the per-owner
broadcasts of R and B1 and, for non-trivial sigma_t, the column exchange.

Compute goes through ``ops`` (default :class:`DeviceOps`, the C ABI of
libranklab_gpu.so on the rank's GPU); communication through ``torch.distributed``
(NCCL on B200; the CPU tests drive the same code over gloo with the oracle as
``ops``).  Storage is int32 (bit pattern of the canonical uint32 values, p < 2^31).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["ColumnTiles", "DeviceOps", "DistCupResult", "dist_cup", "scatter_columns",
           "gather_columns", "random_matrix_local"]


class ColumnTiles:
    """1D block-cyclic map of n columns over ``world`` ranks, tiles of ``tile``."""

    def __init__(self, n: int, world: int, tile: int):
        assert n >= 0 and world >= 1 and tile >= 1
        self.n, self.world, self.tile = n, world, tile
        cols = np.arange(n, dtype=np.int64)
        self.owner = (cols // tile) % world
        self.gpos = [cols[self.owner == g] for g in range(world)]
        self.local = np.zeros(n, np.int64)
        for g in range(world):
            self.local[self.gpos[g]] = np.arange(self.gpos[g].size)

    def width(self, g: int) -> int:
        return int(self.gpos[g].size)

    def lsuf(self, g: int, c: int) -> int:
        """First local column of rank g whose global position is >= c."""
        return int(np.searchsorted(self.gpos[g], c, side="left"))


@dataclass
class DistCupResult:
    rank: int
    row_profile: np.ndarray
    col_perm: np.ndarray
    steps: int


class DeviceOps:
    """The compute of one rank: the C ABI of libranklab_gpu.so on torch CUDA
    views (int32 storage, unit column stride, ld = stride(0)).  No fallback."""

    def __init__(self, p: int):
        from . import cup_dev, mm_dev, trsm_dev
        self.p = int(p)
        self._cup, self._mm, self._trsm = cup_dev, mm_dev, trsm_dev

    @staticmethod
    def _stream():
        return torch.cuda.current_stream()

    def cup(self, t: torch.Tensor):
        m, n = t.shape
        res = self._cup(t, m, n, self.p, lda=t.stride(0), stream=self._stream())
        return res.rank, res.row_profile.astype(np.int64), res.col_perm.astype(np.int64)

    def trsm_right_upper_unit(self, u: torch.Tensor, b: torch.Tensor) -> None:
        """b <- b * U^{-1}, U unit upper (only the strict upper part of u is read)."""
        m, k = b.shape
        self._trsm(1, 0, 1, u, b, m, k, self.p, ldt=u.stride(0), ldb=b.stride(0),
                   stream=self._stream())

    def trsm_left_lower_nonunit(self, t: torch.Tensor, b: torch.Tensor) -> None:
        """b <- T^{-1} b, T lower triangular with a nonzero diagonal."""
        m, n = b.shape
        self._trsm(0, 1, 0, t, b, m, n, self.p, ldt=t.stride(0), ldb=b.stride(0),
                   stream=self._stream())

    def mm_sub(self, a: torch.Tensor, b: torch.Tensor, c: torch.Tensor, max_ctas: int = 0) -> None:
        """c <- c - a * b (mod p); max_ctas > 0 bounds the GEMM grid."""
        m, k = a.shape
        n = b.shape[1]
        if m == 0 or n == 0:
            return
        self._mm(a, b, c, m, k, n, self.p - 1, 1, self.p, lda=a.stride(0), ldb=b.stride(0),
                 ldc=c.stride(0), stream=self._stream(), max_ctas=max_ctas)


def _roundup(a: int, q: int) -> int:
    return -(-a // q) * q


def _comm():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_rank(), dist.get_world_size()
    return None, 0, 1


class _Engine:
    def __init__(self, x: torch.Tensor, m: int, n: int, tiles: ColumnTiles, ops, rank: int,
                 dist, p: int = 0):
        self.x, self.m, self.n, self.tiles, self.ops = x, m, n, tiles, ops
        self.wire = torch.float16 if 0 < p <= 65536 else x.dtype
        self.wire16 = self.wire == torch.float16
        self.rank, self.dist, self.world = rank, dist, tiles.world
        dev = x.device
        self.gpos_t = [torch.as_tensor(gp, dtype=torch.int64, device=dev) for gp in tiles.gpos]
        self.mine = tiles.gpos[rank]
        # on the GPU the data plane around the collectives is one hand-written
        # kernel per piece (csrc/dist.cu); the CPU tests (gloo) use tensor ops
        # point-to-point sends where the backend has them for these tensors
        self.p2p = dist is not None and (not x.is_cuda or dist.get_backend() == "nccl")
        self.G = None
        if x.is_cuda:
            import sys
            self.G = sys.modules[__package__]  # the package's C-ABI bindings

    def _place(self, piece: torch.Tensor, out: torch.Tensor, g: int, la: int, lb: int, c0: int) -> None:
        """out[:, gpos_g[la:lb] - c0] <- the received wire piece."""
        if self.G is not None:
            self.G.dist_unpack_dev(piece, out, self.wire16, self.gpos_t[g][la:lb], c0)
        else:
            out.index_copy_(1, self.gpos_t[g][la:lb] - c0, self._unpack(piece))

    def gather_cols_to(self, dst: int, ra: int, rb: int, c0: int, c1: int, out) -> None:
        """Rows [ra, rb) x global columns [c0, c1) onto rank ``dst`` only (into
        ``out``, global order): every other owner sends its piece point to point."""
        if rb == ra or c1 == c0:
            return
        for g in range(self.world):
            la, lb = self.tiles.lsuf(g, c0), self.tiles.lsuf(g, c1)
            if lb == la:
                continue
            if g == dst:
                if self.rank == dst:
                    out.index_copy_(1, self.gpos_t[g][la:lb] - c0, self.x[ra:rb, la:lb])
                continue
            if self.p2p:
                if self.rank == g:
                    self.dist.send(self._pack(self.x[ra:rb, la:lb]), dst=dst)
                elif self.rank == dst:
                    piece = torch.empty((rb - ra, lb - la), dtype=self.wire, device=self.x.device)
                    self.dist.recv(piece, src=g)
                    self._place(piece, out, g, la, lb, c0)
            else:  # gloo has no point-to-point for CUDA tensors: a broadcast, kept by dst only
                if self.rank == g:
                    piece = self._pack(self.x[ra:rb, la:lb])
                else:
                    piece = torch.empty((rb - ra, lb - la), dtype=self.wire, device=self.x.device)
                self.dist.broadcast(piece, src=g)
                if self.rank == dst:
                    self._place(piece, out, g, la, lb, c0)

    def gather_cols(self, ra: int, rb: int, c0: int, c1: int, out=None) -> torch.Tensor:
        """Rows [ra, rb) x global columns [c0, c1) in global order, on every rank
        (one broadcast from each rank owning a piece), into ``out`` if given.
        With one rank and no ``out`` this is a view of the local matrix (the
        callers solve/update it in place, ld = the local width)."""
        if out is None:
            if self.world == 1:
                return self.x[ra:rb, c0:c1]
            out = torch.empty((rb - ra, c1 - c0), dtype=self.x.dtype, device=self.x.device)
        if rb == ra or c1 == c0:
            return out
        for g in range(self.world):
            la, lb = self.tiles.lsuf(g, c0), self.tiles.lsuf(g, c1)
            if lb == la:
                continue
            if self.world == 1:
                out.copy_(self.x[ra:rb, la:lb])
                continue
            if g == self.rank:
                piece = self._pack(self.x[ra:rb, la:lb])
            else:
                piece = torch.empty((rb - ra, lb - la), dtype=self.wire, device=self.x.device)
            self.dist.broadcast(piece, src=g)
            self._place(piece, out, g, la, lb, c0)
        return out

    # p <= 2^16: field elements cross the links as 16-bit words (half the
    # NVLink volume of the broadcasts and gathers): x - 2^15 fits int16 exactly,
    # carried bit for bit in a 16-bit float tensor (collectives only move bytes)
    def _pack(self, t: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if self.G is not None:
            if out is None:
                out = torch.empty(t.shape, dtype=self.wire, device=t.device)
            self.G.dist_pack_dev(t, out, self.wire16)
            return out
        if self.wire == torch.float16:
            w = (t - 32768).to(torch.int16).view(torch.float16)
        else:
            w = t.contiguous()
        if out is None:
            return w
        out.copy_(w)
        return out

    def _unpack(self, t: torch.Tensor) -> torch.Tensor:
        if self.wire == torch.float16:
            return t.view(torch.int16).to(torch.int32) + 32768
        return t

    def bcast_block(self, R: torch.Tensor, src: int) -> None:
        """R (a contiguous block, identical layout on every rank) from rank src."""
        if R.numel() == 0:
            return
        w = self._pack(R) if self.rank == src else torch.empty(R.shape, dtype=self.wire, device=R.device)
        self.dist.broadcast(w, src=src)
        if self.rank != src:
            if self.G is not None:
                self.G.dist_unpack_dev(w, R, self.wire16)
            else:
                R.copy_(self._unpack(w))

    def put_cols(self, full: torch.Tensor, ra: int, c0: int) -> None:
        """Write this rank's columns of ``full`` (rows [ra, ..), global columns
        [c0, c0 + full.shape[1])) back into the local matrix."""
        rows, w = full.shape
        la, lb = self.tiles.lsuf(self.rank, c0), self.tiles.lsuf(self.rank, c0 + w)
        if lb == la or rows == 0:
            return
        if self.world == 1:
            dst = self.x[ra:ra + rows, la:lb]
            if dst.data_ptr() != full.data_ptr() or dst.stride() != full.stride():
                dst.copy_(full)
        elif self.G is not None:
            self.G.dist_select_cols_dev(full, self.gpos_t[self.rank][la:lb], self.x[ra:ra + rows, la:lb], c0)
        else:
            self.x[ra:ra + rows, la:lb].copy_(
                full.index_select(1, self.gpos_t[self.rank][la:lb] - c0))

    def solve_rows(self, ra: int, rb: int, c0: int, c1: int, U: torch.Tensor) -> torch.Tensor:
        """G = B1 * U^{-1} for B1 = rows [ra, rb) x global columns [c0, c1), U unit
        upper (c1 - c0 square); every rank solves one slice of the rows and the
        slices are all-gathered, so G ends up complete on every rank."""
        rows, k = rb - ra, c1 - c0
        if self.world == 1:
            B1 = self.gather_cols(ra, rb, c0, c1)
            self.ops.trsm_right_upper_unit(U, B1)
            return B1
        B1 = self.gather_cols(ra, rb, c0, c1)
        sl = _roundup(rows, self.world) // self.world
        lo = min(rows, self.rank * sl)
        hi = min(rows, lo + sl)
        mine = torch.zeros((sl, k), dtype=self.wire, device=self.x.device)
        if hi > lo:
            part = B1[lo:hi]
            self.ops.trsm_right_upper_unit(U, part)
            self._pack(part, mine[:hi - lo])
        out = torch.empty((sl * self.world, k), dtype=self.wire, device=self.x.device)
        self.dist.all_gather(list(out.split(sl)), mine)
        if self.G is not None:
            G = torch.empty((rows, k), dtype=self.x.dtype, device=self.x.device)
            self.G.dist_unpack_dev(out[:rows], G, self.wire16)
            return G
        return self._unpack(out[:rows]).contiguous()

    def permute_cols(self, r: int, sig: np.ndarray, row_ranges) -> None:
        """New column r + i = old column r + sig[i] on the given row ranges."""
        moved = np.nonzero(sig != np.arange(sig.size))[0]
        if moved.size == 0:
            return
        dst = r + moved
        src = r + sig[moved]
        t = self.tiles
        for ra, rb in row_ranges:
            if rb <= ra:
                continue
            if self.world == 1:
                li = torch.as_tensor(t.local[src], device=self.x.device)
                lo = torch.as_tensor(t.local[dst], device=self.x.device)
                self.x[ra:rb].index_copy_(1, lo, self.x[ra:rb].index_select(1, li))
                continue
            buf = torch.zeros((rb - ra, moved.size), dtype=self.x.dtype, device=self.x.device)
            own_src = np.nonzero(t.owner[src] == self.rank)[0]
            if own_src.size:
                li = torch.as_tensor(t.local[src[own_src]], device=self.x.device)
                buf.index_copy_(1, torch.as_tensor(own_src, device=self.x.device),
                                self.x[ra:rb].index_select(1, li))
            self.dist.all_reduce(buf)  # one nonzero contributor per column: exact
            own_dst = np.nonzero(t.owner[dst] == self.rank)[0]
            if own_dst.size:
                lo = torch.as_tensor(t.local[dst[own_dst]], device=self.x.device)
                self.x[ra:rb].index_copy_(
                    1, lo, buf.index_select(1, torch.as_tensor(own_dst, device=self.x.device)))

    def shift_u_rows(self, r: int, i0: int, rt: int) -> None:
        """U row j of the block (row i0 + j) moves to row r + j on the columns at
        global position > r + j; the vacated entries become 0 (factor.cpp:62-70)."""
        if i0 == r or rt == 0:
            return
        ls = self.tiles.lsuf(self.rank, r + 1)
        if ls == self.x.shape[1]:
            return
        gp = self.gpos_t[self.rank][ls:]
        if self.G is not None:
            self.G.dist_shift_u_rows_dev(self.x, ls, r, i0, rt, gp)
            return
        j = torch.arange(rt, device=self.x.device, dtype=torch.int64)
        mask = gp[None, :] > (r + j)[:, None]
        src = self.x[i0:i0 + rt, ls:]
        moved = torch.where(mask, src, torch.zeros_like(src))
        src.masked_fill_(mask, 0)
        dst = self.x[r:r + rt, ls:]
        dst.copy_(torch.where(mask, moved, dst))


def dist_cup(x: torch.Tensor, m: int, n: int, p: int, tiles: ColumnTiles, block: int = 1024,
             superblock: int = 4096, ops=None, lookahead: bool = True,
             free_sms: int = 16, window: int | None = None) -> DistCupResult:
    """In-place distributed CUP; ``x`` is this rank's m x tiles.width(rank)
    local matrix (int32, row-major, contiguous).  Collective: every rank of the
    default process group calls it with the same (m, n, p, tiles, block,
    superblock).

    Two levels, like the top of the reference's row-halving recursion
    (factor.cpp:35-53): row blocks of ``block`` rows are factored one after the
    other inside a super-block of ``superblock`` rows (their TRSM and Schur
    updates stop at the super-block's last row); the rows below a super-block
    then receive one TRSM against the super-block's U11 and ONE Schur update
    with K = the super-block's rank (large-K tensor-core GEMMs instead of K =
    block; the G rows are solved in slices, one per rank, and all-gathered).

    Lookahead (CUDA): every Schur update first updates the rows of the NEXT row
    block, then the rest with the GEMM grid bounded to leave ``free_sms`` SMs;
    the next block's gather and factorization run on a second (high-priority)
    stream beside that GEMM -- the serial row-block chain overlaps the
    embarrassingly parallel trailing update.

    Window mode (default with more than one rank): a row block is factored on
    its first ``window`` (default 2 x block) active columns only (every rank, redundantly -- the serial leaf
    chain then runs on a narrow matrix); each rank then forms the block's U rows
    on its OWN columns beyond the window, U_b = C_piv^{-1} * R_b[pivot rows]
    (trsm Left/Lower/NonUnit), and checks that the block's non-pivot rows are
    zero there (R_b - C * U_b = 0, one all-reduce).  If some rank finds a
    nonzero (a pivot beyond the window) the block is refactored over its full
    width.  Identical results either way (the CUP of the block is unique).

    Returns the global rank, row profile and sigma (identical on every rank);
    ``x`` holds this rank's columns of the packed [C\\U] (factor.hpp:10-14)."""
    dist, rank, world = _comm()
    assert world == tiles.world and tiles.n == n
    assert x.dim() == 2 and x.shape == (m, tiles.width(rank)) and x.is_contiguous()
    superblock = max(superblock, block)
    # one rank has nothing redundant to save: full-width blocks (measured faster)
    window = (2 * block if world > 1 else 0) if window is None else window
    if ops is None:
        ops = DeviceOps(p)
    eng = _Engine(x, m, n, tiles, ops, rank, dist, p)
    # The row block is factored in one persistent buffer, its width padded to a
    # few buckets with zero columns (zero columns never hold a pivot and stay
    # in place): the CUP engine caches one plan + CUDA graph per (shape, buffer).
    quantum = _roundup(_roundup(n, 12) // 12, 64)
    rbuf = torch.empty(max(1, min(block, m) * n), dtype=x.dtype, device=x.device)
    wbuf = torch.empty(max(1, min(block, m) * min(n, window)), dtype=x.dtype, device=x.device)
    cuda = x.is_cuda and lookahead
    main = torch.cuda.current_stream(x.device) if cuda else None
    side = torch.cuda.Stream(device=x.device, priority=-1) if cuda else None
    max_ctas = 0
    if cuda:
        max_ctas = max(1, torch.cuda.get_device_properties(x.device).multi_processor_count - free_sms)

    def factor_full(i0, bt, r):
        w = n - r
        wp = min(n, _roundup(w, quantum))
        R = rbuf[:bt * wp].view(bt, wp)
        if wp > w:
            R[:, w:].zero_()
        eng.gather_cols(i0, i0 + bt, r, n, out=R[:, :w])          # (1)
        rt, rrp_t, sig_t = ops.cup(R)                               # (2)
        return R, w, rt, rrp_t, sig_t[:w], None

    def factor_window(i0, bt, r, ww):
        """The block on its first ww columns + this rank's U rows beyond them;
        None when a pivot lies beyond the window (on any rank).  With more than
        one rank only the owner f of column r factors the window (its pieces
        sent to f point to point); f broadcasts the rank, profile, sigma and the
        factored window, so the other ranks' SMs stay on their trailing updates."""
        R = wbuf[:bt * ww].view(bt, ww)
        if world > 1:
            f = int(tiles.owner[r])
            eng.gather_cols_to(f, i0, i0 + bt, r, r + ww, R)
            meta = torch.full((1 + bt + ww,), -1, dtype=torch.int64, device=x.device)
            if rank == f:
                rt, rrp_t, sig_t = ops.cup(R)
                host = np.full(1 + bt + ww, -1, np.int64)
                host[0] = rt
                host[1:1 + rt] = rrp_t[:rt]
                host[1 + bt:] = sig_t[:ww]
                meta.copy_(torch.from_numpy(host))
            dist.broadcast(meta, src=f)
            eng.bcast_block(R, src=f)
            if rank != f:
                host = meta.cpu().numpy()
                rt = int(host[0])
                rrp_t = host[1:1 + bt].copy()
                sig_t = host[1 + bt:].copy()
        else:
            eng.gather_cols(i0, i0 + bt, r, r + ww, out=R)
            rt, rrp_t, sig_t = ops.cup(R)
        ls = tiles.lsuf(rank, r + ww)
        Rb = x[i0:i0 + bt, ls:]
        bad = 0
        Ub = None
        if rt == 0:
            bad = int(bool(torch.any(Rb != 0))) if Rb.numel() else 0
        else:
            piv = torch.as_tensor(rrp_t[:rt], device=x.device)
            Ub = Rb.index_select(0, piv)                            # rt x beyond (copy)
            Cp = torch.tril(R.index_select(0, piv)[:, :rt])         # C at the pivot rows
            if Ub.shape[1]:
                ops.trsm_left_lower_nonunit(Cp, Ub)
            dead = np.setdiff1d(np.arange(bt), rrp_t[:rt])
            if dead.size and Ub.shape[1]:
                dv = torch.as_tensor(dead, device=x.device)
                Cd = R.index_select(0, dv)[:, :rt].contiguous()
                keep = torch.arange(rt, device=x.device)[None, :] <= dv[:, None]
                Cd.masked_fill_(~keep, 0)                           # C(d, k) only for k <= d
                D = Rb.index_select(0, dv)
                ops.mm_sub(Cd, Ub, D)
                bad = int(bool(torch.any(D != 0)))
        if world > 1:
            flag = torch.tensor([bad], dtype=torch.int32, device=x.device)
            dist.all_reduce(flag)
            bad = int(flag.item())
        if bad:
            return None
        sig = np.concatenate([sig_t[:ww], np.arange(ww, n - r, dtype=np.int64)])
        return R, ww, rt, rrp_t, sig, (ls, Ub)

    def factor_block(i0, bt, r):
        w = n - r
        if window and window < w:
            res = factor_window(i0, bt, r, window)
            if res is not None:
                return res
        return factor_full(i0, bt, r)

    def next_block(i_next, r_next, s_end):
        if i_next >= m or r_next >= n:
            return None
        end = s_end if i_next < s_end else min(m, i_next + superblock)
        return i_next, min(block, end - i_next), r_next

    def update(G, ra, rb, ku0, ku1, nb):
        """x[ra:rb, cols >= ku1] -= G * U (U = rows [ku0, ku1)); when the next
        block nb = (i, bt, r) lies in [ra, rb): its rows first, then the rest
        beside the next block's factorization.  Returns the factored block."""
        ls = tiles.lsuf(rank, ku1)
        U = x[ku0:ku1, ls:]
        lo = hi = ra
        if nb is not None and ra <= nb[0] < rb:
            lo, hi = nb[0], min(rb, nb[0] + nb[1])
        if hi > lo:
            ops.mm_sub(G[lo - ra:hi - ra], U, x[lo:hi, ls:])
        if not cuda or hi == lo:
            if lo > ra:
                ops.mm_sub(G[:lo - ra], U, x[ra:lo, ls:])
            if rb > hi:
                ops.mm_sub(G[hi - ra:], U, x[hi:rb, ls:])
            return None
        dbg = os.environ.get("RL_DIST_DEBUG_SYNC", "")
        ev = main.record_event()
        if lo > ra:
            ops.mm_sub(G[:lo - ra], U, x[ra:lo, ls:], max_ctas=max_ctas)
        if rb > hi:
            ops.mm_sub(G[hi - ra:], U, x[hi:rb, ls:], max_ctas=max_ctas)
        if "evall" in dbg:
            ev = main.record_event()
        side.wait_event(ev)
        if "pre" in dbg:
            torch.cuda.synchronize()
        with torch.cuda.stream(side):
            out = (nb, factor_block(*nb))
        if "post" in dbg:
            torch.cuda.synchronize()
        return out

    sigma = np.arange(n, dtype=np.int64)
    rrp: list[np.ndarray] = []
    r, i0, steps = 0, 0, 0
    ahead = None
    while i0 < m and r < n:
        s_end = min(m, i0 + superblock)
        r_s0 = r
        while i0 < s_end and r < n:
            bt = min(block, s_end - i0)
            if ahead is not None:
                assert ahead[0] == (i0, bt, r)
                R, wc, rt, rrp_t, sig_t, beyond = ahead[1]
                main.wait_stream(side)
                ahead = None
            else:
                R, wc, rt, rrp_t, sig_t, beyond = factor_block(i0, bt, r)
            eng.put_cols(R[:, :wc], i0, r)
            if beyond is not None:                                  # window mode
                ls, Ub = beyond
                if Ub is not None:
                    if cuda:  # allocated on the side stream, read here on main: keep its
                        Ub.record_stream(main)  # block from the side pool until main is done
                    x[i0:i0 + rt, ls:].copy_(Ub)
                x[i0 + rt:i0 + bt, ls:].zero_()
            eng.permute_cols(r, sig_t, [(0, r), (i0 + bt, m)])       # (3)
            sigma[r:] = sigma[r + sig_t]
            eng.shift_u_rows(r, i0, rt)                             # (4)
            nb = next_block(i0 + bt, r + rt, s_end)
            if rt and s_end > i0 + bt:                              # (5) + (6) in the SB
                # G = B1 * U11^{-1}: row slices solved one per rank, all-gathered
                B1 = eng.solve_rows(i0 + bt, s_end, r, r + rt, R[:rt, :rt])
                eng.put_cols(B1, i0 + bt, r)
                if tiles.lsuf(rank, r + rt) < x.shape[1]:
                    ahead = update(B1, i0 + bt, s_end, r, r + rt, nb)
            rrp.append(i0 + rrp_t[:rt])
            r += rt
            i0 += bt
            steps += 1
        rs = r - r_s0
        if rs and s_end < m:                                        # rows below the SB
            U = eng.gather_cols(r_s0, r, r_s0, r)
            G = eng.solve_rows(s_end, m, r_s0, r, U)
            eng.put_cols(G, s_end, r_s0)
            if tiles.lsuf(rank, r) < x.shape[1]:
                ahead = update(G, s_end, m, r_s0, r, next_block(s_end, r, s_end))
    if cuda:
        main.wait_stream(side)
    prof = np.concatenate(rrp) if rrp else np.zeros(0, np.int64)
    return DistCupResult(r, prof.astype(np.uint32), sigma.astype(np.uint32), steps)


def scatter_columns(a: torch.Tensor, tiles: ColumnTiles, rank: int) -> torch.Tensor:
    """This rank's local matrix (contiguous) from a full m x n matrix."""
    idx = torch.as_tensor(tiles.gpos[rank], device=a.device)
    return a.index_select(1, idx).contiguous()


def gather_columns(x: torch.Tensor, m: int, tiles: ColumnTiles) -> torch.Tensor:
    """The full m x n matrix on every rank from the local pieces."""
    dist, rank, world = _comm()
    eng = _Engine(x, m, tiles.n, tiles, None, rank, dist)
    return eng.gather_cols(0, m, 0, tiles.n)


def random_matrix_local(m: int, n: int, seed: int, p: int, tiles: ColumnTiles, rank: int,
                        device, chunk_rows: int = 2048) -> torch.Tensor:
    """This rank's columns of ``random_matrix(m, n, seed, GF(p))`` (the reference
    generator, reference.cpp:246-253), generated on the device in row chunks."""
    from . import random_matrix_dev
    x = torch.empty((m, tiles.width(rank)), dtype=torch.int32, device=device)
    idx = torch.as_tensor(tiles.gpos[rank], device=device)
    # the closed form depends on (i*n + j): generate full rows, keep our columns
    buf = torch.empty((min(chunk_rows, max(m, 1)), n), dtype=torch.int32, device=device)
    for i in range(0, m, chunk_rows):
        h = min(chunk_rows, m - i)
        # rows [i, i+h) of the m x n matrix = rows of an (i+h) x n matrix:
        # the generator's counter is i*n + j + 1, so shift the seed instead
        shift = (i * n * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        random_matrix_dev(buf[:h], h, n, (seed + shift) & ((1 << 64) - 1), p, lda=n)
        x[i:i + h].copy_(buf[:h].index_select(1, idx))
    return x
