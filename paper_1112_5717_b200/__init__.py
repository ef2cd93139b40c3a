"""paper_1112_5717_b200 -- B200-native CUP decomposition over GF(p).

Host-side mirror of the reference's hot-path interface (``ranklab``,
/root/reference/proj/include/ranklab) over the C ABI of ``libranklab_gpu.so``
(``include/ranklab_gpu.h``).  Same names, argument meaning and error behaviour:

=====================  =====================================================
this module            reference
=====================  =====================================================
``cup``                ``PackedCup cup(MatView, OpCounter&)``  factor.hpp:34
``mm``                 ``void mm(a, b, c, alpha, beta, OpCounter&)``  kernels.hpp:26
``rank_and_profile``   ``rank_and_profile(MatView, OpCounter&)``  solvers.hpp:13
``determinant``        ``Elem determinant(MatView, OpCounter&)``  solvers.hpp:16
``col_ech_trans``      ``EchelonTransform col_ech_trans(MatView, OpCounter&)``  echelon.hpp:28
``red_col_ech_trans``  ``ReducedEchelonTransform red_col_ech_trans(...)``  echelon.hpp:29
``invert_in_place``    ``void invert_in_place(MatView, OpCounter&)``  solvers.hpp:22
``trsm``               ``void trsm(Side, UpLo, Diag, t, b, OpCounter&, threshold)``  kernels.hpp:37
``PackedCup``          ``struct PackedCup``  factor.hpp:15-19
``OpCounter``          ``struct OpCounter``  field.hpp:16-34
errors                 ``errors.hpp:9-66`` (``Error`` and subclasses)
=====================  =====================================================

Matrices are numpy ``uint32`` arrays (row-major, like ``ranklab::Mat``), or
device buffers given as ``torch`` tensors for the ``*_dev`` entry points.
There is no CPU fallback: importing this package on a machine where the CUDA
library cannot be loaded raises, and every compute call without a GPU returns
``RL_ECUDA`` -> :class:`CudaError`.
"""
from __future__ import annotations

import os as _os

# ~20 streams per factorization: raise the hardware work queues from 8 to 32
# before any CUDA context exists (csrc/runtime.cu does the same when the
# library is loaded first); a user-set value wins.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Error", "DimensionMismatch", "OverlapError", "SingularMatrix", "NotPrime", "CudaError",
    "OpCounter", "PackedCup", "cup", "cup_dev", "cup_batched_dev", "cup_batched", "mm", "mm_dev",
    "rank_and_profile", "determinant", "random_matrix_dev", "LIB_PATH", "lib",
    "EchelonTransform", "ReducedEchelonTransform", "col_ech_trans", "red_col_ech_trans",
    "col_ech_trans_dev", "invert_in_place", "invert_dev", "trsm", "trsm_dev",
    "Side", "UpLo", "Diag", "PackedPle", "ple", "ple_dev", "digest_dev",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libranklab_gpu.so")


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """ranklab::Error (errors.hpp:9)."""


class DimensionMismatch(Error):
    pass


class OverlapError(Error):
    pass


class SingularMatrix(Error):
    pass


class NotPrime(Error):
    """NotPrime / ModulusOutOfRange (errors.hpp:14-24)."""


class CudaError(Error):
    pass


class InvalidArgument(Error):
    pass


_STATUS = {1: DimensionMismatch, 2: OverlapError, 3: SingularMatrix, 4: NotPrime,
           5: CudaError, 6: Error, 7: InvalidArgument, 8: CudaError}


# ------------------------------------------------------------------ types
@dataclass
class OpCounter:
    """Per-bucket field-op tallies (field.hpp:16-34)."""
    n_mul: int = 0
    n_addsub: int = 0
    n_divinv: int = 0
    n_ztest: int = 0

    def arith_total(self) -> int:
        return self.n_mul + self.n_addsub + self.n_divinv

    def full_total(self) -> int:
        return self.arith_total() + self.n_ztest

    def _add(self, ops: np.ndarray) -> None:
        self.n_mul += int(ops[0])
        self.n_addsub += int(ops[1])
        self.n_divinv += int(ops[2])
        self.n_ztest += int(ops[3])


@dataclass
class PackedCup:
    """Metadata of a packed [C\\U] factorization (factor.hpp:15-19)."""
    rank: int = 0
    row_profile: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    col_perm: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


@dataclass
class PackedPle:
    """Metadata of a packed [L\\E] factorization, A = P*L*E (factor.hpp:24-28)."""
    rank: int = 0
    col_profile: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    row_perm: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


# ---------------------------------------------------------------- loading
_lib = None
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_u32 = C.c_uint32
_vp = C.c_void_p

#: every symbol include/ranklab_gpu.h declares
EXPORTS = ["rl_cup_u32", "rl_cup_u32_dev", "rl_cup_batched_u32_dev", "rl_cup_batched_u32", "rl_mm_u32",
           "rl_mm_u32_dev", "rl_mm_u32_dev_grid", "rl_rank_and_profile_u32", "rl_determinant_u32",
           "rl_random_matrix_u32_dev", "rl_last_error", "rl_version", "rl_cup_plan_stats",
           "rl_profile_gemm_dev", "rl_cup_opcount", "rl_col_ech_trans_u32",
           "rl_col_ech_trans_u32_dev", "rl_invert_u32", "rl_invert_u32_dev", "rl_trsm_u32",
           "rl_trsm_u32_dev", "rl_trsm_opcount", "rl_echelon_opcount", "rl_ple_u32",
           "rl_ple_u32_dev", "rl_digest_u32_dev", "rl_dist_pack_u32_dev", "rl_dist_unpack_u32_dev",
           "rl_dist_select_cols_u32_dev", "rl_dist_shift_u_rows_dev"]


def lib():
    """Load libranklab_gpu.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(LIB_PATH)
    L.rl_cup_u32.argtypes = [_vp, _i64, _i64, _i64, _u32, C.POINTER(_i64), _vp, _vp, _vp]
    L.rl_cup_u32_dev.argtypes = [_vp, _i64, _i64, _i64, _u32, C.POINTER(_i64), _vp, _vp, _vp, _vp]
    L.rl_cup_batched_u32_dev.argtypes = [_vp, _i64, _i64, _i64, _i64, _u32, _vp, _vp, _vp, _vp]
    L.rl_cup_batched_u32.argtypes = [_vp, _i64, _i64, _i64, _i64, _u32, _vp, _vp, _vp]
    L.rl_mm_u32.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _u32, _u32, _u32, _vp]
    L.rl_mm_u32_dev.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _u32, _u32, _u32,
                                _vp]
    L.rl_mm_u32_dev_grid.argtypes = [_vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i64, _u32, _u32,
                                     _u32, C.c_int, _vp]
    L.rl_rank_and_profile_u32.argtypes = [_vp, _i64, _i64, _i64, _u32, C.POINTER(_i64), _vp]
    L.rl_determinant_u32.argtypes = [_vp, _i64, _i64, _u32, C.POINTER(_u32)]
    L.rl_random_matrix_u32_dev.argtypes = [_vp, _i64, _i64, _i64, C.c_uint64, _u32, _vp]
    L.rl_last_error.restype = C.c_char_p
    L.rl_cup_plan_stats.argtypes = [_i64, _i64, _i64, _u32, _vp]
    L.rl_profile_gemm_dev.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _u32, C.c_int,
                                      C.POINTER(C.c_float), C.POINTER(C.c_float), _vp]
    L.rl_cup_opcount.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp]
    L.rl_col_ech_trans_u32.argtypes = [_vp, _i64, _i64, _i64, _u32, C.c_int, C.POINTER(_i64), _vp,
                                       _vp, _vp]
    L.rl_col_ech_trans_u32_dev.argtypes = [_vp, _i64, _i64, _i64, _u32, C.c_int, C.POINTER(_i64),
                                           _vp, _vp, _vp, _vp]
    L.rl_invert_u32.argtypes = [_vp, _i64, _i64, _u32, _vp]
    L.rl_invert_u32_dev.argtypes = [_vp, _i64, _i64, _u32, _vp, _vp]
    L.rl_trsm_u32.argtypes = [C.c_int, C.c_int, C.c_int, _vp, _i64, _vp, _i64, _i64, _i64, _u32,
                              _i64, _vp]
    L.rl_trsm_u32_dev.argtypes = [C.c_int, C.c_int, C.c_int, _vp, _i64, _vp, _i64, _i64, _i64,
                                  _u32, _i64, _vp, _vp]
    L.rl_trsm_opcount.argtypes = [C.c_int, C.c_int, C.c_int, _i64, _i64, _i64, _vp]
    L.rl_echelon_opcount.argtypes = [_i64, _i64, _i64, C.c_int, _vp]
    L.rl_ple_u32.argtypes = [_vp, _i64, _i64, _i64, _u32, C.POINTER(_i64), _vp, _vp, _vp]
    L.rl_ple_u32_dev.argtypes = [_vp, _i64, _i64, _i64, _u32, C.POINTER(_i64), _vp, _vp, _vp, _vp]
    L.rl_digest_u32_dev.argtypes = [_vp, _i64, _i64, _i64, C.POINTER(C.c_uint64), _vp]
    L.rl_dist_pack_u32_dev.argtypes = [_vp, _i64, _i64, _i64, C.c_int, _vp, _vp]
    L.rl_dist_unpack_u32_dev.argtypes = [_vp, _i64, _i64, C.c_int, _vp, _i64, _vp, _i64, _vp]
    L.rl_dist_select_cols_u32_dev.argtypes = [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _i64, _vp]
    L.rl_dist_shift_u_rows_dev.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp]
    _lib = L
    return L


def _check(code: int) -> None:
    if code != 0:
        msg = lib().rl_last_error().decode(errors="replace")
        raise _STATUS.get(code, Error)(msg or f"status {code}")


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _as_u32_matrix(a: np.ndarray) -> np.ndarray:
    if not isinstance(a, np.ndarray) or a.dtype != np.uint32 or a.ndim != 2:
        raise InvalidArgument("expected a 2-D numpy uint32 array")
    if a.size and (a.strides[1] != 4 or a.strides[0] % 4):
        raise InvalidArgument("rows must be contiguous uint32")
    return a


def _ld(a: np.ndarray) -> int:
    return max(a.strides[0] // 4, a.shape[1])


# -------------------------------------------------------------------- API
def cup(a: np.ndarray, p: int, ctr: OpCounter | None = None) -> PackedCup:
    """In-place CUP of ``a`` over GF(p): ``a`` <- packed [C\\U], A = C*U*P.

    Mirrors ``ranklab::cup`` (factor.hpp:30-34): any shape including empty,
    rank deficiency is an output.  ``ctr`` receives the reference's exact
    op counts.
    """
    a = _as_u32_matrix(a)
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(1, n), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_cup_u32(_ptr(a), m, n, _ld(a), int(p), C.byref(rank), _ptr(rrp), _ptr(sigma),
                            _ptr(ops)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    return PackedCup(r, rrp[:r].copy(), sigma[:n].copy())


def cup_dev(d_a, m: int, n: int, p: int, lda: int | None = None, stream=None,
            ctr: OpCounter | None = None, want_perm: bool = True, sync: bool = True):
    """CUP of a device-resident matrix (``torch`` tensor or raw pointer).

    With ``sync=False`` nothing is read back: the factorization is only
    enqueued on ``stream`` and None is returned."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    lda = n if lda is None else lda
    if not sync:
        _check(lib().rl_cup_u32_dev(C.c_void_p(ptr), m, n, lda, int(p), None, None, None, None,
                                    _stream_ptr(stream)))
        return None
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(1, n), np.uint32) if want_perm else None
    ops = np.zeros(4, np.uint64) if ctr is not None else None
    _check(lib().rl_cup_u32_dev(C.c_void_p(ptr), m, n, lda, int(p), C.byref(rank), _ptr(rrp),
                                _ptr(sigma), _ptr(ops), _stream_ptr(stream)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    return PackedCup(r, rrp[:r].copy(), sigma[:n].copy() if want_perm else np.zeros(0, np.uint32))


def ple(a: np.ndarray, p: int, ctr: OpCounter | None = None) -> PackedPle:
    """In-place PLE of ``a`` over GF(p): ``a`` <- packed [L\\E], A = P*L*E.

    Mirrors ``ranklab::ple`` (factor.hpp:37, factor.cpp:87-156), cup's
    column-split mirror; computed on the device as cup(A^T)^T."""
    a = _as_u32_matrix(a)
    m, n = a.shape
    rank = _i64(0)
    prof = np.zeros(max(1, min(m, n)), np.uint32)
    perm = np.zeros(max(1, m), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_ple_u32(_ptr(a), m, n, _ld(a), int(p), C.byref(rank), _ptr(prof), _ptr(perm),
                            _ptr(ops)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    return PackedPle(r, prof[:r].copy(), perm[:m].copy())


def ple_dev(d_a, m: int, n: int, p: int, lda: int | None = None, stream=None,
            ctr: OpCounter | None = None) -> PackedPle:
    """PLE of a device-resident m x n matrix (``torch`` tensor or raw pointer)."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    lda = n if lda is None else lda
    rank = _i64(0)
    prof = np.zeros(max(1, min(m, n)), np.uint32)
    perm = np.zeros(max(1, m), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_ple_u32_dev(C.c_void_p(ptr), m, n, lda, int(p), C.byref(rank), _ptr(prof),
                                _ptr(perm), _ptr(ops), _stream_ptr(stream)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    return PackedPle(r, prof[:r].copy(), perm[:m].copy())


def cup_batched_dev(d_a, batch: int, m: int, n: int, p: int, stride: int | None = None,
                    stream=None, want_meta: bool = True):
    """Batched CUP of ``batch`` contiguous m x n device matrices.

    Returns (ranks int64[batch], rrp uint32[batch, min(m,n)], sigma uint32[batch, n])
    or None when ``want_meta`` is False (fully asynchronous)."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    stride = m * n if stride is None else stride
    k = max(1, min(m, n))
    if want_meta:
        ranks = np.zeros(batch, np.int64)
        rrp = np.zeros((batch, k), np.uint32)
        sigma = np.zeros((batch, max(n, 1)), np.uint32)
        _check(lib().rl_cup_batched_u32_dev(C.c_void_p(ptr), batch, m, n, stride, int(p),
                                            _ptr(ranks), _ptr(rrp), _ptr(sigma), _stream_ptr(stream)))
        return ranks, rrp, sigma[:, :n]
    _check(lib().rl_cup_batched_u32_dev(C.c_void_p(ptr), batch, m, n, stride, int(p), None, None,
                                        None, _stream_ptr(stream)))
    return None


def cup_batched(a: np.ndarray, p: int):
    """Batched in-place CUP of host matrices ``a`` (batch x m x n, uint32,
    C-contiguous; pinned memory gets the full PCIe rate): copied in, factored and
    copied back in overlapped chunks (rl_cup_batched_u32).  Returns
    (ranks int64[batch], rrp uint32[batch, min(m,n)], sigma uint32[batch, n])."""
    if a.dtype != np.uint32 or a.ndim != 3 or not a.flags.c_contiguous:
        raise Error("cup_batched expects a C-contiguous uint32 array of shape (batch, m, n)")
    batch, m, n = a.shape
    k = max(1, min(m, n))
    ranks = np.zeros(batch, np.int64)
    rrp = np.zeros((batch, k), np.uint32)
    sigma = np.zeros((batch, max(n, 1)), np.uint32)
    _check(lib().rl_cup_batched_u32(_ptr(a), batch, m, n, m * n, int(p), _ptr(ranks), _ptr(rrp),
                                    _ptr(sigma)))
    return ranks, rrp, sigma[:, :n]


def mm(a: np.ndarray, b: np.ndarray, c: np.ndarray, alpha: int, beta: int, p: int,
       ctr: OpCounter | None = None) -> None:
    """C <- alpha*A*B + beta*C (mod p), the reference's mm seam (kernels.hpp:26-27)."""
    a, b, c = _as_u32_matrix(a), _as_u32_matrix(b), _as_u32_matrix(c)
    m, l = a.shape
    if b.shape[0] != l or c.shape != (m, b.shape[1]):
        raise DimensionMismatch(f"mm {a.shape} * {b.shape} -> {c.shape}")
    n = b.shape[1]
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_mm_u32(_ptr(a), _ld(a), _ptr(b), _ld(b), _ptr(c), _ld(c), m, l, n,
                           int(alpha), int(beta), int(p), _ptr(ops)))
    if ctr is not None:
        ctr._add(ops)


def mm_dev(d_a, d_b, d_c, m, l, n, alpha, beta, p, lda=None, ldb=None, ldc=None, stream=None,
           max_ctas: int = 0):
    """C <- alpha*A*B + beta*C (mod p) on device buffers; ``max_ctas`` > 0 bounds
    the GEMM grid (rl_mm_u32_dev_grid) to leave SMs to a concurrent kernel."""
    pa = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    pb = d_b.data_ptr() if hasattr(d_b, "data_ptr") else int(d_b)
    pc = d_c.data_ptr() if hasattr(d_c, "data_ptr") else int(d_c)
    if max_ctas:
        _check(lib().rl_mm_u32_dev_grid(C.c_void_p(pa), lda or l, C.c_void_p(pb), ldb or n,
                                        C.c_void_p(pc), ldc or n, m, l, n, int(alpha), int(beta),
                                        int(p), int(max_ctas), _stream_ptr(stream)))
        return
    _check(lib().rl_mm_u32_dev(C.c_void_p(pa), lda or l, C.c_void_p(pb), ldb or n, C.c_void_p(pc),
                               ldc or n, m, l, n, int(alpha), int(beta), int(p),
                               _stream_ptr(stream)))


@dataclass
class EchelonTransform:
    """echelon.hpp:12-16: after col_ech_trans the body holds [C\\X], X the strict
    upper part of U^{-1}; A*P^T*X = C with X unit upper triangular."""
    rank: int = 0
    row_profile: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    col_perm: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


@dataclass
class ReducedEchelonTransform(EchelonTransform):
    """echelon.hpp:18-26: the body holds [[X1, X2], [R2, 0]]."""


def _echelon(a: np.ndarray, p: int, reduced: bool, ctr: OpCounter | None):
    a = _as_u32_matrix(a)
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(1, n), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_col_ech_trans_u32(_ptr(a), m, n, _ld(a), int(p), int(reduced), C.byref(rank),
                                      _ptr(rrp), _ptr(sigma), _ptr(ops)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    cls = ReducedEchelonTransform if reduced else EchelonTransform
    return cls(r, rrp[:r].copy(), sigma[:n].copy())


def col_ech_trans(a: np.ndarray, p: int, ctr: OpCounter | None = None) -> EchelonTransform:
    """In place: ``a`` <- [C\\X] (echelon.cpp:5-21)."""
    return _echelon(a, p, False, ctr)


def red_col_ech_trans(a: np.ndarray, p: int,
                      ctr: OpCounter | None = None) -> ReducedEchelonTransform:
    """In place: ``a`` <- [[X1, X2], [R2, 0]] (echelon.cpp:23-47)."""
    return _echelon(a, p, True, ctr)


def col_ech_trans_dev(d_a, m: int, n: int, p: int, reduced: bool = False, lda: int | None = None,
                      stream=None, ctr: OpCounter | None = None) -> EchelonTransform:
    """col_ech_trans / red_col_ech_trans of a device-resident matrix."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    sigma = np.zeros(max(1, n), np.uint32)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_col_ech_trans_u32_dev(C.c_void_p(ptr), m, n, lda or n, int(p), int(reduced),
                                          C.byref(rank), _ptr(rrp), _ptr(sigma), _ptr(ops),
                                          _stream_ptr(stream)))
    if ctr is not None:
        ctr._add(ops)
    r = rank.value
    cls = ReducedEchelonTransform if reduced else EchelonTransform
    return cls(r, rrp[:r].copy(), sigma[:n].copy())


def invert_in_place(a: np.ndarray, p: int, ctr: OpCounter | None = None) -> None:
    """``a`` <- a^{-1} (solvers.cpp:24-31); raises :class:`SingularMatrix` when
    rank < n, leaving red_col_ech_trans's body in ``a`` like the reference."""
    a = _as_u32_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatch("inverse of non-square matrix")
    ops = np.zeros(4, np.uint64)
    try:
        _check(lib().rl_invert_u32(_ptr(a), a.shape[0], _ld(a), int(p), _ptr(ops)))
    finally:
        if ctr is not None:
            ctr._add(ops)


def invert_dev(d_a, n: int, p: int, lda: int | None = None, stream=None,
               ctr: OpCounter | None = None) -> None:
    """invert_in_place of a device-resident n x n matrix."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_invert_u32_dev(C.c_void_p(ptr), n, lda or n, int(p), _ptr(ops),
                                   _stream_ptr(stream)))
    if ctr is not None:
        ctr._add(ops)


class Side:
    Left, Right = 0, 1


class UpLo:
    Upper, Lower = 0, 1


class Diag:
    NonUnit, Unit = 0, 1


def trsm(side: int, uplo: int, diag: int, t: np.ndarray, b: np.ndarray, p: int,
         ctr: OpCounter | None = None, threshold: int = 1) -> None:
    """B <- T^{-1} B (Side.Left) or B T^{-1} (Side.Right), kernels.hpp:37-38.

    A NonUnit zero diagonal raises :class:`SingularMatrix` (the reference's
    SingularDiagonal) with ``b`` untouched."""
    t, b = _as_u32_matrix(t), _as_u32_matrix(b)
    m, n = b.shape
    k = m if side == Side.Left else n
    if t.shape != (k, k):
        raise DimensionMismatch(f"triangular operand {t.shape} vs {k}")
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_trsm_u32(int(side), int(uplo), int(diag), _ptr(t), max(_ld(t), 1), _ptr(b),
                             max(_ld(b), 1), m, n, int(p), int(threshold), _ptr(ops)))
    if ctr is not None:
        ctr._add(ops)


def trsm_dev(side: int, uplo: int, diag: int, d_t, d_b, m: int, n: int, p: int,
             ldt: int | None = None, ldb: int | None = None, stream=None,
             ctr: OpCounter | None = None, threshold: int = 1) -> None:
    pt = d_t.data_ptr() if hasattr(d_t, "data_ptr") else int(d_t)
    pb = d_b.data_ptr() if hasattr(d_b, "data_ptr") else int(d_b)
    k = m if side == Side.Left else n
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_trsm_u32_dev(int(side), int(uplo), int(diag), C.c_void_p(pt), ldt or k,
                                 C.c_void_p(pb), ldb or n, m, n, int(p), int(threshold), _ptr(ops),
                                 _stream_ptr(stream)))
    if ctr is not None:
        ctr._add(ops)


def trsm_opcount(side: int, uplo: int, diag: int, m: int, n: int, threshold: int = 1) -> np.ndarray:
    """The reference's trsm charges (host-only, no device needed)."""
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_trsm_opcount(int(side), int(uplo), int(diag), m, n, int(threshold), _ptr(ops)))
    return ops


def echelon_opcount(m: int, n: int, r: int, reduced: bool) -> np.ndarray:
    """Charges of col_ech_trans / red_col_ech_trans after the cup (host-only)."""
    ops = np.zeros(4, np.uint64)
    _check(lib().rl_echelon_opcount(m, n, r, int(reduced), _ptr(ops)))
    return ops


def rank_and_profile(a: np.ndarray, p: int):
    """(rank, row rank profile); the input is consumed (solvers.hpp:13-14)."""
    a = _as_u32_matrix(a)
    m, n = a.shape
    rank = _i64(0)
    rrp = np.zeros(max(1, min(m, n)), np.uint32)
    _check(lib().rl_rank_and_profile_u32(_ptr(a), m, n, _ld(a), int(p), C.byref(rank), _ptr(rrp)))
    return rank.value, rrp[:rank.value].copy()


def determinant(a: np.ndarray, p: int) -> int:
    """sign(P) * product of pivots; the input is consumed (solvers.hpp:16)."""
    a = _as_u32_matrix(a)
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatch("determinant of non-square matrix")
    d = _u32(0)
    _check(lib().rl_determinant_u32(_ptr(a), a.shape[0], _ld(a), int(p), C.byref(d)))
    return d.value


def random_matrix_dev(d_a, m: int, n: int, seed: int, p: int, lda: int | None = None,
                      stream=None) -> None:
    """Device-side ranklab::random_matrix(m, n, seed, GF(p)) (reference.cpp:246-253)."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    _check(lib().rl_random_matrix_u32_dev(C.c_void_p(ptr), m, n, lda or n,
                                          C.c_uint64(seed & (2**64 - 1)), int(p),
                                          _stream_ptr(stream)))


def digest_dev(d_a, m: int, n: int, lda: int | None = None, stream=None) -> int:
    """Order-independent 64-bit digest of a device matrix (rl_digest_u32_dev; the
    oracle computes the same function on the host)."""
    ptr = d_a.data_ptr() if hasattr(d_a, "data_ptr") else int(d_a)
    h = C.c_uint64(0)
    _check(lib().rl_digest_u32_dev(C.c_void_p(ptr), m, n, n if lda is None else lda, C.byref(h),
                                   _stream_ptr(stream)))
    return h.value


# Data plane of the distributed CUP (dist.py): torch CUDA tensors, enqueued on
# `stream` (torch's current stream when None), no synchronisation.
def _dp(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _cur(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return _stream_ptr(stream)


def dist_pack_dev(src, dst, wire16: bool, stream=None) -> None:
    """dst (rows x cols, contiguous; int16 words x - 2^15 when wire16) <- src
    (a row-major view with unit column stride)."""
    rows, cols = src.shape
    _check(lib().rl_dist_pack_u32_dev(_dp(src), src.stride(0), rows, cols, int(wire16), _dp(dst),
                                      _cur(stream)))


def dist_unpack_dev(src, dst, wire16: bool, colmap=None, off: int = 0, stream=None) -> None:
    """dst[r, colmap[c] - off] <- src[r, c] (colmap: int64 device tensor, or None for c)."""
    rows, cols = src.shape
    _check(lib().rl_dist_unpack_u32_dev(_dp(src), rows, cols, int(wire16), _dp(dst), dst.stride(0),
                                        None if colmap is None else _dp(colmap), off, _cur(stream)))


def dist_select_cols_dev(src, colmap, dst, off: int = 0, stream=None) -> None:
    """dst[r, c] <- src[r, colmap[c] - off] for c < colmap.numel()."""
    rows = dst.shape[0]
    _check(lib().rl_dist_select_cols_u32_dev(_dp(src), src.stride(0), rows, _dp(colmap), off, colmap.numel(),
                                             _dp(dst), dst.stride(0), _cur(stream)))


def dist_shift_u_rows_dev(x, cols_from: int, r: int, i0: int, rt: int, gpos, stream=None) -> None:
    """The U-row move of factor.cpp:62-70 on the local columns from cols_from on
    (gpos: their global positions, int64 device tensor)."""
    v = x[:, cols_from:]
    _check(lib().rl_dist_shift_u_rows_dev(_dp(v), x.stride(0), v.shape[1], r, i0, rt, _dp(gpos),
                                          _cur(stream)))


def plan_stats(m: int, n: int, p: int, lda: int | None = None) -> dict:
    st = np.zeros(6, np.int64)
    _check(lib().rl_cup_plan_stats(m, n, lda or n, int(p), _ptr(st)))
    return dict(gemms=int(st[0]), tc_gemms=int(st[1]), panels=int(st[2]), trsm_leaves=int(st[3]),
                workspace_bytes=int(st[4]), launches=int(st[5]))


def profile_gemm_dev(d_a, d_b, d_c, m: int, l: int, n: int, p: int, iters: int = 5, stream=None):
    """(ms of the two pack kernels, ms of the tcgen05 GEMM kernel) for C <- C - A*B."""
    mp, mg = C.c_float(0), C.c_float(0)
    _check(lib().rl_profile_gemm_dev(C.c_void_p(d_a.data_ptr()), C.c_void_p(d_b.data_ptr()),
                                     C.c_void_p(d_c.data_ptr()), m, l, n, int(p), iters,
                                     C.byref(mp), C.byref(mg), _stream_ptr(stream)))
    return mp.value, mg.value


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def model_ops(m: int, n: int, r: int) -> float:
    """The reference's CUP cost model W(m,n,r) = 2mnr - (m+n)r^2 + (2/3)r^3
    (proj/src/bench.cpp:12-13)."""
    return 2.0 * m * n * r - (m + n) * r * r + (2.0 / 3.0) * r ** 3
