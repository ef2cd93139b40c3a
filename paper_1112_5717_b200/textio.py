"""The reference's matrix text format (proj/include/ranklab/io.hpp:10-15,
proj/src/io.cpp): line 1 "m n p", then m lines of n space-separated entries in
[0, p), LF-only, single spaces, no trailing whitespace.  The parser rejects
anything else with the reference's "line L, column C: ..." diagnostics
(errors.hpp:59-66), including its size cap (m, n <= 2^20, m*n <= 2^28) and the
field validation of the modulus."""
from __future__ import annotations

import io

import numpy as np

U64_MAX = (1 << 64) - 1


class ParseError(ValueError):
    """ranklab::ParseError (errors.hpp:59-66)."""

    def __init__(self, line: int, col: int, msg: str):
        super().__init__(f"line {line}, column {col}: {msg}")
        self.line, self.column = line, col


def is_prime_field(p: int) -> str | None:
    """None if GF(p) is valid (PrimeField, field.cpp:54-76), else the reason."""
    if p < 2 or p >= (1 << 31):
        return f"modulus {p} outside [2, 2^31)"
    if p < 4:
        return None
    if p % 2 == 0:
        return f"modulus {p} is not prime"
    d = 3
    while d * d <= p:
        if p % d == 0:
            return f"modulus {p} is not prime"
        d += 2
    return None


class _Lexer:
    def __init__(self, s: str, line: int):
        self.s, self.line, self.pos = s, line, 0

    def next_uint(self, what: str) -> int:
        s = self.s
        if self.pos >= len(s) or s[self.pos] == " ":
            raise ParseError(self.line, self.pos + 1, f"expected {what}")
        start, v = self.pos, 0
        while self.pos < len(s) and s[self.pos] != " ":
            ch = s[self.pos]
            if not "0" <= ch <= "9":
                raise ParseError(self.line, self.pos + 1, f"invalid character in {what}")
            v = v * 10 + ord(ch) - 48
            if v > U64_MAX // 16:
                raise ParseError(self.line, start + 1, f"{what} too large")
            self.pos += 1
        return v

    def expect_space(self, after: str) -> None:
        if self.pos >= len(self.s) or self.s[self.pos] != " ":
            raise ParseError(self.line, self.pos + 1, f"expected single space after {after}")
        self.pos += 1
        if self.pos < len(self.s) and self.s[self.pos] == " ":
            raise ParseError(self.line, self.pos + 1, "double space")

    def expect_end(self) -> None:
        if self.pos != len(self.s):
            raise ParseError(self.line, self.pos + 1, "trailing characters")


def _get_line(stream, line_no: int) -> str:
    raw = stream.readline()
    if raw == "":
        raise ParseError(line_no, 1, "unexpected end of input")
    s = raw[:-1] if raw.endswith("\n") else raw
    if s.endswith("\r"):
        raise ParseError(line_no, len(s), "carriage return (file must be LF-only)")
    return s


def read_matrix(stream) -> tuple[np.ndarray, int]:
    """Parse one matrix; returns (uint32 array m x n, p)."""
    hl = _Lexer(_get_line(stream, 1), 1)
    m = hl.next_uint("row count")
    hl.expect_space("row count")
    n = hl.next_uint("column count")
    hl.expect_space("column count")
    p = hl.next_uint("modulus")
    hl.expect_end()
    if m > (1 << 20) or n > (1 << 20) or m * n > (1 << 28):
        raise ParseError(1, 1, "matrix dimensions too large")
    why = is_prime_field(p)
    if why is not None:
        raise ParseError(1, 1, why)
    a = np.zeros((m, n), np.uint32)
    for i in range(m):
        row = _get_line(stream, i + 2)
        # fast path: a well-formed row
        parts = row.split(" ")
        if len(parts) == n and n > 0 and all(t.isdigit() and t.isascii() and len(t) <= 18 for t in parts):
            vals = np.array([int(t) for t in parts], dtype=np.uint64)
            if int(vals.max()) < p:
                a[i] = vals
                continue
        lx = _Lexer(row, i + 2)
        for j in range(n):
            if j > 0:
                lx.expect_space("entry")
            col = lx.pos + 1
            v = lx.next_uint("entry")
            if v >= p:
                raise ParseError(i + 2, col, f"entry {v} not in [0, {p})")
            a[i, j] = v
        lx.expect_end()
    return a, p


def read_matrix_file(path: str) -> tuple[np.ndarray, int]:
    try:
        f = open(path, "r", encoding="latin-1", newline="")
    except OSError:
        raise OSError(f"cannot open {path}") from None
    with f:
        return read_matrix(f)


def format_matrix(a: np.ndarray, p: int) -> str:
    """write_matrix (io.cpp): header then rows, LF-terminated."""
    out = io.StringIO()
    m, n = a.shape
    out.write(f"{m} {n} {p}\n")
    for i in range(m):
        out.write(" ".join(map(str, a[i].tolist())))
        out.write("\n")
    return out.getvalue()
