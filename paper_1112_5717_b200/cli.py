"""``python -m paper_1112_5717_b200`` -- the reference's command-line tool
(proj/tools/main.cpp) on the B200 path: the same subcommands, options, output
bytes and exit codes (0 success; 1 usage, IO or singular-matrix errors; 3
inconsistent linear system), with every factorization running through this
package's C ABI.  ``selftest`` (main.cpp:262-296) is not provided here: the
reference's own acceptance suite relinked on the GPU library
(``make -C oracle acceptance-gpu``) is the self-check.

Subcommands (main.cpp:298-349):
  factor  --in F [--algo cup|ple] [--expand] [--count-ops] [--out O]
  echelon --in F [--reduced] [--out O]
  solve   --in F --rhs B [--out O]
  inverse --in F [--out O]
  bench   --algo A --n N [--m M] [--r R] [--field P] [--seed S] [--trials T]
          [--json] [--placement generic|spread] [--threshold K]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

from . import textio

USAGE = __doc__.split("Subcommands", 1)[1]


class Usage(Exception):
    pass


def _default_seed() -> int:
    env = os.environ.get("RANKLAB_SEED")
    if env is not None and env.isdigit():
        return int(env)
    return 1


def _parse(argv: list[str]):
    """CLI11-equivalent parsing of main.cpp:298-342 (required options, flags, defaults)."""
    if not argv or argv[0] in ("-h", "--help"):
        raise Usage("help")
    sub = argv[0]
    spec = {
        "factor": ({"--in": None, "--algo": "cup", "--out": ""}, {"--expand", "--count-ops"},
                   {"--in"}),
        "echelon": ({"--in": None, "--out": ""}, {"--reduced"}, {"--in"}),
        "solve": ({"--in": None, "--rhs": None, "--out": ""}, set(), {"--in", "--rhs"}),
        "inverse": ({"--in": None, "--out": ""}, set(), {"--in"}),
        "bench": ({"--algo": None, "--m": "0", "--n": None, "--r": "0", "--field": "65521",
                   "--seed": None, "--trials": "1", "--placement": "generic", "--threshold": "1"},
                  {"--json"}, {"--algo", "--n"}),
    }
    if sub not in spec:
        raise Usage(f"unknown subcommand '{sub}'")
    opts, flags, required = spec[sub]
    vals = dict(opts)
    on = set()
    i = 1
    while i < len(argv):
        a = argv[i]
        key, eq, inline = a.partition("=")
        if key in flags and not eq:
            on.add(key)
            i += 1
        elif key in opts:
            if eq:
                vals[key] = inline
                i += 1
            else:
                if i + 1 >= len(argv):
                    raise Usage(f"{key} requires an argument")
                vals[key] = argv[i + 1]
                i += 2
        else:
            raise Usage(f"unexpected argument '{a}'")
    for r in required:
        if vals.get(r) is None:
            raise Usage(f"{r} is required")
    return sub, vals, on


def _header(out, algo, rank, profile, perm):
    """write_profile_header (main.cpp:32-43)."""
    out.write(f"algo {algo}\nrank {rank}\nprofile")
    out.write("".join(f" {v}" for v in np.asarray(profile).tolist()))
    out.write("\nperm")
    out.write("".join(f" {v}" for v in np.asarray(perm).tolist()))
    out.write("\n")


class _Sink:
    def __init__(self, path: str):
        self.path = path
        self.parts: list[str] = []

    def write(self, s: str) -> None:
        self.parts.append(s)

    def close(self) -> None:
        data = "".join(self.parts)
        if self.path:
            try:
                with open(self.path, "w", encoding="latin-1", newline="") as f:
                    f.write(data)
            except OSError:
                raise OSError(f"cannot open {self.path} for writing") from None
        else:
            sys.stdout.write(data)
            sys.stdout.flush()


def _open_sink(path: str) -> _Sink:
    if path:
        try:  # the reference opens the sink before computing (main.cpp:47-54)
            open(path, "w").close()
        except OSError:
            raise OSError(f"cannot open {path} for writing") from None
    return _Sink(path)


def cmd_factor(vals, on) -> int:
    from . import OpCounter, cup, ple
    a, p = textio.read_matrix_file(vals["--in"])
    sink = _open_sink(vals["--out"])
    ctr = OpCounter()
    algo = vals["--algo"]
    m, n = a.shape
    if algo == "cup":
        pc = cup(a, p, ctr)
        r = pc.rank
        _header(sink, algo, r, pc.row_profile, pc.col_perm)
        if "--expand" in on:  # expand_cup (factor.cpp:198-211)
            c = np.tril(a[:, :r])
            u = np.triu(a[:r, :], 1)
            u[np.arange(r), np.arange(r)] = 1 % p
            sink.write("C\n" + textio.format_matrix(c, p) + "U\n" + textio.format_matrix(u, p))
        else:
            sink.write("body\n" + textio.format_matrix(a, p))
    elif algo == "ple":
        pp = ple(a, p, ctr)
        r = pp.rank
        _header(sink, algo, r, pp.col_profile, pp.row_perm)
        if "--expand" in on:  # expand_ple (factor.cpp:213-226)
            lo = np.tril(a[:, :r], -1)
            lo[np.arange(r), np.arange(r)] = 1 % p
            e = np.triu(a[:r, :])
            sink.write("L\n" + textio.format_matrix(lo, p) + "E\n" + textio.format_matrix(e, p))
        else:
            sink.write("body\n" + textio.format_matrix(a, p))
    else:
        from . import Error
        raise Error(f"unknown --algo '{algo}' (expected cup or ple)")
    sink.close()
    if "--count-ops" in on:  # print_ops (main.cpp:58-62)
        print(f"ops mul={ctr.n_mul} addsub={ctr.n_addsub} divinv={ctr.n_divinv} "
              f"ztest={ctr.n_ztest} arith={ctr.arith_total()} total={ctr.full_total()}")
    return 0


def cmd_echelon(vals, on) -> int:
    from . import OpCounter, col_ech_trans, red_col_ech_trans
    a, p = textio.read_matrix_file(vals["--in"])
    sink = _open_sink(vals["--out"])
    ctr = OpCounter()
    m, n = a.shape
    if "--reduced" in on:
        t = red_col_ech_trans(a, p, ctr)
        r = t.rank
        _header(sink, "redcolech", r, t.row_profile, t.col_perm)
        # reduced_form (echelon.cpp:67-78)
        rf = np.zeros((m, n), np.uint32)
        rf[np.arange(r), np.arange(r)] = 1 % p
        rf[r:, :r] = a[r:, :r]
        for j in range(r - 1, -1, -1):
            k = int(t.row_profile[j])
            if k != j:
                rf[[j, k]] = rf[[k, j]]
        sink.write("R\n" + textio.format_matrix(rf, p))
    else:
        t = col_ech_trans(a, p, ctr)
        r = t.rank
        _header(sink, "colech", r, t.row_profile, t.col_perm)
        e = np.zeros((m, n), np.uint32)  # echelon_form (echelon.cpp:49-56)
        e[:, :r] = np.tril(a[:, :r])
        sink.write("E\n" + textio.format_matrix(e, p))
    sink.close()
    return 0


def _mod_dot(row: np.ndarray, vec: np.ndarray, p: int) -> int:
    if len(row) == 0:
        return 0
    return int((row.astype(np.uint64) * vec.astype(np.uint64) % np.uint64(p)).sum() % np.uint64(p))


def cmd_solve(vals, on) -> int:
    """solve (solvers.cpp:33-103): cup on the device, then the O(n^2) substitutions."""
    from . import DimensionMismatch, Error, OpCounter, cup
    a, p = textio.read_matrix_file(vals["--in"])
    b, pb = textio.read_matrix_file(vals["--rhs"])
    if p != pb:
        raise Error("matrix and right-hand side use different moduli")
    m, n = a.shape
    if b.shape != (m, 1):
        raise DimensionMismatch(f"right-hand side must be {m}x1")
    pc = cup(a, p, OpCounter())
    r, rrp = pc.rank, pc.row_profile.astype(np.int64)
    bb = b[:, 0]
    z = np.zeros(r, np.uint32)
    for j in range(r):
        row = rrp[j]
        s = (int(bb[row]) - _mod_dot(a[row, :j], z[:j], p)) % p
        z[j] = s * pow(int(a[row, j]), p - 2, p) % p
    is_piv = np.zeros(m, bool)
    is_piv[rrp] = True
    for i in range(m):
        if is_piv[i]:
            continue
        t = min(i + 1, r)
        if _mod_dot(a[i, :t], z[:t], p) != int(bb[i]):
            print(f"INCONSISTENT row {i}")
            return 3
    x = np.zeros(n, np.uint32)
    for ii in range(n - 1, -1, -1):
        v = int(z[ii]) if ii < r else 0
        if ii < r:
            v = (v - _mod_dot(a[ii, ii + 1:], x[ii + 1:], p)) % p
        x[ii] = v
    xf = np.zeros(n, np.uint32)  # perm_apply_rows(x, sigma, inverse): new row sigma(i) = old row i
    xf[pc.col_perm.astype(np.int64)] = x
    sink = _open_sink(vals["--out"])
    sink.write(textio.format_matrix(xf.reshape(n, 1), p))
    sink.close()
    return 0


def cmd_inverse(vals, on) -> int:
    from . import OpCounter, SingularMatrix, invert_in_place
    a, p = textio.read_matrix_file(vals["--in"])
    try:
        invert_in_place(a, p, OpCounter())
    except SingularMatrix:
        sys.stderr.write("SINGULAR\n")
        return 1
    sink = _open_sink(vals["--out"])
    sink.write(textio.format_matrix(a, p))
    sink.close()
    return 0


def _predicted(algo: str, m: int, n: int, r: int) -> float:
    """predicted_arith (bench.cpp:9-23)."""
    dm, dn, dr = float(m), float(n), float(r)
    if algo in ("cup", "ple"):
        return 2.0 * dm * dn * dr - (dm + dn) * dr * dr + (2.0 / 3.0) * dr * dr * dr
    table = {"mm": 2.0, "trsm": 1.0, "colech": 1.0, "redcolech": 2.0}
    return table[algo] * dn * dn * dn


def cmd_bench(vals, on) -> int:
    """cmd_bench (main.cpp:157-250) for the algorithms on the GPU path."""
    from . import (OpCounter, Diag, Error, Side, UpLo, col_ech_trans, cup, mm, ple,
                   red_col_ech_trans, trsm)
    from . import gen
    algo = vals["--algo"]
    n = int(vals["--n"])
    m = int(vals["--m"]) or n
    r = int(vals["--r"])
    p = int(vals["--field"])
    why = textio.is_prime_field(p)
    if why is not None:
        raise Error(why)
    seed = int(vals["--seed"]) if vals["--seed"] is not None else _default_seed()
    trials = int(vals["--trials"])
    placement = vals["--placement"]
    if placement not in ("generic", "spread"):
        raise Usage("--placement: generic or spread")
    threshold = int(vals["--threshold"])
    if r == 0 or r > min(m, n):
        r = min(m, n)
    if algo not in ("cup", "ple", "mm", "trsm", "colech", "redcolech"):
        if algo in ("trtri", "trulm", "trlum", "gaussjordan", "inplacemm"):
            raise Error(f"--algo '{algo}' is not on the GPU path")
        raise Error(f"unknown --algo '{algo}'")
    for t in range(trials):
        s = seed + t
        ctr = OpCounter()
        rm, rr = m, r
        t0 = time.perf_counter()
        if algo in ("cup", "ple"):
            if m == n and r == n:
                a = gen.random_nonsingular_matrix(n, s, p)
            else:
                a = gen.random_rank_matrix(m, n, r, s, p, spread=placement == "spread")
            rr = (cup(a, p, ctr) if algo == "cup" else ple(a, p, ctr)).rank
        elif algo == "mm":
            a = gen.random_matrix(n, n, s, p)
            b = gen.random_matrix(n, n, s + 0x9E37, p)
            c = np.zeros((n, n), np.uint32)
            mm(a, b, c, 1 % p, 0, p, ctr)
            rm = rr = n
        elif algo == "trsm":
            tt = gen.random_triangular_matrix(n, s, p)
            b = gen.random_matrix(n, n, s + 0x9E37, p)
            trsm(Side.Right, UpLo.Upper, Diag.NonUnit, tt, b, p, ctr, threshold=threshold)
            rm = rr = n
        else:
            a = gen.random_nonsingular_matrix(n, s, p)
            (col_ech_trans if algo == "colech" else red_col_ech_trans)(a, p, ctr)
            rm = rr = n
        wall = (time.perf_counter() - t0) * 1e3
        pred = _predicted(algo, rm, n, rr)
        ratio = ctr.arith_total() / pred if pred > 0 else 0.0
        fields = [("algo", algo), ("m", rm), ("n", n), ("r", rr), ("p", p), ("seed", s),
                  ("ops_arith", ctr.arith_total()), ("ops_ztest", ctr.n_ztest),
                  ("ops_mul", ctr.n_mul), ("ops_addsub", ctr.n_addsub),
                  ("ops_divinv", ctr.n_divinv), ("predicted", f"{pred:.0f}"),
                  ("ratio", f"{ratio:.4f}")]
        if "--json" in on:  # format_report_json (bench.cpp:39-51)
            body = ",".join(f'"{k}":"{v}"' if k == "algo" else f'"{k}":{v}' for k, v in fields)
            print("{" + body + "}")
        else:  # format_report_kv (bench.cpp:25-37)
            print(" ".join(f"{k}={v}" for k, v in fields))
        sys.stdout.flush()
        sys.stderr.write(f"wall_ms={wall:.6g}\n")
    return 0


def main(argv: list[str] | None = None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    try:
        sub, vals, on = _parse(argv)
    except Usage as u:
        if str(u) == "help":
            print("ranklab (B200): exact dense linear algebra over GF(p)\n" + USAGE)
            return 0
        sys.stderr.write(f"{u}\n{USAGE}")
        return 1
    from . import Error
    try:
        return {"factor": cmd_factor, "echelon": cmd_echelon, "solve": cmd_solve,
                "inverse": cmd_inverse, "bench": cmd_bench}[sub](vals, on)
    except Usage as u:
        sys.stderr.write(f"{u}\n")
        return 1
    except (Error, textio.ParseError, OSError, ValueError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
