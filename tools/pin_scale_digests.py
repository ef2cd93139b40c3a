#!/usr/bin/env python3
"""Pins bit-exact parity at the BASELINE.json configs (test infrastructure).

For each config the CPU produces (rank, row profile, sigma, packed body) and
records a digest in tests/golden/scale_digests.json, which the -m gpu tests
(tests/test_gpu_scale.py) compare against the device results:

  c1, c2, c4   the UNMODIFIED reference (oracle/_ref/libranklab_ref.so) AND the
               blocked restatement (oracle/blocked.py); both must agree, which
               pins the restatement at those sizes;
  c3, c5, s1   the blocked restatement (the reference would take ~2.7 h, ~7 days
               and ~45 min single-threaded); `c3ref` / `s1ref` run the reference
               itself in the background and add it as a second witness.

Body digest = oracle.blocked.digest (order-independent 64-bit sum of
splitmix_mix((index << 32 | value) + golden), computed on the device by
rl_digest_u32_dev); rrp / sigma digests = sha256 of their uint32 LE bytes.
Usage: pin_scale_digests.py c1|c2|c3|c3ref|c4|c5|s1|s1ref ...
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from oracle import blocked as B  # noqa: E402
from oracle import configs as CF  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "scale_digests.json")


def sha(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(x, dtype=np.uint32)).tobytes()).hexdigest()


def record(a, rank, rrp, sigma, ops, how, seconds):
    n = a.shape[1]
    return {
        "shape": list(a.shape), "rank": int(rank), "body_digest": f"{B.digest(a):016x}",
        "rrp_sha256": sha(rrp), "sigma_sha256": sha(sigma),
        "ops": [int(v) for v in ops],
        "profile_identity": bool(np.array_equal(np.asarray(rrp), np.arange(rank))),
        "sigma_identity": bool(np.array_equal(np.asarray(sigma), np.arange(n))),
        "by": how, "seconds": round(seconds, 1),
    }


def run_blocked(a, p):
    t = time.time()
    r = B.cup(a, p)
    dt = time.time() - t
    ops = B.opcount(a.shape[0], a.shape[1], r.rrp, r.ipiv)
    return record(a, r.rank, r.rrp, r.sigma, ops, "blocked", dt)


def run_ref(a, p):
    t = time.time()
    r = O.ref_cup(a, p)
    dt = time.time() - t
    return record(a, r.rank, r.rrp, r.sigma, r.ops, "reference", dt)


def same(x, y):
    keys = ("shape", "rank", "body_digest", "rrp_sha256", "sigma_sha256", "ops")
    return all(x[k] == y[k] for k in keys)


def load():
    return json.load(open(OUT)) if os.path.exists(OUT) else {}


def save(key, entry):
    import fcntl
    with open(OUT + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        d = load()
        d[key] = entry
        tmp = OUT + ".tmp"
        json.dump(d, open(tmp, "w"), indent=1, sort_keys=True)
        os.replace(tmp, OUT)
    print(f"{key}: {json.dumps(entry)[:400]}", flush=True)


def both(key, make):
    a, p = make()
    x = a.copy()
    rb = run_blocked(x, p)
    del x
    rr = run_ref(a, p)
    if not same(rb, rr):
        raise SystemExit(f"{key}: blocked restatement differs from the reference\n{rb}\n{rr}")
    e = dict(rr)
    e["p"] = p
    e["by"] = "reference+blocked"
    e["seconds_blocked"] = rb["seconds"]
    save(key, e)


def blocked_only(key, make):
    a, p = make()
    e = run_blocked(a, p)
    e["p"] = p
    old = load().get(key)
    if old and "reference" in old.get("by", ""):
        if not same(e, old):
            raise SystemExit(f"{key}: blocked differs from the stored reference digest")
        e["by"] = old["by"] if "blocked" in old["by"] else old["by"] + "+blocked"
        e["seconds_reference"] = old.get("seconds_reference", old.get("seconds"))
    save(key, e)


def ref_witness(key, make):
    """Runs the reference itself on a config the blocked restatement pinned."""
    a, p = make()
    e = run_ref(a, p)
    old = load().get(key)
    if old and not same(e, old):
        raise SystemExit(f"{key}: reference differs from the stored blocked digest\n{e}\n{old}")
    new = dict(old or e)
    new["by"] = "reference+blocked" if old else "reference"
    new["seconds_reference"] = e["seconds"]
    save(key, new)


_C4 = None


def _c4_one(t):
    ranks, ls, rs = _C4
    a = CF.c4_matrix(t, ranks, ls, rs)
    x = a.copy()
    rr = O.ref_cup(x, CF.P23)
    y = a.copy()
    rb = B.cup(y, CF.P23, leaf=16)
    ok = (rr.rank == rb.rank and np.array_equal(rr.rrp, rb.rrp) and np.array_equal(rr.sigma, rb.sigma)
          and np.array_equal(x, y) and tuple(int(v) for v in rr.ops) == B.opcount(256, 256, rb.rrp, rb.ipiv))
    return (t, int(rr.rank), f"{B.digest(x):016x}", sha(rr.rrp), sha(rr.sigma),
            [int(v) for v in rr.ops], bool(ok))


def c4():
    global _C4
    _C4 = CF.c4_recipe(4096, 4)
    t0 = time.time()
    with mp.Pool(os.cpu_count()) as pool:
        res = sorted(pool.map(_c4_one, range(4096), chunksize=16))
    dt = time.time() - t0
    if not all(r[-1] for r in res):
        raise SystemExit(f"c4: blocked differs from the reference on {[r[0] for r in res if not r[-1]]}")
    h = hashlib.sha256()
    for r in res:
        h.update(json.dumps(r[:6]).encode())
    hm = hashlib.sha256()  # without the op counts (the batched device API returns rank, rrp, sigma)
    for r in res:
        hm.update(json.dumps(r[:5]).encode())
    save("c4", {
        "count": 4096, "m": 256, "n": 256, "p": CF.P23, "seed": 4,
        "ranks": [r[1] for r in res], "body_digests": [r[2] for r in res],
        "ops_total": [int(sum(r[5][i] for r in res)) for i in range(4)],
        "records_sha256": h.hexdigest(),
        "record_format": "json.dumps([t, rank, body_digest, rrp_sha256, sigma_sha256, ops]) per matrix, in order",
        "meta_sha256": hm.hexdigest(),
        "meta_format": "json.dumps([t, rank, body_digest, rrp_sha256, sigma_sha256]) per matrix, in order",
        "sigma_identity_all": all(r[4] == sha(np.arange(256)) for r in res),
        "by": "reference+blocked", "seconds_wall": round(dt, 1), "processes": os.cpu_count(),
    })


def main():
    for what in sys.argv[1:]:
        t = time.time()
        if what == "c1":
            both("c1", CF.c1)
        elif what == "c2":
            both("c2", CF.c2)
        elif what == "c3":
            blocked_only("c3", CF.c3)
        elif what == "c3ref":
            ref_witness("c3", CF.c3)
        elif what == "c4":
            c4()
        elif what == "c5":
            blocked_only("c5", CF.c5)
        elif what == "s1":
            blocked_only("s1", CF.s1)
        elif what == "s1ref":
            ref_witness("s1", CF.s1)
        else:
            raise SystemExit(f"unknown config {what}")
        print(f"{what} done in {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
