#!/usr/bin/env python3
"""bench.py -- CUP mod-p ops/s on B200 (BASELINE.json metric, config 3 by default).

Workload (``--workload c3``, the configuration BASELINE.json's metric is quoted
on): in-place CUP of ONE 16384 x 16384 matrix over GF(65521), entries
``ranklab::random_matrix(16384, 16384, seed=3, GF(65521))`` generated on the
device bit-identically to the reference generator (reference.cpp:246-253).
A "step" is one full factorization (rank, row profile, sigma, packed [C\\U]).

Metric: mod-p ops/s with the reference's own cost model
W(m,n,r) = 2mnr - (m+n)r^2 + (2/3)r^3 (bench.cpp:12-13) at the returned rank.

* ``value``     device-resident: input already in HBM; CUDA events on the
                launching stream bracket each factorization (the per-step
                restore of the input is outside the events); 1 GiB input > L2.
* ``e2e``       the same metric through the C ABI with HOST buffers
                (rl_cup_u32: pinned H2D, factorization, D2H of the body,
                rank, profile and sigma), timed by the host around the call.
* ``roofline``  dominant kernel = the tcgen05 limb GEMM; achieved int8 TOPS of
                the root Schur GEMM shape (8192^3) timed live with CUDA events
                vs the measured cuBLAS int8 dense peak on this GPU.
* ``cpu_baseline`` the UNMODIFIED reference (oracle/_ref) on a bounded sample.

``--impl reference`` times the reference's CPU cup on the host cores instead
(T threads, each factoring its own 1024^2 random_matrix sample).

Multi-GPU (torchrun, N>1): ``--workload c5`` factors ONE 65536^2 matrix
distributed over the ranks (paper_1112_5717_b200/dist.py: 1D block-cyclic column
tiles, NCCL broadcasts of each row block and of its pivot columns, local
tensor-core Schur updates), value = W / max-over-ranks time, scaling "strong";
``--dist`` runs the same driver at N = 1.  For C1-C3 every rank factors its
own replica ("replicas only"), value = N * W / max-over-ranks time, scaling "weak".  ``--workload c4``
shards the fixed batch of 4096 matrices across the ranks as contiguous slices
(no collective on the data path), value = 4096 matrices / max-over-ranks time,
scaling "strong".
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

# the factorization's launch sequence spans ~20 streams: 32 hardware work
# queues instead of 8 (set before any CUDA context; see csrc/runtime.cu)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c3": dict(m=16384, n=16384, p=65521, seed=3,
               desc="CUP of one 16384x16384 random_matrix(seed=3) over GF(65521)"),
    "c1": dict(m=1024, n=1024, p=65521, seed=1,
               desc="CUP of one 1024x1024 random_matrix(seed=1) over GF(65521)"),
    "c2048": dict(m=2048, n=2048, p=65521, seed=3,
                  desc="CUP of one 2048x2048 random_matrix(seed=3) over GF(65521)"),
    "c8192": dict(m=8192, n=8192, p=65521, seed=3,
                  desc="CUP of one 8192x8192 random_matrix(seed=3) over GF(65521)"),
    "c5": dict(m=65536, n=65536, p=65521, seed=5, tile=1024, block=1024, superblock=4096,
               desc="CUP of one 65536x65536 random_matrix(seed=5) over GF(65521) (17 GB); one "
                    "GPU: the recursive engine; N > 1 (or --dist): 1D block-cyclic column tiles "
                    "over the ranks, NCCL broadcasts of the row block and the pivot columns"),
    "c2": dict(m=4096, n=8192, p=65521, seed=2, inner=2048,
               desc="CUP of the config-2 4096x8192 rank-2048 matrix (L*R mod p, rows i=2 mod 3 "
                    "zeroed, rows shuffled by SplitMix64(seed+2))"),
    "c4": dict(m=256, n=256, p=8388593, seed=4, batch=4096,
               desc="batched CUP of 4096 config-4 matrices 256x256 over GF(8388593), rank "
                    "128..256 (L_t*R_t mod p); the batch is sharded across ranks"),
}
METRIC = "CUP mod-p ops/s (2n^3/3) at n=16384, % tensor peak; batched matrices/s"


def model_ops(m, n, r):
    return 2.0 * m * n * r - (m + n) * r * r + (2.0 / 3.0) * r ** 3


def limbs(p):
    return max(1, ((p - 1).bit_length() + 7) // 8)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------- reference arm
def _ref_worker_init():
    import oracle  # noqa: F401  (loads oracle/_ref/libranklab_ref.so once per worker)


def _ref_cup_square(job):
    """One reference cup() of random_matrix(size, size, seed) over GF(p): (seconds, rank)."""
    import oracle as O
    size, seed, p = job
    a = O.port_random_matrix(size, size, seed, p)
    t0 = time.perf_counter()
    r = O.ref_cup(a, p)
    return time.perf_counter() - t0, r.rank


def _ref_cup_c4(job):
    """Reference cup() on config-4 matrices [lo, hi): seconds of factorization."""
    import oracle as O
    from paper_1112_5717_b200 import workloads as WL
    from tests.helpers import matmul_mod
    lo, hi, seed, p = job
    ranks, ls, rs = WL.c4_recipe(hi, seed)
    mats = [matmul_mod(O.port_random_matrix(256, ranks[t], ls[t], p),
                       O.port_random_matrix(ranks[t], 256, rs[t], p), p) for t in range(lo, hi)]
    t0 = time.perf_counter()
    for a in mats:
        O.ref_cup(a, p)
    return time.perf_counter() - t0


def _pool(n):
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    return ProcessPoolExecutor(n, mp_context=mp.get_context("fork"), initializer=_ref_worker_init)


def run_cpu_reference(n_proc: int, size: int, steps: int, warmup: int, p: int, seed: int):
    """Each step: n_proc concurrent reference cup() calls (one process per host
    core; the reference is single-threaded) on size^2 samples.  Returns the
    aggregate mod-p ops/s and the mean step time (the slowest worker)."""
    times, ops = [], 0.0
    with _pool(n_proc) as ex:
        for it in range(warmup + steps):
            out = list(ex.map(_ref_cup_square, [(size, seed + 1000 * t, p) for t in range(n_proc)]))
            if it >= warmup:
                times.append(max(o[0] for o in out))
                ops += sum(model_ops(size, size, o[1]) for o in out)
    return ops / sum(times), sum(times) / len(times)


def run_cpu_reference_c4(n_proc: int, per_proc: int, steps: int, warmup: int, p: int, seed: int):
    """Each step: n_proc concurrent processes, each running the reference cup()
    on its own `per_proc` config-4 matrices.  Returns matrices/s, s/step."""
    times = []
    with _pool(n_proc) as ex:
        for it in range(warmup + steps):
            jobs = [(t * per_proc, (t + 1) * per_proc, seed, p) for t in range(n_proc)]
            out = list(ex.map(_ref_cup_c4, jobs))
            if it >= warmup:
                times.append(max(out))
    step = sum(times) / len(times)
    return n_proc * per_proc / step, step


def reference_arm(args, rank, world):
    if world > 1 and rank != 0:
        return
    wl = WORKLOADS[args.workload]
    try:
        import oracle as O
        if not O.have_ref():
            raise FileNotFoundError("oracle/_ref/libranklab_ref.so not built")
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    threads = os.cpu_count() or 1
    if args.workload == "c4":
        per = 4
        val, step_s = run_cpu_reference_c4(threads, per, args.steps, args.warmup, wl["p"], wl["seed"])
        unit = "matrices/s"
        sample = (f"{threads} concurrent processes x {per} reference cup() calls on config-4 "
                  f"256x256 matrices over GF({wl['p']}) per step")
        scaling = "strong"
    else:
        size = 1024
        val, step_s = run_cpu_reference(threads, size, args.steps, args.warmup, wl["p"], wl["seed"])
        unit = "mod-p ops/s"
        sample = (f"{threads} concurrent processes, each one reference cup() of "
                  f"random_matrix({size},{size}) per step (the reference is single-threaded)")
        scaling = "weak"
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": unit,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "u32 (u64 products, % p)", "data": "synthetic",
        "config": {"workload": args.workload, "p": wl["p"], "sample": sample},
        "cpu_baseline": {"value": val, "unit": unit, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.workload != "c4":
        line["config"]["same_config"] = False
        line["config"]["why_sample"] = ("the reference's single-threaded cup() of the full workload "
                                        "takes hours (config 3: ~2.7 h per matrix); each host core "
                                        "factors a bounded sample per step")
    if args.workload == "c3" and not args.no_batched:
        per = 4
        bval, bstep = run_cpu_reference_c4(threads, per, max(1, min(args.steps, 5)), 1,
                                           WORKLOADS["c4"]["p"], WORKLOADS["c4"]["seed"])
        bsample = (f"{threads} concurrent processes x {per} reference cup() calls on config-4 "
                   f"256x256 matrices over GF({WORKLOADS['c4']['p']}) per step")
        line["batched"] = {"value": bval, "unit": "matrices/s", "ms_per_step": bstep * 1e3,
                           "cpu_baseline": {"value": bval, "unit": "matrices/s", "cores": threads,
                                            "kind": "reference", "sample": bsample},
                           "e2e": {"value": bval, "unit": "matrices/s", "h2d_bytes_per_step": 0,
                                   "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------- our arm
def _ncu_traffic():
    """DRAM bytes (read + write) per gemm_tc_kernel launch at 8192^3 from the
    committed ncu --set full capture, or None."""
    path = os.path.join(ROOT, "profiles", "round2", "gemm_8192_ncu.json")
    try:
        with open(path) as f:
            d = json.load(f)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k]["value"]) * scale[d[k]["unit"]]
        return tot
    except Exception:
        return None


def measure_int8_peak(torch, iters=10):
    """cuBLAS int8 dense GEMM (torch._int_mm) 8192^3, best of `iters` (burst)."""
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return 2.0 * n ** 3 / best / 1e12


def ours(args, rank, world, local_rank):
    import torch
    import paper_1112_5717_b200 as G

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wl = WORKLOADS[args.workload]
    m, n, p, seed = wl["m"], wl["n"], wl["p"], wl["seed"]
    L = limbs(p)
    stream = torch.cuda.current_stream()
    if args.workload == "c2":
        from paper_1112_5717_b200 import workloads as WL
        pristine = WL.c2_dev(m, n, wl["inner"], seed, p)
    else:
        pristine = torch.empty((m, n), dtype=torch.int32, device="cuda")
        G.random_matrix_dev(pristine, m, n, seed, p, stream=stream)
    work = torch.empty_like(pristine)

    # warm-up (also builds + captures the plan graph)
    for _ in range(args.warmup):
        work.copy_(pristine)
        G.cup_dev(work, m, n, p, stream=stream, sync=False)
    torch.cuda.synchronize()
    st = G.plan_stats(m, n, p)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            work.copy_(pristine)                    # restore input (outside the events)
            starts[i].record(stream)
            G.cup_dev(work, m, n, p, stream=stream, sync=False)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    elapsed = sum(s.elapsed_time(e) for s, e in zip(starts, ends)) / 1e3
    t_local = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max = float(t_local.item())

    # results of the last factorization + structural verification
    work.copy_(pristine)
    ctr = G.OpCounter()
    res = G.cup_dev(work, m, n, p, stream=stream, ctr=ctr)
    r = res.rank
    # config 2's rank profile is not generic: the model over-counts it, so its
    # algorithmic work is the reference's own counted arith_total
    W = float(ctr.arith_total()) if args.workload == "c2" else model_ops(m, n, r)
    value = world * W * args.steps / t_max
    ms_per_step = t_max / args.steps * 1e3

    # parity of the timed result: the body digest (device) and the row profile /
    # sigma / op counts against the committed CPU digests of this config
    # (tests/golden/scale_digests.json: reference + blocked restatement)
    parity = None
    try:
        want = json.load(open(os.path.join(ROOT, "tests", "golden", "scale_digests.json"))).get(args.workload)
        if want is not None:
            import hashlib

            def sha(x):
                return hashlib.sha256(np.ascontiguousarray(np.asarray(x, np.uint32)).tobytes()).hexdigest()
            got = {"rank": r, "rrp_sha256": sha(res.row_profile), "sigma_sha256": sha(res.col_perm),
                   "ops": [ctr.n_mul, ctr.n_addsub, ctr.n_divinv, ctr.n_ztest],
                   "body_digest": f"{G.digest_dev(work, m, n):016x}"}
            parity = {"bit_exact_vs_committed_digest": all(got[k] == want[k] for k in got),
                      "pinned_by": want.get("by"), "body_digest": got["body_digest"]}
    except Exception as e:  # pragma: no cover
        parity = {"error": str(e)}

    # the metric's second half: batched matrices/s (config 4), every rank
    batched = None
    if args.workload == "c3" and not args.no_batched:
        try:
            batched = batched_record(args, rank, world, dist, max(3, args.steps), max(3, args.warmup))
        except Exception as e:  # pragma: no cover
            batched = {"error": str(e)}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    line = {
        "metric": METRIC, "value": value, "unit": "mod-p ops/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": f"u32 in GF({p}); u8 limbs x{L} on int8 tensor cores (s32 acc, exact)",
        "data": "synthetic",
        "config": {"workload": args.workload, "desc": wl["desc"], "m": m, "n": n, "p": p,
                   "seed": seed, "rank": r, "model_ops": model_ops(m, n, r),
                   "algorithmic_ops": W, "counted_arith_ops": int(ctr.arith_total()),
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "input 1 GiB > 126 MB L2; input restored between steps",
                   "profile_identity": bool(np.array_equal(res.row_profile, np.arange(r))),
                   "sigma_identity": bool(np.array_equal(res.col_perm, np.arange(n)))},
        "gpu_launches": int(st["launches"]) * args.steps,
        "clocks": clk.summary(),
    }

    if parity is not None:
        line["parity"] = parity

    # dominant kernel roofline: root Schur GEMM shape, GEMM kernel alone
    try:
        cublas = measure_int8_peak(torch)
        peak, peak_source = cublas, "measured live: cuBLAS int8 dense GEMM 8192^3 (torch._int_mm), burst"
        try:  # the driver-measured peak: dense int8 = 2 x the measured bf16 rate (same tensor pipe)
            mp_ = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
            peak = 2.0 * float(mp_["bf16_tflops"])
            peak_source = ("MEASURED_PEAKS.json: 2 x bf16_tflops (%.1f, burst; int8 dense runs at twice "
                           "the bf16 rate on B200); live cuBLAS int8 beside it" % float(mp_["bf16_tflops"]))
        except Exception:
            pass
        gm = 8192  # the C3 root Schur GEMM shape (same as the committed ncu capture)
        da = torch.empty((gm, gm), dtype=torch.int32, device="cuda")
        db = torch.empty((gm, gm), dtype=torch.int32, device="cuda")
        dc = torch.empty((gm, gm), dtype=torch.int32, device="cuda")
        G.random_matrix_dev(da, gm, gm, 11, p)
        G.random_matrix_dev(db, gm, gm, 12, p)
        G.random_matrix_dev(dc, gm, gm, 13, p)
        ms_pack, ms_gemm = G.profile_gemm_dev(da, db, dc, gm, gm, gm, p, iters=5, stream=stream)
        tops = 2.0 * gm ** 3 * L * L / (ms_gemm / 1e3) / 1e12
        cup_int8 = W * L * L / (ms_per_step / 1e3) / 1e12
        line["roofline"] = {
            "bound": "tensor", "kernel": "gemm_tc_kernel<L=%d> (tcgen05.mma kind::i8)" % L,
            "achieved": tops, "peak": peak, "unit": "TFLOP/s",
            "unit_note": "int8 tensor TOPS; 1 mod-p MAC = L^2 u8 MACs",
            "frac": tops / peak,
            "peak_source": peak_source,
            "cublas_int8_live": cublas, "frac_vs_cublas": tops / cublas,
            "shape": [gm, gm, gm], "ms_gemm": ms_gemm, "ms_pack": ms_pack,
            "traffic": _ncu_traffic(),
            "traffic_note": "dram read+write bytes per launch of the same shape from one "
                            "ncu --set full capture (profiles/round2/gemm_8192_ncu.json); "
                            "algorithmic bytes 0.94e9",
            "cup_frac_of_peak": cup_int8 / peak,
            "cup_modp_peak": peak * 1e12 / (L * L),
        }
        del da, db, dc
    except Exception as e:  # pragma: no cover
        line["roofline"] = {"error": str(e)}

    # e2e through the C ABI with host buffers
    try:
        e2e_steps = max(1, min(args.steps, 3))
        host = torch.empty((m, n), dtype=torch.int32, pin_memory=True)
        src = pristine.cpu().numpy().view(np.uint32)
        hv = host.numpy().view(np.uint32)
        rrp = np.zeros(min(m, n), np.uint32)
        sig = np.zeros(n, np.uint32)
        tt = []
        for i in range(e2e_steps + 1):
            np.copyto(hv, src)
            rk = ctypes.c_int64(0)
            t0 = time.perf_counter()
            code = G.lib().rl_cup_u32(ctypes.c_void_p(hv.ctypes.data), m, n, n, p,
                                      ctypes.byref(rk), ctypes.c_void_p(rrp.ctypes.data),
                                      ctypes.c_void_p(sig.ctypes.data), None)
            dt = time.perf_counter() - t0
            if code != 0:
                raise RuntimeError(G.lib().rl_last_error().decode())
            if i > 0:
                tt.append(dt)
        e2e_t = sum(tt) / len(tt)
        line["e2e"] = {"value": world * W / e2e_t, "unit": "mod-p ops/s",
                       "h2d_bytes_per_step": m * n * 4,
                       "d2h_bytes_per_step": m * n * 4 + 8 + 4 * min(m, n) * 2 + 4 * n,
                       "ms_per_step": e2e_t * 1e3, "steps": len(tt),
                       "path": "rl_cup_u32 (host pinned buffers)"}
        del host
        # the same through PAGEABLE host memory -- what the C++ drop-in receives
        # from ranklab::Mat's std::vector (matrix.hpp:176): staged through the
        # library's pinned ring by host threads
        pg = np.empty((m, n), np.uint32)
        tp = []
        for i in range(e2e_steps + 1):
            np.copyto(pg, src)
            rk = ctypes.c_int64(0)
            t0 = time.perf_counter()
            code = G.lib().rl_cup_u32(ctypes.c_void_p(pg.ctypes.data), m, n, n, p,
                                      ctypes.byref(rk), ctypes.c_void_p(rrp.ctypes.data),
                                      ctypes.c_void_p(sig.ctypes.data), None)
            dt = time.perf_counter() - t0
            if code != 0:
                raise RuntimeError(G.lib().rl_last_error().decode())
            if i > 0:
                tp.append(dt)
        pt = sum(tp) / len(tp)
        line["e2e_pageable"] = {"value": world * W / pt, "unit": "mod-p ops/s", "ms_per_step": pt * 1e3,
                                "h2d_bytes_per_step": m * n * 4, "d2h_bytes_per_step": m * n * 4,
                                "steps": len(tp),
                                "path": "rl_cup_u32 (pageable host buffer: tile pipeline through two pinned rings filled/drained by host threads)"}
        del pg
    except Exception as e:  # pragma: no cover
        line["e2e"] = {"error": str(e)}

    # CPU baseline: the unmodified reference on a bounded sample, 1 thread
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            size = args.cpu_sample
            a = O.port_random_matrix(size, size, seed, p)
            t0 = time.perf_counter()
            rr = O.ref_cup(a, p) if O.have_ref() else O.port_cup(a, p)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {
                "value": model_ops(size, size, rr.rank) / dt, "unit": "mod-p ops/s", "cores": 1,
                "kind": "reference" if O.have_ref() else "port",
                "sample": f"ranklab::cup of random_matrix({size},{size},seed={seed},GF({p})), "
                          f"single thread, {dt:.1f} s"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)}
    if batched is not None:
        line["batched"] = batched
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def ours_dist(args, rank, world, local_rank):
    """One matrix distributed over the ranks by column tiles (dist.py)."""
    import torch
    import paper_1112_5717_b200 as G
    from paper_1112_5717_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wl = WORKLOADS[args.workload]
    m, n, p, seed = wl["m"], wl["n"], wl["p"], wl["seed"]
    tile, block = wl.get("tile", 1024), wl.get("block", 1024)
    sb = wl.get("superblock", 8192)
    tiles = D.ColumnTiles(n, world, tile)
    stream = torch.cuda.current_stream()
    pristine = D.random_matrix_local(m, n, seed, p, tiles, rank, "cuda")
    x = torch.empty_like(pristine)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        x.copy_(pristine)
        res = D.dist_cup(x, m, n, p, tiles, block=block, superblock=sb)
    barrier()
    times = []
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            x.copy_(pristine)                     # restore input (outside the events)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = D.dist_cup(x, m, n, p, tiles, block=block, superblock=sb)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        barrier()
    t_local = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_max = float(t_local.item())
    r = res.rank
    W = model_ops(m, n, r)
    # launches: the row-block CUP plans (graph-replayed) + per-step trsm/GEMM/copies
    launches = 0
    i0, rr = 0, 0
    quantum = D._roundup(D._roundup(n, 12) // 12, 64)
    while i0 < m and rr < n:
        bt = min(block, m - i0)
        wp = min(n, D._roundup(n - rr, quantum))
        launches += int(G.plan_stats(bt, wp, p)["launches"]) + 4
        i0 += bt
        rr += bt
    # e2e: this rank's columns from pinned host memory, factor, back to the host
    e2e = None
    try:
        host = torch.empty(pristine.shape, dtype=torch.int32, pin_memory=True)
        host.copy_(pristine)
        barrier()
        t0 = time.perf_counter()
        x.copy_(host, non_blocking=True)
        D.dist_cup(x, m, n, p, tiles, block=block, superblock=sb)
        host.copy_(x, non_blocking=True)
        barrier()
        et = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": W / float(et.item()), "unit": "mod-p ops/s",
               "h2d_bytes_per_step": m * n * 4, "d2h_bytes_per_step": m * n * 4,
               "ms_per_step": float(et.item()) * 1e3, "steps": 1,
               "path": "pinned host columns -> dist_cup (every rank) -> host; max over ranks"}
        del host
    except Exception as e:  # pragma: no cover
        e2e = {"error": str(e)}
    if rank == 0:
        L = limbs(p)
        line = {
            "metric": METRIC, "value": W * args.steps / t_max, "unit": "mod-p ops/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": f"u32 in GF({p}); u8 limbs x{L} on int8 tensor cores (s32 acc, exact)",
            "data": "synthetic",
            "config": {"workload": args.workload, "desc": wl["desc"], "m": m, "n": n, "p": p,
                       "seed": seed, "rank": r, "model_ops": W, "tile": tile, "block": block,
                       "superblock": sb,
                       "row_blocks": res.steps,
                       "parallelism": f"1D block-cyclic column tiles over {world} rank(s)",
                       "l2": "input 17 GB > 126 MB L2; input restored between steps",
                       "profile_identity": bool(np.array_equal(res.row_profile, np.arange(r))),
                       "sigma_identity": bool(np.array_equal(res.col_perm, np.arange(n)))},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def batched_record(args, rank, world, dist, steps, warmup):
    """Config 4 -- the metric's second half ("batched matrices/s"): the fixed
    batch of 4096 matrices sharded across ranks (contiguous slices, no
    collective on the data path).  Returns the line (rank 0) or None."""
    import torch
    import paper_1112_5717_b200 as G
    from paper_1112_5717_b200 import workloads as WL

    wl = WORKLOADS["c4"]
    total, m, n, p, seed = wl["batch"], wl["m"], wl["n"], wl["p"], wl["seed"]
    lo, hi = WL.shard_range(total, rank, world)
    cnt = hi - lo
    stream = torch.cuda.current_stream()
    pristine, ranks = WL.c4_dev(total, seed, p, lo, hi)
    work = torch.empty_like(pristine)
    for _ in range(warmup):
        work.copy_(pristine)
        G.cup_batched_dev(work, cnt, m, n, p, stream=stream, want_meta=False)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clk:
        for i in range(steps):
            work.copy_(pristine)
            starts[i].record(stream)
            G.cup_batched_dev(work, cnt, m, n, p, stream=stream, want_meta=False)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    elapsed = sum(s_.elapsed_time(e) for s_, e in zip(starts, ends)) / 1e3
    t_local = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    # verification: ranks equal the recipe's r_t and every body digest equals the
    # reference's (tests/golden/scale_digests.json, pinned by tools/pin_scale_digests.py)
    work.copy_(pristine)
    rk, _, _ = G.cup_batched_dev(work, cnt, m, n, p, stream=stream)
    ok = torch.tensor([int(sum(int(a) == b for a, b in zip(rk, ranks)))], dtype=torch.float64,
                      device="cuda")
    dig_ok = -1
    try:
        want = json.load(open(os.path.join(ROOT, "tests", "golden", "scale_digests.json")))["c4"]
        dig_ok = int(all(f"{G.digest_dev(work[t], m, n):016x}" == want["body_digests"][lo + t]
                         for t in range(cnt)))
    except Exception:
        pass
    dig = torch.tensor([dig_ok], dtype=torch.float64, device="cuda")
    ops = torch.tensor([sum(model_ops(m, n, int(x)) for x in rk)], dtype=torch.float64,
                       device="cuda")
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        dist.all_reduce(ok, op=dist.ReduceOp.SUM)
        dist.all_reduce(dig, op=dist.ReduceOp.MIN)
        dist.all_reduce(ops, op=dist.ReduceOp.SUM)
    t_max = float(t_local.item())
    if rank != 0:
        return None
    value = total * steps / t_max
    line = {
        "metric": METRIC, "value": value, "unit": "matrices/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": t_max / steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": f"u32 in GF({p}); panel: lazy u64 sums, 32-bit Barrett; trailing updates: f64 DMMA (exact, < 2^52)", "data": "synthetic",
        "config": {"workload": "c4", "desc": wl["desc"], "batch": total, "m": m, "n": n, "p": p,
                   "seed": seed, "parallelism": f"batch sharded {world} ways" if world > 1 else "single",
                   "ranks_match_recipe": int(ok.item()),
                   "bodies_match_reference_digests": bool(dig.item() == 1) if dig.item() >= 0 else None,
                   "modp_ops_per_s": float(ops.item()) * steps / t_max,
                   "l2": "256 MB batch > 126 MB L2; batch restored between steps"},
        "gpu_launches": steps,
        "clocks": clk.summary(),
    }
    # e2e: host buffers in, factor, bodies + ranks out (this rank's shard), through
    # the host-buffer C ABI (rl_cup_batched_u32: chunked H2D / factor / D2H overlap)
    try:
        host = torch.empty(pristine.shape, dtype=torch.int32, pin_memory=True)
        src = pristine.cpu()
        hv = host.numpy().view(np.uint32).reshape(cnt, m, n)
        tt = []
        for i in range(4):
            host.copy_(src)                       # restore the inputs (outside the timing)
            t0 = time.perf_counter()
            G.cup_batched(hv, p)                  # ranks, profiles, sigma + bodies back
            tt.append(time.perf_counter() - t0)
        e2e_t = sum(tt[1:]) / len(tt[1:])
        line["e2e"] = {"value": cnt * world / e2e_t, "unit": "matrices/s",
                       "h2d_bytes_per_step": cnt * m * n * 4,
                       "d2h_bytes_per_step": cnt * (m * n * 4 + 8 + 4 * min(m, n) + 4 * n),
                       "ms_per_step": e2e_t * 1e3,
                       "path": "rl_cup_batched_u32 (pinned host matrices; chunked H2D, factor, "
                               "D2H on three streams)"}
    except Exception as e:  # pragma: no cover
        line["e2e"] = {"error": str(e)}
    if world == 1 and not args.no_cpu_baseline:
        try:
            import oracle as O
            from tests.helpers import matmul_mod
            ranks_h, ls, rs = WL.c4_recipe(8, seed)
            t_sum = 0.0
            for t in range(8):
                a = matmul_mod(O.port_random_matrix(256, ranks_h[t], ls[t], p),
                               O.port_random_matrix(ranks_h[t], 256, rs[t], p), p)
                t0 = time.perf_counter()
                (O.ref_cup if O.have_ref() else O.port_cup)(a, p)
                t_sum += time.perf_counter() - t0
            line["cpu_baseline"] = {"value": 8 / t_sum, "unit": "matrices/s", "cores": 1,
                                    "kind": "reference" if O.have_ref() else "port",
                                    "sample": "ranklab::cup of the first 8 config-4 matrices, "
                                              f"single thread, {t_sum:.2f} s"}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(e)}
    return line


def ours_batched(args, rank, world, local_rank):
    """Config 4 alone (--workload c4)."""
    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = batched_record(args, rank, world, dist, args.steps, args.warmup)
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--cpu-sample", type=int, default=2048)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batched", action="store_true",
                    help="c3: skip the config-4 'batched matrices/s' sub-record")
    ap.add_argument("--dist", action="store_true",
                    help="single-matrix workloads: the distributed column-tile driver even at N=1")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
    elif args.workload == "c4":
        ours_batched(args, rank, world, local_rank)
    elif args.dist or (args.workload == "c5" and world > 1):
        ours_dist(args, rank, world, local_rank)
    else:
        ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
