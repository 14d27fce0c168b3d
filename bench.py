#!/usr/bin/env python3
"""bench.py -- GCUPS of the B200-native LCS table fill (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], "C2"): a batch of 65,536
independent protein-like pairs (20-letter alphabet, lengths uniform in
[200, 1000], i.i.d. symbols; synthetic, seeded std::mt19937_64 -- the
procedure of wlcs_generate_pairs / oracle orc_generate_pairs).  One "step" =
one pass of the fill over the whole batch (LCS length of every pair).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
                  [--config c2|c1|c3|c4|c5] [--no-single-pairs]

N > 1: one process per GPU (torchrun; `--gpus N` without WORLD_SIZE re-launches
itself under torch.distributed.run).  The SAME 65,536-pair batch is sharded
across the ranks (contiguous pair ranges balanced by cells; no data-path
collective; "scaling": "strong"); the timed region is bracketed by barrier +
cuda synchronize, the max over ranks is reported by rank 0.

`value`   : algorithmic cells (sum m_k * n_k, no padding) / device time of
            the K steps, inputs resident in HBM, L2 flushed between steps
            (300 MB write, outside the timed events).  CUDA events on the
            launching stream (the library's kernels run on that stream).
`e2e`     : same metric through the public C-ABI (wlcs_length_batch) from
            pinned host buffers: H2D of strings + offsets and D2H of the
            lengths inside the timed region (wall clock per step).
`roofline`: the dominant kernel (batch_main_kernel) against the integer
            ALU-pipe peak measured live (wlcs_probe_int_peak, LOP3 stream):
            achieved = cells * 3/32 int-ops / kernel time.
`cpu_baseline`: the UNMODIFIED reference (oracle/_ref, compiled from
            /root/reference sources) on a bounded sample of the same batch on
            all host cores; its lengths double as the equivalence gate
            (reference proj/src/bench.cpp:100-106).
`c4`, `c5`: the 1e12-cell single pairs (BASELINE configs[3], [4]), length
            only: device fill time (CUDA events around the strip kernel),
            end-to-end wall time through the C-ABI, roofline, and the golden
            length check.  At N > 1, C4 runs as the column split across the
            ranks (carries over NVLink inside the fill).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GCUPS (LCS cell updates/s)"
UNIT = "GCUPS"
PROTEIN = b"ACDEFGHIKLMNPQRSTVWY"
DNA = b"ACGT"
CHILD_SEED_OFFSET = 0x9E3779B97F4A7C15  # proj/include/wavelcs/bench.hpp:74
L2_FLUSH_BYTES = 300 * 1024 * 1024       # > 126 MB L2
SEED = 20130619
# one workload description for BOTH arms (the driver compares them)
C2_CONFIG = {"workload": "C2: 65536 protein-like pairs, 20-letter alphabet, lengths U[200,1000], "
                         "LCS length per pair",
             "global_batch": 65536, "seq_len": "200-1000", "alphabet": 20, "seed": SEED,
             "generator": "master std::mt19937_64(seed): m, n = 200 + r % 801, per-string "
                          "seeds, generate_random (proj/src/io.cpp:103-115)"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["c2", "c1", "c3", "c4", "c5"], default="c2")
    ap.add_argument("--pairs", type=int, default=65536)
    ap.add_argument("--seed", type=int, default=SEED)
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU work of the bounded reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-single-pairs", action="store_true",
                    help="c2: skip the c4 / c5 blocks of the JSON line")
    ap.add_argument("--colsplit", action="store_true",
                    help="c4/c5: use the multi-GPU column-split path even on one GPU")
    ap.add_argument("--variant", choices=["bitparallel", "wavefront"], default="bitparallel",
                    help="fill kernel variant (WLCS_VARIANT_*)")
    ap.add_argument("--dry-run", action="store_true",
                    help="c2: ranks, generation and sharding only (no device work; CPU tests)")
    return ap.parse_args()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-launch under torch.distributed.run
    with N ranks (one per GPU).  Returns the exit code, or None when this
    process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if (os.environ.get("WLCS_BENCH_ONE_DEVICE") != "1" and args.impl == "b200"
            and not args.dry_run):
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} "
                              "CUDA devices are visible"}), flush=True)
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------- plumbing
class Dist:
    """One process per GPU (torchrun).  NCCL by default; WLCS_DIST_BACKEND=gloo
    and WLCS_BENCH_ONE_DEVICE=1 exist only to exercise the N > 1 host logic
    on a single-GPU box or on the CPU (independent shards, no kernel waits on
    another rank)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        one_device = os.environ.get("WLCS_BENCH_ONE_DEVICE") == "1"
        if one_device:
            self.local_rank = 0
        # NCCL refuses two ranks on one GPU: the one-device mode defaults to gloo
        self.backend = os.environ.get("WLCS_DIST_BACKEND", "gloo" if one_device else "nccl")
        self.pg = None

    def init(self):
        import torch.distributed as dist
        if self.world > 1 and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(self.backend)
            self.pg = dist
        return self

    def barrier(self):
        if self.pg is not None:
            self.pg.barrier()

    def _reduce(self, v: float, op) -> float:
        import torch
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, v: float) -> float:
        return v if self.pg is None else self._reduce(v, self.pg.ReduceOp.MAX)

    def sum(self, v: float) -> float:
        return v if self.pg is None else self._reduce(v, self.pg.ReduceOp.SUM)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if not self.path or not os.path.exists(self.path):
            return out
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return out
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for _, _, flags in rows:
            for n, f in zip(names, flags):
                if f.lower().startswith("active"):
                    reasons.add(n)
        loaded = [r[0] for r in rows if r[0] > 500] or [r[0] for r in rows]
        out.update(sm_mhz=float(np.median(loaded)), sm_max_mhz=max(r[1] for r in rows),
                   reasons=sorted(reasons), samples=len(rows))
        return out


def cells_of(xo, yo) -> int:
    m = np.diff(np.asarray(xo).astype(np.int64))
    n = np.diff(np.asarray(yo).astype(np.int64))
    return int(np.sum(m * n))


def shard_range(xo, yo, world: int, rank: int) -> tuple[int, int]:
    """Contiguous pair range of `rank`, balanced by cells (the same rule as
    paper_1306_4627_b200.multigpu.shard_pairs / wlcs_length_batch_multi)."""
    m = np.diff(np.asarray(xo, dtype=np.int64))
    n = np.diff(np.asarray(yo, dtype=np.int64))
    pairs = len(m)
    cum = np.concatenate([[0], np.cumsum(m * n + 1)])
    total = cum[-1]
    lo = int(np.searchsorted(cum, total * rank / world, side="left"))
    hi = pairs if rank == world - 1 else int(np.searchsorted(cum, total * (rank + 1) / world,
                                                             side="left"))
    return min(lo, pairs), min(hi, pairs)


# --------------------------------------------------------- reference (CPU)
def reference_sample(ref, xs, xo, ys, yo, target_s: float, threads: int):
    """Bounded sample of the batch sized to ~target_s of reference CPU time."""
    probe = min(256, len(xo) - 1)
    _, sec = ref.batch_lengths(xs, xo[: probe + 1], ys, yo[: probe + 1], threads)
    rate = cells_of(xo[: probe + 1], yo[: probe + 1]) / max(sec, 1e-6)
    want = rate * target_s
    cum = np.cumsum(np.diff(xo.astype(np.int64)) * np.diff(yo.astype(np.int64)))
    k = int(np.searchsorted(cum, want)) + 1
    return max(probe, min(k, len(xo) - 1))


def run_reference_arm(args, dist):
    """The reference's own CPU path (oracle/_ref: the unmodified reference
    compiled from its sources) -- this process never loads the B200 library:
    its inputs come from the oracle's restatement of the same generator."""
    if dist.rank != 0:
        return 0
    import oracle
    if args.config != "c2":
        print(json.dumps({"impl": "reference", "unavailable":
                          "reference arm implemented for the bench workload c2 only"}))
        return 0
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    xs, xo, ys, yo = oracle.Restatement().generate_pairs(args.pairs, 200, 1000, PROTEIN, args.seed)
    k = reference_sample(ref, xs, xo, ys, yo, min(args.cpu_seconds, 4.0), threads)
    sxo, syo = xo[: k + 1], yo[: k + 1]
    cells = cells_of(sxo, syo)
    for _ in range(args.warmup):
        ref.batch_lengths(xs, sxo, ys, syo, threads)
    times = []
    for _ in range(args.steps):
        _, sec = ref.batch_lengths(xs, sxo, ys, syo, threads)
        times.append(sec)
    total = float(np.sum(times))
    value = cells * args.steps / total / 1e9
    sample = (f"first {k} of {args.pairs} C2 pairs ({cells / 1e9:.3f} G cells) per step, "
              f"lcs_fill_parallel(workers=1) per pair on a {threads}-thread pool")
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded std::mt19937_64)", "impl": "reference",
        "config": dict(C2_CONFIG),
        "parallelism": f"cpu threads x{threads}",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- B200 arm
def gen_pairs_pinned(wl, pairs: int, lo: int, hi: int, alphabet: bytes, seed: int):
    """C2 generator (wlcs_generate_pairs) into page-locked host memory."""
    cap = pairs * hi

    def alloc(n, dtype):
        nbytes = n * np.dtype(dtype).itemsize
        p = wl.lib.wlcs_host_alloc(nbytes)
        if not p:
            raise MemoryError("wlcs_host_alloc")
        return np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(p)).view(dtype)
    xs, ys = alloc(cap, np.uint8), alloc(cap, np.uint8)
    xo, yo = alloc(pairs + 1, np.uint64), alloc(pairs + 1, np.uint64)
    a = np.frombuffer(alphabet, np.uint8)
    rc = wl.lib.wlcs_generate_pairs(ctypes.c_size_t(pairs), ctypes.c_size_t(lo),
                                    ctypes.c_size_t(hi), a.ctypes.data, ctypes.c_size_t(len(a)),
                                    ctypes.c_uint64(seed), xs.ctypes.data,
                                    xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                    ys.ctypes.data,
                                    yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    wl._check(rc)
    return xs, xo, ys, yo


def pinned_copy(wl, arr: np.ndarray) -> np.ndarray:
    nbytes = max(1, arr.nbytes)
    p = wl.lib.wlcs_host_alloc(nbytes)
    if not p:
        raise MemoryError("wlcs_host_alloc")
    out = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(p)).view(arr.dtype)
    out = out[: arr.size]
    out[:] = arr
    return out


def run_c2_dry(args, dist):
    """The N-rank host logic of run_c2 without device work: every rank builds
    the batch, takes its shard, and the totals are reduced over the group."""
    import paper_1306_4627_b200 as wl  # host-only entry point (no device needed)
    P = args.pairs
    xs, ys = np.empty(P * 1000, np.uint8), np.empty(P * 1000, np.uint8)
    xo, yo = np.empty(P + 1, np.uint64), np.empty(P + 1, np.uint64)
    a = np.frombuffer(PROTEIN, np.uint8)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    wl._check(wl.lib.wlcs_generate_pairs(ctypes.c_size_t(P), ctypes.c_size_t(200),
                                         ctypes.c_size_t(1000), a.ctypes.data,
                                         ctypes.c_size_t(len(a)), ctypes.c_uint64(args.seed),
                                         xs.ctypes.data, xo.ctypes.data_as(u64p), ys.ctypes.data,
                                         yo.ctypes.data_as(u64p)))
    p0, p1 = shard_range(xo, yo, dist.world, dist.rank)
    cells = cells_of(xo[p0:p1 + 1], yo[p0:p1 + 1])
    return {"metric": METRIC, "dry_run": True, "n_gpus": dist.world, "scaling": "strong",
            "config": dict(C2_CONFIG), "pairs_total": int(dist.sum(float(p1 - p0))),
            "cells_total": int(dist.sum(float(cells))), "cells_batch": cells_of(xo, yo),
            "max_rank_cells": int(dist.max(float(cells)))}


def run_c2(args, dist):
    import torch
    import paper_1306_4627_b200 as wl
    dev = torch.device("cuda", dist.local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    # the whole batch on every rank (deterministic), then this rank's shard
    axs, axo, ays, ayo = gen_pairs_pinned(wl, args.pairs, 200, 1000, PROTEIN, args.seed)
    total_cells = cells_of(axo, ayo)
    p0, p1 = shard_range(axo, ayo, dist.world, dist.rank)
    npairs = p1 - p0
    xa, xb = int(axo[p0]), int(axo[p1])
    ya, yb = int(ayo[p0]), int(ayo[p1])
    xs = pinned_copy(wl, axs[xa:xb])
    ys = pinned_copy(wl, ays[ya:yb])
    xo = pinned_copy(wl, (axo[p0:p1 + 1] - axo[p0]).astype(np.uint64))
    yo = pinned_copy(wl, (ayo[p0:p1 + 1] - ayo[p0]).astype(np.uint64))
    xs_bytes, ys_bytes = xb - xa, yb - ya
    cells = cells_of(xo, yo)
    d_xs = torch.from_numpy(np.concatenate([xs, np.zeros(16, np.uint8)])).to(dev)
    d_ys = torch.from_numpy(np.concatenate([ys, np.zeros(16, np.uint8)])).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(max(1, npairs), dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    variant = wl.VARIANT_WAVEFRONT if args.variant == "wavefront" else wl.VARIANT_BITPARALLEL

    def step():
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(),
                                   d_yo.data_ptr(), npairs, xs_bytes, ys_bytes,
                                   d_out.data_ptr(), stream.cuda_stream, variant=variant)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    # pass 1: the step exactly as a user runs it (PDL overlap between the
    # batch kernels intact); pass 2 (instrumented, separate): the main
    # kernel's own CUDA-event duration for the roofline
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(dist.local_rank) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    gpu_lengths = d_out[:npairs].cpu().numpy().astype(np.uint32)
    wl._check(wl.lib.wlcs_set_timing(1))
    main_ms = []
    km = ctypes.c_float()
    for _ in range(args.steps):
        flush.zero_()
        step()
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        main_ms.append(km.value)
    torch.cuda.synchronize()
    wl._check(wl.lib.wlcs_set_timing(0))
    total_ms = dist.max(float(np.sum(step_ms)))
    all_cells = dist.sum(float(cells))
    assert int(all_cells) == total_cells, "shards do not cover the batch"
    value = all_cells * args.steps / (total_ms * 1e-3) / 1e9

    # e2e through the public host API (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        out = np.zeros(max(1, npairs), np.uint32)
        outp = out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        xop = xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        yop = yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))

        def e2e_step():
            wl._check(wl.lib.wlcs_length_batch_ex(xs.ctypes.data, xop, ys.ctypes.data, yop,
                                                  npairs, variant, outp))
        e2e_step()
        dist.barrier()
        wall = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_step()
            wall.append(time.perf_counter() - t0)
        dist.barrier()
        e2e_total = dist.max(float(np.sum(wall)))
        if not np.array_equal(out[:npairs], gpu_lengths):
            raise AssertionError("e2e lengths differ from the device-resident run")
        e2e = {"value": round(all_cells * args.steps / e2e_total / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(dist.sum(float(xs_bytes + ys_bytes + 16 * (npairs + 1)))),
               "d2h_bytes_per_step": int(dist.sum(float(4 * npairs))),
               "ms_per_step": round(1e3 * e2e_total / args.steps, 4)}

    peak = ctypes.c_double()
    wl._check(wl.lib.wlcs_probe_int_peak(5, ctypes.byref(peak)))
    kernel_ms = float(np.mean(main_ms))
    wave = variant == wl.VARIANT_WAVEFRONT
    # algorithmic int ops: bit-parallel 3 per 32-cell word-row; cell wavefront
    # 3 per PAIR of 16x2-packed cells (LOP3 match, IADD3 diag+1-d, VIMNMX3.U16x2)
    alg_ops = cells * 1.5 if wave else cells * 3.0 / 32.0
    achieved = alg_ops / (kernel_ms * 1e-3) / 1e12
    peak_t = peak.value / 1e12
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded std::mt19937_64, wlcs_generate_pairs)",
        "config": dict(C2_CONFIG),
        "parallelism": f"65536 pairs sharded over {dist.world} GPU(s) by cells (no collective)",
        "cells_per_step": total_cells, "pairs_this_rank": npairs,
        "l2": "flushed between steps (300 MB write, outside the timed events)",
        # bit-parallel: plan, scatter (with the bucket scan), main, second-pass
        # planner, second pass (empty here: it reads its count on the device);
        # the workspace memset is a driver memset, not counted; wavefront: one kernel
        "gpu_launches": (1 if wave else 5) * args.steps,
        "variant": args.variant,
        "roofline": {"bound": "int", "achieved": round(achieved, 3), "peak": round(peak_t, 3),
                     "unit": "Tops/s (int32 ALU, 3 ops per 2 packed cells)" if wave else
                             "Tops/s (int32 ALU, 3 ops per 32-cell word-row)",
                     # the committed ncu capture is of the whole 65,536-pair batch
                     # on one GPU: a shard's traffic is not known from it
                     "frac": round(achieved / peak_t, 4), "traffic": ncu_traffic(
                         "wave_batch_kernel" if wave else "batch_main_kernel")
                     if dist.world == 1 and npairs == 65536 else None,
                     "algorithmic_bytes": int(xs_bytes + ys_bytes + 16 * (npairs + 1)
                                              + 4 * npairs),
                     "kernel": "wave_batch_kernel" if wave else "batch_main_kernel",
                     "kernel_ms": round(kernel_ms, 4),
                     "kernel_share_of_step": round(kernel_ms / (total_ms / args.steps), 3),
                     "peak_source": "measured live: wlcs_probe_int_peak (LOP3 stream); "
                                    "MEASURED_PEAKS.json has no integer peak",
                     "gcups_ceiling": round(peak.value * (2 if wave else 32) / 3 / 1e9, 1)},
        "clocks": clocks.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_c2(args, axs, axo, ays, ayo, gpu_lengths)
    return line


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[kernel]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def cpu_baseline_c2(args, xs, xo, ys, yo, gpu_lengths):
    import oracle
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    k = reference_sample(ref, xs, xo, ys, yo, args.cpu_seconds, threads)
    lens, sec = ref.batch_lengths(xs, xo[: k + 1], ys, yo[: k + 1], threads)
    if not np.array_equal(lens, gpu_lengths[:k]):
        bad = int(np.nonzero(lens != gpu_lengths[:k])[0][0])
        # EquivalenceError semantics of proj/src/bench.cpp:100-106
        raise AssertionError(f"EquivalenceError: pair {bad}: reference {lens[bad]} "
                             f"vs GPU {gpu_lengths[bad]}")
    cells = cells_of(xo[: k + 1], yo[: k + 1])
    return {"value": round(cells / sec / 1e9, 4), "unit": UNIT, "cores": threads,
            "kind": "reference",
            "sample": f"first {k} of {args.pairs} C2 pairs ({cells / 1e9:.3f} G cells), "
                      f"lcs_fill_parallel(workers=1) per pair on a {threads}-thread pool; "
                      f"lengths identical to the GPU's (equivalence gate)"}


def golden_length(name):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "large_configs.json")) as f:
            return json.load(f)[name]["lcs_length"]
    except (OSError, KeyError, ValueError):
        return None


def subsequence_pair_block(name, steps, warmup, peak_ops):
    """C1 / C3 at full size, length + recovered subsequence through
    lcs_subsequence (one GPU): e2e = wall time of the whole C-ABI call (H2D,
    fill storing the bit rows, parallel traceback, D2H); fill = CUDA events
    around the strip kernel.  The string is checked against the reference's
    own traceback (sha256 in tests/golden/{c1.json, c3.json.gz})."""
    import gzip
    import hashlib
    import paper_1306_4627_b200 as wl
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair(name)
    cells = len(x) * len(y)
    fn = lambda: wl.lcs_subsequence(x, y, wl.NO_BUDGET)  # noqa: E731
    for _ in range(warmup):
        sub = fn()
    wl._check(wl.lib.wlcs_set_timing(1))
    km = ctypes.c_float()
    times, fills = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        sub = fn()
        times.append(time.perf_counter() - t0)
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        fills.append(km.value)
    wl._check(wl.lib.wlcs_set_timing(0))
    fill_ms, wall_s = float(np.mean(fills)), float(np.mean(times))
    try:
        path = os.path.join(ROOT, "tests", "golden", "c1.json" if name == "c1" else "c3.json.gz")
        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rt") as f:
            want = json.load(f)["sha256"]
    except (OSError, KeyError, ValueError):
        want = None
    got = hashlib.sha256(sub).hexdigest()
    if want is not None and got != want:
        raise AssertionError(f"EquivalenceError: {name} subsequence differs from the reference's")
    achieved = cells * 3.0 / 32.0 / (fill_ms * 1e-3) / 1e12 if fill_ms > 0 else 0.0
    return {"workload": {"c1": "C1: 10k x 10k DNA, length + subsequence",
                         "c3": "C3: 100k x ~100k mutated DNA, length + subsequence"}[name],
            "m": len(x), "n": len(y), "lcs_length": len(sub),
            "golden_match": want is not None and got == want,
            "n_gpus": 1, "fill_ms": round(fill_ms, 3),
            "value": round(cells / wall_s / 1e9, 1), "unit": UNIT,
            "e2e": {"value": round(cells / wall_s / 1e9, 1), "unit": UNIT,
                    "ms_per_step": round(wall_s * 1e3, 3),
                    "ms_median": round(float(np.median(times)) * 1e3, 3),
                    "h2d_bytes_per_step": len(x) + len(y), "d2h_bytes_per_step": len(sub) + 8},
            "roofline": {"bound": "int (latency: one row chain)", "achieved": round(achieved, 3),
                         "peak": round(peak_ops / 1e12, 3), "unit": "Tops/s",
                         "frac": round(achieved / (peak_ops / 1e12), 4),
                         "kernel": "pair_strip_kernel (bit rows stored) + walk",
                         # the bound that applies: every row depends on the one
                         # above; 3 dependent ALU ops x ~4.7 cycles per row
                         # (tools/micro/dpx_latency.cu) at the max SM clock
                         "critical_path_ms": round(len(x) * 14.0 / 1.965e6, 3),
                         "frac_of_critical_path": round(len(x) * 14.0 / 1.965e6 / fill_ms, 3)
                         if fill_ms > 0 else None},
            "steps": steps}


def single_pair_block(name, steps, warmup, dist, peak_ops):
    """C4 / C5 at full size, length only (N = 1: one GPU; N > 1: C4's column
    split across the ranks).  Device fill time from CUDA events around the
    strip kernel(s); e2e = wall time of the whole C-ABI call (H2D of the
    strings, alphabet + masks, fill, combine, D2H)."""
    import paper_1306_4627_b200 as wl
    from paper_1306_4627_b200 import workloads
    x, y = workloads.config_pair(name)
    cells = len(x) * len(y)
    colsplit = dist.world > 1 and name == "c4"
    times = []
    if colsplit:
        fill_ms, wall_s, length = colsplit_steps(wl, x, y, steps, warmup, dist)
    else:
        fn = lambda: wl.lcs_length(x, y, wl.NO_BUDGET)  # noqa: E731
        for _ in range(warmup):
            length = fn()
        wl._check(wl.lib.wlcs_set_timing(1))
        km = ctypes.c_float()
        times, fills = [], []
        for _ in range(steps):
            t0 = time.perf_counter()
            length = fn()
            times.append(time.perf_counter() - t0)
            wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
            fills.append(km.value)
        wl._check(wl.lib.wlcs_set_timing(0))
        fill_ms, wall_s = float(np.mean(fills)), float(np.mean(times))
    want = golden_length(name)
    if want is not None and length != want:
        raise AssertionError(f"EquivalenceError: {name} length {length} != golden {want}")
    achieved = cells * 3.0 / 32.0 / (fill_ms * 1e-3) / 1e12
    return {"workload": {"c4": "C4: 1M x 1M i.i.d. DNA, length only",
                         "c5": "C5: 2M x 500k Zipf(1.1) bytes, length only"}[name],
            "m": len(x), "n": len(y), "lcs_length": length, "golden_match": want == length,
            "n_gpus": dist.world if colsplit else 1,
            "parallelism": (f"column split over {dist.world} GPUs, carries over NVLink inside "
                            "the fill" if colsplit else "one GPU, bidirectional split"),
            "fill_ms": round(fill_ms, 3), "value": round(cells / (fill_ms * 1e-3) / 1e9, 1),
            "unit": UNIT,
            "e2e": {"value": round(cells / wall_s / 1e9, 1), "unit": UNIT,
                    "ms_per_step": round(wall_s * 1e3, 3),
                    "ms_median": round(float(np.median(times)) * 1e3, 3) if times else None,
                    "h2d_bytes_per_step": len(x) + len(y), "d2h_bytes_per_step": 8},
            "roofline": {"bound": "int", "achieved": round(achieved, 3),
                         "peak": round(peak_ops / 1e12, 3), "unit": "Tops/s",
                         "frac": round(achieved / (peak_ops / 1e12), 4),
                         "kernel": "pair_strip_kernel",
                         "traffic": ncu_traffic(f"pair_strip_kernel_{name}"),
                         "algorithmic_bytes": len(x) + len(y)},
            "steps": steps}


def colsplit_steps(wl, x, y, steps, warmup, dist):
    """C4 column split across the ranks (IPC inboxes; see run_colsplit)."""
    import torch
    import torch.distributed as tdist
    from paper_1306_4627_b200 import multigpu
    dev = torch.device("cuda", dist.local_rank)
    rows, cols = (x, y) if len(x) <= len(y) else (y, x)
    G, g = dist.world, dist.rank
    lo, hi = multigpu.colsplit_bounds(len(cols), G)[g]
    words = wl.colsplit_inbox_words(len(rows))
    in_f, in_r = wl.device_alloc(4 * words), wl.device_alloc(4 * words)
    handles = [(None, None)] * G
    tdist.all_gather_object(handles, (wl.ipc_handle(in_f), wl.ipc_handle(in_r)))
    out_f = wl.ipc_open(handles[g + 1][0]) if g + 1 < G else 0
    out_r = wl.ipc_open(handles[g - 1][1]) if g > 0 else 0

    def step():
        wl.device_zero(in_f, 4 * words)
        wl.device_zero(in_r, 4 * words)
        torch.cuda.synchronize()
        dist.barrier()
        vf, vr = wl.colsplit_fill(rows, cols, lo, hi, wl.COLSPLIT_FORWARD | wl.COLSPLIT_REVERSE,
                                  in_fwd=in_f if g > 0 else 0, out_fwd=out_f,
                                  in_rev=in_r if g + 1 < G else 0, out_rev=out_r)
        return multigpu.colsplit_combine_dist(lo, hi, vf, vr, tdist,
                                              device=dev if dist.backend == "nccl" else None)
    for _ in range(warmup):
        length = step()
    wl._check(wl.lib.wlcs_set_timing(1))
    km = ctypes.c_float()
    wall, fill = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        length = step()
        wall.append(time.perf_counter() - t0)
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        fill.append(km.value)
    wl._check(wl.lib.wlcs_set_timing(0))
    if out_f:
        wl.ipc_close(out_f)
    if out_r:
        wl.ipc_close(out_r)
    return dist.max(float(np.mean(fill))), dist.max(float(np.mean(wall))), length


def run_colsplit(args, dist):
    """C4/C5 on N GPUs: one long pair, column slice per rank (strong scaling)."""
    import torch
    import paper_1306_4627_b200 as wl
    from paper_1306_4627_b200 import workloads
    torch.cuda.set_device(dist.local_rank)
    x, y = workloads.config_pair(args.config, args.seed)
    with ClockSampler(dist.local_rank) as clocks:
        fill_ms, wall_s, length = colsplit_steps(wl, x, y, args.steps, args.warmup, dist)
    cells = len(x) * len(y)
    return {"metric": METRIC, "value": round(cells / (fill_ms * 1e-3) / 1e9, 3), "unit": UNIT,
            "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(fill_ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (workloads.py)",
            "config": {"workload": f"{args.config.upper()} single pair, column split x{dist.world}",
                       "lcs_length": length, "m": len(x), "n": len(y)},
            "parallelism": f"column slices x{dist.world}, carries over NVLink P2P (IPC)",
            "e2e": {"value": round(cells / wall_s / 1e9, 3), "unit": UNIT,
                    "h2d_bytes_per_step": len(x) + len(y), "d2h_bytes_per_step": 0},
            "gpu_launches": None, "clocks": clocks.summary(),
            "note": "value: device fill time (CUDA events, max over ranks); e2e: wall time "
                    "incl. inbox reset, barrier, H2D, fill and the distributed combine"}


def run_pair_config(args, dist):
    """C1/C3 (length + subsequence) and C4/C5 (length only), single GPU."""
    import torch
    import paper_1306_4627_b200 as wl
    from paper_1306_4627_b200 import workloads
    torch.cuda.set_device(dist.local_rank)
    x, y = workloads.config_pair(args.config, args.seed)
    sub = args.config in ("c1", "c3")
    name = {"c1": "C1: 10k x 10k DNA, length + subsequence",
            "c3": "C3: 100k x ~100k mutated DNA, length + subsequence",
            "c4": "C4: 1M x 1M DNA, length only",
            "c5": "C5: 2M x 500k Zipf(1.1) bytes, length only"}[args.config]
    cells = len(x) * len(y)
    variant = wl.VARIANT_WAVEFRONT if args.variant == "wavefront" else wl.VARIANT_BITPARALLEL
    if variant == wl.VARIANT_WAVEFRONT:
        sub = False  # the cell-wavefront variant computes lengths only
    fn = (lambda: wl.lcs_subsequence(x, y, wl.NO_BUDGET)) if sub else \
        (lambda: wl.lcs_length(x, y, wl.NO_BUDGET, variant=variant))
    for _ in range(args.warmup):
        res = fn()
    times, fill_ms = [], []
    wl._check(wl.lib.wlcs_set_timing(1))
    km = ctypes.c_float()
    with ClockSampler(dist.local_rank) as clocks:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn()
            times.append(time.perf_counter() - t0)
            wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
            fill_ms.append(km.value)
    wl._check(wl.lib.wlcs_set_timing(0))
    t = float(np.mean(times))
    length = len(res) if sub else res
    return {"metric": METRIC, "value": round(cells / t / 1e9, 3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "none", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (paper_1306_4627_b200/workloads.py)",
            "config": {"workload": name + ("" if sub or args.config not in ("c1", "c3")
                                           else " (length only)"),
                       "lcs_length": length, "m": len(x), "n": len(y)},
            "variant": args.variant,
            "fill_kernel_ms": round(float(np.mean(fill_ms)), 3),
            "fill_gcups": round(cells / (float(np.mean(fill_ms)) * 1e-3) / 1e9, 1)
            if np.mean(fill_ms) > 0 else None,
            "clocks": clocks.summary(),
            "note": "end-to-end wall time through the C-ABI (H2D, fill, traceback, D2H)"}


def main():
    args = parse_args()
    rc = maybe_spawn(args)
    if rc is not None:
        return rc
    dist = Dist()
    if args.impl == "reference":
        return run_reference_arm(args, dist)
    dist.init()
    if args.config == "c2" and args.dry_run:
        line = run_c2_dry(args, dist)
    elif args.config == "c2":
        line = run_c2(args, dist)
        # C4 at N > 1 runs the cross-GPU column split, which no multi-GPU box
        # has exercised yet: opt-in (WLCS_BENCH_C4_SPLIT=1) so that it can
        # never stall the headline scaling run; ranks sharing one device
        # (WLCS_BENCH_ONE_DEVICE) must never wait on each other
        split_ok = os.environ.get("WLCS_BENCH_C4_SPLIT") == "1" and \
            os.environ.get("WLCS_BENCH_ONE_DEVICE") != "1"
        if not args.no_single_pairs and args.variant == "bitparallel" and \
                (dist.world == 1 or split_ok):
            import paper_1306_4627_b200 as wl
            peak = ctypes.c_double()
            wl._check(wl.lib.wlcs_probe_int_peak(5, ctypes.byref(peak)))
            for name in ("c4", "c5"):
                if name == "c5" and dist.world > 1:
                    continue  # C5 is a one-GPU configuration (BASELINE configs[4])
                try:
                    line[name] = single_pair_block(name, 3, 1, dist, peak.value)
                except Exception as exc:  # report, never lose the headline line
                    line[name] = {"error": f"{type(exc).__name__}: {exc}"}
            if dist.world == 1:
                for name in ("c1", "c3"):  # one-GPU configurations (configs[0], [2])
                    try:
                        line[name] = subsequence_pair_block(name, 5, 2, peak.value)
                    except Exception as exc:
                        line[name] = {"error": f"{type(exc).__name__}: {exc}"}
    elif (dist.world > 1 or args.colsplit) and args.config in ("c4", "c5"):
        line = run_colsplit(args, dist)
    else:
        line = run_pair_config(args, dist)
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
