#!/usr/bin/env python3
"""bench.py -- GCUPS of the B200-native LCS table fill (BASELINE.json metric).

Default workload (BASELINE.json configs[1], "C2"): a batch of 65,536
independent protein-like pairs (20-letter alphabet, lengths uniform in
[200, 1000], i.i.d. symbols; synthetic, seeded std::mt19937_64 -- see
wlcs_generate_pairs in include/wavelcs_capi.h).  One "step" = one pass of the
fill over the whole batch (LCS length of every pair).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
                  [--config c2|c1|c3|c4|c5]

Under torchrun (N > 1) every rank processes its own 65,536-pair shard (pairs
are independent: no data-path collective; "scaling": "weak"); the timed
region is bracketed by barrier + cuda synchronize and the max over ranks is
reported by rank 0.

`value`   : algorithmic cells (sum m_k * n_k, no padding) / device time of
            the K steps, inputs resident in HBM, L2 flushed between steps
            (300 MB write, untimed).  CUDA events on the launching stream.
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
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
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


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=["c2", "c1", "c3", "c4", "c5"], default="c2")
    ap.add_argument("--pairs", type=int, default=65536)
    ap.add_argument("--seed", type=int, default=20130619)
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU work of the bounded reference sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--colsplit", action="store_true",
                    help="c4/c5: use the multi-GPU column-split path even on one GPU")
    ap.add_argument("--variant", choices=["bitparallel", "wavefront"], default="bitparallel",
                    help="fill kernel variant (WLCS_VARIANT_*)")
    return ap.parse_args()


# ----------------------------------------------------------------- plumbing
class Dist:
    """One process per GPU (torchrun).  NCCL by default; WLCS_DIST_BACKEND=gloo
    and WLCS_BENCH_ONE_DEVICE=1 exist only to exercise the N > 1 host logic
    on a single-GPU box (independent shards, no kernel waits on another)."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        if os.environ.get("WLCS_BENCH_ONE_DEVICE") == "1":
            self.local_rank = 0
        self.backend = os.environ.get("WLCS_DIST_BACKEND", "nccl")
        self.pg = None

    def init(self):
        import torch
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


# ------------------------------------------------------------------ inputs
def gen_pairs(wl, pairs: int, lo: int, hi: int, alphabet: bytes, seed: int, pinned: bool):
    """C2 generator (wlcs_generate_pairs); optionally into page-locked memory."""
    cap = pairs * hi
    if pinned:
        bufs = []

        def alloc(n, dtype):
            p = wl.lib.wlcs_host_alloc(n * np.dtype(dtype).itemsize)
            if not p:
                raise MemoryError("wlcs_host_alloc")
            bufs.append(p)
            arr = np.ctypeslib.as_array(
                (ctypes.c_uint8 * (n * np.dtype(dtype).itemsize)).from_address(p))
            return arr.view(dtype)
        xs, ys = alloc(cap, np.uint8), alloc(cap, np.uint8)
        xo, yo = alloc(pairs + 1, np.uint64), alloc(pairs + 1, np.uint64)
    else:
        xs, ys = np.empty(cap, np.uint8), np.empty(cap, np.uint8)
        xo, yo = np.empty(pairs + 1, np.uint64), np.empty(pairs + 1, np.uint64)
    a = np.frombuffer(alphabet, np.uint8)
    rc = wl.lib.wlcs_generate_pairs(ctypes.c_size_t(pairs), ctypes.c_size_t(lo),
                                    ctypes.c_size_t(hi), a.ctypes.data, ctypes.c_size_t(len(a)),
                                    ctypes.c_uint64(seed), xs.ctypes.data,
                                    xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                    ys.ctypes.data,
                                    yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    wl._check(rc)
    return xs, xo, ys, yo


def cells_of(xo, yo) -> int:
    m = np.diff(xo.astype(np.int64))
    n = np.diff(yo.astype(np.int64))
    return int(np.sum(m * n))


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
    import oracle
    import paper_1306_4627_b200 as wl
    if dist.rank != 0:
        return 0
    ref = oracle.Reference()
    threads = os.cpu_count() or 1
    if args.config != "c2":
        print(json.dumps({"impl": "reference", "unavailable":
                          f"reference arm implemented for the bench workload c2 only"}))
        return 0
    xs, xo, ys, yo = gen_pairs(wl, args.pairs, 200, 1000, PROTEIN, args.seed, pinned=False)
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": "C2: 65536 protein-like pairs, 20 letters, lengths U[200,1000]",
                   "global_batch": args.pairs, "seq_len": "200-1000", "parallelism": "cpu-threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- B200 arm
def run_c2(args, dist):
    import torch
    import paper_1306_4627_b200 as wl
    dev = torch.device("cuda", dist.local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    seed = args.seed + dist.rank
    xs, xo, ys, yo = gen_pairs(wl, args.pairs, 200, 1000, PROTEIN, seed, pinned=True)
    xs_bytes, ys_bytes = int(xo[-1]), int(yo[-1])
    cells = cells_of(xo, yo)
    d_xs = torch.from_numpy(xs[: xs_bytes + 16]).to(dev)
    d_ys = torch.from_numpy(ys[: ys_bytes + 16]).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(args.pairs, dtype=torch.int32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    variant = wl.VARIANT_WAVEFRONT if args.variant == "wavefront" else wl.VARIANT_BITPARALLEL

    def step():
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(),
                                   d_yo.data_ptr(), args.pairs, xs_bytes, ys_bytes,
                                   d_out.data_ptr(), stream.cuda_stream, variant=variant)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    wl._check(wl.lib.wlcs_set_timing(1))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    main_ms = []
    with ClockSampler(dist.local_rank) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
            km = ctypes.c_float()
            wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
            main_ms.append(km.value)
        torch.cuda.synchronize()
        dist.barrier()
    wl._check(wl.lib.wlcs_set_timing(0))
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    total_ms = dist.max(float(np.sum(step_ms)))
    all_cells = dist.sum(float(cells))
    value = all_cells * args.steps / (total_ms * 1e-3) / 1e9
    gpu_lengths = d_out.cpu().numpy().astype(np.uint32)

    # e2e through the public host API (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        out = np.zeros(args.pairs, np.uint32)
        outp = out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
        xop = xo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        yop = yo.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))

        def e2e_step():
            wl._check(wl.lib.wlcs_length_batch_ex(xs.ctypes.data, xop, ys.ctypes.data, yop,
                                                  args.pairs, variant, outp))
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
        if not np.array_equal(out, gpu_lengths):
            raise AssertionError("e2e lengths differ from the device-resident run")
        e2e = {"value": round(all_cells * args.steps / e2e_total / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": int(xs_bytes + ys_bytes + 16 * (args.pairs + 1)),
               "d2h_bytes_per_step": int(4 * args.pairs)}

    peak = ctypes.c_double()
    wl._check(wl.lib.wlcs_probe_int_peak(5, ctypes.byref(peak)))
    kernel_ms = float(np.mean(main_ms))
    wave = variant == wl.VARIANT_WAVEFRONT
    # algorithmic int ops: bit-parallel 3 per 32-cell word-row; cell wavefront
    # 3 per cell (match test, max, add-max)
    alg_ops = cells * 3.0 if wave else cells * 3.0 / 32.0
    achieved = alg_ops / (kernel_ms * 1e-3) / 1e12
    peak_t = peak.value / 1e12
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded std::mt19937_64, wlcs_generate_pairs)",
        "config": {"workload": "C2: 65536 protein-like pairs per GPU, 20-letter alphabet, "
                               "lengths U[200,1000], LCS length per pair",
                   "global_batch": args.pairs * dist.world, "seq_len": "200-1000",
                   "parallelism": f"pair-sharded x{dist.world} (no collective)",
                   "cells_per_gpu_step": cells, "l2": "flushed between steps (300 MB write)"},
        # bit-parallel: plan, scatter (with the bucket scan), main -- the
        # workspace memset is a driver memset, not counted; wavefront: one kernel
        "gpu_launches": (1 if wave else 3) * args.steps,
        "variant": args.variant,
        "roofline": {"bound": "int", "achieved": round(achieved, 3), "peak": round(peak_t, 3),
                     "unit": "Tops/s (int32 ALU, 3 ops per cell)" if wave else
                             "Tops/s (int32 ALU, 3 ops per 32-cell word-row)",
                     "frac": round(achieved / peak_t, 4), "traffic": ncu_traffic(
                         "wave_batch_kernel" if wave else "batch_main_kernel"),
                     "algorithmic_bytes": int(xs_bytes + ys_bytes + 16 * (args.pairs + 1)
                                              + 4 * args.pairs),
                     "kernel": "wave_batch_kernel" if wave else "batch_main_kernel",
                     "kernel_ms": round(kernel_ms, 4),
                     "kernel_share_of_step": round(kernel_ms / (total_ms / args.steps), 3),
                     "peak_source": "measured live: wlcs_probe_int_peak (LOP3 stream)",
                     "gcups_ceiling": round(peak.value * (1 if wave else 32) / 3 / 1e9, 1)},
        "clocks": clocks.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_c2(args, xs, xo, ys, yo, gpu_lengths)
    return line


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "ncu_traffic.json")) as f:
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


def run_colsplit(args, dist):
    """C4/C5 on N GPUs: one long pair, column slice per rank (strong scaling).
    Carries cross GPUs inside the fill (the producer kernel stores into the
    consumer's inbox through an IPC peer pointer); the length comes from one
    all_gather + one MAX all_reduce (multigpu.colsplit_combine_dist)."""
    import torch
    import paper_1306_4627_b200 as wl
    from paper_1306_4627_b200 import multigpu, workloads
    torch.cuda.set_device(dist.local_rank)
    dev = torch.device("cuda", dist.local_rank)
    import torch.distributed as tdist
    x, y = workloads.config_pair(args.config, args.seed)
    rows, cols = (x, y) if len(x) <= len(y) else (y, x)
    G, g = dist.world, dist.rank
    lo, hi = multigpu.colsplit_bounds(len(cols), G)[g]
    words = wl.colsplit_inbox_words(len(rows))
    in_f, in_r = wl.device_alloc(4 * words), wl.device_alloc(4 * words)
    handles = [(None, None)] * G
    if G > 1:
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
        if G == 1:
            return multigpu.colsplit_combine([(lo, hi)], [vf], [vr], len(cols))
        return multigpu.colsplit_combine_dist(lo, hi, vf, vr, tdist,
                                              device=dev if dist.backend == "nccl" else None)

    for _ in range(args.warmup):
        length = step()
    wl._check(wl.lib.wlcs_set_timing(1))
    km = ctypes.c_float()
    wall, fill = [], []
    with ClockSampler(dist.local_rank) as clocks:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            length = step()
            wall.append(time.perf_counter() - t0)
            wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
            fill.append(km.value)
    wl._check(wl.lib.wlcs_set_timing(0))
    fill_ms = dist.max(float(np.mean(fill)))
    wall_s = dist.max(float(np.mean(wall)))
    if out_f:
        wl.ipc_close(out_f)
    if out_r:
        wl.ipc_close(out_r)
    cells = len(x) * len(y)
    return {"metric": METRIC, "value": round(cells / (fill_ms * 1e-3) / 1e9, 3), "unit": UNIT,
            "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(fill_ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (workloads.py)",
            "config": {"workload": f"{args.config.upper()} single pair, column split x{G}",
                       "lcs_length": length, "m": len(x), "n": len(y),
                       "parallelism": f"column slices x{G}, carries over NVLink P2P (IPC)"},
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
    dist = Dist()
    if args.impl == "reference":
        return run_reference_arm(args, dist)
    dist.init()
    if args.config == "c2":
        line = run_c2(args, dist)
    elif (dist.world > 1 or args.colsplit) and args.config in ("c4", "c5"):
        line = run_colsplit(args, dist)
    else:
        line = run_pair_config(args, dist)
    if dist.rank == 0:
        print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
