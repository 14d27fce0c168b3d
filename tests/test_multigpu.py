"""Multi-process (gloo, world_size 2, CPU) coverage of the multi-GPU host logic.

The GPU box has one GPU, so the N>1 paths are exercised here with real
torch.distributed processes and the oracle standing in for the device fill:
  * batch sharding covers every pair exactly once and the all_gathered
    lengths equal the single-process result;
  * the column-strip pipeline (rank g = strip g, per-band carry bits sent
    rank g -> g+1) reproduces the whole-pair length.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _batch_worker(rank, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import oracle
    from paper_1306_4627_b200 import multigpu
    _init(rank, port)
    res = oracle.Restatement()
    rng = np.random.default_rng(99)
    lens_m = rng.integers(0, 400, 301)
    lens_n = rng.integers(0, 400, 301)
    xs = rng.integers(65, 69, int(lens_m.sum())).astype(np.uint8)
    ys = rng.integers(65, 69, int(lens_n.sum())).astype(np.uint8)
    xo = np.concatenate([[0], np.cumsum(lens_m)]).astype(np.uint64)
    yo = np.concatenate([[0], np.cumsum(lens_n)]).astype(np.uint64)
    lo, hi = multigpu.shard_pairs(xo, yo, WORLD, rank)
    mine = res.length_batch(xs, xo[lo:hi + 1] if hi > lo else xo[:1], ys,
                            yo[lo:hi + 1] if hi > lo else yo[:1]) if hi > lo else np.zeros(0, np.uint32)
    full = torch.zeros(301, dtype=torch.int64)
    full[lo:hi] = torch.from_numpy(mine.astype(np.int64))
    covered = torch.zeros(301, dtype=torch.int64)
    covered[lo:hi] = 1
    dist.all_reduce(full)
    dist.all_reduce(covered)
    if rank == 0:
        out["ok"] = bool((covered == 1).all()) and np.array_equal(
            full.numpy(), res.length_batch(xs, xo, ys, yo).astype(np.int64))
    dist.destroy_process_group()


def _strip_worker(rank, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import oracle
    from paper_1306_4627_b200 import multigpu
    _init(rank, port)
    res = oracle.Restatement()
    x = res.generate_random(5000, b"ACGT", 11)
    y = res.generate_random(3333, b"ACGT", 12)
    c0, c1 = multigpu.strip_bounds(len(y), WORLD)[rank]
    V = np.full(max(1, (c1 - c0 + 63) // 64), 2**64 - 1, np.uint64)
    for r0, r1 in multigpu.band_ranges(len(x), 777):
        rows = r1 - r0
        cin = None
        if rank > 0:
            buf = torch.zeros((rows + 7) // 8, dtype=torch.uint8)
            dist.recv(buf, src=rank - 1)
            cin = multigpu.unpack_carries(buf.numpy(), rows)
        cout = res.strip_rows(x[r0:r1], y[c0:c1], V, cin)
        if rank < WORLD - 1:
            dist.send(torch.from_numpy(multigpu.pack_carries(cout).copy()), dst=rank + 1)
    z = torch.tensor([res.strip_zeros(V, c1 - c0)], dtype=torch.int64)
    dist.all_reduce(z)
    if rank == 0:
        out["ok"] = int(z.item()) == res.length_bitpar(x, y)
    dist.destroy_process_group()


def _colsplit_worker(rank, port, out):
    """Bidirectional column split (the C4 multi-GPU decomposition): forward
    carries flow rank 0 -> 1, reverse carries rank 1 -> 0, the length comes
    from colsplit_combine_dist (all_gather of zero totals + MAX all_reduce)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import oracle
    from paper_1306_4627_b200 import multigpu
    _init(rank, port)
    res = oracle.Restatement()
    x = res.generate_random(4001, b"ACGT", 21)
    y = res.generate_random(2999, b"ACGT", 22)
    n = len(y)
    lo, hi = multigpu.colsplit_bounds(n, WORLD)[rank]
    mid = len(x) // 2
    words = max(1, (hi - lo + 63) // 64)
    vf = np.full(words, 2**64 - 1, np.uint64)
    vr = np.full(words, 2**64 - 1, np.uint64)
    top = x[:mid]
    bot = x[mid:][::-1]
    ycol, ycol_rev = y[lo:hi], y[lo:hi][::-1]
    # forward: left to right
    for r0, r1 in multigpu.band_ranges(len(top), 500):
        cin = None
        if rank > 0:
            buf = torch.zeros((r1 - r0 + 7) // 8, dtype=torch.uint8)
            dist.recv(buf, src=rank - 1)
            cin = multigpu.unpack_carries(buf.numpy(), r1 - r0)
        cout = res.strip_rows(top[r0:r1], ycol, vf, cin)
        if rank < WORLD - 1:
            dist.send(torch.from_numpy(multigpu.pack_carries(cout).copy()), dst=rank + 1)
    # reverse: right to left
    for r0, r1 in multigpu.band_ranges(len(bot), 500):
        cin = None
        if rank < WORLD - 1:
            buf = torch.zeros((r1 - r0 + 7) // 8, dtype=torch.uint8)
            dist.recv(buf, src=rank + 1)
            cin = multigpu.unpack_carries(buf.numpy(), r1 - r0)
        cout = res.strip_rows(bot[r0:r1], ycol_rev, vr, cin)
        if rank > 0:
            dist.send(torch.from_numpy(multigpu.pack_carries(cout).copy()), dst=rank - 1)
    got = multigpu.colsplit_combine_dist(lo, hi, vf, vr, dist)
    if rank == 0:
        out["ok"] = got == res.length_bitpar(x, y)
        out["got"] = got
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", [_batch_worker, _strip_worker, _colsplit_worker])
def test_two_process_gloo(worker):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(_free_port(), out), nprocs=WORLD, join=True)
    assert out.get("ok") is True


def test_shard_and_strip_planning():
    from paper_1306_4627_b200 import multigpu
    xo = np.array([0, 10, 10, 500, 700], np.uint64)
    yo = np.array([0, 5, 50, 60, 900], np.uint64)
    for world in (1, 2, 3, 4, 8):
        ranges = [multigpu.shard_pairs(xo, yo, world, r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 4
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    b = multigpu.strip_bounds(1000, 3)
    assert b[0][0] == 0 and b[-1][1] == 1000 and all(c0 % 64 == 0 for c0, _ in b)
    assert multigpu.band_ranges(10, 4) == [(0, 4), (4, 8), (8, 10)]
    bits = np.random.default_rng(0).integers(0, 2, 77).astype(np.uint8)
    assert np.array_equal(multigpu.unpack_carries(multigpu.pack_carries(bits), 77), bits)


def test_colsplit_combine_single_process():
    """colsplit_combine over oracle slices equals the whole-pair length for
    1..4 slices and odd widths."""
    import oracle
    from paper_1306_4627_b200 import multigpu
    res = oracle.Restatement()
    x = res.generate_random(1501, b"ACGT", 5)
    y = res.generate_random(1234, b"ACGT", 6)
    want = res.length_bitpar(x, y)
    mid = len(x) // 2
    for world in (1, 2, 3, 4):
        bounds = multigpu.colsplit_bounds(len(y), world)
        vfs = [None] * world
        vrs = [None] * world
        cin = None
        for g, (lo, hi) in enumerate(bounds):
            v = np.full(max(1, (hi - lo + 63) // 64), 2**64 - 1, np.uint64)
            cin = res.strip_rows(x[:mid], y[lo:hi], v, cin)
            vfs[g] = v
        cin = None
        for g in reversed(range(world)):
            lo, hi = bounds[g]
            v = np.full(max(1, (hi - lo + 63) // 64), 2**64 - 1, np.uint64)
            cin = res.strip_rows(x[mid:][::-1], y[lo:hi][::-1], v, cin)
            vrs[g] = v
        assert multigpu.colsplit_combine(bounds, vfs, vrs, len(y)) == want, world


def test_bench_two_ranks_shard_the_c2_batch():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under
    torch.distributed.run (2 ranks, gloo); the two ranks' shards cover the
    configured 65,536-pair batch exactly once (strong scaling).  --dry-run
    stops before device work, so this runs on the CPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WLCS_DIST_BACKEND="gloo", WLCS_BENCH_ONE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["scaling"] == "strong"
    assert rec["pairs_total"] == 65536
    assert rec["cells_total"] == rec["cells_batch"]
    # balanced by cells: neither rank holds much more than half
    assert rec["max_rank_cells"] <= 0.51 * rec["cells_batch"]
