"""Batch-kernel time vs occupancy: pairs whose column string fits K <= 4
words per lane (masks <= 12 KB per warp), run with the mask budget at 12 KB
(18 warps/SM) and at 24 KB (9 warps/SM)."""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if len(sys.argv) > 1:  # child: one measurement
    import torch
    import paper_1306_4627_b200 as wl
    rng = np.random.default_rng(1)
    pairs = 65536
    prot = np.frombuffer(b"ACDEFGHIKLMNPQRSTVWY", np.uint8)
    lm = rng.integers(100, 129, pairs)   # columns: <= 128 -> K <= 4, S = 1
    ln = rng.integers(600, 1001, pairs)
    xs = prot[rng.integers(0, 20, int(lm.sum()))]
    ys = prot[rng.integers(0, 20, int(ln.sum()))]
    xo = np.concatenate([[0], np.cumsum(lm)]).astype(np.uint64)
    yo = np.concatenate([[0], np.cumsum(ln)]).astype(np.uint64)
    dev = torch.device("cuda")
    d_xs = torch.from_numpy(np.concatenate([xs, np.zeros(16, np.uint8)])).to(dev)
    d_ys = torch.from_numpy(np.concatenate([ys, np.zeros(16, np.uint8)])).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(pairs, dtype=torch.int32, device=dev)
    wl._check(wl.lib.wlcs_set_timing(1))
    km = ctypes.c_float()
    best = 1e9
    for _ in range(8):
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                                   pairs, int(xo[-1]), int(yo[-1]), d_out.data_ptr(), 0)
        wl._check(wl.lib.wlcs_last_kernel_ms(ctypes.byref(km)))
        best = min(best, km.value)
    cells = float((lm * ln).sum())
    print(f"pm_kb={os.environ.get('WLCS_BATCH_PM_KB')} kernel {best:.4f} ms  "
          f"{cells / best / 1e6:.0f} GCUPS")
else:
    for kb in ("12", "24", "12", "24"):
        env = dict(os.environ, WLCS_BATCH_PM_KB=kb)
        subprocess.run([sys.executable, __file__, "run"], env=env, check=True)
