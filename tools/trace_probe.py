"""Per-task timeline of the batch kernel on C2 (library built with
-DWLCS_BATCH_TRACE via tools/exp_build.sh, path in WLCS_LIB_PATH): build vs
sweep time per lane shape, warp / SM finish spread, busy warps over time."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1306_4627_b200 as wl
import bench

xs, xo, ys, yo = bench.gen_pairs_pinned(wl, 65536, 200, 1000, bench.PROTEIN, 20130619)
xs, xo, ys, yo = (np.array(a) for a in (xs, xo, ys, yo))
dev = torch.device("cuda")
d_xs = torch.from_numpy(xs[: int(xo[-1]) + 16]).to(dev)
d_ys = torch.from_numpy(ys[: int(yo[-1]) + 16]).to(dev)
d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
d_out = torch.zeros(65536, dtype=torch.int32, device=dev)
fn = wl.lib.wlcs_debug_batch_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_uint, ctypes.c_int]
buf = np.zeros((1 << 15, 4), np.uint64)
for it in range(3):
    fn(None, 0, 1)
    wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                               65536, int(xo[-1]), int(yo[-1]), d_out.data_ptr(), 0)
    torch.cuda.synchronize()
n = fn(buf.ctypes.data, buf.shape[0], 1)
r = buf[:n].astype(np.int64)
a, b = r[:, 0], r[:, 1]
sm = r[:, 2] >> 32
bld = r[:, 2] & 0xffffffff
cls = r[:, 3] >> 32
rows = r[:, 3] & 0xffffffff
t0 = a.min(); a = a - t0; b = b - t0
end = b.max()
dur = b - a
print(f"tasks {n}  kernel span {end/1e3:.1f} us  task dur mean {dur.mean()/1e3:.1f} max {dur.max()/1e3:.1f} us;"
      f" build share {bld.sum()/dur.sum():.3f}")
for c in sorted(set(cls.tolist())):
    m = cls == c
    print(f"  S={c//16} K={c%16}: {m.sum():5d} tasks, dur {dur[m].mean()/1e3:6.1f} us, build {bld[m].mean()/1e3:5.2f} us,"
          f" rows {rows[m].mean():6.0f}, sweep ns/16rows {np.mean((dur[m]-bld[m])/np.maximum(rows[m],1))*16:6.1f}, "
          f"first start {a[m].min()/1e3:6.1f} last end {b[m].max()/1e3:6.1f}")
smf = np.array([b[sm == s].max() for s in np.unique(sm)])
print(f"SM finish: min {smf.min()/1e3:.1f} p10 {np.percentile(smf,10)/1e3:.1f} p50 {np.median(smf)/1e3:.1f} max {smf.max()/1e3:.1f} us;"
      f" mean SM idle share {(end-smf).mean()/end:.3f}")
# busy warps over time (10 us bins)
edges = np.arange(0, end + 10000, 10000)
busy = [(np.minimum(b, e1) - np.maximum(a, e0)).clip(0).sum() / 10000 for e0, e1 in zip(edges[:-1], edges[1:])]
print("busy warps per 10 us bin:", " ".join(f"{x:.0f}" for x in busy))
o = np.argsort(-b)[:8]
for i in o:
    print(f"  late task S={cls[i]//16} K={cls[i]%16} start {a[i]/1e3:.1f} end {b[i]/1e3:.1f} rows {rows[i]}")
np.savez(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "trace.npz"),
         a=a, b=b, sm=sm, bld=bld, cls=cls, rows=rows)
