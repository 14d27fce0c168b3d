"""Per-task timeline of the batch kernel on C2 (library built with
-DWLCS_TAIL_PROBE, path in WLCS_LIB_PATH)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import torch
    import paper_1306_4627_b200 as wl
    import bench
    xs, xo, ys, yo = (np.array(a) for a in bench.gen_pairs_pinned(wl, 65536, 200, 1000, bench.PROTEIN, 1))
    dev = torch.device("cuda")
    d_xs = torch.from_numpy(xs[: int(xo[-1]) + 16]).to(dev)
    d_ys = torch.from_numpy(ys[: int(yo[-1]) + 16]).to(dev)
    d_xo = torch.from_numpy(xo.view(np.int64)).to(dev)
    d_yo = torch.from_numpy(yo.view(np.int64)).to(dev)
    d_out = torch.zeros(65536, dtype=torch.int32, device=dev)
    for _ in range(2):
        wl.lcs_length_batch_device(d_xs.data_ptr(), d_xo.data_ptr(), d_ys.data_ptr(), d_yo.data_ptr(),
                                   65536, int(xo[-1]), int(yo[-1]), d_out.data_ptr(), 0)
        torch.cuda.synchronize()
    buf = np.zeros(4 * 16384, np.uint64)
    assert wl.lib.wlcs_probe_dump(buf.ctypes.data_as(__import__("ctypes").c_void_p)) == 0
    buf = buf.reshape(-1, 4)
    buf = buf[buf[:, 1] > 0]
    for r in buf:
        print("TASK", 0, int(r[2]) >> 32, int(r[2]) & 0xffffffff, int(r[0]), int(r[1]), int(r[3]) & 0xffffffff,
              int(r[3]) >> 32)
    print("LAUNCH_END")
else:
    out = subprocess.run([sys.executable, __file__, "run"], capture_output=True, text=True).stdout
    part = out.split("LAUNCH_END")[0]
    recs = np.array([list(map(int, l.split()[1:])) for l in part.splitlines() if l.startswith("TASK")],
                    dtype=np.int64)
    t, K, S, a, b, rows, cta = recs.T
    t = np.arange(len(t))
    t0 = a.min(); a -= t0; b -= t0
    dur = b - a
    print(f"tasks {len(t)}  end {b.max()/1e3:.1f} us  dur mean {dur.mean()/1e3:.1f} p50 {np.median(dur)/1e3:.1f} max {dur.max()/1e3:.1f}")
    o = np.argsort(-b)[:12]
    for i in o:
        print(f"  late task t={t[i]} K={K[i]} S={S[i]} start {a[i]/1e3:.1f} end {b[i]/1e3:.1f} dur {dur[i]/1e3:.1f} rows {rows[i]}")
    o = np.argsort(-dur)[:6]
    for i in o:
        print(f"  long task t={t[i]} K={K[i]} S={S[i]} start {a[i]/1e3:.1f} dur {dur[i]/1e3:.1f} rows {rows[i]}")
    fin = np.array([b[cta == c].max() for c in np.unique(cta)])
    print(f"warp finish: p0 {fin.min()/1e3:.1f} p50 {np.median(fin)/1e3:.1f} p90 {np.percentile(fin,90)/1e3:.1f} max {fin.max()/1e3:.1f} idle {(fin.max()-fin).mean()/fin.max():.3f}")
    for k in sorted(set(K)):
        m = K == k
        print(f"  K={k}: {m.sum()} tasks, dur mean {dur[m].mean()/1e3:.1f} us, per-row-chunk {np.mean(dur[m]/np.maximum(rows[m],1))*16:.1f} ns")
