"""Development aid (library built with -DSW_TRACE_ITEMS=1, SW_B200_LIB=<that build>): per-work-item
timeline of the wavefront kernels of one call -- per launch: span, SM busy fraction, the slowest
items.  python tools/item_trace.py c5"""
import ctypes
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2208_12350_b200 import sw, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
b = synth.generate_parallel(cfg)
a = sw.Aligner(0)
q, qo, r, ro = a.to_device(b)
out = a.alloc_out(b.n_pairs)
lib = sw.load()
lib.sw_debug_item_trace.argtypes = [ctypes.c_void_p, ctypes.c_int64]
lib.sw_debug_item_trace.restype = ctypes.c_int64
a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
lib.sw_debug_item_trace(None, 0)  # reset
a.align_tensors(q, qo, r, ro, b.scoring, out=out)
torch.cuda.synchronize()
buf = np.zeros((1 << 21, 4), dtype=np.uint64)
k = lib.sw_debug_item_trace(buf.ctypes.data, buf.shape[0])
t = buf[:k]
item = (t[:, 0] >> 32).astype(np.int64)
smid = ((t[:, 0] >> 16) & 0xffff).astype(np.int64)
rev = ((t[:, 0] >> 8) & 0xff).astype(np.int64)
route = (t[:, 0] & 0xff).astype(np.int64)
t0 = t[:, 1].astype(np.int64)
t1 = t[:, 2].astype(np.int64)
ns = (t[:, 3] >> 48).astype(np.int64)
mmax = ((t[:, 3] >> 24) & 0xffffff).astype(np.int64)
steps = (t[:, 3] & 0xffffff).astype(np.int64)
for rv in (0, 1):
    for rt in np.unique(route[rev == rv]):
        sel = (rev == rv) & (route == rt)
        if not sel.any():
            continue
        T0, T1 = t0[sel].min(), t1[sel].max()
        span = (T1 - T0) / 1e6
        dur = (t1[sel] - t0[sel]) / 1e6
        busy = np.zeros(148)
        np.add.at(busy, smid[sel], dur)
        # warp-level: concurrent items per SM over time -> busy SM-time / (148 * 16 warps * span)
        print(f"{'rev' if rv else 'fwd'} route {rt}: {sel.sum()} items, span {span:.2f} ms, "
              f"item-ms sum {dur.sum():.1f}, mean warps busy {dur.sum() / span:.0f} of 2368")
        ends = np.sort((t1[sel] - T0) / 1e6)
        for f in (0.5, 0.9, 0.99, 1.0):
            print(f"   {int(f*100)}% of items done by {ends[min(len(ends)-1, int(f*len(ends)))]:.2f} ms")
        order = np.argsort(-dur)[:8]
        idx = np.nonzero(sel)[0][order]
        for i in idx:
            print(f"   item {item[i]:6d} sm {smid[i]:3d} start {(t0[i]-T0)/1e6:7.2f} dur {(t1[i]-t0[i])/1e6:7.2f} ms "
                  f"stripes {ns[i]} mmax {mmax[i]} steps {steps[i]}")
        # time profile of active items
        grid = np.linspace(T0, T1, 11)
        act = [int(np.sum((t0[sel] <= g) & (t1[sel] > g))) for g in grid[:-1]]
        print("   items in flight at 0..90% of span:", act)
