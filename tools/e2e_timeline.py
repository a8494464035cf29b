"""GPU timeline of one host-buffer matvec (c2 headline) via torch.profiler/CUPTI: where the e2e time goes."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("H2B_POOL_RESERVE_GB", "16")
import bench  # noqa: E402
import paper_2203_14832_b200 as h2c  # noqa: E402
from paper_2203_14832_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS["c2"]
pts, w = bench.make_inputs(cfg)
kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
h2 = h2c.assemble(h2c.build_tree(h2c.PointCloud.from_points(pts), nu=cfg[6], eta=float(np.sqrt(2.0))), kern, cfg[7])
L = _lib.lib()
s = torch.cuda.current_stream()
wh = torch.from_numpy(np.ascontiguousarray(w)).pin_memory()
uh = torch.empty(w.shape, dtype=torch.float64).pin_memory()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    _lib.check(L.h2b_matvec(h2.handle, wh.data_ptr(), uh.data_ptr(), 1, 0, s.cuda_stream))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        flush.zero_()
        _lib.check(L.h2b_matvec(h2.handle, wh.data_ptr(), uh.data_ptr(), 1, 0, s.cuda_stream))
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev = None
for e in evs:
    st, en = e.time_range.start - t0, e.time_range.end - t0
    gap = st - prev if prev is not None else 0
    print(f"{st:10.1f} {en - st:9.1f} gap {gap:7.1f}  {e.name[:70]}")
    prev = en
