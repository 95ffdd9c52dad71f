"""End-to-end timing breakdown of the C2 host path (dg_last_timing: x upload, kernels, d
download tail, total) for the current environment's plan knobs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2103_09683_b200 as dg  # noqa: E402

ps = bench.workload("c2", int(sys.argv[1]) if len(sys.argv) > 1 else 0)
e = dg.DoseEngine.generate(ps, device=0)
cols = sum(p.cols for p in ps)
xh = torch.from_numpy(dg.seeded_vector(cols, 42)).pin_memory()
yh = torch.empty(e.info["rows"], dtype=torch.float64).pin_memory()
for _ in range(3):
    e.dose_host_ptrs(xh.data_ptr(), cols, yh.data_ptr())
t = []
for _ in range(10):
    e.dose_host_ptrs(xh.data_ptr(), cols, yh.data_ptr())
    t.append(e.last_timing())
print(os.environ.get("TAG", ""), "median", {k: round(float(np.median([d[k] for d in t])), 4) for k in t[0]})
