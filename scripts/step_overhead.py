"""Where does a C2 dose step spend time outside the tile kernel?  (GPU diagnostic)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2103_09683_b200 as dg  # noqa: E402


def timed(fn, n=20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


ps = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
e = dg.DoseEngine.generate(ps, device=0)
cols = sum(p.cols for p in ps)
x = torch.from_numpy(dg.seeded_vector(cols, 42)).cuda()
y = torch.empty(e.info["rows"], dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s = st.cuda_stream
print("zero_ y          ms", timed(lambda: y.zero_()))
print("dose step        ms", timed(lambda: e.dose_device(x.data_ptr(), cols, y.data_ptr(), stream=s, sync=False)))
tot = 0.0
for _ in range(10):
    e.dose_device(x.data_ptr(), cols, y.data_ptr(), stream=s, sync=True, profile=True)
    tot += sum(k["ms"] for k in e.kernel_times())
print("kernels (profiled) ms", tot / 10, e.kernel_times())
print("last_timing", e.last_timing())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for n in (1, 2, 5):
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        e.dose_device(x.data_ptr(), cols, y.data_ptr(), stream=s, sync=False)
    b.record()
    torch.cuda.synchronize()
    print(f"{n} doses back to back: {a.elapsed_time(b):.4f} ms")
