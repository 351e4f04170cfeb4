"""NVML NVLink byte counters around a known peer copy (calibration of
bench.NvlinkCounters): GPU0 pulls 8 GiB from GPU1 with the copy engine and
with the pull kernel (rs_pull_spans); prints each GPU's tx/rx bytes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
from paper_2604_09107_b200 import ros  # noqa: E402

n = 8 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda:1")
b = torch.empty(n, dtype=torch.uint8, device="cuda:0")
ros.synth_bf16(a, 3)
torch.cuda.synchronize(1)
cs = [B.NvlinkCounters(i) for i in range(2)]
print("links", [c.links if not c.err else c.err for c in cs])
for what in ("copy engine", "pull kernel"):
    r0 = [c.read() for c in cs]
    if what == "copy engine":
        b.copy_(a)
        torch.cuda.synchronize(0)
    else:
        code, ms = ros.pull_spans([a.data_ptr()], [b.data_ptr()], [n], device=0)
        print("kernel ms", ms, "code", code, "GB/s", n / ms / 1e6)
    r1 = [c.read() for c in cs]
    for i in range(2):
        if r0[i] and r1[i]:
            print(what, f"gpu{i}", "tx %.3f GB rx %.3f GB (%s); user bytes %.3f GB" % (
                (r1[i][0] - r0[i][0]) / 1e9, (r1[i][1] - r0[i][1]) / 1e9, r1[i][2], n / 1e9))
        else:
            print(what, f"gpu{i}", "no counters", cs[i].err)
