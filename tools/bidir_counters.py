"""NVLink counters of a pull while the same port carries traffic the other
way (diagnostic).  Two processes, GPUs 0 and 1:

  --background S  GPU1 pulls 4 GiB from GPU0 in a loop for S seconds
                  (GPU0's port sends data, receives requests);
  --profiled      GPU0 pulls 4 GiB from GPU1 a few times (GPU0's port
                  receives data, sends requests) -- run under ncu with the
                  nvlrx/nvltx metrics while the background process runs.

tools/bidir_counters.sh runs both and writes the ncu CSV.
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_2604_09107_b200 import ros
    from paper_2604_09107_b200._lib import lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--background", type=float, default=0.0)
    ap.add_argument("--profiled", action="store_true")
    ap.add_argument("--gb", type=float, default=4.0)
    ap.add_argument("--items", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = int(a.gb * (1 << 30)) // a.items // 4096 * 4096
    total = n * a.items
    src_dev, run_dev = (0, 1) if a.background else (1, 0)
    src = torch.empty(total, dtype=torch.uint8, device=torch.device("cuda", src_dev))
    dst = torch.empty(total, dtype=torch.uint8, device=torch.device("cuda", run_dev))
    ros.synth_bf16(src, 3)
    torch.cuda.synchronize(src_dev)
    s_ = np.asarray([src.data_ptr() + i * n for i in range(a.items)], np.uint64)
    d_ = np.asarray([dst.data_ptr() + i * n for i in range(a.items)], np.uint64)
    l_ = np.asarray([n] * a.items, np.uint64)
    code, ms = C.c_int(), C.c_float()

    def pull():
        rc = lib.rs_pull_spans(s_.ctypes.data, d_.ctypes.data, l_.ctypes.data, a.items, 4096, None, None,
                               run_dev, None, C.byref(code), C.byref(ms))
        assert rc == 0 and code.value == 0, (rc, code.value)
        return ms.value

    if a.background:
        print("background ready", flush=True)
        t_end = time.time() + a.background
        times = []
        while time.time() < t_end:
            times.append(pull())
        print(f"background pulls {len(times)}, median {sorted(times)[len(times) // 2]:.3f} ms "
              f"({total / (sorted(times)[len(times) // 2] / 1e3) / 1e9:.1f} GB/s)", flush=True)
    else:
        for _ in range(a.reps):
            t = pull()
            print(f"profiled pull {t:.3f} ms ({total / (t / 1e3) / 1e9:.1f} GB/s)", flush=True)


if __name__ == "__main__":
    main()
