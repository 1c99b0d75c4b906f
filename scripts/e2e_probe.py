"""Host-side cost of one end-to-end C2 estimate through the public API (model + property
creation, estimate, read-back), split by call; prints medians over 30 repetitions."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_0912_2551_b200 as smc  # noqa: E402
import workloads  # noqa: E402


def main():
    torch.cuda.set_device(0)
    smc.use_torch()
    cfg = workloads.c2()
    s = cfg["sampling"]
    rows = []
    for it in range(33):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = smc.Model.from_config(cfg)
        t1 = time.perf_counter()
        p = smc.Property(m, cfg["formula"])
        t2 = time.perf_counter()
        r = smc.estimate(m, p, s["confidence"], s["half_width"], cfg["seed"])
        t3 = time.perf_counter()
        info = m.last_launch(p)
        del p, m
        t4 = time.perf_counter()
        if it >= 3:
            rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, info["kernel_ms"] / 1e3))
    a = np.median(np.array(rows), axis=0) * 1e3
    print("ms: model %.3f property %.3f estimate %.3f (kernels %.3f) free %.3f" % (a[0], a[1], a[2], a[4], a[3]))


if __name__ == "__main__":
    main()
