#!/usr/bin/env python
"""describe() on float64 frames that are not u8-valued (the eval harness's warped + noisy frames): page-locked and
ordinary host memory, 1920x1080 with 10 k keypoints, against the u8-valued float64 frame of the bench."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench                                          # noqa: E402
import paper_1609_03986_b200 as lk                    # noqa: E402

eng = lk.get_engine()
img, kps = bench.synth_inputs("cfg2")
frac = img.astype(np.float64) * 0.93 + np.random.default_rng(0).random(img.shape) * 3.0


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


for name, arr in (("u8-valued float64, page-locked", pinned(img.astype(np.float64))), ("non-integer float64, page-locked", pinned(frac)),
                  ("non-integer float64, ordinary memory", frac)):
    for _ in range(5):
        lk.describe(arr, kps)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        lk.describe(arr, kps)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print(f"{name:40s} describe: median {ts[10]:.3f} ms, min {ts[0]:.3f} ms", flush=True)
