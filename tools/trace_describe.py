#!/usr/bin/env python
"""CLATCH_TRACE=1 python tools/trace_describe.py [cfg2|cfg3]: stage stamps of describe_all on stderr."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle                                   # noqa: E402
import paper_1609_03986_b200 as lk              # noqa: E402

port = oracle.port()
eng = lk.get_engine()
eng.set_pattern(None)
W, H, N = (3840, 2160, 50000) if (len(sys.argv) > 1 and sys.argv[1] == "cfg3") else (1920, 1080, 10000)
img = port.random_image_u8(30000, W, H)
kps = port.random_keypoints(31000, W, H, N)


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


pimg, pkps = pinned(img), pinned(kps)
for dtype_img in (pimg, pinned(img.astype(np.float64))):
    for i in range(4):
        t0 = time.perf_counter()
        r = eng.describe_all(dtype_img, pkps)
        print(f"python describe_all {dtype_img.dtype} ms", (time.perf_counter() - t0) * 1e3, file=sys.stderr)
