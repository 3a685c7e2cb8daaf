#!/usr/bin/env python
"""FAST-9 + NMS + orientation on the device vs the reference on the host, 1920x1080 and 3840x2160."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import oracle                                   # noqa: E402
import paper_1609_03986_b200 as lk              # noqa: E402

port = oracle.port()
ref = oracle.ref()
for w, h in ((1920, 1080), (3840, 2160)):
    img = port.structured_image(11, w, h).astype(np.uint8)
    for name, im in (("u8", img), ("f64", img.astype(np.float64))):
        k = lk.detect(im)
        t0 = time.perf_counter()
        for _ in range(5):
            k = lk.detect(im)
        ms = (time.perf_counter() - t0) / 5 * 1e3
        print(f"{w}x{h} {name}: {len(k)} keypoints, lk.detect {ms:.2f} ms", flush=True)
    if ref is not None:
        t0 = time.perf_counter()
        kr = ref.detect_and_orient(img.astype(np.float64), 20.0, True)
        print(f"{w}x{h} reference detect_and_orient (1 thread): {(time.perf_counter() - t0) * 1e3:.1f} ms, {len(kr)} keypoints, "
              f"identical: {np.array_equal(kr, k)}", flush=True)
