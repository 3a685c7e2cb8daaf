#!/usr/bin/env python
"""Extraction throughput by image kind: u8, integer-valued f64 (promoted on device), non-integer f64."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench                                          # noqa: E402
import paper_1609_03986_b200 as lk                    # noqa: E402

eng = lk.get_engine()
eng.set_pattern(None)
img, kps = bench.synth_inputs("cfg2")
h, w = img.shape
xycs, kept = eng.prepare_keypoints(kps, w, h)
d_x = torch.from_numpy(xycs).cuda()
frac = img.astype(np.float64) + np.random.default_rng(0).random(img.shape) * 0.5
for tag, im in (("u8", img), ("f64 integer-valued", img.astype(np.float64)), ("f64 non-integer", frac)):
    for variant in (6, 5, 4, 3, 2, 1, 0):
        eng.set_option("extract_variant", variant)
        d_img = torch.from_numpy(im).cuda()
        out = eng.extract_device(d_img, d_x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            eng.extract_device(d_img, d_x, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{tag:22s} variant {variant}: {ms:.3f} ms  {len(xycs) / ms * 1e3 / 1e6:.1f} M desc/s", flush=True)
eng.set_option("extract_variant", 5)
