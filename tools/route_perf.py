#!/usr/bin/env python
"""Extraction rate on images with a saturated (exactly flat) left part, with and without the degenerate-image router."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import bench, paper_1609_03986_b200 as lk
eng = lk.get_engine()
eng.set_pattern(None)
img, kps = bench.synth_inputs("cfg2")
h, w = img.shape
yy, xx = np.mgrid[0:h, 0:w]
xycs, _ = eng.prepare_keypoints(kps, w, h)
d_x = torch.from_numpy(xycs).cuda()
for frac in (0.0, 0.1, 0.2, 0.3, 0.5):
    im = np.where(xx < int(w * frac), 255, img).astype(np.uint8)
    d_img = torch.from_numpy(im).cuda()
    for route in (1, 0):
        eng.set_option("extract_route", route)
        out = eng.extract_device(d_img, d_x)
        for _ in range(20): eng.extract_device(d_img, d_x, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(32): eng.extract_device(d_img, d_x, out=out)
        e1.record(); torch.cuda.synchronize()
        print(f"saturated fraction {frac:.1f} router {route}: {len(xycs) / (e0.elapsed_time(e1) / 32) * 1e3 / 1e6:.1f} M desc/s", flush=True)
eng.set_option("extract_route", 1)
