#!/usr/bin/env python
"""Extraction rate on images with a saturated (exactly flat) left part: the default kernel with and without the
degenerate-image router, the all-fp64 quad kernel it routes to, and the share of windows that took the window-wide pass."""
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


def rate(d_img):
    out = eng.extract_device(d_img, d_x)
    for _ in range(40): eng.extract_device(d_img, d_x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(64): eng.extract_device(d_img, d_x, out=out)
    e1.record(); torch.cuda.synchronize()
    return len(xycs) / (e0.elapsed_time(e1) / 64) * 1e3 / 1e6


for frac in (0.0, 0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5, 0.7, 1.0):
    im = np.where(xx < int(w * frac), 255, img).astype(np.uint8)
    d_img = torch.from_numpy(im).cuda()
    eng.set_option("extract_variant", 5)
    eng.set_option("extract_stats", 1)
    eng.extract_device(d_img, d_x)
    torch.cuda.synchronize()
    _, passes = eng.extract_stats()
    eng.set_option("extract_stats", 0)
    eng.set_option("extract_route", 1)
    routed = rate(d_img)
    eng.set_option("extract_route", 0)
    plain = rate(d_img)
    eng.set_option("extract_variant", 1)
    quad = rate(d_img)
    print(f"saturated fraction {frac:.2f}: windows in the exact pass {passes / len(xycs):.3f}; default kernel {plain:.1f}, "
          f"quad kernel {quad:.1f}, with the router {routed:.1f} M desc/s", flush=True)
eng.set_option("extract_variant", 5)
eng.set_option("extract_route", 1)

# A caller that waits for every frame (describe() does): the router's probes of a degenerate stream thin out to one in 128.
flat = torch.full((h, w), 99, dtype=torch.uint8, device="cuda")
for label, variant, route in (("default kernel, router on", 5, 1), ("quad kernel", 1, 0)):
    eng.set_option("extract_variant", variant)
    eng.set_option("extract_route", route)
    out = eng.extract_device(flat, d_x)
    for _ in range(300):
        eng.extract_device(flat, d_x, out=out)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(512):
        eng.extract_device(flat, d_x, out=out)
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    print(f"flat frames, one at a time ({label}): {len(xycs) / (e0.elapsed_time(e1) / 512) * 1e3 / 1e6:.1f} M desc/s", flush=True)
eng.set_option("extract_variant", 5)
eng.set_option("extract_route", 1)
