#!/usr/bin/env python
"""How often the estimate-based extraction kernels fall back to the exact fp64 chains, by image kind."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench                                    # noqa: E402
import oracle                                   # noqa: E402
import paper_1609_03986_b200 as lk              # noqa: E402

port = oracle.port()
eng = lk.get_engine()
img, kps = bench.synth_inputs("cfg2")
h, w = img.shape
rng = np.random.default_rng(7)
yy, xx = np.mgrid[0:h, 0:w]
smooth = (127.5 + 60 * np.sin(xx / 37.0) * np.cos(yy / 23.0) + 40 * np.sin((xx + yy) / 11.0)).round().astype(np.uint8)
images = {
    "cfg2 uniform noise": img,
    "structured (flat regions + edges)": port.structured_image(3986, w, h).astype(np.uint8),
    "smooth sinusoids": smooth,
    "smooth + 2 grey levels of noise": (smooth.astype(int) + rng.integers(-2, 3, smooth.shape)).clip(0, 255).astype(np.uint8),
    "half saturated": np.where(xx < w // 2, 255, img).astype(np.uint8),
    "flat": np.full((h, w), 99, np.uint8),
}
for variant in (5, 50, 6, 4, 3, 2, 1):          # 50 = variant 5 with the degenerate-image router switched off
    eng.set_option("extract_variant", 5 if variant == 50 else variant)
    eng.set_option("extract_route", 0 if variant == 50 else 1)
    for name, im in images.items():
        eng.set_option("extract_stats", 1)
        m = len(lk.describe(im, kps)[1])
        exact, passes = eng.extract_stats() if variant >= 2 else (0, 0)
        if variant in (4, 5, 6):
            eng.set_option("extract_route", 1)      # (resets the router's state between image kinds)
        unit = "windows re-resampled" if variant >= 3 else "warp passes"
        eng.set_option("extract_stats", 0)
        xycs, _ = eng.prepare_keypoints(kps, w, h)
        d_img, d_x = torch.from_numpy(im).cuda(), torch.from_numpy(xycs).cuda()
        out = eng.extract_device(d_img, d_x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            eng.extract_device(d_img, d_x, out=out)
        e1.record()
        torch.cuda.synchronize()
        rate = len(xycs) / (e0.elapsed_time(e1) / 10) * 1e3 / 1e6
        print(f"variant {'5 (router off)' if variant == 50 else variant}  {name:36s} exact triplets {exact:9d} of {m * 512} = {exact / (m * 512):.2e}; "
              f"{unit}: {passes} ({passes / m:.3f} per descriptor); {rate:.1f} M desc/s", flush=True)
eng.set_option("extract_stats", 0)
eng.set_option("extract_variant", 5)
eng.set_option("extract_route", 1)
