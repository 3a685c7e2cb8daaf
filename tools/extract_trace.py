#!/usr/bin/env python
"""Per-CTA timeline of the default extraction kernel (CLATCH_EX_TRACE=1) by image kind and keypoint count.

Usage: CLATCH_EX_TRACE=1 python tools/extract_trace.py   — the library prints one line per launch on stderr.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

os.environ.setdefault("CLATCH_EX_TRACE", "1")
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench                                    # noqa: E402
import paper_1609_03986_b200 as lk              # noqa: E402

eng = lk.get_engine()
eng.set_pattern(None)
eng.set_option("extract_route", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in ("cfg2", "cfg3"):
    img, kps = bench.synth_inputs(cfg)
    h, w = img.shape
    yy, xx = np.mgrid[0:h, 0:w]
    smooth = (127.5 + 60 * np.sin(xx / 37.0) * np.cos(yy / 23.0) + 40 * np.sin((xx + yy) / 11.0)).round().astype(np.uint8)
    xycs, _ = eng.prepare_keypoints(kps, w, h)
    d_x = torch.from_numpy(xycs).cuda()
    for name, im in (("noise", img), ("smooth", smooth)):
        d_img = torch.from_numpy(im).cuda()
        out = eng.extract_device(d_img, d_x)
        torch.cuda.synchronize()
        for rep in range(3):
            flush.zero_()
            torch.cuda.synchronize()
            print(f"== {cfg} {name} ({len(xycs)} keypoints), launch {rep}", file=sys.stderr, flush=True)
            eng.extract_device(d_img, d_x, out=out)
            torch.cuda.synchronize()
