#!/usr/bin/env python
"""Matcher throughput sweep on device-resident sets (CUDA events), per kernel variant."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

eng = get_engine()
shapes = [(2_000, 2_000), (8_000, 8_000), (10_000, 10_000), (20_000, 20_000), (100_000, 100_000), (20_000, 1_000_000),
          (1_000_000, 1_000_000)]
variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 3, 4]
rows = []
g = torch.Generator(device="cuda").manual_seed(0)
for q, n in shapes:
    dq = torch.randint(0, 256, (q, 64), dtype=torch.uint8, device="cuda", generator=g)
    dt = torch.randint(0, 256, (n, 64), dtype=torch.uint8, device="cuda", generator=g)
    ref = None
    for v in variants:
        eng.set_option("match_variant", v)
        if v == 1 and q * n > 2e10:
            continue
        out = eng.match_top2_device(dq, dt)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        same = bool(torch.equal(ref, out))
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            eng.match_top2_device(dq, dt, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        rows.append({"Q": q, "N": n, "variant": v, "ms": ms, "compares_per_s": q * n / ms * 1e3, "same_as_first": same})
        print(rows[-1], flush=True)
print(json.dumps(rows))
