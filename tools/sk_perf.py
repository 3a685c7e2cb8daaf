#!/usr/bin/env python
"""Tensor matcher: (query tile, split) rounds vs stream-K on single CTAs vs stream-K on CTA pairs, small self-matches
(CUDA events)."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

eng = get_engine()
g = torch.Generator(device="cuda").manual_seed(0)
for q, n in [(2000, 2000), (4000, 4000), (8000, 8000), (10000, 10000), (20000, 20000), (30000, 30000), (50000, 50000), (5000, 90000)]:
    dq = torch.randint(0, 256, (q, 64), dtype=torch.uint8, device="cuda", generator=g)
    dt = dq if q == n else torch.randint(0, 256, (n, 64), dtype=torch.uint8, device="cuda", generator=g)
    for sk in (0, 1, 2):
        eng.set_option("match_streamk", 1 if sk else 0)
        eng.set_option("match_streamk_pairs", 1 if sk == 2 else 0)
        out = eng.match_top2_device(dq, dt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            eng.match_top2_device(dq, dt, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{q:6d} x {n:6d}  streamk={sk} (0 rounds, 1 single CTAs, 2 CTA pairs): {ms * 1e3:8.1f} us  {q * n / ms * 1e3:.3e} compares/s", flush=True)
eng.set_option("match_streamk", 1)
eng.set_option("match_streamk_pairs", 0)
