#!/usr/bin/env python
"""One matcher problem on device-resident random sets (for ncu captures): match_one.py Q N variant [reps]."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

q, n, v = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
eng = get_engine()
eng.set_option("match_variant", v)
eng.set_option("match_form_auto", 0)
g = torch.Generator(device="cuda").manual_seed(0)
dq = torch.randint(0, 256, (q, 64), dtype=torch.uint8, device="cuda", generator=g)
dt = torch.randint(0, 256, (n, 64), dtype=torch.uint8, device="cuda", generator=g)
out = eng.match_top2_device(dq, dt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    eng.match_top2_device(dq, dt, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print({"Q": q, "N": n, "variant": v, "ms": ms, "compares_per_s": q * n / ms * 1e3})
