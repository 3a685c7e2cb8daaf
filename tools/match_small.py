#!/usr/bin/env python
"""One small self-match on device-resident descriptors, L2 flushed between calls: median / min time of
match_top2_device (expansion + tensor-core kernel + merge), by `pdl` setting.

    CLATCH_MATCH_STREAMK_PAIRS=0|1 python tools/match_small.py [rows]
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
eng = get_engine()
g = torch.Generator(device="cuda").manual_seed(0)
d = torch.randint(0, 256, (n, 64), dtype=torch.uint8, device="cuda", generator=g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for pdl in (1, 0):
    eng.set_option("pdl", pdl)
    out = eng.match_top2_device(d, d)
    torch.cuda.synchronize()
    ts = []
    for _ in range(40):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.match_top2_device(d, d, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{n} x {n}  pdl={pdl}: median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f} us", flush=True)
eng.set_option("pdl", 1)
