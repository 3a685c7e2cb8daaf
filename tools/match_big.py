#!/usr/bin/env python
"""One large device-resident match (for ncu): python tools/match_big.py [Q] [N]"""
import sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1609_03986_b200.engine import get_engine   # noqa: E402
q, n = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (60000, 60000)
eng = get_engine()
g = torch.Generator(device="cuda").manual_seed(0)
dq = torch.randint(0, 256, (q, 64), dtype=torch.uint8, device="cuda", generator=g)
dt = torch.randint(0, 256, (n, 64), dtype=torch.uint8, device="cuda", generator=g)
for _ in range(3):
    out = eng.match_top2_device(dq, dt)
torch.cuda.synchronize()
print("done", out.shape)
