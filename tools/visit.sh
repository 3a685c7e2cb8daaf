nproc; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/cpu.stat 2>/dev/null | head -6
cat > /tmp/t.py <<'PY'
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle, paper_1609_03986_b200 as lk
port = oracle.port(); eng = lk.get_engine(); eng.set_pattern(None)
W, H, N = 3840, 2160, 50000
img = port.random_image_u8(30000, W, H); kps = port.random_keypoints(31000, W, H, N)
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True); t.numpy()[...] = a; return t.numpy()
pimg, pkps = pinned(img), pinned(kps)
for workers in (0, 12, 8, 4, 2):
    ts=[]
    for i in range(8):
        t0=time.perf_counter(); r=eng.describe_batch([pimg]*8, [pkps]*8, workers); ts.append((time.perf_counter()-t0)*1e3)
    print(f"workers={workers}: describe_batch 8 images: min {min(ts):.2f} median {sorted(ts)[4]:.2f} max {max(ts):.2f} ms")
PY
python /tmp/t.py 2>&1 | tail -6
cat /sys/fs/cgroup/cpu.stat 2>/dev/null | head -6
