#!/usr/bin/env bash
# A short GPU-box visit: smoke, GPU parity tests, both bench arms, the NCCL path at world size 1.
# Usage: gpurun --timeout 2400 -- 'bash tools/gpu_visit.sh <tag> [skip-tests]'
set -u
TAG="${1:-v}"
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
(nproc; free -g) > "$OUT/host.txt" 2>&1
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" | tee -a "$OUT/smoke.log"
if [ "${2:-}" != "skip-tests" ]; then
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" | tee -a "$OUT/pytest_gpu.log"
tail -25 "$OUT/pytest_gpu.log"
fi
echo "== bench ours"; timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; tail -8 "$OUT/bench.err"
python - "$OUT/bench.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
except Exception as e:
    print("bench line unreadable:", e); sys.exit(0)
print("headline", d["value"], d["unit"][:20], "ms", d["ms_per_step"], "e2e ms", d["e2e"]["ms_per_step"], "pageable", d.get("e2e_pageable", {}).get("ms_per_step"), "u8", d.get("e2e_u8", {}).get("ms_per_step"))
print("roofline", d["roofline"]["kernel"], d["roofline"]["bound"], round(d["roofline"]["frac"], 3))
for k, c in d.get("configs", {}).items():
    print(k, "%.4g" % c["value"], c["unit"][:24], "ms %.3f" % c["ms_per_step"], "e2e %.4g (%.3f ms)" % (c["e2e"]["value"], c["e2e"].get("ms_per_step", 0)),
          "u8 e2e %.4g" % c["e2e_u8"]["value"] if "e2e_u8" in c else "", "roof", round(c.get("roofline", {}).get("frac", 0), 3),
          "cpu %.4g" % c["cpu_baseline"]["value"] if c.get("cpu_baseline") else "", "wall", c.get("bench_wall_s"))
PY
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "rc=$?"; cut -c1-600 "$OUT/bench_reference.json"
echo "== torchrun world size 1 (NCCL path)"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_torchrun1.json" 2> "$OUT/bench_torchrun1.err"; echo "rc=$?"; tail -3 "$OUT/bench_torchrun1.err"; cut -c1-300 "$OUT/bench_torchrun1.json"
ls -la "$OUT"
