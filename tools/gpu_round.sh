#!/usr/bin/env bash
# One GPU-box visit: smoke, GPU parity tests, pipe-rate microbench, bench (both arms),
# ncu launch list and one full capture per hot kernel. Everything lands in gpurun_out/.
# Usage (from the build container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
set -u
TAG="${1:-r1}"
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" | tee -a "$OUT/smoke.log"
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" | tee -a "$OUT/pytest_gpu.log"
tail -5 "$OUT/pytest_gpu.log"
echo "== pipe peaks"; timeout 120 ./tools/pipe_peaks > "$OUT/pipe_peaks.json" 2> "$OUT/pipe_peaks.err"; cat "$OUT/pipe_peaks.json"
echo "== bench ours"; timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; cat "$OUT/bench.json"; tail -3 "$OUT/bench.err"
if [ "${VARIANTS:-0}" = "1" ]; then
for v in 0 1 2 3 4; do
  echo "== extraction variant $v"
  timeout 300 python bench.py --steps 20 --warmup 5 --phase extract --no-cpu-baseline --extract-variant $v > "$OUT/bench_extract_v$v.json" 2>> "$OUT/bench.err"
  python -c "import json;d=json.load(open('$OUT/bench_extract_v$v.json'));print('extract variant $v desc/s', d['descriptors_per_s'])"
done
for v in 0 1 2 3; do
  echo "== matcher variant $v"
  timeout 300 python bench.py --steps 20 --warmup 5 --phase match --no-cpu-baseline --match-variant $v > "$OUT/bench_match_v$v.json" 2>> "$OUT/bench.err"
  python -c "import json;d=json.load(open('$OUT/bench_match_v$v.json'));print('variant $v compares/s', d['compares_per_s'], 'ms', list(d['kernels'].values())[0]['ms'])"
done
fi
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; cat "$OUT/bench_reference.json"
if [ "${SKIP_NCU:-0}" != "1" ]; then
echo "== ncu launch list"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
echo "== ncu full: extraction"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:extract_roles -s 3 -c 1 -f -o "$OUT/prof_extract" \
    python bench.py --steps 2 --warmup 3 --phase extract --no-cpu-baseline > "$OUT/ncu_extract.log" 2>&1
echo "== ncu full: tensor-core matching"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -f -o "$OUT/prof_match_tc" \
    python bench.py --steps 2 --warmup 3 --phase match --no-cpu-baseline --match-variant 3 > "$OUT/ncu_match_tc.log" 2>&1
echo "== e2e breakdown, extraction by image kind, configs 3-5"
timeout 300 python tools/e2e_breakdown.py > "$OUT/e2e_breakdown.log" 2>&1
timeout 300 python tools/extract_perf.py > "$OUT/extract_perf.log" 2>&1
timeout 900 python tools/run_configs.py > "$OUT/configs.json" 2> "$OUT/configs.err"
timeout 120 ./tools/tex_probe > "$OUT/tex_probe.json" 2>&1
timeout 120 ./tools/lat_probe > "$OUT/lat_probe.json" 2>&1
timeout 300 python tools/sk_perf.py > "$OUT/sk_perf.log" 2>&1
timeout 600 python tools/cfg3_breakdown.py > "$OUT/cfg3_breakdown.log" 2>&1
echo "== compute-sanitizer"
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > "$OUT/sanitize_memcheck.log" 2>&1; tail -2 "$OUT/sanitize_memcheck.log"
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize.py > "$OUT/sanitize_racecheck.log" 2>&1; tail -2 "$OUT/sanitize_racecheck.log"
fi
ls -la "$OUT"
