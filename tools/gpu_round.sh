#!/usr/bin/env bash
# One full GPU-box visit: smoke, GPU parity tests, pipe / tensor microbenchmarks, bench (both arms), the NCCL path at
# world size 1, ncu launch list and one full capture per hot kernel, breakdown tools, soak, sanitizer.
# Usage (from the build container): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh <tag>'
set -u
TAG="${1:-r3}"
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
(nproc; free -g) > "$OUT/host.txt" 2>&1
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" | tee -a "$OUT/smoke.log"
echo "== pytest -m gpu"; timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" | tee -a "$OUT/pytest_gpu.log"; tail -4 "$OUT/pytest_gpu.log"
echo "== microbenchmarks"
timeout 120 ./tools/pipe_peaks > "$OUT/pipe_peaks.json" 2> "$OUT/pipe_peaks.err"
timeout 120 ./tools/tc_peak > "$OUT/tc_peak.json" 2>&1
timeout 120 ./tools/tmem_ld_probe > "$OUT/tmem_ld_probe.json" 2>&1
timeout 120 ./tools/tmem_contention > "$OUT/tmem_contention.json" 2>&1
timeout 120 ./tools/tc_pair_probe > "$OUT/tc_pair_probe.json" 2>&1
timeout 120 ./tools/tex_probe > "$OUT/tex_probe.json" 2>&1
echo "== bench ours"; timeout 900 python bench.py --steps 20 --warmup 5 > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"; tail -6 "$OUT/bench.err"
echo "== bench reference"; timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "rc=$?"
echo "== torchrun world size 1 (NCCL path)"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > "$OUT/bench_torchrun1.json" 2> "$OUT/bench_torchrun1.err"; echo "rc=$?"
echo "== matcher sweep"; timeout 600 python tools/match_perf.py 1,3,4 > "$OUT/match_perf.log" 2>&1
timeout 300 python tools/pairs_one.py 32 8000 3 > "$OUT/pairs_perf.log" 2>&1
for s in "2000 2000" "10000 10000" "100000 100000" "1000000 1000000"; do CLATCH_TC_TRACE=1 timeout 300 python tools/match_one.py $s 4 1 2>&1 | grep "tc trace" | tail -1; done > "$OUT/match_trace.log"
if [ "${SKIP_NCU:-0}" != "1" ]; then
echo "== ncu launch list"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" \
    python bench.py --workload cfg2 --steps 2 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
echo "== ncu full: extraction"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:extract_h16_kernel -s 3 -c 1 -f -o "$OUT/prof_extract" \
    python bench.py --workload cfg2 --steps 2 --warmup 3 --phase extract --no-cpu-baseline > "$OUT/ncu_extract.log" 2>&1
echo "== ncu full: tensor-core matching (cfg2 size, 100k x 100k, batched pairs)"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 3 -c 1 -f -o "$OUT/prof_match_tc" \
    python bench.py --workload cfg2 --steps 2 --warmup 3 --phase match --no-cpu-baseline > "$OUT/ncu_match_tc.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 1 -c 1 -f -o "$OUT/prof_match_tc_100k" python tools/match_one.py 100000 100000 4 1 > "$OUT/ncu_match_100k.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:match_tc -s 1 -c 1 -f -o "$OUT/prof_match_tc_pairs" python tools/pairs_one.py 32 8000 1 > "$OUT/ncu_match_pairs.log" 2>&1
fi
if [ "${SKIP_EXTRA:-0}" != "1" ]; then
echo "== e2e breakdown, extraction by image kind"
timeout 300 python tools/e2e_breakdown.py > "$OUT/e2e_breakdown.log" 2>&1
timeout 300 python tools/extract_perf.py > "$OUT/extract_perf.log" 2>&1
timeout 300 python tools/exact_rate.py > "$OUT/exact_rate.log" 2>&1
echo "== soak"; timeout 700 python tools/soak.py 420 > "$OUT/soak.log" 2>&1; tail -2 "$OUT/soak.log"
echo "== compute-sanitizer"
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py all > "$OUT/sanitize_memcheck.log" 2>&1; tail -2 "$OUT/sanitize_memcheck.log"
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize.py > "$OUT/sanitize_racecheck.log" 2>&1; tail -2 "$OUT/sanitize_racecheck.log"
fi
ls -la "$OUT"
