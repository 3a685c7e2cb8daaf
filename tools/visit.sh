set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python tools/e2e_breakdown.py 2>&1 | tee $OUT/e2e_breakdown.log | grep -v "workers="
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json | python -c "import sys,json; d=json.load(sys.stdin); print({k:d[k] for k in ['value','ms_per_step','descriptors_per_s','compares_per_s','gpu_launches']}); print(d['e2e']['ms_per_step'], d['e2e_u8']['ms_per_step'])"
