set -u
OUT=gpurun_out/r1z; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "extraction_variant or filtered" 2>&1 | tail -5
timeout 300 python tools/extract_perf.py 2>&1 | grep "^u8" | tee $OUT/extract_perf.log
