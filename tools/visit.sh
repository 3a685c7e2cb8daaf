set -u
OUT=gpurun_out/r1w; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "extraction_variant or filtered or golden or reference_vectors" > $OUT/pytest_sel.log 2>&1; echo "rc=$?"; tail -3 $OUT/pytest_sel.log
timeout 300 python tools/extract_perf.py 2>&1 | grep "variant [23]" | tee $OUT/extract_perf.log
