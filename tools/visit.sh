set -u
OUT=gpurun_out/r1z; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "match or knn or pairs or sets" 2>&1 | tail -5
timeout 300 python tools/sk_perf.py 2>&1 | tee $OUT/sk_perf.log
