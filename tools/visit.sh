set -u
OUT=gpurun_out/r1z; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -k "trained_pattern or custom_patterns" 2>&1 | tail -15
