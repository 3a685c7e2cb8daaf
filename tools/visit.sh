set -u
timeout 900 python -m pytest tests -m gpu -x -q -k "banded or promotion or golden" 2>&1 | tail -3
for b in 2 3 4; do echo "=== bands $b"; CLATCH_UPLOAD_BANDS=$b CLATCH_TRACE=1 python tools/trace_describe.py cfg2 2>&1 | grep -B2 "describe_all float64" | tail -3; done
echo "=== cfg3 f64"; for b in 1 2 4 6; do echo "bands $b"; CLATCH_UPLOAD_BANDS=$b CLATCH_TRACE=1 python tools/trace_describe.py cfg3 2>&1 | grep "describe_all float64" | tail -1; done
