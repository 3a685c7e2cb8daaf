set -u
OUT=gpurun_out/r1v; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "extraction_variant or filtered or golden or reference_vectors" > $OUT/pytest_sel.log 2>&1; echo "rc=$?"; tail -15 $OUT/pytest_sel.log
for v in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --phase extract --no-cpu-baseline --extract-variant $v > $OUT/bench_extract_v$v.json 2>> $OUT/bench.err
python -c "import json;d=json.load(open('$OUT/bench_extract_v$v.json'));print('extract variant $v desc/s', d['descriptors_per_s'])"
done
timeout 300 python tools/extract_perf.py 2>&1 | tee $OUT/extract_perf.log
