set -u
OUT=gpurun_out/r1w; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "extraction_variant or filtered or golden or reference_vectors" > $OUT/pytest_sel.log 2>&1; echo "rc=$?"; tail -3 $OUT/pytest_sel.log
timeout 300 python tools/extract_perf.py 2>&1 | grep "variant [23]" | tee $OUT/extract_perf.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:extract_pipe -s 3 -c 1 -f -o $OUT/prof_extract_pipe \
    python bench.py --steps 2 --warmup 3 --phase extract --no-cpu-baseline > $OUT/ncu_extract.log 2>&1
