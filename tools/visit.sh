for d in 2 3 4 5 6; do echo "depth $d"; CLATCH_PIPE_DEPTH=$d python tools/extract_perf.py 2>&1 | grep "^u8 .*variant 3"; done
