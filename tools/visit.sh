set -u
OUT=gpurun_out/r1z; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "pairs or sets or match" 2>&1 | tail -8
timeout 900 python tools/run_configs.py > $OUT/configs2.json 2> $OUT/configs2.err; python -c "
import json;c=json.load(open('$OUT/configs2.json'));print(c['cfg3']['kernel_descriptors_per_s'],c['cfg3']['batch_e2e_descriptors_per_s'],c['cfg3']['e2e_descriptors_per_s']);print(c['cfg5']); print(c['cfg5_detail'])"
