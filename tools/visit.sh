set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "recycled or describe or batch or golden" 2>&1 | tail -3
timeout 900 python tools/run_configs.py > $OUT/configs.json 2> $OUT/configs.err; python -c "
import json;c=json.load(open('$OUT/configs.json'));print(c['cfg3']['kernel_descriptors_per_s'],c['cfg3']['batch_e2e_descriptors_per_s'],c['cfg3']['e2e_descriptors_per_s'],c['cfg4']['compares_per_s'],c['cfg5']['batched']['pairs_per_s'], c['cfg5']['pairs_per_s'])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline | python -c "import sys,json; d=json.load(sys.stdin); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_u8']['ms_per_step'])"
