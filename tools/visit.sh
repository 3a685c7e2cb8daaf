set -u
OUT=gpurun_out/r1z; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > $OUT/bench_torchrun.json 2> $OUT/bench_torchrun.err; echo "torchrun bench rc=$?"; python -c "
import json;d=json.load(open('$OUT/bench_torchrun.json'));print(d['n_gpus'], d['ms_per_step'], d['e2e']['ms_per_step'], d['cpu_baseline'] is not None)"
tail -3 $OUT/bench_torchrun.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 | cut -c1-200
