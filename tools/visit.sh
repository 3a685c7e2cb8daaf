mkdir -p gpurun_out/r1z; timeout 600 python tools/exact_rate.py 2>&1 | tee gpurun_out/r1z/exact_rate.log
