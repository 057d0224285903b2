PBG_RW96G=16 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_batch.py -x -q > gpurun_out/t12.log 2>&1; tail -2 gpurun_out/t12.log
for G in 8 16; do PBG_RW96G=$G python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_g$G.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5_g$G.json').read().strip().splitlines()[-1]); print($G, d['value']/1e9, d['config']['per_variant_ms_per_step'])"; done
