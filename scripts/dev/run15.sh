python -m pytest tests/test_gpu_shapes.py tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q > gpurun_out/t15.log 2>&1; tail -2 gpurun_out/t15.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWTMA": "0"}, {"PBG_ROWTMA": "2"}]' > gpurun_out/ab15.txt 2>&1; cat gpurun_out/ab15.txt
python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_15.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5_15.json').read().strip().splitlines()[-1]); print(d['value']/1e9, d['config']['per_variant_ms_per_step'])"
