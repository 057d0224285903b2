python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_batch.py tests/test_gpu_slab.py -x -q > gpurun_out/t40.log 2>&1; tail -3 gpurun_out/t40.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_PDL": "0"}, {}]' > gpurun_out/ab40.txt 2>&1; cat gpurun_out/ab40.txt
