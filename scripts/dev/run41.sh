python -m pytest tests/test_gpu_batch.py tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t41.log 2>&1; tail -5 gpurun_out/t41.log
python scripts/dev/c5_axes.py > gpurun_out/c5axes41.txt 2>&1; cat gpurun_out/c5axes41.txt
PBG_ROWLEAN=0 python scripts/dev/c5_axes.py > gpurun_out/c5axes41b.txt 2>&1; cat gpurun_out/c5axes41b.txt
python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{}]' > gpurun_out/ab41.txt 2>&1; cat gpurun_out/ab41.txt
