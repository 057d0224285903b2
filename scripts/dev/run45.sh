python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py tests/test_gpu_scale.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/t45.log 2>&1; tail -5 gpurun_out/t45.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{}]' > gpurun_out/ab45.txt 2>&1; cat gpurun_out/ab45.txt
python scripts/dev/slab_model.py 8 queued > gpurun_out/slab45.jsonl 2>gpurun_out/slab45.err; cat gpurun_out/slab45.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_slab" -c 1200 --csv --log-file gpurun_out/slab_launches45.csv python scripts/dev/slab_model.py 8 > gpurun_out/ncu45.log 2>&1
