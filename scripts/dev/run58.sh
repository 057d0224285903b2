python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t58.log 2>&1; tail -3 gpurun_out/t58.log
for B in 6 0 3; do
PBG_SLAB_BETA=$B python scripts/dev/slab_model.py 4 queued >> gpurun_out/slab58.jsonl 2>gpurun_out/slab58.err
done
cut -c1-330 gpurun_out/slab58.jsonl
