python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t51.log 2>&1; tail -3 gpurun_out/t51.log
for B in 6 4 3; do
PBG_SLAB_BETA=$B python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab51.jsonl 2>gpurun_out/slab51.err
done
cut -c1-420 gpurun_out/slab51.jsonl
