python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t50.log 2>&1; tail -3 gpurun_out/t50.log
for B in 0 6 4 8; do
PBG_SLAB_BETA=$B python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab50.jsonl 2>gpurun_out/slab50.err
done
python scripts/dev/slab_model.py 4 queued >> gpurun_out/slab50.jsonl 2>gpurun_out/slab50.err
python scripts/dev/slab_model.py 2 queued >> gpurun_out/slab50.jsonl 2>gpurun_out/slab50.err
cut -c1-420 gpurun_out/slab50.jsonl
