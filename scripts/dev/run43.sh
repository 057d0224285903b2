python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t43.log 2>&1; tail -5 gpurun_out/t43.log
for P4 in 0 1; do for Q in plain queued; do
PBG_P4=$P4 python scripts/dev/slab_model.py 8 $Q >> gpurun_out/slab43.jsonl 2>gpurun_out/slab43.err
done; done
cat gpurun_out/slab43.jsonl
