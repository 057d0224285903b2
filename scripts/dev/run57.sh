python -m pytest tests/test_gpu_shapes.py tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t57.log 2>&1; tail -3 gpurun_out/t57.log
for N in 8 4; do for P in 1 0; do
PBG_P4S20=$P python scripts/dev/slab_model.py $N queued >> gpurun_out/slab57.jsonl 2>gpurun_out/slab57.err
done; done
cut -c1-330 gpurun_out/slab57.jsonl
