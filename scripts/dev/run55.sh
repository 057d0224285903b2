python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t55.log 2>&1; tail -3 gpurun_out/t55.log
for B in 6 0; do
PBG_SLAB_BETA=$B python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab55.jsonl 2>gpurun_out/slab55.err
done
cut -c1-330 gpurun_out/slab55.jsonl
