python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t59.log 2>&1; tail -8 gpurun_out/t59.log
for N in 8 4 2; do
python scripts/dev/slab_model.py $N queued >> gpurun_out/slab59.jsonl 2>gpurun_out/slab59.err
done
PBG_SLAB_SPIKE=0 python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab59.jsonl 2>gpurun_out/slab59.err
cut -c1-330 gpurun_out/slab59.jsonl
