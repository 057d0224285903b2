python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t53.log 2>&1; tail -5 gpurun_out/t53.log
for B in 6 0; do
PBG_SLAB_BETA=$B python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab53.jsonl 2>gpurun_out/slab53.err
done
PBG_SLAB_ENDS=0 python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab53.jsonl 2>gpurun_out/slab53.err
cut -c1-420 gpurun_out/slab53.jsonl
