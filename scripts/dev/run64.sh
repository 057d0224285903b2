TAG=r02d bash scripts/collect_round.sh > gpurun_out/collect64.log 2>&1
for N in 2 4 8; do python scripts/dev/slab_model.py $N queued >> gpurun_out/slab_model_r02d.jsonl 2>>gpurun_out/slab64.err; done
PBG_SLAB_BETA=0 python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab_model_r02d.jsonl 2>>gpurun_out/slab64.err
tail -3 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/bench_c4.json
