TAG=r02c bash scripts/collect_round.sh > gpurun_out/collect56.log 2>&1
for N in 2 4 8; do python scripts/dev/slab_model.py $N queued >> gpurun_out/slab_model_r02c.jsonl 2>>gpurun_out/slab56.err; done
PBG_SLAB_BETA=0 python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab_model_r02c.jsonl 2>>gpurun_out/slab56.err
tail -3 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/bench_c4.json; cut -c1-200 gpurun_out/bench_ref.json
