# Round collection + the slab model at N = 2/4/8 (weighted) and 8 (equal slabs).
#   gpurun -- 'TAG=r02f bash scripts/dev/collect_final.sh'
TAG=${TAG:-rXX}
TAG=$TAG bash scripts/collect_round.sh > gpurun_out/collect_$TAG.log 2>&1
rm -f gpurun_out/slab_model_$TAG.jsonl
for N in 2 4 8; do python scripts/dev/slab_model.py $N queued >> gpurun_out/slab_model_$TAG.jsonl 2>>gpurun_out/slab_$TAG.err; done
PBG_SLAB_BETA=0 python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab_model_$TAG.jsonl 2>>gpurun_out/slab_$TAG.err
tail -3 gpurun_out/pytest_gpu.log; cut -c1-300 gpurun_out/bench_c4.json
