python -m pytest tests/test_gpu_slab.py tests/test_gpu_plan.py -x -q > gpurun_out/t_slab.log 2>&1; tail -3 gpurun_out/t_slab.log
PBG_SLAB_CHUNKS=1 python -m pytest tests/test_gpu_slab.py -x -q > gpurun_out/t_slab1.log 2>&1; tail -2 gpurun_out/t_slab1.log
for n in 8 4 2; do python scripts/dev/slab_model.py $n; done > gpurun_out/slab_model.jsonl 2>&1; cat gpurun_out/slab_model.jsonl
PBG_SLAB_CHUNKS=1 python scripts/dev/slab_model.py 8 >> gpurun_out/slab_model.jsonl 2>&1; tail -1 gpurun_out/slab_model.jsonl
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode slab --steps 20 --warmup 3 --no-e2e > gpurun_out/bench_slab1.json 2> gpurun_out/bench_slab1.err; tail -1 gpurun_out/bench_slab1.json | cut -c1-300; tail -3 gpurun_out/bench_slab1.err
