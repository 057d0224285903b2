# Round collection on the GPU box: tests, bench lines, ncu launch list and full capture.
#   gpurun -- 'TAG=r01e bash scripts/collect_round.sh'
set -x
TAG=${TAG:-rXX}
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --mode slab --steps 20 --warmup 3 > gpurun_out/bench_slab1.json 2> gpurun_out/bench_slab1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 9 -c 3 -o gpurun_out/c4_full_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 9 -c 3 -o gpurun_out/c3_full_$TAG python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c3.log 2>&1
# the two reports together exceed gpurun's 64 MiB copy-back: keep their raw pages only
for c in c4 c3; do
  ncu -i gpurun_out/${c}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${c}_full_${TAG}_raw.csv 2>/dev/null && rm -f gpurun_out/${c}_full_$TAG.ncu-rep
done
