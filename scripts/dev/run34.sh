python -m pytest tests -m gpu -x -q > gpurun_out/t34.log 2>&1; tail -3 gpurun_out/t34.log
python bench.py --steps 20 --warmup 5 > gpurun_out/b34_c4.json 2> gpurun_out/b34_c4.err; tail -c 400 gpurun_out/b34_c4.json
python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b34_c3.json 2> gpurun_out/b34_c3.err; tail -c 300 gpurun_out/b34_c3.json
python bench.py --config c5 --steps 100 --warmup 5 > gpurun_out/b34_c5.json 2> gpurun_out/b34_c5.err; tail -c 300 gpurun_out/b34_c5.json
