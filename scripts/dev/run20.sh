python -m pytest tests -m gpu -x -q > gpurun_out/t20.log 2>&1; tail -3 gpurun_out/t20.log
python bench.py --steps 20 --warmup 5 > gpurun_out/b20_c4.json 2> gpurun_out/b20_c4.err; tail -c 600 gpurun_out/b20_c4.json
python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/b20_c3.json 2> gpurun_out/b20_c3.err; tail -c 300 gpurun_out/b20_c3.json
