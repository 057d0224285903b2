python -m pytest tests -m gpu -x -q > gpurun_out/t_all14.log 2>&1; tail -3 gpurun_out/t_all14.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1; tail -2 gpurun_out/smoke14.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench14.json 2> gpurun_out/bench14.err; tail -1 gpurun_out/bench14.json
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/ref14.json 2> gpurun_out/ref14.err; tail -1 gpurun_out/ref14.json; tail -3 gpurun_out/ref14.err
