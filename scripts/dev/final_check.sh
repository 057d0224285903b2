# Round-end rehearsal: what the driver runs (GPU tests, smoke, both bench arms with its flags).
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; tail -2 gpurun_out/final_smoke.log
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -4 gpurun_out/final_ref.err; cut -c1-300 gpurun_out/final_ref.json
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -4 gpurun_out/final_bench.err; cut -c1-300 gpurun_out/final_bench.json
