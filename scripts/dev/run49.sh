python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t49.log 2>&1; tail -3 gpurun_out/t49.log
for CH in 4 2 1; do
PBG_SLAB_CHUNKS=$CH python scripts/dev/slab_model.py 8 queued >> gpurun_out/slab49.jsonl 2>gpurun_out/slab49.err
done
cat gpurun_out/slab49.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_slab" -c 100 --csv --log-file gpurun_out/slab_launches49_warm.csv python scripts/dev/slab_model.py 8 > gpurun_out/ncu49.log 2>&1
grep k_slab_interface gpurun_out/slab_launches49_warm.csv | tail -3 | awk -F'","' '{print $NF}'
