for E in "PBG_ROWWARP=1" "PBG_ROWWARP=0" "PBG_INPLACE=0" "PBG_INPLACE=1"; do env $E python bench.py --config c5 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_e.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/c5_e.json').read().strip().splitlines()[-1]); print('$E', d['value']/1e9, d['config']['per_variant_ms_per_step'])"; done
