# config 2 schedule sweep (streams x sub-batches)
for cfg in "1 1" "2 2" "2 1" "3 3" "4 4" "2 4"; do
  set -- $cfg
  timeout 300 python bench.py --width 512 --step-size 0.0016914558667664816 --steps 50 --config1 0 --config2 0 --config3 0 --config4 0 --fields 0 --res256 0 --cpu-baseline 0 --phases 0 --streams $1 --chunks $2 > gpurun_out/c2s_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c2s_$1_$2.json').read().strip().splitlines()[-1]); print('c2 S=$1 K=$2', round(d['ms_per_step'],4))"
done
