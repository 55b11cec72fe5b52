# resident-step schedule sweep: streams x sub-batches, with and without the skew
for cfg in "2 2 0" "2 2 1" "2 4 1" "2 8 1" "3 6 1" "2 4 0" "4 8 1"; do
  set -- $cfg
  timeout 300 python bench.py --config1 0 --config2 0 --config3 0 --fields 0 --cpu-baseline 0 --steps 30 --streams $1 --chunks $2 --skew $3 > gpurun_out/skew_$1_$2_$3.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/skew_$1_$2_$3.json').read().strip().splitlines()[-1])
print('S=$1 K=$2 skew=$3', round(d['ms_per_step'],4), d['pipeline'])"
done
