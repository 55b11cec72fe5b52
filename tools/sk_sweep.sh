# resident-step streams x sub-batches sweep for the given library variants
for n in "$@"; do
  if [ "$n" = main ]; then lib=paper_2210_04847_b200/lib/libvoxmarch_b200.so; else lib=paper_2210_04847_b200/lib/variants/libvoxmarch_b200_$n.so; fi
  for cfg in "2 2" "3 3" "4 4" "2 4" "3 6"; do
    set -- $cfg
    VMB_LIB_PATH=$lib timeout 300 python bench.py --config1 0 --config2 0 --config3 0 --fields 0 --cpu-baseline 0 --phases 0 --steps 30 --streams $1 --chunks $2 > gpurun_out/sk_${n}_$1_$2.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/sk_${n}_$1_$2.json').read().strip().splitlines()[-1])
print('$n S=$1 K=$2', round(d['ms_per_step'],4), d['pipeline']['matches_single_call_outputs'])"
  done
done
