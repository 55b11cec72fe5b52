# config 3 (cascade + cone) A/B of library variants: tools/c3_ab.sh name...
for rep in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then lib=paper_2210_04847_b200/lib/libvoxmarch_b200.so; else lib=paper_2210_04847_b200/lib/variants/libvoxmarch_b200_$n.so; fi
    VMB_LIB_PATH=$lib timeout 600 python bench.py --workload config3 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/c3ab_${n}_$rep.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/c3ab_${n}_$rep.json').read().strip().splitlines()[-1]); print('$n', $rep, round(d['ms_per_step'],3))"
  done
done
