# config 1 (4096 rays, CUDA graph) A/B of library variants
for rep in 1 2; do for n in "$@"; do
  if [ "$n" = main ]; then lib=paper_2210_04847_b200/lib/libvoxmarch_b200.so; else lib=paper_2210_04847_b200/lib/variants/libvoxmarch_b200_$n.so; fi
  VMB_LIB_PATH=$lib timeout 300 python bench.py --workload config1 --steps 200 --warmup 20 > gpurun_out/c1ab_${n}_$rep.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/c1ab_${n}_$rep.json').read().strip().splitlines()[-1]); print('$n', $rep, round(d['ms_per_step']*1e3,2), 'us graph;', round(d.get('calls_ms_per_step',0)*1e3,2), 'us calls')"
done; done
