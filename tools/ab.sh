# A/B of library builds on the config 5 step: tools/ab.sh name1 name2 ... (variants
# under paper_2210_04847_b200/lib/variants/libvoxmarch_b200_<name>.so; "main" = the
# default build), each timed twice, interleaved. Extra bench flags via $AB_FLAGS.
for rep in 1 2; do
  for n in "$@"; do
    if [ "$n" = main ]; then lib=paper_2210_04847_b200/lib/libvoxmarch_b200.so; else lib=paper_2210_04847_b200/lib/variants/libvoxmarch_b200_$n.so; fi
    VMB_LIB_PATH=$lib timeout 600 python bench.py --config1 0 --config2 0 --config3 0 --fields 0 --cpu-baseline 0 --steps 30 $AB_FLAGS \
      > gpurun_out/ab_${n}_$rep.json 2> gpurun_out/ab_${n}_$rep.err
    python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_${n}_$rep.json').read().strip().splitlines()[-1])
print('$n', $rep, round(d['ms_per_step'],4), {k: round(v,4) for k,v in d.get('phases_ms',{}).items()}, d['roofline']['step']['frac'] if 'roofline' in d else '', 'cfg2', round(d['config2']['ms_per_step'],4) if d.get('config2') else '')"
  done
done
