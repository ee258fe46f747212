#!/bin/bash
# Leaf variants on the bench configs: value, leaf ms per launch, error.
# usage: tools/leaf_probe.sh "ENV1=.. ENV2=.." "ENV=.." ...   (each arg one variant)
for cfg in ${CONFIGS:-c3-sw2-16384 c2-sw1-4096 c5-sw2-32768}; do
  for v in "$@"; do
    line=$(env $v python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': '$cfg', 'variant': '$v', 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],3), 'leaf_ms': round(r['ms_per_launch'],3), 'leaf_frac': round(r['frac'],4), 'err': d.get('max_scaled_error')}))" "$line"
  done
done
