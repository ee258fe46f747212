#!/bin/bash
# Leaf shapes under the proxy-fenced ring: unfused, ordered fold on one / two
# CTAs per SM, bulk fold; bench.py step time.
for cfg in ${CONFIGS:-c3-sw2-16384 x-sw3-16384 x-sw4-16384-hybrid}; do
  for v in "MF_LEAF_2CTA=0|" "MF_LEAF_2CTA=1|" "MF_LEAF_2CTA=0|--fuse 1" "MF_LEAF_2CTA=1|--fuse 1" "MF_LEAF_2CTA=1|--fuse 2"; do
    envs=${v%%|*}; args=${v#*|}
    line=$(env $envs python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants $args 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': '$cfg', 'variant': '$envs $args'.strip(), 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],3), 'leaf_ms': round(r['ms_per_launch'],3), 'err': d.get('max_scaled_error'), 'bitwise_equal_unfused': d.get('bitwise_equal_unfused'), 'clocks': d.get('clocks')}))" "$line"
  done
done
