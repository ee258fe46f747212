#!/bin/bash
# One-CTA (8 warps, 128x128) vs two-CTA (4 warps, 128x64, 2 per SM) leaf, unfused
# and with the bulk-reduction fold, on the bench configs (bench.py step time).
for cfg in ${CONFIGS:-c3-sw2-16384 x-sw3-16384 c2-sw1-4096 c4a-ld1-13824 c4b-sw2-13824}; do
  for v in "MF_LEAF_2CTA=0" "MF_LEAF_2CTA=1" "MF_LEAF_2CTA=0 FUSE=2" "MF_LEAF_2CTA=1 FUSE=2"; do
    fuse=""; case "$v" in *FUSE=2*) fuse="--fuse 2";; esac
    line=$(env ${v% FUSE=2} python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants $fuse 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': '$cfg', 'variant': '$v', 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],3), 'leaf_ms': round(r['ms_per_launch'],3), 'phases': {k: round(x,3) for k,x in r['phase_ms_per_step'].items()}, 'err': d.get('max_scaled_error'), 'clocks': d.get('clocks')}))" "$line"
  done
done
