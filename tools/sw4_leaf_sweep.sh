#!/bin/bash
# Leaf shape at m = 1024 (the SW^4 hybrid's children): one-CTA 128x128 vs two-CTA
# 128x64 and rasterisation group sizes, bench.py step time.
for v in "MF_LEAF_2CTA=0" "MF_LEAF_2CTA=1" "MF_LEAF_GROUPM=4" "MF_LEAF_GROUPM=16" "MF_LEAF_KSUB=1"; do
  line=$(env $v python bench.py --config ${CFG:-x-sw4-16384-hybrid} --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants 2>/dev/null | tail -n 1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'variant': '$v', 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],3), 'clocks': d.get('clocks')}))" "$line"
done
