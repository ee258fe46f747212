#!/bin/bash
# One-CTA vs two-CTA leaf (unfused) against the leaf side m: bench.py step time
# at (n, levels) of Strassen-Winograd.  SPECS="n:levels n:levels ..."; VARIANTS="0 1 d"
# (d = the library's default choice)
for spec in ${SPECS:-4096:2 8192:3 8192:2 2048:2 4096:3 12288:3 6144:2 8192:1}; do
  n=${spec%%:*}; lv=${spec##*:}
  for v in ${VARIANTS:-0 1}; do
    if [ "$v" = d ]; then envs=""; else envs="MF_LEAF_2CTA=$v"; fi
    line=$(env $envs python bench.py --n $n --levels $lv --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'n': $n, 'levels': $lv, 'm': $n >> $lv, 'two_cta': '$v', 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],4)}))" "$line"
  done
done
