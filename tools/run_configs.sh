#!/bin/bash
# Runs every BASELINE config preset of bench.py once (1 GPU) -> gpurun_out/configs.jsonl
out=gpurun_out/configs.jsonl; [ -z "$CONFIG_APPEND" ] && : > $out
for c in ${CONFIG_LIST:-c1-sw1-64 c2-sw1-4096 c3-sw2-16384 c3b-sw1-16384 c4a-ld1-13824 c4b-sw2-13824 c5-sw2-32768 x-sw3-16384 x-ld2-13824 x-sw3-32768 x-swld-13824 x-ldsw-13824 x-sw2-49152-bounded x-sw4-16384-hybrid x-sw4-32768-hybrid x-sw5-32768-hybrid}; do
  extra=""
  case $c in c5-*|x-sw3-32768|x-sw2-49152-bounded|x-sw4-32768-hybrid|x-sw5-32768-hybrid) extra="--steps 3 --warmup 3 --no-e2e --no-variants";; c1-*) extra="--steps 50 --warmup 5";; c2-*) extra="--steps 20 --warmup 5";; esac
  timeout 900 python bench.py --config $c $extra --no-cpu --no-variants >> $out 2> gpurun_out/cfg_$c.err || echo "{\"preset\": \"$c\", \"failed\": true}" >> $out
done
python - <<'PY'
import json
for l in open('gpurun_out/configs.jsonl'):
    d=json.loads(l)
    if d.get('failed'): print(d); continue
    c=d['config']; r=d['roofline']; cl=d.get('classical',{})
    print(c['preset'], 'TF=%.2f ms=%.3f leaf_frac=%.3f cublas=%.2f speedup=%.3f err=%.2e e2e=%s' % (d['value'], d['ms_per_step'], r['frac'], cl.get('cublas_dgemm_tflops',0), d.get('speedup_vs_cublas',0), d.get('max_scaled_error',-1), d.get('e2e',{}).get('value')))
PY
