#!/bin/bash
# One-CTA vs two-CTA leaf (unfused) against the leaf side m: bench.py step time
# at (n, triple, levels) giving m = 512 .. 3072.
for spec in ${SPECS:-"4096 2" "8192 3" "8192 2" "16384 4" "2048 2" "4096 3" "12288 3" "6144 2" "8192 1"}; do
  set -- $spec
  for v in 0 1; do
    extra=""; [ "$1" = 16384 ] && [ "$2" = 4 ] && extra="--recurse-levels 1"
    line=$(MF_LEAF_2CTA=$v python bench.py --n $1 --levels $2 $extra --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu --no-classical --no-variants 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'n': $1, 'levels': $2, 'm': $1 >> $2, 'two_cta': $v, 'tflops': round(d['value'],3), 'ms_per_step': round(d['ms_per_step'],4)}))" "$line"
  done
done
