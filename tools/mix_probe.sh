#!/bin/bash
# Phase times of the table-driven K4/K6 (grouped vs term-list) against the
# compile-time specialised kernels, from bench.py's live phase events.
for cfg in c3-sw2-16384 c4a-ld1-13824 c4b-sw2-13824; do
  for mode in fixed jit generic generic-terms; do
    env=""
    [ "$mode" != fixed ] && env="MF_MIX_GENERIC=1"
    [ "$mode" = generic ] && env="$env MF_MIX_NOJIT=1"
    [ "$mode" = generic-terms ] && env="$env MF_MIX_NOJIT=1"
    [ "$mode" = generic-terms ] && env="$env MF_MIX_UNGROUPED=1"
    line=$(env $env python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-classical --no-variants 2>/dev/null | tail -n 1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'config': '$cfg', 'mix': '$mode', 'ms_per_step': round(d['ms_per_step'],3), 'phases': {k: round(v,3) for k,v in d['roofline']['phase_ms_per_step'].items()}}))" "$line"
  done
done
