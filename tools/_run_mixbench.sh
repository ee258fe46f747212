for rep in 1 2; do for eager in 0 1; do for c in c3-sw2-16384 x-sw3-16384; do
  if [ $eager = 1 ]; then export MF_E2E_EAGER_D2H=1; else unset MF_E2E_EAGER_D2H; fi
  timeout 300 python bench.py --config $c --no-cpu --no-classical --no-variants --steps 4 > gpurun_out/e.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e.json')); print('rep$rep eager=$eager $c', round(d['value'],2), round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],1))"
done; done; done
