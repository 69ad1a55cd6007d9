#!/bin/bash
# A/B of one environment switch inside bench.py (precond kernel times and the step rate):
#   bash tools/ab_bench.sh VAR "val1 val2 ..." [steps]
var=$1; vals=$2; steps=${3:-3}
for v in $vals; do
  env $var=$v python bench.py --steps $steps --no-e2e 2>/dev/null | tail -1 | python -c "
import json, sys; d = json.loads(sys.stdin.read()); k = d['precond_kernels']
print('$var=$v', d['value'], {n: k[n]['ms'] for n in k})"
done
