#!/bin/bash
# A/B a bench environment switch on the GPU box:  tools/ab.sh <tiles> <VAR> <val_a> <val_b> [bench args]
tiles=$1; var=$2; a=$3; b=$4; shift 4
for val in $a $b $a $b; do
  env $var=$val timeout 600 python bench.py --tiles $tiles --steps 100 --warmup 10 --no-cpu --no-f64 --e2e-steps 0 \
    --amortised-steps 0 --prof-steps 8 "$@" 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d['kernel_ms_per_step']
    print('$var=$val', round(d['value'],1), 'ms/step', round(d['ms_per_step'],3), 'ss', round(k['k_contacts_ss'],3), 'int', round(k['k_integrate'],3), 'kT/cyc', round(k['kT_per_cycle'],3))"
done
