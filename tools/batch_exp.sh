# design tool (GPU): cfg2 batch throughput over "batch,workers,budget" triples in $SPECS
for spec in ${SPECS:-"16,8,32"}; do IFS=, read b w s <<< "$spec"; python bench.py --config cfg2 --batch $b --batch-workers $w --batch-sm-budget $s --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-by-config ${NOE2E:+--no-e2e} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=d['e2e']['value'] if d.get('e2e') else float('nan')
print('$ENVX batch $b workers $w budget $s: value %.1f ms/step %.3f e2e %.1f' % (d['value'], d['ms_per_step'], e))
"; done
