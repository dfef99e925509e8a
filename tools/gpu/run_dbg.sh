export PYTHONUNBUFFERED=1
O=gpurun_out/r2c123; mkdir -p $O
for c in 1 2 3; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_c$c.json 2> $O/bench_c$c.err; echo "rc=$?" >> $O/bench_c$c.err; done
python -c "
import json
for c in (1,2,3):
    for l in open('$O/bench_c%d.json' % c):
        if l.startswith('{'):
            d=json.loads(l); print(c, round(d['value'],1), round(d['e2e']['value'],1), d['newton_iters'], d.get('cpu_baseline',{}).get('value'))"
