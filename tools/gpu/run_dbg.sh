# allocation poisoning at full size (C4): bootstrapped Newton parity, free-running steps, bench Newton count
export PYTHONUNBUFFERED=1
O=gpurun_out/r2poison; mkdir -p $O
MSIM_POISON=1 timeout 600 python -m pytest tests/test_gpu_newton_fullsize.py -q -rA -p no:cacheprovider -k "C4 or C3x10" > $O/c4_poison.log 2>&1; echo "rc=$?" >> $O/c4_poison.log
MSIM_POISON=1 timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_poison.json 2> $O/bench_poison.err; echo "rc=$?" >> $O/bench_poison.err
tail -8 $O/c4_poison.log; python -c "
import json
for l in open('$O/bench_poison.json'):
    if l.startswith('{'):
        d=json.loads(l); print('poison bench', d['value'], d['newton_iters'], d['e2e']['value'])"
