timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/e27_tests.log 2>&1; tail -3 gpurun_out/e27_tests.log
for c in c2 c5 c1 c3 c4; do s=10; [ $c = c4 ] && s=3; [ $c = c3 ] && s=5; python bench.py --config $c --steps $s --no-cpu --no-g500 > gpurun_out/e27_$c.json 2> gpurun_out/e27_$c.err; done
for c in c2 c5 c1 c3 c4; do python -c "
import json; d=json.loads(open('gpurun_out/e27_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['config'].get('work_inflation'), d['roofline']['frac'], d['clocks'])"; done
