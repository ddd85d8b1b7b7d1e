set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/gputest_r02e.txt 2>&1
tail -5 gpurun_out/gputest_r02e.txt
for c in cfg3 cfg2; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-eigensolver > gpurun_out/bench_${c}_r02e.json 2> gpurun_out/bench_${c}_r02e.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_${c}_r02e.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['e2e']['value'], {k: d['roofline'][k] for k in ('achieved','frac','executed_fraction','scalar_fill_fraction','achieved_stored_tiles','trsm_share_of_step')})"
done
