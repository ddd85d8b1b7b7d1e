python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "sweep profile|apply_filter" | cut -c1-200
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/t6_gputest.txt 2>&1; tail -3 gpurun_out/t6_gputest.txt
python bench.py --config cfg5 --no-cpu-baseline --no-eigensolver --steps 3 --warmup 3 > gpurun_out/t6_cfg5.json 2> gpurun_out/t6_cfg5.err
python -c "
import json; d=json.loads(open('gpurun_out/t6_cfg5.json').read().strip().splitlines()[-1]); print('cfg5', d['value'], d['roofline']['trsm_launches'], d['steps'], d['gmres_iterations'])"
