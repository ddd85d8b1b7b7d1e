for v in pc1 pc2 pc4; do echo "== $v"; ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python tools/quick_check.py cfg2 cfg3 2>&1 | grep -E "apply_filter|chunk_slots" | sed -n '1p;3p;4p;6p' | cut -c1-150
ZOLO_LIB_PATH=tools/dev/variants/libzolo_$v.so python bench.py --config cfg5 --no-cpu-baseline --no-eigensolver --steps 3 --warmup 3 > gpurun_out/pc_cfg5_$v.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/pc_cfg5_$v.json').read().strip().splitlines()[-1]); print('cfg5', round(d['value'],2), d['roofline']['trsm_launches'] // d['steps'], 'launches/step')"
done
