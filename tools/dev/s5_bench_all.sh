mkdir -p gpurun_out/s5
python bench.py --steps 5 --warmup 3 > gpurun_out/s5/bench3_cfg3.json 2> gpurun_out/s5/bench3_cfg3.err
python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/s5/bench3_cfg2.json 2> gpurun_out/s5/bench3_cfg2.err
python bench.py --config cfg4s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5/bench3_cfg4s.json 2> gpurun_out/s5/bench3_cfg4s.err
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5/bench3_cfg5.json 2> gpurun_out/s5/bench3_cfg5.err
for c in cfg3 cfg2 cfg4s cfg5; do python - <<EOF
import json
try:
    d=json.load(open("gpurun_out/s5/bench3_$c.json"))
    t=d.get("time_to_all_eigenpairs",{})
    print("$c", round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "frac", round(d["roofline"]["frac"],3), "t_factor_ms", round(d["t_factor_ms"],1), "ttae", t.get("value"), t.get("found"), t.get("converged"), t.get("residual"), d["clocks"]["sm_mhz"])
except Exception as e:
    print("$c failed", e)
EOF
done
