# the round-end sequence on one box: GPU tests, smoke(), the reference arm, the default bench
mkdir -p gpurun_out/final
(time python -m pytest tests -m gpu -x -q) > gpurun_out/final/gputest.log 2>&1; tail -3 gpurun_out/final/gputest.log | head -1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -2 gpurun_out/final/smoke.log
(time python bench.py --impl reference) > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; tail -3 gpurun_out/final/bench_reference.err
(time python bench.py) > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -3 gpurun_out/final/bench.err
python - <<EOF
import json
d=json.load(open("gpurun_out/final/bench.json"))
t=d["time_to_all_eigenpairs"]
print("bench", round(d["value"],2), "e2e", round(d["e2e"]["value"],2), "frac", round(d["roofline"]["frac"],3), "ttae", round(t["value"],3), t["found"], t["converged"], d["clocks"], "sibling", d.get("sibling_comparison",{}).get("ratio"))
r=json.load(open("gpurun_out/final/bench_reference.json"))
print("reference", r.get("value"), r.get("unavailable","")[:60], r["cpu_baseline"]["value"], r.get("product_library_mapped"))
EOF
