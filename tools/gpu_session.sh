mkdir -p gpurun_out
timeout 300 python tools/prof_overhead.py
timeout 900 python bench.py > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench_full.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2_bench_full.json').read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "parity", d["parity"]["ok"], d["stage_ms_last_step"], d["roofline"]["frac"], d["lloyd_distances_per_s"])
for k,v in d.get("by_config",{}).items():
    print(k, round(v["value"],1), "e2e", round(v["e2e"]["value"],1), "parity", v["parity"]["ok"], v["stage_ms_last_step"])
PY
