# pipelined e2e leg (back-to-back steps) beside the per-step one
for r in 1 2; do
timeout 600 python bench.py --no-secondary --no-cpu > gpurun_out/r4d_bench_$r.log 2>&1; echo "exit $?" >> gpurun_out/r4d_bench_$r.log
python - <<PY
import json
l=[x for x in open("gpurun_out/r4d_bench_$r.log") if x.startswith("{")][-1]
j=json.loads(l); e=j["e2e"]
print("value", round(j["value"]), "e2e", round(e["value"]), e["ms_per_step"], "iso", round(e["isolated_step"]["value"]), "check", e.get("check",{}).get("pass"), j["check"]["pass"], "frac", round(j["roofline"]["frac"],4))
PY
done
