for tc in 0 2 0 2; do
  BMOE_COACT_TC=$tc timeout 900 python bench.py --workload profile 2>/dev/null | sed "s/^{/{\"coact_tc\": $tc, /"
done > gpurun_out/r2s_profile_mxf4_ab.jsonl
python - <<'P'
import json
for l in open("gpurun_out/r2s_profile_mxf4_ab.jsonl"):
    r = json.loads(l); print(r["coact_tc"], r["value"], r["ms_per_step"], r["roofline"]["avg_launch_ms"], r["roofline"]["frac"], r.get("tables_sha16") or r.get("digest"))
P
