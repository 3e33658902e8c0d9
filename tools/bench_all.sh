#!/usr/bin/env bash
# Every bench.py workload on one B200, one JSON line each -> gpurun_out/wl_<name>.json
#   /usr/local/graft/bin/gpurun --timeout 3600 -- bash tools/bench_all.sh [workloads...]
mkdir -p gpurun_out
WL=${@:-cascade default-raw default-icp default-ranked fast intermediate slow scenes stress adapt}
for w in $WL; do
  extra=""
  [ "$w" = "adapt" ] && extra="--steps 200 --warmup 5"
  timeout 900 python bench.py --workload $w ${extra:---steps 5} > gpurun_out/wl_$w.json 2> gpurun_out/wl_$w.err \
    || { echo "$w failed"; tail -5 gpurun_out/wl_$w.err; continue; }
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
d = json.loads(open(f"gpurun_out/wl_{w}.json").read().strip().splitlines()[-1])
acc = d.get("accuracy", {})
print(w, "value", d["value"], d["unit"], "e2e", d.get("e2e", {}).get("value"), "succ", acc.get("success_5cm_5deg"),
      "mix", acc.get("stage_mix"), "cpu", (d.get("cpu_baseline") or {}).get("value"),
      "parity", {k: v for k, v in (d.get("parity") or {}).items() if k in ("bit_exact_results", "frames_compared", "adapted_table_bit_exact")},
      "dom", (d.get("roofline") or {}).get("kernel"), (d.get("roofline") or {}).get("frac"))
PY
done
