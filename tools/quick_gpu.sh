#!/usr/bin/env bash
# One gpurun iteration: parity tests, a short bench (no CPU leg) and the ncu launch list of the
# same command; prints the headline numbers and the per-kernel launch summary.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- bash tools/quick_gpu.sh [pytest targets]
mkdir -p gpurun_out
T=${1:-tests/test_gpu_parity.py}
timeout 900 python -m pytest $T -q -x > gpurun_out/q_tests.log 2>&1; tail -2 gpurun_out/q_tests.log
timeout 600 python bench.py --no-cpu --steps 5 ${BENCH_ARGS:-} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err || tail -5 gpurun_out/q_bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/q_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "ms/step", d["ms_per_step"], "succ", d["accuracy"]["success_5cm_5deg"],
      "mix", d["accuracy"]["stage_mix"], "clk", d["clocks"]["sm_mhz"])
print({k: v for k, v in sorted(d["kernel_share"].items(), key=lambda x: -x[1])[:8]})
PY
if [ -z "${NO_LAUNCHES:-}" ]; then
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --profile-window ${BENCH_ARGS:-} \
      > gpurun_out/ncu_launch.log 2>&1
  python profiles/launch_summary.py gpurun_out/launches.csv | head -24
fi
