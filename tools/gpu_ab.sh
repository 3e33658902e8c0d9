#!/usr/bin/env bash
# A/B timing of build variants on one B200: tools/gpu_ab.sh "<defs A>" "<defs B>" ...
# (first runs the GPU tests on the default build). Outputs: gpurun_out/ab_<i>.json
mkdir -p gpurun_out
python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
i=0
for defs in "$@"; do
  SCR_NVCC_DEFS="$defs" python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$defs" gpurun_out/ab_$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
ks = d["kernel_share"]
print(f"[{sys.argv[1]}] value {d['value']} e2e {d['e2e']['value']} ms/step {d['ms_per_step']} "
      f"instr {d['instrumented_pass_ms_per_step']} clocks {d['clocks'].get('sm_mhz')}x{d['clocks'].get('samples')} "
      f"succ {d['accuracy']['success_5cm_5deg']}")
print("   ", {k: v for k, v in sorted(ks.items(), key=lambda x: -x[1])[:6]})
print("   ", {k: (v['achieved'], v['frac']) for k, v in [(d['roofline']['kernel'], d['roofline'])] + list(d.get('rooflines_other', {}).items())})
PY
  i=$((i+1))
done
python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
