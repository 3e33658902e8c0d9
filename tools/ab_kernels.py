"""Per-kernel ms per bench step from bench.py JSON lines (A/B runs of tools/gpu_ab.sh).

  python tools/ab_kernels.py gpurun_out/ab_0.json gpurun_out/ab_1.json ...
"""
import json
import sys

for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    ks, ins = d["kernel_share"], d["instrumented_pass_ms_per_step"]
    top = sorted(ks.items(), key=lambda x: -x[1])[:6]
    print(f, "value", d["value"], "e2e", d["e2e"]["value"], "stage_mix", d["accuracy"]["stage_mix"])
    print("   ", {k: round(v * ins, 3) for k, v in top}, "ms/step (instrumented pass)")
