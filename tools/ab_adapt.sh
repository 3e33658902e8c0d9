#!/usr/bin/env bash
# A/B of build variants on the per-frame adaptation workload
mkdir -p gpurun_out
for defs in "$@"; do
  SCR_NVCC_DEFS="$defs" python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --workload adapt --no-cpu --steps 100 --warmup 5 > gpurun_out/aba.json 2> gpurun_out/aba.err
  python -c "
import json; d=json.loads(open('gpurun_out/aba.json').read().strip().splitlines()[-1]); print('[$defs]', d['value'], d['ms_per_step'], {k: v for k, v in list(d['kernel_ms_per_frame'].items())[:3]})"
done
python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
