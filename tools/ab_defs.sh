#!/usr/bin/env bash
# A/B of build variants: tools/ab_defs.sh "<defs A>" "<defs B>" ... (each: rebuild + short bench)
mkdir -p gpurun_out
for defs in "$@"; do
  SCR_NVCC_DEFS="$defs" python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu --steps 5 ${BENCH_ARGS:-} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('[$defs]', d['value'], d['e2e']['value'], d['ms_per_step'], d['instrumented_pass'], 'assoc', d['work'].get('lm_assoc_evals'), {k: v for k, v in sorted(d['kernel_share'].items(), key=lambda x: -x[1])[:5]})"
done
python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
