#!/usr/bin/env bash
# A/B of prebuilt library variants: tools/ab_libs.sh ablibs/a.so ablibs/b.so ... (each: short bench)
mkdir -p gpurun_out
LIB=paper_1810_12163_b200/lib/libscreloc_gpu.so
cp $LIB /tmp/ab_keep.so
for so in "$@"; do
  cp "$so" $LIB
  timeout 300 python bench.py --no-cpu --steps 5 ${BENCH_ARGS:-} > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('[$so]', d['value'], d['e2e']['value'], d['ms_per_step'], d['instrumented_pass'], {k: v for k, v in sorted(d['kernel_share'].items(), key=lambda x: -x[1])[:5]})"
done
cp /tmp/ab_keep.so $LIB
