#!/usr/bin/env bash
# Run on a B200 (gpurun): plain bench, then the ncu launch list of the same command, then one
# `--set full` capture per top kernel. Outputs land in gpurun_out/ (scratch); summaries are
# extracted into profiles/ by profiles/summarise.py.
set -uo pipefail
CMD="python bench.py --steps 3 --warmup 3 --batch 128 --test-frames 256 --no-cpu"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
    > gpurun_out/ncu_launch.log 2>&1
for k in k_hypgen k_energy k_icp_score k_energy_small k_leaves; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}\$|::${k}\(" -s 2 -c 1 \
      -o gpurun_out/full_${k} $CMD > gpurun_out/ncu_full_${k}.log 2>&1
done
ls -la gpurun_out/
