#!/usr/bin/env bash
# On a B200 (gpurun), one ncu tool per call:
#   bash profiles/run_profiles.sh plain     # bench without ncu (must exit 0 first)
#   bash profiles/run_profiles.sh launches  # ncu launch list of the timed region
#   bash profiles/run_profiles.sh full      # ncu --set full of the top kernels, first timed step
# Outputs land in gpurun_out/; profiles/summarise.py turns them into tracked summaries.
set -uo pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --profile-window"
case "${1:-plain}" in
  plain) $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err; tail -c 600 gpurun_out/prof_plain.json ;;
  launches)
    $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
        --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
    tail -3 gpurun_out/ncu_launch.log ;;
  full)
    $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || { echo "plain run failed"; exit 1; }
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:"${NCU_REGEX:-k_hypgen|k_icp_score|k_energy_small|k_leaves}" -c ${NCU_COUNT:-10} \
        -o gpurun_out/full_top $CMD > gpurun_out/ncu_full.log 2>&1
    tail -3 gpurun_out/ncu_full.log ;;
esac
