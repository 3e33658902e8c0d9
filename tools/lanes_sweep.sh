# Lane / batch sweep of the default workload: tools/lanes_sweep.sh ["<bench args>" ...]
mkdir -p gpurun_out
[ $# -eq 0 ] && set -- "" "--lanes 4" "--lanes 6" "--lanes 8" "--lanes 6 --batch 96" "--lanes 4 --batch 160"
for a in "$@"; do
  timeout 300 python bench.py --no-cpu --steps 5 $a > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('[$a]', d['value'], d['e2e']['value'], d['ms_per_step'])"
done
