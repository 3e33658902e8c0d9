mkdir -p gpurun_out
for ms in 50 0 50 0 250 1000; do
  SCR_CLOCK_MS=$ms timeout 300 python bench.py --no-cpu --steps 5 > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('[clock ms $ms]', d['value'], d['e2e']['value'], d['ms_per_step'], d['clocks'])"
done
