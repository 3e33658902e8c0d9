set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b8.json 2> gpurun_out/b8.err; tail -c 1500 gpurun_out/b8.json
SCR_NVCC_DEFS="-DSCR_HYPGEN_MINB=4" python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b4.json 2> gpurun_out/b4.err; tail -c 1500 gpurun_out/b4.json
