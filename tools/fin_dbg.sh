SCR_NVCC_DEFS="-DSCR_FIN_DEBUG" python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --lanes 1 > gpurun_out/fin_dbg.json 2> gpurun_out/fin_dbg.err
grep -h "hypfin" gpurun_out/fin_dbg.json gpurun_out/fin_dbg.err | python -c "
import sys,re,collections
tent=fail=0; conts=[]; sus=[]
for l in sys.stdin:
    m=re.search(r'tent=(\d+) fail=(\d+)',l)
    if m: tent+=int(m.group(1)); fail+=int(m.group(2))
    m=re.search(r'hypfin-sus a=\d+ n=(\d+)',l)
    if m: sus.append(int(m.group(1)))
    m=re.search(r'att=(\d+) it=(\d+) ok=(\d+)',l)
    if m: conts.append(tuple(map(int,m.groups())))
print('suspects',sum(sus),'frames with suspects',len(sus),'max',max(sus or [0]),'continuations',len(conts))
print(conts[:40])
"
python paper_1810_12163_b200/build.py --force > /dev/null 2>&1
