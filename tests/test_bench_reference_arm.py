"""bench.py --impl reference (CPU): the reference arm runs the oracle restatement on the
host cores and must never import or load the B200 package (reference-arm
hygiene)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

GUARD = """
import sys, json
class Block:
    def find_spec(self, name, path=None, target=None):
        if name.split('.')[0] == 'paper_1810_12163_b200':
            raise ImportError('reference arm imported the B200 package')
        return None
sys.meta_path.insert(0, Block())
sys.argv = ['bench.py'] + sys.argv[1:]
sys.path.insert(0, %r)
import bench
bench.main()
maps = open('/proc/self/maps').read()
assert 'libscreloc_gpu' not in maps, 'B200 library mapped by the reference arm'
"""


def test_reference_arm_never_loads_product():
    cmd = [sys.executable, "-c", GUARD % ROOT, "--impl", "reference", "--workload", "fast", "--adapt-frames", "12",
           "--test-frames", "4", "--ref-batch", "2", "--steps", "1", "--warmup", "1", "--cpu-seconds", "0.5"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["cpu_baseline"]["one_thread"]["cores"] == 1 and d["cpu_baseline"]["one_thread"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload_key"] == "fast"
