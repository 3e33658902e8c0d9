"""Aggregate ncu per-instruction stall samples onto source lines.

  python tools/sass_lines.py <rep.ncu-rep> <kernel-substring> [top]

Reads `ncu --page source --print-source sass` for the kernel (one launch), maps every
SASS offset to its source line with `nvdisasm -g` on the library's cubin (built with
-lineinfo), and prints the source lines with the most warp-stall samples together with
their executed instruction counts. The library must be the same build as the capture.
"""
from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1810_12163_b200", "lib", "libscreloc_gpu.so")


def sass_rows(rep: str, kernel: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    # the first row names the kernel, the second is the header
    name = rows[0][1] if rows and len(rows[0]) > 1 else "?"
    hdr = rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            break
        out.append(dict(zip(hdr, r)))
    return name, out


def mangled_sub(kernel: str, demangled: str) -> str:
    """Substring of the mangled name selecting exactly the profiled instantiation
    (k_icp_score<(bool)0> -> k_icp_scoreILb0E); SASS_FN overrides."""
    if os.environ.get("SASS_FN"):
        return os.environ["SASS_FN"]
    m = re.search(re.escape(kernel) + r"<\(bool\)(\d)>", demangled)
    if m:
        return f"{kernel}ILb{m.group(1)}E"
    m = re.search(re.escape(kernel) + r"<(\d+)>", demangled)
    if m:
        return f"{kernel}ILi{m.group(1)}E"
    return kernel


def line_map(kernel_mangled_sub: str):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    m = {}
    for cub in os.listdir(tmp):
        dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
        cur = None
        in_fn = False
        for ln in dis.splitlines():
            if ln.startswith(".text.") and ln.rstrip().endswith(":"):
                in_fn = kernel_mangled_sub in ln
                continue
            if not in_fn:
                continue
            g = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
            if g:
                cur = (os.path.basename(g.group(1)), int(g.group(2)))
                continue
            g = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
            if g and cur:
                m[int(g.group(1), 16)] = cur
        if m:
            break
    return m


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    by_exec = len(sys.argv) > 4 and sys.argv[4] == "exec"
    name, rows = sass_rows(rep, kernel)
    base = int(rows[0]["Address"], 16)
    lm = line_map(mangled_sub(kernel, name))
    samples = collections.Counter()
    execd = collections.Counter()
    tot = 0
    for r in rows:
        off = int(r["Address"], 16) - base
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        key = lm.get(off, ("?", 0))
        samples[key] += s
        execd[key] += int(r["Instructions Executed"] or 0)
        tot += s
    src = {}
    for f in ("reloc.cu", "common.cuh", "scene.cu", "internal.cuh"):
        p = os.path.join(ROOT, "paper_1810_12163_b200", "csrc", f)
        if os.path.exists(p):
            src[f] = open(p).read().splitlines()
    print(f"{name[:100]}\n{tot} samples, {len(rows)} SASS instructions, {len(lm)} mapped")
    order = execd.most_common(top) if by_exec else samples.most_common(top)
    tot_exec = max(1, sum(execd.values()))
    print(f"{sum(execd.values())} warp instructions executed")
    for key, _ in order:
        s = samples[key]
        f, l = key
        text = src.get(f, [])[l - 1].strip() if f in src and 0 < l <= len(src[f]) else ""
        print(f"{100 * s / tot:5.1f}%  {execd[key]:>12d} ({100 * execd[key] / tot_exec:4.1f}%)  {f}:{l:<5d} {text[:80]}")


def dump_line(rep: str, kernel: str, fname: str, line: int):
    """SASS of one source line with executed counts (debug helper)."""
    name, rows = sass_rows(rep, kernel)
    base = int(rows[0]["Address"], 16)
    lm = line_map(mangled_sub(kernel, name))
    for r in rows:
        off = int(r["Address"], 16) - base
        if lm.get(off) == (fname, line):
            print(f"{off:6x} {int(r['Instructions Executed'] or 0):>11d} {r['Warp Stall Sampling (All Samples)']:>7s}  "
                  f"{r['Source'].strip()}")


if __name__ == "__main__":
    main()
