"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    out = []
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e6 if u in ("nsecond", "ns") else (v / 1e3 if u in ("usecond", "us") else v)
        out.append((d["Kernel Name"].split("(")[0].replace("scr::", ""), v))
    return out


if __name__ == "__main__":
    launches = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    launches = launches[skip:]
    agg = collections.defaultdict(list)
    for n, v in launches:
        agg[n].append(v)
    tot = sum(v for _, v in launches)
    print(f"{'kernel':22s} {'launches':>8s} {'total ms':>9s} {'share':>6s}  per-launch ms (last 8)")
    for n, l in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{n:22s} {len(l):8d} {sum(l):9.2f} {100 * sum(l) / tot:5.1f}%  {[round(x, 3) for x in l[-8:]]}")
