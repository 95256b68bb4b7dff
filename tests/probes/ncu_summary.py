"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
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
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)  # -> microseconds
        out.append((d["Kernel Name"].split("(")[0].split("<")[0], v))
    return out


def summary(path):
    seq = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in seq:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':28s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:28s} {n:8d} {t / 1e3:10.3f} {t / n:10.1f} {100 * t / tot:5.1f}%")
    lines.append(f"{'TOTAL':28s} {len(seq):8d} {tot / 1e3:10.3f}")
    return "\n".join(lines), seq


if __name__ == "__main__":
    s, seq = summary(sys.argv[1])
    print(s)
    if len(sys.argv) > 2:
        print([(n[:10], round(v)) for n, v in seq[: int(sys.argv[2])]])
