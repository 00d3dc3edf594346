"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import io
import sys


def summarize(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["Metric Unit"]]
        name = r["Kernel Name"].replace("void ", "").split("(")[0] + "(" + r["Kernel Name"].split("(")[1].split(")")[0] + ")" if "(" in r["Kernel Name"] else r["Kernel Name"]
        a = agg[name]
        a[0] += 1
        a[1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'total_ms':>10} {'share':>6} {'launches':>8} {'avg_us':>9}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t / 1e3:10.3f} {100 * t / tot:5.1f}% {n:8d} {t / n:9.1f}  {k}")
    lines.append(f"{tot / 1e3:10.3f} 100.0% {sum(v[0] for v in agg.values()):8d}  (all kernels, serialised)")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
