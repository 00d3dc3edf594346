"""Dynamic SASS opcode histogram + stall totals of one kernel in an .ncu-rep
(per `unit` = launch-wide instruction count / unit count, e.g. warp-pages).

    python tools/ncu_ophist.py gpurun_out/x.ncu-rep [--per N] [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    R = rows[2:]
    iE = h.index("Instructions Executed")
    iS = h.index("Warp Stall Sampling (All Samples)")
    stalls = [c for c in h if c.startswith("stall_") and "Not" not in c]
    ops = collections.Counter()
    st = collections.Counter()
    for r in R:
        op = r[1].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1]
        ops[op.split()[0]] += int(r[iE] or 0)
        for c in stalls:
            st[c] += int(r[h.index(c)] or 0)
    tot = sum(ops.values())
    print(f"instructions {tot}  per unit {tot / a.per:.1f}  samples {sum(int(r[iS] or 0) for r in R)}")
    for k, v in ops.most_common(a.top):
        print(f"  {k:34s} {v / a.per:9.2f} {v / tot * 100:5.1f}%")
    print("stalls:", ", ".join(f"{k[6:]}={v}" for k, v in st.most_common(10)))


if __name__ == "__main__":
    main()
