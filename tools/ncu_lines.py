"""Executed instructions and stall samples per CUDA source line of one kernel
in an .ncu-rep (needs -lineinfo + --import-source on).

    python tools/ncu_lines.py rep.ncu-rep [--per N] [--top 40]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--per", type=float, default=1.0)
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, res = None, []
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0].isdigit() and len(r) > 8 and r[2] == "-":
            try:
                res.append((int(r[7] or 0), int(r[4] or 0), f"{cur}:{r[0]}", r[1][:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in res)
    print(f"total {tot} per unit {tot / a.per:.1f}")
    for ex, smp, loc, src in sorted(res, reverse=True)[:a.top]:
        print(f"{ex / a.per:7.2f} {smp:5d} {loc:24s} {src}")


if __name__ == "__main__":
    main()
