"""Stall samples per CUDA source line (top reasons) of one kernel in an .ncu-rep.

    python tools/ncu_stall_lines.py rep.ncu-rep [--top 25]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, res = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif r and r[0].isdigit() and len(r) > 8 and r[2] == "-":
            d = dict(zip(hdr, r))
            smp = int(d.get("Warp Stall Sampling (All Samples)") or 0)
            st = {k[6:]: int(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not" not in k}
            res.append((smp, f"{cur}:{r[0]}", r[1][:64], sorted(st.items(), key=lambda x: -x[1])[:3]))
    tot = sum(x[0] for x in res)
    print("samples", tot)
    for smp, loc, src, st in sorted(res, reverse=True)[:a.top]:
        print(f"{smp:5d} {smp / tot * 100:5.1f}% {loc:22s} {src:64s} {st}")


if __name__ == "__main__":
    main()
