"""Print selected (section, metric) pairs of an ncu report's details page."""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput",
        "Issued Ipc Active", "Eligible Warps Per Scheduler", "No Eligible", "Registers Per Thread",
        "Grid Size", "Waves Per SM", "Achieved Occupancy", "L2 Hit Rate", "Mem Busy",
        "Max Bandwidth", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction")


def main(path, extra=()):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out[out.index('"ID"'):])))
    hdr = rows[0]
    ki, si, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name",
                                                  "Metric Unit", "Metric Value"))
    seen = set()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if r[mi] in WANT or r[mi] in extra:
            key = (r[ki], r[mi])
            if key in seen:
                continue
            seen.add(key)
            print(f"{r[ki][:40]:40s} {r[mi]:38s} {r[vi]:>12s} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
