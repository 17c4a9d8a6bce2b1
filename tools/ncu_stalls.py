"""Stall-reason shares and the top stalled SASS lines of an ncu report (source page).
usage: ncu_stalls.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    iS = h.index("Warp Stall Sampling (All Samples)")
    names = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = {n: sum(int(r[h.index(n)] or 0) for r in data) for n in names}
    T = sum(tot.values()) or 1
    print("stall shares:", {k: round(v / T, 3) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
    for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:top]:
        why = {n[6:]: r[h.index(n)] for n in names if r[h.index(n)] not in ("0", "")}
        print(r[0][-5:], r[iS].rjust(6), r[1].strip()[:60].ljust(60), why)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
