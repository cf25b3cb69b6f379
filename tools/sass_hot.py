"""Top SASS instructions by warp-stall samples from an ncu report (source page).

python tools/sass_hot.py report.ncu-rep [--top 40] [--range A B]
Prints index, samples, executions, the dominant stall reasons and the SASS.
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--range", type=int, nargs=2, default=None)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(rows[0][1][:150])
    h, data = rows[1], rows[2:]
    i_s, i_src, i_ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
    st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(int(r[i_s]) for r in data)
    print("total samples", tot, "instructions executed", sum(int(r[i_ex]) for r in data))
    if a.range:
        idx = range(a.range[0], a.range[1])
    else:
        idx = sorted(sorted(range(len(data)), key=lambda k: -int(data[k][i_s]))[: a.top])
    for k in idx:
        r = data[k]
        reasons = sorted(((int(r[i]), h[i][6:]) for i in st if r[i] not in ("", "0")), reverse=True)[:2]
        rs = " ".join(f"{n}:{v}" for v, n in reasons)
        print(f"{k:5d} {int(r[i_s]):8d} {100 * int(r[i_s]) / tot:5.1f}% {int(r[i_ex]):11d}  {r[i_src].strip()[:70]:70s} {rs}")


if __name__ == "__main__":
    main()
