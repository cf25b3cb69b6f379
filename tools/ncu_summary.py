"""Summarise ncu outputs into a text file for profiles/.

python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <out.txt> [steps]
- launch list: per-kernel total device time and share (cold-cache, serialised)
- full capture: key metrics per captured kernel (duration, DRAM bytes, hit
  rates, issue, occupancy, stall breakdown)
"""
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = {}
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
        name = r[ki].split("(")[0]
        t = tot.setdefault(name, [0.0, 0])
        t[0] += v
        t[1] += 1
    return tot


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    res = {}
    for x in r[1:]:
        res.setdefault(x[ki].split("(")[0], []).append((x[mi], x[vi], x[ui]))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    traffic = {}
    if rr:
        hh = rr[0]
        want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
                "smsp__inst_executed.sum", "l1tex__t_bytes.sum"]
        idx = {w: hh.index(w) for w in want if w in hh}
        kidx = hh.index("Kernel Name")
        units = rr[1] if len(rr) > 1 else []
        for x in rr[2:]:
            traffic[x[kidx].split("(")[0]] = {w: (x[i], units[i] if i < len(units) else "") for w, i in idx.items()}
    return res, traffic


def main():
    lp, rep, outp = sys.argv[1], sys.argv[2], sys.argv[3]
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    lines = []
    tot = launches(lp)
    s = sum(v[0] for v in tot.values())
    lines.append(f"# launch list ({lp}): {s:.2f} ms device time over all launches (cold-cache, serialised)")
    for k, (v, n) in sorted(tot.items(), key=lambda x: -x[1][0]):
        if v / s > 0.0005:
            lines.append(f"{v:10.3f} ms {n:5d} launches {100 * v / s:6.2f}%  {k}")
    res, traffic = details(rep)
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
            "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
            "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Grid Size", "Block Size",
            "Dynamic Shared Memory Per Block"}
    for k, ms in res.items():
        lines.append(f"\n# ncu --set full: {k}")
        for m, v, u in ms:
            if m in keep:
                lines.append(f"  {m} = {v} {u}")
        for m, (v, u) in traffic.get(k, {}).items():
            lines.append(f"  {m} = {v} {u}")
    open(outp, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # per-kernel DRAM traffic per launch, for bench.py's roofline.traffic
    import json
    import os
    import math
    tpath = os.path.join(os.path.dirname(outp) or ".", "roofline_traffic.json")
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tj = {k: v for k, v in tj.items() if math.isfinite(v.get("dram_bytes", float("nan")))}
    for k, t in traffic.items():
        try:
            rd, ru = t["dram__bytes_read.sum"]
            wr, wu = t["dram__bytes_write.sum"]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            b = float(rd) * scale.get(ru, 1) + float(wr) * scale.get(wu, 1)
            if math.isfinite(b):
                tj[k.replace("void ", "").split("<")[0]] = {"dram_bytes": b, "source": os.path.basename(outp)}
        except (KeyError, ValueError):
            pass
    if tj:
        json.dump(tj, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
