"""Summarise an ncu report: headline metrics + SASS instruction mix (per 16-px block if --blocks given)."""
import csv, collections, subprocess, sys, io

def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        if len(r) == len(hdr):
            d = dict(zip(hdr, r))
            res[(d["Section Name"], d["Metric Name"])] = (d["Metric Value"], d["Metric Unit"])
    return res

def sass_mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]; ie = hdr.index("Instructions Executed"); src = hdr.index("Source"); smp = hdr.index("Warp Stall Sampling (All Samples)")
    cnt = collections.Counter(); samples = collections.Counter()
    for r in rows[2:]:
        try: n = int(r[ie])
        except (ValueError, IndexError): continue
        s = r[src].strip().split()
        if not s: continue
        op = (s[1] if s[0].startswith('@') else s[0]).split('.')[0]
        cnt[op] += n; samples[op] += int(r[smp] or 0)
    return cnt, samples

if __name__ == "__main__":
    rep = sys.argv[1]; blocks = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    d = details(rep)
    keys = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
            "Achieved Occupancy", "Eligible Warps Per Scheduler", "No Eligible", "DRAM Throughput", "Memory Throughput",
            "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
    for (sec, name), (v, u) in d.items():
        if name in keys: print(f"{name:36s} {v} {u}")
    cnt, samples = sass_mix(rep)
    tot = sum(cnt.values())
    print(f"warp instructions {tot}  per block {tot / blocks:.1f}")
    for op, n in cnt.most_common(24):
        print(f"  {op:10s} {n / blocks:8.1f}   stall samples {samples[op]}")
