"""Per-region stall breakdown of an ncu source page: samples summed over
address ranges split at the main loop (development aid).
    python tools/ncu_hot.py report.ncu-rep [top]"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows[2:]:
    try:
        addr = int(r[ix["Address"]], 16)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(r[ix["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    recs.append((addr, r[ix["Source"]].strip(), s, n, {k: int(r[ix[k]] or 0) for k in reasons}))
tot = sum(x[2] for x in recs)
print("total samples", tot)
by_op = collections.defaultdict(lambda: collections.Counter())
for a, src, s, n, rs in recs:
    t = src.split()
    op = (t[1] if t and t[0].startswith("@") else t[0]).split(".")[0] if t else "?"
    by_op[op]["samples"] += s
    for k, v in rs.items():
        by_op[op][k] += v
print("by opcode (share of samples, top reasons):")
for op, c in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:16]:
    rs = sorted(((k, v) for k, v in c.items() if k != "samples"), key=lambda kv: -kv[1])[:4]
    print(f"  {op:8s} {100 * c['samples'] / tot:5.1f}%  " + " ".join(f"{k[6:]}={100 * v / tot:.1f}" for k, v in rs))
print("top instructions:")
for a, src, s, n, rs in sorted(recs, key=lambda x: -x[2])[:top]:
    rr = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
    print(f"  {a:05x} {100 * s / tot:5.2f}% n={n:8d} {src[:60]:60s} " + " ".join(f"{k[6:]}={v}" for k, v in rr))
