"""Write a committed text summary of an ncu --set full report (profiles/)."""
import csv, io, re, subprocess, sys, json, collections

KEYS = re.compile(r"^(gpu__time_duration.sum|dram__bytes_(read|write)\.sum|sm__cycles_elapsed.avg|smsp__inst_executed.sum|"
                  r"launch__(registers_per_thread|grid_size|block_size|shared_mem_per_block_dynamic)|"
                  r"sm__inst_executed_pipe_(xu|fma|alu|tensor_subpipe_hmma)\.avg\.pct_of_peak_sustained_active|"
                  r"sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_active|"
                  r"smsp__issue_active\.avg\.pct_of_peak_sustained_active|sm__warps_active\.avg\.pct_of_peak_sustained_active|"
                  r"smsp__average_warps_issue_stalled_(wait|not_selected|short_scoreboard|long_scoreboard|math_pipe_throttle|"
                  r"barrier|mio_throttle|branch_resolving|dispatch_stall|no_instruction)_per_issue_active\.ratio)$")

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [(h, u, v) for h, u, v in zip(rows[0], rows[1], rows[2])]

def mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]; ie = hdr.index("Instructions Executed"); src = hdr.index("Source")
    c = collections.Counter()
    for r in rows[2:]:
        try: n = int(r[ie])
        except (ValueError, IndexError): continue
        s = r[src].strip().split()
        if s: c[(s[1] if s[0].startswith('@') else s[0]).split('.')[0]] += n
    return c, rows[0][0] if rows and rows[0] else ""

if __name__ == "__main__":
    rep, title, units, tag = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
    lines = [f"# {title}", f"# source: {rep} (ncu --set full --clock-control none; cold, serialised launch)"]
    vals = {}
    for h, u, v in raw(rep):
        if KEYS.match(h):
            lines.append(f"{h:95s} {v} {u}")
            vals[h] = (v, u)
    c, kname = mix(rep)
    tot = sum(c.values())
    lines.append(f"\n# SASS instruction mix (warp instructions), total {tot}, per 16-pixel block {tot / units:.1f}")
    for op, n in c.most_common(30):
        lines.append(f"  {op:10s} {n:12d}  {n / units:8.2f} / block")
    print("\n".join(lines))
    def to_bytes(v, u):
        v = float(v.replace(",", "")); return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    rd = to_bytes(*vals["dram__bytes_read.sum"]); wr = to_bytes(*vals["dram__bytes_write.sum"])
    summ = {}
    try: summ = json.load(open("profiles/ncu_summary.json"))
    except (OSError, ValueError): pass
    summ[tag] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                 "duration_us_cold": float(vals["gpu__time_duration.sum"][0].replace(",", "")) *
                 {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(vals["gpu__time_duration.sum"][1], 1.0),
                 "xu_pct_active": float(vals["sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"][0]),
                 "issue_pct_active": float(vals["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
                 "tensor_pct_active": float(vals["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"][0]),
                 "report": rep}
    json.dump(summ, open("profiles/ncu_summary.json", "w"), indent=1)
