"""Static instruction mix of the innermost SASS loop that contains HMMA (or a
given opcode) in one kernel of the built library.

    python tools/sass_loop.py <mangled-kernel-substring> [--op HMMA] [--skip-forward]

--skip-forward drops instructions jumped over by forward predicated branches
whose target lies inside the loop (cold paths such as the normalise divide).
"""

import argparse
import collections
import re
import subprocess
import sys
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2306_16699_b200" / "_lib" / "librinr_b200.so"


def kernel_sass(sub):
    out = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s+Function : ", out)
    hits = [b for b in blocks[1:] if sub in b.split("\n", 1)[0]]
    if len(hits) != 1:
        sys.exit(f"{len(hits)} kernels match {sub!r}")
    ins = []
    for l in hits[0].splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    return hits[0].split("\n", 1)[0], ins


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kernel")
    ap.add_argument("--op", default="HMMA")
    ap.add_argument("--skip-forward", action="store_true")
    a = ap.parse_args()
    name, ins = kernel_sass(a.kernel)
    first = next(addr for addr, t in ins if a.op in t)
    # innermost backward branch spanning `first`
    best = None
    for addr, t in ins:
        m = re.search(r"BRA (?:`\(.*?\) )?0x([0-9a-f]+)", t)
        if m and "CALL" not in t:
            tgt = int(m.group(1), 16)
            if tgt <= first <= addr and (best is None or addr - tgt < best[1] - best[0]):
                best = (tgt, addr)
    lo, hi = best
    body = [(addr, t) for addr, t in ins if lo <= addr <= hi]
    skip = set()
    if a.skip_forward:
        for addr, t in body:
            m = re.match(r"@!?U?P\d BRA 0x([0-9a-f]+)", t)
            if m and lo < int(m.group(1), 16) <= hi and int(m.group(1), 16) > addr:
                skip.update(x for x, _ in body if addr < x < int(m.group(1), 16))
    c = collections.Counter()
    for addr, t in body:
        if addr in skip:
            continue
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        c[op.split(".")[0]] += 1
    print(name[:120])
    print(f"loop 0x{lo:x}-0x{hi:x}: {sum(c.values())} instructions" + (" (forward-skipped removed)" if a.skip_forward else ""))
    print("  " + "  ".join(f"{k} {v}" for k, v in c.most_common()))


if __name__ == "__main__":
    main()
