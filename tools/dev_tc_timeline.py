"""Per-slot timeline of decode_tc in CTA 0 (library built with
RINR_EXTRA_NVCC_FLAGS=-DRINR_DEV_KNOBS): for each tile slot and round, the
exposed MMA wait and the epilogue time of every layer, and how many slots are
in their epilogue (sine) phase at once.

    python tools/dev_tc_timeline.py [fp32|bf16]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16699_b200 import Store, _native, synth  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
B = 256
st = Store(synth.gpu_store_bytes("c3", 4096, seed=3))
ids = torch.randint(0, len(st), (8, B), device="cuda")
p = st.decode_params(224, 224, precision=prec, overlap_prologue=True)
out = torch.empty((B, 3, 224, 224), device="cuda")
for k in range(6):
    st.decode(ids[k], out=out, params=p, check=False)
torch.cuda.synchronize()
t = np.zeros((8, 8, 12, 4), np.int64)
assert _native.lib().rinr_dev_tc_times(t.ctypes.data_as(C.c_void_p)) == 0
T = int((t[:, 0, 0, 0] != 0).sum())
NL = 10
print(f"{prec}: {T} slots")
base = t[:T][t[:T] > 0].min()
epi, wait, fly, l0, iss = [], [], [], [], []
events = []  # (time, +1/-1) epilogue phases
for s in range(T):
    for r in range(8):
        x = t[s, r]
        if x[0, 0] == 0 or x[NL, 0] == 0:
            continue
        l0.append(x[0, 2] - x[0, 0])
        events += [(x[0, 0], 1), (x[0, 2], -1)]
        for l in range(1, NL - 1):
            wait.append(x[l, 1] - x[l, 0])
            epi.append(x[l, 2] - x[l, 1])
            fly.append(x[l, 1] - x[l - 1, 2])
            iss.append(x[l - 1, 3] - x[l - 1, 2])
            events += [(x[l, 1], 1), (x[l, 2], -1)]
        wait.append(x[NL - 1, 1] - x[NL - 1, 0])
        fly.append(x[NL - 1, 1] - x[NL - 2, 2])
        print(f"slot {s} round {r}: tile {(x[NL, 0] - x[0, 0])} cyc, start {x[0, 0] - base}")
print(f"layer 0 (FFMA + sine + store A): median {np.median(l0):.0f} cycles")
print(f"hidden epilogue (ld, sine, split, st, barrier): median {np.median(epi):.0f} p90 {np.percentile(epi, 90):.0f}")
print(f"exposed MMA wait: median {np.median(wait):.0f} p90 {np.percentile(wait, 90):.0f}")
print(f"issue_layer duration: median {np.median(iss):.0f} p90 {np.percentile(iss, 90):.0f}")
print(f"MMA issue -> completion seen: median {np.median(fly):.0f} p90 {np.percentile(fly, 90):.0f}")
ev = sorted(events)
t0, t1 = ev[0][0], ev[-1][0]
cur, last, hist = 0, t0, np.zeros(T + 1)
for tm, d in ev:
    hist[cur] += tm - last
    cur += d
    last = tm
hist /= hist.sum()
print("share of time with k slots in epilogue:", {k: round(float(v), 3) for k, v in enumerate(hist)})
