"""Per-CTA phase timeline of decode_persist (library built with
RINR_EXTRA_NVCC_FLAGS=-DRINR_DEV_KNOBS; tools/dev_timeline.sh)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_16699_b200 import Store, _native, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
B = 1024 if cfg == "c2" else 256
st = Store(synth.gpu_store_bytes(cfg, 65536, seed=3))
ids = torch.randint(0, len(st), (16, B), device="cuda")
p = st.decode_params(32, 32, precision="fp32", overlap_prologue=True)
out = torch.empty((B, 3, 32, 32), device="cuda")
for k in range(12):  # back to back on one stream (PDL chain), last 4 recorded
    st.decode(ids[k], out=out, params=p, check=False)
torch.cuda.synchronize()
t = np.zeros((4, 512, 8), np.uint64)
assert _native.lib().rinr_dev_times(t.ctypes.data_as(C.c_void_p)) == 0
grid = int((t[0, :, 0] != 0).sum())  # CTAs that stamped (2 x 148 for 8-warp CTAs)
print(f"grid {grid}")
t = t[:, :grid, :].astype(np.int64)
base = t[:, :, 0].min()
names = ["entry", "ids+cp.async issued", "records in smem", "dequant done", "pdl_wait done", "phase2 done", "exit"]
for s in range(4):
    tt = t[s] - base
    print(f"launch slot {s}: entry {tt[:, 0].min() / 1e3:.2f}..{tt[:, 0].max() / 1e3:.2f} us, "
          f"exit {tt[:, 6].min() / 1e3:.2f}..{tt[:, 6].max() / 1e3:.2f} us")
    d7 = (t[s][:, 7] - t[s][:, 0]) / 1e3
    print(f"   entry -> first id loaded: median {np.median(d7):.2f} us  max {d7.max():.2f}")
    for k in range(1, 7):
        d = (t[s][:, k] - t[s][:, k - 1]) / 1e3
        print(f"   {names[k - 1]:>22s} -> {names[k]:<22s} median {np.median(d):6.2f} us  max {d.max():6.2f}")
tk = np.zeros((512, 16, 2), np.uint64)
assert _native.lib().rinr_dev_task_times(tk.ctypes.data_as(C.c_void_p)) == 0
d = tk[:grid, :, 1].astype(np.int64)
for h in (0, 1):
    sel = d[(d >= h * 1000000) & (d < (h + 1) * 1000000)] - h * 1000000
    if sel.size:
        print(f"task h={h}: {sel.size} samples, median {np.median(sel):.0f} cycles, max {sel.max()}")

# per-CTA phase 2 (pdl_wait done -> exit) against images spanned and SM
sm = tk[:grid, 15, 0].astype(np.int64)
gpi = 32
total = B * gpi
qg, rg = divmod(total, grid)
b = np.arange(grid)
G0 = b * qg + np.minimum(b, rg)
G1 = G0 + qg + (b < rg)
nimg = (G1 - 1) // gpi - G0 // gpi + 1
for s in range(4):
    d = (t[s][:, 6] - t[s][:, 4]) / 1e3
    e = (t[s][:, 4] - t[s][:, 0]) / 1e3
    print(f"slot {s}: phase2+exit p10 {np.percentile(d, 10):.2f} p50 {np.median(d):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.2f} us;"
          f" entry->phase2 p50 {np.median(e):.2f} max {e.max():.2f}")
    for k in sorted(set(nimg.tolist())):
        print(f"   nimg {k}: {int((nimg == k).sum())} CTAs, phase2 mean {d[nimg == k].mean():.2f} max {d[nimg == k].max():.2f}")
    slow = np.argsort(d)[-8:]
    print("   slowest CTAs (cta, sm, nimg, us, entry):", [(int(c), int(sm[c]), int(nimg[c]), round(float(d[c]), 2), round(float((t[s][c, 0] - t[s][:, 0].min()) / 1e3), 2)) for c in slow])
    # SM pairs: both CTAs of an SM
    per_sm = {}
    for c in range(grid):
        per_sm.setdefault(int(sm[c]), []).append(c)
    multi = [v for v in per_sm.values() if len(v) == 2]
    print(f"   SMs used {len(per_sm)}; with 2 CTAs {len(multi)}")

# absolute exit times (from the launch's first CTA entry) by wave and images spanned
for s in range(4):
    base_s = t[s][:, 0].min()
    ex = (t[s][:, 6] - base_s) / 1e3
    en = (t[s][:, 0] - base_s) / 1e3
    p4 = (t[s][:, 4] - base_s) / 1e3
    wave = (np.arange(grid) >= grid // 2).astype(int)
    print(f"slot {s}: exit p50 {np.median(ex):.2f} p90 {np.percentile(ex, 90):.2f} max {ex.max():.2f} us")
    for w in (0, 1):
        for k in sorted(set(nimg.tolist())):
            m = (wave == w) & (nimg == k)
            if m.any():
                print(f"   wave {w} nimg {k}: {int(m.sum())} CTAs, entry {en[m].mean():.2f}, phase2 start {p4[m].mean():.2f}, "
                      f"exit mean {ex[m].mean():.2f} max {ex[m].max():.2f}")
