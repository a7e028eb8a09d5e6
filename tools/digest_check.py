import sys, hashlib, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from conftest import load_golden
from paper_2306_16699_b200 import Store, bench
g = load_golden("digests")
for case in ["c1_r0", "c1_r1", "c2", "zoo", "fitted_A"]:
    data = load_golden("fitted")["A/archive"].tobytes() if case == "fitted_A" else load_golden(case)["archive"].tobytes()
    rep = bench(data, batch=4)
    print(case, rep.digest == str(g[f"{case}/digest"]))
