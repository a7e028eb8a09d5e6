"""Reference-arm sensitivity: the oracle port of rinr.decode_batch (what
`bench.py --impl reference` times) under a jobs x BLAS-threads sweep on the
host cores, c2 (32x32) and c3 (224x224 + crop/flip/normalise).  Answers
whether 1 BLAS thread per worker process (bench.py's choice) understates the
CPU baseline.

    python tools/cpu_sweep.py            # whole sweep, one JSON line per point
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(cfg: str, jobs: int, threads: int):
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = str(threads)
    sys.path.insert(0, ROOT)
    import numpy as np
    import bench
    W = bench.workload(cfg)
    n_rec = 4096 if cfg != "c3" else 64
    data = bench.host_store_bytes(cfg, n_rec, seed=12345)
    pool = bench.CpuPool(data, W["h"], W["w"], jobs)
    rng = np.random.default_rng(0)
    n = 32768 if cfg == "c2" else 192
    try:
        warm = rng.integers(0, n_rec, max(jobs, 16))
        pool.run(warm, bench.crop_params_np(len(warm), 0) if cfg == "c3" else None)
        ids = rng.integers(0, n_rec, n)
        t = pool.run(ids, bench.crop_params_np(n, 1) if cfg == "c3" else None)
    finally:
        pool.close()
    print(json.dumps({"config": cfg, "jobs": jobs, "blas_threads": threads, "images": n,
                      "seconds": round(t, 3), "images_per_s": round(n / t, 1)}), flush=True)


def main():
    cores = len(os.sched_getaffinity(0))
    print(json.dumps({"host_cores": cores}), flush=True)
    points = sorted({(cores, 1), (max(1, cores // 2), 2), (max(1, cores // 4), 4), (1, cores)})
    for cfg in ("c2", "c3"):
        for jobs, thr in points:
            subprocess.run([sys.executable, __file__, "--one", cfg, str(jobs), str(thr)], check=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        main()
