"""Store build throughput (rinr_store_create: host C++ header/index parse, CRC32
per record, record parse, one HBM upload) next to the reference reader's
ArchiveReader + read_raw + materialize per record (oracle restatement, one
core).  Prints one JSON line.

    python tools/bench_loader.py [--records 262144]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from oracle import rinr_oracle as O  # noqa: E402
from paper_2306_16699_b200 import Store  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--records", type=int, default=262144)
    a = ap.parse_args()
    data = bench.store_bytes("c2", a.records, seed=0)
    Store(data).close()  # warm-up (CUDA context, allocator)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = Store(data)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st.close()
    k = 20000
    t0 = time.perf_counter()
    blobs = O.record_blobs(data)
    for i, b in enumerate(blobs[:k]):
        O.materialize(O.parse_record(O.check_crc(b, f"record {i}"), f"record {i}"))
    cdt = (time.perf_counter() - t0) * len(blobs) / k
    print(json.dumps({"metric": "store build records/sec (parse + CRC + HBM upload)", "value": a.records / dt,
                      "unit": "records/s", "seconds": dt, "bytes": len(data),
                      "cpu_baseline": {"value": a.records / cdt, "unit": "records/s", "cores": 1, "kind": "port",
                                       "sample": f"{k} records read + CRC + materialize by the oracle restatement "
                                                 "of archive.py:278-400, extrapolated"}}))


if __name__ == "__main__":
    main()
