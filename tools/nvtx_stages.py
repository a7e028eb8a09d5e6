"""Run harness.bench (the reference's rinr.bench mirror) on a synthetic c2
store with NVTX stage ranges on, and print the report.  Under ncu the
ranges filter a capture to one stage:

    RINR_NVTX=1 ncu --nvtx --nvtx-include "rinr.forward/" \
        --metrics gpu__time_duration.sum --csv python tools/nvtx_stages.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RINR_NVTX", "1")

from paper_2306_16699_b200 import harness, synth, trace  # noqa: E402

assert trace.enabled()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
data = synth.gpu_store_bytes("c2", n, seed=7)
r = harness.bench(data, batch=256)
print(json.dumps({"images": r.images, "stage_seconds": r.stage_seconds, "images_per_s": r.images_per_s,
                  "digest": r.digest}))
