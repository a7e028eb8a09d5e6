#!/bin/bash
# development loop on the GPU box: decode parity tests, then the quick bench sweep
python -m pytest tests/test_gpu_parity.py tests/test_gpu_zeropoint.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q 2>&1 | tail -3
bash tools/quick_bench.sh "$@"
