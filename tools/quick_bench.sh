#!/bin/bash
# quick bench sweep used during development (prints value / roofline frac / ms per step)
set -o pipefail
run() {
  python bench.py --no-cpu --no-e2e "$@" > gpurun_out/b.json 2>gpurun_out/b.err || { tail -3 gpurun_out/b.err; return 1; }
  python -c "import json,sys;d=json.load(open('gpurun_out/b.json'));print(' '.join(sys.argv[1:]),round(d['value']),round(d['roofline']['frac'],3),round(d['ms_per_step'],4))" "$@"
}
run --config c2 && run --config c2 --precision bf16 && run --config c3 --steps 20 --warmup 3 --precision bf16 && run --config c3 --steps 20 --warmup 3 --precision fp32
