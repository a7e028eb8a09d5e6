#!/bin/bash
# A/B of two library builds (A: paper_2306_16699_b200/_lib, B: _lib_ab) on the
# decode benches, interleaved twice.  Usage: bash tools/ab_bench.sh [bench args...]
set -o pipefail
B=paper_2306_16699_b200/_lib_ab/librinr_b200.so
one() {
  local tag=$1; shift
  python bench.py --no-cpu --no-e2e --no-subs "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err || { tail -3 gpurun_out/ab.err; return 1; }
  python -c "import json,sys;d=json.load(open('gpurun_out/ab.json'));print(sys.argv[1],' '.join(sys.argv[2:]),round(d['value']),round(d['roofline']['frac'],4),round(d['ms_per_step']*1000,2),'us')" "$tag" "$@"
}
for rep in 1 2; do
  one A --config c2 "$@"
  RINR_LIB_PATH=$B one B --config c2 "$@"
  one A --config c2 --precision bf16 "$@"
  RINR_LIB_PATH=$B one B --config c2 --precision bf16 "$@"
  one A --config c1 "$@"
  RINR_LIB_PATH=$B one B --config c1 "$@"
done
