#!/bin/bash
# A/B of two library builds (A: paper_2306_16699_b200/_lib, B: _lib_ab) on the
# decode benches, interleaved twice.
#   bash tools/ab_bench.sh            c2 fp32 / bf16 and c1
#   bash tools/ab_bench.sh c3         c3 fp32 / bf16
set -o pipefail
B=paper_2306_16699_b200/_lib_ab/librinr_b200.so
one() {
  local tag=$1; shift
  python bench.py --no-cpu --no-e2e --no-subs "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err || { tail -3 gpurun_out/ab.err; return 1; }
  python -c "import json,sys;d=json.load(open('gpurun_out/ab.json'));print(sys.argv[1],' '.join(sys.argv[2:]),round(d['value']),round(d['roofline']['frac'],4),round(d['ms_per_step']*1000,2),'us')" "$tag" "$@"
}
if [ "$1" = "c3" ]; then
  sets=("--config c3 --steps 20 --warmup 3 --precision fp32" "--config c3 --steps 20 --warmup 3 --precision bf16")
else
  sets=("--config c2" "--config c2 --precision bf16" "--config c1")
fi
for rep in 1 2; do
  for s in "${sets[@]}"; do
    one A $s
    RINR_LIB_PATH=$B one B $s
  done
done
