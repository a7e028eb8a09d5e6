#!/bin/bash
# Round evidence refresh (run on the GPU box via gpurun); outputs under gpurun_out/.
#   bash tools/profile_round.sh [c2|c3|all]
set -o pipefail
what=${1:-all}
o=gpurun_out
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; tail -1 $o/pytest_gpu.log
if [ "$what" != "c3" ]; then
  python bench.py > $o/bench_c2.json 2> $o/bench_c2.err || tail -5 $o/bench_c2.err
  python bench.py --precision bf16 --no-cpu --no-e2e > $o/bench_c2_bf16.json 2>> $o/bench_c2.err
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_c2.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $o/ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:decode_persist -s 10 -c 1 -o $o/full_c2 -f \
    python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $o/ncu_full_c2.log 2>&1
fi
if [ "$what" != "c2" ]; then
  python bench.py --config c3 --steps 20 --warmup 3 > $o/bench_c3.json 2> $o/bench_c3.err || tail -5 $o/bench_c3.err
  python bench.py --config c3 --steps 20 --warmup 3 --precision fp32 --no-cpu --no-e2e > $o/bench_c3_fp32.json 2>> $o/bench_c3.err
  ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 5 -c 1 -o $o/full_c3 -f \
    python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e --store-records 512 > $o/ncu_full_c3.log 2>&1
fi
for f in $o/bench_*.json; do echo "$f: $(python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value']), d['unit'], 'frac', round(d['roofline']['frac'],3), 'ms', round(d['ms_per_step'],5), 'e2e', (d.get('e2e') or {}).get('value'))")"; done
