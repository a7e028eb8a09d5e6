#!/bin/bash
# Round evidence refresh on the GPU box (gpurun); outputs under gpurun_out/r02/.
#   bash tools/profile_round.sh
# 1. the GPU suite; 2. the driver's bench commands (ours + reference arm);
# 3. c4 / c5 training benches; 4. ncu launch list of the default bench;
# 5. one `ncu --set full` capture per decode kernel of the metric (c2 fp32,
#    c1 fp32, c3 fp32, c3 bf16), each after the same command ran clean.
set -o pipefail
o=gpurun_out/r02
mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; tail -1 $o/pytest_gpu.log
python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err || tail -5 $o/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_ref.json 2> $o/bench_ref.err || tail -5 $o/bench_ref.err
python bench.py --config c4 --steps 20 --warmup 5 > $o/bench_c4.json 2> $o/bench_c4.err || tail -5 $o/bench_c4.err
python bench.py --config c5 --steps 20 --warmup 5 > $o/bench_c5.json 2> $o/bench_c5.err || tail -5 $o/bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $o/launches_bench.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $o/ncu_launch.log 2>&1
# units per launch for the per-block instruction counts: 16-pixel blocks
for spec in "c2 fp32 decode_persist 65536" "c1 fp32 decode_persist 16384" "c3 fp32 decode_tc 802816" "c3 bf16 decode_tc 802816"; do
  set -- $spec
  cmd="python tools/ncu_decode.py --config $1 --precision $2 --launches 6 --records 65536"
  [ "$1" = "c3" ] && cmd="python tools/ncu_decode.py --config $1 --precision $2 --launches 4 --records 16384"
  $cmd > $o/plain_$1_$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 -o $o/full_$1_$2 -f $cmd \
    > $o/ncu_full_$1_$2.log 2>&1
  tail -1 $o/ncu_full_$1_$2.log
  # summaries here (the .ncu-rep files are too large to bring back)
  python tools/ncu_report.py $o/full_$1_$2.ncu-rep "$3 ($1, $2): bench workload, ncu --set full" $4 $1_$2 \
    > $o/ncu_$1_$2.txt 2>&1
  python tools/ncu_hot.py $o/full_$1_$2.ncu-rep 30 > $o/ncu_hot_$1_$2.txt 2>&1
  rm -f $o/full_$1_$2.ncu-rep
done
cp profiles/ncu_summary.json $o/ncu_summary.json
ls $o
