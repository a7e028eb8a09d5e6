bash tools/ab_bench.sh c3
