bash tools/ab_bench.sh
