python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
bash tools/ab_bench.sh c3
