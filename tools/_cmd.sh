python -m pytest tests -m gpu -x -q --timeout 300 -k "parity or layout or wide or accuracy or fitted or fuzz or epilogue or augment or edges" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
bash tools/ab_bench.sh c3
