python -m pytest tests -m gpu -x -q -k "parity or layout or edges or digest or dropin or fitted or zeropoint or fuzz" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
RINR_LIB_PATH=paper_2306_16699_b200/_lib_ab/librinr_b200.so python tools/dev_timeline.py c2
bash tools/quick_bench.sh
