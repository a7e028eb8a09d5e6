timeout 1200 bash tools/checked_build.sh test > gpurun_out/checked.log 2>&1; tail -2 gpurun_out/checked.log; grep -c "RINR_DCHECK" gpurun_out/checked.log || true
python -m pytest tests -m gpu -x -q --timeout 300 -k "parity or layout or edges" 2>&1 | tail -1
