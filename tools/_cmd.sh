set -x
python -m pytest tests -m gpu -x -q -k "parity or layout or edges or digest or dropin" 2>&1 | tail -3
bash tools/ab_bench.sh
