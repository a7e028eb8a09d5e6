RINR_NW=16 python -m pytest tests -m gpu -x -q --timeout 300 -k "parity or layout or edges or fuzz or digest" 2>&1 | tail -1
