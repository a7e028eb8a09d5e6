#!/bin/bash
# Bounds-asserting build (-DRINR_CHECKED: RINR_DCHECK on shared-memory
# accesses, record reads, output stores and TMEM columns; device printf +
# trap on failure) into paper_2306_16699_b200/_lib_checked/, then (on a GPU
# box) the whole GPU suite against it.  compute-sanitizer is closed on the
# GPU pool; this is the substitute evidence (profiles/r02_checked_build.txt).
#   bash tools/checked_build.sh build   # here (cross-compiles)
#   bash tools/checked_build.sh test    # on the GPU box
set -e
case "$1" in
  build)
    RINR_LIB_DIR=paper_2306_16699_b200/_lib_checked RINR_EXTRA_NVCC_FLAGS=-DRINR_CHECKED \
      python -c "from paper_2306_16699_b200 import build as B; print(B.build(force=True))" ;;
  test)
    RINR_LIB_PATH=$PWD/paper_2306_16699_b200/_lib_checked/librinr_b200.so python -m pytest tests -m gpu -q -p no:cacheprovider ;;
esac
