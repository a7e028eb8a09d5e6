RINR_LIB_PATH=paper_2306_16699_b200/_lib_ab/librinr_b200.so python tools/dev_tc_timeline.py fp32 2>&1 | tail -7
RINR_LIB_PATH=paper_2306_16699_b200/_lib_ab/librinr_b200.so python tools/dev_tc_timeline.py bf16 2>&1 | tail -7
