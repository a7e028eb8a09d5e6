#!/bin/bash
# c2 per-launch time with phases skipped (library built with RINR_EXTRA_NVCC_FLAGS=-DRINR_DEV_KNOBS;
# the skipped variants produce wrong images and are timing diagnostics only)
for s in ${SKIPS:-0 1 2 3}; do
  RINR_DEBUG_SKIP=$s python bench.py --no-cpu --no-e2e "$@" > gpurun_out/pb.json 2>gpurun_out/pb.err || tail -3 gpurun_out/pb.err
  python -c "import json,sys;d=json.load(open('gpurun_out/pb.json'));print('skip',$s,round(d['ms_per_step']*1e3,2),'us')"
done
