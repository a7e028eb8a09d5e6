for f in umma_lat umma_multi umma_first; do echo "## tools/micro/$f"; timeout 120 ./tools/micro/$f; done > gpurun_out/umma.txt 2>&1; tail -3 gpurun_out/umma.txt
