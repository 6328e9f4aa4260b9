#!/bin/bash
# ncu --set full of the folded scan (source-level stall samples), CFG4 at 4000 queries per batch as in gpu_evidence.sh
OUT=gpurun_out/t33; mkdir -p $OUT
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"scan_fold" -s 2 -c 1 -o $OUT/fold $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
