#!/bin/bash
# timeline of the folded scan's CTA 0 (RABITQ_DIAG build), CFG4
OUT=gpurun_out/t38; mkdir -p $OUT
cp paper_2605_16007_b200/librabitq.so /tmp/lib_keep.so
cp variants/lib_T.so paper_2605_16007_b200/librabitq.so
RABITQ_FOLD_TIMELINE=$OUT/tl.bin timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_T.json 2> $OUT/cfg4_T.err
python tools/fold_timeline.py $OUT/tl.bin > $OUT/timeline.txt 2>&1
cp /tmp/lib_keep.so paper_2605_16007_b200/librabitq.so
