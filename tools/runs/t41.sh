#!/bin/bash
# folded scan, RABITQ_DIAG build of the committed kernel: cost of the slow path (FOLD_DIAG 1: flagged chunks
# dropped, 2: no exact row ip; results are wrong on purpose, only stage_ms.scan is read) and the CTA-0 timeline
OUT=gpurun_out/t41; mkdir -p $OUT
cp paper_2605_16007_b200/librabitq.so /tmp/lib_keep.so
cp variants/lib_D.so paper_2605_16007_b200/librabitq.so
for fd in 0 1 2; do
  RABITQ_FOLD_DIAG=$fd timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_fd$fd.json 2> $OUT/cfg4_fd$fd.err
done
RABITQ_FOLD_TIMELINE=$OUT/tl.bin timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_T.json 2> $OUT/cfg4_T.err
python tools/fold_timeline.py $OUT/tl.bin > $OUT/timeline.txt 2>&1
cp /tmp/lib_keep.so paper_2605_16007_b200/librabitq.so
