#!/bin/bash
# folded scan: slot released as soon as the last TMEM read has landed
OUT=gpurun_out/t39; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_scan_identical or latency" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_P.json 2> $OUT/cfg4_P.err
timeout 600 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg5_P.json 2> $OUT/cfg5_P.err
cp paper_2605_16007_b200/librabitq.so /tmp/lib_keep.so
cp variants/lib_TP.so paper_2605_16007_b200/librabitq.so
RABITQ_FOLD_TIMELINE=$OUT/tl.bin timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_T.json 2> $OUT/cfg4_T.err
python tools/fold_timeline.py $OUT/tl.bin > $OUT/timeline.txt 2>&1
cp /tmp/lib_keep.so paper_2605_16007_b200/librabitq.so
