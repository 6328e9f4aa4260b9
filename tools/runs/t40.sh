#!/bin/bash
# folded scan: static-size fast pass (valid 16-column chunks only) + slow-path load/atomic overlap; 16 epilogue warps variant
OUT=gpurun_out/t40; mkdir -p $OUT
for v in Q R16; do
  cp variants/lib_$v.so paper_2605_16007_b200/librabitq.so
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "small_scan_identical or latency" > $OUT/pytest_$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_$v.log
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_$v.json 2> $OUT/cfg4_$v.err
done
cp variants/lib_Q.so paper_2605_16007_b200/librabitq.so
timeout 600 python bench.py --config 5 --shard 0/8 --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg5_Q.json 2> $OUT/cfg5_Q.err
