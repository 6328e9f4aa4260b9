#!/bin/bash
# A-stage sensitivity (FX_SA=3) and the full GPU test suite with the early-release folded scan
OUT=gpurun_out/t37; mkdir -p $OUT
cp variants/lib_N.so paper_2605_16007_b200/librabitq.so
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-recall > $OUT/cfg4_N.json 2> $OUT/cfg4_N.err
cp variants/lib_K.so paper_2605_16007_b200/librabitq.so
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
