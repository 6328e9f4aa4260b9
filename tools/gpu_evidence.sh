#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the ncu launch list of
# the bench command and one `ncu --set full` capture of the top kernels.
# Usage (on the box): bash tools/gpu_evidence.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-recall"
$CMD > $OUT/plain_launch.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall --nq 4000"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"scan_imma|select_rerank" -s 6 -c 2 -o $OUT/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
