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
  timeout 900 ncu --nvtx --nvtx-include "rabitq:search/" --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "launch_rc=$?" >> $OUT/ncu_launch.log
CMD2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-recall"
$CMD2 > $OUT/plain_full.log 2>&1 && \
  timeout 1200 ncu --nvtx --nvtx-include "rabitq:search/" --set full --clock-control none --import-source on -k regex:"scan_fold|scan_imma|scan_small|select_rerank|seed_near|quantize_kernel|probe_select|tgemm_kernel" -s 22 -c 11 -o $OUT/full $CMD2 > $OUT/ncu_full.log 2>&1
echo "full_rc=$?" >> $OUT/ncu_full.log
./tools/ubench/tmem_ld > $OUT/tmem_ld.txt 2>&1
timeout 600 python bench.py --config 5 --shard 0/8 --no-cpu-baseline > $OUT/cfg5.json 2> $OUT/cfg5.err
timeout 900 python bench.py --config 3 --nprobe-sweep 16,32,64,128 > $OUT/cfg3_sweep.json 2> $OUT/cfg3_sweep.err
timeout 600 python bench.py --config 2 > $OUT/cfg2.json 2> $OUT/cfg2.err
timeout 300 python bench.py --config 1 > $OUT/cfg1.json 2> $OUT/cfg1.err
